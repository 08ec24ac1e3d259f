/*
 * subsurf_oracle.c -- CPU restatement of the reference SUBSURF hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see subsurf_oracle.h): the parity checker for the
 * CUDA path, never shipped or measured as the product.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).  Every
 * expression keeps the reference's evaluation order; x86-64 SSE2 without FMA
 * contraction makes the results bit-identical to the reference's -O3 build.
 * File:line citations are into /root/reference/proj/src.
 */
#include "subsurf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define IMAX(g) ((g)->n1 + 2)
#define JMAX(g) ((g)->n2 + 2)
#define KMAX(g) ((g)->n3 + 2)
#define LMAX(g) ((g)->n4 + 2)

static inline size_t off4(const or_grid* g, int i, int j, int k, int l) {
    return (((size_t)l * KMAX(g) + k) * JMAX(g) + j) * IMAX(g) + i;
}

static inline double spacing(const or_grid* g, int axis) {
    return axis == 0 ? g->h1 : axis == 1 ? g->h2 : axis == 2 ? g->h3 : g->h4;
}

static inline ptrdiff_t stride(const or_grid* g, int axis) {
    switch (axis) {
        case 0: return 1;
        case 1: return IMAX(g);
        case 2: return (ptrdiff_t)IMAX(g) * JMAX(g);
        default: return (ptrdiff_t)IMAX(g) * JMAX(g) * KMAX(g);
    }
}

size_t or_padded_size(const or_grid* g) {
    return (size_t)IMAX(g) * JMAX(g) * KMAX(g) * LMAX(g);
}

/* grid.cpp:126-136 */
void or_apply_dirichlet(const or_grid* g, double* f, double value) {
    for (int l = 0; l <= g->n4 + 1; ++l)
        for (int k = 0; k <= g->n3 + 1; ++k)
            for (int j = 0; j <= g->n2 + 1; ++j)
                for (int i = 0; i <= g->n1 + 1; ++i) {
                    int ghost = i == 0 || i == g->n1 + 1 || j == 0 || j == g->n2 + 1 || k == 0 ||
                                k == g->n3 + 1 || l == 0 || l == g->n4 + 1;
                    if (ghost) f[off4(g, i, j, k, l)] = value;
                }
}

/* grid.cpp:138-156: one axis at a time over the padded box, so later axes
 * carry mirrored values into edges and corners. */
void or_apply_mirror_ghosts(const or_grid* g, double* f) {
    const int hi[4] = {g->n1 + 1, g->n2 + 1, g->n3 + 1, g->n4 + 1};
    for (int axis = 0; axis < 4; ++axis) {
        const ptrdiff_t st = stride(g, axis);
        for (int l = 0; l <= g->n4 + 1; ++l)
            for (int k = 0; k <= g->n3 + 1; ++k)
                for (int j = 0; j <= g->n2 + 1; ++j)
                    for (int i = 0; i <= g->n1 + 1; ++i) {
                        const int c[4] = {i, j, k, l};
                        if (c[axis] != 0 && c[axis] != hi[axis]) continue;
                        double* p = f + off4(g, i, j, k, l);
                        *p = c[axis] == 0 ? p[st] : p[-st];
                    }
    }
}

/* grid.cpp:158-171 */
void or_interior_minmax(const or_grid* g, const double* f, double* lo, double* hi) {
    double a = INFINITY, b = -INFINITY;
    for (int l = 1; l <= g->n4; ++l)
        for (int k = 1; k <= g->n3; ++k)
            for (int j = 1; j <= g->n2; ++j)
                for (int i = 1; i <= g->n1; ++i) {
                    const double v = f[off4(g, i, j, k, l)];
                    a = (v < a) ? v : a; /* std::min(lo, v) */
                    b = (b < v) ? v : b; /* std::max(hi, v) */
                }
    *lo = a;
    *hi = b;
}

/* edge.cpp:16-22 : 0.25 * (((p0 + pa) + pb) + pab) */
static inline double corner_average(const double* p, ptrdiff_t sa, ptrdiff_t sb) {
    return 0.25 * (p[0] + p[sa] + p[sb] + p[sa + sb]);
}

/* edge.cpp:33-48 */
void or_face_gradient(const or_grid* g, const double* u, int i, int j, int k, int l, int face,
                      double grad[4]) {
    const int axis = face >> 1;
    const int sign = (face & 1) ? 1 : -1;
    const double* p = u + off4(g, i, j, k, l);
    const ptrdiff_t sn = sign * stride(g, axis);
    grad[axis] = (double)sign * (p[sn] - p[0]) / spacing(g, axis);
    for (int t = 0; t < 4; ++t) {
        if (t == axis) continue;
        const double plus = corner_average(p, sn, stride(g, t));
        const double minus = corner_average(p, sn, -stride(g, t));
        grad[t] = (plus - minus) / spacing(g, t);
    }
}

/* edge.cpp:50-57 */
void or_face_gradient_sq(const or_grid* g, const double* u, int i, int j, int k, int l,
                         double out[8]) {
    for (int f = 0; f < 8; ++f) {
        double gr[4];
        or_face_gradient(g, u, i, j, k, l, f, gr);
        out[f] = gr[0] * gr[0] + gr[1] * gr[1] + gr[2] * gr[2] + gr[3] * gr[3];
    }
}

/* edge.cpp:9-14 */
static int edge_params_ok(double K, double delta, double vartheta) {
    if (K < 0.0) return 0;
    if (delta < 0.0 || delta > 1.0) return 0;
    if (vartheta < 0.0 || vartheta > 1.0) return 0;
    return 1;
}

/* edge.cpp:73-99 ; perona_malik edge.hpp:21 */
int or_face_coefficients(const or_grid* g, const double* I0s, const double* ITs, double K,
                         double delta, double vartheta, double* G) {
    if (!edge_params_ok(K, delta, vartheta)) return OR_ERR_VALIDATION;
    const size_t P = or_padded_size(g);
    for (size_t n = 0; n < 8 * P; ++n) G[n] = 1.0; /* FaceCoefficientField fill */
    for (int l = 1; l <= g->n4; ++l)
        for (int k = 1; k <= g->n3; ++k)
            for (int j = 1; j <= g->n2; ++j)
                for (int i = 1; i <= g->n1; ++i) {
                    double* out = G + 8 * off4(g, i, j, k, l);
                    for (int f = 0; f < 8; ++f) {
                        double gi[4], gt[4];
                        or_face_gradient(g, I0s, i, j, k, l, f, gi);
                        or_face_gradient(g, ITs, i, j, k, l, f, gt);
                        const double ni =
                            sqrt(gi[0] * gi[0] + gi[1] * gi[1] + gi[2] * gi[2] + gi[3] * gi[3]);
                        const double nt =
                            sqrt(gt[0] * gt[0] + gt[1] * gt[1] + gt[2] * gt[2] + gt[3] * gt[3]);
                        const double s = delta * ni + vartheta * nt;
                        out[f] = 1.0 / (1.0 + K * s * s);
                    }
                }
    return OR_OK;
}

/* solver.cpp:13-21 (the subset assemble/sor check) */
static int solver_params_ok(double tau, double eps, double omega, double tol, int max_iter) {
    if (tau < 0.0) return 0;
    if (!(eps > 0.0)) return 0;
    if (!(omega > 0.0) || !(omega < 2.0)) return 0;
    if (!(tol > 0.0)) return 0;
    if (max_iter < 1) return 0;
    return 1;
}

/* solver.cpp:23-77 */
int or_assemble_step(const or_grid* g, const double* u_prev, const double* G, double tau,
                     double eps, double* off, double* diag, double* abar) {
    if (!solver_params_ok(tau, eps, 1.0, 1.0, 1)) return OR_ERR_VALIDATION;
    const size_t P = or_padded_size(g);
    memset(off, 0, 8 * P * sizeof(double));
    memset(diag, 0, P * sizeof(double));
    memset(abar, 0, P * sizeof(double));
    double t_h2[4];
    for (int a = 0; a < 4; ++a) t_h2[a] = tau / (spacing(g, a) * spacing(g, a));
    int bad = 0;
    for (int l = 1; l <= g->n4; ++l)
        for (int k = 1; k <= g->n3; ++k)
            for (int j = 1; j <= g->n2; ++j)
                for (int i = 1; i <= g->n1; ++i) {
                    double g2[8];
                    or_face_gradient_sq(g, u_prev, i, j, k, l, g2);
                    double a_face[8];
                    double a_sq_sum = 0.0;
                    for (int f = 0; f < 8; ++f) {
                        const double a_sq = eps + g2[f];
                        a_face[f] = sqrt(a_sq);
                        a_sq_sum += a_sq;
                    }
                    const double ab = sqrt(eps + 0.125 * a_sq_sum);
                    const size_t at = off4(g, i, j, k, l);
                    const double* gp = G ? G + 8 * at : NULL;
                    double sum = 0.0;
                    for (int f = 0; f < 8; ++f) {
                        const double gf = gp ? gp[f] : 1.0;
                        const double o = (double)(float)(-(t_h2[f >> 1] * ab * gf / a_face[f]));
                        off[8 * at + f] = o;
                        sum += o;
                    }
                    diag[at] = 1.0 - sum;
                    abar[at] = ab;
                    if (!isfinite(diag[at])) bad = 1;
                }
    return bad ? OR_ERR_NONFINITE : OR_OK;
}

/* solver.cpp:79-116 */
int or_assemble_heat_step(const or_grid* g, double dt, double* off, double* diag, double* abar) {
    if (!(dt > 0.0)) return OR_ERR_VALIDATION;
    const size_t P = or_padded_size(g);
    memset(off, 0, 8 * P * sizeof(double));
    memset(diag, 0, P * sizeof(double));
    memset(abar, 0, P * sizeof(double));
    double d_h2[4];
    for (int a = 0; a < 4; ++a) d_h2[a] = dt / (spacing(g, a) * spacing(g, a));
    const int hi[4] = {g->n1, g->n2, g->n3, g->n4};
    for (int l = 1; l <= g->n4; ++l)
        for (int k = 1; k <= g->n3; ++k)
            for (int j = 1; j <= g->n2; ++j)
                for (int i = 1; i <= g->n1; ++i) {
                    const size_t at = off4(g, i, j, k, l);
                    const int c[4] = {i, j, k, l};
                    double sum = 0.0;
                    for (int f = 0; f < 8; ++f) {
                        const int axis = f >> 1;
                        const int nb = c[axis] + ((f & 1) ? 1 : -1);
                        if (nb < 1 || nb > hi[axis]) {
                            off[8 * at + f] = 0.0;
                        } else {
                            off[8 * at + f] = (double)(float)(-d_h2[axis]);
                            sum += off[8 * at + f];
                        }
                    }
                    diag[at] = 1.0 - sum;
                    abar[at] = 1.0;
                }
    return OR_OK;
}

/* One colour half-sweep, solver.cpp:267-317.  Returns nothing; per-slice
 * residual sums go to slice_sq when non-NULL (black phase, :309-315). */
static void sweep(const or_grid* g, const float* cf, const double* rhs, double* u, double omega,
                  int color, double* slice_sq) {
    const ptrdiff_t sj = IMAX(g), sk = sj * JMAX(g), sl = sk * KMAX(g);
    const double keep = 1.0 - omega;
    for (int l = 1; l <= g->n4; ++l) {
        double res_sum = 0.0;
        for (int k = 1; k <= g->n3; ++k)
            for (int j = 1; j <= g->n2; ++j) {
                const size_t row = off4(g, 0, j, k, l);
                double* uu = u + row;
                const double* rr = rhs + row;
                const int i0 = (((1 + j + k + l + color) & 1) == 0) ? 1 : 2;
                for (int i = i0; i <= g->n1; i += 2) {
                    const float* c = cf + 8 * (row + i);
                    const double c0 = c[0], c1 = c[1], c2 = c[2], c3 = c[3];
                    const double c4 = c[4], c5 = c[5], c6 = c[6], c7 = c[7];
                    const double dg = 1.0 - (c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7);
                    double acc = rr[i];
                    acc -= c0 * uu[i - 1];
                    acc -= c1 * uu[i + 1];
                    acc -= c2 * uu[i - sj];
                    acc -= c3 * uu[i + sj];
                    acc -= c4 * uu[i - sk];
                    acc -= c5 * uu[i + sk];
                    acc -= c6 * uu[i - sl];
                    acc -= c7 * uu[i + sl];
                    const double ubar = acc / dg;
                    const double unew = omega * ubar + keep * uu[i];
                    uu[i] = unew;
                    const double res = dg * (unew - ubar);
                    res_sum += res * res;
                }
            }
        if (slice_sq) slice_sq[l] = res_sum;
    }
}

/* solver.cpp:319-361 */
static void red_residuals(const or_grid* g, const float* cf, const double* rhs, const double* u,
                          const double* black_sq, double* slice_res) {
    const ptrdiff_t sj = IMAX(g), sk = sj * JMAX(g), sl = sk * KMAX(g);
    for (int l = 1; l <= g->n4; ++l) {
        double sum = 0.0;
        for (int k = 1; k <= g->n3; ++k)
            for (int j = 1; j <= g->n2; ++j) {
                const size_t row = off4(g, 0, j, k, l);
                const double* uu = u + row;
                const double* rr = rhs + row;
                const int i0 = (((1 + j + k + l) & 1) == 0) ? 1 : 2;
                for (int i = i0; i <= g->n1; i += 2) {
                    const float* c = cf + 8 * (row + i);
                    const double c0 = c[0], c1 = c[1], c2 = c[2], c3 = c[3];
                    const double c4 = c[4], c5 = c[5], c6 = c[6], c7 = c[7];
                    const double dg = 1.0 - (c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7);
                    double res = dg * uu[i] - rr[i];
                    res += c0 * uu[i - 1];
                    res += c1 * uu[i + 1];
                    res += c2 * uu[i - sj];
                    res += c3 * uu[i + sj];
                    res += c4 * uu[i - sk];
                    res += c5 * uu[i + sk];
                    res += c6 * uu[i - sl];
                    res += c7 * uu[i + sl];
                    sum += res * res;
                }
            }
        slice_res[l] = black_sq[l] + sum;
    }
}

/* solver.cpp:379-397 via SorRun (:124-375), single worker. */
int or_redblack_sor(const or_grid* g, const double* off, const double* rhs, double* u,
                    double omega, double tol, int max_iter, int* iters, double* res) {
    if (!solver_params_ok(1.0, 1.0, omega, tol, max_iter)) return OR_ERR_VALIDATION;
    const size_t P = or_padded_size(g);
    /* pack_coefficients (solver.cpp:233-249): float copies of the rows */
    float* cf = (float*)malloc(8 * P * sizeof(float));
    double* black_sq = (double*)calloc((size_t)g->n4 + 2, sizeof(double));
    double* slice_res = (double*)calloc((size_t)g->n4 + 2, sizeof(double));
    if (!cf || !black_sq || !slice_res) {
        free(cf);
        free(black_sq);
        free(slice_res);
        return OR_ERR_VALIDATION;
    }
    for (size_t n = 0; n < 8 * P; ++n) cf[n] = (float)off[n];
    int it = 0, done = 0;
    double r = 0.0;
    for (;;) {
        sweep(g, cf, rhs, u, omega, 0, NULL);
        sweep(g, cf, rhs, u, omega, 1, black_sq);
        red_residuals(g, cf, rhs, u, black_sq, slice_res);
        double total = 0.0;
        for (int l = 1; l <= g->n4; ++l) total += slice_res[l];
        r = sqrt(total);
        ++it;
        if (r <= tol) {
            done = 1;
            break;
        }
        if (it >= max_iter) break;
    }
    free(cf);
    free(black_sq);
    free(slice_res);
    *iters = it;
    *res = r;
    return done ? OR_OK : OR_ERR_NOCONVERGE;
}

/* preprocess.cpp:25-51 */
int or_heat_smooth(const or_grid* g, const double* image, double sigma, int steps, double omega,
                   double tol, int max_iter, double* out) {
    if (sigma < 0.0 || steps < 1 || !(tol > 0.0) || max_iter < 1 || !(omega > 0.0) ||
        !(omega < 2.0))
        return OR_ERR_VALIDATION;
    const size_t P = or_padded_size(g);
    memcpy(out, image, P * sizeof(double));
    if (sigma == 0.0) {
        or_apply_mirror_ghosts(g, out);
        return OR_OK;
    }
    const double dt = 0.5 * sigma * sigma / steps;
    double* off = (double*)malloc(8 * P * sizeof(double));
    double* dg = (double*)malloc(P * sizeof(double));
    double* ab = (double*)malloc(P * sizeof(double));
    double* rhs = (double*)malloc(P * sizeof(double));
    int st = or_assemble_heat_step(g, dt, off, dg, ab);
    for (int s = 0; s < steps && st == OR_OK; ++s) {
        int it;
        double r;
        memcpy(rhs, out, P * sizeof(double)); /* redblack_sor(coeff, u, u, ...) */
        st = or_redblack_sor(g, off, rhs, out, omega, tol, max_iter, &it, &r);
    }
    free(off);
    free(dg);
    free(ab);
    free(rhs);
    if (st != OR_OK) return st;
    or_apply_mirror_ghosts(g, out);
    return OR_OK;
}

/* io.cpp:128-140 */
int or_validate_centers(const or_grid* g, const or_center* c, int n) {
    for (int m = 0; m < n; ++m) {
        if (c[m].frame < 0 || c[m].frame >= g->n4) return OR_ERR_VALIDATION;
        if (!(c[m].radius > 0.0)) return OR_ERR_VALIDATION;
        if (c[m].x < 0.0 || c[m].x > g->n1 - 1 || c[m].y < 0.0 || c[m].y > g->n2 - 1 ||
            c[m].z < 0.0 || c[m].z > g->n3 - 1)
            return OR_ERR_VALIDATION;
    }
    return OR_OK;
}

typedef struct {
    int i0, i1, j0, j1, k0, k1;
} ball_box;

/* seedinit.cpp:22-31 (same bounds as preprocess.cpp:63-68) */
static ball_box ball_bounds(const or_center* c, double r, const or_grid* g) {
    ball_box b;
    int t;
    t = (int)ceil(c->x - r) + 1;
    b.i0 = t > 1 ? t : 1;
    t = (int)floor(c->x + r) + 1;
    b.i1 = t < g->n1 ? t : g->n1;
    t = (int)ceil(c->y - r) + 1;
    b.j0 = t > 1 ? t : 1;
    t = (int)floor(c->y + r) + 1;
    b.j1 = t < g->n2 ? t : g->n2;
    t = (int)ceil(c->z - r) + 1;
    b.k0 = t > 1 ? t : 1;
    t = (int)floor(c->z + r) + 1;
    b.k1 = t < g->n3 ? t : g->n3;
    return b;
}

/* seedinit.cpp:33-40 / preprocess.cpp:70-75 */
static inline double dist_sq(const or_center* c, int i, int j, int k) {
    const double dx = (i - 1) - c->x;
    const double dy = (j - 1) - c->y;
    const double dz = (k - 1) - c->z;
    return dx * dx + dy * dy + dz * dz;
}

/* preprocess.cpp:53-102 */
int or_local_threshold(const or_grid* g, const double* image, const or_center* c, int n,
                       double lambda, double background, double* out) {
    if (lambda < 0.0 || lambda > 1.0) return OR_ERR_VALIDATION;
    if (or_validate_centers(g, c, n) != OR_OK) return OR_ERR_VALIDATION;
    const size_t P = or_padded_size(g);
    for (size_t q = 0; q < P; ++q) out[q] = background;
    for (int m = 0; m < n; ++m) {
        const int l = c[m].frame + 1;
        const double r_sq = c[m].radius * c[m].radius;
        const ball_box b = ball_bounds(&c[m], c[m].radius, g);
        double alpha = INFINITY, beta = -INFINITY;
        for (int k = b.k0; k <= b.k1; ++k)
            for (int j = b.j0; j <= b.j1; ++j)
                for (int i = b.i0; i <= b.i1; ++i) {
                    if (!(dist_sq(&c[m], i, j, k) <= r_sq)) continue;
                    const double v = image[off4(g, i, j, k, l)];
                    alpha = (v < alpha) ? v : alpha;
                    beta = (beta < v) ? v : beta;
                }
        if (alpha > beta) return OR_ERR_VALIDATION; /* ball covers no doxels */
        const double th = lambda * alpha + (1.0 - lambda) * beta;
        for (int k = b.k0; k <= b.k1; ++k)
            for (int j = b.j0; j <= b.j1; ++j)
                for (int i = b.i0; i <= b.i1; ++i) {
                    if (!(dist_sq(&c[m], i, j, k) <= r_sq)) continue;
                    const size_t at = off4(g, i, j, k, l);
                    out[at] = image[at] >= th ? beta : alpha;
                }
    }
    return OR_OK;
}

/* seedinit.cpp:42-66 */
int or_build_initial(const or_grid* g, const or_center* c, int n, double v, double R,
                     int profile, double* u) {
    if (!(v > 0.0) || !(R > 0.0)) return OR_ERR_VALIDATION;
    if (or_validate_centers(g, c, n) != OR_OK) return OR_ERR_VALIDATION;
    memset(u, 0, or_padded_size(g) * sizeof(double));
    const double floor_value = 1.0 / (R + v);
    for (int m = 0; m < n; ++m) {
        const int l = c[m].frame + 1;
        const ball_box b = ball_bounds(&c[m], R, g);
        for (int k = b.k0; k <= b.k1; ++k)
            for (int j = b.j0; j <= b.j1; ++j)
                for (int i = b.i0; i <= b.i1; ++i) {
                    const double d = sqrt(dist_sq(&c[m], i, j, k));
                    if (d > R) continue;
                    const double value = profile == 0 ? 1.0 / (d + v) - floor_value : 1.0 - d / R;
                    double* cell = u + off4(g, i, j, k, l);
                    *cell = (*cell < value) ? value : *cell; /* std::max */
                }
    }
    return OR_OK;
}

/* seedinit.cpp:68-99 */
int or_local_rescale(const or_grid* g, double* u, const or_center* c, int n, double radius) {
    if (or_validate_centers(g, c, n) != OR_OK) return OR_ERR_VALIDATION;
    for (int m = 0; m < n; ++m) {
        const double r = isnan(radius) ? c[m].radius : radius; /* NaN = std::nullopt (value_or) */
        const int l = c[m].frame + 1;
        const ball_box b = ball_bounds(&c[m], r, g);
        const double r_sq = r * r;
        double lo = INFINITY, hi = -INFINITY;
        for (int k = b.k0; k <= b.k1; ++k)
            for (int j = b.j0; j <= b.j1; ++j)
                for (int i = b.i0; i <= b.i1; ++i) {
                    if (dist_sq(&c[m], i, j, k) > r_sq) continue;
                    const double v = u[off4(g, i, j, k, l)];
                    lo = (v < lo) ? v : lo;
                    hi = (hi < v) ? v : hi;
                }
        if (!(hi > lo)) continue;
        const double scale = 1.0 / (hi - lo);
        for (int k = b.k0; k <= b.k1; ++k)
            for (int j = b.j0; j <= b.j1; ++j)
                for (int i = b.i0; i <= b.i1; ++i) {
                    if (dist_sq(&c[m], i, j, k) > r_sq) continue;
                    double* p = u + off4(g, i, j, k, l);
                    *p = (*p - lo) * scale;
                }
    }
    return OR_OK;
}

/* tracking.cpp:35-52 */
void or_extract_mask(const or_grid* g, const double* u, double level, unsigned char* mask) {
    size_t q = 0;
    for (int l = 1; l <= g->n4; ++l)
        for (int k = 1; k <= g->n3; ++k)
            for (int j = 1; j <= g->n2; ++j)
                for (int i = 1; i <= g->n1; ++i) mask[q++] = u[off4(g, i, j, k, l)] >= level;
}

static double interior_norm2(const or_grid* g, const double* u) {
    double s = 0.0;
    for (int l = 1; l <= g->n4; ++l)
        for (int k = 1; k <= g->n3; ++k)
            for (int j = 1; j <= g->n2; ++j)
                for (int i = 1; i <= g->n1; ++i) {
                    const double v = u[off4(g, i, j, k, l)];
                    s += v * v;
                }
    return sqrt(s);
}

/* solver.cpp:405-441 */
int or_segment(const or_grid* g, const double* image, const or_center* c, int n,
               const or_seg_params* p, const double* u0, double* u_out, or_step_diag* diags) {
    if (!solver_params_ok(p->tau, p->epsilon, p->omega, p->sor_tol, p->sor_max_iter) ||
        p->n_steps < 1)
        return OR_ERR_VALIDATION;
    if (or_validate_centers(g, c, n) != OR_OK) return OR_ERR_VALIDATION;
    const size_t P = or_padded_size(g);
    double* th = (double*)malloc(P * sizeof(double));
    double* I0s = (double*)malloc(P * sizeof(double));
    double* ITs = (double*)malloc(P * sizeof(double));
    double* G = (double*)malloc(8 * P * sizeof(double));
    double* off = (double*)malloc(8 * P * sizeof(double));
    double* dg = (double*)malloc(P * sizeof(double));
    double* ab = (double*)malloc(P * sizeof(double));
    double* rhs = (double*)malloc(P * sizeof(double));
    int st = OR_OK;
    const double rr = p->rescale_radius;

    if (u0) {
        memcpy(u_out, u0, P * sizeof(double));
    } else {
        st = or_build_initial(g, c, n, p->init_v, p->init_R, p->init_profile, u_out);
    }
    if (st == OR_OK) st = or_local_rescale(g, u_out, c, n, rr);
    if (st == OR_OK) st = or_local_threshold(g, image, c, n, p->lambda, p->background, th);
    if (st == OR_OK)
        st = or_heat_smooth(g, image, p->sigma, p->smooth_steps, p->smooth_omega, p->smooth_tol,
                            p->smooth_max_iter, I0s);
    if (st == OR_OK)
        st = or_heat_smooth(g, th, p->sigma, p->smooth_steps, p->smooth_omega, p->smooth_tol,
                            p->smooth_max_iter, ITs);
    if (st == OR_OK) st = or_face_coefficients(g, I0s, ITs, p->K, p->delta, p->vartheta, G);
    if (st == OR_OK) or_apply_dirichlet(g, u_out, 0.0);
    for (int step = 1; step <= p->n_steps && st == OR_OK; ++step) {
        st = or_assemble_step(g, u_out, G, p->tau, p->epsilon, off, dg, ab);
        if (st != OR_OK) break;
        const double tol = p->sor_rel_tol > 0.0 ? p->sor_rel_tol * interior_norm2(g, u_out)
                                                : p->sor_tol;
        memcpy(rhs, u_out, P * sizeof(double));
        int it = 0;
        double r = 0.0;
        st = or_redblack_sor(g, off, rhs, u_out, p->omega, tol, p->sor_max_iter, &it, &r);
        if (st != OR_OK) break;
        if (p->rescale_each_step) st = or_local_rescale(g, u_out, c, n, rr);
        if (diags) {
            diags[step - 1].iterations = it;
            diags[step - 1].residual = r;
            diags[step - 1].tol = tol;
            or_interior_minmax(g, u_out, &diags[step - 1].umin, &diags[step - 1].umax);
        }
    }
    free(th);
    free(I0s);
    free(ITs);
    free(G);
    free(off);
    free(dg);
    free(ab);
    free(rhs);
    return st;
}

/* eoc.cpp:19-37 (exact_u, centre coordinates) */
static inline double exact_u(double x0, double x1, double x2, double x3, double t) {
    return (x0 * x0 + x1 * x1 + x2 * x2 + x3 * x3 - 1.0) / 6.0 + t;
}
static inline double ccoord(int v, double dmin, double h) { return dmin + (v - 0.5) * h; }

/* eoc.cpp:55-79 */
static void eoc_fill_ghosts(const or_grid* g, double* u, double dmin, double h, double t) {
    const int n = g->n1;
    for (int l = 0; l <= g->n4 + 1; ++l) {
        const double xl = ccoord(l, dmin, h);
        const int lg = l == 0 || l == g->n4 + 1;
        for (int k = 0; k <= g->n3 + 1; ++k) {
            const double xk = ccoord(k, dmin, h);
            const int klg = lg || k == 0 || k == g->n3 + 1;
            for (int j = 0; j <= g->n2 + 1; ++j) {
                const double xj = ccoord(j, dmin, h);
                if (klg || j == 0 || j == g->n2 + 1) {
                    for (int i = 0; i <= n + 1; ++i)
                        u[off4(g, i, j, k, l)] = exact_u(ccoord(i, dmin, h), xj, xk, xl, t);
                } else {
                    u[off4(g, 0, j, k, l)] = exact_u(ccoord(0, dmin, h), xj, xk, xl, t);
                    u[off4(g, n + 1, j, k, l)] = exact_u(ccoord(n + 1, dmin, h), xj, xk, xl, t);
                }
            }
        }
    }
}

/* eoc.cpp:83-137 (EocConfig defaults eoc.hpp:16-28) */
int or_eoc_row(int n, double omega, double sor_tol, int max_iter, double* err) {
    static const int sched[5][2] = {{10, 1}, {20, 4}, {40, 16}, {80, 64}, {160, 256}};
    int steps = 0;
    for (int s = 0; s < 5; ++s)
        if (sched[s][0] == n) steps = sched[s][1];
    if (!steps) return OR_ERR_VALIDATION;
    const double dmin = -1.25, dmax = 1.25, T = 0.0625;
    const double h = (dmax - dmin) / n;
    const double tau = T / steps;
    const or_grid g = {n, n, n, n, h, h, h, h};
    const size_t P = or_padded_size(&g);
    double* u = (double*)malloc(P * sizeof(double));
    double* off = (double*)malloc(8 * P * sizeof(double));
    double* dg = (double*)malloc(P * sizeof(double));
    double* ab = (double*)malloc(P * sizeof(double));
    double* rhs = (double*)malloc(P * sizeof(double));
    for (int l = 0; l <= n + 1; ++l)
        for (int k = 0; k <= n + 1; ++k)
            for (int j = 0; j <= n + 1; ++j)
                for (int i = 0; i <= n + 1; ++i)
                    u[off4(&g, i, j, k, l)] = exact_u(ccoord(i, dmin, h), ccoord(j, dmin, h),
                                                      ccoord(k, dmin, h), ccoord(l, dmin, h), 0.0);
    const double cell = h * h * h * h;
    double err_sq = 0.0;
    int st = OR_OK;
    for (int step = 1; step <= steps && st == OR_OK; ++step) {
        const double t_n = step * tau;
        st = or_assemble_step(&g, u, NULL, tau, h * h, off, dg, ab);
        if (st != OR_OK) break;
        eoc_fill_ghosts(&g, u, dmin, h, t_n);
        memcpy(rhs, u, P * sizeof(double));
        int it;
        double r;
        st = or_redblack_sor(&g, off, rhs, u, omega, sor_tol, max_iter, &it, &r);
        if (st != OR_OK) break;
        double step_sum = 0.0;
        for (int l = 1; l <= n; ++l) {
            const double xl = ccoord(l, dmin, h);
            double sum = 0.0;
            for (int k = 1; k <= n; ++k) {
                const double xk = ccoord(k, dmin, h);
                for (int j = 1; j <= n; ++j) {
                    const double xj = ccoord(j, dmin, h);
                    for (int i = 1; i <= n; ++i) {
                        const double e =
                            u[off4(&g, i, j, k, l)] - exact_u(ccoord(i, dmin, h), xj, xk, xl, t_n);
                        sum += e * e;
                    }
                }
            }
            step_sum += sum;
        }
        err_sq += tau * cell * step_sum;
    }
    free(u);
    free(off);
    free(dg);
    free(ab);
    free(rhs);
    *err = sqrt(err_sq);
    return st;
}
