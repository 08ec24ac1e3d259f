/*
 * subsurf_oracle.h -- CPU restatement of the reference SUBSURF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker, never the product:
 * only tests/ (incl. the reference-timing harnesses in tests/perf/),
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may load it.  The product path (paper_2111_11866_b200) never links it
 * and has no CPU fallback.
 *
 * Every function restates one reference function in plain C with the same
 * floating-point operation order (compiled with -ffp-contract=off, SSE2, like
 * the reference's `-O3` build without -march), so results are bit-identical
 * to /root/reference/proj.  Pinned against the reference itself by
 * tests/test_oracle_pin.py (oracle/_ref, built from the reference sources) and
 * by the committed fixtures in tests/golden/.
 *
 * Layout: ghost-padded fp64 arrays, i fastest,
 *   idx = ((l*kMax + k)*jMax + j)*iMax + i       (grid.hpp:108-110)
 * Face order f = 2*axis + (sign > 0)               (grid.cpp:67-80)
 */
#ifndef SUBSURF_ORACLE_H
#define SUBSURF_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int n1, n2, n3, n4;
    double h1, h2, h3, h4;
} or_grid;

typedef struct {
    int frame;
    double x, y, z, radius;
} or_center;

enum {
    OR_OK = 0,
    OR_ERR_VALIDATION = 1,
    OR_ERR_NOCONVERGE = 2,
    OR_ERR_NONFINITE = 3
};

size_t or_padded_size(const or_grid* g);

/* grid.cpp:126-136 */
void or_apply_dirichlet(const or_grid* g, double* f, double value);
/* grid.cpp:138-156 */
void or_apply_mirror_ghosts(const or_grid* g, double* f);
/* grid.cpp:158-171 */
void or_interior_minmax(const or_grid* g, const double* f, double* lo, double* hi);

/* edge.cpp:33-48 : gradient on one face of interior doxel (i,j,k,l) */
void or_face_gradient(const or_grid* g, const double* u, int i, int j, int k, int l, int face,
                      double grad[4]);
/* edge.cpp:50-57 */
void or_face_gradient_sq(const or_grid* g, const double* u, int i, int j, int k, int l,
                         double out[8]);

/* edge.cpp:73-99 ; G has 8 doubles per padded doxel, ghosts = 1 */
int or_face_coefficients(const or_grid* g, const double* I0s, const double* ITs, double K,
                         double delta, double vartheta, double* G);

/* solver.cpp:23-77 ; G may be NULL (G == 1). off: 8*P, diag: P, abar: P (zeroed on ghosts) */
int or_assemble_step(const or_grid* g, const double* u_prev, const double* G, double tau,
                     double eps, double* off, double* diag, double* abar);
/* solver.cpp:79-116 */
int or_assemble_heat_step(const or_grid* g, double dt, double* off, double* diag, double* abar);

/* solver.cpp:124-397 restated single-worker (the reference is worker-count
 * invariant, solver.cpp:144-205).  u: in = guess, out = result.  Returns
 * OR_ERR_NOCONVERGE (with *iters/*res set and u holding the last iterate)
 * where the reference throws SolverError. slice_res (n4+2 doubles, may be NULL)
 * receives the per-slice residual partials of the last iteration. */
int or_redblack_sor(const or_grid* g, const double* off, const double* rhs, double* u,
                    double omega, double tol, int max_iter, int* iters, double* res);

/* preprocess.cpp:25-51 */
int or_heat_smooth(const or_grid* g, const double* image, double sigma, int steps, double omega,
                   double tol, int max_iter, double* out);
/* preprocess.cpp:53-102 */
int or_local_threshold(const or_grid* g, const double* image, const or_center* c, int n,
                       double lambda, double background, double* out);
/* io.cpp:128-140 */
int or_validate_centers(const or_grid* g, const or_center* c, int n);

/* seedinit.cpp:42-66 ; profile 0 = peak, 1 = linear */
int or_build_initial(const or_grid* g, const or_center* c, int n, double v, double R,
                     int profile, double* u);
/* seedinit.cpp:68-99 ; radius <= 0 means per-row radii */
int or_local_rescale(const or_grid* g, double* u, const or_center* c, int n, double radius);

/* tracking.cpp:35-52 : mask[(l-1)*n1*n2*n3 + ((k-1)*n2 + (j-1))*n1 + (i-1)] */
void or_extract_mask(const or_grid* g, const double* u, double level, unsigned char* mask);

typedef struct {
    /* SolverParams (solver.hpp:19-29) */
    double tau, epsilon, omega, sor_tol;
    int sor_max_iter, n_steps, rescale_each_step;
    /* harness extension: if > 0, sor_tol = sor_rel_tol * ||u^{n-1}||_2 per step */
    double sor_rel_tol;
    /* SmoothingParams (preprocess.hpp:10-18) */
    double sigma;
    int smooth_steps;
    double smooth_tol;
    int smooth_max_iter;
    double smooth_omega;
    /* ThresholdParams */
    double lambda, background;
    /* EdgeParams */
    double K, delta, vartheta;
    /* InitParams */
    double init_v, init_R;
    int init_profile;
    /* rescale radius (NaN: per-row radii = std::nullopt; else explicit) */
    double rescale_radius;
} or_seg_params;

typedef struct {
    int iterations;
    double residual, tol, umin, umax;
} or_step_diag;

/* solver.cpp:405-441 ; u0 may be NULL (build_initial), else used instead of
 * build_initial (then rescaled exactly as segment() rescales build_initial's
 * output). diags: n_steps entries or NULL. */
int or_segment(const or_grid* g, const double* image, const or_center* c, int n,
               const or_seg_params* p, const double* u0, double* u_out, or_step_diag* diags);

/* eoc.cpp:83-137 : the G == 1 verification row; returns the space-time L2 error */
int or_eoc_row(int n, double omega, double sor_tol, int max_iter, double* err);

#ifdef __cplusplus
}
#endif
#endif
