// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (/root/reference/proj/src, compiled in place by oracle/Makefile into
// oracle/_ref/libsubsurf_ref.so).
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by tests/ to pin the C
// restatement (oracle/subsurf_oracle.c) against the real reference, and by
// bench.py's reference arm / cpu_baseline leg to time the reference's own CPU
// solver.  Never linked into the product.
//
// The signatures mirror oracle/subsurf_oracle.h (prefix ref_ instead of or_)
// plus a worker count where the reference takes one.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <thread>

#include "subsurf/edge.hpp"
#include "subsurf/eoc.hpp"
#include "subsurf/grid.hpp"
#include "subsurf/io.hpp"
#include "subsurf/preprocess.hpp"
#include "subsurf/seedinit.hpp"
#include "subsurf/solver.hpp"
#include "subsurf/tracking.hpp"

#include "subsurf_oracle.h"

using namespace subsurf;

namespace {

GridSpec spec_of(const or_grid* g) { return GridSpec(g->n1, g->n2, g->n3, g->n4, g->h1, g->h2, g->h3, g->h4); }

Field4D field_of(const or_grid* g, const double* data) {
    Field4D f(spec_of(g));
    std::memcpy(f.data(), data, f.size() * sizeof(double));
    return f;
}

void store(const Field4D& f, double* out) { std::memcpy(out, f.data(), f.size() * sizeof(double)); }

CentersTable table_of(const or_center* c, int n) {
    CentersTable t;
    for (int m = 0; m < n; ++m) {
        CenterRow r;
        r.frame = c[m].frame;
        r.x = c[m].x;
        r.y = c[m].y;
        r.z = c[m].z;
        r.radius = c[m].radius;
        t.rows.push_back(r);
    }
    return t;
}

StepCoefficients coeff_of(const or_grid* g, const double* off) {
    StepCoefficients c;
    c.spec = spec_of(g);
    const std::size_t P = c.spec.padded_size();
    c.offdiag.resize(P);
    c.diag.resize(P);
    c.abar.resize(P);
    for (std::size_t n = 0; n < P; ++n) {
        double s = 0.0;
        for (int f = 0; f < 8; ++f) {
            c.offdiag[n][f] = off[8 * n + f];
            s += off[8 * n + f];
        }
        c.diag[n] = 1.0 - s;
    }
    return c;
}

thread_local char g_err[512];

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return OR_OK;
    } catch (const SolverError& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return OR_ERR_NOCONVERGE;
    } catch (const NumericalError& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return OR_ERR_NONFINITE;
    } catch (const std::exception& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return OR_ERR_VALIDATION;
    }
}

double interior_norm2(const Field4D& u) {
    const GridSpec& s = u.spec();
    double acc = 0.0;
    for (int l = 1; l <= s.n4; ++l)
        for (int k = 1; k <= s.n3; ++k)
            for (int j = 1; j <= s.n2; ++j)
                for (int i = 1; i <= s.n1; ++i) {
                    const double v = u.at(i, j, k, l);
                    acc += v * v;
                }
    return std::sqrt(acc);
}

SegmentationParams seg_of(const or_seg_params* p, int workers) {
    SegmentationParams sp;
    sp.solver.tau = p->tau;
    sp.solver.epsilon = p->epsilon;
    sp.solver.omega = p->omega;
    sp.solver.sor_tol = p->sor_tol;
    sp.solver.sor_max_iter = p->sor_max_iter;
    sp.solver.n_steps = p->n_steps;
    sp.solver.rescale_each_step = p->rescale_each_step != 0;
    sp.smoothing.sigma = p->sigma;
    sp.smoothing.steps = p->smooth_steps;
    sp.smoothing.sor_tol = p->smooth_tol;
    sp.smoothing.sor_max_iter = p->smooth_max_iter;
    sp.smoothing.omega = p->smooth_omega;
    sp.threshold.lambda = p->lambda;
    sp.threshold.background = p->background;
    sp.edge.K = p->K;
    sp.edge.delta = p->delta;
    sp.edge.vartheta = p->vartheta;
    sp.init.v = p->init_v;
    sp.init.R = p->init_R;
    sp.init.profile = p->init_profile == 0 ? InitProfile::peak : InitProfile::linear;
    if (!std::isnan(p->rescale_radius)) sp.rescale_radius = p->rescale_radius;
    sp.workers = workers;
    return sp;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

int ref_hardware_threads() { return int(std::max(1u, std::thread::hardware_concurrency())); }

int ref_face_coefficients(const or_grid* g, const double* I0s, const double* ITs, double K,
                          double delta, double vartheta, int workers, double* G) {
    return guarded([&] {
        EdgeParams p;
        p.K = K;
        p.delta = delta;
        p.vartheta = vartheta;
        const FaceCoefficientField out =
            face_coefficients(field_of(g, I0s), field_of(g, ITs), p, spec_of(g), workers);
        std::memcpy(G, out.data(), out.spec().padded_size() * 8 * sizeof(double));
    });
}

int ref_face_gradient_sq(const or_grid* g, const double* u, int i, int j, int k, int l,
                         double out[8]) {
    return guarded([&] {
        const Field4D f = field_of(g, u);
        const auto r = face_gradient_sq(f, f.spec(), Index4{i, j, k, l});
        for (int q = 0; q < 8; ++q) out[q] = r[q];
    });
}

int ref_assemble_step(const or_grid* g, const double* u_prev, const double* G, double tau,
                      double eps, int workers, double* off, double* diag, double* abar) {
    return guarded([&] {
        SolverParams sp;
        sp.tau = tau;
        sp.epsilon = eps;
        const GridSpec spec = spec_of(g);
        FaceCoefficientField gf;
        if (G) {
            gf = FaceCoefficientField(spec);
            for (int l = 0; l <= spec.n4 + 1; ++l)
                for (int k = 0; k <= spec.n3 + 1; ++k)
                    for (int j = 0; j <= spec.n2 + 1; ++j)
                        for (int i = 0; i <= spec.n1 + 1; ++i) {
                            auto& a = gf.at(i, j, k, l);
                            const std::size_t n = gf.flat(i, j, k, l);
                            for (int f = 0; f < 8; ++f) a[f] = G[8 * n + f];
                        }
        }
        const StepCoefficients c =
            assemble_step(field_of(g, u_prev), G ? &gf : nullptr, sp, spec, workers);
        for (std::size_t n = 0; n < c.offdiag.size(); ++n) {
            for (int f = 0; f < 8; ++f) off[8 * n + f] = c.offdiag[n][f];
            diag[n] = c.diag[n];
            abar[n] = c.abar[n];
        }
    });
}

int ref_assemble_heat_step(const or_grid* g, double dt, double* off, double* diag, double* abar) {
    return guarded([&] {
        const StepCoefficients c = assemble_heat_step(spec_of(g), dt, 1);
        for (std::size_t n = 0; n < c.offdiag.size(); ++n) {
            for (int f = 0; f < 8; ++f) off[8 * n + f] = c.offdiag[n][f];
            diag[n] = c.diag[n];
            abar[n] = c.abar[n];
        }
    });
}

int ref_redblack_sor(const or_grid* g, const double* off, const double* rhs, double* u,
                     double omega, double tol, int max_iter, int workers, int* iters,
                     double* res) {
    *iters = 0;
    *res = 0.0;
    return guarded([&] {
        SolverParams sp;
        sp.omega = omega;
        sp.sor_tol = tol;
        sp.sor_max_iter = max_iter;
        const GridSpec spec = spec_of(g);
        const Partition part = Partition::create(spec.n4, Partition::clamp_workers(spec.n4, workers));
        try {
            SorResult r = redblack_sor(coeff_of(g, off), field_of(g, rhs), field_of(g, u), sp, part);
            store(r.u, u);
            *iters = r.iterations;
            *res = r.residual;
        } catch (const SolverError& e) {
            *iters = e.iterations;
            *res = e.last_residual;
            throw;
        }
    });
}

int ref_heat_smooth(const or_grid* g, const double* image, double sigma, int steps, double omega,
                    double tol, int max_iter, int workers, double* out) {
    return guarded([&] {
        SmoothingParams p;
        p.sigma = sigma;
        p.steps = steps;
        p.omega = omega;
        p.sor_tol = tol;
        p.sor_max_iter = max_iter;
        store(heat_smooth(field_of(g, image), p, workers), out);
    });
}

int ref_local_threshold(const or_grid* g, const double* image, const or_center* c, int n,
                        double lambda, double background, double* out) {
    return guarded([&] {
        ThresholdParams p;
        p.lambda = lambda;
        p.background = background;
        store(local_threshold(field_of(g, image), table_of(c, n), p), out);
    });
}

int ref_build_initial(const or_grid* g, const or_center* c, int n, double v, double R,
                      int profile, double* u) {
    return guarded([&] {
        InitParams p;
        p.v = v;
        p.R = R;
        p.profile = profile == 0 ? InitProfile::peak : InitProfile::linear;
        store(build_initial(table_of(c, n), p, spec_of(g)), u);
    });
}

int ref_local_rescale(const or_grid* g, double* u, const or_center* c, int n, double radius) {
    return guarded([&] {
        Field4D f = field_of(g, u);
        local_rescale(f, table_of(c, n), std::isnan(radius) ? std::nullopt : std::optional<double>(radius));
        store(f, u);
    });
}

void ref_apply_mirror_ghosts(const or_grid* g, double* f) {
    Field4D x = field_of(g, f);
    apply_mirror_ghosts(x);
    store(x, f);
}

void ref_extract_mask(const or_grid* g, const double* u, double level, unsigned char* mask) {
    const MaskFrames m = extract_mask(field_of(g, u), level);
    std::size_t q = 0;
    for (const auto& fr : m.frames)
        for (auto b : fr) mask[q++] = b;
}

// ---- tracking (tracking.cpp), flat arrays: frames of n1*n2*n3, x fastest
static LabelField labels_of(const or_grid* g, const int* labels, const int* lpf) {
    LabelField L;
    L.n1 = g->n1;
    L.n2 = g->n2;
    L.n3 = g->n3;
    const std::size_t fs = L.frame_size();
    L.frames.resize(g->n4);
    L.labels_per_frame.assign(lpf, lpf + g->n4);
    for (int f = 0; f < g->n4; ++f) L.frames[f].assign(labels + f * fs, labels + (f + 1) * fs);
    return L;
}

/* label_components: labels n4*fs, lpf n4 */
int ref_label_components(const or_grid* g, const unsigned char* mask, int* labels, int* lpf) {
    return guarded([&] {
        MaskFrames m;
        m.n1 = g->n1;
        m.n2 = g->n2;
        m.n3 = g->n3;
        const std::size_t fs = m.frame_size();
        m.frames.resize(g->n4);
        for (int f = 0; f < g->n4; ++f) m.frames[f].assign(mask + f * fs, mask + (f + 1) * fs);
        const LabelField L = label_components(m);
        for (int f = 0; f < g->n4; ++f) {
            std::memcpy(labels + f * fs, L.frames[f].data(), fs * sizeof(int));
            lpf[f] = L.labels_per_frame[f];
        }
    });
}

/* distance_centers: 7 ints per record (frame, label, cx, cy, cz, max_distance, voxel_count) */
int ref_distance_centers(const or_grid* g, const int* labels, const int* lpf, long long* out, int capacity,
                         int* n) {
    return guarded([&] {
        const std::vector<CellRecord> r = distance_centers(labels_of(g, labels, lpf));
        *n = int(r.size());
        if (int(r.size()) > capacity) throw std::runtime_error("capacity");
        for (std::size_t i = 0; i < r.size(); ++i) {
            long long* o = out + 7 * i;
            o[0] = r[i].frame;
            o[1] = r[i].label;
            o[2] = r[i].center[0];
            o[3] = r[i].center[1];
            o[4] = r[i].center[2];
            o[5] = r[i].max_distance;
            o[6] = (long long)r[i].voxel_count;
        }
    });
}

/* backtrack_link on the reference's own records: per chain the (frame, label)
 * pairs, chains concatenated; chain_start n_chains+1 entries */
int ref_backtrack_link(const or_grid* g, const int* labels, const int* lpf, int* frame_label, int* chain_start,
                       int* n_chains) {
    return guarded([&] {
        const LabelField L = labels_of(g, labels, lpf);
        const std::vector<CellRecord> recs = distance_centers(L);
        const std::vector<Trajectory> t = backtrack_link(recs, L);
        int k = 0;
        for (std::size_t c = 0; c < t.size(); ++c) {
            chain_start[c] = k;
            for (const CellRecord& r : t[c].records) {
                frame_label[2 * k] = r.frame;
                frame_label[2 * k + 1] = r.label;
                ++k;
            }
        }
        chain_start[t.size()] = k;
        *n_chains = int(t.size());
    });
}

/* prolong_and_merge on partials given as records (frame, x, y, z) concatenated;
 * sizes[np]; output: merged trajectories as records concatenated + sizes */
int ref_prolong_and_merge(int np, const int* sizes, const int* fxyz, int window, double radius, int* out_fxyz,
                          int* out_sizes, int* n_out) {
    return guarded([&] {
        std::vector<Trajectory> parts(np);
        int k = 0;
        for (int p = 0; p < np; ++p) {
            parts[p].id = p + 1;
            for (int r = 0; r < sizes[p]; ++r, ++k) {
                CellRecord c;
                c.frame = fxyz[4 * k];
                c.center = {fxyz[4 * k + 1], fxyz[4 * k + 2], fxyz[4 * k + 3]};
                c.label = k + 1;
                parts[p].records.push_back(c);
            }
        }
        const std::vector<Trajectory> m = prolong_and_merge(parts, window, radius);
        int q = 0;
        for (std::size_t t = 0; t < m.size(); ++t) {
            out_sizes[t] = int(m[t].records.size());
            for (const CellRecord& c : m[t].records) {
                out_fxyz[4 * q] = c.frame;
                out_fxyz[4 * q + 1] = c.center[0];
                out_fxyz[4 * q + 2] = c.center[1];
                out_fxyz[4 * q + 3] = c.center[2];
                ++q;
            }
        }
        *n_out = int(m.size());
    });
}

/* track(u): points (id, frame) ints + (x, y, z) doubles */
int ref_track(const or_grid* g, const double* u, double level, int window, double radius, int* id_frame,
              double* xyz, int capacity, int* n) {
    return guarded([&] {
        TrackParams p;
        p.level = level;
        p.window = window;
        p.radius = radius;
        const TrajectoryFile tf = track(field_of(g, u), p);
        *n = int(tf.points.size());
        if (*n > capacity) throw std::runtime_error("capacity");
        for (int i = 0; i < *n; ++i) {
            id_frame[2 * i] = tf.points[i].trajectory_id;
            id_frame[2 * i + 1] = tf.points[i].frame;
            xyz[3 * i] = tf.points[i].x;
            xyz[3 * i + 1] = tf.points[i].y;
            xyz[3 * i + 2] = tf.points[i].z;
        }
    });
}

int ref_eoc_row(int n, double omega, double sor_tol, int max_iter, int workers, double* err) {
    return guarded([&] {
        EocConfig cfg;
        cfg.omega = omega;
        cfg.sor_tol = sor_tol;
        cfg.sor_max_iter = max_iter;
        cfg.workers = workers;
        *err = run_levelset_row(n, cfg);
    });
}

// segment() (solver.cpp:405-441) unchanged when rel_tol <= 0 and u0 == NULL.
// Otherwise the harness loop of SURVEY.md section 8(d): the same sequence of
// public reference calls with a per-step sor_tol = rel_tol * ||u^{n-1}||_2
// and/or a caller-built u0.  Per-step diagnostics and phase timings go to
// diags / times (seconds: [setup, assemble_total, sor_total, rescale_total]);
// step_seconds[n] is the wall time of time step n+1 (assemble + SOR + rescale).
int ref_segment(const or_grid* g, const double* image, const or_center* c, int n,
                const or_seg_params* p, const double* u0, int workers, double* u_out,
                or_step_diag* diags, double* times, long long* sor_sweeps, double* step_seconds) {
    using clk = std::chrono::steady_clock;
    return guarded([&] {
        SegmentationParams sp = seg_of(p, workers);

        const Field4D image_f = field_of(g, image);
        const CentersTable centers = table_of(c, n);
        if (p->sor_rel_tol <= 0.0 && !u0 && !diags && !times && !step_seconds) {
            store(segment(image_f, centers, sp), u_out);
            return;
        }
        // the loop of solver.cpp:405-441 through the same public calls
        const auto t0 = clk::now();
        const GridSpec& spec = image_f.spec();
        sp.solver.validate();
        validate_centers(centers, spec);
        const int w = Partition::clamp_workers(spec.n4, sp.workers);
        Field4D u = u0 ? field_of(g, u0) : build_initial(centers, sp.init, spec);
        local_rescale(u, centers, sp.rescale_radius);
        const Field4D th = local_threshold(image_f, centers, sp.threshold);
        const Field4D I0s = heat_smooth(image_f, sp.smoothing, w);
        const Field4D ITs = heat_smooth(th, sp.smoothing, w);
        const FaceCoefficientField G = face_coefficients(I0s, ITs, sp.edge, spec, w);
        apply_dirichlet(u, 0.0);
        const Partition part = Partition::create(spec.n4, w);
        double t_asm = 0, t_sor = 0, t_resc = 0;
        long long sweeps = 0;
        const auto t1 = clk::now();
        for (int step = 1; step <= sp.solver.n_steps; ++step) {
            const auto a0 = clk::now();
            const StepCoefficients coeff = assemble_step(u, &G, sp.solver, spec, w);
            const auto a1 = clk::now();
            SolverParams stp = sp.solver;
            if (p->sor_rel_tol > 0.0) stp.sor_tol = p->sor_rel_tol * interior_norm2(u);
            SorResult sor = redblack_sor(coeff, u, u, stp, part);
            const auto a2 = clk::now();
            u = std::move(sor.u);
            if (sp.solver.rescale_each_step) local_rescale(u, centers, sp.rescale_radius);
            const auto a3 = clk::now();
            t_asm += std::chrono::duration<double>(a1 - a0).count();
            t_sor += std::chrono::duration<double>(a2 - a1).count();
            t_resc += std::chrono::duration<double>(a3 - a2).count();
            if (step_seconds) step_seconds[step - 1] = std::chrono::duration<double>(a3 - a0).count();
            sweeps += sor.iterations;
            if (diags) {
                diags[step - 1].iterations = sor.iterations;
                diags[step - 1].residual = sor.residual;
                diags[step - 1].tol = stp.sor_tol;
                const auto [lo, hi] = interior_minmax(u);
                diags[step - 1].umin = lo;
                diags[step - 1].umax = hi;
            }
        }
        store(u, u_out);
        if (times) {
            times[0] = std::chrono::duration<double>(t1 - t0).count();
            times[1] = t_asm;
            times[2] = t_sor;
            times[3] = t_resc;
        }
        if (sor_sweeps) *sor_sweeps = sweeps;
    });
}

// Fixed-sweep time steps (BASELINE config 4: "fixed 50 SOR sweeps per time step, no early
// stop") through the reference's public calls.  The reference has no such mode:
// redblack_sor throws SolverError{last_residual, iterations} at max_iter and discards the
// iterate (solver.cpp:201-206, :391-395).  Same preamble as ref_segment, then per step
// assemble_step + redblack_sor(max_iter = n_sweeps, sor_tol = 1e-300) + local_rescale.
//   mode 0 (parity pin): the iterate after exactly n_sweeps sweeps is recovered from the
//     reference itself by a second call with sor_tol = the thrown residual r_n: it stops at
//     the first iteration whose residual is <= r_n, which must be n_sweeps (checked;
//     residuals decrease strictly in practice), and returns that iterate.
//   mode 1 (bench): only the throwing call is made (timed with the assembly and the
//     rescale); the reference discards its iterate, so u is not advanced -- every step
//     repeats the same work.
int ref_segment_fixed(const or_grid* g, const double* image, const or_center* c, int n,
                      const or_seg_params* p, const double* u0, int workers, int n_sweeps, int mode,
                      double* u_out, or_step_diag* diags, double* times, double* step_seconds) {
    using clk = std::chrono::steady_clock;
    return guarded([&] {
        SegmentationParams sp = seg_of(p, workers);
        const Field4D image_f = field_of(g, image);
        const CentersTable centers = table_of(c, n);
        const auto t0 = clk::now();
        const GridSpec& spec = image_f.spec();
        sp.solver.validate();
        validate_centers(centers, spec);
        const int w = Partition::clamp_workers(spec.n4, sp.workers);
        Field4D u = u0 ? field_of(g, u0) : build_initial(centers, sp.init, spec);
        local_rescale(u, centers, sp.rescale_radius);
        const Field4D th = local_threshold(image_f, centers, sp.threshold);
        const Field4D I0s = heat_smooth(image_f, sp.smoothing, w);
        const Field4D ITs = heat_smooth(th, sp.smoothing, w);
        const FaceCoefficientField G = face_coefficients(I0s, ITs, sp.edge, spec, w);
        apply_dirichlet(u, 0.0);
        const Partition part = Partition::create(spec.n4, w);
        const auto t1 = clk::now();
        for (int step = 1; step <= sp.solver.n_steps; ++step) {
            const auto a0 = clk::now();
            const StepCoefficients coeff = assemble_step(u, &G, sp.solver, spec, w);
            SolverParams stp = sp.solver;
            stp.sor_tol = 1e-300;
            stp.sor_max_iter = n_sweeps;
            double r = 0.0;
            int it = 0;
            try {
                SorResult sor = redblack_sor(coeff, u, u, stp, part);  // converged below 1e-300
                r = sor.residual;
                it = sor.iterations;
                if (mode == 0) u = std::move(sor.u);
            } catch (const SolverError& e) {
                r = e.last_residual;
                it = e.iterations;
                if (mode == 0) {
                    stp.sor_tol = r;
                    SorResult sor = redblack_sor(coeff, u, u, stp, part);
                    if (sor.iterations != n_sweeps || sor.residual != r)
                        throw std::runtime_error("fixed-sweep pin: residual not strictly decreasing (stopped at " +
                                                 std::to_string(sor.iterations) + ")");
                    u = std::move(sor.u);
                }
            }
            if (sp.solver.rescale_each_step) local_rescale(u, centers, sp.rescale_radius);
            const auto a1 = clk::now();
            if (step_seconds) step_seconds[step - 1] = std::chrono::duration<double>(a1 - a0).count();
            if (diags) {
                diags[step - 1].iterations = it;
                diags[step - 1].residual = r;
                diags[step - 1].tol = 1e-300;
                const auto [lo, hi] = interior_minmax(u);
                diags[step - 1].umin = lo;
                diags[step - 1].umax = hi;
            }
        }
        store(u, u_out);
        if (times) times[0] = std::chrono::duration<double>(t1 - t0).count();
    });
}

// Steady-state sweep rate of the reference's redblack_sor (bench.py cpu_baseline): the
// system assemble_step(u, G == 1) on the caller's grid, then two calls of n_a and n_b
// sweeps (max_iter, sor_tol = 1e-300: both end in SolverError, caught).  secs[0], secs[1]
// are their wall times; (secs[1] - secs[0]) / (n_b - n_a) is the time per sweep with the
// per-call scatter / coefficient packing / thread start-up cancelled out.
int ref_sor_rate(const or_grid* g, const double* u0, double tau, double eps, double omega, int n_a, int n_b,
                 int workers, double* secs) {
    using clk = std::chrono::steady_clock;
    return guarded([&] {
        SolverParams sp;
        sp.tau = tau;
        sp.epsilon = eps;
        sp.omega = omega;
        sp.sor_tol = 1e-300;
        const GridSpec spec = spec_of(g);
        const int w = Partition::clamp_workers(spec.n4, workers);
        const Field4D u = field_of(g, u0);
        const StepCoefficients coeff = assemble_step(u, nullptr, sp, spec, w);
        const Partition part = Partition::create(spec.n4, w);
        const int ns[2] = {n_a, n_b};
        for (int q = 0; q < 2; ++q) {
            sp.sor_max_iter = ns[q];
            const auto t0 = clk::now();
            try {
                (void)redblack_sor(coeff, u, u, sp, part);
            } catch (const SolverError&) {
            }
            secs[q] = std::chrono::duration<double>(clk::now() - t0).count();
        }
    });
}

// The reference's own writers (io.cpp), for byte-for-byte comparison of the CLI drop-in's
// output files: write_image4d (io.cpp:99-119), export_frame_vtk (io.cpp:198-223),
// write_trajectories (io.cpp:170-177), and the track subcommand's label-field VTKs
// (cli.cpp:174-188: label_components of extract_mask, exported frame by frame).
int ref_write_image4d(const or_grid* g, const double* u, const char* header, const char* data) {
    return guarded([&] { write_image4d(field_of(g, u), header, data); });
}

int ref_export_frame_vtk(const or_grid* g, const double* u, int l, const char* path) {
    return guarded([&] { export_frame_vtk(field_of(g, u), l, path); });
}

int ref_write_trajectories(int n, const int* id_frame, const double* xyz, const char* path) {
    return guarded([&] {
        TrajectoryFile t;
        for (int q = 0; q < n; ++q) {
            TrajectoryPoint pt;
            pt.trajectory_id = id_frame[2 * q];
            pt.frame = id_frame[2 * q + 1];
            pt.x = xyz[3 * q];
            pt.y = xyz[3 * q + 1];
            pt.z = xyz[3 * q + 2];
            t.points.push_back(pt);
        }
        write_trajectories(t, path);
    });
}

int ref_export_label_vtks(const or_grid* g, const double* u, double level, const char* prefix) {
    return guarded([&] {
        const Field4D f = field_of(g, u);
        const LabelField labels = label_components(extract_mask(f, level));
        const GridSpec& spec = f.spec();
        Field4D label_field(spec, 0.0);
        for (int l = 1; l <= spec.n4; ++l)
            for (int k = 1; k <= spec.n3; ++k)
                for (int j = 1; j <= spec.n2; ++j)
                    for (int i = 1; i <= spec.n1; ++i)
                        label_field.at(i, j, k, l) = double(labels.frames[l - 1][labels.voxel(i - 1, j - 1, k - 1)]);
        for (int l = 1; l <= spec.n4; ++l)
            export_frame_vtk(label_field, l, std::string(prefix) + "_f" + std::to_string(l - 1) + ".vtk");
    });
}

}  // extern "C"
