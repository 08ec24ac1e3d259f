// capi.cu -- the C ABI (include/subsurf_b200.h).
//
// Per-call entry points mirror the reference's free functions: they reuse a
// cached single-slab Domain for their grid, upload reference-layout host
// arrays, run the kernels and download the results.  ss_session_* expose the
// device-resident Domain (single GPU, an in-process slab group, or one rank
// of an NCCL job).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "domain.cuh"
#include "track.cuh"

namespace ssb {

static thread_local std::string t_err;
void set_last_error(const std::string& m) { t_err = m; }

static std::unique_ptr<Domain> g_cached;

static bool same_grid(const ss_grid& a, const ss_grid& b) {
    return a.n1 == b.n1 && a.n2 == b.n2 && a.n3 == b.n3 && a.n4 == b.n4 && a.h1 == b.h1 && a.h2 == b.h2 &&
           a.h3 == b.h3 && a.h4 == b.h4;
}

static void require_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n < 1)
        throw Error(SS_ERR_CUDA, std::string("no usable CUDA device (") +
                                     (e != cudaSuccess ? cudaGetErrorString(e) : "count 0") +
                                     "); this library has no CPU fallback");
}

// The per-call entry points share one cached Domain: a call holds its lock from
// cached() to the end of guard(), so concurrent per-call use from several host
// threads is serialised (sessions are independent objects and are not locked).
static std::mutex g_cached_mu;
static thread_local std::unique_lock<std::mutex> t_cached_lock;

static Domain& cached(const ss_grid& g) {
    if (!t_cached_lock.owns_lock()) t_cached_lock = std::unique_lock<std::mutex>(g_cached_mu);
    require_device();
    if (!g_cached || !same_grid(g_cached->g, g)) {
        g_cached.reset();
        int dev = 0;
        SSB_CUDA(cudaGetDevice(&dev));
        g_cached.reset(new Domain(g, dev, 1));
    }
    g_cached->prepared = false;
    return *g_cached;
}

template <class F>
static ss_status guard(F&& fn) {
    struct Release {
        ~Release() {
            if (t_cached_lock.owns_lock()) t_cached_lock.unlock();
        }
    } release;
    try {
        fn();
        t_err.clear();
        return SS_OK;
    } catch (const Error& e) {
        t_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        t_err = "host allocation failed";
        return SS_ERR_CUDA;
    } catch (const std::exception& e) {
        t_err = e.what();
        return SS_ERR_CUDA;
    }
}

static void heat_consts(const ss_grid& g, double dt, double hc[4]) {
    const double h[4] = {g.h1, g.h2, g.h3, g.h4};
    for (int a = 0; a < 4; ++a) hc[a] = (double)(float)(-(dt / (h[a] * h[a])));  // solver.cpp:89-90,107
}

}  // namespace ssb

using namespace ssb;

struct ss_session {
    std::unique_ptr<Domain> d;
};

extern "C" {

const char* ss_last_error(void) { return t_err.c_str(); }
int ss_abi_version(void) { return 6; }
unsigned long long ss_launch_count(void) { return g_launches.load(); }

int ss_device_available(void) {
    return guard([] { require_device(); }) == SS_OK ? 1 : 0;
}

double ss_sor_pass_bytes(const ss_grid* g) {
    // SURVEY.md 8(d) contract figure: 56 B per interior doxel per red+black sweep
    // (8 fp32 coefficients + rhs + u read + u write); one colour pass = half.
    const double N = (double)g->n1 * g->n2 * g->n3 * g->n4;
    return 0.5 * N * 56.0;
}

ss_status ss_assemble_step(const ss_grid* g, const double* u_prev, const double* G, double tau, double epsilon,
                           double* offdiag, double* diag, double* abar) {
    return guard([&] {
        validate_grid(g);
        validate_solver(tau, epsilon, 1.0, 1.0, 1, 1);
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        s.upload_state(u_prev, 0);
        if (G) {
            double* d8 = s.stage8_p();
            copy_h2d(d8, G, s.L.P * 8 * sizeof(double), d.stream);
            s.G[0].alloc(s.L.cs * 8);
            s.G[1].alloc(s.L.cs * 8);
            launch_pack8(d.stream, s.L, d8, s.G[0].p, s.G[1].p);
        }
        double* off = s.stage8_p();
        Dev<double> dg, ab;
        dg.alloc(s.L.P);
        ab.alloc(s.L.P);
        SSB_CUDA(cudaMemsetAsync(off, 0, s.L.P * 8 * sizeof(double), d.stream));
        SSB_CUDA(cudaMemsetAsync(dg.p, 0, s.L.P * sizeof(double), d.stream));
        SSB_CUDA(cudaMemsetAsync(ab.p, 0, s.L.P * sizeof(double), d.stream));
        s.assemble(s.S[0].pf(), G != nullptr, tau, epsilon, off, dg.p, ab.p);
        copy_d2h(offdiag, off, s.L.P * 8 * sizeof(double), d.stream);
        copy_d2h(diag, dg.p, s.L.P * sizeof(double), d.stream);
        copy_d2h(abar, ab.p, s.L.P * sizeof(double), d.stream);
        int bad = 0;
        SSB_CUDA(cudaMemcpyAsync(&bad, s.flags.p, sizeof(int), cudaMemcpyDeviceToHost, d.stream));
        d.sync();
        s.have_G = false;
        if (bad) throw Error(SS_ERR_NONFINITE, "assemble_step: non-finite coefficient (bad input field?)");
    });
}

ss_status ss_assemble_heat_step(const ss_grid* g, double dt, double* offdiag, double* diag, double* abar) {
    return guard([&] {
        validate_grid(g);
        require(dt > 0.0, "assemble_heat_step: dt must be > 0");
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        double hc[4];
        heat_consts(*g, dt, hc);
        double* off = s.stage8_p();
        Dev<double> dg, ab;
        dg.alloc(s.L.P);
        ab.alloc(s.L.P);
        launch_heat_export(d.stream, s.L, hc, off, dg.p, ab.p);
        copy_d2h(offdiag, off, s.L.P * 8 * sizeof(double), d.stream);
        copy_d2h(diag, dg.p, s.L.P * sizeof(double), d.stream);
        copy_d2h(abar, ab.p, s.L.P * sizeof(double), d.stream);
        d.sync();
    });
}

ss_status ss_redblack_sor(const ss_grid* g, const double* offdiag, const double* rhs, double* u, double omega,
                          double sor_tol, int sor_max_iter, int workers, int* iterations, double* residual) {
    if (iterations) *iterations = 0;
    if (residual) *residual = 0.0;
    return guard([&] {
        validate_grid(g);
        validate_solver(1.0, 1.0, omega, sor_tol, sor_max_iter, 1);
        require(workers >= 1, "Partition: worker count must be >= 1");
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        double* d8 = s.stage8_p();
        copy_h2d(d8, offdiag, s.L.P * 8 * sizeof(double), d.stream);
        launch_pack_coef(d.stream, s.L, d8, s.coef[0].p, s.coef[1].p);  // pack_coefficients, solver.cpp:233-249
        s.rhs_sep.alloc(s.L);
        s.upload(rhs, s.rhs_sep.pf());
        s.upload_state(u, 0);
        const int roles[kStateBuffers] = {0, 1, 2, 3};
        int rr = 0;
        const SolveOut o = d.solve(d.role_triples(roles), {s.rhs_sep.pf()}, false, omega, nullptr, sor_tol, false,
                                   0.0, sor_max_iter, false, &rr);
        s.download(s.S[rr].pf(), u);
        d.sync();
        if (iterations) *iterations = o.iterations;
        if (residual) *residual = o.residual;
        if (!o.converged) throw SolverErrT(o);
    });
}

ss_status ss_face_coefficients(const ss_grid* g, const double* I0s, const double* ITs, double K, double delta,
                               double vartheta, double* G) {
    return guard([&] {
        validate_grid(g);
        validate_edge(K, delta, vartheta);
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        DevField a, b;
        a.alloc(s.L);
        b.alloc(s.L);
        s.upload(I0s, a.pf());
        s.upload(ITs, b.pf());
        double* out = s.stage8_p();
        launch_fill_raw(d.stream, out, s.L.P * 8, 1.0);  // ghost entries = 1 (edge.hpp:73)
        s.face_coefficients(a.pf(), b.pf(), K, delta, vartheta, out);
        copy_d2h(G, out, s.L.P * 8 * sizeof(double), d.stream);
        d.sync();
        s.have_G = false;
    });
}

ss_status ss_heat_smooth(const ss_grid* g, const double* image, double sigma, int steps, double omega,
                         double sor_tol, int sor_max_iter, double* out) {
    return guard([&] {
        validate_grid(g);
        validate_smoothing(sigma, steps, sor_tol, sor_max_iter, omega);
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        DevField a, b, c, e;
        a.alloc(s.L);
        b.alloc(s.L);
        c.alloc(s.L);
        e.alloc(s.L);
        s.upload(image, a.pf());
        const std::vector<Domain::Triple> B = {{a.pf(), b.pf(), c.pf(), e.pf()}};
        const int r = d.heat_smooth(B, sigma, steps, omega, sor_tol, sor_max_iter);
        s.download(B[0][r], out);
        d.sync();
    });
}

ss_status ss_local_threshold(const ss_grid* g, const double* image, const ss_center* c, int n, double lambda,
                             double background, double* out) {
    return guard([&] {
        validate_grid(g);
        require(!(lambda < 0.0 || lambda > 1.0), "ThresholdParams: lambda must be in [0,1]");
        validate_centers(*g, c, n);
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        DevField a, b;
        a.alloc(s.L);
        b.alloc(s.L);
        s.upload(image, a.pf());
        BallSet bs;
        build_balls(bs, s.gl, 0, c, n, std::nan(""), false);  // per-row radii
        Dev<double> ab;
        ab.alloc(2 * (size_t)std::max(1, bs.count()));
        launch_fill(d.stream, s.L, b.pf(), background);
        if (bs.count()) {
            s.threshold_minmax(a.pf(), bs, ab.p);
            std::vector<double> h(2 * bs.count());
            SSB_CUDA(cudaMemcpyAsync(h.data(), ab.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, d.stream));
            d.sync();
            int first = INT_MAX;
            for (int q = 0; q < bs.count(); ++q)
                if (h[2 * q] > h[2 * q + 1]) first = std::min(first, bs.row[q]);
            if (first != INT_MAX)  // preprocess.cpp:89-91
                throw Error(SS_ERR_VALIDATION,
                            "local_threshold: ball in centers row " + std::to_string(first + 1) + " covers no doxels");
            s.threshold_write(a.pf(), b.pf(), bs, ab.p, lambda);
        }
        s.download(b.pf(), out);
        d.sync();
    });
}

ss_status ss_build_initial(const ss_grid* g, const ss_center* c, int n, double v, double R, int profile, double* u) {
    return guard([&] {
        validate_grid(g);
        require(v > 0.0, "InitParams: v must be > 0");
        require(R > 0.0, "InitParams: R must be > 0");
        validate_centers(*g, c, n);
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        DevField a;
        a.alloc(s.L);
        s.initial(a.pf(), c, n, v, R, profile);
        s.download(a.pf(), u);
        d.sync();
    });
}

ss_status ss_local_rescale(const ss_grid* g, double* u, const ss_center* c, int n, double radius) {
    return guard([&] {
        validate_grid(g);
        validate_centers(*g, c, n);
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        build_balls(s.rescale_balls, s.gl, 0, c, n, radius, false);
        s.upload_state(u, 0);
        s.rescale(0);
        s.download(s.S[0].pf(), u);
        d.sync();
    });
}

ss_status ss_apply_dirichlet(const ss_grid* g, double* f, double value) {
    return guard([&] {
        validate_grid(g);
        require(f != nullptr, "null field");
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        s.upload(f, s.S[0].pf());
        launch_set_ghosts(d.stream, s.L, s.S[0].pf(), value);
        s.download(s.S[0].pf(), f);
        d.sync();
    });
}

ss_status ss_apply_mirror_ghosts(const ss_grid* g, double* f) {
    return guard([&] {
        validate_grid(g);
        require(f != nullptr, "null field");
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        s.upload(f, s.S[0].pf());
        launch_mirror_ghosts(d.stream, s.L, s.S[0].pf());
        s.download(s.S[0].pf(), f);
        d.sync();
    });
}

ss_status ss_interior_minmax(const ss_grid* g, const double* f, double* lo, double* hi) {
    return guard([&] {
        validate_grid(g);
        require(f && lo && hi, "null argument");
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        s.upload(f, s.S[0].pf());
        launch_minmax(d.stream, s.L, s.S[0].pf(), s.scratch.p, s.scal.p + 1);
        double h[2];
        SSB_CUDA(cudaMemcpyAsync(h, s.scal.p + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, d.stream));
        d.sync();
        *lo = h[0];
        *hi = h[1];
    });
}

ss_status ss_extract_mask(const ss_grid* g, const double* u, double level, uint8_t* mask) {
    return guard([&] {
        validate_grid(g);
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        s.upload_state(u, 0);
        d.cur = 0;
        d.get_mask(level, mask);
    });
}

// ---------------------------------------------------------------- tracking
static cudaStream_t track_stream() {
    static cudaStream_t s = [] {
        cudaStream_t t;
        SSB_CUDA(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
        return t;
    }();
    return s;
}

static std::vector<ssb_track::Cell> to_cells(const ss_cell_record* r, int n) {
    std::vector<ssb_track::Cell> c(n);
    for (int i = 0; i < n; ++i) {
        c[i].frame = r[i].frame;
        c[i].label = r[i].label;
        c[i].cx = r[i].cx;
        c[i].cy = r[i].cy;
        c[i].cz = r[i].cz;
        c[i].max_distance = r[i].max_distance;
        c[i].voxel_count = r[i].voxel_count;
    }
    return c;
}

static void put_points(const std::vector<ss_track_point>& pts, ss_track_point* out, int capacity, int* n_points) {
    *n_points = (int)pts.size();
    if ((int)pts.size() > capacity || (!out && !pts.empty()))
        throw Error(SS_ERR_VALIDATION, "track: " + std::to_string(pts.size()) + " points, capacity " +
                                           std::to_string(capacity));
    if (!pts.empty()) std::memcpy(out, pts.data(), pts.size() * sizeof(ss_track_point));
}

ss_status ss_label_components(const ss_grid* g, const uint8_t* mask, int32_t* labels, int* labels_per_frame) {
    return guard([&] {
        validate_grid(g);
        require(mask && labels && labels_per_frame, "null buffer");
        require_device();
        Tracker t(g->n1, g->n2, g->n3, g->n4, track_stream());
        SSB_CUDA(cudaMemcpyAsync(t.mask(), mask, (size_t)t.frame_size() * g->n4, cudaMemcpyHostToDevice,
                                 track_stream()));
        t.label();
        SSB_CUDA(cudaMemcpyAsync(labels, t.labels(), (size_t)t.frame_size() * g->n4 * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost, track_stream()));
        SSB_CUDA(cudaStreamSynchronize(track_stream()));
        std::copy(t.labels_per_frame().begin(), t.labels_per_frame().end(), labels_per_frame);
    });
}

ss_status ss_distance_centers(const ss_grid* g, const int32_t* labels, const int* labels_per_frame,
                              ss_cell_record* out, int capacity, int* n_records) {
    return guard([&] {
        validate_grid(g);
        require(labels && labels_per_frame && n_records, "null buffer");
        require_device();
        Tracker t(g->n1, g->n2, g->n3, g->n4, track_stream());
        t.set_labels(labels, std::vector<int>(labels_per_frame, labels_per_frame + g->n4));
        t.centers();
        const std::vector<ssb_track::Cell>& c = t.cells();
        *n_records = (int)c.size();
        if ((int)c.size() > capacity || (!out && !c.empty()))
            throw Error(SS_ERR_VALIDATION, "distance_centers: " + std::to_string(c.size()) + " records, capacity " +
                                               std::to_string(capacity));
        for (size_t i = 0; i < c.size(); ++i)
            out[i] = ss_cell_record{c[i].frame, c[i].label, c[i].cx, c[i].cy, c[i].cz, c[i].max_distance,
                                    c[i].voxel_count};
    });
}

ss_status ss_backtrack_link(const ss_grid* g, const int32_t* labels, const int* labels_per_frame,
                            const ss_cell_record* records, int n_records, int* record_index, int* chain_start,
                            int* n_chains) {
    return guard([&] {
        validate_grid(g);
        require(labels && labels_per_frame && (records || n_records == 0) && record_index && chain_start && n_chains,
                "null buffer");
        require_device();
        Tracker t(g->n1, g->n2, g->n3, g->n4, track_stream());
        t.set_labels(labels, std::vector<int>(labels_per_frame, labels_per_frame + g->n4));
        t.set_cells(to_cells(records, n_records));
        std::vector<int> proj, overlap;
        t.targets(proj, overlap);
        const std::vector<ssb_track::Chain> ch =
            ssb_track::backtrack(t.labels_per_frame(), t.first(), t.cells(), proj, overlap);
        int k = 0;
        for (size_t c = 0; c < ch.size(); ++c) {
            chain_start[c] = k;
            for (int r : ch[c]) record_index[k++] = r;
        }
        chain_start[ch.size()] = k;
        *n_chains = (int)ch.size();
    });
}

ss_status ss_track(const ss_grid* g, const double* u, double level, int window, double radius, ss_track_point* out,
                   int capacity, int* n_points) {
    return guard([&] {
        validate_grid(g);
        require(u && n_points, "null buffer");
        Domain& d = cached(*g);
        Slab& s = *d.sp[0];
        s.upload_state(u, 0);
        Tracker t(g->n1, g->n2, g->n3, g->n4, d.stream);
        launch_mask(d.stream, s.L, s.S[0].pf(), level, t.mask());
        std::vector<ss_track_point> pts;
        track_points(t, window, radius, pts);
        put_points(pts, out, capacity, n_points);
    });
}

ss_status ss_segment(const ss_grid* g, const double* image, const ss_center* c, int n, const ss_seg_params* p,
                     const double* u0, double* u_out, ss_step_diag* diags) {
    return guard([&] {
        validate_grid(g);
        require(p != nullptr, "null params");
        Domain& d = cached(*g);
        d.prepare(image, c, n, *p, u0);
        if (diags) std::memset(diags, 0, sizeof(ss_step_diag) * p->n_steps);
        for (int step = 0; step < p->n_steps; ++step) {
            try {
                d.step(diags ? diags + step : nullptr);
            } catch (const SolverErrT& e) {  // the failing step's diag: SolverError's payload
                if (diags) {
                    diags[step].iterations = e.iterations;
                    diags[step].residual = e.residual;
                    diags[step].tol = -1.0;  // marks the failing step
                }
                d.prepared = false;
                throw;
            }
        }
        d.get_u(u_out);
        d.prepared = false;
    });
}

ss_status ss_session_create(const ss_grid* g, int device, ss_session** out) {
    return ss_session_create_group(g, 1, device, out);
}

ss_status ss_session_create_group(const ss_grid* g, int n_slabs, int device, ss_session** out) {
    return guard([&] {
        validate_grid(g);
        require(out != nullptr, "null output pointer");
        require_device();
        *out = nullptr;
        std::unique_ptr<ss_session> h(new ss_session);
        h->d.reset(new Domain(*g, device, n_slabs));
        *out = h.release();
    });
}

ss_status ss_nccl_unique_id(uint8_t out[128]) {
    return guard([&] {
        require(out != nullptr, "null output pointer");
        nccl_unique_id(out);
    });
}

ss_status ss_session_create_dist(const ss_grid* g, int rank, int world, const uint8_t uid[128], int device,
                                 ss_session** out) {
    return guard([&] {
        validate_grid(g);
        require(out != nullptr && uid != nullptr, "null argument");
        require_device();
        *out = nullptr;
        SSB_CUDA(cudaSetDevice(device));
        std::unique_ptr<ss_session> h(new ss_session);
        h->d.reset(new Domain(*g, device, rank, world, uid));
        *out = h.release();
    });
}

ss_status ss_session_create_dist_host(const ss_grid* g, int rank, int world, const ss_host_comm* comm, int device,
                                      ss_session** out) {
    return guard([&] {
        validate_grid(g);
        require(out != nullptr && comm != nullptr, "null argument");
        require_device();
        *out = nullptr;
        SSB_CUDA(cudaSetDevice(device));
        std::unique_ptr<ss_session> h(new ss_session);
        h->d.reset(new Domain(*g, device, rank, world, *comm));
        *out = h.release();
    });
}

ss_status ss_session_slab(ss_session* s, int* l_begin, int* l_count, int* world) {
    return guard([&] {
        require(s != nullptr, "null session");
        Domain& d = *s->d;
        if (l_begin) *l_begin = d.sp[0]->L.l0 + 1;
        if (l_count) *l_count = d.distributed ? d.sp[0]->L.n4 : d.g.n4;
        if (world) *world = d.world;
    });
}

ss_status ss_session_destroy(ss_session* s) {
    return guard([&] { delete s; });
}

void* ss_session_stream(ss_session* s) { return s ? (void*)s->d->stream : nullptr; }

ss_status ss_session_prepare(ss_session* s, const double* image, const ss_center* c, int n, const ss_seg_params* p,
                             const double* u0) {
    return guard([&] {
        require(s && p, "null session / params");
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->prepare(image, c, n, *p, u0);
    });
}

ss_status ss_session_step(ss_session* s, ss_step_diag* diag) {
    return guard([&] {
        require(s != nullptr, "null session");
        SSB_CUDA(cudaSetDevice(s->d->device));
        try {
            s->d->step(diag);
        } catch (const SolverErrT& e) {  // SolverError{last_residual, iterations} (solver.cpp:391-395)
            if (diag) {
                diag->iterations = e.iterations;
                diag->residual = e.residual;
            }
            throw;
        }
    });
}

ss_status ss_session_set_u(ss_session* s, const double* host_u) {
    return guard([&] {
        require(s && host_u, "null session / buffer");
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->set_u(host_u);
    });
}

ss_status ss_session_get_u(ss_session* s, double* host_u) {
    return guard([&] {
        require(s && host_u, "null session / buffer");
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->get_u(host_u);
    });
}

ss_status ss_session_get_mask(ss_session* s, double level, uint8_t* mask) {
    return guard([&] {
        require(s && mask, "null session / buffer");
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->get_mask(level, mask);
    });
}

ss_status ss_session_track(ss_session* s, double level, int window, double radius, ss_track_point* out,
                           int capacity, int* n_points) {
    return guard([&] {
        require(s && n_points, "null session / output");
        Domain& d = *s->d;
        require(!d.distributed, "track on a distributed session: gather u on one rank first");
        SSB_CUDA(cudaSetDevice(d.device));
        Tracker t(d.g.n1, d.g.n2, d.g.n3, d.g.n4, d.stream);
        const long long fr = t.frame_size();
        for (Slab* sl : d.sp) launch_mask(d.stream, sl->L, sl->S[d.cur].pf(), level, t.mask() + fr * sl->L.l0);
        std::vector<ss_track_point> pts;
        track_points(t, window, radius, pts);
        put_points(pts, out, capacity, n_points);
    });
}

ss_status ss_session_fixed_sweeps(ss_session* s, int n_sweeps, double* residual) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(n_sweeps >= 1, "n_sweeps must be >= 1");
        SSB_CUDA(cudaSetDevice(s->d->device));
        const double r = s->d->fixed_sweeps(n_sweeps);
        if (residual) *residual = r;
    });
}

ss_status ss_session_step_fixed(ss_session* s, int n_sweeps, ss_step_diag* diag) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(n_sweeps >= 1, "n_sweeps must be >= 1");
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->step(diag, n_sweeps, true);
    });
}

ss_status ss_session_step_host(ss_session* s, const double* u_in, double* u_out, int n_sweeps, ss_step_diag* diag) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(n_sweeps >= 0, "n_sweeps must be >= 0");
        SSB_CUDA(cudaSetDevice(s->d->device));
        try {
            s->d->step_host(u_in, u_out, n_sweeps, diag);
        } catch (const SolverErrT& e) {
            if (diag) {
                diag->iterations = e.iterations;
                diag->residual = e.residual;
            }
            throw;
        }
    });
}

ss_status ss_session_step_host_async(ss_session* s, const double* u_in, double* u_out, int n_sweeps,
                                     ss_step_diag* diag) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(n_sweeps >= 0, "n_sweeps must be >= 0");
        SSB_CUDA(cudaSetDevice(s->d->device));
        try {
            s->d->step_host_async(u_in, u_out, n_sweeps, diag);
        } catch (const SolverErrT& e) {
            if (diag) {
                diag->iterations = e.iterations;
                diag->residual = e.residual;
            }
            throw;
        }
    });
}

ss_status ss_session_wait(ss_session* s) {
    return guard([&] {
        require(s != nullptr, "null session");
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->wait_transfers();
        s->d->sync();
    });
}

ss_status ss_session_set_u_interior(ss_session* s, const double* u) {
    return guard([&] {
        require(s && u, "null session / buffer");
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->wait_transfers();
        s->d->set_u_interior(u);
        s->d->sync();
    });
}

ss_status ss_session_get_u_interior(ss_session* s, double* u) {
    return guard([&] {
        require(s && u, "null session / buffer");
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->wait_transfers();
        s->d->get_u_interior(u);
    });
}

ss_status ss_session_assemble_export(ss_session* s, double* offdiag) {
    return guard([&] {
        require(s && offdiag, "null session / output");
        Domain& d = *s->d;
        require(d.prepared, "session not prepared");
        require(d.single(), "assemble_export: single-slab sessions");
        SSB_CUDA(cudaSetDevice(d.device));
        Slab& x = *d.sp[0];
        x.assemble(x.S[d.cur].pf(), x.have_G, d.prm.tau, d.prm.epsilon, nullptr, nullptr, nullptr);
        Dev<double> off;
        off.alloc((size_t)x.L.P * 8);
        launch_unpack_coef(d.stream, x.L, x.coef[0].p, x.coef[1].p, off.p);
        int bad = 0;
        SSB_CUDA(cudaMemcpyAsync(&bad, x.flags.p, sizeof(int), cudaMemcpyDeviceToHost, d.stream));
        copy_d2h(offdiag, off.p, (size_t)x.L.P * 8 * sizeof(double), d.stream);
        d.sync();
        if (bad) throw Error(SS_ERR_NONFINITE, "assemble_step: non-finite coefficient (bad input field?)");
    });
}

ss_status ss_selftest_rsqrt(double* eps0) {
    return guard([&] {
        require(eps0 != nullptr, "null output");
        require_device();
        *eps0 = rsqrt_approx_bound();
    });
}

ss_status ss_session_eoc_row(ss_session* s, int n, double omega, double sor_tol, int sor_max_iter, double* err,
                             long long* sweeps) {
    return guard([&] {
        require(s && err, "null session / output");
        validate_solver(1.0, 1.0, omega, sor_tol, sor_max_iter, 1);
        SSB_CUDA(cudaSetDevice(s->d->device));
        s->d->prepared = false;
        *err = s->d->eoc_row(n, omega, sor_tol, sor_max_iter, sweeps);
    });
}

ss_status ss_session_set_loop_mode(ss_session* s, int mode) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(mode == 0 || mode == 1, "loop mode must be 0 or 1");
        s->d->loop_mode = mode;
    });
}

ss_status ss_session_set_kernel(ss_session* s, int kernel) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(kernel >= 0 && kernel <= 7 && kernel != 6,
                "kernel must be 0 (LDG), 1 (TMA), 2 (TMA wavefront), 3 (resident), 4 (auto), 5 (2D-tiled TMA) "
                "or 7 (one-sweep k-wavefront)");
        if (s->d->kernel != kernel) {  // captured loops of the old kernel are not reused
            s->d->clear_graphs();
        }
        s->d->kernel = kernel;
    });
}

ss_status ss_session_sor_kernel(ss_session* s, int* kernel) {
    return guard([&] {
        require(s != nullptr && kernel != nullptr, "null argument");
        *kernel = s->d->last_kernel;
    });
}

ss_status ss_session_set_profiling(ss_session* s, int enable) {
    return guard([&] {
        require(s != nullptr, "null session");
        s->d->profiling = enable != 0;
    });
}

ss_status ss_session_profile(ss_session* s, ss_profile* out) {
    return guard([&] {
        require(s && out, "null session / output");
        *out = s->d->prof;
        s->d->prof = ss_profile{};
    });
}

}  // extern "C"
