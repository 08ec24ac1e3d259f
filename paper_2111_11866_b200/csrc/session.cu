// session.cu -- device-resident SUBSURF state and the C ABI (include/subsurf_b200.h).
//
// A Session owns every device buffer of one grid: three rotating colour-packed
// state fields (guess/rhs + two SOR output buffers), fp32 colour-packed
// coefficients, colour-packed fp64 edge coefficients G, residual partials and
// the SOR loop state.  segment() (solver.cpp:405-441) runs entirely on the
// device; host <-> device copies happen only at the API boundary.
//
// The stateless per-call entry points (ss_assemble_step, ss_redblack_sor, ...)
// reuse a cached Session for their grid, upload the reference-layout host
// arrays, run the same kernels and download the results.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace ssb {

std::atomic<unsigned long long> g_launches{0};
static thread_local std::string t_err;
void set_last_error(const std::string& m) { t_err = m; }

template <class T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    Dev() = default;
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    ~Dev() { reset(); }
    void alloc(size_t count) {
        if (count == n && p) return;
        reset();
        if (count == 0) return;
        SSB_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

struct DevField {
    Dev<double> c[2];
    void alloc(const Layout& L) {
        c[0].alloc(L.cs);
        c[1].alloc(L.cs);
    }
    PField pf() const {
        PField f;
        f.c[0] = c[0].p;
        f.c[1] = c[1].p;
        return f;
    }
    void reset() {
        c[0].reset();
        c[1].reset();
    }
};

// ------------------------------------------------------------------ balls
// Ball bounds exactly as seedinit.cpp:22-31 / preprocess.cpp:63-68.
static Ball make_ball(const ss_grid& g, const ss_center& c, double r) {
    Ball b{};
    b.l = c.frame + 1;
    b.i0 = std::max(1, int(std::ceil(c.x - r)) + 1);
    b.i1 = std::min(g.n1, int(std::floor(c.x + r)) + 1);
    b.j0 = std::max(1, int(std::ceil(c.y - r)) + 1);
    b.j1 = std::min(g.n2, int(std::floor(c.y + r)) + 1);
    b.k0 = std::max(1, int(std::ceil(c.z - r)) + 1);
    b.k1 = std::min(g.n3, int(std::floor(c.z + r)) + 1);
    b.x = c.x;
    b.y = c.y;
    b.z = c.z;
    b.r = r;
    b.r_sq = r * r;
    return b;
}

static bool boxes_meet(const Ball& a, const Ball& b) {
    return a.l == b.l && a.i0 <= b.i1 && b.i0 <= a.i1 && a.j0 <= b.j1 && b.j0 <= a.j1 &&
           a.k0 <= b.k1 && b.k0 <= a.k1;
}

// Balls grouped into waves preserving table order among overlapping balls.
struct BallSet {
    std::vector<Ball> host;     // wave-sorted
    std::vector<int> row;       // wave-sorted index -> centres-table row
    std::vector<int> wave_off;  // waves + 1 offsets into host
    Dev<Ball> dev;
    int count() const { return (int)host.size(); }
    int waves() const { return (int)wave_off.size() - 1; }
};

static void build_balls(BallSet& bs, const ss_grid& g, const ss_center* c, int n,
                        double radius_override, bool fixed_radius) {
    std::vector<Ball> table(n);
    for (int m = 0; m < n; ++m)
        table[m] = make_ball(g, c[m], fixed_radius || radius_override > 0.0 ? radius_override : c[m].radius);
    std::vector<int> wave(n, 0);
    int nw = 0;
    for (int b = 0; b < n; ++b) {
        int w = 0;
        for (int a = 0; a < b; ++a)
            if (wave[a] + 1 > w && boxes_meet(table[a], table[b])) w = wave[a] + 1;
        wave[b] = w;
        nw = std::max(nw, w + 1);
    }
    bs.host.clear();
    bs.row.clear();
    bs.wave_off.assign(1, 0);
    for (int w = 0; w < nw; ++w) {
        for (int b = 0; b < n; ++b)
            if (wave[b] == w) {
                bs.host.push_back(table[b]);
                bs.row.push_back(b);
            }
        bs.wave_off.push_back((int)bs.host.size());
    }
    bs.dev.alloc(std::max<size_t>(1, bs.host.size()));
    if (!bs.host.empty())
        SSB_CUDA(cudaMemcpy(bs.dev.p, bs.host.data(), bs.host.size() * sizeof(Ball),
                            cudaMemcpyHostToDevice));
}

// ------------------------------------------------------------------ validation
// (solver.cpp:13-21, preprocess.cpp:11-23, edge.cpp:9-14, seedinit.cpp:9-12, io.cpp:128-140)
static void require(bool ok, const std::string& msg) {
    if (!ok) throw Error(SS_ERR_VALIDATION, msg);
}
static void validate_grid(const ss_grid* g) {
    require(g != nullptr, "null grid");
    require(g->n1 >= 1 && g->n2 >= 1 && g->n3 >= 1 && g->n4 >= 1, "GridSpec: doxel counts must be >= 1");
    require(g->h1 > 0.0 && g->h2 > 0.0 && g->h3 > 0.0 && g->h4 > 0.0, "GridSpec: spacings must be > 0");
}
static void validate_solver(double tau, double eps, double omega, double tol, int max_iter, int n_steps) {
    require(!(tau < 0.0), "SolverParams: tau must be >= 0");
    require(eps > 0.0, "SolverParams: epsilon must be > 0");
    require(omega > 0.0 && omega < 2.0, "SolverParams: omega must lie in (0,2)");
    require(tol > 0.0, "SolverParams: sor_tol must be > 0");
    require(max_iter >= 1, "SolverParams: sor_max_iter must be >= 1");
    require(n_steps >= 1, "SolverParams: n_steps must be >= 1");
}
static void validate_smoothing(double sigma, int steps, double tol, int max_iter, double omega) {
    require(!(sigma < 0.0), "SmoothingParams: sigma must be >= 0");
    require(steps >= 1, "SmoothingParams: steps must be >= 1");
    require(tol > 0.0, "SmoothingParams: sor_tol must be > 0");
    require(max_iter >= 1, "SmoothingParams: sor_max_iter must be >= 1");
    require(omega > 0.0 && omega < 2.0, "SmoothingParams: omega must lie in (0,2)");
}
static void validate_edge(double K, double delta, double vartheta) {
    require(!(K < 0.0), "EdgeParams: K must be >= 0");
    require(!(delta < 0.0 || delta > 1.0), "EdgeParams: delta must be in [0,1]");
    require(!(vartheta < 0.0 || vartheta > 1.0), "EdgeParams: vartheta must be in [0,1]");
}
static void validate_centers(const ss_grid& g, const ss_center* c, int n) {
    require(n == 0 || c != nullptr, "null centres table");
    for (int m = 0; m < n; ++m) {
        const std::string where = "centers row " + std::to_string(m + 1);
        require(c[m].frame >= 0 && c[m].frame < g.n4,
                where + ": frame " + std::to_string(c[m].frame) + " out of range [0," +
                    std::to_string(g.n4 - 1) + "]");
        require(c[m].radius > 0.0, where + ": radius must be > 0");
        require(!(c[m].x < 0.0 || c[m].x > g.n1 - 1 || c[m].y < 0.0 || c[m].y > g.n2 - 1 ||
                  c[m].z < 0.0 || c[m].z > g.n3 - 1),
                where + ": center outside volume bounds");
    }
}

// ------------------------------------------------------------------ session
struct SolveOut {
    int iterations = 0;
    double residual = 0.0, tol = 0.0;
    bool converged = false;
};

// A captured loop body bakes in its kernel arguments: key on all of them.
struct GraphKey {
    int heat;
    const void* ptr[8];  // 6 state arrays + 2 rhs arrays
    double omega;
    double hc[4];
    bool operator==(const GraphKey& o) const {
        if (heat != o.heat || omega != o.omega) return false;
        for (int q = 0; q < 8; ++q)
            if (ptr[q] != o.ptr[q]) return false;
        for (int q = 0; q < 4; ++q)
            if (hc[q] != o.hc[q]) return false;
        return true;
    }
};

struct Session {
    ss_grid g{};
    Layout L{};
    int device = 0;
    cudaStream_t stream = nullptr, cap_stream = nullptr;

    DevField S[3];        // rotating state buffers
    int cur = 0;          // S[cur] holds u
    DevField rhs_sep;     // separate rhs (per-call redblack_sor only)
    Dev<float> coef[2];
    Dev<double> G[2];
    bool have_G = false;
    Dev<double> part[2];
    Dev<double> slice_res;
    Dev<SorState> st;
    SorState* st_host = nullptr;  // pinned
    Dev<double> scratch;          // reductions
    Dev<double> scal;             // [0] norm_sq, [1..2] minmax
    double* scal_host = nullptr;  // pinned
    Dev<int> flags;               // [0] bad (assembly non-finite), [1] empty ball
    int* flags_host = nullptr;    // pinned
    Dev<double> stage;            // P doubles (host transfers)
    Dev<double> stage8;           // 8 P doubles (per-call coefficient / G transfers)

    // prepared segment() state
    bool prepared = false;
    ss_seg_params prm{};
    BallSet rescale_balls;

    // loop control
    int loop_mode = 1;
    bool profiling = false;
    struct GraphEntry {
        GraphKey key;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
    };
    std::vector<GraphEntry> graphs;
    ss_profile prof{};
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_c = nullptr, ev_d = nullptr;

    explicit Session(const ss_grid& grid, int dev) : g(grid), L(Layout::make(grid)), device(dev) {
        SSB_CUDA(cudaSetDevice(device));
        SSB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        SSB_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
        for (auto& f : S) f.alloc(L);
        coef[0].alloc(L.cs * 8);
        coef[1].alloc(L.cs * 8);
        SorArgs tmp{};
        pass_tiles(L, tmp);
        part[0].alloc((size_t)tmp.tiles * kPassBY);
        part[1].alloc((size_t)tmp.tiles * kPassBY);
        slice_res.alloc(L.n4);
        st.alloc(1);
        scratch.alloc(2 * kReduceBlocks);
        scal.alloc(8);
        flags.alloc(4);
        SSB_CUDA(cudaMallocHost(&st_host, sizeof(SorState)));
        SSB_CUDA(cudaMallocHost(&scal_host, 8 * sizeof(double)));
        SSB_CUDA(cudaMallocHost(&flags_host, 4 * sizeof(int)));
        SSB_CUDA(cudaEventCreate(&ev_a));
        SSB_CUDA(cudaEventCreate(&ev_b));
        SSB_CUDA(cudaEventCreate(&ev_c));
        SSB_CUDA(cudaEventCreate(&ev_d));
        // zero everything once: ghosts of all buffers are defined from the start
        for (auto& f : S) launch_fill(stream, L, f.pf(), 0.0);
        SSB_CUDA(cudaMemsetAsync(coef[0].p, 0, coef[0].n * sizeof(float), stream));
        SSB_CUDA(cudaMemsetAsync(coef[1].p, 0, coef[1].n * sizeof(float), stream));
        SSB_CUDA(cudaStreamSynchronize(stream));
    }
    ~Session() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        for (auto& e : graphs) {
            if (e.exec) cudaGraphExecDestroy(e.exec);
            if (e.graph) cudaGraphDestroy(e.graph);
        }
        for (auto e : ev_pool) cudaEventDestroy(e);
        for (cudaEvent_t e : {ev_a, ev_b, ev_c, ev_d})
            if (e) cudaEventDestroy(e);
        if (st_host) cudaFreeHost(st_host);
        if (scal_host) cudaFreeHost(scal_host);
        if (flags_host) cudaFreeHost(flags_host);
        if (stream) cudaStreamDestroy(stream);
        if (cap_stream) cudaStreamDestroy(cap_stream);
    }

    void sync() { SSB_CUDA(cudaStreamSynchronize(stream)); }

    double* stage_p() {
        stage.alloc(L.P);
        return stage.p;
    }
    double* stage8_p() {
        stage8.alloc(L.P * 8);
        return stage8.p;
    }

    // host padded -> S[role] (ghosts into all three state buffers)
    void upload_state(const double* host, int role) {
        double* d = stage_p();
        SSB_CUDA(cudaMemcpyAsync(d, host, L.P * sizeof(double), cudaMemcpyDefault, stream));
        const int a = (role + 1) % 3, b = (role + 2) % 3;
        launch_pack(stream, L, d, S[role].pf(), S[a].pf(), S[b].pf());
    }
    void upload_field(const double* host, PField dst) {
        double* d = stage_p();
        SSB_CUDA(cudaMemcpyAsync(d, host, L.P * sizeof(double), cudaMemcpyDefault, stream));
        PField none;
        launch_pack(stream, L, d, dst, none, none);
    }
    void download_field(PField src, double* host) {
        double* d = stage_p();
        launch_unpack(stream, L, src, d);
        SSB_CUDA(cudaMemcpyAsync(host, d, L.P * sizeof(double), cudaMemcpyDefault, stream));
    }
    void sync_ghosts_from(int role) {
        for (int r = 0; r < 3; ++r)
            if (r != role) launch_copy_ghosts(stream, L, S[r].pf(), S[role].pf());
    }

    // ------------------------------------------------------------ SOR solve
    SorArgs sor_args(const PField B[3], const PField& rhs, bool heat, double omega,
                     const double hc[4]) {
        SorArgs a{};
        a.L = L;
        for (int b = 0; b < 3; ++b)
            for (int c = 0; c < 2; ++c) a.U[b][c] = B[b].c[c];
        a.rhs[0] = rhs.c[0];
        a.rhs[1] = rhs.c[1];
        a.coef[0] = coef[0].p;
        a.coef[1] = coef[1].p;
        a.part[0] = part[0].p;
        a.part[1] = part[1].p;
        a.slice_res = slice_res.p;
        a.st = st.p;
        a.omega = omega;
        a.keep = 1.0 - omega;
        for (int q = 0; q < 4; ++q) a.hc[q] = heat ? hc[q] : 0.0;
        pass_tiles(L, a);
        a.use_cond = 0;
        return a;
    }

    cudaGraphExec_t graph_for(const SorArgs& base, const GraphKey& key, bool heat) {
        for (auto& e : graphs)
            if (e.key == key) return e.exec;
        GraphEntry e;
        e.key = key;
        SSB_CUDA(cudaGraphCreate(&e.graph, 0));
        cudaGraphConditionalHandle h;
        SSB_CUDA(cudaGraphConditionalHandleCreate(&h, e.graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        SSB_CUDA(cudaGraphAddNode(&node, e.graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        SorArgs a = base;
        a.use_cond = 1;
        a.cond = h;
        const unsigned long long saved = g_launches.load();
        SSB_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal));
        launch_sor_body(cap_stream, a, heat, nullptr);
        cudaGraph_t captured = nullptr;
        SSB_CUDA(cudaStreamEndCapture(cap_stream, &captured));
        g_launches.store(saved);
        SSB_CUDA(cudaGraphInstantiate(&e.exec, e.graph, 0));
        graphs.push_back(e);
        if (graphs.size() > 8) {  // bound the cache
            cudaGraphExecDestroy(graphs.front().exec);
            cudaGraphDestroy(graphs.front().graph);
            graphs.erase(graphs.begin());
        }
        return graphs.back().exec;
    }

    cudaEvent_t pool_event(size_t idx) {
        while (ev_pool.size() <= idx) {
            cudaEvent_t e;
            SSB_CUDA(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        return ev_pool[idx];
    }

    // Solves with guess B[0] (never written; its ghosts must equal those of
    // B[1], B[2]) and rhs `rhs` (may alias B[0]).  The iterate lands in
    // B[*result]; tolerance = tol_abs, or rel*sqrt(*norm_sq) when norm_sq
    // (device) is given.  Non-convergence is reported, not thrown: the caller
    // maps !converged to SS_ERR_NOCONVERGE (SolverError).
    SolveOut sor(const PField B[3], const PField& rhs, bool heat, double omega, const double hc[4],
                 double tol_abs, const double* norm_sq, double rel, int max_iter, bool fixed,
                 int* result) {
        launch_sor_init(stream, st.p, tol_abs, norm_sq, rel, max_iter, fixed ? 1 : 0);
        SorArgs a = sor_args(B, rhs, heat, omega, hc);
        const int limit = max_iter + 1;  // red(max_iter+1) evaluates the last residual
        if (loop_mode == 1 && !profiling) {
            GraphKey key{};
            key.heat = heat;
            for (int b = 0; b < 3; ++b)
                for (int c = 0; c < 2; ++c) key.ptr[2 * b + c] = a.U[b][c];
            key.ptr[6] = a.rhs[0];
            key.ptr[7] = a.rhs[1];
            key.omega = omega;
            for (int q = 0; q < 4; ++q) key.hc[q] = a.hc[q];
            cudaGraphExec_t ex = graph_for(a, key, heat);
            SSB_CUDA(cudaGraphLaunch(ex, stream));
            SSB_CUDA(cudaMemcpyAsync(st_host, st.p, sizeof(SorState), cudaMemcpyDeviceToHost, stream));
            sync();
            count_launch(3ull * (unsigned long long)std::min(limit, st_host->iterations + 1));
        } else {
            // host-driven: chunks of loop bodies, one chunk of look-ahead
            int launched = 0, chunk = 4;
            int* flag = flags_host;  // [2],[3] ping-pong done flags
            cudaEvent_t done_ev[2] = {ev_a, ev_b};
            int slot = 0, pending = -1;
            size_t ev_used = 0;
            std::vector<int> body_ev;  // event base index per body (profiling)
            while (launched < limit) {
                const int nb = std::min(chunk, limit - launched);
                for (int b = 0; b < nb; ++b) {
                    cudaEvent_t* ev = nullptr;
                    cudaEvent_t evs[4];
                    if (profiling) {
                        for (int q = 0; q < 4; ++q) evs[q] = pool_event(ev_used + q);
                        body_ev.push_back((int)ev_used);
                        ev_used += 4;
                        ev = evs;
                    }
                    launch_sor_body(stream, a, heat, ev);
                }
                launched += nb;
                SSB_CUDA(cudaMemcpyAsync(flag + 2 + slot, &st.p->done, sizeof(int),
                                         cudaMemcpyDeviceToHost, stream));
                SSB_CUDA(cudaEventRecord(done_ev[slot], stream));
                if (profiling) {
                    // no look-ahead while profiling: keeps the event list exact
                    SSB_CUDA(cudaEventSynchronize(done_ev[slot]));
                    if (flag[2 + slot]) break;
                } else if (pending >= 0) {
                    SSB_CUDA(cudaEventSynchronize(done_ev[pending]));
                    if (flag[2 + pending]) break;
                }
                pending = slot;
                slot ^= 1;
                chunk = std::min(chunk * 2, 64);
            }
            SSB_CUDA(cudaMemcpyAsync(st_host, st.p, sizeof(SorState), cudaMemcpyDeviceToHost, stream));
            sync();
            if (profiling) {
                const int it = st_host->iterations;
                for (size_t b = 0; b < body_ev.size(); ++b) {
                    float ms = 0.f;
                    const int base = body_ev[b];
                    if ((int)b <= it) {  // red(b+1) did real work (b+1 <= it+1)
                        SSB_CUDA(cudaEventElapsedTime(&ms, ev_pool[base], ev_pool[base + 1]));
                        prof.red_ms += ms;
                        prof.red_n++;
                    }
                    if ((int)b < it) {   // black(b+1) did real work
                        SSB_CUDA(cudaEventElapsedTime(&ms, ev_pool[base + 2], ev_pool[base + 3]));
                        prof.black_ms += ms;
                        prof.black_n++;
                    }
                }
            }
        }
        SolveOut o;
        o.iterations = st_host->iterations;
        o.residual = st_host->residual;
        o.tol = st_host->tol;
        o.converged = st_host->converged != 0;
        prof.sweeps += o.iterations;
        *result = o.iterations == 0 ? 0 : ((o.iterations & 1) ? 1 : 2);
        return o;
    }

    // ------------------------------------------------------------ kernels wrappers
    void assemble(PField u, bool with_G, double tau, double eps, double* off_out, double* diag_out,
                  double* abar_out) {
        AsmArgs a{};
        a.L = L;
        a.u[0] = u.c[0];
        a.u[1] = u.c[1];
        a.G[0] = with_G ? G[0].p : nullptr;
        a.G[1] = with_G ? G[1].p : nullptr;
        a.coef[0] = coef[0].p;
        a.coef[1] = coef[1].p;
        const double h[4] = {g.h1, g.h2, g.h3, g.h4};
        for (int q = 0; q < 4; ++q) {
            a.t_h2[q] = tau / (h[q] * h[q]);  // solver.cpp:36-38
            a.h[q] = h[q];
        }
        a.eps = eps;
        a.bad = flags.p;
        a.off_out = off_out;
        a.diag_out = diag_out;
        a.abar_out = abar_out;
        SSB_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), stream));
        launch_assemble(stream, a);
    }
    void check_assembly() {
        SSB_CUDA(cudaMemcpyAsync(flags_host, flags.p, sizeof(int), cudaMemcpyDeviceToHost, stream));
        sync();
        if (flags_host[0])
            throw Error(SS_ERR_NONFINITE, "assemble_step: non-finite coefficient (bad input field?)");
    }

    void face_coefficients(PField I0s, PField ITs, double K, double delta, double vartheta,
                           double* G_out) {
        G[0].alloc(L.cs * 8);
        G[1].alloc(L.cs * 8);
        EdgeArgs e{};
        e.L = L;
        e.I0[0] = I0s.c[0];
        e.I0[1] = I0s.c[1];
        e.IT[0] = ITs.c[0];
        e.IT[1] = ITs.c[1];
        e.G[0] = G[0].p;
        e.G[1] = G[1].p;
        e.G_out = G_out;
        e.K = K;
        e.delta = delta;
        e.vartheta = vartheta;
        e.h[0] = g.h1;
        e.h[1] = g.h2;
        e.h[2] = g.h3;
        e.h[3] = g.h4;
        launch_face_coefficients(stream, e);
        have_G = true;
    }

    static void heat_constants(const ss_grid& g, double dt, double hc[4]) {
        const double h[4] = {g.h1, g.h2, g.h3, g.h4};
        for (int a = 0; a < 4; ++a) hc[a] = (double)(float)(-(dt / (h[a] * h[a])));  // solver.cpp:89-90,107
    }

    struct SolverErrT : Error {
        int iterations;
        double residual;
        explicit SolverErrT(const SolveOut& o)
            : Error(SS_ERR_NOCONVERGE, "redblack_sor: no convergence after " +
                                           std::to_string(o.iterations) + " iterations (residual " +
                                           std::to_string(o.residual) + ")"),
              iterations(o.iterations),
              residual(o.residual) {}
    };

    // heat_smooth (preprocess.cpp:25-51) of the image in B[0], using B[1], B[2]
    // as SOR outputs.  Returns the index into B of the result (ghosts mirrored).
    int heat_smooth(PField B[3], double sigma, int steps, double omega, double tol, int max_iter) {
        if (sigma == 0.0) {
            launch_mirror_ghosts(stream, L, B[0]);
            return 0;
        }
        const double dt = 0.5 * sigma * sigma / steps;
        double hc[4];
        heat_constants(g, dt, hc);
        // the SOR buffers' ghosts = the input's (they only meet zero couplings)
        launch_copy_ghosts(stream, L, B[1], B[0]);
        launch_copy_ghosts(stream, L, B[2], B[0]);
        int idx[3] = {0, 1, 2};
        for (int s = 0; s < steps; ++s) {
            const PField T[3] = {B[idx[0]], B[idx[1]], B[idx[2]]};
            int r = 0;
            const SolveOut o = sor(T, T[0], true, omega, hc, tol, nullptr, 0.0, max_iter, false, &r);
            if (!o.converged) throw SolverErrT(o);
            const int nidx[3] = {idx[r], idx[(r + 1) % 3], idx[(r + 2) % 3]};
            std::memcpy(idx, nidx, sizeof idx);
        }
        launch_mirror_ghosts(stream, L, B[idx[0]]);
        return idx[0];
    }

    void rescale(int role) {
        if (!rescale_balls.count()) return;
        for (int w = 0; w < rescale_balls.waves(); ++w) {
            const int o = rescale_balls.wave_off[w], n = rescale_balls.wave_off[w + 1] - o;
            launch_rescale(stream, L, S[role].pf(), rescale_balls.dev.p + o, n);
        }
    }

    // local_threshold (preprocess.cpp:53-102): img -> out
    void threshold(PField img, PField out, const ss_center* c, int n, double lambda,
                   double background) {
        BallSet bs;
        build_balls(bs, g, c, n, 0.0, false);
        launch_fill(stream, L, out, background);
        if (!bs.count()) return;
        Dev<double> ab;
        ab.alloc(2 * (size_t)bs.count());
        SSB_CUDA(cudaMemsetAsync(flags.p + 1, 0x7f, sizeof(int), stream));
        launch_ball_minmax(stream, L, img, bs.dev.p, bs.count(), ab.p, flags.p + 1);
        SSB_CUDA(cudaMemcpyAsync(flags_host + 1, flags.p + 1, sizeof(int), cudaMemcpyDeviceToHost, stream));
        sync();
        if (flags_host[1] != 0x7f7f7f7f) {
            // report the first offending row in table order
            int first = INT_MAX;
            std::vector<double> h(2 * bs.count());
            SSB_CUDA(cudaMemcpy(h.data(), ab.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
            for (int b = 0; b < bs.count(); ++b)
                if (h[2 * b] > h[2 * b + 1]) first = std::min(first, bs.row[b]);
            throw Error(SS_ERR_VALIDATION, "local_threshold: ball in centers row " +
                                               std::to_string(first + 1) + " covers no doxels");
        }
        for (int w = 0; w < bs.waves(); ++w) {
            const int o = bs.wave_off[w], m = bs.wave_off[w + 1] - o;
            launch_threshold_write(stream, L, img, out, bs.dev.p + o, m, ab.p + 2 * o, lambda);
        }
        sync();  // ab / bs are freed on return
    }

    void initial(PField u, const ss_center* c, int n, double v, double R, int profile) {
        BallSet bs;
        build_balls(bs, g, c, n, R, true);
        launch_fill(stream, L, u, 0.0);
        for (int w = 0; w < bs.waves(); ++w) {
            const int o = bs.wave_off[w], m = bs.wave_off[w + 1] - o;
            launch_initial(stream, L, u, bs.dev.p + o, m, v, R, profile);
        }
        sync();
    }

    // ------------------------------------------------------------ segment()
    void prepare(const double* image, const ss_center* c, int n, const ss_seg_params& p,
                 const double* u0) {
        validate_solver(p.tau, p.epsilon, p.omega, p.sor_tol, p.sor_max_iter, p.n_steps);
        validate_smoothing(p.sigma, p.smooth_steps, p.smooth_tol, p.smooth_max_iter, p.smooth_omega);
        require(!(p.lambda < 0.0 || p.lambda > 1.0), "ThresholdParams: lambda must be in [0,1]");
        validate_edge(p.K, p.delta, p.vartheta);
        require(p.init_v > 0.0, "InitParams: v must be > 0");
        require(p.init_R > 0.0, "InitParams: R must be > 0");
        validate_centers(g, c, n);
        prepared = false;
        prm = p;
        build_balls(rescale_balls, g, c, n, p.rescale_radius, false);

        // u0 (solver.cpp:416-417)
        cur = 0;
        if (u0) {
            upload_state(u0, cur);
        } else {
            initial(S[cur].pf(), c, n, p.init_v, p.init_R, p.init_profile);
            sync_ghosts_from(cur);
        }
        rescale(cur);

        // image, thresholded image, heat smoothing, G (solver.cpp:419-422)
        DevField img, th, t1, t2;
        img.alloc(L);
        th.alloc(L);
        t1.alloc(L);
        t2.alloc(L);
        upload_field(image, img.pf());
        threshold(img.pf(), th.pf(), c, n, p.lambda, p.background);
        PField b1[3] = {img.pf(), t1.pf(), t2.pf()};
        const int r1 = heat_smooth(b1, p.sigma, p.smooth_steps, p.smooth_omega, p.smooth_tol,
                                   p.smooth_max_iter);
        const PField I0s = b1[r1];
        PField b2[3] = {th.pf(), b1[(r1 + 1) % 3], b1[(r1 + 2) % 3]};
        const int r2 = heat_smooth(b2, p.sigma, p.smooth_steps, p.smooth_omega, p.smooth_tol,
                                   p.smooth_max_iter);
        const PField ITs = b2[r2];
        face_coefficients(I0s, ITs, p.K, p.delta, p.vartheta, nullptr);
        sync();

        // apply_dirichlet(u, 0) (solver.cpp:425) on every state buffer
        for (auto& f : S) launch_set_ghosts(stream, L, f.pf(), 0.0);
        sync();
        prepared = true;
    }

    void step(ss_step_diag* diag) {
        if (!prepared) throw Error(SS_ERR_STATE, "session not prepared");
        const int roles[3] = {cur, (cur + 1) % 3, (cur + 2) % 3};
        if (profiling) SSB_CUDA(cudaEventRecord(ev_c, stream));
        assemble(S[cur].pf(), have_G, prm.tau, prm.epsilon, nullptr, nullptr, nullptr);
        if (profiling) SSB_CUDA(cudaEventRecord(ev_d, stream));
        const bool rel = prm.sor_rel_tol > 0.0;
        if (rel) launch_norm_sq(stream, L, S[cur].pf(), scratch.p, scal.p);
        check_assembly();
        if (profiling) {
            float ms = 0.f;
            SSB_CUDA(cudaEventElapsedTime(&ms, ev_c, ev_d));
            prof.assemble_ms += ms;
            prof.assemble_n++;
        }
        const PField B[3] = {S[roles[0]].pf(), S[roles[1]].pf(), S[roles[2]].pf()};
        int rr = 0;
        const SolveOut o = sor(B, B[0], false, prm.omega, nullptr, prm.sor_tol,
                               rel ? scal.p : nullptr, prm.sor_rel_tol, prm.sor_max_iter, false, &rr);
        if (!o.converged) throw SolverErrT(o);
        cur = roles[rr];
        if (prm.rescale_each_step) {
            if (profiling) SSB_CUDA(cudaEventRecord(ev_c, stream));
            rescale(cur);
            if (profiling) SSB_CUDA(cudaEventRecord(ev_d, stream));
        }
        if (diag) {
            launch_minmax(stream, L, S[cur].pf(), scratch.p, scal.p + 1);
            SSB_CUDA(cudaMemcpyAsync(scal_host + 1, scal.p + 1, 2 * sizeof(double),
                                     cudaMemcpyDeviceToHost, stream));
        }
        sync();
        if (profiling && prm.rescale_each_step) {
            float ms = 0.f;
            SSB_CUDA(cudaEventElapsedTime(&ms, ev_c, ev_d));
            prof.rescale_ms += ms;
            prof.rescale_n++;
        }
        if (diag) {
            diag->iterations = o.iterations;
            diag->residual = o.residual;
            diag->tol = o.tol;
            diag->umin = scal_host[1];
            diag->umax = scal_host[2];
        }
    }

    double fixed_sweeps(int n_sweeps) {
        if (!prepared) throw Error(SS_ERR_STATE, "session not prepared");
        const int roles[3] = {cur, (cur + 1) % 3, (cur + 2) % 3};
        assemble(S[cur].pf(), have_G, prm.tau, prm.epsilon, nullptr, nullptr, nullptr);
        check_assembly();
        const PField B[3] = {S[roles[0]].pf(), S[roles[1]].pf(), S[roles[2]].pf()};
        int rr = 0;
        const SolveOut o = sor(B, B[0], false, prm.omega, nullptr, 1.0, nullptr, 0.0, n_sweeps,
                               true, &rr);
        cur = roles[rr];
        return o.residual;
    }
};

// ------------------------------------------------------------------ session cache (per-call API)
static std::unique_ptr<Session> g_cached;

static bool same_grid(const ss_grid& a, const ss_grid& b) {
    return a.n1 == b.n1 && a.n2 == b.n2 && a.n3 == b.n3 && a.n4 == b.n4 && a.h1 == b.h1 &&
           a.h2 == b.h2 && a.h3 == b.h3 && a.h4 == b.h4;
}

static void require_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n < 1)
        throw Error(SS_ERR_CUDA, std::string("no usable CUDA device (") +
                                     (e != cudaSuccess ? cudaGetErrorString(e) : "count 0") +
                                     "); this library has no CPU fallback");
}

static Session& cached_session(const ss_grid& g) {
    require_device();
    if (!g_cached || !same_grid(g_cached->g, g)) {
        g_cached.reset();
        int dev = 0;
        SSB_CUDA(cudaGetDevice(&dev));
        g_cached.reset(new Session(g, dev));
    }
    return *g_cached;
}

template <class F>
static ss_status guard(F&& fn) {
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

}  // namespace ssb

using namespace ssb;

struct ss_session {
    std::unique_ptr<Session> s;
};

extern "C" {

const char* ss_last_error(void) { return t_err.c_str(); }
int ss_abi_version(void) { return 1; }
unsigned long long ss_launch_count(void) { return g_launches.load(); }

int ss_device_available(void) {
    const ss_status st = guard([] { require_device(); });
    return st == SS_OK ? 1 : 0;
}

double ss_sor_pass_bytes(const ss_grid* g) {
    // SURVEY.md 8(d) contract figure: 56 B per interior doxel per red+black sweep
    // (8 fp32 coefficients + rhs + u read + u write); one colour pass = half.
    const double N = (double)g->n1 * g->n2 * g->n3 * g->n4;
    return 0.5 * N * 56.0;
}

ss_status ss_assemble_step(const ss_grid* g, const double* u_prev, const double* G, double tau,
                           double epsilon, double* offdiag, double* diag, double* abar) {
    return guard([&] {
        validate_grid(g);
        validate_solver(tau, epsilon, 1.0, 1.0, 1, 1);
        Session& s = cached_session(*g);
        s.upload_state(u_prev, s.cur);
        if (G) {
            double* d8 = s.stage8_p();
            SSB_CUDA(cudaMemcpyAsync(d8, G, s.L.P * 8 * sizeof(double), cudaMemcpyDefault, s.stream));
            s.G[0].alloc(s.L.cs * 8);
            s.G[1].alloc(s.L.cs * 8);
            launch_pack8(s.stream, s.L, d8, s.G[0].p, s.G[1].p);
        }
        // export buffers: off (8P) in stage8 after G was packed, diag/abar in scratch fields
        double* off = s.stage8_p();
        Dev<double> dg, ab;
        dg.alloc(s.L.P);
        ab.alloc(s.L.P);
        SSB_CUDA(cudaMemsetAsync(off, 0, s.L.P * 8 * sizeof(double), s.stream));
        SSB_CUDA(cudaMemsetAsync(dg.p, 0, s.L.P * sizeof(double), s.stream));
        SSB_CUDA(cudaMemsetAsync(ab.p, 0, s.L.P * sizeof(double), s.stream));
        s.assemble(s.S[s.cur].pf(), G != nullptr, tau, epsilon, off, dg.p, ab.p);
        SSB_CUDA(cudaMemcpyAsync(offdiag, off, s.L.P * 8 * sizeof(double), cudaMemcpyDefault, s.stream));
        SSB_CUDA(cudaMemcpyAsync(diag, dg.p, s.L.P * sizeof(double), cudaMemcpyDefault, s.stream));
        SSB_CUDA(cudaMemcpyAsync(abar, ab.p, s.L.P * sizeof(double), cudaMemcpyDefault, s.stream));
        s.check_assembly();
        s.have_G = false;
        s.prepared = false;
    });
}

ss_status ss_assemble_heat_step(const ss_grid* g, double dt, double* offdiag, double* diag,
                                double* abar) {
    return guard([&] {
        validate_grid(g);
        require(dt > 0.0, "assemble_heat_step: dt must be > 0");
        Session& s = cached_session(*g);
        double hc[4];
        Session::heat_constants(*g, dt, hc);
        double* off = s.stage8_p();
        Dev<double> dg, ab;
        dg.alloc(s.L.P);
        ab.alloc(s.L.P);
        launch_heat_export(s.stream, s.L, hc, off, dg.p, ab.p);
        SSB_CUDA(cudaMemcpyAsync(offdiag, off, s.L.P * 8 * sizeof(double), cudaMemcpyDefault, s.stream));
        SSB_CUDA(cudaMemcpyAsync(diag, dg.p, s.L.P * sizeof(double), cudaMemcpyDefault, s.stream));
        SSB_CUDA(cudaMemcpyAsync(abar, ab.p, s.L.P * sizeof(double), cudaMemcpyDefault, s.stream));
        s.sync();
    });
}

ss_status ss_redblack_sor(const ss_grid* g, const double* offdiag, const double* rhs, double* u,
                          double omega, double sor_tol, int sor_max_iter, int workers,
                          int* iterations, double* residual) {
    if (iterations) *iterations = 0;
    if (residual) *residual = 0.0;
    return guard([&] {
        validate_grid(g);
        validate_solver(1.0, 1.0, omega, sor_tol, sor_max_iter, 1);
        require(workers >= 1, "Partition: worker count must be >= 1");
        Session& s = cached_session(*g);
        s.prepared = false;
        double* d8 = s.stage8_p();
        SSB_CUDA(cudaMemcpyAsync(d8, offdiag, s.L.P * 8 * sizeof(double), cudaMemcpyDefault, s.stream));
        launch_pack_coef(s.stream, s.L, d8, s.coef[0].p, s.coef[1].p);
        s.rhs_sep.alloc(s.L);
        s.upload_field(rhs, s.rhs_sep.pf());
        s.cur = 0;
        s.upload_state(u, 0);
        const PField B[3] = {s.S[0].pf(), s.S[1].pf(), s.S[2].pf()};
        int rr = 0;
        const SolveOut o = s.sor(B, s.rhs_sep.pf(), false, omega, nullptr, sor_tol, nullptr, 0.0,
                                 sor_max_iter, false, &rr);
        s.download_field(s.S[rr].pf(), u);
        s.sync();
        if (iterations) *iterations = o.iterations;
        if (residual) *residual = o.residual;
        if (!o.converged) throw Session::SolverErrT(o);
    });
}

ss_status ss_face_coefficients(const ss_grid* g, const double* I0s, const double* ITs, double K,
                               double delta, double vartheta, double* G) {
    return guard([&] {
        validate_grid(g);
        validate_edge(K, delta, vartheta);
        Session& s = cached_session(*g);
        s.prepared = false;
        DevField a, b;
        a.alloc(s.L);
        b.alloc(s.L);
        s.upload_field(I0s, a.pf());
        s.upload_field(ITs, b.pf());
        double* out = s.stage8_p();
        launch_fill_raw(s.stream, out, s.L.P * 8, 1.0);  // ghost entries = 1 (edge.hpp:73)
        s.face_coefficients(a.pf(), b.pf(), K, delta, vartheta, out);
        SSB_CUDA(cudaMemcpyAsync(G, out, s.L.P * 8 * sizeof(double), cudaMemcpyDefault, s.stream));
        s.sync();
    });
}

ss_status ss_heat_smooth(const ss_grid* g, const double* image, double sigma, int steps,
                         double omega, double sor_tol, int sor_max_iter, double* out) {
    return guard([&] {
        validate_grid(g);
        validate_smoothing(sigma, steps, sor_tol, sor_max_iter, omega);
        Session& s = cached_session(*g);
        s.prepared = false;
        DevField a, b, c;
        a.alloc(s.L);
        b.alloc(s.L);
        c.alloc(s.L);
        s.upload_field(image, a.pf());
        PField B[3] = {a.pf(), b.pf(), c.pf()};
        const int r = s.heat_smooth(B, sigma, steps, omega, sor_tol, sor_max_iter);
        s.download_field(B[r], out);
        s.sync();
    });
}

ss_status ss_local_threshold(const ss_grid* g, const double* image, const ss_center* c, int n,
                             double lambda, double background, double* out) {
    return guard([&] {
        validate_grid(g);
        require(!(lambda < 0.0 || lambda > 1.0), "ThresholdParams: lambda must be in [0,1]");
        validate_centers(*g, c, n);
        Session& s = cached_session(*g);
        s.prepared = false;
        DevField a, b;
        a.alloc(s.L);
        b.alloc(s.L);
        s.upload_field(image, a.pf());
        s.threshold(a.pf(), b.pf(), c, n, lambda, background);
        s.download_field(b.pf(), out);
        s.sync();
    });
}

ss_status ss_build_initial(const ss_grid* g, const ss_center* c, int n, double v, double R,
                           int profile, double* u) {
    return guard([&] {
        validate_grid(g);
        require(v > 0.0, "InitParams: v must be > 0");
        require(R > 0.0, "InitParams: R must be > 0");
        validate_centers(*g, c, n);
        Session& s = cached_session(*g);
        s.prepared = false;
        DevField a;
        a.alloc(s.L);
        s.initial(a.pf(), c, n, v, R, profile);
        s.download_field(a.pf(), u);
        s.sync();
    });
}

ss_status ss_local_rescale(const ss_grid* g, double* u, const ss_center* c, int n, double radius) {
    return guard([&] {
        validate_grid(g);
        validate_centers(*g, c, n);
        Session& s = cached_session(*g);
        s.prepared = false;
        build_balls(s.rescale_balls, *g, c, n, radius, false);
        s.cur = 0;
        s.upload_state(u, 0);
        s.rescale(0);
        s.download_field(s.S[0].pf(), u);
        s.sync();
    });
}

ss_status ss_apply_dirichlet(const ss_grid* g, double* f, double value) {
    return guard([&] {
        validate_grid(g);
        require(f != nullptr, "null field");
        Session& s = cached_session(*g);
        s.prepared = false;
        s.upload_field(f, s.S[0].pf());
        launch_set_ghosts(s.stream, s.L, s.S[0].pf(), value);
        s.download_field(s.S[0].pf(), f);
        s.sync();
    });
}

ss_status ss_apply_mirror_ghosts(const ss_grid* g, double* f) {
    return guard([&] {
        validate_grid(g);
        require(f != nullptr, "null field");
        Session& s = cached_session(*g);
        s.prepared = false;
        s.upload_field(f, s.S[0].pf());
        launch_mirror_ghosts(s.stream, s.L, s.S[0].pf());
        s.download_field(s.S[0].pf(), f);
        s.sync();
    });
}

ss_status ss_interior_minmax(const ss_grid* g, const double* f, double* lo, double* hi) {
    return guard([&] {
        validate_grid(g);
        require(f && lo && hi, "null argument");
        Session& s = cached_session(*g);
        s.prepared = false;
        s.upload_field(f, s.S[0].pf());
        launch_minmax(s.stream, s.L, s.S[0].pf(), s.scratch.p, s.scal.p + 1);
        SSB_CUDA(cudaMemcpyAsync(s.scal_host + 1, s.scal.p + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                 s.stream));
        s.sync();
        *lo = s.scal_host[1];
        *hi = s.scal_host[2];
    });
}

ss_status ss_extract_mask(const ss_grid* g, const double* u, double level, uint8_t* mask) {
    return guard([&] {
        validate_grid(g);
        Session& s = cached_session(*g);
        s.prepared = false;
        s.cur = 0;
        s.upload_state(u, 0);
        const size_t N = (size_t)g->n1 * g->n2 * g->n3 * g->n4;
        Dev<uint8_t> m;
        m.alloc(N);
        launch_mask(s.stream, s.L, s.S[0].pf(), level, m.p);
        SSB_CUDA(cudaMemcpyAsync(mask, m.p, N, cudaMemcpyDefault, s.stream));
        s.sync();
    });
}

ss_status ss_segment(const ss_grid* g, const double* image, const ss_center* c, int n,
                     const ss_seg_params* p, const double* u0, double* u_out, ss_step_diag* diags) {
    return guard([&] {
        validate_grid(g);
        require(p != nullptr, "null params");
        Session& s = cached_session(*g);
        s.prepare(image, c, n, *p, u0);
        for (int step = 0; step < p->n_steps; ++step) s.step(diags ? diags + step : nullptr);
        s.download_field(s.S[s.cur].pf(), u_out);
        s.sync();
        s.prepared = false;
    });
}

ss_status ss_session_create(const ss_grid* g, int device, ss_session** out) {
    return guard([&] {
        validate_grid(g);
        require(out != nullptr, "null output pointer");
        require_device();
        *out = nullptr;
        std::unique_ptr<ss_session> h(new ss_session);
        h->s.reset(new Session(*g, device));
        *out = h.release();
    });
}

ss_status ss_session_destroy(ss_session* s) {
    return guard([&] { delete s; });
}

void* ss_session_stream(ss_session* s) { return s ? (void*)s->s->stream : nullptr; }

ss_status ss_session_prepare(ss_session* s, const double* image, const ss_center* c, int n,
                             const ss_seg_params* p, const double* u0) {
    return guard([&] {
        require(s && p, "null session / params");
        SSB_CUDA(cudaSetDevice(s->s->device));
        s->s->prepare(image, c, n, *p, u0);
    });
}

ss_status ss_session_step(ss_session* s, ss_step_diag* diag) {
    return guard([&] {
        require(s != nullptr, "null session");
        SSB_CUDA(cudaSetDevice(s->s->device));
        s->s->step(diag);
    });
}

ss_status ss_session_set_u(ss_session* s, const double* host_u) {
    return guard([&] {
        require(s && host_u, "null session / buffer");
        Session& x = *s->s;
        SSB_CUDA(cudaSetDevice(x.device));
        x.upload_state(host_u, x.cur);
    });
}

ss_status ss_session_get_u(ss_session* s, double* host_u) {
    return guard([&] {
        require(s && host_u, "null session / buffer");
        Session& x = *s->s;
        SSB_CUDA(cudaSetDevice(x.device));
        x.download_field(x.S[x.cur].pf(), host_u);
        x.sync();
    });
}

ss_status ss_session_get_mask(ss_session* s, double level, uint8_t* mask) {
    return guard([&] {
        require(s && mask, "null session / buffer");
        Session& x = *s->s;
        SSB_CUDA(cudaSetDevice(x.device));
        const size_t N = (size_t)x.g.n1 * x.g.n2 * x.g.n3 * x.g.n4;
        Dev<uint8_t> m;
        m.alloc(N);
        launch_mask(x.stream, x.L, x.S[x.cur].pf(), level, m.p);
        SSB_CUDA(cudaMemcpyAsync(mask, m.p, N, cudaMemcpyDefault, x.stream));
        x.sync();
    });
}

ss_status ss_session_fixed_sweeps(ss_session* s, int n_sweeps, double* residual) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(n_sweeps >= 1, "n_sweeps must be >= 1");
        SSB_CUDA(cudaSetDevice(s->s->device));
        const double r = s->s->fixed_sweeps(n_sweeps);
        if (residual) *residual = r;
    });
}

ss_status ss_session_set_loop_mode(ss_session* s, int mode) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(mode == 0 || mode == 1, "loop mode must be 0 or 1");
        s->s->loop_mode = mode;
    });
}

ss_status ss_session_set_profiling(ss_session* s, int enable) {
    return guard([&] {
        require(s != nullptr, "null session");
        s->s->profiling = enable != 0;
    });
}

ss_status ss_session_profile(ss_session* s, ss_profile* out) {
    return guard([&] {
        require(s && out, "null session / output");
        *out = s->s->prof;
        s->s->prof = ss_profile{};
    });
}

}  // extern "C"
