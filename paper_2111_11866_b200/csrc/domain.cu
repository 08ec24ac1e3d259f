// domain.cu -- slabs, the in-process transport and the device-resident
// segment() domain (solver.cpp:405-441) with its red-black SOR driver
// (solver.cpp:124-397).  See domain.cuh for the structure.
#include "domain.cuh"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <cstring>

namespace ssb {

std::atomic<unsigned long long> g_launches{0};

// ------------------------------------------------------------------ validation
// (solver.cpp:13-21, preprocess.cpp:11-23, edge.cpp:9-14, seedinit.cpp:9-12, io.cpp:128-140)
void require(bool ok, const std::string& msg) {
    if (!ok) throw Error(SS_ERR_VALIDATION, msg);
}
void validate_grid(const ss_grid* g) {
    require(g != nullptr, "null grid");
    require(g->n1 >= 1 && g->n2 >= 1 && g->n3 >= 1 && g->n4 >= 1, "GridSpec: doxel counts must be >= 1");
    require(g->h1 > 0.0 && g->h2 > 0.0 && g->h3 > 0.0 && g->h4 > 0.0, "GridSpec: spacings must be > 0");
}
void validate_solver(double tau, double eps, double omega, double tol, int max_iter, int n_steps) {
    require(!(tau < 0.0), "SolverParams: tau must be >= 0");
    require(eps > 0.0, "SolverParams: epsilon must be > 0");
    require(omega > 0.0 && omega < 2.0, "SolverParams: omega must lie in (0,2)");
    require(tol > 0.0, "SolverParams: sor_tol must be > 0");
    require(max_iter >= 1, "SolverParams: sor_max_iter must be >= 1");
    require(n_steps >= 1, "SolverParams: n_steps must be >= 1");
}
void validate_smoothing(double sigma, int steps, double tol, int max_iter, double omega) {
    require(!(sigma < 0.0), "SmoothingParams: sigma must be >= 0");
    require(steps >= 1, "SmoothingParams: steps must be >= 1");
    require(tol > 0.0, "SmoothingParams: sor_tol must be > 0");
    require(max_iter >= 1, "SmoothingParams: sor_max_iter must be >= 1");
    require(omega > 0.0 && omega < 2.0, "SmoothingParams: omega must lie in (0,2)");
}
void validate_edge(double K, double delta, double vartheta) {
    require(!(K < 0.0), "EdgeParams: K must be >= 0");
    require(!(delta < 0.0 || delta > 1.0), "EdgeParams: delta must be in [0,1]");
    require(!(vartheta < 0.0 || vartheta > 1.0), "EdgeParams: vartheta must be in [0,1]");
}
void validate_centers(const ss_grid& g, const ss_center* c, int n) {
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
void validate_seg_params(const ss_seg_params& p) {
    validate_solver(p.tau, p.epsilon, p.omega, p.sor_tol, p.sor_max_iter, p.n_steps);
    validate_smoothing(p.sigma, p.smooth_steps, p.smooth_tol, p.smooth_max_iter, p.smooth_omega);
    require(!(p.lambda < 0.0 || p.lambda > 1.0), "ThresholdParams: lambda must be in [0,1]");
    validate_edge(p.K, p.delta, p.vartheta);
    require(p.init_v > 0.0, "InitParams: v must be > 0");
    require(p.init_R > 0.0, "InitParams: R must be > 0");
}

SolverErrT::SolverErrT(const SolveOut& o)
    : Error(SS_ERR_NOCONVERGE, "redblack_sor: no convergence after " + std::to_string(o.iterations) +
                                   " iterations (residual " + std::to_string(o.residual) + ")"),
      iterations(o.iterations),
      residual(o.residual) {}

// ------------------------------------------------------------------ balls
// Bounds exactly as seedinit.cpp:22-31 / preprocess.cpp:63-68 (on global coordinates).
static Ball make_ball(const ss_grid& g, const ss_center& c, double r, int l0) {
    Ball b{};
    b.l = c.frame + 1 - l0;
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
    return a.l == b.l && a.i0 <= b.i1 && b.i0 <= a.i1 && a.j0 <= b.j1 && b.j0 <= a.j1 && a.k0 <= b.k1 &&
           b.k0 <= a.k1;
}

// Waves: a ball's wave is one past the latest wave of any EARLIER ball whose
// index box meets its own (same frame), so sequential table order is kept
// wherever it matters and disjoint balls run concurrently.
void build_balls(BallSet& bs, const ss_grid& gl, int l0, const ss_center* c, int n, double radius,
                 bool fixed_radius) {
    std::vector<Ball> table;
    std::vector<int> rows;
    for (int m = 0; m < n; ++m) {
        if (c[m].frame + 1 - l0 < 1 || c[m].frame + 1 - l0 > gl.n4) continue;  // other slab
        table.push_back(make_ball(gl, c[m], fixed_radius || !std::isnan(radius) ? radius : c[m].radius, l0));
        rows.push_back(m);
    }
    const int nb = (int)table.size();
    std::vector<int> wave(nb, 0);
    int nw = 0;
    for (int b = 0; b < nb; ++b) {
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
        for (int b = 0; b < nb; ++b)
            if (wave[b] == w) {
                bs.host.push_back(table[b]);
                bs.row.push_back(rows[b]);
            }
        bs.wave_off.push_back((int)bs.host.size());
    }
    bs.dev.alloc(std::max<size_t>(1, bs.host.size()));
    if (!bs.host.empty())
        SSB_CUDA(cudaMemcpy(bs.dev.p, bs.host.data(), bs.host.size() * sizeof(Ball), cudaMemcpyHostToDevice));
}

// ------------------------------------------------------------------ slab
Slab::~Slab() {
    for (auto& e : map_cache) cudaFree(e.dev);
}

Slab::Slab(const ss_grid& global, int l0, int n4_local, int idx, int chunk, int world, cudaStream_t s)
    : index(idx), stream(s) {
    gl = global;
    gl.n4 = n4_local;
    L = Layout::make(gl, l0, global.n4);
    for (auto& f : S) f.alloc(L);
    coef[0].alloc(L.rows * L.Wc * 8);
    coef[1].alloc(L.rows * L.Wc * 8);
    SorArgs t{};
    pass_tiles(L, t);
    const size_t nparts = std::max({(size_t)t.tiles * kPassBY, tma_partials(L), resident_partials(L),
                                    kwave_supported(L) ? kwave_partials(L) : (size_t)0});
    for (auto& pp : part) {
        pp[0].alloc(nparts);
        pp[1].alloc(nparts);
    }
    slice_res.alloc(chunk);
    norm_loc.alloc(chunk);
    norm_part.alloc((size_t)chunk * kNormChunks);
    if (world > 1) {
        bad_all.alloc(world);
        all_slices.alloc((size_t)world * chunk);
        norm_all.alloc((size_t)world * chunk);
        SSB_CUDA(cudaMemsetAsync(all_slices.p, 0, all_slices.n * sizeof(double), stream));
        SSB_CUDA(cudaMemsetAsync(norm_all.p, 0, norm_all.n * sizeof(double), stream));
    }
    gloc.alloc(8);
    gall.alloc((size_t)world * 8);
    if (world == 1 && (wave_supported(L) || kwave_supported(L))) {
        wflags.alloc(std::max(wave_supported(L) ? wave_flags(L) : (size_t)0,
                              kwave_supported(L) ? kwave_flags(L) : (size_t)0));
        SSB_CUDA(cudaMemsetAsync(wflags.p, 0, wflags.n * sizeof(int), stream));
    }
    SSB_CUDA(cudaMemsetAsync(slice_res.p, 0, slice_res.n * sizeof(double), stream));
    SSB_CUDA(cudaMemsetAsync(norm_loc.p, 0, norm_loc.n * sizeof(double), stream));
    st.alloc(1);
    scratch.alloc(2 * kReduceBlocks);
    scal.alloc(8);
    flags.alloc(4);
    // zero everything once: ghosts and halos of all buffers are defined from the start
    for (auto& f : S) launch_fill(stream, L, f.pf(), 0.0);
    SSB_CUDA(cudaMemsetAsync(coef[0].p, 0, coef[0].n * sizeof(float), stream));
    SSB_CUDA(cudaMemsetAsync(coef[1].p, 0, coef[1].n * sizeof(float), stream));
}

double* Slab::stage_p() {
    stage.alloc(L.P);
    return stage.p;
}

double* Slab::dstage_p() {
    dstage.alloc(L.P);
    return dstage.p;
}
double* Slab::stage8_p() {
    stage8.alloc(L.P * 8);
    return stage8.p;
}

void Slab::upload(const double* host, PField dst, PField t0, PField t1, PField t2) {
    double* d = stage_p();
    copy_h2d(d, host, L.P * sizeof(double), stream);
    launch_pack(stream, L, d, dst, t0, t1, t2);
}

void Slab::upload_state(const double* host, int role) {
    upload(host, S[role].pf(), S[(role + 1) % kStateBuffers].pf(), S[(role + 2) % kStateBuffers].pf(),
           S[(role + 3) % kStateBuffers].pf());
}

void Slab::download(PField src, double* host) {
    double* d = stage_p();
    launch_unpack(stream, L, src, d);
    copy_d2h(host, d, L.P * sizeof(double), stream);
}

void Slab::sync_ghosts_from(int role) {
    for (int r = 0; r < kStateBuffers; ++r)
        if (r != role) launch_copy_ghosts(stream, L, S[r].pf(), S[role].pf());
}

AsmArgs Slab::asm_args(PField u, bool with_G, double tau, double eps) const {
    AsmArgs a{};
    a.L = L;
    a.u[0] = u.c[0];
    a.u[1] = u.c[1];
    a.G[0] = with_G ? G[0].p : nullptr;
    a.G[1] = with_G ? G[1].p : nullptr;
    a.coef[0] = coef[0].p;
    a.coef[1] = coef[1].p;
    const double h[4] = {gl.h1, gl.h2, gl.h3, gl.h4};
    for (int q = 0; q < 4; ++q) {
        a.t_h2[q] = tau / (h[q] * h[q]);  // solver.cpp:36-38
        a.h[q] = h[q];
    }
    a.eps = eps;
    a.bad = flags.p;
    a.guard = flags.p + 2;  // the tile kernel's range guard: flags[2] out of range, flags[3] max |u| high word
    return a;
}

void Slab::assemble(PField u, bool with_G, double tau, double eps, double* off_out, double* diag_out,
                    double* abar_out) {
    AsmArgs a{};
    a.L = L;
    a.u[0] = u.c[0];
    a.u[1] = u.c[1];
    a.G[0] = with_G ? G[0].p : nullptr;
    a.G[1] = with_G ? G[1].p : nullptr;
    a.coef[0] = coef[0].p;
    a.coef[1] = coef[1].p;
    const double h[4] = {gl.h1, gl.h2, gl.h3, gl.h4};
    for (int q = 0; q < 4; ++q) {
        a.t_h2[q] = tau / (h[q] * h[q]);  // solver.cpp:36-38
        a.h[q] = h[q];
    }
    a.eps = eps;
    a.bad = flags.p;
    a.guard = flags.p + 2;  // the tile kernel's range guard: flags[2] out of range, flags[3] max |u| high word (flags[1]: threshold)
    a.off_out = off_out;
    a.diag_out = diag_out;
    a.abar_out = abar_out;
    SSB_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int), stream));
    launch_assemble(stream, a);
}

void Slab::face_coefficients(PField I0s, PField ITs, double K, double delta, double vartheta,
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
    e.h[0] = gl.h1;
    e.h[1] = gl.h2;
    e.h[2] = gl.h3;
    e.h[3] = gl.h4;
    e.guard = flags.p + 2;  // the scaled gradients' range guard (reset by every assembly before use)
    launch_face_coefficients(stream, e);
    have_G = true;
}

void Slab::rescale(int role) {
    for (int w = 0; w < rescale_balls.waves(); ++w) {
        const int o = rescale_balls.wave_off[w], n = rescale_balls.wave_off[w + 1] - o;
        launch_rescale(stream, L, S[role].pf(), rescale_balls.dev.p + o, n);
    }
}

void Slab::threshold_minmax(PField img, const BallSet& bs, double* ab) {
    SSB_CUDA(cudaMemsetAsync(flags.p + 1, 0x7f, sizeof(int), stream));
    launch_ball_minmax(stream, L, img, bs.dev.p, bs.count(), ab, flags.p + 1);
}

void Slab::threshold_write(PField img, PField out, const BallSet& bs, const double* ab, double lambda) {
    for (int w = 0; w < bs.waves(); ++w) {
        const int o = bs.wave_off[w], m = bs.wave_off[w + 1] - o;
        launch_threshold_write(stream, L, img, out, bs.dev.p + o, m, ab + 2 * o, lambda);
    }
}

void Slab::initial(PField u, const ss_center* c, int n, double v, double R, int profile) {
    BallSet bs;
    build_balls(bs, gl, L.l0, c, n, R, true);
    launch_fill(stream, L, u, 0.0);
    for (int w = 0; w < bs.waves(); ++w) {
        const int o = bs.wave_off[w], m = bs.wave_off[w + 1] - o;
        launch_initial(stream, L, u, bs.dev.p + o, m, v, R, profile);
    }
    SSB_CUDA(cudaStreamSynchronize(stream));  // bs is freed on return
}

SorArgs Slab::sor_args(const PField B[kStateBuffers], const PField& rhs, bool heat, double omega, const double hc[4],
                       int world, int kernel) const {
    SorArgs a{};
    a.L = L;
    for (int b = 0; b < kStateBuffers; ++b)
        for (int c = 0; c < 2; ++c) a.U[b][c] = B[b].c[c];
    a.rhs[0] = rhs.c[0];
    a.rhs[1] = rhs.c[1];
    a.coef[0] = coef[0].p;
    a.coef[1] = coef[1].p;
    for (int q = 0; q < 4; ++q) {
        a.part[q][0] = part[q][0].p;
        a.part[q][1] = part[q][1].p;
    }
    a.slice_res = slice_res.p;
    a.all_slices = world == 1 ? slice_res.p : all_slices.p;
    a.inline_decide = world == 1 ? 1 : 0;
    a.st = st.p;
    a.omega = omega;
    a.keep = 1.0 - omega;
    for (int q = 0; q < 4; ++q) a.hc[q] = heat ? hc[q] : 0.0;
    a.tma = kernel >= 1 && tma_pass_supported(L) ? 1 : 0;
    a.l_lo = 1;
    a.l_hi = L.n4;
    a.l_step = 1;
    a.dyn = 1;  // whole-slab pass launches; ranges clear it (sor.cu)
    a.wave = kernel == 2 && world == 1 && wflags.p != nullptr && wave_supported(L) ? 1 : 0;
    if (kernel == 7 && !heat && world == 1 && wflags.p != nullptr && kwave_supported(L)) {
        a.wave = 2;
        a.kwj = kwave_axis_j(L);
    }
    a.flags = wflags.p;
    a.snake = pass_snake();
    a.l2hint = pass_l2hint();
    a.order = pass_order();
    a.fuse_final = a.tma && world == 1 && !a.wave && pass_fuse_final() && tma_fuse_ok(L) ? 1 : 0;
    // halo push pointers are filled in by the Domain (it knows the neighbours)
    // 2D-tiled items on request, or (auto) when whole-row items leave many lanes idle:
    // rows of 150 / 284 slots (n1 = 300 / 567) -14..-29% per sweep; 16..256-slot rows
    // that fill the 256 threads keep whole rows
    const double u_rows = tma_lane_utilization(L, false), u_2d = tma_lane_utilization(L, true);
    a.tile2d = a.tma && !a.wave && (kernel == 5 || pass_tile2d() || (kernel == 6 && u_rows < 0.8 && u_2d > u_rows))
                   ? 1 : 0;
    if (a.tile2d) {
        a.maps = maps_for(a);
        if (!a.maps) a.tile2d = 0;  // no tensor-map encoder: whole-row items
    }
    if (a.tma)
        tma_pass_tiles(L, a);
    else
        pass_tiles(L, a);
    if (a.wave == 2) a.bps = kwave_bps(L);  // one partial per (plane-chunk item, warp)
    a.use_cond = 0;
    return a;
}

// ------------------------------------------------------------------ local transport
void LocalTransport::exchange(std::vector<Slab*>& slabs, const std::vector<PField>& F, int colours,
                              cudaStream_t st) {
    for (size_t s = 0; s + 1 < slabs.size(); ++s) {
        Slab& a = *slabs[s];
        const long long P1 = a.L.plane();
        const int n4 = a.L.n4;
        for (int c = 0; c < 2; ++c) {
            if (!(colours & (1 << c))) continue;
            // a's last owned plane -> b's halo plane 0; b's first owned plane -> a's halo plane n4+1
            SSB_CUDA(cudaMemcpyAsync(F[s + 1].c[c], F[s].c[c] + n4 * P1, P1 * sizeof(double),
                                     cudaMemcpyDeviceToDevice, st));
            SSB_CUDA(cudaMemcpyAsync(F[s].c[c] + (n4 + 1) * P1, F[s + 1].c[c] + P1, P1 * sizeof(double),
                                     cudaMemcpyDeviceToDevice, st));
        }
    }
}

void LocalTransport::allgather(std::vector<Slab*>& slabs, const std::vector<double*>& local,
                               const std::vector<double*>& all, int chunk, cudaStream_t st) {
    for (size_t d = 0; d < slabs.size(); ++d)
        for (size_t s = 0; s < slabs.size(); ++s)
            SSB_CUDA(cudaMemcpyAsync(all[d] + s * chunk, local[s], chunk * sizeof(double),
                                     cudaMemcpyDeviceToDevice, st ? st : slabs[d]->stream));
}

// ------------------------------------------------------------------ domain
struct Domain::GraphEntry {
    const void* key_ptr[2 * kStateBuffers + 2];
    const void* maps;
    int heat;
    int variant[7];  // every launch-shape switch of the captured pass kernels (graph_variant)
    double omega, hc[4];
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ~GraphEntry() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
    }
};

void Domain::init_common() {
    SSB_CUDA(cudaSetDevice(device));
    SSB_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    SSB_CUDA(cudaStreamCreateWithFlags(&cap_stream, cudaStreamNonBlocking));
    SSB_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    SSB_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    // the end slices and the halo exchange run on high-priority streams: the interior
    // pass is a persistent grid that fills every CTA slot, and pending CTAs of a
    // higher-priority stream (the end slices, the NCCL exchange kernels) are scheduled
    // first on the slots that free up, so the exchange overlaps the interior instead of
    // waiting for its end
    int prio_lo = 0, prio_hi = 0;
    SSB_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    SSB_CUDA(cudaStreamCreateWithPriority(&comm, cudaStreamNonBlocking, prio_hi));
    SSB_CUDA(cudaStreamCreateWithPriority(&bnd, cudaStreamNonBlocking, prio_hi));
    SSB_CUDA(cudaStreamCreateWithPriority(&dec, cudaStreamNonBlocking, prio_hi));
    SSB_CUDA(cudaEventCreateWithFlags(&ev_red, cudaEventDisableTiming));
    SSB_CUDA(cudaEventCreateWithFlags(&ev_dec, cudaEventDisableTiming));
    SSB_CUDA(cudaEventCreateWithFlags(&ev_pre, cudaEventDisableTiming));
    SSB_CUDA(cudaEventCreateWithFlags(&ev_bnd, cudaEventDisableTiming));
    SSB_CUDA(cudaEventCreateWithFlags(&ev_xchg, cudaEventDisableTiming));
    SSB_CUDA(cudaMallocHost(&st_host, sizeof(SorState)));
    SSB_CUDA(cudaMallocHost(&flag_host, 8 * sizeof(int)));
    SSB_CUDA(cudaMallocHost(&scal_host, 64 * sizeof(double)));
    for (auto& e : ev) SSB_CUDA(cudaEventCreate(&e));
}

Domain::Domain(const ss_grid& grid, int dev, int n_slabs) : g(grid), world(n_slabs), device(dev) {
    require(n_slabs >= 1, "Partition: worker count must be >= 1");
    chunk = (g.n4 + n_slabs - 1) / n_slabs;  // parallel.cpp:9-19
    const int last = g.n4 - (n_slabs - 1) * chunk;
    require(last >= 1, "Partition: " + std::to_string(n_slabs) + " workers leave the last one with " +
                           std::to_string(last) + " slices of " + std::to_string(g.n4));
    init_common();
    for (int s = 0; s < n_slabs; ++s) {
        const int n4l = s == n_slabs - 1 ? last : chunk;
        slabs.emplace_back(new Slab(g, s * chunk, n4l, s, chunk, world, stream));
        sp.push_back(slabs.back().get());
    }
    if (world == 1)
        tr.reset(new NullTransport);
    else
        tr.reset(new LocalTransport);
    sync();
}

void Domain::init_rank(int rank) {
    require(world >= 1 && rank >= 0 && rank < world, "invalid rank / world size");
    chunk = (g.n4 + world - 1) / world;
    const int last = g.n4 - (world - 1) * chunk;
    require(last >= 1, "Partition: " + std::to_string(world) + " workers leave the last one with " +
                           std::to_string(last) + " slices of " + std::to_string(g.n4));
    init_common();
    const int n4l = rank == world - 1 ? last : chunk;
    slabs.emplace_back(new Slab(g, rank * chunk, n4l, rank, chunk, world, stream));
    sp.push_back(slabs.back().get());
}

Domain::Domain(const ss_grid& grid, int dev, int rank, int w, const ss_host_comm& comm)
    : g(grid), world(w), device(dev), distributed(true) {
    init_rank(rank);
    tr = make_host_transport(comm, rank, w);
    sync();
}

Domain::Domain(const ss_grid& grid, int dev, int rank, int w, const unsigned char* uid)
    : g(grid), world(w), device(dev), distributed(true) {
    init_rank(rank);
    tr = make_nccl_transport(uid, rank, w);
    const char* e = std::getenv("SSB_P2P");
    if (w > 1 && e && std::atoi(e) != 0) setup_peer_links(*tr, *sp[0], rank, w, chunk, g.n4, peers);
    // ncclSend/ncclRecv are kernels: the interior launch of a pass is a persistent grid that fills
    // every CTA slot, so it leaves a few free for them (SSB_COMM_RESERVE, default 8 of 296: measured
    // free of charge on config 4, scripts/gpu_r02_s5i.sh); the in-kernel push needs none
    const char* r = std::getenv("SSB_COMM_RESERVE");
    comm_reserve = w > 1 && !peers.on ? (r ? std::max(0, std::atoi(r)) : 8) : 0;
    sync();
}

Domain::~Domain() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    graphs.clear();
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto e : ev)
        if (e) cudaEventDestroy(e);
    tr.reset();
    sp.clear();
    slabs.clear();
    if (st_host) cudaFreeHost(st_host);
    if (flag_host) cudaFreeHost(flag_host);
    if (scal_host) cudaFreeHost(scal_host);
    if (comm) cudaStreamSynchronize(comm);
    if (ev_bnd) cudaEventDestroy(ev_bnd);
    if (ev_pre) cudaEventDestroy(ev_pre);
    if (bnd) cudaStreamDestroy(bnd);
    if (dec) cudaStreamDestroy(dec);
    if (ev_red) cudaEventDestroy(ev_red);
    if (ev_dec) cudaEventDestroy(ev_dec);
    if (ev_xchg) cudaEventDestroy(ev_xchg);
    if (stream) cudaStreamDestroy(stream);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (h2d) cudaStreamSynchronize(h2d);
    for (auto e : up_ev) cudaEventDestroy(e);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamSynchronize(d2h);
    for (auto e : dn_ev) cudaEventDestroy(e);
    if (d2h) cudaStreamDestroy(d2h);
    if (comm) cudaStreamDestroy(comm);
}

void Domain::sync() { SSB_CUDA(cudaStreamSynchronize(stream)); }

void Domain::clear_graphs() {
    sync();
    graphs.clear();
}

long long Domain::host_plane() const { return (long long)(g.n1 + 2) * (g.n2 + 2) * (g.n3 + 2); }

// host arrays are global (local group / single) or the rank's slab (distributed)
const double* Domain::host_slab(const double* base, const Slab& s) const {
    return distributed ? base : base + (long long)s.L.l0 * host_plane();
}
double* Domain::host_slab(double* base, const Slab& s) const {
    return distributed ? base : base + (long long)s.L.l0 * host_plane();
}

std::vector<PField> Domain::role_fields(int role) const {
    std::vector<PField> F;
    for (Slab* s : sp) F.push_back(s->S[role].pf());
    return F;
}

std::vector<Domain::Triple> Domain::role_triples(const int roles[kStateBuffers]) const {
    std::vector<Triple> B;
    for (Slab* s : sp) {
        Triple t;
        for (int q = 0; q < kStateBuffers; ++q) t[q] = s->S[roles[q]].pf();
        B.push_back(t);
    }
    return B;
}

// every exchange runs on the comm stream, fenced by events against the main
// stream (one stream per communicator keeps the NCCL issue order identical on
// every rank)
void Domain::exchange(const std::vector<PField>& F, int colours) {
    if (world == 1) return;
    SSB_CUDA(cudaEventRecord(ev_bnd, stream));
    SSB_CUDA(cudaStreamWaitEvent(comm, ev_bnd, 0));
    tr->exchange(sp, F, colours, comm);
    SSB_CUDA(cudaEventRecord(ev_xchg, comm));
    SSB_CUDA(cudaStreamWaitEvent(stream, ev_xchg, 0));
}
void Domain::exchange_role(int role, int colours) { exchange(role_fields(role), colours); }

std::vector<double> Domain::gather_values(const std::vector<std::vector<double>>& per_slab, int k) {
    if (world == 1) return per_slab[0];
    std::vector<double*> loc, all;
    for (size_t s = 0; s < sp.size(); ++s) {
        SSB_CUDA(cudaMemcpyAsync(sp[s]->gloc.p, per_slab[s].data(), k * sizeof(double), cudaMemcpyHostToDevice,
                                 stream));
        loc.push_back(sp[s]->gloc.p);
        all.push_back(sp[s]->gall.p);
    }
    tr->allgather(sp, loc, all, k);
    std::vector<double> out((size_t)world * k);
    SSB_CUDA(cudaMemcpyAsync(out.data(), sp[0]->gall.p, out.size() * sizeof(double), cudaMemcpyDeviceToHost,
                             stream));
    sync();
    return out;
}

// profiling events per host-driven loop body: the red/black pass bounds + 3 per exchange
constexpr int kBodyEvents = 10;

cudaEvent_t Domain::pool_event(size_t idx) {
    while (ev_pool.size() <= idx) {
        cudaEvent_t e;
        SSB_CUDA(cudaEventCreate(&e));
        ev_pool.push_back(e);
    }
    return ev_pool[idx];
}

// 2D-tiled TMA items (env SSB_TILE2D; kernel 5 selects them explicitly)
bool pass_tile2d() {
    static const int v = [] {
        const char* e = std::getenv("SSB_TILE2D");
        return e ? std::atoi(e) : 0;
    }();
    return v != 0;
}

// device copies of the tensor maps, one per set of array pointers (the cached
// graphs bake the map address in, so a map set is never rewritten)
const TmaMaps* Slab::maps_for(const SorArgs& a) const {
    const void* key[2 * kStateBuffers + 4];
    for (int b = 0; b < kStateBuffers; ++b)
        for (int c = 0; c < 2; ++c) key[2 * b + c] = a.U[b][c];
    key[2 * kStateBuffers] = a.rhs[0];
    key[2 * kStateBuffers + 1] = a.rhs[1];
    key[2 * kStateBuffers + 2] = a.coef[0];
    key[2 * kStateBuffers + 3] = a.coef[1];
    for (const auto& e : map_cache)
        if (std::memcmp(e.key, key, sizeof key) == 0) return e.dev;
    TmaMaps h;
    if (!encode_tma_maps(a, h)) return nullptr;
    MapEntry e;
    std::memcpy(e.key, key, sizeof key);
    SSB_CUDA(cudaMalloc(&e.dev, sizeof(TmaMaps)));
    SSB_CUDA(cudaMemcpy(e.dev, &h, sizeof h, cudaMemcpyHostToDevice));
    map_cache.push_back(e);
    return e.dev;
}

// halo push for in-process slab groups (env SSB_PUSH, default on)
bool halo_push() {
    static const int v = [] {
        const char* e = std::getenv("SSB_PUSH");
        return e ? std::atoi(e) : 1;
    }();
    return v != 0;
}

// loop bodies per conditional-node iteration (env SSB_UNROLL)
int graph_unroll() {
    static const int v = [] {
        const char* e = std::getenv("SSB_UNROLL");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    return v;
}

// the switches that select which pass kernels / item shapes a captured loop body launches:
// a graph is reused only when all of them agree (ss_session_set_kernel may change them)
static void graph_variant(const SorArgs& a, int v[7]) {
    v[0] = a.tma;
    v[1] = a.wave;
    v[2] = a.tile2d;
    v[3] = a.fuse_final;
    v[4] = a.order;
    v[5] = a.snake;
    v[6] = a.l2hint;
}

cudaGraphExec_t Domain::graph_for(const SorArgs& base, bool heat) {
    constexpr int NK = 2 * kStateBuffers + 2;
    int variant[7];
    graph_variant(base, variant);
    const void* key[NK];
    for (int b = 0; b < kStateBuffers; ++b)
        for (int c = 0; c < 2; ++c) key[2 * b + c] = base.U[b][c];
    key[NK - 2] = base.rhs[0];
    key[NK - 1] = base.rhs[1];
    for (auto& e : graphs) {
        bool same = e->heat == (int)heat && e->omega == base.omega && e->maps == (const void*)base.maps &&
                    std::memcmp(e->variant, variant, sizeof variant) == 0;
        for (int q = 0; q < NK && same; ++q) same = e->key_ptr[q] == key[q];
        for (int q = 0; q < 4 && same; ++q) same = e->hc[q] == base.hc[q];
        if (same) return e->exec;
    }
    std::unique_ptr<GraphEntry> e(new GraphEntry);
    std::memcpy(e->key_ptr, key, sizeof key);
    e->heat = (int)heat;
    e->maps = base.maps;
    std::memcpy(e->variant, variant, sizeof variant);
    e->omega = base.omega;
    std::memcpy(e->hc, base.hc, sizeof e->hc);
    SSB_CUDA(cudaGraphCreate(&e->graph, 0));
    cudaGraphConditionalHandle h;
    SSB_CUDA(cudaGraphConditionalHandleCreate(&h, e->graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    SSB_CUDA(cudaGraphAddNode(&node, e->graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    SorArgs a = base;
    a.use_cond = 1;
    a.cond = h;
    const unsigned long long saved = g_launches.load();
    SSB_CUDA(cudaStreamBeginCaptureToGraph(cap_stream, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    // the body holds graph_unroll() iterations: a decided loop makes the rest no-ops
    for (int u = 0; u < graph_unroll(); ++u) launch_sor_body(cap_stream, a, heat, nullptr);
    cudaGraph_t captured = nullptr;
    SSB_CUDA(cudaStreamEndCapture(cap_stream, &captured));
    g_launches.store(saved);
    SSB_CUDA(cudaGraphInstantiate(&e->exec, e->graph, 0));
    graphs.push_back(std::move(e));
    if (graphs.size() > 8) graphs.erase(graphs.begin());
    return graphs.back()->exec;
}

void Domain::body_single(const SorArgs& a, bool heat, cudaEvent_t* ev4) {
    launch_sor_body(stream, a, heat, ev4);
}

// Multi-slab iteration n (solver.cpp:181-193): red on every slab, exchange the
// new red boundary planes, per-slice residuals + all-gather + decision, black,
// exchange the new black boundary planes.
void Domain::body_multi(const std::vector<SorArgs>& a, const std::vector<Triple>& B, bool heat, int n,
                        cudaEvent_t* ev4, cudaEvent_t* xev6) {
    const int bout = out_buf(n);
    std::vector<PField> F;
    for (const Triple& t : B) F.push_back(t[bout]);
    // boundary slices first, their exchange on the comm stream overlapped with
    // the interior slices (the paper overlaps Isend/Irecv the same way)
    const bool push = a[0].push_lo[0][0] != nullptr || a[0].push_hi[0][0] != nullptr;
    auto pass = [&](int colour) {
        if (push && distributed) {  // NVLink: wait for the neighbours' previous pass, push, signal
            const unsigned long long k = ++peers.count;
            launch_p2p_wait(stream, peers, k - 1);
            launch_sor_pass(stream, a[0], colour, heat);
            launch_p2p_signal(stream, peers, k);
            return;
        }
        if (push) {  // the pass kernels write the neighbours' halo planes themselves
            for (const SorArgs& x : a) launch_sor_pass(stream, x, colour, heat);
            return;
        }
        // the end slices (the planes the neighbours need) on the high-priority stream, one
        // launch per slab, running concurrently with the interior slices on the main stream
        SSB_CUDA(cudaEventRecord(ev_pre, stream));
        SSB_CUDA(cudaStreamWaitEvent(bnd, ev_pre, 0));
        for (const SorArgs& x : a) launch_sor_pass_ends(bnd, x, colour, heat);
        // halo timing (every timed multi-slab solve): x[0] exchange start (comm), x[1]
        // exchange end (comm), x[2] interior slices done (main stream)
        cudaEvent_t* xe = xev6 ? xev6 + 3 * colour : nullptr;
        SSB_CUDA(cudaEventRecord(ev_bnd, bnd));
        SSB_CUDA(cudaStreamWaitEvent(comm, ev_bnd, 0));
        if (xe) SSB_CUDA(cudaEventRecord(xe[0], comm));
        tr->exchange(sp, F, colour == 0 ? 1 : 2, comm);
        SSB_CUDA(cudaEventRecord(xe ? xe[1] : ev_xchg, comm));
        for (SorArgs x : a) {
            x.grid_short = comm_reserve;
            launch_sor_pass_range(stream, x, colour, heat, 2, x.L.n4 - 1, true);
        }
        if (xe) SSB_CUDA(cudaEventRecord(xe[2], stream));
        SSB_CUDA(cudaStreamWaitEvent(stream, xe ? xe[1] : ev_xchg, 0));
    };
    if (ev4) SSB_CUDA(cudaEventRecord(ev4[0], stream));
    pass(0);
    if (ev4) SSB_CUDA(cudaEventRecord(ev4[1], stream));
    // the decision of iteration n-1 (slice residuals, their all-gather, the test) on the side
    // stream, overlapped with the black pass n: black(n) does not depend on it (the red pass
    // handed it n; if n-1 turns out converged, black(n) only wrote out(n), which nobody reads)
    SSB_CUDA(cudaEventRecord(ev_red, stream));
    SSB_CUDA(cudaStreamWaitEvent(dec, ev_red, 0));
    for (const SorArgs& x : a) launch_sor_finalize(dec, x);
    std::vector<double*> loc, all;
    for (Slab* s : sp) {
        loc.push_back(s->slice_res.p);
        all.push_back(s->all_slices.p);
    }
    tr->allgather(sp, loc, all, chunk, dec);
    for (const SorArgs& x : a) launch_sor_decide(dec, x);
    SSB_CUDA(cudaEventRecord(ev_dec, dec));
    if (ev4) SSB_CUDA(cudaEventRecord(ev4[2], stream));
    pass(1);
    if (ev4) SSB_CUDA(cudaEventRecord(ev4[3], stream));
    SSB_CUDA(cudaStreamWaitEvent(stream, ev_dec, 0));  // the next red pass reads the decision
}

SolveOut Domain::solve(const std::vector<Triple>& B, const std::vector<PField>& rhs, bool heat, double omega,
                       const double hc[4], double tol_abs, bool use_norm, double rel, int max_iter, bool fixed,
                       int* result, bool check_assembly) {
    std::vector<SorArgs> a;
    // resident loop: single slab whose working set fits L2 (auto) or on request
    bool resident = single() && (kernel == 3 || (kernel == 4 && resident_supported(sp[0]->L)));
    // per-slab kernel code: 0 LDG (also the resident loop's tiles), 1 TMA whole rows,
    // 2 wavefront, 5 TMA 2D-tiled, 6 TMA with the item shape chosen per grid (auto)
    int kern = resident ? 0 : (kernel == 4 ? 6 : kernel == 3 ? 1 : kernel);
    solve_count = (solve_count + 1) & 0x3fff;
    const int epoch_base = (solve_count + 1) << 16;  // differs from the previous solve's
    if (check_assembly && world > 1) {  // every slab's assembly flag to every slab, on the device
        std::vector<double*> loc, all;
        for (Slab* s : sp) {
            launch_flag_to_double(stream, s->flags.p, s->gloc.p);
            loc.push_back(s->gloc.p);
            all.push_back(s->bad_all.p);
        }
        tr->allgather(sp, loc, all, 1);
    }
    for (size_t s = 0; s < sp.size(); ++s) {
        Slab& x = *sp[s];
        const double* ns = use_norm ? (world == 1 ? x.norm_loc.p : x.norm_all.p) : nullptr;
        launch_sor_init(stream, x.st.p, tol_abs, ns, g.n4, rel, max_iter, fixed ? fixed_mode : 0, epoch_base,
                        check_assembly && world == 1 ? x.flags.p : nullptr,
                        check_assembly && world > 1 ? x.bad_all.p : nullptr, world);
        a.push_back(x.sor_args(B[s].data(), rhs[s], heat, omega, hc, world, kern));
    }
    // in-process slab group with the TMA pass: neighbours' halo planes are written by
    // the pass kernels themselves (no exchange copies between the passes)
    if (distributed && peers.on && a[0].tma && !a[0].wave) {
        // ranks: the neighbours' arrays of the same buffer roles, mapped with CUDA IPC
        Slab& x = *sp[0];
        const long long P1 = x.L.plane();
        bool mapped = true;
        for (int b = 0; b < kStateBuffers && mapped; ++b)
            for (int c = 0; c < 2 && mapped; ++c) {
                int k = -1;  // which of this slab's state arrays is role b
                for (int q = 0; q < kStateBuffers; ++q)
                    if (x.S[q].c[c].p == B[0][b].c[c]) k = q;
                mapped = k >= 0;
                if (mapped) {
                    a[0].push_lo[b][c] = peers.S[0][k][c];
                    a[0].push_hi[b][c] = peers.S[1][k][c];
                }
            }
        if (mapped) {
            a[0].push_lo_off = (long long)peers.n4[0] * P1;
            a[0].push_hi_off = -(long long)x.L.n4 * P1;
        } else {
            for (int b = 0; b < kStateBuffers; ++b)
                for (int c = 0; c < 2; ++c) a[0].push_lo[b][c] = a[0].push_hi[b][c] = nullptr;
        }
    }
    if (!distributed && sp.size() > 1 && a[0].tma && !a[0].wave && halo_push()) {
        const long long P1 = sp[0]->L.plane();
        for (size_t s = 0; s < sp.size(); ++s) {
            for (int b = 0; b < kStateBuffers; ++b)
                for (int c = 0; c < 2; ++c) {
                    a[s].push_lo[b][c] = s > 0 ? B[s - 1][b].c[c] : nullptr;
                    a[s].push_hi[b][c] = s + 1 < sp.size() ? B[s + 1][b].c[c] : nullptr;
                }
            a[s].push_lo_off = s > 0 ? (long long)sp[s - 1]->L.n4 * P1 : 0;  // my plane 1 -> its plane n4'+1
            a[s].push_hi_off = -(long long)sp[s]->L.n4 * P1;                 // my plane n4 -> its plane 0
        }
    }
    if (!heat)
        last_kernel = resident ? 3 : a[0].wave == 2 ? 7 : a[0].wave == 1 ? 2 : !a[0].tma ? 0 : a[0].tile2d ? 5 : 1;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (resident) {  // events around the single launch: profiling split and the live loop time
        e0 = pool_event(0);
        e1 = pool_event(1);
        SSB_CUDA(cudaEventRecord(e0, stream));
        if (!launch_sor_resident(stream, a[0], heat)) {  // cannot be co-resident: pass kernels
            resident = false;
            kern = kernel == 4 ? 6 : 1;
            a[0] = sp[0]->sor_args(B[0].data(), rhs[0], heat, omega, hc, world, kern);
            if (!heat) last_kernel = a[0].tile2d ? 5 : 1;
        }
    }
    if (resident) {
        SSB_CUDA(cudaEventRecord(e1, stream));
        SSB_CUDA(cudaMemcpyAsync(st_host, sp[0]->st.p, sizeof(SorState), cudaMemcpyDeviceToHost, stream));
        sync();
        float lms = 0.f;
        SSB_CUDA(cudaEventElapsedTime(&lms, e0, e1));
        if (!heat) {  // passes run: red 1..it+1, black 1..it+1 (the last one speculative)
            prof.loop_ms += lms;
            prof.loop_passes += 2LL * st_host->iterations + 2;
        }
        if (profiling) {  // one launch: split its time evenly over the colour passes it ran
            const float ms = lms;
            const int it = st_host->iterations;
            const double per = ms / (2.0 * it + 1.0);
            prof.red_ms += per * (it + 1);
            prof.red_n += it + 1;
            prof.black_ms += per * it;
            prof.black_n += it;
        }
        SolveOut o;
        o.iterations = st_host->iterations;
        o.residual = st_host->residual;
        o.tol = st_host->tol;
        o.converged = st_host->converged != 0;
        o.nonfinite = st_host->nonfinite != 0;
        prof.sweeps += o.iterations;
        *result = o.iterations == 0 ? 0 : out_buf(o.iterations);
        return o;
    }
    const bool wave = a[0].wave != 0;
    // exchanges on the comm stream (not the in-kernel halo push): timed in every multi-slab
    // segmentation solve, profiling or not (events on the comm / main streams; the accounting
    // reads them once the solve is over), so the bench reports the timed run's own halo time
    const bool halo_timed = !heat && !single() && !wave && a[0].push_lo[0][0] == nullptr &&
                            a[0].push_hi[0][0] == nullptr;
    // loop bodies: red(max_iter+1) evaluates the last residual; a wavefront body
    // covers two iterations
    const int WI = a[0].wave == 1 ? wave_iters() : 1;
    const int limit = wave ? (max_iter + WI) / WI : max_iter + 1;
    if (single() && loop_mode == 1 && !profiling) {
        cudaGraphExec_t ex = graph_for(a[0], heat);
        cudaEvent_t l0 = pool_event(0), l1 = pool_event(1);
        SSB_CUDA(cudaEventRecord(l0, stream));
        SSB_CUDA(cudaGraphLaunch(ex, stream));
        SSB_CUDA(cudaEventRecord(l1, stream));
        SSB_CUDA(cudaMemcpyAsync(st_host, sp[0]->st.p, sizeof(SorState), cudaMemcpyDeviceToHost, stream));
        sync();
        if (!heat) {  // live SOR-loop time (the bench's roofline): events around the graph
            float ms = 0.f;
            SSB_CUDA(cudaEventElapsedTime(&ms, l0, l1));
            prof.loop_ms += ms;
            // passes run: red 1..it+1, black 1..it (+1 when the finalize sits in the black pass)
            // (a fixed-sweep solve's last black pass carries only the decision: not counted)
            prof.loop_passes += a[0].wave == 2 ? 2LL * (st_host->iterations + 1)  // k-wavefront bodies
                                               : 2LL * st_host->iterations + (fixed && fixed_mode == 2 ? 0 : 1) +
                                                     (a[0].fuse_final && !fixed ? 1 : 0);
        }
        const int bodies = wave ? st_host->iterations / WI + 1 : st_host->iterations + 1;
        const int U = graph_unroll();
        // kernels per loop body: red, finalize, black (finalize folded into black: 2;
        // wavefront: the wave kernel + one finalize per iteration it covers)
        const unsigned long long per = wave ? 1ull + WI : (a[0].fuse_final ? 2ull : 3ull);
        count_launch(per * U * (unsigned long long)((std::min(limit, bodies) + U - 1) / U));
    } else {
        // host-driven: chunks of loop bodies with one chunk of look-ahead; every
        // rank runs the same schedule (the decision is identical everywhere)
        int launched = 0, nb_chunk = 4;
        int slot = 0, pending = -1;
        size_t ev_used = 0;
        std::vector<size_t> body_ev;
        while (launched < limit) {
            const int nb = std::min(nb_chunk, limit - launched);
            for (int b = 0; b < nb; ++b) {
                const int n = launched + b + 1;
                // per body: red/black pass bounds (4) + the two exchanges' events (multi-slab, 6)
                cudaEvent_t evs[kBodyEvents];
                cudaEvent_t* e4 = nullptr;
                if (profiling || halo_timed) {
                    for (int q = 0; q < kBodyEvents; ++q) evs[q] = pool_event(ev_used + q);
                    body_ev.push_back(ev_used);
                    ev_used += kBodyEvents;
                    e4 = evs;
                }
                if (single())
                    body_single(a[0], heat, profiling ? e4 : nullptr);
                else
                    body_multi(a, B, heat, n, profiling ? e4 : nullptr, halo_timed ? e4 + 4 : nullptr);
            }
            launched += nb;
            SSB_CUDA(cudaMemcpyAsync(flag_host + slot, &sp[0]->st.p->done, sizeof(int), cudaMemcpyDeviceToHost,
                                     stream));
            SSB_CUDA(cudaEventRecord(ev[slot], stream));
            if (profiling) {
                SSB_CUDA(cudaEventSynchronize(ev[slot]));
                if (flag_host[slot]) break;
            } else if (pending >= 0) {
                SSB_CUDA(cudaEventSynchronize(ev[pending]));
                if (flag_host[pending]) break;
            }
            pending = slot;
            slot ^= 1;
            nb_chunk = std::min(nb_chunk * 2, 64);
        }
        SSB_CUDA(cudaMemcpyAsync(st_host, sp[0]->st.p, sizeof(SorState), cudaMemcpyDeviceToHost, stream));
        sync();
        if (profiling && wave) {  // wave kernel time per body, 2 * WI colour passes each
            const int bodies = st_host->iterations / WI + 1;
            for (size_t b = 0; b < body_ev.size() && (int)b < bodies; ++b) {
                float ms = 0.f;
                SSB_CUDA(cudaEventElapsedTime(&ms, ev_pool[body_ev[b]], ev_pool[body_ev[b] + 1]));
                prof.red_ms += ms;
                prof.red_n += 2 * WI;
            }
        } else if (profiling || halo_timed) {
            const int it = st_host->iterations;
            for (size_t b = 0; b < body_ev.size(); ++b) {
                float ms = 0.f;
                const size_t base = body_ev[b];
                // red(b+1) did real work (b+1 <= it+1; a fixed-sweep solve without diagnostics: <= it)
                if (profiling && (int)b < it + (fixed && fixed_mode == 2 ? 0 : 1)) {
                    SSB_CUDA(cudaEventElapsedTime(&ms, ev_pool[base], ev_pool[base + 1]));
                    prof.red_ms += ms;
                    prof.red_n++;
                }
                if (profiling && (int)b < it) {  // black(b+1) did real work
                    SSB_CUDA(cudaEventElapsedTime(&ms, ev_pool[base + 2], ev_pool[base + 3]));
                    prof.black_ms += ms;
                    prof.black_n++;
                }
                if (halo_timed)  // both exchanges of the body: duration, and the part not hidden
                    for (int c = 0; c < 2; ++c) {
                        if (c == 0 ? (int)b > it : (int)b >= it) continue;
                        const size_t x = base + 4 + 3 * c;
                        float xm = 0.f, wait = 0.f;
                        SSB_CUDA(cudaEventElapsedTime(&xm, ev_pool[x], ev_pool[x + 1]));
                        SSB_CUDA(cudaEventElapsedTime(&wait, ev_pool[x + 2], ev_pool[x + 1]));
                        prof.halo_ms += xm;
                        prof.halo_exposed_ms += wait > 0.f ? wait : 0.f;
                        prof.halo_n++;
                    }
            }
        }
    }
    SolveOut o;
    o.iterations = st_host->iterations;
    o.residual = st_host->residual;
    o.tol = st_host->tol;
    o.converged = st_host->converged != 0;
    o.nonfinite = st_host->nonfinite != 0;
    prof.sweeps += o.iterations;
    *result = o.iterations == 0 ? 0 : out_buf(o.iterations);
    return o;
}

void Domain::mirror_all(const std::vector<PField>& F) {
    // axes 0..2 on every local plane (halo planes hold exact copies of the
    // neighbours' planes, so mirroring them locally reproduces the neighbours'
    // result), then axis 3 at the global ends only (grid.cpp:138-156)
    for (size_t s = 0; s < sp.size(); ++s) launch_mirror_ghosts(stream, sp[s]->L, F[s], 0, 4);
}

static void heat_constants(const ss_grid& g, double dt, double hc[4]) {
    const double h[4] = {g.h1, g.h2, g.h3, g.h4};
    for (int a = 0; a < 4; ++a) hc[a] = (double)(float)(-(dt / (h[a] * h[a])));  // solver.cpp:89-90,107
}

int Domain::heat_smooth(const std::vector<Triple>& B, double sigma, int steps, double omega, double tol,
                        int max_iter) {
    std::vector<PField> F0;
    for (const Triple& t : B) F0.push_back(t[0]);
    if (sigma == 0.0) {
        mirror_all(F0);
        return 0;
    }
    const double dt = 0.5 * sigma * sigma / steps;
    double hc[4];
    heat_constants(g, dt, hc);
    for (size_t s = 0; s < sp.size(); ++s)  // the SOR buffers' ghosts/halos = the input's
        for (int q = 1; q < kStateBuffers; ++q) launch_copy_ghosts(stream, sp[s]->L, B[s][q], B[s][0]);
    int idx[kStateBuffers];
    for (int q = 0; q < kStateBuffers; ++q) idx[q] = q;
    for (int st = 0; st < steps; ++st) {
        std::vector<Triple> T;
        std::vector<PField> rhs;
        for (const Triple& t : B) {
            Triple x;
            for (int q = 0; q < kStateBuffers; ++q) x[q] = t[idx[q]];
            T.push_back(x);
            rhs.push_back(t[idx[0]]);
        }
        int r = 0;
        const SolveOut o = solve(T, rhs, true, omega, hc, tol, false, 0.0, max_iter, false, &r);
        if (!o.converged) throw SolverErrT(o);
        int nidx[kStateBuffers];
        for (int q = 0; q < kStateBuffers; ++q) nidx[q] = idx[(r + q) % kStateBuffers];
        std::memcpy(idx, nidx, sizeof idx);
    }
    std::vector<PField> R;
    for (const Triple& t : B) R.push_back(t[idx[0]]);
    mirror_all(R);
    return idx[0];
}

void Domain::set_u(const double* host) {
    for (Slab* s : sp) s->upload_state(host_slab(host, *s), cur);
}

void Domain::get_u(double* host) {
    // owned planes (and global ghost planes) of every slab; halo planes are the
    // neighbours' and are left alone
    const long long hp = host_plane();
    for (Slab* s : sp) {
        double* d = s->stage_p();
        launch_unpack(stream, s->L, s->S[cur].pf(), d);
        const int p0 = s->L.glo ? 0 : 1;
        const int p1 = s->L.ghi ? s->L.n4 + 1 : s->L.n4;
        copy_d2h(host_slab(host, *s) + p0 * hp, d + p0 * hp, (p1 - p0 + 1) * hp * sizeof(double), stream);
    }
    sync();
}

void Domain::get_mask(double level, uint8_t* mask) {
    const size_t fr = (size_t)g.n1 * g.n2 * g.n3;
    for (Slab* s : sp) {
        Dev<uint8_t> m;
        m.alloc(fr * s->L.n4);
        launch_mask(stream, s->L, s->S[cur].pf(), level, m.p);
        SSB_CUDA(cudaMemcpyAsync(mask + (distributed ? 0 : fr * s->L.l0), m.p, fr * s->L.n4, cudaMemcpyDefault,
                                 stream));
        sync();
    }
}

void Domain::prepare(const double* image, const ss_center* c, int n, const ss_seg_params& p, const double* u0) {
    // SSB_TIMING=1: per-phase wall times of prepare on stderr (device synchronised)
    static const bool timing = std::getenv("SSB_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!timing) return;
        sync();
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "prepare %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    validate_seg_params(p);
    validate_centers(g, c, n);
    require(image != nullptr, "null image");
    prepared = false;
    prm = p;
    for (Slab* s : sp) build_balls(s->rescale_balls, s->gl, s->L.l0, c, n, p.rescale_radius, false);

    // u0 (solver.cpp:416-417): caller's u0 or build_initial, then local_rescale
    cur = 0;
    for (Slab* s : sp) {
        if (u0) {
            s->upload_state(host_slab(u0, *s), 0);
        } else {
            s->initial(s->S[0].pf(), c, n, p.init_v, p.init_R, p.init_profile);
            s->sync_ghosts_from(0);
        }
        s->rescale(0);
    }
    mark("u0 + rescale");

    // local_threshold, heat_smooth x2, face_coefficients (solver.cpp:419-422)
    // the heat solves' three rotating outputs are the state buffers S[1..3]: unused until
    // the first step (which overwrites their interiors; their ghosts are reset below), so
    // prepare's peak is 2 fields above the steady state -- config 3 fits two GPUs
    std::vector<std::unique_ptr<DevField>> img, th;
    for (Slab* s : sp) {
        img.emplace_back(new DevField);
        th.emplace_back(new DevField);
        img.back()->alloc(s->L);
        th.back()->alloc(s->L);
        s->upload(host_slab(image, *s), img.back()->pf());
    }
    sync();
    for (Slab* s : sp) s->stage.reset();  // the upload staging buffer comes back on demand
    mark("alloc + image upload");
    {
        std::vector<std::unique_ptr<BallSet>> bsets;
        std::vector<std::unique_ptr<Dev<double>>> abs;
        std::vector<std::vector<double>> bad(sp.size(), std::vector<double>(1, (double)INT_MAX));
        for (size_t s = 0; s < sp.size(); ++s) {
            Slab& x = *sp[s];
            bsets.emplace_back(new BallSet);
            build_balls(*bsets.back(), x.gl, x.L.l0, c, n, std::nan(""), false);  // per-row radii
            abs.emplace_back(new Dev<double>);
            abs.back()->alloc(2 * (size_t)std::max(1, bsets.back()->count()));
            launch_fill(stream, x.L, th[s]->pf(), p.background);
            if (bsets.back()->count()) x.threshold_minmax(img[s]->pf(), *bsets.back(), abs.back()->p);
        }
        sync();
        for (size_t s = 0; s < sp.size(); ++s) {  // "ball covers no doxels" (preprocess.cpp:89-91)
            const BallSet& bs = *bsets[s];
            if (!bs.count()) continue;
            std::vector<double> h(2 * bs.count());
            SSB_CUDA(cudaMemcpy(h.data(), abs[s]->p, h.size() * sizeof(double), cudaMemcpyDeviceToHost));
            for (int b = 0; b < bs.count(); ++b)
                if (h[2 * b] > h[2 * b + 1]) bad[s][0] = std::min(bad[s][0], (double)bs.row[b]);
        }
        const std::vector<double> allbad = gather_values(bad, 1);
        const double first = *std::min_element(allbad.begin(), allbad.end());
        if (first < (double)INT_MAX)
            throw Error(SS_ERR_VALIDATION,
                        "local_threshold: ball in centers row " + std::to_string((long long)first + 1) +
                            " covers no doxels");
        for (size_t s = 0; s < sp.size(); ++s)
            if (bsets[s]->count()) sp[s]->threshold_write(img[s]->pf(), th[s]->pf(), *bsets[s], abs[s]->p, p.lambda);
        sync();
    }
    std::vector<PField> thf;
    for (auto& f : th) thf.push_back(f->pf());
    exchange(thf, 3);  // halos of the thresholded image (the heat solve reads them)
    mark("local_threshold");

    std::vector<Triple> b1, b2;
    for (size_t s = 0; s < sp.size(); ++s)
        b1.push_back({img[s]->pf(), sp[s]->S[1].pf(), sp[s]->S[2].pf(), sp[s]->S[3].pf()});
    const int r1 = heat_smooth(b1, p.sigma, p.smooth_steps, p.smooth_omega, p.smooth_tol, p.smooth_max_iter);
    mark("heat_smooth(I0)");
    for (size_t s = 0; s < sp.size(); ++s)
        b2.push_back({th[s]->pf(), b1[s][(r1 + 1) % kStateBuffers], b1[s][(r1 + 2) % kStateBuffers],
                      b1[s][(r1 + 3) % kStateBuffers]});
    const int r2 = heat_smooth(b2, p.sigma, p.smooth_steps, p.smooth_omega, p.smooth_tol, p.smooth_max_iter);
    mark("heat_smooth(ITH)");
    for (size_t s = 0; s < sp.size(); ++s)
        sp[s]->face_coefficients(b1[s][r1], b2[s][r2], p.K, p.delta, p.vartheta, nullptr);
    sync();
    mark("face_coefficients");

    // apply_dirichlet(u, 0) (solver.cpp:425) on every state buffer; halo planes
    // are refreshed by the exchange at the start of every step
    for (Slab* s : sp)
        for (auto& f : s->S) launch_set_ghosts(stream, s->L, f.pf(), 0.0);
    sync();
    mark("dirichlet");
    prepared = true;
}

// One time step of the segment() loop (solver.cpp:428-438): exchange the u^{n-1} halos,
// assemble_step, the per-step tolerance, redblack_sor (rhs = guess = u^{n-1}), local_rescale.
// Everything up to the end of the SOR loop is one stream sequence: the assembly's
// non-finite flag (solver.cpp:71-75) reaches the loop control on the device (sor_init,
// all-gathered across slabs), and the host learns of it with the solve's final state.
SolveOut Domain::step(ss_step_diag* diag, int fixed, bool rescale) { return step_impl(diag, fixed, rescale, nullptr); }

void Domain::set_u_interior(const double* host) {
    const long long fr = (long long)g.n1 * g.n2 * g.n3;
    for (Slab* s : sp) {
        double* d = s->stage_p();
        copy_h2d(d, host + (distributed ? 0 : fr * s->L.l0), fr * s->L.n4 * sizeof(double), stream);
        launch_pack_interior(stream, s->L, d, s->S[cur].pf(), 1, s->L.n4);
    }
}

// slice chunks of the host-buffer transfers (step_host*, get_u_interior): the chained upload
// of step_host_async trails its download by one chunk
#ifndef SSB_HOST_CHUNKS
#define SSB_HOST_CHUNKS 16
#endif
constexpr int kHostChunks = SSB_HOST_CHUNKS;

void Domain::get_u_interior(double* host) {
    const long long fr = (long long)g.n1 * g.n2 * g.n3;
    if (single() && host_pinned(host)) {  // slice chunks: unpack chunk q+1 while chunk q moves
        Slab& x = *sp[0];
        const int n4 = x.L.n4, C = std::min(n4, kHostChunks);
        while ((int)up_ev.size() < C + 1) {
            cudaEvent_t e;
            SSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            up_ev.push_back(e);
        }
        double* d = x.stage_p();
        for (int q = 0; q < C; ++q) {
            const int a = 1 + (int)((long long)q * n4 / C), b = (int)((long long)(q + 1) * n4 / C);
            launch_unpack_interior(stream, x.L, x.S[cur].pf(), d, a, b);
            SSB_CUDA(cudaEventRecord(up_ev[q], stream));
            SSB_CUDA(cudaStreamWaitEvent(h2d, up_ev[q], 0));
            SSB_CUDA(cudaMemcpyAsync(host + (a - 1) * fr, d + (a - 1) * fr, (size_t)(b - a + 1) * fr * sizeof(double),
                                     cudaMemcpyDeviceToHost, h2d));
        }
        SSB_CUDA(cudaEventRecord(up_ev[C], h2d));
        SSB_CUDA(cudaStreamWaitEvent(stream, up_ev[C], 0));  // later users of the staging buffer
        SSB_CUDA(cudaStreamSynchronize(h2d));
        return;
    }
    for (Slab* s : sp) {
        double* d = s->stage_p();
        launch_unpack_interior(stream, s->L, s->S[cur].pf(), d);
        copy_d2h(host + (distributed ? 0 : fr * s->L.l0), d, fr * s->L.n4 * sizeof(double), stream);
    }
    sync();
}

// one slab, page-locked input: slice chunks H2D on the copy stream; per chunk the main
// stream packs it and (assemble) assembles the slices whose l+1 neighbour is in (the last
// chunk: all)
void Domain::upload_chunks(const double* host, bool assemble) {
    Slab& x = *sp[0];
    const long long fr = (long long)g.n1 * g.n2 * g.n3;
    const int n4 = x.L.n4, C = std::min(n4, kHostChunks);
    while ((int)up_ev.size() < C + 1) {
        cudaEvent_t e;
        SSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        up_ev.push_back(e);
    }
    double* st = x.stage_p();
    SSB_CUDA(cudaEventRecord(up_ev[C], stream));  // earlier users of the staging buffer are done
    SSB_CUDA(cudaStreamWaitEvent(h2d, up_ev[C], 0));
    auto lo = [&](int q) { return 1 + (int)((long long)q * n4 / C); };
    // this input is the previous step's result still on its way down (step_host_async): each
    // chunk goes up as soon as it has come down (same chunks), device-ordered, no host wait
    const bool chained = dn_host == host && (int)dn_ev.size() >= 2 * C + 1;
    for (int q = 0; q < C; ++q) {
        const int a = lo(q), b = lo(q + 1) - 1;
        if (chained) SSB_CUDA(cudaStreamWaitEvent(h2d, dn_ev[q], 0));
        SSB_CUDA(cudaMemcpyAsync(st + (a - 1) * fr, host + (a - 1) * fr, (size_t)(b - a + 1) * fr * sizeof(double),
                                 cudaMemcpyHostToDevice, h2d));
        SSB_CUDA(cudaEventRecord(up_ev[q], h2d));
    }
    if (!assemble) {
        for (int q = 0; q < C; ++q) {
            SSB_CUDA(cudaStreamWaitEvent(stream, up_ev[q], 0));
            launch_pack_interior(stream, x.L, st, x.S[cur].pf(), lo(q), lo(q + 1) - 1);
        }
        return;
    }
    SSB_CUDA(cudaMemsetAsync(x.flags.p, 0, sizeof(int), stream));
    const AsmArgs args = x.asm_args(x.S[cur].pf(), x.have_G, prm.tau, prm.epsilon);
    int done = 0;
    for (int q = 0; q < C; ++q) {
        const int a = lo(q), b = lo(q + 1) - 1;
        SSB_CUDA(cudaStreamWaitEvent(stream, up_ev[q], 0));
        launch_pack_interior(stream, x.L, st, x.S[cur].pf(), a, b);
        const int hi = q == C - 1 ? n4 : b - 1;
        if (!launch_assemble_tile_range(stream, args, done + 1, hi))
            throw Error(SS_ERR_CUDA, "assemble: tensor-map encoding failed");
        done = std::max(done, hi);
    }
}

SolveOut Domain::step_host(const double* in, double* out, int fixed, ss_step_diag* diag) {
    const SolveOut o = step_impl(diag, fixed, true, in);
    wait_transfers();
    if (out) get_u_interior(out);
    return o;
}

// the result's compact interior to page-locked `host` in slice chunks on the d2h stream: the
// unpack of chunk q + 1 (main stream, its own staging buffer) overlaps the copy of chunk q; no
// host wait (wait_transfers)
void Domain::download_async(double* host) {
    Slab& x = *sp[0];
    const long long fr = (long long)g.n1 * g.n2 * g.n3;
    const int n4 = x.L.n4, C = std::min(n4, kHostChunks);
    while ((int)dn_ev.size() < 2 * C + 1) {
        cudaEvent_t e;
        SSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        dn_ev.push_back(e);
    }
    double* d = x.dstage_p();
    for (int q = 0; q < C; ++q) {
        const int a = 1 + (int)((long long)q * n4 / C), b = (int)((long long)(q + 1) * n4 / C);
        SSB_CUDA(cudaStreamWaitEvent(stream, dn_ev[q], 0));  // the previous copy out of this staging chunk
        launch_unpack_interior(stream, x.L, x.S[cur].pf(), d, a, b);
        SSB_CUDA(cudaEventRecord(dn_ev[C + q], stream));
        SSB_CUDA(cudaStreamWaitEvent(d2h, dn_ev[C + q], 0));
        SSB_CUDA(cudaMemcpyAsync(host + (a - 1) * fr, d + (a - 1) * fr, (size_t)(b - a + 1) * fr * sizeof(double),
                                 cudaMemcpyDeviceToHost, d2h));
        SSB_CUDA(cudaEventRecord(dn_ev[q], d2h));
    }
    dn_host = host;
}

SolveOut Domain::step_host_async(const double* in, double* out, int fixed, ss_step_diag* diag) {
    const bool async = sp.size() == 1 && out && host_pinned(out) && (!in || host_pinned(in)) &&
                       assemble_tile_supported(sp[0]->L);
    if (!async) return step_host(in, out, fixed, diag);
    if (dn_host && dn_host != in) wait_transfers();  // only a chained input may still be in flight
    const SolveOut o = step_impl(diag, fixed, true, in);
    if (dn_host) wait_transfers();  // (a chained download is complete: the upload waited for it)
    download_async(out);
    return o;
}

// every transfer of step_host_async complete (host), and the main stream ordered after them
void Domain::wait_transfers() {
    if (!dn_host) return;
    const int C = (int)(dn_ev.size() - 1) / 2;
    SSB_CUDA(cudaEventRecord(dn_ev[2 * C], d2h));
    SSB_CUDA(cudaStreamWaitEvent(stream, dn_ev[2 * C], 0));
    SSB_CUDA(cudaStreamSynchronize(d2h));
    dn_host = nullptr;
}

SolveOut Domain::step_impl(ss_step_diag* diag, int fixed, bool rescale, const double* host_in) {
    if (!prepared) throw Error(SS_ERR_STATE, "session not prepared");
    int roles[kStateBuffers];
    for (int q = 0; q < kStateBuffers; ++q) roles[q] = (cur + q) % kStateBuffers;
    // page-locked input of a one-slab process: chunked upload (chained to an in-flight download
    // of the same buffer); a single domain also overlaps it with the assembly
    const bool chunked = host_in && sp.size() == 1 && assemble_tile_supported(sp[0]->L) && host_pinned(host_in);
    const bool overlap = chunked && single();
    if (host_in && !chunked) set_u_interior(host_in);
    if (chunked && !overlap) upload_chunks(host_in, false);
    exchange_role(cur, 3);  // u^{n-1} halos for the face gradients and the first red pass
    if (profiling) SSB_CUDA(cudaEventRecord(ev[2], stream));
    if (overlap)
        upload_chunks(host_in, true);
    else
        for (Slab* s : sp) s->assemble(s->S[cur].pf(), s->have_G, prm.tau, prm.epsilon, nullptr, nullptr, nullptr);
    if (profiling) SSB_CUDA(cudaEventRecord(ev[3], stream));
    const bool rel = !fixed && prm.sor_rel_tol > 0.0;
    if (rel) {
        std::vector<double*> loc, all;
        for (Slab* s : sp) {
            launch_norm_slices(stream, s->L, s->S[cur].pf(), s->norm_part.p, s->norm_loc.p);
            loc.push_back(s->norm_loc.p);
            all.push_back(s->norm_all.p);
        }
        if (world > 1) tr->allgather(sp, loc, all, chunk);
    }
    const std::vector<Triple> B = role_triples(roles);
    std::vector<PField> rhs;
    for (const Triple& t : B) rhs.push_back(t[0]);  // rhs = guess = u^{n-1} (solver.cpp:430)
    int rr = 0;
    // without a diag struct nobody reads a fixed-sweep solve's residual (ss_session_fixed_sweeps returns it
    // and asks for it): the pass that would only evaluate it stays idle
    fixed_mode = diag || want_residual ? 1 : 2;
    const SolveOut o = fixed ? solve(B, rhs, false, prm.omega, nullptr, 1.0, false, 0.0, fixed, true, &rr, true)
                             : solve(B, rhs, false, prm.omega, nullptr, prm.sor_tol, rel, prm.sor_rel_tol,
                                     prm.sor_max_iter, false, &rr, true);
    if (profiling) {
        float ms = 0.f;
        SSB_CUDA(cudaEventElapsedTime(&ms, ev[2], ev[3]));
        prof.assemble_ms += ms;
        prof.assemble_n++;
    }
    if (o.nonfinite) throw Error(SS_ERR_NONFINITE, "assemble_step: non-finite coefficient (bad input field?)");
    if (!o.converged) throw SolverErrT(o);
    cur = roles[rr];
    const bool do_rescale = rescale && prm.rescale_each_step;
    if (do_rescale) {
        if (profiling) SSB_CUDA(cudaEventRecord(ev[2], stream));
        for (Slab* s : sp) s->rescale(cur);
        if (profiling) SSB_CUDA(cudaEventRecord(ev[3], stream));
    }
    std::vector<double> mh(2 * sp.size(), 0.0);
    if (diag)
        for (size_t s = 0; s < sp.size(); ++s) {
            launch_minmax(stream, sp[s]->L, sp[s]->S[cur].pf(), sp[s]->scratch.p, sp[s]->scal.p + 1);
            SSB_CUDA(cudaMemcpyAsync(&mh[2 * s], sp[s]->scal.p + 1, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                     stream));
        }
    if (diag || profiling) sync();
    if (profiling && do_rescale) {
        float ms = 0.f;
        SSB_CUDA(cudaEventElapsedTime(&ms, ev[2], ev[3]));
        prof.rescale_ms += ms;
        prof.rescale_n++;
    }
    if (diag) {
        std::vector<std::vector<double>> mm(sp.size());
        for (size_t s = 0; s < sp.size(); ++s) mm[s] = {mh[2 * s], mh[2 * s + 1]};
        const std::vector<double> all = gather_values(mm, 2);
        double lo = INFINITY, hi = -INFINITY;
        for (int r = 0; r < world; ++r) {
            lo = std::min(lo, all[2 * r]);
            hi = std::max(hi, all[2 * r + 1]);
        }
        diag->iterations = o.iterations;
        diag->residual = o.residual;
        diag->tol = o.tol;
        diag->umin = lo;
        diag->umax = hi;
    }
    return o;
}

// fixed-sweep mode without the rescale (ss_session_fixed_sweeps): assemble + exactly
// n_sweeps sweeps; non-finite coefficients are reported like step()'s
double Domain::fixed_sweeps(int n_sweeps) {
    struct Want {
        bool& w;
        explicit Want(bool& x) : w(x) { w = true; }
        ~Want() { w = false; }
    } want(want_residual);
    return step(nullptr, n_sweeps, false).residual;
}

}  // namespace ssb
