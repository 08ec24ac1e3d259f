// eoc.cu -- the EOC verification harness on the device (eoc.cpp:83-137): the
// pure level-set step (G == 1, no rescaling) against the exact solution
// u(x, t) = (|x|^2 - 1)/6 + t on [-1.25, 1.25]^4, Dirichlet ghosts from the
// exact solution at the new time level, space-time L2 error.
//
// Expressions follow eoc.cpp: centre coordinate dmin + (v - 0.5) h,
// exact_u = (x0*x0 + x1*x1 + x2*x2 + x3*x3 - 1.0) / 6.0 + t (left to right,
// -fmad=false), so ghost and initial values are bit-identical to the reference.
#include <cmath>

#include "domain.cuh"

namespace ssb {

namespace {

__device__ __forceinline__ double exact_u(double x0, double x1, double x2, double x3, double t) {
    return (x0 * x0 + x1 * x1 + x2 * x2 + x3 * x3 - 1.0) / 6.0 + t;
}

__device__ __forceinline__ double ccoord(int v, double dmin, double h) { return dmin + (v - 0.5) * h; }

// fill_all (eoc.cpp:40-53) or fill_ghosts (eoc.cpp:55-79) on a colour-packed field
__global__ void exact_fill_kernel(const Layout L, PField f, double dmin, double h, double t, int ghosts_only) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= L.P) return;
    const int i = (int)(e % L.iMax);
    const long long row = e / L.iMax;
    const int j = (int)(row % L.jMax);
    const int k = (int)((row / L.jMax) % L.kMax);
    const int l = (int)(row / ((long long)L.jMax * L.kMax));
    const bool ghost =
        i == 0 || i > L.n1 || j == 0 || j > L.n2 || k == 0 || k > L.n3 || l == 0 || l > L.n4;
    if (ghosts_only && !ghost) return;
    const int lg = l + L.l0;
    f.c[L.colour(i, j, k, l)][row * L.W + (i >> 1)] =
        exact_u(ccoord(i, dmin, h), ccoord(j, dmin, h), ccoord(k, dmin, h), ccoord(lg, dmin, h), t);
}

// per owned slice: sum over the slice of (u - exact)^2 (eoc.cpp:115-131), fixed order
__global__ void __launch_bounds__(256) err_slices_kernel(const Layout L, PField f, double dmin, double h,
                                                         double t, double* out) {
    const int l = blockIdx.x + 1;
    const long long N = (long long)L.n1 * L.n2 * L.n3;
    double s = 0.0;
    for (long long e = threadIdx.x; e < N; e += blockDim.x) {
        const int i = (int)(e % L.n1) + 1;
        const long long r = e / L.n1;
        const int j = (int)(r % L.n2) + 1;
        const int k = (int)(r / L.n2) + 1;
        const double u = f.c[L.colour(i, j, k, l)][L.packed(i, j, k, l)];
        const double d = u - exact_u(ccoord(i, dmin, h), ccoord(j, dmin, h), ccoord(k, dmin, h),
                                     ccoord(l + L.l0, dmin, h), t);
        s += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    __shared__ double ws[8];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += ws[w];
        out[blockIdx.x] = tot;
    }
}

}  // namespace

void launch_exact_fill(cudaStream_t s, const Layout& L, PField f, double dmin, double h, double t, bool ghosts_only) {
    exact_fill_kernel<<<ceil_div(L.P, 256), 256, 0, s>>>(L, f, dmin, h, t, ghosts_only ? 1 : 0);
    SSB_LAUNCHED();
}

void launch_err_slices(cudaStream_t s, const Layout& L, PField f, double dmin, double h, double t, double* out) {
    err_slices_kernel<<<L.n4, 256, 0, s>>>(L, f, dmin, h, t, out);
    SSB_LAUNCHED();
}

// run_levelset_row (eoc.cpp:83-137) for grid n, EocConfig defaults (eoc.hpp:16-28)
double Domain::eoc_row(int n, double omega, double sor_tol, int max_iter, long long* total_sweeps) {
    static const int sched[5][2] = {{10, 1}, {20, 4}, {40, 16}, {80, 64}, {160, 256}};
    int steps = 0;
    for (auto& r : sched)
        if (r[0] == n) steps = r[1];
    if (!steps) throw Error(SS_ERR_VALIDATION, "EOC schedule has no row n=" + std::to_string(n) +
                                                   " (valid: 10, 20, 40, 80, 160)");
    require(g.n1 == n && g.n2 == n && g.n3 == n && g.n4 == n, "eoc_row: the session grid must be n^4");
    const double dmin = -1.25, dmax = 1.25, T = 0.0625;
    const double h = (dmax - dmin) / n;
    const double tau = T / steps;
    cur = 0;
    for (Slab* s : sp) {
        launch_exact_fill(stream, s->L, s->S[0].pf(), dmin, h, 0.0, false);
        s->sync_ghosts_from(0);
    }
    exchange_role(0, 3);
    const double cell = h * h * h * h;
    double err_sq = 0.0;
    long long sweeps = 0;
    std::vector<double> host_slices(g.n4);
    for (int step = 1; step <= steps; ++step) {
        const double t_n = step * tau;
        // coefficients at u^{n-1} with the previous time level's ghosts (eoc.cpp:110)
        for (Slab* s : sp) s->assemble(s->S[cur].pf(), false, tau, h * h, nullptr, nullptr, nullptr);
        // fresh Dirichlet data in every state buffer (eoc.cpp:111)
        for (Slab* s : sp)
            for (auto& f : s->S) launch_exact_fill(stream, s->L, f.pf(), dmin, h, t_n, true);
        exchange_role(cur, 3);  // slabs: halo planes are the neighbours' u^{n-1}, not ghosts
        int roles[kStateBuffers];
        for (int q = 0; q < kStateBuffers; ++q) roles[q] = (cur + q) % kStateBuffers;
        const std::vector<Triple> B = role_triples(roles);
        std::vector<PField> rhs;
        for (const Triple& t : B) rhs.push_back(t[0]);
        int rr = 0;
        const SolveOut o = solve(B, rhs, false, omega, nullptr, sor_tol, false, 0.0, max_iter, false, &rr);
        if (!o.converged) throw SolverErrT(o);
        cur = roles[rr];
        sweeps += o.iterations;
        // per-slice error sums, summed in l order (eoc.cpp:115-134)
        std::vector<double*> loc, all;
        for (Slab* s : sp) {
            launch_err_slices(stream, s->L, s->S[cur].pf(), dmin, h, t_n, s->norm_loc.p);
            loc.push_back(s->norm_loc.p);
            all.push_back(s->norm_all.p);
        }
        if (world > 1) tr->allgather(sp, loc, all, chunk);
        SSB_CUDA(cudaMemcpyAsync(host_slices.data(), world > 1 ? sp[0]->norm_all.p : sp[0]->norm_loc.p,
                                 g.n4 * sizeof(double), cudaMemcpyDeviceToHost, stream));
        sync();
        double step_sum = 0.0;
        for (int l = 0; l < g.n4; ++l) step_sum += host_slices[l];
        err_sq += tau * cell * step_sum;
    }
    if (total_sweeps) *total_sweeps = sweeps;
    return std::sqrt(err_sq);
}

}  // namespace ssb
