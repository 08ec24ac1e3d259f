// sor.cu -- red-black SOR for the 4D 9-point system (solver.cpp:124-397).
//
// One iteration = red pass, finalize, black pass:
//   red(n)      updates red doxels of state n-1 into buffer out(n) and, from the
//               same loads, evaluates the red-row residual of state n-1
//               (the reference's separate red_residuals pass, solver.cpp:319-361,
//               lagged by one pass so it costs no extra sweep);
//   finalize    sums per-slice residuals of state n-1 (black partials from
//               black(n-1) + red partials from red(n)), tests res <= tol /
//               iter >= max_iter (solver.cpp:195-205) and advances counters;
//   black(n)    updates black doxels with the new red values; its in-sweep
//               residual diag*(unew-ubar) (solver.cpp:309-312) is the black
//               part of state n's residual.
// Rotating buffers (SorArgs::U): red(n+1) writes a different buffer than the
// one holding state n, so stopping after red(n+1) returns exactly the
// reference's iterate n; the guess buffer is never written, so it can double
// as the rhs (segment() solves with rhs = guess = u^{n-1}, solver.cpp:430).
// Per-doxel arithmetic is the reference's expression order compiled with
// -fmad=false: iterates are bit-identical to the oracle.
#include "kernels.cuh"

namespace ssb {

namespace {

__device__ __forceinline__ double block_sum(double v) {
    // fixed-shape tree => deterministic
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __shared__ double ws[32];
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    const int nw = (blockDim.x * blockDim.y + 31) >> 5;
    if ((tid & 31) == 0) ws[tid >> 5] = v;
    __syncthreads();
    if (tid < 32) {
        v = tid < nw ? ws[tid] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;  // valid in thread 0
}

template <int C, bool HEAT>
__global__ void __launch_bounds__(kPassBX * kPassBY) sor_pass(const SorArgs a) {
    const SorState* st = a.st;
    if (*(volatile const int*)&st->done) return;
    const int n = C == 0 ? *(volatile const int*)&st->n_red : *(volatile const int*)&st->n_black;
    const int bout = (n & 1) ? 1 : 2;
    const int bin = n == 1 ? 0 : (((n - 1) & 1) ? 1 : 2);
    const Layout& L = a.L;
    const double* __restrict__ uc = a.U[bin][C];
    const double* __restrict__ uo = C == 0 ? a.U[bin][1] : a.U[bout][0];
    double* __restrict__ ucw = a.U[bout][C];

    const int z = blockIdx.z;
    const int k = z % L.n3 + 1;
    const int l = z / L.n3 + 1;
    const int j = blockIdx.y * kPassBY + threadIdx.y + 1;
    const int i = 1 + ((1 + j + k + l + C) & 1) + 2 * (int)(blockIdx.x * kPassBX + threadIdx.x);

    double r2 = 0.0;
    if (j <= L.n2 && i <= L.n1) {
        const long long rb = L.row(j, k, l) * L.W;
        const long long p = rb + (i >> 1);
        double c0, c1, c2, c3, c4, c5, c6, c7;
        if constexpr (HEAT) {
            // assemble_heat_step: couplings into ghosts are dropped (solver.cpp:100-103)
            c0 = i > 1 ? a.hc[0] : 0.0;
            c1 = i < L.n1 ? a.hc[0] : 0.0;
            c2 = j > 1 ? a.hc[1] : 0.0;
            c3 = j < L.n2 ? a.hc[1] : 0.0;
            c4 = k > 1 ? a.hc[2] : 0.0;
            c5 = k < L.n3 ? a.hc[2] : 0.0;
            c6 = l > 1 ? a.hc[3] : 0.0;
            c7 = l < L.n4 ? a.hc[3] : 0.0;
        } else {
            const float4* cp = reinterpret_cast<const float4*>(a.coef[C] + p * 8);
            const float4 lo = __ldcs(cp);
            const float4 hi = __ldcs(cp + 1);
            c0 = lo.x; c1 = lo.y; c2 = lo.z; c3 = lo.w;
            c4 = hi.x; c5 = hi.y; c6 = hi.z; c7 = hi.w;
        }
        const double rhs = __ldcs(a.rhs[C] + p);
        const double u0 = __ldg(uc + p);
        const double n0 = __ldg(uo + rb + ((i - 1) >> 1));
        const double n1 = __ldg(uo + rb + ((i + 1) >> 1));
        const double n2 = __ldg(uo + p - L.sj);
        const double n3 = __ldg(uo + p + L.sj);
        const double n4 = __ldg(uo + p - L.sk);
        const double n5 = __ldg(uo + p + L.sk);
        const double n6 = __ldg(uo + p - L.sl);
        const double n7 = __ldg(uo + p + L.sl);

        // solver.cpp:296-312
        const double dg = 1.0 - (c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7);
        double acc = rhs;
        acc -= c0 * n0;
        acc -= c1 * n1;
        acc -= c2 * n2;
        acc -= c3 * n3;
        acc -= c4 * n4;
        acc -= c5 * n5;
        acc -= c6 * n6;
        acc -= c7 * n7;
        const double ubar = acc / dg;
        const double unew = a.omega * ubar + a.keep * u0;
        ucw[p] = unew;
        if constexpr (C == 1) {
            const double res = dg * (unew - ubar);
            r2 = res * res;
        } else {
            // red residual of the incoming state (solver.cpp:347-356)
            double res = dg * u0 - rhs;
            res += c0 * n0;
            res += c1 * n1;
            res += c2 * n2;
            res += c3 * n3;
            res += c4 * n4;
            res += c5 * n5;
            res += c6 * n6;
            res += c7 * n7;
            r2 = res * res;
        }
    }
    r2 = block_sum(r2);
    if (threadIdx.x == 0 && threadIdx.y == 0)
        a.part[C][((long long)z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = r2;
}

// grid = n4 blocks (one per local l-slice), 256 threads
__global__ void __launch_bounds__(256) sor_finalize(const SorArgs a) {
    SorState* st = a.st;
    if (*(volatile int*)&st->done) return;
    const int n = *(volatile int*)&st->n_red;
    if (n >= 2) {
        const int l = blockIdx.x;
        const double* pr = a.part[0] + (long long)l * a.bps;
        const double* pb = a.part[1] + (long long)l * a.bps;
        double r = 0.0, b = 0.0;
        for (int q = threadIdx.x; q < a.bps; q += blockDim.x) {
            r += pr[q];
            b += pb[q];
        }
        r = block_sum(r);
        __syncthreads();
        b = block_sum(b);
        if (threadIdx.x == 0) a.slice_res[l] = b + r;  // slice_black + red (solver.cpp:359)
    }
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    st->counter = 0;
    if (n >= 2) {
        double total = 0.0;
        for (int l = 0; l < (int)gridDim.x; ++l) total += __ldcg(a.slice_res + l);
        const double res = sqrt(total);
        const int it = n - 1;
        st->residual = res;
        st->iterations = it;
        if (!st->fixed && res <= st->tol) {
            st->done = 1;
            st->converged = 1;
        } else if (it >= st->max_iter) {
            st->done = 1;
            st->converged = st->fixed;
        }
    }
    st->n_black = n;
    st->n_red = n + 1;
    if (a.use_cond) cudaGraphSetConditional(a.cond, st->done ? 0u : 1u);
}

__global__ void sor_init(SorState* st, double tol, const double* norm_sq, double rel, int max_iter,
                         int fixed) {
    st->n_red = 1;
    st->n_black = 0;
    st->done = 0;
    st->converged = 0;
    st->iterations = 0;
    st->max_iter = max_iter;
    st->fixed = fixed;
    st->counter = 0;
    st->residual = 0.0;
    st->tol = norm_sq ? rel * sqrt(*norm_sq) : tol;
}

}  // namespace

dim3 pass_grid(const Layout& L) {
    const int nq = (L.n1 + 1) / 2;  // max doxels of one colour per row
    return dim3(ceil_div(nq, kPassBX), ceil_div(L.n2, kPassBY), (unsigned)(L.n3 * L.n4));
}

void launch_sor_init(cudaStream_t s, SorState* st, double tol, const double* norm_sq, double rel,
                     int max_iter, int fixed) {
    sor_init<<<1, 1, 0, s>>>(st, tol, norm_sq, rel, max_iter, fixed);
    SSB_LAUNCHED();
}

void launch_sor_body(cudaStream_t s, const SorArgs& a, bool heat, cudaEvent_t* ev) {
    const dim3 grid = pass_grid(a.L);
    const dim3 block(kPassBX, kPassBY);
    if (ev) SSB_CUDA(cudaEventRecord(ev[0], s));
    if (heat)
        sor_pass<0, true><<<grid, block, 0, s>>>(a);
    else
        sor_pass<0, false><<<grid, block, 0, s>>>(a);
    SSB_LAUNCHED();
    if (ev) SSB_CUDA(cudaEventRecord(ev[1], s));
    sor_finalize<<<a.L.n4, 256, 0, s>>>(a);
    SSB_LAUNCHED();
    if (ev) SSB_CUDA(cudaEventRecord(ev[2], s));
    if (heat)
        sor_pass<1, true><<<grid, block, 0, s>>>(a);
    else
        sor_pass<1, false><<<grid, block, 0, s>>>(a);
    SSB_LAUNCHED();
    if (ev) SSB_CUDA(cudaEventRecord(ev[3], s));
}

}  // namespace ssb
