// sor_final.cuh -- the end-of-red-pass bookkeeping of one SOR iteration
// (solver.cpp:195-205), shared by the stand-alone finalize kernel (sor.cu), the
// TMA black pass that performs it in its head (sor_tma.cu) and the resident
// solve (sor.cu).
//
// slice_res[l] = (sum of the black(n-1) partials of slice l) + (sum of the
// red(n) partials of slice l), each summed by 256 threads in one fixed order;
// the decision sums the slices in global l order.  Both callers use exactly
// these functions, so iterates and iteration counts do not depend on which
// path ran.
#pragma once

#include "kernels.cuh"

namespace ssb {

// The fixed-shape 256-lane tree, run by NT = 256 or 128 threads (tid 0..NT-1,
// named barrier 1): thread tid plays lanes tid + k*NT, k < 256/NT, so the sum is
// the same bits whichever NT runs it.
template <int NT = 256>
__device__ __forceinline__ double group256_sum(const double (&v)[256 / NT], double* ws, int tid) {
    constexpr int V = 256 / NT;
#pragma unroll
    for (int k = 0; k < V; ++k) {
        double x = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if ((tid & 31) == 0) ws[(tid + k * NT) >> 5] = x;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    double x = 0.0;
    if (tid < 32) {
        x = tid < 8 ? ws[tid] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    }
    return x;  // valid in tid 0
}
__device__ __forceinline__ double group256_sum(double v, double* ws, int tid) {
    const double a[1] = {v};
    return group256_sum<256>(a, ws, tid);
}

// residual of slice l (local, 0-based) of state n-1; valid in tid 0
template <int NT = 256>
__device__ __forceinline__ double slice_residual(const SorArgs& a, int n, int l, double* ws, int tid) {
    constexpr int V = 256 / NT;
    const double* pr = a.part[n & 3][0] + (long long)l * a.bps;        // red(n)
    const double* pb = a.part[(n - 1) & 3][1] + (long long)l * a.bps;  // black(n-1)
    double r[V], b[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        r[k] = 0.0;
        b[k] = 0.0;
        for (int q = tid + k * NT; q < a.bps; q += 256) {
            r[k] += __ldcg(pr + q);
            b[k] += __ldcg(pb + q);
        }
    }
    const double rs = group256_sum<NT>(r, ws, tid);
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    const double bs = group256_sum<NT>(b, ws, tid);
    return bs + rs;  // slice_black + red (solver.cpp:359)
}

// Decision of iteration n-1 from the per-slice residuals of ALL slices in
// global l order (solver.cpp:195-205): identical on every rank.
__device__ __forceinline__ void sor_decide_state(const SorArgs& a, SorState* st, int n) {
    if (n >= 2) {
        double total = 0.0;  // sequential in l; loads issued 8 at a time
        for (int l0 = 0; l0 < a.L.n4g; l0 += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = l0 + q < a.L.n4g ? __ldcg(a.all_slices + l0 + q) : 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (l0 + q < a.L.n4g) total += v[q];
        }
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

// Finalize in the head of the black pass (fuse_final): CTAs l < n4 (grid-stride)
// compute slice l's residual of state n-1 -- red(n) is complete, the black pass
// runs after it -- and the CTA that completes the last slice decides.  The
// black pass of iteration n runs whatever the decision (if iterate n-1 has
// converged it only writes buffer out(n), which nobody reads).  Called by the
// NT consumer threads of a CTA (the same bits for NT = 128 or 256).
template <int NT = 256>
__device__ __forceinline__ void black_head_finalize(const SorArgs& a, int n, double* ws, int* last, int tid) {
    int mine = 0;
    for (int l = blockIdx.x; l < a.L.n4; l += gridDim.x) {
        if (n >= 2) {
            const double v = slice_residual<NT>(a, n, l, ws, tid);
            if (tid == 0) a.slice_res[l] = v;
        }
        ++mine;
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
    }
    if (!mine) return;
    if (tid == 0) {
        __threadfence();
        SorState* st = a.st;
        *last = atomicAdd(&st->counter, (unsigned)mine) + mine == (unsigned)a.L.n4;
        if (*last) {
            __threadfence();
            st->counter = 0;
            sor_decide_state(a, st, n);
        }
    }
}

}  // namespace ssb
