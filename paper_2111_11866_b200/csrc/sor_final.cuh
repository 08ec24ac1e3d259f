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

// 256 threads (tid 0..255) synchronised with named barrier 1: fixed-shape tree
__device__ __forceinline__ double group256_sum(double v, double* ws, int tid) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) ws[tid >> 5] = v;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (tid < 32) {
        v = tid < 8 ? ws[tid] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;  // valid in tid 0
}

// residual of slice l (local, 0-based) of state n-1; valid in tid 0
__device__ __forceinline__ double slice_residual(const SorArgs& a, int n, int l, double* ws, int tid) {
    const double* pr = a.part[n & 3][0] + (long long)l * a.bps;        // red(n)
    const double* pb = a.part[(n - 1) & 3][1] + (long long)l * a.bps;  // black(n-1)
    double r = 0.0, b = 0.0;
    for (int q = tid; q < a.bps; q += 256) {
        r += __ldcg(pr + q);
        b += __ldcg(pb + q);
    }
    r = group256_sum(r, ws, tid);
    asm volatile("bar.sync 1, 256;" ::: "memory");
    b = group256_sum(b, ws, tid);
    return b + r;  // slice_black + red (solver.cpp:359)
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
// 256 consumer threads of a CTA.
__device__ __forceinline__ void black_head_finalize(const SorArgs& a, int n, double* ws, int* last, int tid) {
    int mine = 0;
    for (int l = blockIdx.x; l < a.L.n4; l += gridDim.x) {
        if (n >= 2) {
            const double v = slice_residual(a, n, l, ws, tid);
            if (tid == 0) a.slice_res[l] = v;
        }
        ++mine;
        asm volatile("bar.sync 1, 256;" ::: "memory");
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
