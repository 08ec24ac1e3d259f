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
#include <algorithm>

#include <cooperative_groups.h>

#include "sor_final.cuh"
#include "sor_math.cuh"

namespace cg = cooperative_groups;

namespace ssb {

namespace {


// CG: the state arrays were written earlier in the SAME launch (resident loop):
// read them through L2 (ld.global.cg), not the non-coherent read-only path.
template <bool CG>
__device__ __forceinline__ double ld_state(const double* p) {
    if constexpr (CG)
        return __ldcg(p);
    else
        return __ldg(p);
}

template <int C, bool HEAT, bool CG = false>
__device__ __forceinline__ void load_doxel(const SorArgs& a, const float* __restrict__ cf,
                                           const double* __restrict__ rh,
                                           const double* __restrict__ uc,
                                           const double* __restrict__ uo, int i, int j, int k,
                                           int l, DoxelIn& d) {
    const Layout& L = a.L;
    const long long rb = L.row(j, k, l) * L.W;
    const long long p = rb + (i >> 1);
    d.p = p;
    if constexpr (HEAT) {
        // assemble_heat_step: couplings into ghosts are dropped (solver.cpp:100-103)
        d.c[0] = i > 1 ? (float)a.hc[0] : 0.f;
        d.c[1] = i < L.n1 ? (float)a.hc[0] : 0.f;
        d.c[2] = j > 1 ? (float)a.hc[1] : 0.f;
        d.c[3] = j < L.n2 ? (float)a.hc[1] : 0.f;
        d.c[4] = k > 1 ? (float)a.hc[2] : 0.f;
        d.c[5] = k < L.n3 ? (float)a.hc[2] : 0.f;
        d.c[6] = l + L.l0 > 1 ? (float)a.hc[3] : 0.f;  // global l boundaries
        d.c[7] = l + L.l0 < L.n4g ? (float)a.hc[3] : 0.f;
    } else {
        const float4* cp = reinterpret_cast<const float4*>(cf + (L.row(j, k, l) * L.Wc + ((i - 1) >> 1)) * 8);
        const float4 lo = __ldcs(cp);
        const float4 hi = __ldcs(cp + 1);
        d.c[0] = lo.x; d.c[1] = lo.y; d.c[2] = lo.z; d.c[3] = lo.w;
        d.c[4] = hi.x; d.c[5] = hi.y; d.c[6] = hi.z; d.c[7] = hi.w;
    }
    d.rhs = __ldcs(rh + p);
    d.u0 = ld_state<CG>(uc + p);
    d.nb[0] = ld_state<CG>(uo + rb + ((i - 1) >> 1));
    d.nb[1] = ld_state<CG>(uo + rb + ((i + 1) >> 1));
    d.nb[2] = ld_state<CG>(uo + p - L.sj);
    d.nb[3] = ld_state<CG>(uo + p + L.sj);
    d.nb[4] = ld_state<CG>(uo + p - L.sk);
    d.nb[5] = ld_state<CG>(uo + p + L.sk);
    d.nb[6] = ld_state<CG>(uo + p - L.sl);
    d.nb[7] = ld_state<CG>(uo + p + L.sl);
}

// Persistent colour pass: a resident grid walks the tiles (kPassBX doxels of one
// colour along i) x (kPassBY rows j) x (kPassKC planes k) of one slice l.  Each
// warp (one row j of a tile) reduces its squared residuals with shuffles and
// writes one partial; the partials of a slice are contiguous and indexed by
// (tile, warp), so the per-slice sums do not depend on the grid size, and no
// block barrier stalls the load pipeline between tiles.
template <int C, bool HEAT, bool CG>
__device__ __forceinline__ void pass_body(const SorArgs& a, int n) {
    const int bout = out_buf(n);
    const int bin = in_buf(n);
    const Layout& L = a.L;
    const double* __restrict__ uc = a.U[bin][C];
    const double* __restrict__ uo = C == 0 ? a.U[bin][1] : a.U[bout][0];
    double* __restrict__ ucw = a.U[bout][C];

    const float* __restrict__ cf = a.coef[C];
    const double* __restrict__ rh = a.rhs[C];
    const long long per_slice = a.tiles / L.n4;
    const long long t_end = (long long)a.l_hi * per_slice;
    for (long long t = (long long)(a.l_lo - 1) * per_slice + blockIdx.x; t < t_end; t += gridDim.x) {
        const int bx = (int)(t % a.tx);
        long long r = t / a.tx;
        const int by = (int)(r % a.ty);
        r /= a.ty;
        const int bk = (int)(r % a.tk);
        const int l = (int)(r / a.tk) + 1;
        const int j = by * kPassBY + threadIdx.y + 1;
        const int q = bx * kPassBX + threadIdx.x;
        const int k0 = bk * kPassKC + 1;
        double r2 = 0.0;
        if (j <= L.n2) {
#pragma unroll
            for (int kb = 0; kb < kPassKC; kb += kPassBatch) {
                DoxelIn d[kPassBatch];
                bool ok[kPassBatch];
#pragma unroll
                for (int b = 0; b < kPassBatch; ++b) {  // all loads of the batch first
                    const int k = k0 + kb + b;
                    const int i = 1 + ((1 + j + k + l + L.lpar + C) & 1) + 2 * q;
                    ok[b] = k <= L.n3 && i <= L.n1;
                    if (ok[b]) load_doxel<C, HEAT, CG>(a, cf, rh, uc, uo, i, j, k, l, d[b]);
                }
#pragma unroll
                for (int b = 0; b < kPassBatch; ++b)
                    if (ok[b]) r2 += compute_doxel<C>(a, d[b], ucw);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r2 += __shfl_down_sync(0xffffffffu, r2, o);
        if (threadIdx.x == 0) a.part[n & 3][C][t * kPassBY + threadIdx.y] = r2;
    }
}

template <int C, bool HEAT>
__global__ void __launch_bounds__(kPassBX * kPassBY, SSB_PASS_MINB) sor_pass(const SorArgs a) {
    SorState* st = a.st;
    if (*(volatile const int*)&st->done) return;
    const int n = C == 0 ? *(volatile const int*)&st->n_red : *(volatile const int*)&st->n_black;
    // the red pass hands its n to the black pass (the decision may run concurrently)
    if (C == 0 && blockIdx.x == 0 && threadIdx.x == 0 && threadIdx.y == 0) st->n_black = n;
    pass_body<C, HEAT, false>(a, n);
}

// Resident pass: the pass's doxel slots of slice l, (k, j, q) with q fastest over
// nq = (n1+1)/2, are cut into aligned chunks of 32; a warp computes one chunk per
// lane set (lane = slot), kResidentBatch chunks with all their loads issued
// first (the state lives in L2: latency, not bandwidth, bounds a pass), and
// writes one partial per chunk at (slice, chunk) -- so per-slice sums do not
// depend on the grid size.  All CTAs' warps share one grid-stride over chunks.
#ifndef SSB_RES_BATCH
#define SSB_RES_BATCH 1
#endif
#ifndef SSB_RES_MINB
#define SSB_RES_MINB 2
#endif
constexpr int kResidentBatch = SSB_RES_BATCH;

__host__ __device__ inline long long resident_chunks(const Layout& L) {
    return ((long long)L.n2 * L.n3 * ((L.n1 + 1) / 2) + 31) / 32;
}

template <int C, bool HEAT>
__device__ __forceinline__ void resident_body(const SorArgs& a, int n) {
    const int bout = out_buf(n);
    const int bin = in_buf(n);
    const Layout& L = a.L;
    const double* __restrict__ uc = a.U[bin][C];
    const double* __restrict__ uo = C == 0 ? a.U[bin][1] : a.U[bout][0];
    double* __restrict__ ucw = a.U[bout][C];
    const float* __restrict__ cf = a.coef[C];
    const double* __restrict__ rh = a.rhs[C];
    const int nq = (L.n1 + 1) / 2;
    const long long cps = resident_chunks(L);  // chunks per slice
    const long long total = cps * L.n4;
    const int lane = threadIdx.x;  // blockDim = (32, 8)
    const long long w0 = (long long)blockIdx.x * blockDim.y + threadIdx.y;
    const long long nw = (long long)gridDim.x * blockDim.y;
    for (long long c0 = w0; c0 < total; c0 += nw * kResidentBatch) {
        DoxelIn d[kResidentBatch];
        bool ok[kResidentBatch];
#pragma unroll
        for (int b = 0; b < kResidentBatch; ++b) {  // all loads of the batch first
            const long long c = c0 + b * nw;
            ok[b] = false;
            if (c >= total) continue;
            const int l = (int)(c / cps) + 1;
            const long long e = (c % cps) * 32 + lane;  // slot within the slice
            const int q = (int)(e % nq);
            const long long rr = e / nq;
            const int j = (int)(rr % L.n2) + 1, k = (int)(rr / L.n2) + 1;
            const int i = 1 + ((1 + j + k + l + L.lpar + C) & 1) + 2 * q;
            ok[b] = k <= L.n3 && i <= L.n1;
            if (ok[b]) load_doxel<C, HEAT, true>(a, cf, rh, uc, uo, i, j, k, l, d[b]);
        }
#pragma unroll
        for (int b = 0; b < kResidentBatch; ++b) {
            const long long c = c0 + b * nw;
            if (c >= total) continue;  // warp-uniform
            double r2 = ok[b] ? compute_doxel<C>(a, d[b], ucw) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) r2 += __shfl_down_sync(0xffffffffu, r2, o);
            if (lane == 0) a.part[n & 3][C][c] = r2;
        }
    }
}

// Resident solve (grids whose working set fits in L2, e.g. BASELINE config 0):
// ONE cooperative launch runs the whole loop -- red pass, grid barrier, slice
// residuals and black pass, grid barrier, the decision (taken by every CTA from
// the same slice values in the same order, so all agree; CTA 0 publishes it) --
// instead of three launches per iteration.  Same tiles, partials,
// per-doxel arithmetic and slice reductions as the other kernels (partials per
// 32-slot chunk, resident_body): iterates bit for bit, iteration counts equal.
// State arrays are read through L2 (they change between passes of the launch).
template <bool HEAT>
__global__ void __launch_bounds__(kPassBX * kPassBY, SSB_RES_MINB) sor_resident(const SorArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double ws[32];
    __shared__ int stop;
    SorState* st = a.st;
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    if (*(volatile int*)&st->done) return;  // uniform: nobody has written st yet
    int n = *(volatile int*)&st->n_red;
    const double tol = st->tol;
    const int fixed = st->fixed, max_iter = st->max_iter;
    grid.sync();  // everyone has read the state before CTA 0 rewrites it
    while (true) {
        resident_body<0, HEAT>(a, n);
        grid.sync();
        // slice residuals of state n-1, then (without waiting for the decision) the
        // black pass of iteration n: if iterate n-1 turns out converged, black(n)
        // only wrote buffer out(n), which nobody reads -- one wasted pass per
        // solve instead of a grid barrier per iteration
        if (n >= 2)
            for (int l = blockIdx.x; l < a.L.n4; l += gridDim.x) {
                const double v = slice_residual(a, n, l, ws, tid);
                if (tid == 0) a.slice_res[l] = v;
                asm volatile("bar.sync 1, 256;" ::: "memory");
            }
        resident_body<1, HEAT>(a, n);
        grid.sync();
        if (tid == 0) {  // sor_decide_state, evaluated by every CTA
            int done = 0, conv = 0;
            double res = 0.0;
            if (n >= 2) {
                double total = 0.0;
                for (int l = 0; l < a.L.n4g; ++l) total += __ldcg(a.all_slices + l);
                res = sqrt(total);
                if (!fixed && res <= tol) {
                    done = conv = 1;
                } else if (n - 1 >= max_iter) {
                    done = 1;
                    conv = fixed;
                }
            }
            if (blockIdx.x == 0) {
                if (n >= 2) {
                    st->residual = res;
                    st->iterations = n - 1;
                }
                st->done = done;
                st->converged = conv;
                st->n_black = n;
                st->n_red = n + 1;
            }
            stop = done;
        }
        __syncthreads();
        if (stop) break;
        ++n;
    }
}

// grid = local n4 blocks (one per owned slice), 256 threads: slice_res[l] via
// slice_residual (sor_final.cuh).  With inline_decide (single slab) the last
// block also takes the decision; otherwise the slices are all-gathered first
// (sor_decide).  The TMA black pass does the same in its head (fuse_final).
__global__ void __launch_bounds__(256) sor_finalize(const SorArgs a) {
    __shared__ double ws[32];
    SorState* st = a.st;
    if (*(volatile int*)&st->done) return;
    const int n = *(volatile int*)&st->n_red;
    if (n >= 2) {
        const double v = slice_residual(a, n, blockIdx.x, ws, threadIdx.x);
        if (threadIdx.x == 0) a.slice_res[blockIdx.x] = v;
    }
    if (!a.inline_decide) return;
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&st->counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    st->counter = 0;
    sor_decide_state(a, st, n);
}

__global__ void sor_decide(const SorArgs a) {
    SorState* st = a.st;
    if (*(volatile int*)&st->done) return;
    sor_decide_state(a, st, *(volatile int*)&st->n_red);
}

// tol = rel * sqrt(sum over all slices in global l order) when norm_slices is given
__global__ void sor_init(SorState* st, double tol, const double* norm_slices, int n_slices, double rel,
                         int max_iter, int fixed, int epoch_base, const int* bad_local,
                         const double* bad_all, int n_all) {
    st->epoch_base = epoch_base;
    st->n_red = 1;
    st->n_black = 0;
    st->done = 0;
    st->converged = 0;
    st->iterations = 0;
    st->max_iter = max_iter;
    st->fixed = fixed;
    st->counter = 0;
    st->item_ctr[0] = st->item_ctr[1] = 0;
    st->residual = 0.0;
    if (norm_slices) {
        double s = 0.0;
        for (int l = 0; l < n_slices; ++l) s += norm_slices[l];
        st->tol = rel * sqrt(s);
    } else {
        st->tol = tol;
    }
    // NumericalError (solver.cpp:71-75) decided on the device: one iteration, not converged,
    // flagged (every slab sees the same all-gathered flags, so every rank stops alike)
    int bad = bad_local && *bad_local != 0;
    for (int q = 0; bad_all && q < n_all; ++q) bad |= bad_all[q] != 0.0;
    st->nonfinite = bad;
    if (bad) {
        st->max_iter = 1;
        st->fixed = 0;
    }
}

__global__ void flag_to_double(const int* flag, double* out) { out[0] = flag[0] != 0 ? 1.0 : 0.0; }

}  // namespace

dim3 pass_grid(const Layout& L) {
    const int nq = (L.n1 + 1) / 2;  // max doxels of one colour per row
    return dim3(ceil_div(nq, kPassBX), ceil_div(L.n2, kPassBY), (unsigned)(L.n3 * L.n4));
}

void pass_tiles(const Layout& L, SorArgs& a) {
    const int nq = (L.n1 + 1) / 2;
    a.tx = (int)ceil_div(nq, kPassBX);
    a.ty = (int)ceil_div(L.n2, kPassBY);
    a.tk = (int)ceil_div(L.n3, kPassKC);
    a.tiles = (long long)a.tx * a.ty * a.tk * L.n4;
    a.bps = a.tx * a.ty * a.tk * kPassBY;  // one partial per warp-row of a tile
}

static int resident_blocks() {
    static int blocks = 0;
    if (!blocks) {
        int dev = 0, sms = 0, per = 0;
        SSB_CUDA(cudaGetDevice(&dev));
        SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sor_pass<0, false>,
                                                               kPassBX * kPassBY, 0));
        blocks = sms * std::max(1, per);
    }
    return blocks;
}

void launch_sor_init(cudaStream_t s, SorState* st, double tol, const double* norm_slices,
                     int n_slices, double rel, int max_iter, int fixed, int epoch_base,
                     const int* bad_local, const double* bad_all, int n_all) {
    sor_init<<<1, 1, 0, s>>>(st, tol, norm_slices, n_slices, rel, max_iter, fixed, epoch_base, bad_local,
                             bad_all, n_all);
    SSB_LAUNCHED();
}

void launch_flag_to_double(cudaStream_t s, const int* flag, double* out) {
    flag_to_double<<<1, 1, 0, s>>>(flag, out);
    SSB_LAUNCHED();
}

void launch_sor_pass(cudaStream_t s, const SorArgs& a, int colour, bool heat) {
    if (a.tma) {
        launch_sor_pass_tma(s, a, colour, heat);
        return;
    }
    const long long items = a.tiles / a.L.n4 * (a.l_hi - a.l_lo + 1);
    const unsigned grid = (unsigned)std::min<long long>(items, resident_blocks());
    const dim3 block(kPassBX, kPassBY);
    if (colour == 0) {
        if (heat)
            sor_pass<0, true><<<grid, block, 0, s>>>(a);
        else
            sor_pass<0, false><<<grid, block, 0, s>>>(a);
    } else {
        if (heat)
            sor_pass<1, true><<<grid, block, 0, s>>>(a);
        else
            sor_pass<1, false><<<grid, block, 0, s>>>(a);
    }
    SSB_LAUNCHED();
}

void launch_sor_pass_range(cudaStream_t s, const SorArgs& a, int colour, bool heat, int lo, int hi, bool dyn) {
    if (lo > hi) return;
    SorArgs b = a;
    b.l_lo = lo;
    b.l_hi = hi;
    b.l_step = 1;
    b.dyn = dyn ? 1 : 0;  // only the interior launch of a pass takes items from the counter
    launch_sor_pass(s, b, colour, heat);
}

void launch_sor_pass_ends(cudaStream_t s, const SorArgs& a, int colour, bool heat) {
    const int n4 = a.L.n4;
    if (n4 <= 2 || !a.tma || a.wave) {  // contiguous, or kernels without strided slice ranges
        launch_sor_pass_range(s, a, colour, heat, 1, 1);
        if (n4 > 1) launch_sor_pass_range(s, a, colour, heat, n4, n4);
        return;
    }
    SorArgs b = a;  // slices 1 and n4 in one launch
    b.l_lo = 1;
    b.l_hi = n4;
    b.l_step = n4 - 1;
    b.pdl_off = 1;
    b.dyn = 0;
    launch_sor_pass(s, b, colour, heat);
}

void launch_sor_finalize(cudaStream_t s, const SorArgs& a) {
    sor_finalize<<<a.L.n4, 256, 0, s>>>(a);
    SSB_LAUNCHED();
}

void launch_sor_decide(cudaStream_t s, const SorArgs& a) {
    sor_decide<<<1, 1, 0, s>>>(a);
    SSB_LAUNCHED();
}

bool resident_supported(const Layout& L) {
    // active working set of one iteration: coefficients + rhs/guess + in + out buffers
    const double bytes = 2.0 * L.rows * L.Wc * 32.0 + 3.0 * 2.0 * L.cs * 8.0;
    return bytes <= 96.0 * 1024 * 1024 && L.glo && L.ghi;
}

size_t resident_partials(const Layout& L) { return (size_t)resident_chunks(L) * L.n4; }

bool launch_sor_resident(cudaStream_t s, const SorArgs& a, bool heat) {
    static int blocks = 0;
    if (!blocks) {
        int dev = 0, sms = 0, per0 = 0, per1 = 0;
        SSB_CUDA(cudaGetDevice(&dev));
        SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per0, sor_resident<false>, kPassBX * kPassBY, 0));
        SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, sor_resident<true>, kPassBX * kPassBY, 0));
        blocks = sms * std::max(1, std::min(per0, per1));
    }
    SorArgs b = a;
    b.bps = (int)resident_chunks(a.L);  // slice partials of resident_body
    const unsigned grid = (unsigned)std::max(1LL, std::min<long long>((resident_chunks(a.L) * a.L.n4 + 7) / 8, blocks));
    void* args[] = {&b};
    const void* fn = heat ? (const void*)sor_resident<true> : (const void*)sor_resident<false>;
    const cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kPassBX, kPassBY), args, 0, s);
    if (e == cudaErrorCooperativeLaunchTooLarge) {  // fewer SMs available than at startup (MPS, ...)
        (void)cudaGetLastError();
        return false;
    }
    SSB_CUDA(e);
    SSB_LAUNCHED();
    return true;
}

void launch_sor_body(cudaStream_t s, const SorArgs& a, bool heat, cudaEvent_t* ev) {
    if (a.wave == 2) {  // one sweep (red + black) in one k-wavefront launch, then the decision
        if (ev) SSB_CUDA(cudaEventRecord(ev[0], s));
        launch_sor_kwave(s, a);
        if (ev) SSB_CUDA(cudaEventRecord(ev[1], s));
        sor_finalize<<<a.L.n4, 256, 0, s>>>(a);
        SSB_LAUNCHED();
        if (ev) {
            SSB_CUDA(cudaEventRecord(ev[2], s));
            SSB_CUDA(cudaEventRecord(ev[3], s));
        }
        return;
    }
    if (a.wave) {  // iterations n and n+1 in one wavefront launch, then both decisions
        if (ev) SSB_CUDA(cudaEventRecord(ev[0], s));
        launch_sor_wave(s, a, heat);
        if (ev) SSB_CUDA(cudaEventRecord(ev[1], s));
        for (int q = 0; q < wave_iters(); ++q) {
            sor_finalize<<<a.L.n4, 256, 0, s>>>(a);
            SSB_LAUNCHED();
        }
        if (ev) {
            SSB_CUDA(cudaEventRecord(ev[2], s));
            SSB_CUDA(cudaEventRecord(ev[3], s));
        }
        return;
    }
    if (ev) SSB_CUDA(cudaEventRecord(ev[0], s));
    launch_sor_pass(s, a, 0, heat);
    if (ev) SSB_CUDA(cudaEventRecord(ev[1], s));
    if (!a.fuse_final) {  // else the black pass takes the decision in its head
        sor_finalize<<<a.L.n4, 256, 0, s>>>(a);
        SSB_LAUNCHED();
    }
    if (ev) SSB_CUDA(cudaEventRecord(ev[2], s));
    launch_sor_pass(s, a, 1, heat);
    if (ev) SSB_CUDA(cudaEventRecord(ev[3], s));
}

}  // namespace ssb
