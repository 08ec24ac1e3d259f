// sor_tma.cu -- TMA-fed red-black SOR colour pass (the hot kernel).
//
// The LDG pass (sor.cu) is latency-bound: every thread waits on eleven global
// loads per doxel.  Here one producer thread per CTA streams, with
// cp.async.bulk (TMA) and mbarrier completion, everything a work item needs
// into a ring of shared-memory stages, and eight consumer warps compute from
// shared memory only; up to kStages-3 planes are in flight per CTA.
//
// Work item = R consecutive rows j0..j0+R-1 (all W packed slots of a row) x a
// chunk of planes k0..k1 of one slice l.  Stage q of an item holds, for plane
// p = k0-1+q:
//     UK   rows j0-1..j0+R of the other colour at (p, l)       (always)
//     COEF R rows of fp32 coefficients of colour C at (p, l)  (interior planes)
//     RHS  R rows of rhs, UC R rows of colour C's own values
//     ULM / ULP  R rows of the other colour at (p, l-1) / (p, l+1)
// so the consumer of plane p reads UK of stages q-1, q, q+1 (the k-1, k, k+1
// neighbours: a rolling window -- each other-colour row is fetched once per
// item, not three times) and everything else from stage q.  Rows of a plane
// are consecutive in the packed layout, so every stream of a stage is ONE
// contiguous bulk copy (W is even: rows are 16-byte aligned).
//
// Residual partials: one per (item, warp), items ordered l-major, so the
// per-slice sums do not depend on the grid size (same contract as sor.cu).
#include <algorithm>

#include "sor_math.cuh"

namespace ssb {

namespace {

constexpr int kWarps = 8;  // "virtual" consumer warps: one row (segment) each, one residual partial each
#ifndef SSB_RPW
#define SSB_RPW 1
#endif
constexpr int kRPW = SSB_RPW;                   // virtual warps computed (interleaved) per physical warp
constexpr int kConsumers = kWarps / kRPW;       // physical consumer warps
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr int kStages = 5;
constexpr int kPlanesPerItem = 8;
#ifndef SSB_WAVE_SKEW
#define SSB_WAVE_SKEW 0  // 0: 2 * nkc sub-slices (measured: nkc+1 starves, 16..48 equal)
#endif

__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sptr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(sptr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sptr(dst)),
        "l"(src), "r"(bytes), "r"(sptr(bar))
        : "memory");
}

struct Geo {  // per-launch tiling (identical on host and device)
    int R;    // rows per item
    int wpr;  // warps per row
    int njg;  // row groups per plane
    int nkc;  // plane chunks per slice
    long long items;
    uint32_t row_bytes;   // one packed row of doubles
    uint32_t stage_bytes;
    uint32_t off_coef, off_rhs, off_uc, off_ulm, off_ulp, off_uk;
};

__host__ __device__ inline Geo make_geo(const Layout& L) {
    Geo g;
    const uint32_t rb = (uint32_t)L.W * 8u;
    int R = 8;
    while (R > 1 && rb * (9u * R + 2u) > 24576u) R >>= 1;
    if (R > L.n2) R = L.n2 < 1 ? 1 : L.n2;
    // keep R a divisor of kWarps so warps map evenly onto rows
    while (kWarps % R) --R;
    g.R = R;
    g.wpr = kWarps / R;
    g.njg = (L.n2 + R - 1) / R;
    g.nkc = (L.n3 + kPlanesPerItem - 1) / kPlanesPerItem;
    g.items = (long long)g.njg * g.nkc * L.n4;
    g.row_bytes = rb;
    g.off_coef = 0;
    g.off_rhs = g.off_coef + 4u * R * rb;  // fp32 x 8 per slot = 4 x a double row
    g.off_uc = g.off_rhs + R * rb;
    g.off_ulm = g.off_uc + R * rb;
    g.off_ulp = g.off_ulm + R * rb;
    g.off_uk = g.off_ulp + R * rb;
    g.stage_bytes = g.off_uk + (R + 2u) * rb;
    return g;
}

// Work item geometry (item = row group jg x plane chunk kc of slice l)
struct Item {
    int l, j0, rows, k0, k1;
};
__device__ __forceinline__ Item make_item(const Layout& L, const Geo& G, int l, int jg, int kc) {
    Item it;
    it.l = l;
    it.j0 = jg * G.R + 1;
    it.rows = min(G.R, L.n2 - it.j0 + 1);
    it.k0 = kc * kPlanesPerItem + 1;
    it.k1 = min(it.k0 + kPlanesPerItem - 1, L.n3);
    return it;
}

struct Ring {  // producer-side position of the next stage
    uint32_t slot = 0, phase = 0, used = 0;
};

// Producer: issue the k1-k0+3 stages of one item (planes k0-1 .. k1+1).
template <bool HEAT>
__device__ __forceinline__ void produce_item(const Layout& L, const Geo& G, unsigned char* smem, uint64_t* full,
                                             uint64_t* empty, Ring& rg, const Item& it, const float* coef,
                                             const double* rhs, const double* uc, const double* uo) {
    const long long W = L.W;
    const long long plane_rows = (long long)L.jMax * L.kMax;
    const uint32_t rb = G.row_bytes;
    for (int p = it.k0 - 1; p <= it.k1 + 1; ++p) {
        if (rg.used >= kStages) mbar_wait(&empty[rg.slot], rg.phase ^ 1);
        unsigned char* s = smem + rg.slot * G.stage_bytes;
        const bool interior = p >= it.k0 && p <= it.k1;
        uint32_t bytes = (it.rows + 2) * rb;
        if (interior) bytes += (HEAT ? 4u : 8u) * it.rows * rb;
        uint64_t* bar = &full[rg.slot];
        mbar_expect_tx(bar, bytes);
        const long long row0 = ((long long)it.l * L.kMax + p) * L.jMax + it.j0;  // row (j0, p, l)
        bulk_g2s(s + G.off_uk, uo + (row0 - 1) * W, (it.rows + 2) * rb, bar);
        if (interior) {
            if (!HEAT) bulk_g2s(s + G.off_coef, coef + row0 * W * 8, 4 * it.rows * rb, bar);
            bulk_g2s(s + G.off_rhs, rhs + row0 * W, it.rows * rb, bar);
            bulk_g2s(s + G.off_uc, uc + row0 * W, it.rows * rb, bar);
            bulk_g2s(s + G.off_ulm, uo + (row0 - plane_rows) * W, it.rows * rb, bar);
            bulk_g2s(s + G.off_ulp, uo + (row0 + plane_rows) * W, it.rows * rb, bar);
        }
        ++rg.used;
        if (++rg.slot == kStages) {
            rg.slot = 0;
            rg.phase ^= 1;
        }
    }
}

// Consumers: update colour C on the item's planes from the staged rows.  Each
// physical warp computes kRPW virtual warps (rows / row segments) with their
// loads and dependency chains interleaved (ILP), and returns each virtual
// warp's sum of squared residuals in r2[].  (s0, ph0) is the ring position of
// the item's first stage and is advanced past the item.
template <int C, bool HEAT>
__device__ __forceinline__ void consume_item(const SorArgs& a, const Layout& L, const Geo& G,
                                             unsigned char* smem, uint64_t* full, uint64_t* empty,
                                             uint32_t& s0, uint32_t& ph0, const Item& it,
                                             double* __restrict__ ucw, int warp, int lane,
                                             double r2[kRPW]) {
    const long long W = L.W;
    const int nq = (L.n1 + 1) / 2;
    const int l = it.l;
    int rloc[kRPW], seg[kRPW], jv[kRPW];
#pragma unroll
    for (int v = 0; v < kRPW; ++v) {
        const int vw = warp * kRPW + v;
        rloc[v] = vw / G.wpr;
        seg[v] = vw % G.wpr;
        jv[v] = it.j0 + rloc[v];
        r2[v] = 0.0;
    }
    // (slot, phase) of stages q-1 (plane p-1), q (p), q+1 (p+1)
    uint32_t sm = s0, pm = ph0;
    uint32_t sc = sm + 1 == kStages ? 0 : sm + 1, pc = sm + 1 == kStages ? pm ^ 1 : pm;
    mbar_wait(&full[sm], pm);
    mbar_wait(&full[sc], pc);
    for (int p = it.k0; p <= it.k1; ++p) {
        const uint32_t sp = sc + 1 == kStages ? 0 : sc + 1, pp = sc + 1 == kStages ? pc ^ 1 : pc;
        mbar_wait(&full[sp], pp);
        const unsigned char* scb = smem + sc * G.stage_bytes;
        const double* ukm = reinterpret_cast<const double*>(smem + sm * G.stage_bytes + G.off_uk);
        const double* ukc = reinterpret_cast<const double*>(scb + G.off_uk);
        const double* ukp = reinterpret_cast<const double*>(smem + sp * G.stage_bytes + G.off_uk);
        const float* cf = reinterpret_cast<const float*>(scb + G.off_coef);
        const double* rh = reinterpret_cast<const double*>(scb + G.off_rhs);
        const double* u0r = reinterpret_cast<const double*>(scb + G.off_uc);
        const double* ulm = reinterpret_cast<const double*>(scb + G.off_ulm);
        const double* ulp = reinterpret_cast<const double*>(scb + G.off_ulp);
        for (int q0 = lane; q0 < nq; q0 += 32 * G.wpr) {
            DoxelIn d[kRPW];
            bool ok[kRPW];
#pragma unroll
            for (int v = 0; v < kRPW; ++v) {  // all loads first
                const int j = jv[v], r = rloc[v];
                const int i = 1 + ((1 + j + p + l + L.lpar + C) & 1) + 2 * (q0 + 32 * seg[v]);
                ok[v] = r < it.rows && q0 + 32 * seg[v] < nq && i <= L.n1;
                if (!ok[v]) continue;
                const int m = i >> 1;
                if constexpr (HEAT) {
                    d[v].c[0] = i > 1 ? (float)a.hc[0] : 0.f;
                    d[v].c[1] = i < L.n1 ? (float)a.hc[0] : 0.f;
                    d[v].c[2] = j > 1 ? (float)a.hc[1] : 0.f;
                    d[v].c[3] = j < L.n2 ? (float)a.hc[1] : 0.f;
                    d[v].c[4] = p > 1 ? (float)a.hc[2] : 0.f;
                    d[v].c[5] = p < L.n3 ? (float)a.hc[2] : 0.f;
                    d[v].c[6] = l + L.l0 > 1 ? (float)a.hc[3] : 0.f;
                    d[v].c[7] = l + L.l0 < L.n4g ? (float)a.hc[3] : 0.f;
                } else {
                    const float* c8 = cf + ((long long)r * W + m) * 8;
                    const float4 lo = *reinterpret_cast<const float4*>(c8);
                    const float4 hi = *reinterpret_cast<const float4*>(c8 + 4);
                    d[v].c[0] = lo.x; d[v].c[1] = lo.y; d[v].c[2] = lo.z; d[v].c[3] = lo.w;
                    d[v].c[4] = hi.x; d[v].c[5] = hi.y; d[v].c[6] = hi.z; d[v].c[7] = hi.w;
                }
                const double* ur = ukc + (r + 1) * W;  // this row in the (rows+2)-row block
                d[v].rhs = rh[r * W + m];
                d[v].u0 = u0r[r * W + m];
                d[v].nb[0] = ur[(i - 1) >> 1];
                d[v].nb[1] = ur[(i + 1) >> 1];
                d[v].nb[2] = ukc[r * W + m];
                d[v].nb[3] = ukc[(r + 2) * W + m];
                d[v].nb[4] = ukm[(r + 1) * W + m];
                d[v].nb[5] = ukp[(r + 1) * W + m];
                d[v].nb[6] = ulm[r * W + m];
                d[v].nb[7] = ulp[r * W + m];
                d[v].p = (((long long)l * L.kMax + p) * L.jMax + j) * W + m;
            }
#ifndef SSB_NOCOMPUTE
#pragma unroll
            for (int v = 0; v < kRPW; ++v)
                if (ok[v]) r2[v] += compute_doxel<C>(a, d[v], ucw);
#else  // data-movement floor experiment: touch the operands, store u0
#pragma unroll
            for (int v = 0; v < kRPW; ++v)
                if (ok[v]) {
                    double s = d[v].rhs + d[v].u0 + (double)d[v].c[0] + (double)d[v].c[7];
                    for (int f = 0; f < 8; ++f) s += d[v].nb[f];
                    ucw[d[v].p] = s;
                    r2[v] += s * 1e-300;
                }
#endif
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sm]);  // plane p-1's stage is done
        sm = sc;
        pm = pc;
        sc = sp;
        pc = pp;
    }
    // the last two stages of the item (planes k1, k1+1)
    __syncwarp();
    if (lane == 0) {
        mbar_arrive(&empty[sm]);
        mbar_arrive(&empty[sc]);
    }
    s0 = sc + 1 == kStages ? 0 : sc + 1;
    ph0 = sc + 1 == kStages ? pc ^ 1 : pc;
#pragma unroll
    for (int v = 0; v < kRPW; ++v)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r2[v] += __shfl_down_sync(0xffffffffu, r2[v], o);
}

__device__ __forceinline__ void init_barriers(uint64_t* full, uint64_t* empty) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

template <int C, bool HEAT>
__global__ void __launch_bounds__(kThreads, 2) sor_pass_tma(const SorArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    const SorState* st = a.st;
    if (*(volatile const int*)&st->done) return;
    const int n = C == 0 ? *(volatile const int*)&st->n_red : *(volatile const int*)&st->n_black;
    const int bout = out_buf(n);
    const int bin = in_buf(n);
    const Layout& L = a.L;
    const double* uc = a.U[bin][C];
    const double* uo = C == 0 ? a.U[bin][1] : a.U[bout][0];
    double* ucw = a.U[bout][C];
    const Geo G = make_geo(L);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long per_slice = (long long)G.njg * G.nkc;
    const long long t_begin = (long long)(a.l_lo - 1) * per_slice, t_end = (long long)a.l_hi * per_slice;
    init_barriers(full, empty);

    if (warp == kConsumers) {  // producer: one thread issues every bulk copy
        if (lane != 0) return;
        Ring rg;
        for (long long t = t_begin + blockIdx.x; t < t_end; t += gridDim.x) {
            const int jg = (int)(t % G.njg);
            const long long r = t / G.njg;
            const Item it = make_item(L, G, (int)(r / G.nkc) + 1, jg, (int)(r % G.nkc));
            produce_item<HEAT>(L, G, smem, full, empty, rg, it, a.coef[C], a.rhs[C], uc, uo);
        }
        return;
    }
    uint32_t s0 = 0, ph0 = 0;
    for (long long t = t_begin + blockIdx.x; t < t_end; t += gridDim.x) {
        const int jg = (int)(t % G.njg);
        const long long r = t / G.njg;
        const Item it = make_item(L, G, (int)(r / G.nkc) + 1, jg, (int)(r % G.nkc));
        double r2[kRPW];
        consume_item<C, HEAT>(a, L, G, smem, full, empty, s0, ph0, it, ucw, warp, lane, r2);
        if (lane == 0)
#pragma unroll
            for (int v = 0; v < kRPW; ++v) a.part[n & 3][C][t * kWarps + warp * kRPW + v] = r2[v];
    }
}

// ---------------------------------------------------------------------------
// Two-iteration wavefront (temporal blocking through L2).
//
// One launch computes iterations n and n+1 as a wavefront over sub-slices
// s = (l-1)*nkc + kc (a slice split into its plane chunks): step sigma runs
// red(n, s=sigma), black(n, sigma-S), red(n+1, sigma-2S), black(n+1, sigma-3S)
// with skew S = 2*nkc sub-slices, each split into the row-group items above.
// A phase depends on the previous phase at most one slice + one chunk ahead,
// i.e. on items of earlier steps only.
// MEASURED (config 1, B200): 122 us per colour pass vs 111 us for the two-pass
// kernel -- DRAM reads per two sweeps only fall from 2.07 to 1.76 GB: with
// enough skew for ~300 CTAs to find independent work, a slice's rows are
// evicted from L2 before the second iteration reuses them.  Kept as an
// option (kernel 2), not the default.  An item waits (producer, spinning on
// per-item completion flags in global memory) for the items of the previous
// phase that produced the rows it reads: the same chunk at l-1, l, l+1 and
// the in-plane neighbour chunks (jg +- 1, kc +- 1) at l.  Items are taken in
// sequence order by a resident persistent grid, so the earliest unfinished
// item never waits on an unfinished one (no deadlock).  With the slices of
// ~4 wavefront steps resident in L2 (config 1: ~67 MB of 126 MB), the
// coefficient, rhs and state rows of a slice are read from DRAM about once
// per TWO sweeps.  Iterates are unchanged: every update reads exactly the
// values it reads in the two-pass order (the outputs rotate over 3 buffers, so
// nothing a later phase writes is read by an earlier one), and residual
// partials go to the same per-iteration slots, decided afterwards by two
// finalize launches.
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <bool HEAT>
__global__ void __launch_bounds__(kThreads, 2) sor_wave_tma(const SorArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    const SorState* st = a.st;
    if (*(volatile const int*)&st->done) return;
    const int n = *(volatile const int*)&st->n_red;
    const int epoch = *(volatile const int*)&st->epoch_base + n;
    const Layout& L = a.L;
    const Geo G = make_geo(L);
    const int CH = G.njg * G.nkc;  // items per slice and phase
    // wavefront over sub-slices s = (l-1)*nkc + kc: phase d of step sigma works on
    // s = sigma - skew*d; each step has 4 phases x njg row groups
    const int skew = SSB_WAVE_SKEW > 0 ? SSB_WAVE_SKEW : 2 * G.nkc;
    const long long NS = (long long)L.n4 * G.nkc;
    const long long NT = (NS + 3LL * skew) * 4 * G.njg;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    init_barriers(full, empty);

    auto decode = [&](long long t, int& d, int& l, int& c) {
        const int jg = (int)(t % G.njg);
        const long long r = t / G.njg;
        d = (int)(r & 3);
        const long long s = (r >> 2) - (long long)skew * d;  // sub-slice of this phase
        if (s < 0 || s >= NS) {
            l = 0;
            c = 0;
            return;
        }
        l = (int)(s / G.nkc) + 1;
        c = (int)(s % G.nkc) * G.njg + jg;
    };

    if (warp == kConsumers) {  // producer
        if (lane != 0) return;
        Ring rg;
        for (long long t = blockIdx.x; t < NT; t += gridDim.x) {
            int d, l, c;
            decode(t, d, l, c);
            if (l < 1 || l > L.n4) continue;
            const int m = n + (d >> 1), C = d & 1;
            const int jg = c % G.njg, kc = c / G.njg;
            if (d > 0) {  // wait for the producing phase d-1 around this item
                const int* f = a.flags + (long long)(d - 1) * L.n4 * CH;
                auto wait = [&](int ll, int cc) {
                    const int* q = f + (long long)(ll - 1) * CH + cc;
                    while (ld_acquire(q) != epoch) __nanosleep(64);
                };
                wait(l, c);
                if (l > 1) wait(l - 1, c);
                if (l < L.n4) wait(l + 1, c);
                if (jg > 0) wait(l, c - 1);
                if (jg + 1 < G.njg) wait(l, c + 1);
                if (kc > 0) wait(l, c - G.njg);
                if (kc + 1 < G.nkc) wait(l, c + G.njg);
                asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
            }
            const int bin = in_buf(m), bout = out_buf(m);
            const double* uc = a.U[bin][C];
            const double* uo = C == 0 ? a.U[bin][1] : a.U[bout][0];
            const Item it = make_item(L, G, l, jg, kc);
            produce_item<HEAT>(L, G, smem, full, empty, rg, it, a.coef[C], a.rhs[C], uc, uo);
        }
        return;
    }
    uint32_t s0 = 0, ph0 = 0;
    for (long long t = blockIdx.x; t < NT; t += gridDim.x) {
        int d, l, c;
        decode(t, d, l, c);
        if (l < 1 || l > L.n4) continue;
        const int m = n + (d >> 1), C = d & 1;
        const int jg = c % G.njg, kc = c / G.njg;
        const Item it = make_item(L, G, l, jg, kc);
        double* ucw = a.U[out_buf(m)][C];
        double r2[kRPW];
        if (C == 0)
            consume_item<0, HEAT>(a, L, G, smem, full, empty, s0, ph0, it, ucw, warp, lane, r2);
        else
            consume_item<1, HEAT>(a, L, G, smem, full, empty, s0, ph0, it, ucw, warp, lane, r2);
        if (lane == 0)
#pragma unroll
            for (int v = 0; v < kRPW; ++v)
                a.part[m & 3][C][((long long)(l - 1) * CH + c) * kWarps + warp * kRPW + v] = r2[v];
        // publish: every consumer's stores, then one flag store (release)
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
        if (threadIdx.x == 0) {
            int* q = a.flags + ((long long)d * L.n4 + (l - 1)) * CH + c;
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(q), "r"(epoch) : "memory");
        }
    }
}

template <int C, bool HEAT>
void configure() {
    static bool done = false;
    if (!done) {
        SSB_CUDA(cudaFuncSetAttribute(sor_pass_tma<C, HEAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      96 * 1024 + 64 * 1024));
        done = true;
    }
}

template <bool HEAT>
void configure_wave() {
    static bool done = false;
    if (!done) {
        SSB_CUDA(cudaFuncSetAttribute(sor_wave_tma<HEAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      96 * 1024 + 64 * 1024));
        done = true;
    }
}

// resident CTAs for this kernel and shared-memory size (the wavefront kernel
// relies on every CTA being resident: items wait only on earlier items)
int tma_blocks(const void* fn, size_t smem_bytes) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        SSB_CUDA(cudaGetDevice(&dev));
        SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    int per = 0;
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kThreads, smem_bytes));
    return sms * std::max(1, per);
}

}  // namespace

bool tma_pass_supported(const Layout& L) {
    const Geo G = make_geo(L);
    return (size_t)G.stage_bytes * kStages <= 160 * 1024;
}

void tma_pass_tiles(const Layout& L, SorArgs& a) {
    const Geo G = make_geo(L);
    a.tiles = G.items;
    a.bps = G.njg * G.nkc * kWarps;  // partials per slice: one per (item, warp)
    a.tx = G.njg;
    a.ty = G.nkc;
    a.tk = 1;
}

size_t tma_partials(const Layout& L) { return (size_t)make_geo(L).items * kWarps; }

size_t wave_flags(const Layout& L) {
    const Geo G = make_geo(L);
    return (size_t)4 * L.n4 * G.njg * G.nkc;
}

bool wave_supported(const Layout& L) {
    // the slices of ~4 wavefront steps (coefficients 32 B + rhs + 3 states ~ 64 B per
    // doxel) must stay in L2 for the temporal blocking to pay; one slab only
    const double slice = (double)L.n1 * L.n2 * L.n3 * 64.0;
    return tma_pass_supported(L) && L.glo && L.ghi && 4.0 * slice <= 80.0 * 1024 * 1024;
}

void launch_sor_wave(cudaStream_t s, const SorArgs& a, bool heat) {
    const Geo G = make_geo(a.L);
    const size_t smem = (size_t)G.stage_bytes * kStages;
    configure_wave<false>();
    configure_wave<true>();
    configure<0, false>();
    static size_t last_smem = 0;
    static int blocks = 0;
    if (smem != last_smem) {
        blocks = std::min(tma_blocks((const void*)sor_wave_tma<false>, smem),
                          tma_blocks((const void*)sor_wave_tma<true>, smem));
        last_smem = smem;
    }
    const int skew = SSB_WAVE_SKEW > 0 ? SSB_WAVE_SKEW : 2 * G.nkc;
    const long long NT = ((long long)a.L.n4 * G.nkc + 3LL * skew) * 4 * G.njg;
    const unsigned grid = (unsigned)std::min<long long>(NT, blocks);
    if (heat)
        sor_wave_tma<true><<<grid, kThreads, smem, s>>>(a);
    else
        sor_wave_tma<false><<<grid, kThreads, smem, s>>>(a);
    SSB_LAUNCHED();
}

void launch_sor_pass_tma(cudaStream_t s, const SorArgs& a, int colour, bool heat) {
    const Geo G = make_geo(a.L);
    const size_t smem = (size_t)G.stage_bytes * kStages;
    configure<0, false>();
    configure<1, false>();
    configure<0, true>();
    configure<1, true>();
    static size_t last_smem = 0;
    static int blocks = 0;
    if (smem != last_smem) {
        blocks = tma_blocks((const void*)sor_pass_tma<0, false>, smem);
        last_smem = smem;
    }
    const long long items = (long long)G.njg * G.nkc * (a.l_hi - a.l_lo + 1);
    const unsigned grid = (unsigned)std::min<long long>(items, blocks);
    if (colour == 0) {
        if (heat)
            sor_pass_tma<0, true><<<grid, kThreads, smem, s>>>(a);
        else
            sor_pass_tma<0, false><<<grid, kThreads, smem, s>>>(a);
    } else {
        if (heat)
            sor_pass_tma<1, true><<<grid, kThreads, smem, s>>>(a);
        else
            sor_pass_tma<1, false><<<grid, kThreads, smem, s>>>(a);
    }
    SSB_LAUNCHED();
}

}  // namespace ssb
