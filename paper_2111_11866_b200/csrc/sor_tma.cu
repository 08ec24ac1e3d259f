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

constexpr int kWarps = 8;         // consumer warps
constexpr int kThreads = (kWarps + 1) * 32;
constexpr int kStages = 5;
constexpr int kPlanesPerItem = 8;

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
    const double* __restrict__ uc = a.U[bin][C];
    const double* __restrict__ uo = C == 0 ? a.U[bin][1] : a.U[bout][0];
    double* __restrict__ ucw = a.U[bout][C];
    const Geo G = make_geo(L);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const long long W = L.W;
    const long long plane_rows = (long long)L.jMax * L.kMax;  // rows per l-plane
    if (warp == kWarps) {
        // ---------------- producer: one thread issues every bulk copy
        if (lane != 0) return;
        uint32_t slot = 0, phase = 0, used = 0;  // ring position of the next stage
        for (long long t = blockIdx.x; t < G.items; t += gridDim.x) {
            const int jg = (int)(t % G.njg);
            long long r = t / G.njg;
            const int kc = (int)(r % G.nkc);
            const int l = (int)(r / G.nkc) + 1;
            const int j0 = jg * G.R + 1;
            const int rows = min(G.R, L.n2 - j0 + 1);
            const int k0 = kc * kPlanesPerItem + 1;
            const int k1 = min(k0 + kPlanesPerItem - 1, L.n3);
            for (int p = k0 - 1; p <= k1 + 1; ++p) {
                if (used >= kStages) mbar_wait(&empty[slot], phase ^ 1);
                unsigned char* s = smem + slot * G.stage_bytes;
                const bool interior = p >= k0 && p <= k1;
                const uint32_t rb = G.row_bytes;
                uint32_t bytes = (rows + 2) * rb;
                if (interior) bytes += (HEAT ? 4u : 8u) * rows * rb;
                mbar_expect_tx(&full[slot], bytes);
                const long long row0 = ((long long)l * L.kMax + p) * L.jMax + j0;  // row (j0, p, l)
                bulk_g2s(s + G.off_uk, uo + (row0 - 1) * W, (rows + 2) * rb, &full[slot]);
                if (interior) {
                    if (!HEAT) bulk_g2s(s + G.off_coef, a.coef[C] + row0 * W * 8, 4 * rows * rb, &full[slot]);
                    bulk_g2s(s + G.off_rhs, a.rhs[C] + row0 * W, rows * rb, &full[slot]);
                    bulk_g2s(s + G.off_uc, uc + row0 * W, rows * rb, &full[slot]);
                    bulk_g2s(s + G.off_ulm, uo + (row0 - plane_rows) * W, rows * rb, &full[slot]);
                    bulk_g2s(s + G.off_ulp, uo + (row0 + plane_rows) * W, rows * rb, &full[slot]);
                }
                ++used;
                if (++slot == kStages) {
                    slot = 0;
                    phase ^= 1;
                }
            }
        }
        return;
    }

    // ---------------- consumers
    const int rloc = warp / G.wpr, seg = warp % G.wpr;
    const int nq = (L.n1 + 1) / 2;
    uint32_t s0 = 0, ph0 = 0;  // ring slot / phase of the item's first stage (plane k0-1)
    for (long long t = blockIdx.x; t < G.items; t += gridDim.x) {
        const int jg = (int)(t % G.njg);
        long long r = t / G.njg;
        const int kc = (int)(r % G.nkc);
        const int l = (int)(r / G.nkc) + 1;
        const int j0 = jg * G.R + 1;
        const int rows = min(G.R, L.n2 - j0 + 1);
        const int k0 = kc * kPlanesPerItem + 1;
        const int k1 = min(k0 + kPlanesPerItem - 1, L.n3);
        double r2 = 0.0;
        const int j = j0 + rloc;
        // (slot, phase) of stages q-1 (plane p-1), q (p), q+1 (p+1)
        uint32_t sm = s0, pm = ph0;
        uint32_t sc = sm + 1 == kStages ? 0 : sm + 1, pc = sm + 1 == kStages ? pm ^ 1 : pm;
        mbar_wait(&full[sm], pm);
        mbar_wait(&full[sc], pc);
        for (int p = k0; p <= k1; ++p) {
            const uint32_t sp = sc + 1 == kStages ? 0 : sc + 1, pp = sc + 1 == kStages ? pc ^ 1 : pc;
            mbar_wait(&full[sp], pp);
            if (rloc < rows) {
                const unsigned char* scb = smem + sc * G.stage_bytes;
                const double* ukm = reinterpret_cast<const double*>(smem + sm * G.stage_bytes + G.off_uk);
                const double* ukc = reinterpret_cast<const double*>(scb + G.off_uk);
                const double* ukp = reinterpret_cast<const double*>(smem + sp * G.stage_bytes + G.off_uk);
                const float* cf = reinterpret_cast<const float*>(scb + G.off_coef) + (long long)rloc * W * 8;
                const double* rh = reinterpret_cast<const double*>(scb + G.off_rhs) + rloc * W;
                const double* u0r = reinterpret_cast<const double*>(scb + G.off_uc) + rloc * W;
                const double* ulm = reinterpret_cast<const double*>(scb + G.off_ulm) + rloc * W;
                const double* ulp = reinterpret_cast<const double*>(scb + G.off_ulp) + rloc * W;
                const double* ukc_r = ukc + (rloc + 1) * W;  // this row in the (rows+2)-row block
                const long long grow = (((long long)l * L.kMax + p) * L.jMax + j) * W;
                const int i0 = 1 + ((1 + j + p + l + L.lpar + C) & 1);
                for (int qq = seg * 32 + lane; qq < nq; qq += 32 * G.wpr) {
                    const int i = i0 + 2 * qq;
                    if (i > L.n1) break;
                    const int m = i >> 1;
                    DoxelIn d;
                    if constexpr (HEAT) {
                        d.c[0] = i > 1 ? (float)a.hc[0] : 0.f;
                        d.c[1] = i < L.n1 ? (float)a.hc[0] : 0.f;
                        d.c[2] = j > 1 ? (float)a.hc[1] : 0.f;
                        d.c[3] = j < L.n2 ? (float)a.hc[1] : 0.f;
                        d.c[4] = p > 1 ? (float)a.hc[2] : 0.f;
                        d.c[5] = p < L.n3 ? (float)a.hc[2] : 0.f;
                        d.c[6] = l + L.l0 > 1 ? (float)a.hc[3] : 0.f;
                        d.c[7] = l + L.l0 < L.n4g ? (float)a.hc[3] : 0.f;
                    } else {
                        const float4 lo = *reinterpret_cast<const float4*>(cf + m * 8);
                        const float4 hi = *reinterpret_cast<const float4*>(cf + m * 8 + 4);
                        d.c[0] = lo.x; d.c[1] = lo.y; d.c[2] = lo.z; d.c[3] = lo.w;
                        d.c[4] = hi.x; d.c[5] = hi.y; d.c[6] = hi.z; d.c[7] = hi.w;
                    }
                    d.rhs = rh[m];
                    d.u0 = u0r[m];
                    d.nb[0] = ukc_r[(i - 1) >> 1];
                    d.nb[1] = ukc_r[(i + 1) >> 1];
                    d.nb[2] = ukc[rloc * W + m];
                    d.nb[3] = ukc[(rloc + 2) * W + m];
                    d.nb[4] = ukm[(rloc + 1) * W + m];
                    d.nb[5] = ukp[(rloc + 1) * W + m];
                    d.nb[6] = ulm[m];
                    d.nb[7] = ulp[m];
                    d.p = grow + m;
                    r2 += compute_doxel<C>(a, d, ucw);
                }
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
        for (int o = 16; o > 0; o >>= 1) r2 += __shfl_down_sync(0xffffffffu, r2, o);
        if (lane == 0) a.part[n & 3][C][t * kWarps + warp] = r2;
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

int tma_blocks(size_t smem_bytes) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        SSB_CUDA(cudaGetDevice(&dev));
        SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    int per = 0;
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sor_pass_tma<0, false>, kThreads, smem_bytes));
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
        blocks = tma_blocks(smem);
        last_smem = smem;
    }
    const unsigned grid = (unsigned)std::min<long long>(G.items, blocks);
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
