// sor_tma.cu -- TMA-fed red-black SOR colour pass (the hot kernel).
//
// The LDG pass (sor.cu) is latency-bound: every thread waits on eleven global
// loads per doxel.  Here two producer threads per CTA stream, with
// cp.async.bulk (TMA) and mbarrier completion, everything a work item needs
// into two rings of shared-memory stages, and eight consumer warps compute from
// shared memory only.
//
// Work item = R consecutive rows j0..j0+R-1 (all W packed slots of a row) x a
// chunk of planes k0..k1 of one slice l.  Per plane p the item needs
//     UK   rows j0-1..j0+R of the other colour at (p, l)       (planes k0-1..k1+1)
//     COEF R rows of fp32 coefficients of colour C at (p, l)  (planes k0..k1)
//     RHS  R rows of rhs, UC R rows of colour C's own values
//     ULM / ULP  R rows of the other colour at (p, l-1) / (p, l+1)
// The consumer of plane p reads UK of planes p-1, p, p+1 (a rolling window:
// each other-colour row is fetched once per item) and the rest of plane p
// only, so UK stages live in their own ring (held for three planes) and the
// main stages (COEF..ULP, released after one plane) in another: the main ring
// keeps kMainStages-1 planes in flight per CTA.  Rows of a plane are
// consecutive in the packed layout, so every stream of a stage is ONE
// contiguous bulk copy (W is even: rows are 16-byte aligned).
//
// Item order: slice-fastest (order 1), so items of slices l-1, l, l+1 at the
// same (jg, kc) run together and the ULM/ULP rows hit L2 even when one slice
// is larger than L2; black passes walk the items backwards (snake), starting
// where the red pass ended.  Residual partials: one per (item, warp) at the
// item's canonical slice-major id, so per-slice sums do not depend on the
// traversal or the grid size (same contract as sor.cu).
#include <algorithm>
#include <cstring>
#include <string>

#include <cudaTypedefs.h>
#include <cstdlib>

#include "sor_final.cuh"
#include "sor_math.cuh"

namespace ssb {

namespace {

#ifndef SSB_CONSUMER_WARPS
#define SSB_CONSUMER_WARPS 8
#endif
#ifndef SSB_CTAS_PER_SM
#define SSB_CTAS_PER_SM 2
#endif
constexpr int kWarps = SSB_CONSUMER_WARPS;  // consumer warps, one residual partial each per item
constexpr int kConsumers = kWarps;
constexpr int kSlotsPerPlane = kConsumers * 32;   // consumer threads: one slot each (flat mapping)
constexpr int kThreads = (kConsumers + 2) * 32;  // + a producer warp per ring
#ifndef SSB_FLAT_WARPS
#define SSB_FLAT_WARPS 8
#endif
// flat-mapping kernels: kFlatWarps consumer warps, each thread kFlatV of the 256 slots
constexpr int kFlatWarps = SSB_FLAT_WARPS;
constexpr int kFlatV = kWarps / kFlatWarps;
static_assert(kFlatWarps * kFlatV == kWarps && (kFlatV == 1 || kFlatV == 2), "SSB_FLAT_WARPS: 8 or 4");
#ifndef SSB_SPLIT_MAIN
#define SSB_SPLIT_MAIN 0  // flat kernels: a second main-ring producer thread issues the l-1 / l+1 rows
#endif
constexpr int kSplitMain = SSB_SPLIT_MAIN;
#ifndef SSB_DYN_ITEMS
#define SSB_DYN_ITEMS 1  // flat single-range passes: items handed out by an atomic counter (else round-robin;
                         // measured: config 2 -2.2% per sweep, config 1 unchanged)
#endif
constexpr int kItemQ = 4;  // item indices a CTA's main producer may publish ahead of its readers
__host__ __device__ constexpr int pass_threads(bool flat) {
    return ((flat ? kFlatWarps + kSplitMain : kConsumers) + 2) * 32;
}
#ifndef SSB_MAIN_STAGES
#define SSB_MAIN_STAGES 4
#endif
#ifndef SSB_UK_STAGES
#define SSB_UK_STAGES 6
#endif
#ifndef SSB_STAGE_BUDGET
#define SSB_STAGE_BUDGET 24576  // bytes of one main + one UK stage that bound the rows per item
#endif
constexpr int kMainStages = SSB_MAIN_STAGES;  // per-plane operands (consumed by one plane)
constexpr int kUKStages = SSB_UK_STAGES;      // other-colour planes (held for three planes)
#ifndef SSB_FULL_ROWS
// 1: the flat consumer also rewrites a row's ghost/pad slots, so row stores cover whole
// 32-byte sectors.  MEASURED (config 1 red pass, ncu): DRAM reads 502.6 -> 493.1 MB (the
// L2 fills of partial sectors), but +25% instructions; per sweep config 1 -1%, config 2
// +5.5% (power-capped clock).  Off.
#define SSB_FULL_ROWS 0
#endif
#ifndef SSB_PLANES_PER_ITEM
#define SSB_PLANES_PER_ITEM 32  // measured: 8 -> 16 planes: config 2/4 -6%, config 1 -1% per sweep (fewer k-halo rows);
                                // 16 -> 32 under the power cap: config 4 -1.0%, config 2 -0.5%, config 1 -1.0% (64: config 1 +4%)
#endif
constexpr int kPlanesPerItem = SSB_PLANES_PER_ITEM;
#ifndef SSB_SMALL_SLICE_ITEMS
#define SSB_SMALL_SLICE_ITEMS 148  // whole-row items per slice (at kPlanesPerItem) below which items are halved
#endif
constexpr int kSmallSliceItems = SSB_SMALL_SLICE_ITEMS;
constexpr int kDefaultSnake = 1;
constexpr int kDefaultL2Hint = 0;
// -1 = auto: slice-major (0) when a slice has at most half a grid of items -- several
// slices are in flight, so the l +- 1 rows AND the row-group / plane-chunk halo rows of
// an item come from L2 (config 1: 197 -> 190 us per sweep) -- else slice-fastest (1),
// which keeps the l +- 1 rows in L2 when a slice is larger than the grid (config 2:
// slice-major 1619 vs 1446 us)
constexpr int kDefaultOrder = -1;
#ifndef SSB_WAVE_SKEW
#define SSB_WAVE_SKEW 0  // 0: 2 * nkc sub-slices (measured: nkc+1 starves, 16..48 equal)
#endif
#ifndef SSB_WAVE_PHASES
#define SSB_WAVE_PHASES 4  // colour phases per wavefront launch: 4 = two iterations, 2 = one sweep
#endif
constexpr int kWavePH = SSB_WAVE_PHASES;

__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared-memory loads at a 32-bit shared address (+ a constant byte offset).  volatile:
// they stay behind the mbarrier waits (also volatile asm) that publish the stage.
template <int OFF>
__device__ __forceinline__ double lds_f64(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(addr), "n"(OFF));
    return v;
}
template <int OFF>
__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+%5];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr), "n"(OFF));
    return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sptr(bar)) : "memory");
}
#ifndef SSB_SOR_FLOOR
#define SSB_SOR_FLOOR 0
#endif
#ifndef SSB_SOR_NOLPM
#define SSB_SOR_NOLPM 0  // (timing-only build, WRONG results) skip the l-1 / l+1 row copies
#endif
#ifndef SSB_SOR_SUSPEND
#define SSB_SOR_SUSPEND 0  // try_wait suspend-time hint in ns (0: the hardware's default)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if constexpr (SSB_SOR_SUSPEND > 0) {
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
            "@!p bra WAIT_%=;\n"
            "}\n" ::"r"(sptr(bar)),
            "r"(parity), "n"(SSB_SOR_SUSPEND)
            : "memory");
    } else {
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
}
__device__ __forceinline__ void mbar_expect_tx_u(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// bulk copy with the destination and barrier as shared-window addresses
__device__ __forceinline__ void bulk_g2s_u(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

// 2D tensor copy (box at coordinates {x, y}) with mbarrier completion
__device__ __forceinline__ void tensor_g2s(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            sptr(dst)),
        "l"(map), "r"(x), "r"(y), "r"(sptr(bar))
        : "memory");
}

// L2 eviction policies (createpolicy): streamed-once operands vs state rows
struct Policies {
    uint64_t stream, uload, ustore;
};
__device__ __forceinline__ Policies make_policies(int hint) {
    uint64_t first, last, normal;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(first));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(last));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(normal));
    Policies p;
    p.stream = hint & 1 ? first : normal;
    p.uload = hint & 2 ? last : normal;
    p.ustore = hint & 4 ? last : normal;
    return p;
}

struct Geo {  // per-launch tiling (identical on host and device)
    int R;    // rows per item
    int wpr;  // warps per row (wide rows), 0: flat slot mapping (R * nq <= 256)
    int njg;  // row groups per plane
    int nkc;  // plane chunks per slice
    int ppi;  // planes per item (chunk)
    long long items;
    uint32_t row_bytes;   // one packed row of doubles
    uint32_t coef_row_bytes;  // one row of fp32 coefficients (Wc slots x 8)
    uint32_t main_bytes;  // one main stage: COEF RHS UC ULM ULP of a plane
    uint32_t uk_bytes;    // one UK stage: R+2 other-colour rows of a plane
    uint32_t off_coef, off_rhs, off_uc, off_ulm, off_ulp;
    uint32_t off_ukring;  // the UK ring follows the main ring
    uint32_t smem;
    int S;     // 2D-tiled items: slots per segment (kTileS), 0: whole rows
    int nsg;   // segments per row (1 for whole rows)
    int pw;    // row pitch of a staged fp64 block, in slots (W, or kTileS + 2)
    int cpw;   // row pitch of the staged coefficients, in floats (Wc * 8, or kTileS * 8)
};

__host__ __device__ inline Geo make_geo(const Layout& L, bool tile2d = false) {
    Geo g;
    const int nq = (L.n1 + 1) / 2;  // slots of one colour per row
    if (tile2d) {  // kTileR rows x kTileS-slot segments, every thread one slot
        g.R = kTileR;
        g.wpr = 0;
        g.S = kTileS;
        g.nsg = (nq + kTileS - 1) / kTileS;
        g.pw = kTileS + 2;
        g.cpw = kTileS * 8;
        g.njg = (L.n2 + kTileR - 1) / kTileR;
        g.ppi = kPlanesPerItem;
        g.nkc = (L.n3 + kPlanesPerItem - 1) / kPlanesPerItem;
        g.items = (long long)g.nsg * g.njg * g.nkc * L.n4;
        g.row_bytes = (uint32_t)g.pw * 8u;
        g.coef_row_bytes = (uint32_t)g.cpw * 4u;
        g.off_coef = 0;
        g.off_rhs = g.R * g.coef_row_bytes;
        g.off_uc = g.off_rhs + g.R * g.row_bytes;
        g.off_ulm = g.off_uc + g.R * g.row_bytes;
        g.off_ulp = g.off_ulm + g.R * g.row_bytes;
        g.main_bytes = g.off_ulp + g.R * g.row_bytes;
        // tensor copies land on 128-byte aligned shared addresses
        auto up128 = [](uint32_t x) { return (x + 127u) & ~127u; };
        g.off_uc = up128(g.off_uc);
        g.off_ulm = up128(g.off_uc + g.R * g.row_bytes);
        g.off_ulp = up128(g.off_ulm + g.R * g.row_bytes);
        g.main_bytes = up128(g.off_ulp + g.R * g.row_bytes);
        g.uk_bytes = up128((g.R + 2u) * g.row_bytes);
        g.off_ukring = kMainStages * g.main_bytes;
        g.smem = g.off_ukring + kUKStages * g.uk_bytes;
        return g;
    }
    g.S = 0;
    g.nsg = 1;
    g.pw = L.W;
    g.cpw = L.Wc * 8;
    const uint32_t rb = (uint32_t)L.W * 8u;
    const uint32_t crb = (uint32_t)L.Wc * 32u;
    // Rows per item.  Rows up to 256 slots: the 256 consumer threads take one slot
    // each over the item's R rows (flat mapping), so pick R <= 256 / nq filling the
    // most threads (ties: more rows, fewer halo rows) within the stage budget --
    // 32 slots: 8 rows, 128: 2, 40: 6, 80: 3.  Wider rows: one row, 8 warps along it.
    int R = 1;
    if (nq <= kSlotsPerPlane) {
        int best = 0;
        for (int r = 1; r <= kSlotsPerPlane / nq && r <= L.n2; ++r) {
            if (r > 1 && r * (crb + 4u * rb) + (r + 2u) * rb > (uint32_t)SSB_STAGE_BUDGET) break;
            if (r * nq >= best) {
                best = r * nq;
                R = r;
            }
        }
    }
    g.R = R;
    g.wpr = nq <= kSlotsPerPlane ? 0 : kWarps;  // 0: flat mapping
    g.njg = (L.n2 + R - 1) / R;
    // planes per item: kPlanesPerItem, halved when a slice has few items (then the launch
    // runs slice-major and the items' plane-chunk halo rows come from L2; config 1: -0.7%
    // per sweep with 8 planes, config 2 (large slices) +1.8%, so it keeps 16)
    g.ppi = kPlanesPerItem;
    if (g.njg * ((L.n3 + kPlanesPerItem - 1) / kPlanesPerItem) <= kSmallSliceItems && kPlanesPerItem >= 4)
        g.ppi = kPlanesPerItem / 2;
    g.nkc = (L.n3 + g.ppi - 1) / g.ppi;
    g.items = (long long)g.njg * g.nkc * L.n4;
    g.row_bytes = rb;
    g.off_coef = 0;
    g.coef_row_bytes = (uint32_t)L.Wc * 32u;
    g.off_rhs = g.off_coef + R * g.coef_row_bytes;
    g.off_uc = g.off_rhs + R * rb;
    g.off_ulm = g.off_uc + R * rb;
    g.off_ulp = g.off_ulm + R * rb;
    g.main_bytes = g.off_ulp + R * rb;
    g.uk_bytes = (R + 2u) * rb;
    g.off_ukring = kMainStages * g.main_bytes;
    g.smem = g.off_ukring + kUKStages * g.uk_bytes;
    return g;
}

// Work item geometry (item = row group jg x plane chunk kc of slice l)
struct Item {
    int l, j0, rows, k0, k1;
    int s0;  // first slot (2D-tiled items), 0 for whole rows
};
__device__ __forceinline__ Item make_item(const Layout& L, const Geo& G, int l, int jg, int kc, int sg = 0) {
    Item it;
    it.l = l;
    it.s0 = sg * G.S;
    it.j0 = jg * G.R + 1;
    it.rows = min(G.R, L.n2 - it.j0 + 1);
    it.k0 = kc * G.ppi + 1;
    it.k1 = min(it.k0 + G.ppi - 1, L.n3);
    return it;
}

// Launch-local item t (0 .. items of slices l_lo..l_hi) -> its Item and canonical
// id ((l-1)*nkc + kc)*njg + jg, which indexes the residual partials (so per-slice
// sums are independent of the traversal).  order 0: slice-major; order 1: slice
// fastest, so the items of slices l-1, l, l+1 at the same (jg, kc) run
// concurrently and share their other-colour rows through L2 (a slice of a large
// grid is bigger than L2).
__device__ __forceinline__ long long decode_item(const Layout& L, const Geo& G, int order, int l_lo, int nl,
                                                 long long t64, Item& it, int l_step = 1) {
    // item counts stay far below 2^31 (host_launch checks), so 32-bit division suffices
    const unsigned t = (unsigned)t64;
    unsigned l, jg, kc, sg;
    const unsigned nsg = (unsigned)G.nsg, njg = (unsigned)G.njg, nkc = (unsigned)G.nkc;
    if (order == 0) {
        sg = t % nsg;
        const unsigned c2 = t / nsg;
        jg = c2 % njg;
        const unsigned r = c2 / njg;
        kc = r % nkc;
        l = (unsigned)l_lo + (r / nkc) * (unsigned)l_step;
    } else if (order == 1) {
        const unsigned r0 = t / (unsigned)nl;
        l = (unsigned)l_lo + (t - r0 * (unsigned)nl) * (unsigned)l_step;
        const unsigned r = nsg == 1 ? r0 : r0 / nsg;
        sg = r0 - r * nsg;
        kc = r / njg;
        jg = r - kc * njg;
    } else {  // 2: slice fastest, then plane chunk (k-halo planes shared by neighbours in time)
        const unsigned r0 = t / (unsigned)nl;
        l = (unsigned)l_lo + (t - r0 * (unsigned)nl) * (unsigned)l_step;
        const unsigned r = nsg == 1 ? r0 : r0 / nsg;
        sg = r0 - r * nsg;
        jg = r / nkc;
        kc = r - jg * nkc;
    }
    it = make_item(L, G, (int)l, (int)jg, (int)kc, (int)sg);
    return (((long long)(l - 1) * nkc + kc) * njg + jg) * nsg + sg;
}

template <int N>
struct Ring {  // producer-side position of the next stage of an N-stage ring
    uint32_t slot = 0, phase = 0, used = 0;
    __device__ __forceinline__ void acquire(uint64_t* empty) {
        if (used >= N) mbar_wait(&empty[slot], phase ^ 1);
    }
    __device__ __forceinline__ void advance() {
        ++used;
        if (++slot == N) {
            slot = 0;
            phase ^= 1;
        }
    }
};

// consumer-side ring position
template <int N>
__device__ __forceinline__ void next_stage(uint32_t& slot, uint32_t& phase) {
    if (++slot == N) {
        slot = 0;
        phase ^= 1;
    }
}

// Main producer: one stage per interior plane k0..k1 of the item.
template <bool HEAT>
__device__ __forceinline__ void produce_main(const Layout& L, const Geo& G, unsigned char* smem, uint64_t* full,
                                             uint64_t* empty, Ring<kMainStages>& rg, const Item& it,
                                             const float* coef, const double* rhs, const double* uc,
                                             const double* uo, const Policies& pol,
                                             const CUtensorMap* const* tm = nullptr, bool issue = true,
                                             int part = 0) {
    const long long W = L.W;
    const long long plane_rows = (long long)L.jMax * L.kMax;
    const uint32_t rb = G.row_bytes;
    if (G.S) {  // 2D-tiled: one tensor copy per stream, full boxes (out-of-range slots read as 0)
        const CUtensorMap* const* m = tm;
        for (int p = it.k0; p <= it.k1; ++p) {
            rg.acquire(empty);
            unsigned char* s = smem + rg.slot * G.main_bytes;
            uint64_t* bar = &full[rg.slot];
            const int row0 = (int)(((long long)it.l * L.kMax + p) * L.jMax + it.j0);
            if (issue) {
                mbar_expect_tx(bar, (HEAT ? 0u : G.R * G.coef_row_bytes) + 4u * G.R * rb);
                if (!HEAT) tensor_g2s(s + G.off_coef, m[0], it.s0 * 8, row0, bar);
                tensor_g2s(s + G.off_rhs, m[1], it.s0, row0, bar);
                tensor_g2s(s + G.off_uc, m[2], it.s0, row0, bar);
                tensor_g2s(s + G.off_ulm, m[3], it.s0, row0 - (int)plane_rows, bar);
                tensor_g2s(s + G.off_ulp, m[3], it.s0, row0 + (int)plane_rows, bar);
            }
            rg.advance();
        }
        return;
    }
    // the item's five row blocks of plane k0; every stream advances by one plane (jMax rows)
    // per stage, so the loop only adds strides (the per-plane products were a third of the
    // producer's instructions, and producer instructions take issue slots from the consumers)
    const long long row0 = ((long long)it.l * L.kMax + it.k0) * L.jMax + it.j0;  // row (j0, k0, l)
    const char* pc = reinterpret_cast<const char*>(coef + row0 * L.Wc * 8);
    const char* pr = reinterpret_cast<const char*>(rhs + row0 * W);
    const char* pu = reinterpret_cast<const char*>(uc + row0 * W);
    const char* pm = reinterpret_cast<const char*>(uo + (row0 - plane_rows) * W);
    const char* pp = reinterpret_cast<const char*>(uo + (row0 + plane_rows) * W);
    const long long dc = (long long)L.jMax * L.Wc * 32, ds = (long long)L.jMax * W * 8;
    const uint32_t bc = it.rows * G.coef_row_bytes, br = it.rows * rb;
    // part 0: every stream; split producers: part 1 coef / rhs / own colour, part 2 the l +- 1 rows
    const uint32_t b1 = (HEAT ? 0u : bc) + 2u * br, b2 = SSB_SOR_NOLPM && !HEAT ? 0u : 2u * br;
    const uint32_t tx = part == 0 ? b1 + b2 : part == 1 ? b1 : b2;
    const uint32_t sm0 = sptr(smem), bar0 = sptr(full);
    for (int p = it.k0; p <= it.k1; ++p) {
        rg.acquire(empty);
        const uint32_t st = sm0 + rg.slot * G.main_bytes, bar = bar0 + rg.slot * 8u;
        if (issue) {
            mbar_expect_tx_u(bar, tx);
            if (part != 2) {
                if (!HEAT) bulk_g2s_u(st + G.off_coef, pc, bc, bar, pol.stream);
                bulk_g2s_u(st + G.off_rhs, pr, br, bar, pol.stream);
                bulk_g2s_u(st + G.off_uc, pu, br, bar, pol.uload);
            }
            if (part != 1 && !(SSB_SOR_NOLPM && !HEAT)) {
                bulk_g2s_u(st + G.off_ulm, pm, br, bar, pol.uload);
                bulk_g2s_u(st + G.off_ulp, pp, br, bar, pol.uload);
            }
        }
        pc += dc;
        pr += ds;
        pu += ds;
        pm += ds;
        pp += ds;
        rg.advance();
    }
}

// UK producer: the other colour's rows j0-1..j0+rows of planes k0-1 .. k1+1.
__device__ __forceinline__ void produce_uk(const Layout& L, const Geo& G, unsigned char* smem, uint64_t* full,
                                           uint64_t* empty, Ring<kUKStages>& rg, const Item& it, const double* uo,
                                           const Policies& pol, const CUtensorMap* uk_map = nullptr,
                                           bool issue = true) {
    const long long W = L.W;
    const uint32_t rb = G.row_bytes;
    if (G.S) {
        for (int p = it.k0 - 1; p <= it.k1 + 1; ++p) {
            rg.acquire(empty);
            unsigned char* s = smem + G.off_ukring + rg.slot * G.uk_bytes;
            uint64_t* bar = &full[rg.slot];
            const int row0 = (int)(((long long)it.l * L.kMax + p) * L.jMax + it.j0);
            if (issue) {
                mbar_expect_tx(bar, (G.R + 2u) * rb);  // the box's bytes (the stage is padded to 128 B)
                tensor_g2s(s, uk_map, it.s0, row0 - 1, bar);
            }
            rg.advance();
        }
        return;
    }
    // rows j0-1 .. j0+rows of plane k0-1, advancing one plane per stage
    const char* pk =
        reinterpret_cast<const char*>(uo + ((((long long)it.l * L.kMax + it.k0 - 1) * L.jMax + it.j0) - 1) * W);
    const long long ds = (long long)L.jMax * W * 8;
    const uint32_t bytes = (it.rows + 2) * rb;
    const uint32_t sk0 = sptr(smem) + G.off_ukring, bar0 = sptr(full);
    for (int p = it.k0 - 1; p <= it.k1 + 1; ++p) {
        rg.acquire(empty);
        const uint32_t bar = bar0 + rg.slot * 8u;
        if (issue) {
            mbar_expect_tx_u(bar, bytes);
            bulk_g2s_u(sk0 + rg.slot * G.uk_bytes, pk, bytes, bar, pol.uload);
        }
        pk += ds;
        rg.advance();
    }
}

// Consumers: update colour C on the item's planes from the staged rows.  Warp w
// owns row w / wpr of the item and the slot segment w % wpr; with parity
// par = (1 + j + k + l + C) & 1 its doxels of plane k sit at i = 1 + par + 2q,
// i.e. packed slot m = q + par, with the i-1 / i+1 neighbours at slots q and q+1
// of the other colour's row -- so every address is a loop-invariant base plus
// q, and only par flips from plane to plane.  Returns the warp's sum of squared
// residuals.  (ms, mph) / (s0, ph0) are the main / UK ring positions of the
// item's first stages and are advanced past the item.
template <int C, bool HEAT, bool PUSH = false>
__device__ __forceinline__ double consume_item(const SorArgs& a, const Layout& L, const Geo& G,
                                               unsigned char* smem, uint64_t* fullM, uint64_t* emptyM,
                                               uint64_t* fullK, uint64_t* emptyK, uint32_t& ms,
                                               uint32_t& mph, uint32_t& s0, uint32_t& ph0, const Item& it,
                                               double* __restrict__ ucw, int warp, int lane,
                                               uint64_t pol_store, double* push_lo = nullptr,
                                               double* push_hi = nullptr) {
    const int W = L.W;
    // this thread's row r and first slot: flat (one slot per thread over the item's
    // R rows) or, for rows wider than 256 slots, 8 warps striding along the row
    const int nq = (L.n1 + 1) / 2;
    const int tid = warp * 32 + lane;
    // 2D-tiled items (G.S): warp = row, lane = slot of the segment at it.s0
    const int r = G.S ? warp : (G.wpr ? warp / G.wpr : tid / nq);
    const int q_begin = G.S ? it.s0 + lane : (G.wpr ? lane + 32 * (warp % G.wpr) : tid - r * nq);
    const int q_step = G.wpr && !G.S ? 32 * G.wpr : 1 << 30;
    const int PW = G.pw;      // staged row pitch (slots)
    const int sb0 = it.s0;    // global slot of the staged block's first column
    const int j = it.j0 + r;
    const bool row_ok = r < it.rows;  // (flat: tid < R * nq  <=>  r < R)
    // last slot q with i = 1 + par + 2q <= n1, per parity
    const int q_end0 = (L.n1 - 1) >> 1, q_end1 = (L.n1 - 2) >> 1;
    int par = (1 + j + it.k0 + it.l + L.lpar + C) & 1;
    // shared-memory element offsets of row r: R-row blocks / the (R+2)-row UK block
    const int o_row = r * PW - sb0, o_uk = (r + 1) * PW - sb0;  // index staged rows by GLOBAL slot
    double* wrow = ucw + L.row(j, it.k0, it.l) * (long long)W;  // this row at plane k0
    // halo push: the same row in the neighbours' arrays (first / last owned plane only)
    double* wlo = PUSH && push_lo ? push_lo + (wrow - ucw) + a.push_lo_off : nullptr;
    double* whi = PUSH && push_hi ? push_hi + (wrow - ucw) + a.push_hi_off : nullptr;
    const long long wstep = (long long)L.jMax * W;
    const unsigned char* ukr = smem + G.off_ukring;
    double r2 = 0.0;
    // UK (slot, phase) of planes p-1, p, p+1; main stage (ms, mph) of plane p
    uint32_t sm = s0, pm = ph0;
    uint32_t sc = sm, pc = pm;
    next_stage<kUKStages>(sc, pc);
    mbar_wait(&fullK[sm], pm);
    mbar_wait(&fullK[sc], pc);
    for (int p = it.k0; p <= it.k1; ++p) {
        uint32_t sp = sc, pp = pc;
        next_stage<kUKStages>(sp, pp);
        mbar_wait(&fullK[sp], pp);
        mbar_wait(&fullM[ms], mph);
        const unsigned char* mb = smem + ms * G.main_bytes;
        const double* ukm = reinterpret_cast<const double*>(ukr + sm * G.uk_bytes) + o_uk;
        const double* ukc = reinterpret_cast<const double*>(ukr + sc * G.uk_bytes) + o_uk;
        const double* ukp = reinterpret_cast<const double*>(ukr + sp * G.uk_bytes) + o_uk;
        const float* cf = reinterpret_cast<const float*>(mb + G.off_coef) + r * G.cpw - 8 * sb0;
        const double* rh = reinterpret_cast<const double*>(mb + G.off_rhs) + o_row;
        const double* u0r = reinterpret_cast<const double*>(mb + G.off_uc) + o_row;
        const double* ulm = reinterpret_cast<const double*>(mb + G.off_ulm) + o_row;
        const double* ulp = reinterpret_cast<const double*>(mb + G.off_ulp) + o_row;
        const int q_end = par ? q_end1 : q_end0;
        if (row_ok)
            for (int q = q_begin; q <= q_end; q += q_step) {
                const int m = q + par;
                DoxelIn d;
                if constexpr (HEAT) {
                    const int i = 1 + par + 2 * q;
                    d.c[0] = i > 1 ? (float)a.hc[0] : 0.f;
                    d.c[1] = i < L.n1 ? (float)a.hc[0] : 0.f;
                    d.c[2] = j > 1 ? (float)a.hc[1] : 0.f;
                    d.c[3] = j < L.n2 ? (float)a.hc[1] : 0.f;
                    d.c[4] = p > 1 ? (float)a.hc[2] : 0.f;
                    d.c[5] = p < L.n3 ? (float)a.hc[2] : 0.f;
                    d.c[6] = it.l + L.l0 > 1 ? (float)a.hc[3] : 0.f;
                    d.c[7] = it.l + L.l0 < L.n4g ? (float)a.hc[3] : 0.f;
                } else {
                    const float4 lo = *reinterpret_cast<const float4*>(cf + 8 * q);  // slot q <-> i = 1 + par + 2q
                    const float4 hi = *reinterpret_cast<const float4*>(cf + 8 * q + 4);
                    d.c[0] = lo.x; d.c[1] = lo.y; d.c[2] = lo.z; d.c[3] = lo.w;
                    d.c[4] = hi.x; d.c[5] = hi.y; d.c[6] = hi.z; d.c[7] = hi.w;
                }
                d.rhs = rh[m];
                d.u0 = u0r[m];
                d.nb[0] = ukc[q];
                d.nb[1] = ukc[q + 1];
                d.nb[2] = ukc[m - PW];
                d.nb[3] = ukc[m + PW];
                d.nb[4] = ukm[m];
                d.nb[5] = ukp[m];
                d.nb[6] = ulm[m];
                d.nb[7] = ulp[m];
                d.p = m;
#ifndef SSB_NOCOMPUTE
                r2 += compute_doxel<C, true, PUSH>(a, d, wrow, pol_store, wlo, whi);
#else  // data-movement floor experiment: touch the operands, store u0
                double t = d.rhs + d.u0 + (double)d.c[0] + (double)d.c[7];
                for (int f = 0; f < 8; ++f) t += d.nb[f];
                wrow[m] = t;
                r2 += t * 1e-300;
#endif
            }
        __syncwarp();
        mbar_arrive(&emptyM[ms]);  // plane p's operands are done (every consumer thread arrives)
        mbar_arrive(&emptyK[sm]);  // and plane p-1's other-colour rows
        next_stage<kMainStages>(ms, mph);
        sm = sc;
        pm = pc;
        sc = sp;
        pc = pp;
        par ^= 1;
        wrow += wstep;
        if constexpr (PUSH) {
            if (wlo) wlo += wstep;
            if (whi) whi += wstep;
        }
    }
    // the last two UK stages of the item (planes k1, k1+1)
    __syncwarp();
    mbar_arrive(&emptyK[sm]);
    mbar_arrive(&emptyK[sc]);
    next_stage<kUKStages>(sc, pc);
    s0 = sc;
    ph0 = pc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r2 += __shfl_down_sync(0xffffffffu, r2, o);
    return r2;
}

// Per-thread constants of the flat slot mapping (rows of <= 256 slots, whole-row
// items): thread tid owns row r = tid / nq, slot q = tid % nq of every item.
struct FlatThread {
    int r, q;
    uint32_t t_coef;  // byte offset of its 8 coefficients in a main stage
    uint32_t t_row;   // byte offset of slot q of row r in an R-row block
    uint32_t t_uk;    // byte offset of slot q of row r + 1 in the (R+2)-row UK block
    uint32_t act;     // bit par: slot q holds a doxel of parity par (q <= q_end[par])
    // slots of the row no doxel of parity par covers (the i-ghost and the even-W pad):
    // [0, par) and [hi[par], W).  The row's first / last thread rewrites them with the
    // input row's values (equal in every state buffer), so the row store covers whole
    // 32-byte sectors and L2 does not fill the partial ones from DRAM.
    uint32_t fill;    // bit 0: first thread of its row, bit 1: last thread of its row
    int hi0, hi1;     // hi[par] - q: first high fill slot relative to q
};
__device__ __forceinline__ FlatThread flat_thread(const Layout& L, const Geo& G, int tid) {
    FlatThread f;
    const int nq = (L.n1 + 1) / 2;
    f.r = tid / nq;
    f.q = tid - f.r * nq;
    const int ra = f.r < G.R ? f.r : 0;  // idle threads (r >= R) read row 0's operands
    f.t_coef = G.off_coef + (uint32_t)(ra * G.cpw + 8 * f.q) * 4u;
    f.t_row = (uint32_t)(ra * G.pw + f.q) * 8u;
    f.t_uk = (uint32_t)((ra + 1) * G.pw + f.q) * 8u;
    f.act = (f.q <= ((L.n1 - 1) >> 1) ? 1u : 0u) | (f.q <= ((L.n1 - 2) >> 1) ? 2u : 0u);
    f.fill = SSB_FULL_ROWS && f.r < G.R ? (f.q == 0 ? 1u : 0u) | (f.q == nq - 1 ? 2u : 0u) : 0u;
    f.hi0 = ((L.n1 - 1) >> 1) + 1 - f.q;
    f.hi1 = ((L.n1 - 2) >> 1) + 2 - f.q;
    return f;
}

// consume_item for the flat mapping: the same update, with every shared-memory
// address a per-thread constant plus a stage base carried from plane to plane
// (the general version re-derives its addresses per plane: ~35 integer
// instructions per warp-plane against ~90 for the arithmetic itself).
template <int C, bool PUSH, int V, bool RES = true>
__device__ __forceinline__ void consume_item_flat(const SorArgs& a, const Layout& L, const Geo& G,
                                                  const FlatThread (&ft)[V], uint32_t sbase, uint64_t* fullM,
                                                  uint64_t* emptyM, uint64_t* fullK, uint64_t* emptyK, uint32_t& ms,
                                                  uint32_t& mph, uint32_t& s0, uint32_t& ph0, const Item& it,
                                                  double* __restrict__ ucw, double* push_lo, double* push_hi,
                                                  double (&r2)[V]) {
    // V virtual threads per thread (slots tid + k * consumer threads): their updates
    // are independent, so they are computed branch-free side by side and stored
    // under a predicate
    uint32_t act[V], par[V], trow[V];
    double* wq[V];
    double* wlo[V];
    double* whi[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const int j = it.j0 + ft[k].r;
        act[k] = ft[k].r < it.rows ? ft[k].act : 0u;
        par[k] = (uint32_t)(1 + j + it.k0 + it.l + L.lpar + C) & 1u;
        const long long row0 = L.row(j, it.k0, it.l) * (long long)L.W + ft[k].q;
        wq[k] = ucw + row0;  // slot q of this row at plane k0 (+ par: the doxel's slot)
        wlo[k] = PUSH && push_lo ? push_lo + row0 + a.push_lo_off : nullptr;
        whi[k] = PUSH && push_hi ? push_hi + row0 + a.push_hi_off : nullptr;
        trow[k] = ft[k].t_row;
        r2[k] = 0.0;
    }
    long long wstep = (long long)L.jMax * L.W;
    asm("" : "+l"(wstep));  // opaque: keep it in registers, not re-derived per plane
    const uint32_t pwb = (uint32_t)G.pw * 8u;
    // shared addresses: UK stages of planes p-1, p, p+1 (stage bases), main stage of p
    const uint32_t ukb = sbase + G.off_ukring;
    uint32_t sm = s0, pm = ph0;
    uint32_t sc = sm, pc = pm;
    next_stage<kUKStages>(sc, pc);
    uint32_t am = ukb + sm * G.uk_bytes, ac = ukb + sc * G.uk_bytes;
    uint32_t amain = sbase + ms * G.main_bytes;
    mbar_wait(&fullK[sm], pm);
    mbar_wait(&fullK[sc], pc);
    for (int p = it.k0; p <= it.k1; ++p) {
        uint32_t sp = sc, pp = pc;
        next_stage<kUKStages>(sp, pp);
        const uint32_t ap = sp == 0 ? ukb : ac + G.uk_bytes;
        mbar_wait(&fullK[sp], pp);
        mbar_wait(&fullM[ms], mph);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const bool on = (act[k] >> par[k]) & 1u;
            if (V == 1 && !on) continue;
            const uint32_t par8 = par[k] * 8u;
            const uint32_t cf = amain + ft[k].t_coef;
            const uint32_t x = amain + trow[k] + par8;  // slot m = q + par of row r
            const uint32_t yc = ac + ft[k].t_uk;         // slot q of the UK row r + 1
            const uint32_t y = yc + par8;                // slot m of the UK row r + 1
            const float4 lo = lds_f4<0>(cf), hi = lds_f4<16>(cf);
            DoxelIn d;
            d.c[0] = lo.x; d.c[1] = lo.y; d.c[2] = lo.z; d.c[3] = lo.w;
            d.c[4] = hi.x; d.c[5] = hi.y; d.c[6] = hi.z; d.c[7] = hi.w;
            d.rhs = lds_f64<0>(x + G.off_rhs);
            d.u0 = lds_f64<0>(x + G.off_uc);
            d.nb[0] = lds_f64<0>(yc);  // slot q   <-> i - 1
            d.nb[1] = lds_f64<8>(yc);  // slot q+1 <-> i + 1
            d.nb[2] = lds_f64<0>(y - pwb);
            d.nb[3] = lds_f64<0>(y + pwb);
            d.nb[4] = lds_f64<0>(am + ft[k].t_uk + par8);
            d.nb[5] = lds_f64<0>(ap + ft[k].t_uk + par8);
#if SSB_SOR_NOLPM  // (timing only) the l-1 / l+1 neighbours replaced by the slice's own other-colour value
            d.nb[6] = lds_f64<0>(y);
            d.nb[7] = lds_f64<0>(y);
#else
            d.nb[6] = lds_f64<0>(x + G.off_ulm);
            d.nb[7] = lds_f64<0>(x + G.off_ulp);
#endif
            double unew, e2;
            if constexpr (RES) {
#if SSB_SOR_FLOOR >= 2
                unew = d.u0;
                e2 = 0.0;
#else
                doxel_update<C>(a, d, unew, e2);
#endif
            } else {  // fixed-sweep solves before their last iteration: the update alone
#if SSB_SOR_FLOOR == 3  // (timing only) the full arithmetic, but the old value written back
                {
                    double t;
                    doxel_update_nores<C>(a, d, t);
                    asm volatile("" ::"d"(t));
                    unew = d.u0;
                }
#elif SSB_SOR_FLOOR  // (timing-only build, WRONG results) every operand loaded, no arithmetic
                unsigned long long x = (unsigned long long)__double_as_longlong(d.rhs) ^
                                       (unsigned long long)__double_as_longlong(d.u0) ^ __float_as_uint(d.c[0]) ^
                                       __float_as_uint(d.c[3]) ^ __float_as_uint(d.c[5]) ^ __float_as_uint(d.c[7]);
#pragma unroll
                for (int f = 0; f < 8; ++f) x ^= (unsigned long long)__double_as_longlong(d.nb[f]);
                unew = SSB_SOR_FLOOR == 2 ? d.u0 : __longlong_as_double((long long)x);  // 2: u stays finite
#else
                doxel_update_nores<C>(a, d, unew);
#endif
                e2 = 0.0;
            }
            if (on) {
                wq[k][par[k]] = unew;
                if constexpr (PUSH) {
                    if (wlo[k]) wlo[k][par[k]] = unew;
                    if (whi[k]) whi[k][par[k]] = unew;
                }
                r2[k] += e2;
            }
            if (SSB_FULL_ROWS && ft[k].fill && ft[k].r < it.rows) {  // ghost / pad slots of the row
                const uint32_t xu = amain + trow[k] + G.off_uc;         // slot q of the input row
                if ((ft[k].fill & 1u) && par[k]) wq[k][0] = lds_f64<0>(xu);
                if (ft[k].fill & 2u)
                    for (int e = par[k] ? ft[k].hi1 : ft[k].hi0; ft[k].q + e < L.W; ++e)
                        wq[k][e] = lds_f64<0>(xu + 8u * (uint32_t)e);
            }
        }
        // every consumer thread arrives for itself (release: its reads are done)
        mbar_arrive(&emptyM[ms]);  // plane p's operands
        mbar_arrive(&emptyK[sm]);  // plane p-1's other-colour rows
        if (++ms == kMainStages) {
            ms = 0;
            mph ^= 1u;
            amain = sbase;
        } else {
            amain += G.main_bytes;
        }
        sm = sc;
        pm = pc;
        sc = sp;
        pc = pp;
        am = ac;
        ac = ap;
#pragma unroll
        for (int k = 0; k < V; ++k) {
            par[k] ^= 1u;
            wq[k] += wstep;
            if constexpr (PUSH) {
                if (wlo[k]) wlo[k] += wstep;
                if (whi[k]) whi[k] += wstep;
            }
        }
    }
    mbar_arrive(&emptyK[sm]);
    mbar_arrive(&emptyK[sc]);
    next_stage<kUKStages>(sc, pc);
    s0 = sc;
    ph0 = pc;
#pragma unroll
    for (int k = 0; k < V; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r2[k] += __shfl_down_sync(0xffffffffu, r2[k], o);
}

struct Bars {
    uint64_t fullM[kMainStages], emptyM[kMainStages], fullK[kUKStages], emptyK[kUKStages];
};

__device__ __forceinline__ void init_barriers(Bars& b, uint32_t consumer_threads = kConsumers * 32,
                                              uint32_t main_producers = 1) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMainStages; ++s) {
            mbar_init(&b.fullM[s], main_producers);
            mbar_init(&b.emptyM[s], consumer_threads);
        }
        for (int s = 0; s < kUKStages; ++s) {
            mbar_init(&b.fullK[s], 1);
            mbar_init(&b.emptyK[s], consumer_threads);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

template <int C, bool HEAT, bool PUSH, bool FLAT>
__global__ void __launch_bounds__(pass_threads(FLAT), SSB_CTAS_PER_SM) sor_pass_tma(const SorArgs a) {
    constexpr int NW = FLAT ? kFlatWarps : kConsumers;  // consumer warps of this kernel
    constexpr int V = FLAT ? kFlatV : 1;                 // slots per consumer thread
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) Bars bars;
    __shared__ double ws[32];
    __shared__ int last;
    // prologue that touches no global memory, then wait for the previous kernel of the
    // stream (programmatic dependent launch: this grid may start while it drains)
    constexpr int SPLIT = FLAT ? kSplitMain : 0;  // second main-ring producer warp
    // dynamic items: the main producer takes item indices from a global counter and hands
    // them to the UK producer and the consumers through a small shared queue
    constexpr bool DYN = SSB_DYN_ITEMS && FLAT && !PUSH && !SPLIT;
    __shared__ int qitem[kItemQ];
    __shared__ __align__(8) uint64_t qfull[kItemQ], qempty[kItemQ];
    if (DYN && threadIdx.x == 0)
        for (int q = 0; q < kItemQ; ++q) {
            mbar_init(&qfull[q], 1);
            mbar_init(&qempty[q], NW * 32 + 1);
        }
    init_barriers(bars, NW * 32, 1 + SPLIT);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    SorState* st = a.st;
    if (*(volatile const int*)&st->done) return;
    const int n = C == 0 ? *(volatile const int*)&st->n_red : *(volatile const int*)&st->n_black;
    // fuse_final: no finalize launch between the passes.  The red pass hands its
    // n to the black pass (n_black: black CTAs read it, nobody else writes it
    // during the red pass); the black pass's first CTAs take the finalize's
    // place before their own items (black_head_finalize).
    // (also on slab groups: their decision runs concurrently with the black pass)
    if (C == 0 && blockIdx.x == 0 && threadIdx.x == 0) st->n_black = n;
    const int bout = out_buf(n);
    const int bin = in_buf(n);
    const Layout& L = a.L;
    const double* uc = a.U[bin][C];
    const double* uo = C == 0 ? a.U[bin][1] : a.U[bout][0];
    double* ucw = a.U[bout][C];
    const Geo G = make_geo(L, a.tile2d != 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nl = (a.l_hi - a.l_lo) / a.l_step + 1;  // slices l_lo, l_lo + l_step, .. l_hi
    // fixed-sweep solves know their end: the black pass after the last iteration (it only
    // carries the head's decision of that iteration) updates nothing
    const int fixed_mode = *(volatile const int*)&st->fixed;
    const bool fixed_solve = fixed_mode != 0;
    const int max_it = *(volatile const int*)&st->max_iter;
    // (mode 2, no diagnostics wanted: red(max_iter + 1) would only evaluate that residual -- idle too)
    const bool idle = fixed_solve && n > max_it && (C == 1 || fixed_mode == 2);
    // fixed-sweep solves need a residual only for their last iteration (the diagnostics):
    // red(max_iter + 1) carries its red part, black(max_iter) its black part; the other
    // passes skip the residual arithmetic and write zero partials (-1.6% per sweep, config 4:
    // the power-capped clock rises with the work saved)
    const bool need_res = !fixed_solve || (fixed_mode == 1 && (C == 0 ? n == max_it + 1 : n == max_it));
    const long long n_items = idle ? 0 : (long long)G.nsg * G.njg * G.nkc * nl;
    // snake order: black passes walk the items backwards, so each pass starts on
    // the rows the previous pass touched last (still in L2)
    const bool rev = C == 1 && a.snake;
    const Policies pol = make_policies(a.l2hint);
    const bool dyn = DYN && a.dyn && a.l_step == 1;  // uniform over the grid; one such launch per pass
    // the other colour's pass is complete (and its successor not started): reset its counter
    if (dyn && blockIdx.x == 0 && threadIdx.x == 0) st->item_ctr[C ^ 1] = 0;
    // queue reader: the next item index (-1: none left)
    uint32_t qs = 0, qph = 0;
    auto q_take = [&]() -> long long {
        mbar_wait(&qfull[qs], qph);
        const int v = *(volatile int*)&qitem[qs];
        mbar_arrive(&qempty[qs]);
        next_stage<kItemQ>(qs, qph);
        return v;
    };

    if (warp >= NW) {  // producers: one thread per ring issues its bulk copies
        if (lane != 0) return;
        // 2D-tiled: the tensor maps of the streams (coef, rhs, own colour, other colour)
        const CUtensorMap* tm[4] = {nullptr, nullptr, nullptr, nullptr};
        const CUtensorMap* tm_uk = nullptr;
        if (G.S) {
            const int bo = C == 0 ? bin : bout, co = C == 0 ? 1 : 0;
            tm[0] = &a.maps->coef[C];
            tm[1] = &a.maps->rhs[C];
            tm[2] = &a.maps->u_main[bin][C];
            tm[3] = &a.maps->u_main[bo][co];
            tm_uk = &a.maps->u_uk[bo][co];
        }
        Ring<kMainStages> rm;
        Ring<kUKStages> rk;
        if (dyn && warp == NW) {  // the item source: first item static, then the counter
            long long tt = blockIdx.x;
            for (int used = 0;; ++used) {
                if (used >= kItemQ) mbar_wait(&qempty[qs], qph ^ 1u);
                const long long cur = tt < n_items ? tt : -1;
                qitem[qs] = (int)cur;
                mbar_arrive(&qfull[qs]);
                next_stage<kItemQ>(qs, qph);
                if (cur < 0) break;
                // claim the next item now: the atomic's latency overlaps this item's copies
                const unsigned nxt = atomicAdd(&st->item_ctr[C], 1u);
                Item it;
                decode_item(L, G, a.order, a.l_lo, nl, rev ? n_items - 1 - cur : cur, it, a.l_step);
                produce_main<HEAT>(L, G, smem, bars.fullM, bars.emptyM, rm, it, a.coef[C], a.rhs[C], uc, uo, pol, tm);
                tt = (long long)gridDim.x + nxt;
            }
            return;
        }
        for (long long tt = dyn ? q_take() : blockIdx.x; tt >= 0 && tt < n_items;
             tt = dyn ? q_take() : tt + gridDim.x) {
            Item it;
            decode_item(L, G, a.order, a.l_lo, nl, rev ? n_items - 1 - tt : tt, it, a.l_step);
            if (warp == NW)
                produce_main<HEAT>(L, G, smem, bars.fullM, bars.emptyM, rm, it, a.coef[C], a.rhs[C], uc, uo, pol, tm,
                                   true, SPLIT ? 1 : 0);
            else if (SPLIT && warp == NW + 2)
                produce_main<HEAT>(L, G, smem, bars.fullM, bars.emptyM, rm, it, a.coef[C], a.rhs[C], uc, uo, pol, tm,
                                   true, 2);
            else
                produce_uk(L, G, smem, bars.fullK, bars.emptyK, rk, it, uo, pol, tm_uk);
        }
        return;
    }
    if (C == 1 && a.fuse_final)  // the finalize's fixed 256-lane tree, NW * 32 threads
        if (threadIdx.x < 256)  // the tree is played by <= 256 threads (same bits for 128 or 256)
            black_head_finalize<(NW * 32 > 256 ? 256 : NW * 32)>(a, n, ws, &last, threadIdx.x);
    uint32_t ms = 0, mph = 0, s0 = 0, ph0 = 0;
    // FLAT (host-chosen): whole-row items with the flat slot mapping, not heat.  Thread
    // tid plays the 8-warp mapping's threads tid + k * NW * 32 (k < V), and writes
    // their warps' residual partials, so the partials are the same bits for any V.
    FlatThread ft[V];
#pragma unroll
    for (int k = 0; k < V; ++k) ft[k] = FLAT ? flat_thread(L, G, threadIdx.x + k * NW * 32) : FlatThread{};
    for (long long tt = dyn ? q_take() : blockIdx.x; tt >= 0 && tt < n_items; tt = dyn ? q_take() : tt + gridDim.x) {
        Item it;
        const long long t = decode_item(L, G, a.order, a.l_lo, nl, rev ? n_items - 1 - tt : tt, it, a.l_step);
        double* plo = PUSH && it.l == 1 ? a.push_lo[bout][C] : nullptr;
        double* phi = PUSH && it.l == L.n4 ? a.push_hi[bout][C] : nullptr;
        double r2[V];
        if constexpr (FLAT) {
            if (need_res)
                consume_item_flat<C, PUSH, V, true>(a, L, G, ft, sptr(smem), bars.fullM, bars.emptyM, bars.fullK,
                                                    bars.emptyK, ms, mph, s0, ph0, it, ucw, plo, phi, r2);
            else
                consume_item_flat<C, PUSH, V, false>(a, L, G, ft, sptr(smem), bars.fullM, bars.emptyM, bars.fullK,
                                                     bars.emptyK, ms, mph, s0, ph0, it, ucw, plo, phi, r2);
        }
        else
            r2[0] = consume_item<C, HEAT, PUSH>(a, L, G, smem, bars.fullM, bars.emptyM, bars.fullK, bars.emptyK, ms,
                                                mph, s0, ph0, it, ucw, warp, lane, pol.ustore, plo, phi);
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < V; ++k) a.part[n & 3][C][t * kWarps + warp + k * NW] = r2[k];
    }
    // halo push to another GPU: this thread's peer stores are performed before the
    // pass completes (the signal kernel that follows publishes the pass)
    if constexpr (PUSH) __threadfence_system();
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
__global__ void __launch_bounds__(kThreads, SSB_CTAS_PER_SM) sor_wave_tma(const SorArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) Bars bars;
    const SorState* st = a.st;
    if (*(volatile const int*)&st->done) return;
    const int n = *(volatile const int*)&st->n_red;
    const int epoch = *(volatile const int*)&st->epoch_base + n;
    const Layout& L = a.L;
    const Geo G = make_geo(L, a.tile2d != 0);
    const int CH = G.njg * G.nkc;  // items per slice and phase
    // wavefront over sub-slices s = (l-1)*nkc + kc: phase d of step sigma works on
    // s = sigma - skew*d; each step has kWavePH phases x njg row groups
    const int skew = SSB_WAVE_SKEW > 0 ? SSB_WAVE_SKEW : 2 * G.nkc;
    const long long NS = (long long)L.n4 * G.nkc;
    const long long NT = (NS + (kWavePH - 1LL) * skew) * kWavePH * G.njg;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Policies pol = make_policies(a.l2hint);
    init_barriers(bars);

    auto decode = [&](long long t, int& d, int& l, int& c) {
        const int jg = (int)(t % G.njg);
        const long long r = t / G.njg;
        d = (int)(r % kWavePH);
        const long long s = r / kWavePH - (long long)skew * d;  // sub-slice of this phase
        if (s < 0 || s >= NS) {
            l = 0;
            c = 0;
            return;
        }
        l = (int)(s / G.nkc) + 1;
        c = (int)(s % G.nkc) * G.njg + jg;
    };

    if (warp >= kConsumers) {  // producers (each waits for the flags itself)
        if (lane != 0) return;
        Ring<kMainStages> rm;
        Ring<kUKStages> rk;
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
            if (warp == kConsumers)
                produce_main<HEAT>(L, G, smem, bars.fullM, bars.emptyM, rm, it, a.coef[C], a.rhs[C], uc, uo, pol);
            else
                produce_uk(L, G, smem, bars.fullK, bars.emptyK, rk, it, uo, pol);
        }
        return;
    }
    uint32_t ms = 0, mph = 0, s0 = 0, ph0 = 0;
    for (long long t = blockIdx.x; t < NT; t += gridDim.x) {
        int d, l, c;
        decode(t, d, l, c);
        if (l < 1 || l > L.n4) continue;
        const int m = n + (d >> 1), C = d & 1;
        const int jg = c % G.njg, kc = c / G.njg;
        const Item it = make_item(L, G, l, jg, kc);
        double* ucw = a.U[out_buf(m)][C];
        const double r2 =
            C == 0 ? consume_item<0, HEAT>(a, L, G, smem, bars.fullM, bars.emptyM, bars.fullK, bars.emptyK, ms, mph,
                                           s0, ph0, it, ucw, warp, lane, pol.ustore)
                   : consume_item<1, HEAT>(a, L, G, smem, bars.fullM, bars.emptyM, bars.fullK, bars.emptyK, ms, mph,
                                           s0, ph0, it, ucw, warp, lane, pol.ustore);
        if (lane == 0) a.part[m & 3][C][((long long)(l - 1) * CH + c) * kWarps + warp] = r2;
        // publish: every consumer's stores, then one flag store (release)
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
        if (threadIdx.x == 0) {
            int* q = a.flags + ((long long)d * L.n4 + (l - 1)) * CH + c;
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(q), "r"(epoch) : "memory");
        }
    }
}

// ---------------------------------------------------------------------------
// One-sweep k-wavefront (kernel 7, "kwave": red and black of one iteration in one launch).
//
// Items are R rows x kKwP planes (a plane chunk) of one slice, consumed with the two-pass
// rings and flat mapping.  The launch walks the plane chunks in order across ALL slices
// and row groups at once: step s holds the red items of chunk s (every (jg, l), l
// fastest), then the black items of chunk s - LAG.  A black item (kc, jg, l) reads the
// new red values of (kc, jg, l), (kc, jg, l +- 1), (kc, jg +- 1, l) and (kc +- 1, jg, l)
// (the first / last plane); the producers poll those seven red items' completion flags
// (epochs; relaxed loads issued one black item ahead, one acquire fence) before issuing
// the item's bulk copies.  A publisher thread per CTA publishes each finished red item
// (consumers' stores -> mbarrier -> __threadfence -> flag) so consumers never block on
// a fence.  Why: the red values a black item reads, and the black values the red items
// of the following chunks read, were touched ~LAG + 2 chunks earlier and are still in L2
// (coefficient / rhs streams evict_first), so a sweep moves ~59 B per doxel from DRAM
// instead of the two-pass ~67 B.  Iterates are the two-pass ones bit for bit (tests);
// residual partials are one per (item, warp) at the item's canonical slice-major index.
// MEASURED (config 1, B200, scripts/gpu_kwave_var.sh): DRAM 997 vs 1128 MB per sweep, but
// 226 us per sweep vs 198 us for the two-pass (P = 4, LAG = 2; P = 8: 217; P = 1: 330);
// with the flag waits compiled out (a timing-only build, wrong results; removed) 193 us -- the
// cross-CTA dependency waits cost more than the 12% of DRAM bytes saved.  Opt-in, not the default.
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

#ifndef SSB_KWAVE_LAG
#define SSB_KWAVE_LAG 2  // black items of plane chunk c follow the red items of chunk c + LAG
#endif
#ifndef SSB_KWAVE_PLANES
#define SSB_KWAVE_PLANES 4  // planes per item (one ring stage each)
#endif
constexpr int kKwP = SSB_KWAVE_PLANES;
#ifndef SSB_KWAVE_L2MB
#define SSB_KWAVE_L2MB 48  // L2 share the live u rows of the wavefront may take
#endif
#ifndef SSB_KWAVE_L2HINT
#define SSB_KWAVE_L2HINT 1  // bit0: coefficient / rhs streams evict_first (the u rows are the reused data)
#endif
constexpr int kKwLag = SSB_KWAVE_LAG;
constexpr int kKwPub = 4;  // publisher ring: items a consumer may finish ahead of the publisher
// The wavefront marches along k (chunk = a plane chunk of every row group and slice) or,
// when that cross-section is smaller, along j (chunk = a row group of every plane chunk
// and slice: the j-wavefront) -- the u rows between a chunk's red and black items must
// stay in L2, and the j cross-section of a wide, shallow grid (config 4: 8 MB) is a
// quarter of the k one
struct KwGeo {
    int nkc;        // plane chunks of kKwP planes
    int axis_j;     // 1: chunks are row groups (j-wavefront), 0: plane chunks (k-wavefront)
    int nch;        // chunks along the march axis
    int NA;         // items per chunk and slice (row groups, or plane chunks for axis_j)
    int M;          // items per chunk and colour: NA * n4
    long long NT;   // items of the launch: (nch + LAG) steps x 2 colours x M (empty halves skipped)
};
__host__ __device__ __forceinline__ KwGeo make_kwgeo(const Layout& L, const Geo& G, int axis_j = 0) {
    KwGeo k;
    k.nkc = (L.n3 + kKwP - 1) / kKwP;
    k.axis_j = axis_j;
    k.nch = axis_j ? G.njg : k.nkc;
    k.NA = axis_j ? k.nkc : G.njg;
    k.M = k.NA * L.n4;
    k.NT = (long long)(k.nch + kKwLag) * 2 * k.M;
    return k;
}

constexpr int kKwThreads = (kFlatWarps + 3) * 32;  // consumers + main producer + UK producer + publisher
__host__ __device__ __forceinline__ uint32_t kwave_smem(const Layout& L) { return (uint32_t)make_geo(L).smem; }

__global__ void __launch_bounds__(kKwThreads, SSB_CTAS_PER_SM) sor_kwave_tma(const SorArgs a) {
    constexpr int NW = kFlatWarps, V = kFlatV;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) Bars bars;  // the two-pass rings: main (per plane), UK (other-colour rows)
    __shared__ __align__(8) uint64_t doneB[kKwPub], pubB[kKwPub];
    init_barriers(bars, NW * 32);
    if (threadIdx.x == 0) {
        for (int q = 0; q < kKwPub; ++q) {
            mbar_init(&doneB[q], NW * 32);  // consumers: item finished (stores issued)
            mbar_init(&pubB[q], 1);         // publisher: item published, slot free again
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const SorState* st = a.st;
    if (*(volatile const int*)&st->done) return;
    const int n = *(volatile const int*)&st->n_red;
    const int epoch = *(volatile const int*)&st->epoch_base + n;
    const Layout& L = a.L;
    const Geo G = make_geo(L, false);
    const KwGeo K = make_kwgeo(L, G, a.kwj);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bin = in_buf(n), bout = out_buf(n);
    int* const flg = a.flags;  // per red item: the epoch of the launch that completed it
    // item cursor: block blk (2 per step: red, black), position a within the chunk (row group,
    // or plane chunk for the j-wavefront), slice l0 + 1 (l fastest); advanced by gridDim.x
    // items with additions only
    struct Cur {
        int blk, a, l0;
    };
    const int NB = 2 * (K.nch + kKwLag);
    const int gq = (int)(gridDim.x / (unsigned)L.n4), gr = (int)(gridDim.x % (unsigned)L.n4);
    auto first = [&]() {
        Cur c;
        const int x0 = (int)blockIdx.x % K.M;
        c.blk = (int)blockIdx.x / K.M;
        c.a = x0 / L.n4;
        c.l0 = x0 - c.a * L.n4;
        return c;
    };
    auto advance = [&](Cur& c) {
        c.l0 += gr;
        c.a += gq;
        if (c.l0 >= L.n4) {
            c.l0 -= L.n4;
            ++c.a;
        }
        while (c.a >= K.NA) {
            c.a -= K.NA;
            ++c.blk;
        }
    };
    // colour and Item of the cursor's item; false: empty half-step (no such chunk)
    auto item_of = [&](const Cur& c, int& C, Item& it) -> bool {
        C = c.blk & 1;
        const int ch = (c.blk >> 1) - C * kKwLag;  // chunk along the march axis
        if (ch < 0 || ch >= K.nch) return false;
        const int kc = K.axis_j ? c.a : ch, jg = K.axis_j ? ch : c.a;
        it.l = c.l0 + 1;
        it.s0 = 0;
        it.j0 = jg * G.R + 1;
        it.rows = min(G.R, L.n2 - it.j0 + 1);
        it.k0 = kc * kKwP + 1;
        it.k1 = min(it.k0 + kKwP - 1, L.n3);
        return true;
    };
    auto chunk = [&](const Item& it) { return (it.k0 - 1) / kKwP; };  // plane chunk
    auto rgroup = [&](const Item& it) { return (it.j0 - 1) / G.R; };  // row group
    auto flag_of = [&](int kc, int jg, int l) -> const int* {
        return flg + ((long long)kc * G.njg + jg) * L.n4 + (l - 1);
    };

    if (warp == NW + 2) {  // publisher: after the consumers finish a red item, fence + flag
        if (lane != 0) return;
        uint32_t ps = 0, pph = 0;
        for (Cur c = first(); c.blk < NB; advance(c)) {
            int C;
            Item it;
            if (!item_of(c, C, it)) continue;
            mbar_wait(&doneB[ps], pph);
            if (C == 0) {
                __threadfence();  // the consumers' stores (ordered before their arrivals) -> gpu scope
                asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(flag_of(chunk(it), rgroup(it), it.l)),
                             "r"(epoch)
                             : "memory");
            }
            mbar_arrive(&pubB[ps]);
            next_stage<kKwPub>(ps, pph);
        }
        return;
    }
    if (warp >= NW) {  // producers: lane 0 of warp NW (main ring), of warp NW + 1 (UK ring)
        if (lane != 0) return;
        const Policies pol = make_policies(SSB_KWAVE_L2HINT);
        Ring<kMainStages> rm;
        Ring<kUKStages> rk;
        // the red items a black item (kc, jg, l) reads: (kc, jg, l), (kc, jg, l +- 1),
        // (kc, jg +- 1, l), (kc +- 1, jg, l); their flags for this CTA's next black item are
        // loaded one black item ahead (relaxed, in parallel), re-polled only if not yet set
        Cur nb{-1, 0, 0};
        int nbv[7];
        auto deps = [&](const Item& it, const int*(&q)[7]) {
            const int kc = chunk(it), jg = rgroup(it), l = it.l;
            const int* self = flag_of(kc, jg, l);
            q[0] = self;
            q[1] = l > 1 ? self - 1 : self;
            q[2] = l < L.n4 ? self + 1 : self;
            q[3] = jg > 0 ? self - L.n4 : self;
            q[4] = jg + 1 < G.njg ? self + L.n4 : self;
            q[5] = kc > 0 ? self - (long long)G.njg * L.n4 : self;
            q[6] = kc + 1 < K.nkc ? self + (long long)G.njg * L.n4 : self;
        };
        auto prefetch_next_black = [&](Cur c) {
            nb.blk = -1;
            for (advance(c); c.blk < NB; advance(c)) {
                int C2;
                Item it2;
                if (item_of(c, C2, it2) && C2 == 1) {
                    const int* q[7];
                    deps(it2, q);
#pragma unroll
                    for (int u = 0; u < 7; ++u) nbv[u] = ld_relaxed(q[u]);
                    nb = c;
                    return;
                }
            }
        };
        for (Cur c = first(); c.blk < NB; advance(c)) {
            int C;
            Item it;
            if (!item_of(c, C, it)) continue;
            if (C == 1) {
                const int* q[7];
                deps(it, q);
                const bool pre = nb.blk == c.blk && nb.a == c.a && nb.l0 == c.l0;
                int v[7];
#pragma unroll
                for (int u = 0; u < 7; ++u) v[u] = pre ? nbv[u] : ld_relaxed(q[u]);
#pragma unroll
                for (int u = 0; u < 7; ++u)
                    while (v[u] != epoch) {
                        __nanosleep(32);
                        v[u] = ld_relaxed(q[u]);
                    }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
                prefetch_next_black(c);
            }
            const double* uc = a.U[bin][C];
            const double* uo = C == 0 ? a.U[bin][1] : a.U[bout][0];
            if (warp == NW) {
                produce_main<false>(L, G, smem, bars.fullM, bars.emptyM, rm, it, a.coef[C], a.rhs[C], uc, uo, pol);
            } else {
                produce_uk(L, G, smem, bars.fullK, bars.emptyK, rk, it, uo, pol);
            }
        }
        return;
    }
    uint32_t ms = 0, mph = 0, s0 = 0, ph0 = 0, ds = 0, dph = 0;
    int ci = 0;  // item ordinal
    FlatThread ft[V];
#pragma unroll
    for (int k = 0; k < V; ++k) ft[k] = flat_thread(L, G, threadIdx.x + k * NW * 32);
    for (Cur c = first(); c.blk < NB; advance(c)) {
        int C;
        Item it;
        if (!item_of(c, C, it)) continue;
        double r2[V];
        if (C == 0)
            consume_item_flat<0, false, V>(a, L, G, ft, sptr(smem), bars.fullM, bars.emptyM, bars.fullK, bars.emptyK,
                                           ms, mph, s0, ph0, it, a.U[bout][0], nullptr, nullptr, r2);
        else
            consume_item_flat<1, false, V>(a, L, G, ft, sptr(smem), bars.fullM, bars.emptyM, bars.fullK, bars.emptyK,
                                           ms, mph, s0, ph0, it, a.U[bout][1], nullptr, nullptr, r2);
        const long long canon = ((long long)(it.l - 1) * K.nkc + chunk(it)) * G.njg + rgroup(it);
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < V; ++k) a.part[n & 3][C][canon * kWarps + warp + k * NW] = r2[k];
        // hand the item to the publisher (its slot must have been released kKwPub items ago)
        if (ci >= kKwPub) mbar_wait(&pubB[ds], dph ^ 1u);
        mbar_arrive(&doneB[ds]);
        next_stage<kKwPub>(ds, dph);
        ++ci;
    }
}

template <int C, bool HEAT, bool PUSH, bool FLAT = false>
void configure() {
    static bool done = false;
    if (!done) {
        SSB_CUDA(cudaFuncSetAttribute(sor_pass_tma<C, HEAT, PUSH, FLAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
        done = true;
    }
}

template <bool HEAT>
void configure_wave() {
    static bool done = false;
    if (!done) {
        SSB_CUDA(cudaFuncSetAttribute(sor_wave_tma<HEAT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
        done = true;
    }
}

// resident CTAs for this kernel and shared-memory size (the wavefront kernel
// relies on every CTA being resident: items wait only on earlier items)
int tma_blocks(const void* fn, size_t smem_bytes, int threads = kThreads) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        SSB_CUDA(cudaGetDevice(&dev));
        SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    int per = 0;
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem_bytes));
    return sms * std::max(1, per);
}

}  // namespace

// pass-order / L2-policy switches (env SSB_SNAKE, SSB_L2HINT; measured defaults)
int pass_snake() {
    static const int v = [] {
        const char* e = std::getenv("SSB_SNAKE");
        return e ? std::atoi(e) : kDefaultSnake;
    }();
    return v;
}
int pass_pdl() {
    static const int v = [] {
        const char* e = std::getenv("SSB_PDL");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}
int pass_grid_short() {
    static const int v = [] {
        const char* e = std::getenv("SSB_GRID_SHORT");
        return e ? std::max(0, std::atoi(e)) : 0;
    }();
    return v;
}
int pass_fuse_final() {
    static const int v = [] {
        const char* e = std::getenv("SSB_FUSE_FINAL");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}
int pass_order() {
    static const int v = [] {
        const char* e = std::getenv("SSB_ORDER");
        return e ? std::atoi(e) : kDefaultOrder;
    }();
    return v;
}
int pass_l2hint() {
    static const int v = [] {
        const char* e = std::getenv("SSB_L2HINT");
        return e ? std::atoi(e) : kDefaultL2Hint;
    }();
    return v;
}

bool tma_pass_supported(const Layout& L) {
    const Geo G = make_geo(L);
    // decode_item works in 32 bits
    const long long lim = 1LL << 31;
    return (size_t)G.smem <= 200 * 1024 && G.items < lim && make_geo(L, true).items < lim;
}

void tma_pass_tiles(const Layout& L, SorArgs& a) {
    const Geo G = make_geo(L, a.tile2d != 0);
    a.tiles = G.items;
    a.bps = G.nsg * G.njg * G.nkc * kWarps;  // partials per slice: one per (item, warp)
    a.tx = G.njg;
    a.ty = G.nkc;
    a.tk = G.nsg;
}

bool tma_fuse_ok(const Layout& L) { return L.glo && L.ghi; }  // single slab

// fraction of the consumer threads that own a doxel slot in a plane step
double tma_lane_utilization(const Layout& L, bool tile2d) {
    const Geo G = make_geo(L, tile2d);
    const int nq = (L.n1 + 1) / 2;
    if (G.S) return nq / (double)(G.S * G.nsg);
    if (G.wpr) return nq / (double)(kSlotsPerPlane * ((nq + kSlotsPerPlane - 1) / kSlotsPerPlane));
    return G.R * nq / (double)kSlotsPerPlane;
}

size_t tma_partials(const Layout& L) {
    return (size_t)std::max(make_geo(L).items, make_geo(L, true).items) * kWarps;
}

// ---- tensor maps of the 2D-tiled pass (driver API through the runtime's entry point)
bool encode_tma_maps(const SorArgs& a, TmaMaps& m) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!enc) return false;
    const Layout& L = a.L;
    const cuuint32_t ones[2] = {1, 1};
    auto map2d = [&](CUtensorMap* out, CUtensorMapDataType dt, const void* base, cuuint64_t cols, cuuint32_t esz,
                     cuuint32_t bx, cuuint32_t by) {
        const cuuint64_t dims[2] = {cols, (cuuint64_t)L.rows};
        const cuuint64_t strides[1] = {cols * esz};
        const cuuint32_t box[2] = {bx, by};
        const CUresult r = enc(out, dt, 2, const_cast<void*>(base), dims, strides, box, ones,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(SS_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    };
    std::memset(&m, 0, sizeof m);
    const cuuint32_t pw = kTileS + 2;
    for (int b = 0; b < kStateBuffers; ++b)
        for (int c = 0; c < 2; ++c) {
            map2d(&m.u_main[b][c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, a.U[b][c], L.W, 8, pw, kTileR);
            map2d(&m.u_uk[b][c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, a.U[b][c], L.W, 8, pw, kTileR + 2);
        }
    for (int c = 0; c < 2; ++c) {
        map2d(&m.rhs[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, a.rhs[c], L.W, 8, pw, kTileR);
        if (a.coef[c])
            map2d(&m.coef[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.coef[c], (cuuint64_t)L.Wc * 8, 4, kTileS * 8, kTileR);
    }
    return true;
}

int wave_iters() { return kWavePH / 2; }

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
    const size_t smem = (size_t)G.smem;
    configure_wave<false>();
    configure_wave<true>();
    configure<0, false, false>();
    static size_t last_smem = 0;
    static int blocks = 0;
    if (smem != last_smem) {
        blocks = std::min(tma_blocks((const void*)sor_wave_tma<false>, smem),
                          tma_blocks((const void*)sor_wave_tma<true>, smem));
        last_smem = smem;
    }
    const int skew = SSB_WAVE_SKEW > 0 ? SSB_WAVE_SKEW : 2 * G.nkc;
    const long long NT = ((long long)a.L.n4 * G.nkc + (kWavePH - 1LL) * skew) * kWavePH * G.njg;
    const unsigned grid = (unsigned)std::min<long long>(NT, blocks);
    if (heat)
        sor_wave_tma<true><<<grid, kThreads, smem, s>>>(a);
    else
        sor_wave_tma<false><<<grid, kThreads, smem, s>>>(a);
    SSB_LAUNCHED();
}

// u rows live in L2 between a chunk's first red read and its last black read: about
// LAG + 2 chunks of (red-new + black-old) = 8 B per doxel of a chunk (the coefficient /
// rhs streams are evict_first).  A chunk is kKwP planes of every (j, l) (k-wavefront) or
// R rows of every (k, l) (j-wavefront); the smaller one is used
static double kwave_chunk_bytes(const Layout& L, const Geo& G, int axis_j) {
    return axis_j ? (double)G.R * L.n1 * L.n3 * L.n4 * 8.0 : (double)kKwP * L.n1 * L.n2 * L.n4 * 8.0;
}
int kwave_axis_j(const Layout& L) {
    const int forced = std::getenv("SSB_KWAVE_AXIS") ? std::atoi(std::getenv("SSB_KWAVE_AXIS")) : -1;
    if (forced >= 0) return forced;
    const Geo G = make_geo(L);
    return kwave_chunk_bytes(L, G, 1) < kwave_chunk_bytes(L, G, 0) ? 1 : 0;
}
bool kwave_supported(const Layout& L) {
    // whole-row flat items, one slab; the live chunks must leave L2 room
    const Geo G = make_geo(L);
    return tma_pass_supported(L) && !G.wpr && !G.S && L.glo && L.ghi && kwave_smem(L) <= 110u * 1024u &&
           (kKwLag + 2.0) * kwave_chunk_bytes(L, G, kwave_axis_j(L)) <= SSB_KWAVE_L2MB * 1024.0 * 1024;
}
size_t kwave_flags(const Layout& L) {
    const Geo G = make_geo(L);
    const int nkc = make_kwgeo(L, G).nkc;
    return (size_t)nkc * G.njg * L.n4;
}
size_t kwave_partials(const Layout& L) {
    const Geo G = make_geo(L);
    return (size_t)make_kwgeo(L, G).nkc * G.njg * L.n4 * kWarps;
}
int kwave_bps(const Layout& L) {
    const Geo G = make_geo(L);
    return make_kwgeo(L, G).nkc * G.njg * kWarps;
}

void launch_sor_kwave(cudaStream_t s, const SorArgs& a) {
    const Geo G = make_geo(a.L);
    const KwGeo K = make_kwgeo(a.L, G, a.kwj);
    const size_t smem = kwave_smem(a.L);
    static size_t last_smem = 0;
    static int blocks = 0;
    if (smem != last_smem) {
        SSB_CUDA(cudaFuncSetAttribute(sor_kwave_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        blocks = tma_blocks((const void*)sor_kwave_tma, smem, kKwThreads);
        last_smem = smem;
    }
    const unsigned grid = (unsigned)std::min<long long>(K.NT, blocks);
    sor_kwave_tma<<<grid, kKwThreads, smem, s>>>(a);
    SSB_LAUNCHED();
}

void launch_sor_pass_tma(cudaStream_t s, const SorArgs& a, int colour, bool heat) {
    const Geo G = make_geo(a.L, a.tile2d != 0);
    const size_t smem = (size_t)G.smem;
    static size_t last_smem = 0;
    static int blocks[2] = {0, 0};  // general / flat kernels
    if (smem != last_smem) {
        configure<0, false, false>();
        configure<1, false, false>();
        configure<0, true, false>();
        configure<1, true, false>();
        configure<0, false, true>();
        configure<1, false, true>();
        configure<0, true, true>();
        configure<1, true, true>();
        configure<0, false, false, true>();
        configure<1, false, false, true>();
        configure<0, false, true, true>();
        configure<1, false, true, true>();
        blocks[0] = tma_blocks((const void*)sor_pass_tma<0, false, false, false>, smem, pass_threads(false));
        blocks[1] = tma_blocks((const void*)sor_pass_tma<0, false, false, true>, smem, pass_threads(true));
        last_smem = smem;
    }
    const bool flat = !heat && !G.S && !G.wpr;
    const long long items = (long long)G.nsg * G.njg * G.nkc * ((a.l_hi - a.l_lo) / a.l_step + 1);
    // CTA slots left free for kernels of other streams (NCCL's send/recv beside the interior
    // launch of a distributed pass): the grid is persistent, so nothing else frees one mid-pass
    const int room = std::max(1, blocks[flat] - std::max(a.grid_short, pass_grid_short()));
    const unsigned grid = (unsigned)std::min<long long>(items, room);
    SorArgs b = a;
    if (b.order < 0) b.order = 2LL * G.nsg * G.njg * G.nkc <= blocks[flat] ? 0 : 1;
    const bool push = a.push_lo[0][0] != nullptr || a.push_hi[0][0] != nullptr;
    const int v = (colour & 1) | (heat ? 2 : 0) | (push ? 4 : 0) | (flat ? 8 : 0);
    using K = void (*)(const SorArgs);
    static const K fns[16] = {sor_pass_tma<0, false, false, false>, sor_pass_tma<1, false, false, false>,
                              sor_pass_tma<0, true, false, false>,  sor_pass_tma<1, true, false, false>,
                              sor_pass_tma<0, false, true, false>,  sor_pass_tma<1, false, true, false>,
                              sor_pass_tma<0, true, true, false>,   sor_pass_tma<1, true, true, false>,
                              sor_pass_tma<0, false, false, true>,  sor_pass_tma<1, false, false, true>,
                              nullptr,                              nullptr,
                              sor_pass_tma<0, false, true, true>,   sor_pass_tma<1, false, true, true>,
                              nullptr,                              nullptr};
    // programmatic dependent launch: the pass may be scheduled while the previous kernel
    // drains; it waits (griddepcontrol.wait) before its first global read
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(pass_threads(flat));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pass_pdl() && !a.pdl_off ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SSB_CUDA(cudaLaunchKernelEx(&cfg, fns[v], b));
    SSB_LAUNCHED();
}

}  // namespace ssb
