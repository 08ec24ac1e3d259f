// assemble.cu -- reduced-diamond-cell face gradients (edge.cpp:16-57), per-face
// coefficient assembly (solver.cpp:23-77) and the Perona-Malik edge
// coefficients (edge.cpp:73-99), plus coefficient packing for the per-call API.
//
// Every expression keeps the reference's evaluation order and the file is
// compiled with -fmad=false, so the fp32 off-diagonals are bit-identical to the
// reference's (IEEE sqrt/div are correctly rounded on the GPU as on x86).
#include <algorithm>
#include <cmath>

#include "kernels.cuh"

namespace ssb {

namespace {

// Loader of a colour-packed field around doxel (i, j, k, l) of colour C.
struct Stencil {
    const double* f[2];
    long long row;  // row(j,k,l)
    int i, C;
    int jMax, kMax, W;
    __device__ __forceinline__ double at(int di, int dj, int dk, int dl) const {
        const long long r = row + dj + (long long)dk * jMax + (long long)dl * jMax * kMax;
        const int c = C ^ ((di + dj + dk + dl) & 1);
        return __ldg(f[c] + r * W + ((i + di) >> 1));
    }
};

template <int A>
__device__ __forceinline__ void unit(int& di, int& dj, int& dk, int& dl, int s) {
    di = A == 0 ? s : 0;
    dj = A == 1 ? s : 0;
    dk = A == 2 ? s : 0;
    dl = A == 3 ? s : 0;
}

// x / h_a.  When every spacing is a power of two (h = 1/32, 1/64, ...),
// x / h == x * (1/h) exactly in IEEE arithmetic (both are exact rescalings by
// 2^k), so the division is replaced by the multiplication bit for bit.
template <bool POW2>
__device__ __forceinline__ double div_h(double x, const double h[4], const double hinv[4], int a) {
    if constexpr (POW2)
        return x * hinv[a];
    else
        return x / h[a];
}

// face_gradient (edge.cpp:33-48) for face F of the stencil's doxel
template <int F, bool POW2>
__device__ __forceinline__ void face_gradient(const Stencil& S, const double h[4], const double hinv[4],
                                              double p0, double g[4]) {
    constexpr int A = F >> 1;
    constexpr int SG = (F & 1) ? 1 : -1;
    int ai, aj, ak, al;
    unit<A>(ai, aj, ak, al, SG);
    const double pn = S.at(ai, aj, ak, al);
    g[A] = div_h<POW2>((double)SG * (pn - p0), h, hinv, A);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        if (t == A) continue;
        const int ti = t == 0, tj = t == 1, tk = t == 2, tl = t == 3;
        // corner_average (edge.cpp:16-22): 0.25 * (p0 + p[sa] + p[sb] + p[sa+sb])
        const double plus =
            0.25 * (p0 + pn + S.at(ti, tj, tk, tl) + S.at(ai + ti, aj + tj, ak + tk, al + tl));
        const double minus = 0.25 * (p0 + pn + S.at(-ti, -tj, -tk, -tl) +
                                     S.at(ai - ti, aj - tj, ak - tk, al - tl));
        g[t] = div_h<POW2>(plus - minus, h, hinv, t);
    }
}

template <int F, bool POW2>
__device__ __forceinline__ double face_g2(const Stencil& S, const double h[4], const double hinv[4], double p0) {
    double g[4];
    face_gradient<F, POW2>(S, h, hinv, p0, g);
    return g[0] * g[0] + g[1] * g[1] + g[2] * g[2] + g[3] * g[3];  // edge.cpp:53-54
}

// thread -> interior doxel of colour C in tile t of a persistent grid-stride
// loop over (kPassBX doxels along i) x (kPassBY rows j) x (k, l) tiles
struct Site {
    int i, j, k, l;
    bool valid;
};
__device__ __forceinline__ Site site(const Layout& L, int C, long long t, int tx, int ty) {
    Site s;
    const int bx = (int)(t % tx);
    long long r = t / tx;
    const int by = (int)(r % ty);
    const long long z = r / ty;
    s.k = (int)(z % L.n3) + 1;
    s.l = (int)(z / L.n3) + 1;
    s.j = by * kPassBY + threadIdx.y + 1;
    s.i = 1 + ((1 + s.j + s.k + s.l + L.lpar + C) & 1) + 2 * (bx * kPassBX + (int)threadIdx.x);
    s.valid = s.j <= L.n2 && s.i <= L.n1;
    return s;
}

struct TileGrid {
    int tx, ty;
    long long tiles;
};
__host__ __device__ inline TileGrid tile_grid(const Layout& L) {
    TileGrid g;
    g.tx = ((L.n1 + 1) / 2 + kPassBX - 1) / kPassBX;
    g.ty = (L.n2 + kPassBY - 1) / kPassBY;
    g.tiles = (long long)g.tx * g.ty * L.n3 * L.n4;
    return g;
}

template <int C, bool EXPORT, bool POW2>
#ifndef SSB_ASM_MINB
#define SSB_ASM_MINB 3  // 3 CTAs/SM: 449 vs 464 us per colour on config 1 (fp64-latency bound)
#endif
__global__ void __launch_bounds__(kPassBX * kPassBY, SSB_ASM_MINB) assemble_kernel(const AsmArgs a) {
    const Layout& L = a.L;
    const TileGrid tg = tile_grid(L);
    for (long long t = blockIdx.x; t < tg.tiles; t += gridDim.x) {
    const Site q = site(L, C, t, tg.tx, tg.ty);
    if (!q.valid) continue;
    Stencil S;
    S.f[0] = a.u[0];
    S.f[1] = a.u[1];
    S.row = L.row(q.j, q.k, q.l);
    S.i = q.i;
    S.C = C;
    S.jMax = L.jMax;
    S.kMax = L.kMax;
    S.W = L.W;
    const double p0 = S.at(0, 0, 0, 0);

    double g2[8];
    g2[0] = face_g2<0, POW2>(S, a.h, a.hinv, p0);
    g2[1] = face_g2<1, POW2>(S, a.h, a.hinv, p0);
    g2[2] = face_g2<2, POW2>(S, a.h, a.hinv, p0);
    g2[3] = face_g2<3, POW2>(S, a.h, a.hinv, p0);
    g2[4] = face_g2<4, POW2>(S, a.h, a.hinv, p0);
    g2[5] = face_g2<5, POW2>(S, a.h, a.hinv, p0);
    g2[6] = face_g2<6, POW2>(S, a.h, a.hinv, p0);
    g2[7] = face_g2<7, POW2>(S, a.h, a.hinv, p0);

    // solver.cpp:48-56
    double af[8];
    double a_sq_sum = 0.0;
#pragma unroll
    for (int f = 0; f < 8; ++f) {
        const double a_sq = a.eps + g2[f];
        af[f] = sqrt(a_sq);
        a_sq_sum += a_sq;
    }
    const double abar = sqrt(a.eps + 0.125 * a_sq_sum);

    const long long p = S.row * L.W + (q.i >> 1);
    double gv[8];
    if (a.G[C]) {
        const double2* gp = reinterpret_cast<const double2*>(a.G[C] + p * 8);
#pragma unroll
        for (int h2 = 0; h2 < 4; ++h2) {
            const double2 v = __ldcs(gp + h2);
            gv[2 * h2] = v.x;
            gv[2 * h2 + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int f = 0; f < 8; ++f) gv[f] = 1.0;
    }
    // solver.cpp:58-69
    float cf[8];
    double off[8];
    double sum = 0.0;
#pragma unroll
    for (int f = 0; f < 8; ++f) {
        cf[f] = __double2float_rn(-(a.t_h2[f >> 1] * abar * gv[f] / af[f]));
        off[f] = (double)cf[f];
        sum += off[f];
    }
    const double diag = 1.0 - sum;
    if (!isfinite(diag)) atomicOr(a.bad, 1);
    float4* cw = reinterpret_cast<float4*>(a.coef[C] + (S.row * L.Wc + ((q.i - 1) >> 1)) * 8);
    cw[0] = make_float4(cf[0], cf[1], cf[2], cf[3]);
    cw[1] = make_float4(cf[4], cf[5], cf[6], cf[7]);
    if constexpr (EXPORT) {
        const long long pp = L.padded(q.i, q.j, q.k, q.l);
#pragma unroll
        for (int f = 0; f < 8; ++f) a.off_out[pp * 8 + f] = off[f];
        a.diag_out[pp] = diag;
        a.abar_out[pp] = abar;
    }
    }
}

template <int C, bool EXPORT, bool POW2>
__global__ void __launch_bounds__(kPassBX * kPassBY) edge_kernel(const EdgeArgs a) {
    const Layout& L = a.L;
    const TileGrid tg = tile_grid(L);
    for (long long t = blockIdx.x; t < tg.tiles; t += gridDim.x) {
    const Site q = site(L, C, t, tg.tx, tg.ty);
    if (!q.valid) continue;
    Stencil SI, ST;
    SI.f[0] = a.I0[0];
    SI.f[1] = a.I0[1];
    ST.f[0] = a.IT[0];
    ST.f[1] = a.IT[1];
    SI.row = ST.row = L.row(q.j, q.k, q.l);
    SI.i = ST.i = q.i;
    SI.C = ST.C = C;
    SI.jMax = ST.jMax = L.jMax;
    SI.kMax = ST.kMax = L.kMax;
    SI.W = ST.W = L.W;
    const double pi0 = SI.at(0, 0, 0, 0), pt0 = ST.at(0, 0, 0, 0);
    double G[8];
    // edge.cpp:86-94
#define SSB_EDGE_FACE(F)                                                                   \
    {                                                                                      \
        double gi[4], gt[4];                                                               \
        face_gradient<F, POW2>(SI, a.h, a.hinv, pi0, gi);                                  \
        face_gradient<F, POW2>(ST, a.h, a.hinv, pt0, gt);                                  \
        const double ni = sqrt(gi[0] * gi[0] + gi[1] * gi[1] + gi[2] * gi[2] + gi[3] * gi[3]); \
        const double nt = sqrt(gt[0] * gt[0] + gt[1] * gt[1] + gt[2] * gt[2] + gt[3] * gt[3]); \
        const double s = a.delta * ni + a.vartheta * nt;                                   \
        G[F] = 1.0 / (1.0 + a.K * s * s);                                                  \
    }
    SSB_EDGE_FACE(0)
    SSB_EDGE_FACE(1)
    SSB_EDGE_FACE(2)
    SSB_EDGE_FACE(3)
    SSB_EDGE_FACE(4)
    SSB_EDGE_FACE(5)
    SSB_EDGE_FACE(6)
    SSB_EDGE_FACE(7)
#undef SSB_EDGE_FACE
    const long long p = SI.row * L.W + (q.i >> 1);
    double2* gw = reinterpret_cast<double2*>(a.G[C] + p * 8);
#pragma unroll
    for (int h2 = 0; h2 < 4; ++h2) gw[h2] = make_double2(G[2 * h2], G[2 * h2 + 1]);
    if constexpr (EXPORT) {
        const long long pp = L.padded(q.i, q.j, q.k, q.l);
#pragma unroll
        for (int f = 0; f < 8; ++f) a.G_out[pp * 8 + f] = G[f];
    }
    }
}

// thread per padded doxel (i fastest)
__global__ void pack_coef_kernel(const Layout L, const double* __restrict__ off, float* c0,
                                 float* c1) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= L.P) return;
    const int i = (int)(e % L.iMax);
    long long r = e / L.iMax;
    const int j = (int)(r % L.jMax);
    const int k = (int)((r / L.jMax) % L.kMax);
    const int l = (int)(r / ((long long)L.jMax * L.kMax));
    if (i < 1 || i > L.n1 || j < 1 || j > L.n2 || k < 1 || k > L.n3 || l < 1 || l > L.n4) return;
    float* dst = (L.colour(i, j, k, l) ? c1 : c0) + L.coef_slot(i, j, k, l) * 8;
#pragma unroll
    for (int f = 0; f < 8; ++f) dst[f] = (float)off[e * 8 + f];
}

// colour-packed fp32 rows -> padded fp64 off-diagonals (8 per doxel; ghost doxels 0)
__global__ void unpack_coef_kernel(const Layout L, const float* __restrict__ c0, const float* __restrict__ c1,
                                   double* off) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= L.P) return;
    const int i = (int)(e % L.iMax);
    long long r = e / L.iMax;
    const int j = (int)(r % L.jMax);
    const int k = (int)((r / L.jMax) % L.kMax);
    const int l = (int)(r / ((long long)L.jMax * L.kMax));
    const bool in = i >= 1 && i <= L.n1 && j >= 1 && j <= L.n2 && k >= 1 && k <= L.n3 && l >= 1 && l <= L.n4;
    const float* src = in ? (L.colour(i, j, k, l) ? c1 : c0) + L.coef_slot(i, j, k, l) * 8 : nullptr;
#pragma unroll
    for (int f = 0; f < 8; ++f) off[e * 8 + f] = in ? (double)src[f] : 0.0;
}

__global__ void pack8_kernel(const Layout L, const double* __restrict__ src, double* d0,
                             double* d1) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= L.P) return;
    const int i = (int)(e % L.iMax);
    long long r = e / L.iMax;
    const int j = (int)(r % L.jMax);
    const int k = (int)((r / L.jMax) % L.kMax);
    const int l = (int)(r / ((long long)L.jMax * L.kMax));
    double* dst = (L.colour(i, j, k, l) ? d1 : d0) + (r * L.W + (i >> 1)) * 8;
#pragma unroll
    for (int f = 0; f < 8; ++f) dst[f] = src[e * 8 + f];
}

struct HeatC {
    double c[4];
};

__global__ void heat_export_kernel(const Layout L, const HeatC hc, double* off, double* diag,
                                   double* abar) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= L.P) return;
    const int i = (int)(e % L.iMax);
    long long r = e / L.iMax;
    const int j = (int)(r % L.jMax);
    const int k = (int)((r / L.jMax) % L.kMax);
    const int l = (int)(r / ((long long)L.jMax * L.kMax));
    const bool interior =
        i >= 1 && i <= L.n1 && j >= 1 && j <= L.n2 && k >= 1 && k <= L.n3 && l >= 1 && l <= L.n4;
    if (!interior) {
#pragma unroll
        for (int f = 0; f < 8; ++f) off[e * 8 + f] = 0.0;
        diag[e] = 0.0;
        abar[e] = 0.0;
        return;
    }
    const int c[4] = {i, j, k, l};
    const int hi[4] = {L.n1, L.n2, L.n3, L.n4};
    double sum = 0.0;
#pragma unroll
    for (int f = 0; f < 8; ++f) {
        const int ax = f >> 1;
        const int nb = c[ax] + ((f & 1) ? 1 : -1);
        if (nb < 1 || nb > hi[ax]) {
            off[e * 8 + f] = 0.0;
        } else {
            off[e * 8 + f] = hc.c[ax];
            sum += hc.c[ax];
        }
    }
    diag[e] = 1.0 - sum;
    abar[e] = 1.0;
}

}  // namespace

static unsigned persistent_grid(const void* fn, long long tiles) {
    int dev = 0, sms = 0, per = 0;
    SSB_CUDA(cudaGetDevice(&dev));
    SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kPassBX * kPassBY, 0));
    return (unsigned)std::min<long long>(tiles, (long long)sms * std::max(1, per));
}

static bool pow2(double h) {
    int e = 0;
    return std::frexp(h, &e) == 0.5;  // mantissa exactly 1 => power of two
}

template <int C, bool EXPORT, bool POW2>
static void asm_launch(cudaStream_t s, const AsmArgs& a) {
    static unsigned grid = 0;
    const TileGrid tg = tile_grid(a.L);
    if (!grid) grid = persistent_grid((const void*)assemble_kernel<C, EXPORT, POW2>, 1LL << 40);
    assemble_kernel<C, EXPORT, POW2><<<(unsigned)std::min<long long>(tg.tiles, grid), dim3(kPassBX, kPassBY), 0, s>>>(a);
    SSB_LAUNCHED();
}

template <int C, bool EXPORT, bool POW2>
static void edge_launch(cudaStream_t s, const EdgeArgs& a) {
    static unsigned grid = 0;
    const TileGrid tg = tile_grid(a.L);
    if (!grid) grid = persistent_grid((const void*)edge_kernel<C, EXPORT, POW2>, 1LL << 40);
    edge_kernel<C, EXPORT, POW2><<<(unsigned)std::min<long long>(tg.tiles, grid), dim3(kPassBX, kPassBY), 0, s>>>(a);
    SSB_LAUNCHED();
}

void launch_assemble(cudaStream_t s, const AsmArgs& a0) {
    AsmArgs a = a0;
    bool p2 = true;
    for (int q = 0; q < 4; ++q) {
        p2 = p2 && pow2(a.h[q]);
        a.hinv[q] = 1.0 / a.h[q];
    }
    // the TMA-staged tile kernel (both colours in one launch) unless the per-call API asks
    // for the padded fp64 exports
    if (!a.off_out && assemble_tile_supported(a.L) && launch_assemble_tile(s, a, p2)) return;
    if (a.off_out) {
        if (p2) { asm_launch<0, true, true>(s, a); asm_launch<1, true, true>(s, a); }
        else { asm_launch<0, true, false>(s, a); asm_launch<1, true, false>(s, a); }
    } else {
        if (p2) { asm_launch<0, false, true>(s, a); asm_launch<1, false, true>(s, a); }
        else { asm_launch<0, false, false>(s, a); asm_launch<1, false, false>(s, a); }
    }
}

void launch_face_coefficients(cudaStream_t s, const EdgeArgs& a0) {
    EdgeArgs a = a0;
    bool p2 = true;
    for (int q = 0; q < 4; ++q) {
        p2 = p2 && pow2(a.h[q]);
        a.hinv[q] = 1.0 / a.h[q];
    }
    // the TMA-staged tile kernel, also for the per-call API's padded export
    if (assemble_tile_supported(a.L) && launch_edge_tile(s, a, p2)) return;
    if (a.G_out) {
        if (p2) { edge_launch<0, true, true>(s, a); edge_launch<1, true, true>(s, a); }
        else { edge_launch<0, true, false>(s, a); edge_launch<1, true, false>(s, a); }
    } else {
        if (p2) { edge_launch<0, false, true>(s, a); edge_launch<1, false, true>(s, a); }
        else { edge_launch<0, false, false>(s, a); edge_launch<1, false, false>(s, a); }
    }
}

void launch_pack_coef(cudaStream_t s, const Layout& L, const double* off, float* c0, float* c1) {
    pack_coef_kernel<<<ceil_div(L.P, 256), 256, 0, s>>>(L, off, c0, c1);
    SSB_LAUNCHED();
}

void launch_unpack_coef(cudaStream_t s, const Layout& L, const float* c0, const float* c1, double* off) {
    unpack_coef_kernel<<<ceil_div(L.P, 256), 256, 0, s>>>(L, c0, c1, off);
    SSB_LAUNCHED();
}

void launch_pack8(cudaStream_t s, const Layout& L, const double* src, double* d0, double* d1) {
    pack8_kernel<<<ceil_div(L.P, 256), 256, 0, s>>>(L, src, d0, d1);
    SSB_LAUNCHED();
}

void launch_heat_export(cudaStream_t s, const Layout& L, double hcv[4], double* off, double* diag,
                        double* abar) {
    HeatC hc;
    for (int a = 0; a < 4; ++a) hc.c[a] = hcv[a];
    heat_export_kernel<<<ceil_div(L.P, 256), 256, 0, s>>>(L, hc, off, diag, abar);
    SSB_LAUNCHED();
}

}  // namespace ssb
