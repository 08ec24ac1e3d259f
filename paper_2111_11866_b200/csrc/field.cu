// field.cu -- layout conversion and whole-field kernels: pack/unpack between
// the reference's ghost-padded Field4D layout and the colour-packed device
// layout, Dirichlet / mirror ghosts (grid.cpp:126-156), deterministic interior
// reductions (grid.cpp:158-171) and the 0.5-superlevel mask (tracking.cpp:35-52).
#include "kernels.cuh"

namespace ssb {

namespace {

struct Pos {
    int i, j, k, l;
    long long row;
};

__device__ __forceinline__ Pos decode_padded(const Layout& L, long long e) {
    Pos p;
    p.i = (int)(e % L.iMax);
    p.row = e / L.iMax;
    p.j = (int)(p.row % L.jMax);
    p.k = (int)((p.row / L.jMax) % L.kMax);
    p.l = (int)(p.row / ((long long)L.jMax * L.kMax));
    return p;
}

__device__ __forceinline__ Pos decode_interior(const Layout& L, long long e) {
    Pos p;
    p.i = (int)(e % L.n1) + 1;
    long long r = e / L.n1;
    p.j = (int)(r % L.n2) + 1;
    r /= L.n2;
    p.k = (int)(r % L.n3) + 1;
    p.l = (int)(r / L.n3) + 1;
    p.row = L.row(p.j, p.k, p.l);
    return p;
}

__device__ __forceinline__ double* at(const Layout& L, PField f, int i, int j, int k, int l) {
    return f.c[L.colour(i, j, k, l)] + L.packed(i, j, k, l);
}

// Ghost-shell enumeration: the two hyperplanes c[axis] = 0 / max of one axis
// (face_count(axis) positions each, the other three coordinates over their whole
// padded range, lowest axis fastest).  Kernels over ghosts walk these instead of
// the whole padded box (config 1: 2.3 M instead of 19 M positions).
__host__ __device__ __forceinline__ long long face_count(const Layout& L, int axis) {
    const long long ext[4] = {L.iMax, L.jMax, L.kMax, L.lMax};
    long long n = 1;
    for (int b = 0; b < 4; ++b)
        if (b != axis) n *= ext[b];
    return n;
}

__device__ __forceinline__ void face_pos(const Layout& L, int axis, long long e, int c[4]) {
    const long long F = face_count(L, axis);
    const int ext[4] = {L.iMax, L.jMax, L.kMax, L.lMax};
    const int side = (int)(e / F);
    long long r = e - side * F;
    for (int b = 0; b < 4; ++b) {
        if (b == axis) continue;
        c[b] = (int)(r % ext[b]);
        r /= ext[b];
    }
    c[axis] = side ? ext[axis] - 1 : 0;
}

// e over the 8 hyperplanes of all axes -> a ghost position (edges repeat)
__device__ __forceinline__ void shell_pos(const Layout& L, long long e, int c[4]) {
    int axis = 0;
    while (axis < 3 && e >= 2 * face_count(L, axis)) {
        e -= 2 * face_count(L, axis);
        ++axis;
    }
    face_pos(L, axis, e, c);
}

__host__ __device__ __forceinline__ long long shell_count(const Layout& L) {
    return 2 * (face_count(L, 0) + face_count(L, 1) + face_count(L, 2) + face_count(L, 3));
}

// one warp per padded row (j, k, l): coalesced reads of the reference layout,
// half-warp-contiguous writes into each colour's packed row
struct RowPos {
    int j, k, l;
    bool ghost_row;  // j, k or l is a ghost/halo index: every doxel of the row is a ghost
};
__device__ __forceinline__ RowPos decode_row(const Layout& L, long long r) {
    RowPos p;
    p.j = (int)(r % L.jMax);
    const long long t = r / L.jMax;
    p.k = (int)(t % L.kMax);
    p.l = (int)(t / L.kMax);
    p.ghost_row = p.j == 0 || p.j > L.n2 || p.k == 0 || p.k > L.n3 || p.l == 0 || p.l > L.n4;
    return p;
}

__global__ void pack_kernel(const Layout L, const double* __restrict__ src, PField dst, PField t0,
                            PField t1, PField t2) {
    const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= L.rows) return;
    const RowPos p = decode_row(L, r);
    const int par = (p.j + p.k + p.l + L.lpar) & 1;
    for (int i = lane; i < L.iMax; i += 32) {
        const int c = (i + par) & 1;
        const long long q = r * L.W + (i >> 1);
        const double v = src[r * L.iMax + i];
        dst.c[c][q] = v;
        if (p.ghost_row || i == 0 || i > L.n1) {
            if (t0.c[c]) t0.c[c][q] = v;
            if (t1.c[c]) t1.c[c][q] = v;
            if (t2.c[c]) t2.c[c][q] = v;
        }
    }
}

// compact interior rows (n1 doubles, i fastest, then j, k, l; no ghosts) of slices
// [l_lo, l_hi] <-> the colour-packed field: one warp per interior row
__global__ void pack_interior_kernel(const Layout L, const double* __restrict__ src, PField dst, int l_lo,
                                     long long nrows) {
    const long long q = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= nrows) return;
    const int j = (int)(q % L.n2) + 1;
    const long long t = q / L.n2;
    const int k = (int)(t % L.n3) + 1;
    const int l = (int)(t / L.n3) + l_lo;
    const long long r = L.row(j, k, l);
    const long long cq = ((long long)(l - 1) * L.n3 + (k - 1)) * L.n2 + (j - 1);
    const int par = (j + k + l + L.lpar) & 1;
    for (int i = 1 + lane; i <= L.n1; i += 32) dst.c[(i + par) & 1][r * L.W + (i >> 1)] = src[cq * L.n1 + i - 1];
}

__global__ void unpack_interior_kernel(const Layout L, PField src, double* __restrict__ dst, int l_lo,
                                       long long nrows) {
    const long long q0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q0 >= nrows) return;
    const long long q = q0 + (long long)(l_lo - 1) * L.n2 * L.n3;  // compact row index from slice 1
    const int j = (int)(q % L.n2) + 1;
    const long long t = q / L.n2;
    const int k = (int)(t % L.n3) + 1;
    const int l = (int)(t / L.n3) + 1;
    const long long r = L.row(j, k, l);
    const int par = (j + k + l + L.lpar) & 1;
    for (int i = 1 + lane; i <= L.n1; i += 32) dst[q * L.n1 + i - 1] = src.c[(i + par) & 1][r * L.W + (i >> 1)];
}

__global__ void unpack_kernel(const Layout L, PField src, double* __restrict__ dst) {
    const long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= L.rows) return;
    const RowPos p = decode_row(L, r);
    const int par = (p.j + p.k + p.l + L.lpar) & 1;
    for (int i = lane; i < L.iMax; i += 32) dst[r * L.iMax + i] = src.c[(i + par) & 1][r * L.W + (i >> 1)];
}

__global__ void fill_kernel(const Layout L, PField f, double v) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= L.P) return;
    const Pos p = decode_padded(L, e);
    f.c[L.colour(p.i, p.j, p.k, p.l)][p.row * L.W + (p.i >> 1)] = v;
}

__global__ void set_ghosts_kernel(const Layout L, PField f, double v) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= shell_count(L)) return;
    int c[4];
    shell_pos(L, e, c);
    *at(L, f, c[0], c[1], c[2], c[3]) = v;
}

// grid.cpp:138-156, one launch per axis (axis order 0..3 carries edges/corners)
__global__ void mirror_kernel(const Layout L, PField f, int axis) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= 2 * face_count(L, axis)) return;
    int c[4];
    face_pos(L, axis, e, c);
    const int hi[4] = {L.n1 + 1, L.n2 + 1, L.n3 + 1, L.n4 + 1};
    // slab halo planes are the neighbours' data, not ghosts
    if (axis == 3 && ((c[3] == 0 && !L.glo) || (c[3] == hi[3] && !L.ghi))) return;
    const int dst[4] = {c[0], c[1], c[2], c[3]};
    c[axis] += c[axis] == 0 ? 1 : -1;
    *at(L, f, dst[0], dst[1], dst[2], dst[3]) = *at(L, f, c[0], c[1], c[2], c[3]);
}

__global__ void fill_raw_kernel(double* p, long long n, double v) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        p[e] = v;
}

__global__ void copy_ghosts_kernel(const Layout L, PField dst, PField src) {
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= shell_count(L)) return;
    int p[4];
    shell_pos(L, e, p);
    const int c = L.colour(p[0], p[1], p[2], p[3]);
    const long long q = L.packed(p[0], p[1], p[2], p[3]);
    dst.c[c][q] = src.c[c][q];
}

__global__ void copy_kernel(long long n, double* __restrict__ d, const double* __restrict__ s) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x)
        d[e] = s[e];
}

__device__ __forceinline__ double bsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    __shared__ double ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? ws[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    }
    return v;
}

__device__ __forceinline__ void bminmax(double& lo, double& hi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_down_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_down_sync(0xffffffffu, hi, o));
    }
    __shared__ double wl[32], wh[32];
    if ((threadIdx.x & 31) == 0) {
        wl[threadIdx.x >> 5] = lo;
        wh[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const bool ok = threadIdx.x < (blockDim.x >> 5);
        lo = ok ? wl[threadIdx.x] : INFINITY;
        hi = ok ? wh[threadIdx.x] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fmin(lo, __shfl_down_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_down_sync(0xffffffffu, hi, o));
        }
    }
}

__global__ void __launch_bounds__(256) norm_part_kernel(const Layout L, PField f, double* part) {
    const long long N = (long long)L.n1 * L.n2 * L.n3 * L.n4;
    double s = 0.0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N;
         e += (long long)gridDim.x * blockDim.x) {
        const Pos p = decode_interior(L, e);
        const double v = *at(L, f, p.i, p.j, p.k, p.l);
        s += v * v;
    }
    s = bsum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// Per-slice sum of squares, in two fixed-shape steps: block (c, l) sums the
// interior slots of rows c, c + kNormChunks, ... of slice l (both colours,
// one warp per row, coalesced), then one thread per slice adds the kNormChunks
// partials in order.  The result depends only on the slice's values (not on
// the slab decomposition).
__global__ void __launch_bounds__(256) slice_norm_part_kernel(const Layout L, PField f, double* part) {
    const int l = blockIdx.y + 1;
    const int rows = L.n2 * L.n3;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int U = 4;  // rows whose loads are in flight together
    double s = 0.0;
    for (int r0 = blockIdx.x + kNormChunks * warp; r0 < rows; r0 += kNormChunks * 8 * U) {
        for (int m0 = 0; m0 < L.W; m0 += 32) {
            const int m = m0 + lane;
            double v[U][2];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = r0 + u * kNormChunks * 8;
                const int j = r % L.n2 + 1, k = r / L.n2 + 1;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    // slot m of colour c holds i = 2m + b
                    const int i = 2 * m + ((c + j + k + l + L.lpar) & 1);
                    v[u][c] = r < rows && m < L.W && i >= 1 && i <= L.n1 ? f.c[c][L.row(j, k, l) * L.W + m] : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int c = 0; c < 2; ++c) s += v[u][c] * v[u][c];
        }
    }
    s = bsum(s);
    if (threadIdx.x == 0) part[(long long)blockIdx.y * kNormChunks + blockIdx.x] = s;
}

__global__ void norm_slices_kernel(const double* part, int n4, double* out) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= n4) return;
    double s = 0.0;
    for (int c = 0; c < kNormChunks; ++c) s += part[(long long)l * kNormChunks + c];
    out[l] = s;
}

__global__ void __launch_bounds__(256) sum_final_kernel(const double* part, int n, double* out) {
    double s = 0.0;
    for (int q = threadIdx.x; q < n; q += blockDim.x) s += part[q];
    s = bsum(s);
    if (threadIdx.x == 0) *out = s;
}

__global__ void __launch_bounds__(256) minmax_part_kernel(const Layout L, PField f, double* part) {
    const long long N = (long long)L.n1 * L.n2 * L.n3 * L.n4;
    double lo = INFINITY, hi = -INFINITY;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N;
         e += (long long)gridDim.x * blockDim.x) {
        const Pos p = decode_interior(L, e);
        const double v = *at(L, f, p.i, p.j, p.k, p.l);
        lo = fmin(lo, v);
        hi = fmax(hi, v);
    }
    bminmax(lo, hi);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = lo;
        part[2 * blockIdx.x + 1] = hi;
    }
}

__global__ void __launch_bounds__(256) minmax_final_kernel(const double* part, int n, double* out) {
    double lo = INFINITY, hi = -INFINITY;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        lo = fmin(lo, part[2 * q]);
        hi = fmax(hi, part[2 * q + 1]);
    }
    bminmax(lo, hi);
    if (threadIdx.x == 0) {
        out[0] = lo;
        out[1] = hi;
    }
}

__global__ void mask_kernel(const Layout L, PField f, double level, uint8_t* mask) {
    const long long N = (long long)L.n1 * L.n2 * L.n3 * L.n4;
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= N) return;
    const Pos p = decode_interior(L, e);
    mask[e] = *at(L, f, p.i, p.j, p.k, p.l) >= level ? 1 : 0;
}

}  // namespace

void launch_pack(cudaStream_t s, const Layout& L, const double* src, PField dst, PField t0,
                 PField t1, PField t2) {
    pack_kernel<<<ceil_div(L.rows * 32, 256), 256, 0, s>>>(L, src, dst, t0, t1, t2);
    SSB_LAUNCHED();
}

void launch_fill_raw(cudaStream_t s, double* p, long long n, double v) {
    fill_raw_kernel<<<kReduceBlocks * 2, 256, 0, s>>>(p, n, v);
    SSB_LAUNCHED();
}

void launch_copy_ghosts(cudaStream_t s, const Layout& L, PField dst, PField src) {
    copy_ghosts_kernel<<<ceil_div(shell_count(L), 256), 256, 0, s>>>(L, dst, src);
    SSB_LAUNCHED();
}

void launch_pack_interior(cudaStream_t s, const Layout& L, const double* src, PField dst, int l_lo, int l_hi) {
    const long long nrows = (long long)L.n2 * L.n3 * (l_hi - l_lo + 1);
    if (nrows <= 0) return;
    pack_interior_kernel<<<ceil_div(nrows * 32, 256), 256, 0, s>>>(L, src, dst, l_lo, nrows);
    SSB_LAUNCHED();
}

void launch_unpack_interior(cudaStream_t s, const Layout& L, PField src, double* dst, int l_lo, int l_hi) {
    if (l_hi < 0) l_hi = L.n4;
    const long long nrows = (long long)L.n2 * L.n3 * (l_hi - l_lo + 1);
    if (nrows <= 0) return;
    unpack_interior_kernel<<<ceil_div(nrows * 32, 256), 256, 0, s>>>(L, src, dst, l_lo, nrows);
    SSB_LAUNCHED();
}

void launch_unpack(cudaStream_t s, const Layout& L, PField src, double* dst) {
    unpack_kernel<<<ceil_div(L.rows * 32, 256), 256, 0, s>>>(L, src, dst);
    SSB_LAUNCHED();
}

void launch_fill(cudaStream_t s, const Layout& L, PField f, double v) {
    fill_kernel<<<ceil_div(L.P, 256), 256, 0, s>>>(L, f, v);
    SSB_LAUNCHED();
}

void launch_set_ghosts(cudaStream_t s, const Layout& L, PField f, double v) {
    set_ghosts_kernel<<<ceil_div(shell_count(L), 256), 256, 0, s>>>(L, f, v);
    SSB_LAUNCHED();
}

void launch_mirror_ghosts(cudaStream_t s, const Layout& L, PField f, int a0, int a1) {
    for (int axis = a0; axis < a1; ++axis) {
        mirror_kernel<<<ceil_div(2 * face_count(L, axis), 256), 256, 0, s>>>(L, f, axis);
        SSB_LAUNCHED();
    }
}

void launch_copy_field(cudaStream_t s, const Layout& L, PField dst, PField src) {
    for (int c = 0; c < 2; ++c) {
        copy_kernel<<<kReduceBlocks * 2, 256, 0, s>>>(L.cs, dst.c[c], src.c[c]);
        SSB_LAUNCHED();
    }
}

void launch_norm_sq(cudaStream_t s, const Layout& L, PField f, double* scratch, double* out) {
    norm_part_kernel<<<kReduceBlocks, 256, 0, s>>>(L, f, scratch);
    SSB_LAUNCHED();
    sum_final_kernel<<<1, 256, 0, s>>>(scratch, kReduceBlocks, out);
    SSB_LAUNCHED();
}

void launch_norm_slices(cudaStream_t s, const Layout& L, PField f, double* scratch, double* out) {
    slice_norm_part_kernel<<<dim3(kNormChunks, L.n4), 256, 0, s>>>(L, f, scratch);
    SSB_LAUNCHED();
    norm_slices_kernel<<<ceil_div(L.n4, 128), 128, 0, s>>>(scratch, L.n4, out);
    SSB_LAUNCHED();
}

void launch_minmax(cudaStream_t s, const Layout& L, PField f, double* scratch, double* out2) {
    minmax_part_kernel<<<kReduceBlocks, 256, 0, s>>>(L, f, scratch);
    SSB_LAUNCHED();
    minmax_final_kernel<<<1, 256, 0, s>>>(scratch, kReduceBlocks, out2);
    SSB_LAUNCHED();
}

void launch_mask(cudaStream_t s, const Layout& L, PField f, double level, uint8_t* mask) {
    const long long N = (long long)L.n1 * L.n2 * L.n3 * L.n4;
    mask_kernel<<<ceil_div(N, 256), 256, 0, s>>>(L, f, level, mask);
    SSB_LAUNCHED();
}

}  // namespace ssb
