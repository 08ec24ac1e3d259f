// balls.cu -- per-seed-ball operations: local_threshold (preprocess.cpp:53-102),
// local_rescale (seedinit.cpp:68-99) and build_initial (seedinit.cpp:42-66).
//
// The reference walks the centres table sequentially; later balls see (and
// overwrite) the results of earlier overlapping balls.  The host groups balls
// into waves (session.cu: ball_waves) such that a ball's wave is later than
// that of every earlier ball whose index box intersects it; balls inside one
// wave are disjoint, so one CTA per ball runs them concurrently and the result
// equals the sequential one bit for bit.
#include "kernels.cuh"

namespace ssb {

namespace {

__device__ __forceinline__ double dist_sq(const Ball& b, int i, int j, int k) {
    const double dx = (double)(i - 1) - b.x;
    const double dy = (double)(j - 1) - b.y;
    const double dz = (double)(k - 1) - b.z;
    return dx * dx + dy * dy + dz * dz;
}

__device__ __forceinline__ long long box_size(const Ball& b) {
    if (b.i1 < b.i0 || b.j1 < b.j0 || b.k1 < b.k0) return 0;
    return (long long)(b.i1 - b.i0 + 1) * (b.j1 - b.j0 + 1) * (b.k1 - b.k0 + 1);
}

__device__ __forceinline__ void box_pos(const Ball& b, long long t, int& i, int& j, int& k) {
    const int ni = b.i1 - b.i0 + 1, nj = b.j1 - b.j0 + 1;
    i = b.i0 + (int)(t % ni);
    t /= ni;
    j = b.j0 + (int)(t % nj);
    k = b.k0 + (int)(t / nj);
}

__device__ __forceinline__ double* at(const Layout& L, PField f, int i, int j, int k, int l) {
    return f.c[L.colour(i, j, k, l)] + L.packed(i, j, k, l);
}

// block-wide (min, max); result broadcast to all threads
__device__ void block_minmax(double& lo, double& hi) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double a = __shfl_xor_sync(0xffffffffu, lo, o);
        const double b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = hi < b ? b : hi;
    }
    __shared__ double wl[32], wh[32];
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        wl[threadIdx.x >> 5] = lo;
        wh[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    const int nw = blockDim.x >> 5;
    lo = INFINITY;
    hi = -INFINITY;
    for (int w = 0; w < nw; ++w) {
        lo = wl[w] < lo ? wl[w] : lo;
        hi = hi < wh[w] ? wh[w] : hi;
    }
}

__global__ void __launch_bounds__(256) ball_minmax_kernel(const Layout L, PField f,
                                                          const Ball* balls, double* ab,
                                                          int* empty) {
    const Ball b = balls[blockIdx.x];
    const long long nb = box_size(b);
    double lo = INFINITY, hi = -INFINITY;
    for (long long t = threadIdx.x; t < nb; t += blockDim.x) {
        int i, j, k;
        box_pos(b, t, i, j, k);
        if (!(dist_sq(b, i, j, k) <= b.r_sq)) continue;
        const double v = *at(L, f, i, j, k, b.l);
        lo = v < lo ? v : lo;
        hi = hi < v ? v : hi;
    }
    block_minmax(lo, hi);
    if (threadIdx.x == 0) {
        ab[2 * blockIdx.x] = lo;
        ab[2 * blockIdx.x + 1] = hi;
        if (lo > hi) atomicMin(empty, (int)blockIdx.x);  // "ball covers no doxels"
    }
}

__global__ void __launch_bounds__(256) threshold_write_kernel(const Layout L, PField img,
                                                              PField out, const Ball* balls,
                                                              const double* ab, double lambda) {
    const Ball b = balls[blockIdx.x];
    const double alpha = ab[2 * blockIdx.x], beta = ab[2 * blockIdx.x + 1];
    const double th = lambda * alpha + (1.0 - lambda) * beta;  // preprocess.cpp:93
    const long long nb = box_size(b);
    for (long long t = threadIdx.x; t < nb; t += blockDim.x) {
        int i, j, k;
        box_pos(b, t, i, j, k);
        if (!(dist_sq(b, i, j, k) <= b.r_sq)) continue;
        const double v = *at(L, img, i, j, k, b.l);
        *at(L, out, i, j, k, b.l) = v >= th ? beta : alpha;
    }
}

__global__ void __launch_bounds__(512) rescale_kernel(const Layout L, PField u, const Ball* balls) {
    const Ball b = balls[blockIdx.x];
    const long long nb = box_size(b);
    double lo = INFINITY, hi = -INFINITY;
    for (long long t = threadIdx.x; t < nb; t += blockDim.x) {
        int i, j, k;
        box_pos(b, t, i, j, k);
        if (dist_sq(b, i, j, k) > b.r_sq) continue;
        const double v = *at(L, u, i, j, k, b.l);
        lo = v < lo ? v : lo;
        hi = hi < v ? v : hi;
    }
    block_minmax(lo, hi);
    if (!(hi > lo)) return;  // seedinit.cpp:90
    const double scale = 1.0 / (hi - lo);
    for (long long t = threadIdx.x; t < nb; t += blockDim.x) {
        int i, j, k;
        box_pos(b, t, i, j, k);
        if (dist_sq(b, i, j, k) > b.r_sq) continue;
        double* p = at(L, u, i, j, k, b.l);
        *p = (*p - lo) * scale;
    }
}

__global__ void __launch_bounds__(256) initial_kernel(const Layout L, PField u, const Ball* balls,
                                                      double v, double R, int profile) {
    const Ball b = balls[blockIdx.x];
    const double floor_value = 1.0 / (R + v);
    const long long nb = box_size(b);
    for (long long t = threadIdx.x; t < nb; t += blockDim.x) {
        int i, j, k;
        box_pos(b, t, i, j, k);
        const double d = sqrt(dist_sq(b, i, j, k));
        if (d > R) continue;
        const double value = profile == 0 ? 1.0 / (d + v) - floor_value : 1.0 - d / R;
        double* p = at(L, u, i, j, k, b.l);
        *p = *p < value ? value : *p;
    }
}

}  // namespace

void launch_ball_minmax(cudaStream_t s, const Layout& L, PField f, const Ball* balls, int n,
                        double* ab, int* empty_flag) {
    if (n <= 0) return;
    ball_minmax_kernel<<<n, 256, 0, s>>>(L, f, balls, ab, empty_flag);
    SSB_LAUNCHED();
}

void launch_threshold_write(cudaStream_t s, const Layout& L, PField img, PField out,
                            const Ball* balls, int n, const double* ab, double lambda) {
    if (n <= 0) return;
    threshold_write_kernel<<<n, 256, 0, s>>>(L, img, out, balls, ab, lambda);
    SSB_LAUNCHED();
}

void launch_rescale(cudaStream_t s, const Layout& L, PField u, const Ball* balls, int n) {
    if (n <= 0) return;
    rescale_kernel<<<n, 512, 0, s>>>(L, u, balls);
    SSB_LAUNCHED();
}

void launch_initial(cudaStream_t s, const Layout& L, PField u, const Ball* balls, int n, double v,
                    double R, int profile) {
    if (n <= 0) return;
    initial_kernel<<<n, 256, 0, s>>>(L, u, balls, v, R, profile);
    SSB_LAUNCHED();
}

}  // namespace ssb
