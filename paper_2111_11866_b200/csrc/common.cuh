// common.cuh -- shared layout, error handling and launch bookkeeping of the
// B200 SUBSURF library.
//
// Device layout ("colour-packed"): the ghost-padded box of the reference
// (grid.hpp:91-119) is split by red/black colour, colour(i,j,k,l) = (i+j+k+l)&1
// (red = 0 = even, solver.cpp:244/291/341, 1-based padded GLOBAL indices).
// Each colour is a dense array of rows; row r = (l*kMax + k)*jMax + j holds the
// doxels of that colour at packed position m = i >> 1 (W = (n1+3)/2 slots per
// row, rounded up to even so rows are 16-byte aligned for bulk copies).  For any
// doxel the j/k/l neighbours sit at the same m in the other
// colour's array one row stride away, and the i-1 / i+1 neighbours at
// m' = (i-1)>>1 and (i+1)>>1.  A colour half-sweep therefore reads and writes
// whole 32-byte sectors only (no half-used sectors as with the interleaved
// Field4D layout).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "subsurf_b200.h"

namespace ssb {

struct Layout {
    int n1, n2, n3, n4;   // local extents (n4 = slices owned by this slab)
    int l0;               // global l of local plane 0 (slab offset; 0 for a whole grid)
    int n4g;              // global number of slices
    int lpar;             // l0 & 1: colour parity uses GLOBAL l (solver.cpp:244)
    int glo, ghi;         // local planes 0 / n4+1 are global ghosts (else: halos)
    int iMax, jMax, kMax, lMax;
    int W;            // packed slots per row
    int Wc;           // coefficient slots per row: interior doxels of one colour, (n1+1)/2
                      // (slot s <-> i = 2s + 1 + parity; no ghost slot, rows stay 32-byte aligned)
    long long rows;   // jMax * kMax * lMax
    long long cs;     // elements per colour array = rows * W
    long long sj, sk, sl;  // packed row strides for j, k, l neighbours
    long long P;      // padded doxels of the reference layout

    static Layout make(const ss_grid& g, int l0 = 0, int n4g = -1) {
        Layout L;
        L.n1 = g.n1; L.n2 = g.n2; L.n3 = g.n3; L.n4 = g.n4;
        L.l0 = l0;
        L.n4g = n4g < 0 ? g.n4 : n4g;
        L.lpar = l0 & 1;
        L.glo = l0 == 0;
        L.ghi = l0 + g.n4 == L.n4g;
        L.iMax = g.n1 + 2; L.jMax = g.n2 + 2; L.kMax = g.n3 + 2; L.lMax = g.n4 + 2;
        L.W = (((L.iMax + 1) / 2) + 1) & ~1;  // even: every packed row starts 16-byte aligned (TMA)
        L.Wc = (g.n1 + 1) / 2;
        L.rows = (long long)L.jMax * L.kMax * L.lMax;
        L.cs = L.rows * L.W;
        L.sj = L.W;
        L.sk = (long long)L.W * L.jMax;
        L.sl = (long long)L.W * L.jMax * L.kMax;
        L.P = (long long)L.iMax * L.rows;
        return L;
    }
    __host__ __device__ __forceinline__ long long row(int j, int k, int l) const {
        return ((long long)l * kMax + k) * jMax + j;
    }
    __host__ __device__ __forceinline__ long long padded(int i, int j, int k, int l) const {
        return row(j, k, l) * iMax + i;
    }
    __host__ __device__ __forceinline__ long long packed(int i, int j, int k, int l) const {
        return row(j, k, l) * W + (i >> 1);
    }
    // red = 0 <=> (i + j + k + l_global) even
    __host__ __device__ __forceinline__ int colour(int i, int j, int k, int l) const {
        return (i + j + k + l + lpar) & 1;
    }
    long long plane() const { return (long long)jMax * kMax * W; }  // one colour, one l-plane
    // index of doxel (i, j, k, l) in a colour's coefficient rows (8 floats each)
    __host__ __device__ __forceinline__ long long coef_slot(int i, int j, int k, int l) const {
        return row(j, k, l) * Wc + ((i - 1) >> 1);
    }
};

// A colour-packed scalar field: two device arrays (red, black).
struct PField {
    double* c[2] = {nullptr, nullptr};
};

// Error plumbing: internal failures throw ssb::Error, the C ABI catches and
// converts to a status code + message (ss_last_error()).
struct Error : std::runtime_error {
    ss_status code;
    Error(ss_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);
extern std::atomic<unsigned long long> g_launches;

inline void count_launch(unsigned long long n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define SSB_CUDA(expr)                                                                      \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            throw ::ssb::Error(SS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define SSB_LAUNCHED()                                                                      \
    do {                                                                                    \
        ::ssb::count_launch();                                                              \
        cudaError_t _e = cudaGetLastError();                                                \
        if (_e != cudaSuccess)                                                              \
            throw ::ssb::Error(SS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

inline unsigned ceil_div(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

}  // namespace ssb
