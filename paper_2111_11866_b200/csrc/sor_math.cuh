// sor_math.cuh -- the per-doxel red-black SOR arithmetic (solver.cpp:292-313,
// 347-356), shared by the LDG and the TMA-fed pass kernels.  Expression order
// is the reference's; the library is compiled with -fmad=false.
#pragma once

#include "kernels.cuh"

namespace ssb {

// Operands of one doxel update; loads are split from the arithmetic so a
// thread can put the loads of several doxels in flight before the first store.
struct DoxelIn {
    float c[8];  // heat: exact float values of float(-dt/h^2), so nothing is lost
    double rhs, u0, nb[8];
    long long p;
};

// store of the new value; with an L2 cache policy (TMA pass) or plain (LDG pass)
__device__ __forceinline__ void store_u(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// The update of solver.cpp:292-313: the new value and the squared residual
// contribution (black: in-sweep, :309-312; red: of the incoming state, :347-356).
// Every rounding is the reference's: the products c_f * u_f are formed once and
// feed both the update (acc -= p_f) and the red residual (res += p_f) -- the
// reference evaluates the same products in both places -- so the three
// dependency chains (diag sum, acc, residual) can overlap.
template <int C>
__device__ __forceinline__ void doxel_update(const SorArgs& a, const DoxelIn& d, double& unew, double& r2) {
    const double c0 = (double)d.c[0], c1 = (double)d.c[1], c2 = (double)d.c[2];
    const double c3 = (double)d.c[3], c4 = (double)d.c[4], c5 = (double)d.c[5];
    const double c6 = (double)d.c[6], c7 = (double)d.c[7];
    const double p0 = c0 * d.nb[0], p1 = c1 * d.nb[1], p2 = c2 * d.nb[2], p3 = c3 * d.nb[3];
    const double p4 = c4 * d.nb[4], p5 = c5 * d.nb[5], p6 = c6 * d.nb[6], p7 = c7 * d.nb[7];
    const double dg = 1.0 - (c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7);
    double acc = d.rhs;
    acc -= p0;
    acc -= p1;
    acc -= p2;
    acc -= p3;
    acc -= p4;
    acc -= p5;
    acc -= p6;
    acc -= p7;
    if constexpr (C == 0) {
        double res = dg * d.u0 - d.rhs;
        res += p0;
        res += p1;
        res += p2;
        res += p3;
        res += p4;
        res += p5;
        res += p6;
        res += p7;
        const double ubar = acc / dg;
        unew = a.omega * ubar + a.keep * d.u0;
        r2 = res * res;
    } else {
        const double ubar = acc / dg;
        unew = a.omega * ubar + a.keep * d.u0;
        const double res = dg * (unew - ubar);
        r2 = res * res;
    }
}

// the update alone (no residual): the same bits of unew
template <int C>
__device__ __forceinline__ void doxel_update_nores(const SorArgs& a, const DoxelIn& d, double& unew) {
    const double c0 = (double)d.c[0], c1 = (double)d.c[1], c2 = (double)d.c[2];
    const double c3 = (double)d.c[3], c4 = (double)d.c[4], c5 = (double)d.c[5];
    const double c6 = (double)d.c[6], c7 = (double)d.c[7];
    const double dg = 1.0 - (c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7);
    double acc = d.rhs;
    acc -= c0 * d.nb[0];
    acc -= c1 * d.nb[1];
    acc -= c2 * d.nb[2];
    acc -= c3 * d.nb[3];
    acc -= c4 * d.nb[4];
    acc -= c5 * d.nb[5];
    acc -= c6 * d.nb[6];
    acc -= c7 * d.nb[7];
    const double ubar = acc / dg;
    unew = a.omega * ubar + a.keep * d.u0;
}

// doxel_update + the store(s) of the new value; returns the squared residual
template <int C, bool HINT = false, bool MIRROR = false>
__device__ __forceinline__ double compute_doxel(const SorArgs& a, const DoxelIn& d,
                                                double* __restrict__ ucw, uint64_t pol = 0,
                                                double* mir_lo = nullptr, double* mir_hi = nullptr) {
    double unew, r2;
    doxel_update<C>(a, d, unew, r2);
    if constexpr (HINT)
        store_u(ucw + d.p, unew, pol);
    else
        ucw[d.p] = unew;
    if constexpr (MIRROR) {  // halo push (uniform per work item)
        if (mir_lo) mir_lo[d.p] = unew;
        if (mir_hi) mir_hi[d.p] = unew;
    }
    return r2;
}

}  // namespace ssb
