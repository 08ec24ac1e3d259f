"""The error bound behind the certified face gradients (assemble_tile.cu face_sq_cert,
cert_threshold), checked on the CPU with the reference's own rounding sequence.

The reference's scaled tangential difference is d_T = RN(X - Y) with the rounded corner sums
X = RN(RN(RN(p0 + pn) + p_+T) + pn_+T) and Y = RN(RN(RN(p0 + pn) + p_-T) + pn_-T) (edge.cpp:16-22,
:43-45, the 0.25 and 1/h pulled out exactly); the certified value is d'_T = RN(c_T(p) + c_T(pn))
with the central differences c_T = RN(x_+T - x_-T).  The kernel's exactness argument needs

  (1) |d_T - d'_T| <= 26.05 M u_r  (E = 32 M u_r is what the kernel uses), M >= every |u|;
  (2) |F_ex - F'| <= 8.1 u_r F + 2 sqrt(3) E sqrt(F) + 3.1 E^2 for the sum of the four squares
      (reference: sequential RN(d_a^2) sums; certified: one product and three fused multiply-adds);
  (3) |sigma (F_ex - F')| <= rho (eps + sigma F_ex), rho = 40 u_r + 1.75 E r + 3.1 (E r)^2,
      r = sqrt(sigma) / sqrt(eps).

numpy float64 scalar operations are IEEE round-to-nearest like the device's -fmad=false code;
the fused multiply-add is emulated exactly with fractions (one rounding).  Inputs: random
stencils in [0, 1] and [-M, M], near-equal values (cancellation), values one ulp apart around
powers of two, mixed magnitudes, exact zeros.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

UR = 2.0 ** -53


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def face(vals, A):
    """vals: dict of the stencil of one face with normal axis A (sign folded into pn):
    p0, pn and per tangent T: (pt, pmt, pnt, pnmt).  Returns (F_ex, F', max |d - d'|, M)."""
    p0, pn = vals["p0"], vals["pn"]
    d = [0.0] * 4
    dc = [0.0] * 4
    d[A] = dc[A] = 4.0 * (pn - p0)
    s0 = p0 + pn
    err = 0.0
    M = max(abs(p0), abs(pn))
    for T in range(4):
        if T == A:
            continue
        pt, pmt, pnt, pnmt = vals[T]
        M = max(M, abs(pt), abs(pmt), abs(pnt), abs(pnmt))
        X = (s0 + pt) + pnt
        Y = (s0 + pmt) + pnmt
        d[T] = X - Y
        dc[T] = (pt - pmt) + (pnt - pnmt)
        err = max(err, abs(d[T] - dc[T]))
    F_ex = d[0] * d[0] + d[1] * d[1] + d[2] * d[2] + d[3] * d[3]
    acc = dc[A] * dc[A]
    for T in range(4):
        if T != A:
            acc = fma(dc[T], dc[T], acc)
    return F_ex, acc, err, M


def samples(rng, n):
    kinds = ["unit", "signed", "cancel", "ulp", "mixed", "zeros", "powers"]
    for t in range(n):
        kind = kinds[t % len(kinds)]
        k = 2 + 3 * 4
        if kind == "unit":
            v = rng.random(k)
        elif kind == "signed":
            v = rng.uniform(-1, 1, k) * 10.0 ** rng.uniform(-3, 3)
        elif kind == "cancel":  # all near one value: the differences are tiny, the sums large
            v = 0.7 + rng.normal(0, 1e-9, k)
        elif kind == "ulp":  # one or two ulps around a power of two
            base = 2.0 ** rng.integers(-4, 4)
            v = base + rng.integers(-3, 4, k) * base * UR
        elif kind == "mixed":  # a few large, the rest tiny
            v = rng.random(k) * 1e-6
            v[rng.integers(0, k, 3)] = rng.random(3)
        elif kind == "zeros":
            v = rng.random(k)
            v[rng.random(k) < 0.5] = 0.0
        else:
            v = 2.0 ** rng.integers(-10, 3, k).astype(float) * rng.choice([-1.0, 1.0], k)
        A = int(rng.integers(0, 4))
        vals = {"p0": float(v[0]), "pn": float(v[1])}
        q = 2
        for T in range(4):
            if T == A:
                continue
            vals[T] = tuple(float(x) for x in v[q:q + 4])
            q += 4
        yield vals, A


def test_certified_gradient_bound():
    rng = np.random.default_rng(2111)
    worst_d = 0.0
    worst_F = 0.0
    worst_rho = 0.0
    for vals, A in samples(rng, 120000):
        F_ex, F_c, err, M = face(vals, A)
        if M == 0.0:
            continue
        E = 32.0 * M * UR
        # (1) the tangential differences
        ratio_d = err / (M * UR)
        worst_d = max(worst_d, ratio_d)
        assert ratio_d <= 26.05, (vals, A, ratio_d)
        # (2) the sum of squares
        F = max(F_ex, F_c)
        bound = 8.1 * UR * F + 2.0 * math.sqrt(3.0) * E * math.sqrt(F) + 3.1 * E * E
        assert abs(F_ex - F_c) <= bound, (vals, A, F_ex, F_c, bound)
        worst_F = max(worst_F, abs(F_ex - F_c) / bound if bound else 0.0)
        # (3) relative to A_f^2 = eps + sigma F for the BASELINE spacings and a range of eps
        for h in (1 / 32, 1 / 64, 1 / 128, 1.0):
            sig = (0.25 / h) ** 2
            for eps in (1e-3, 1e-6, 1.0):
                r = math.sqrt(sig) / math.sqrt(eps)
                rho = 40 * UR + 1.75 * E * r + 3.1 * (E * r) ** 2
                lhs = abs(sig * (F_ex - F_c))
                assert lhs <= rho * (eps + sig * F_ex), (vals, A, h, eps, lhs, rho)
                worst_rho = max(worst_rho, lhs / (rho * (eps + sig * F_ex)))
    print(f"max |d - d'| = {worst_d:.2f} M u_r (bound 26.05, kernel uses 32); "
          f"sum-of-squares error at most {worst_F:.3f} of its bound; rho at most {worst_rho:.3f} of its bound")


def test_threshold_formula_matches_the_kernel():
    """cert_threshold (assemble_tile.cu) restated: T = 1.25 (11700 + rho 2^53) ulps, in use only
    below 2^17; the BASELINE settings (u in [0, 1], eps = 1e-3) give T ~ 2^15 at h = 1/32 and
    certified gradients at h = 1/64 too."""
    def T(M, h, eps, nr1=True):
        Er = 32.0 * M * UR * (0.25 / h) / math.sqrt(eps)
        rho = 40 * UR + 1.75 * Er + 3.1 * Er * Er
        t = 1.25 * ((11700.0 if nr1 else 20.0) + rho * 2.0 ** 53)
        return max(16384 if nr1 else 512, int(t) + 1) if t < 131072.0 else 0

    assert 16384 < T(1.0, 1 / 32, 1e-3) < 65536
    assert 0 < T(1.0, 1 / 64, 1e-3) < 131072
    assert T(1e3, 1 / 32, 1e-3) == 0  # large |u|: exact scaled gradients
    assert T(1.0, 1 / 32, 1e-12) == 0  # tiny eps: the bound is too loose to pay
