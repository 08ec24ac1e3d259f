"""ctypes front-end for the parity checkers (TEST INFRASTRUCTURE ONLY).

Loads ``oracle/liboracle.so`` (the C restatement, ``subsurf_oracle.c``) and,
when present, ``oracle/_ref/libsubsurf_ref.so`` (the unmodified reference
compiled in place).  Only tests/ (incl. tests/perf/), ``__graft_entry__.smoke()``
and bench.py's cpu_baseline / reference legs import this module; the product
package never does.

Arrays are numpy fp64 in the reference's ghost-padded layout, shape
``(n4+2, n3+2, n2+2, n1+2)`` (i fastest), coefficient arrays
``(n4+2, n3+2, n2+2, n1+2, 8)``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsubsurf_ref.so")

OK, ERR_VALIDATION, ERR_NOCONVERGE, ERR_NONFINITE = 0, 1, 2, 3


class Grid(C.Structure):
    _fields_ = [("n1", C.c_int), ("n2", C.c_int), ("n3", C.c_int), ("n4", C.c_int),
                ("h1", C.c_double), ("h2", C.c_double), ("h3", C.c_double), ("h4", C.c_double)]

    @classmethod
    def make(cls, dims, h):
        hs = (h,) * 4 if np.isscalar(h) else tuple(h)
        return cls(*[int(d) for d in dims], *[float(x) for x in hs])

    @property
    def shape(self):
        return (self.n4 + 2, self.n3 + 2, self.n2 + 2, self.n1 + 2)


class Center(C.Structure):
    _fields_ = [("frame", C.c_int), ("x", C.c_double), ("y", C.c_double), ("z", C.c_double),
                ("radius", C.c_double)]


class SegParams(C.Structure):
    _fields_ = [("tau", C.c_double), ("epsilon", C.c_double), ("omega", C.c_double),
                ("sor_tol", C.c_double), ("sor_max_iter", C.c_int), ("n_steps", C.c_int),
                ("rescale_each_step", C.c_int), ("sor_rel_tol", C.c_double),
                ("sigma", C.c_double), ("smooth_steps", C.c_int), ("smooth_tol", C.c_double),
                ("smooth_max_iter", C.c_int), ("smooth_omega", C.c_double),
                ("lambda_", C.c_double), ("background", C.c_double),
                ("K", C.c_double), ("delta", C.c_double), ("vartheta", C.c_double),
                ("init_v", C.c_double), ("init_R", C.c_double), ("init_profile", C.c_int),
                ("rescale_radius", C.c_double)]


class StepDiag(C.Structure):
    _fields_ = [("iterations", C.c_int), ("residual", C.c_double), ("tol", C.c_double),
                ("umin", C.c_double), ("umax", C.c_double)]


def seg_params(**kw) -> SegParams:
    """Defaults of cli.cpp:73-107 / solver.hpp:19-29 / preprocess.hpp:10-30 / edge.hpp:12-18."""
    d = dict(tau=1.0, epsilon=1e-4, omega=1.85, sor_tol=1e-8, sor_max_iter=10000, n_steps=10,
             rescale_each_step=1, sor_rel_tol=0.0, sigma=0.0, smooth_steps=1, smooth_tol=1e-10,
             smooth_max_iter=10000, smooth_omega=1.85, lambda_=0.5, background=0.0, K=1.0,
             delta=1.0, vartheta=0.0, init_v=1.0, init_R=10.0, init_profile=0,
             rescale_radius=float("nan"))  # NaN = std::nullopt: per-row radii
    if kw.get("rescale_radius", 0.0) is None:
        kw["rescale_radius"] = float("nan")
    if "lam" in kw:
        kw["lambda_"] = kw.pop("lam")
    d.update(kw)
    return SegParams(**d)


def centers_array(rows):
    arr = (Center * max(1, len(rows)))()
    for n, r in enumerate(rows):
        arr[n] = Center(int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]))
    return arr, len(rows)


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when the reference is present)."""
    out = subprocess.run(["make", "-C", HERE, "-s"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


_D = C.POINTER(C.c_double)
_G = C.POINTER(Grid)
_CEN = C.POINTER(Center)


class _Lib:
    def __init__(self, path: str, prefix: str, with_workers: bool):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.w = with_workers
        L, pre = self.lib, prefix
        W = [C.c_int] if with_workers else []

        def sig(name, args, res=C.c_int):
            f = getattr(L, pre + name)
            f.argtypes = args
            f.restype = res
            return f

        self._fc = sig("face_coefficients", [_G, _D, _D, C.c_double, C.c_double, C.c_double] + W + [_D])
        self._gsq = sig("face_gradient_sq", [_G, _D, C.c_int, C.c_int, C.c_int, C.c_int, _D])
        self._asm = sig("assemble_step", [_G, _D, _D, C.c_double, C.c_double] + W + [_D, _D, _D])
        self._heat_asm = sig("assemble_heat_step", [_G, C.c_double, _D, _D, _D])
        self._sor = sig("redblack_sor", [_G, _D, _D, _D, C.c_double, C.c_double, C.c_int] + W
                        + [C.POINTER(C.c_int), _D])
        self._heat = sig("heat_smooth", [_G, _D, C.c_double, C.c_int, C.c_double, C.c_double,
                                         C.c_int] + W + [_D])
        self._thr = sig("local_threshold", [_G, _D, _CEN, C.c_int, C.c_double, C.c_double, _D])
        self._init = sig("build_initial", [_G, _CEN, C.c_int, C.c_double, C.c_double, C.c_int, _D])
        self._resc = sig("local_rescale", [_G, _D, _CEN, C.c_int, C.c_double])
        self._mirror = sig("apply_mirror_ghosts", [_G, _D], None)
        self._mask = sig("extract_mask", [_G, _D, C.c_double, C.POINTER(C.c_ubyte)], None)
        self._eoc = sig("eoc_row", [C.c_int, C.c_double, C.c_double, C.c_int] + W + [_D])
        seg_args = [_G, _D, _CEN, C.c_int, C.POINTER(SegParams), _D] + W + [_D, C.POINTER(StepDiag)]
        if with_workers:
            seg_args += [_D, C.POINTER(C.c_longlong), _D]
        self._seg = sig("segment", seg_args)
        if with_workers:
            self._sorrate = sig("sor_rate", [_G, _D, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                             C.c_int, _D])
            self._wimg = sig("write_image4d", [_G, _D, C.c_char_p, C.c_char_p])
            self._wvtk = sig("export_frame_vtk", [_G, _D, C.c_int, C.c_char_p])
            self._wtrj = sig("write_trajectories", [C.c_int, C.POINTER(C.c_int), _D, C.c_char_p])
            self._wlab = sig("export_label_vtks", [_G, _D, C.c_double, C.c_char_p])
            self._segfix = sig("segment_fixed", [_G, _D, _CEN, C.c_int, C.POINTER(SegParams), _D, C.c_int,
                                                 C.c_int, C.c_int, _D, C.POINTER(StepDiag), _D, _D])
        if with_workers:  # tracking: the reference itself (tracking.cpp) is the checker
            _I = C.POINTER(C.c_int)
            self._lab = sig("label_components", [_G, C.POINTER(C.c_ubyte), _I, _I])
            self._dc = sig("distance_centers", [_G, _I, _I, C.POINTER(C.c_longlong), C.c_int, _I])
            self._bt = sig("backtrack_link", [_G, _I, _I, _I, _I, _I])
            self._trk = sig("track", [_G, _D, C.c_double, C.c_int, C.c_double, _I, _D, C.c_int, _I])

    def _wk(self, workers):
        return [int(workers)] if self.w else []

    # ---- wrappers (numpy in, numpy out; status code returned where meaningful) ----
    def face_coefficients(self, g, I0s, ITs, K, delta, vartheta, workers=1):
        G = np.empty(g.shape + (8,))
        st = self._fc(C.byref(g), _p(I0s), _p(ITs), K, delta, vartheta, *self._wk(workers), _p(G))
        return st, G

    def face_gradient_sq(self, g, u, i, j, k, l):
        out = np.empty(8)
        self._gsq(C.byref(g), _p(u), i, j, k, l, _p(out))
        return out

    def assemble_step(self, g, u, G, tau, eps, workers=1):
        off = np.zeros(g.shape + (8,))
        dg = np.zeros(g.shape)
        ab = np.zeros(g.shape)
        st = self._asm(C.byref(g), _p(u), _p(G), tau, eps, *self._wk(workers), _p(off), _p(dg), _p(ab))
        return st, off, dg, ab

    def assemble_heat_step(self, g, dt):
        off = np.zeros(g.shape + (8,))
        dg = np.zeros(g.shape)
        ab = np.zeros(g.shape)
        st = self._heat_asm(C.byref(g), dt, _p(off), _p(dg), _p(ab))
        return st, off, dg, ab

    def redblack_sor(self, g, off, rhs, u_guess, omega, tol, max_iter, workers=1):
        u = np.array(u_guess, dtype=np.float64, copy=True)
        it = C.c_int(0)
        res = C.c_double(0.0)
        st = self._sor(C.byref(g), _p(np.ascontiguousarray(off)), _p(np.ascontiguousarray(rhs)),
                       _p(u), omega, tol, max_iter, *self._wk(workers), C.byref(it), C.byref(res))
        return st, u, it.value, res.value

    def heat_smooth(self, g, image, sigma, steps=1, omega=1.85, tol=1e-10, max_iter=10000, workers=1):
        out = np.empty(g.shape)
        st = self._heat(C.byref(g), _p(image), sigma, steps, omega, tol, max_iter,
                        *self._wk(workers), _p(out))
        return st, out

    def local_threshold(self, g, image, rows, lam, background=0.0):
        arr, n = centers_array(rows)
        out = np.empty(g.shape)
        st = self._thr(C.byref(g), _p(image), arr, n, lam, background, _p(out))
        return st, out

    def build_initial(self, g, rows, v=1.0, R=10.0, profile=0):
        arr, n = centers_array(rows)
        out = np.empty(g.shape)
        st = self._init(C.byref(g), arr, n, v, R, profile, _p(out))
        return st, out

    def local_rescale(self, g, u, rows, radius=None):
        """radius None = std::nullopt (each row's own radius); any number is explicit"""
        radius = float("nan") if radius is None else float(radius)
        arr, n = centers_array(rows)
        u = np.array(u, dtype=np.float64, copy=True)
        st = self._resc(C.byref(g), _p(u), arr, n, radius)
        return st, u

    def apply_mirror_ghosts(self, g, f):
        f = np.array(f, dtype=np.float64, copy=True)
        self._mirror(C.byref(g), _p(f))
        return f

    def extract_mask(self, g, u, level=0.5):
        m = np.empty(g.n1 * g.n2 * g.n3 * g.n4, dtype=np.uint8)
        self._mask(C.byref(g), _p(u), level, m.ctypes.data_as(C.POINTER(C.c_ubyte)))
        return m.reshape(g.n4, g.n3, g.n2, g.n1)

    # ---- tracking (reference only; frames (n4, n3, n2, n1), x fastest) ----
    def label_components(self, g, mask):
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        lab = np.empty(mask.shape, dtype=np.int32)
        lpf = np.empty(g.n4, dtype=np.int32)
        st = self._lab(C.byref(g), mask.ctypes.data_as(C.POINTER(C.c_ubyte)),
                       lab.ctypes.data_as(C.POINTER(C.c_int)), lpf.ctypes.data_as(C.POINTER(C.c_int)))
        assert st == 0, st
        return lab, lpf.tolist()

    def distance_centers(self, g, labels, lpf):
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        lpf = np.asarray(lpf, dtype=np.int32)
        cap = int(lpf.sum())
        out = np.zeros((max(cap, 1), 7), dtype=np.int64)
        n = C.c_int(0)
        st = self._dc(C.byref(g), labels.ctypes.data_as(C.POINTER(C.c_int)), lpf.ctypes.data_as(C.POINTER(C.c_int)),
                      out.ctypes.data_as(C.POINTER(C.c_longlong)), cap, C.byref(n))
        assert st == 0, st
        return out[:n.value]

    def backtrack_link(self, g, labels, lpf):
        """chains as lists of (frame, label), the reference's own records"""
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        lpf = np.asarray(lpf, dtype=np.int32)
        cap = int(lpf.sum())
        fl = np.zeros((max(cap, 1), 2), dtype=np.int32)
        cs = np.zeros(cap + 2, dtype=np.int32)
        nc = C.c_int(0)
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))
        st = self._bt(C.byref(g), ip(labels), ip(lpf), ip(fl), ip(cs), C.byref(nc))
        assert st == 0, st
        return [[tuple(x) for x in fl[cs[c]:cs[c + 1]].tolist()] for c in range(nc.value)]

    def track(self, g, u, level=0.5, window=3, radius=5.0):
        """rows (trajectory_id, frame, x, y, z)"""
        cap = 1 << 16
        while True:
            idf = np.zeros((cap, 2), dtype=np.int32)
            xyz = np.zeros((cap, 3))
            n = C.c_int(0)
            st = self._trk(C.byref(g), _p(np.ascontiguousarray(u, dtype=np.float64)), level, window, radius,
                           idf.ctypes.data_as(C.POINTER(C.c_int)), _p(xyz), cap, C.byref(n))
            if st == 0:
                return [(int(a), int(b), float(x), float(y), float(z))
                        for (a, b), (x, y, z) in zip(idf[:n.value].tolist(), xyz[:n.value].tolist())]
            assert n.value > cap, st
            cap = n.value

    def eoc_row(self, n, omega=1.5, tol=1e-8, max_iter=10000, workers=1):
        err = C.c_double(0.0)
        st = self._eoc(n, omega, tol, max_iter, *self._wk(workers), C.byref(err))
        return st, err.value

    def segment(self, g, image, rows, params: SegParams, u0=None, workers=1):
        arr, n = centers_array(rows)
        out = np.empty(g.shape)
        diags = (StepDiag * params.n_steps)()
        extra = []
        times = np.zeros(4)
        sweeps = C.c_longlong(0)
        step_s = np.zeros(params.n_steps)
        if self.w:
            extra = [_p(times), C.byref(sweeps), _p(step_s)]
        st = self._seg(C.byref(g), _p(image), arr, n, C.byref(params), _p(u0), *self._wk(workers),
                       _p(out), diags, *extra)
        d = [dict(iterations=x.iterations, residual=x.residual, tol=x.tol, umin=x.umin,
                  umax=x.umax) for x in diags]
        info = dict(diags=d)
        if self.w:
            info.update(times=times.tolist(), sweeps=sweeps.value, step_seconds=step_s.tolist())
        return st, out, info

    def segment_fixed(self, g, image, rows, params: SegParams, u0=None, workers=1, n_sweeps=50, mode=0):
        """Reference only (ref_shim.cpp ref_segment_fixed): n_steps time steps of exactly
        n_sweeps red-black sweeps each.  mode 0 returns the reference's own iterate (parity
        pin), mode 1 times the throwing redblack_sor call without advancing u (bench)."""
        arr, n = centers_array(rows)
        out = np.empty(g.shape)
        diags = (StepDiag * params.n_steps)()
        times = np.zeros(4)
        step_s = np.zeros(params.n_steps)
        st = self._segfix(C.byref(g), _p(image), arr, n, C.byref(params), _p(u0), int(workers), int(n_sweeps),
                          int(mode), _p(out), diags, _p(times), _p(step_s))
        d = [dict(iterations=x.iterations, residual=x.residual, tol=x.tol, umin=x.umin,
                  umax=x.umax) for x in diags]
        return st, out, dict(diags=d, times=times.tolist(), step_seconds=step_s.tolist())

    def sor_rate(self, g, u0, tau, eps, omega, n_a, n_b, workers):
        """Reference only: wall seconds of redblack_sor calls of n_a and n_b sweeps."""
        secs = np.zeros(2)
        st = self._sorrate(C.byref(g), _p(np.ascontiguousarray(u0)), tau, eps, omega, int(n_a), int(n_b),
                           int(workers), _p(secs))
        return st, secs.tolist()

    # ---- the reference's writers (io.cpp), reference only
    def write_image4d(self, g, u, header, data):
        return self._wimg(C.byref(g), _p(np.ascontiguousarray(u)), header.encode(), data.encode())

    def export_frame_vtk(self, g, u, l, path):
        return self._wvtk(C.byref(g), _p(np.ascontiguousarray(u)), int(l), path.encode())

    def write_trajectories(self, points, path):
        idf = np.ascontiguousarray(np.array([p[:2] for p in points], dtype=np.int32).reshape(-1, 2))
        xyz = np.ascontiguousarray(np.array([p[2:] for p in points], dtype=np.float64).reshape(-1, 3))
        return self._wtrj(len(points), idf.ctypes.data_as(C.POINTER(C.c_int)), _p(xyz), path.encode())

    def export_label_vtks(self, g, u, level, prefix):
        return self._wlab(C.byref(g), _p(np.ascontiguousarray(u)), float(level), prefix.encode())


_oracle = None
_ref = None


def oracle() -> _Lib:
    """The C restatement."""
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _oracle = _Lib(ORACLE_SO, "or_", False)
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> _Lib:
    """The unmodified reference (oracle/_ref)."""
    global _ref
    if _ref is None:
        _ref = _Lib(REF_SO, "ref_", True)
    return _ref
