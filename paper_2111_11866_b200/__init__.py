"""B200-native SUBSURF time step (arXiv 2111.11866 hot path).

Python host mirror of the reference's solver API (namespace ``subsurf`` in
/root/reference/proj/include/subsurf/*.hpp) over the C ABI of
``libsubsurf_b200.so`` (include/subsurf_b200.h).  Same function names, the same
argument meaning and the same error taxonomy (errors.hpp:9-39):

=======================  ==============================================
reference                this module
=======================  ==============================================
assemble_step            :func:`assemble_step`      solver.hpp:50-51
assemble_heat_step       :func:`assemble_heat_step` solver.hpp:55
redblack_sor             :func:`redblack_sor`       solver.hpp:69-70
face_coefficients        :func:`face_coefficients`  edge.hpp:95-97
heat_smooth              :func:`heat_smooth`        preprocess.hpp:23
local_threshold          :func:`local_threshold`    preprocess.hpp:36-37
build_initial            :func:`build_initial`      seedinit.hpp:25-26
local_rescale            :func:`local_rescale`      seedinit.hpp:32-33
extract_mask             :func:`extract_mask`       tracking.hpp:55
segment                  :func:`segment`            solver.hpp:91-92
=======================  ==============================================

Fields are numpy fp64 arrays in the reference's ghost-padded layout, shape
``(n4+2, n3+2, n2+2, n1+2)`` (i fastest); per-face arrays add a trailing axis
of 8 (kFaceOffsets order).  Everything runs on the GPU; there is no CPU path:
without the built library or a CUDA device every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SUBSURF_B200_LIB") or os.path.join(_HERE, "libsubsurf_b200.so")

SS_OK, SS_ERR_VALIDATION, SS_ERR_NOCONVERGE, SS_ERR_NONFINITE, SS_ERR_CUDA, SS_ERR_NCCL, SS_ERR_STATE = range(7)


# ----------------------------------------------------------------------------- errors (errors.hpp)
class SubsurfError(RuntimeError):
    """Base of the reference's exception taxonomy."""


class ValidationError(SubsurfError):
    """errors.hpp:15-18"""


class SolverError(SubsurfError):
    """errors.hpp:26-33: carries ``last_residual`` and ``iterations``."""

    def __init__(self, msg: str, last_residual: float = 0.0, iterations: int = 0):
        super().__init__(msg)
        self.last_residual = last_residual
        self.iterations = iterations


class NumericalError(SubsurfError):
    """errors.hpp:36-39"""


class DeviceError(SubsurfError):
    """No usable CUDA device / CUDA failure (the library has no CPU fallback)."""


class StateError(SubsurfError):
    """API misuse."""


# ----------------------------------------------------------------------------- ABI structs
class Grid(C.Structure):
    """GridSpec (grid.hpp:16-46)."""
    _fields_ = [("n1", C.c_int), ("n2", C.c_int), ("n3", C.c_int), ("n4", C.c_int),
                ("h1", C.c_double), ("h2", C.c_double), ("h3", C.c_double), ("h4", C.c_double)]

    @classmethod
    def make(cls, dims, h) -> "Grid":
        hs = (h,) * 4 if np.isscalar(h) else tuple(h)
        return cls(*[int(d) for d in dims], *[float(x) for x in hs])

    @property
    def shape(self):
        return (self.n4 + 2, self.n3 + 2, self.n2 + 2, self.n1 + 2)

    @property
    def interior(self):
        return (slice(1, self.n4 + 1), slice(1, self.n3 + 1), slice(1, self.n2 + 1),
                slice(1, self.n1 + 1))

    def padded_size(self) -> int:
        return int(np.prod(self.shape))


class Center(C.Structure):
    """CenterRow (io.hpp:23-27)."""
    _fields_ = [("frame", C.c_int), ("x", C.c_double), ("y", C.c_double), ("z", C.c_double),
                ("radius", C.c_double)]


class SegParams(C.Structure):
    """SegmentationParams (solver.hpp:77-85), flattened as ss_seg_params."""
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


class CellRecord(C.Structure):  # ss_cell_record (CellRecord, tracking.hpp:36-42)
    _fields_ = [("frame", C.c_int), ("label", C.c_int), ("cx", C.c_int), ("cy", C.c_int), ("cz", C.c_int),
                ("max_distance", C.c_int), ("voxel_count", C.c_longlong)]


class TrackPoint(C.Structure):  # ss_track_point (TrajectoryPoint, io.hpp:36-40)
    _fields_ = [("trajectory_id", C.c_int), ("frame", C.c_int), ("x", C.c_double), ("y", C.c_double),
                ("z", C.c_double)]


class Profile(C.Structure):
    _fields_ = [("red_ms", C.c_double), ("black_ms", C.c_double), ("assemble_ms", C.c_double),
                ("rescale_ms", C.c_double), ("red_n", C.c_longlong), ("black_n", C.c_longlong),
                ("assemble_n", C.c_longlong), ("rescale_n", C.c_longlong),
                ("sweeps", C.c_longlong), ("loop_ms", C.c_double), ("loop_passes", C.c_longlong),
                ("halo_ms", C.c_double), ("halo_exposed_ms", C.c_double), ("halo_n", C.c_longlong)]


def seg_params(**kw) -> SegParams:
    """Defaults of the reference (cli.cpp:73-107, solver.hpp:19-29, preprocess.hpp:10-30,
    edge.hpp:12-18, seedinit.hpp:14-20).  ``lam`` is accepted for ``lambda``."""
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


# ----------------------------------------------------------------------------- library
_lib = None
_D = C.POINTER(C.c_double)
_GP = C.POINTER(Grid)
_CP = C.POINTER(Center)


def library() -> C.CDLL:
    """Load libsubsurf_b200.so (raises ImportError when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)

    def sig(name, args, res=C.c_int):
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res

    sig("ss_last_error", [], C.c_char_p)
    sig("ss_abi_version", [])
    sig("ss_launch_count", [], C.c_ulonglong)
    sig("ss_device_available", [])
    sig("ss_sor_pass_bytes", [_GP], C.c_double)
    sig("ss_assemble_step", [_GP, _D, _D, C.c_double, C.c_double, _D, _D, _D])
    sig("ss_assemble_heat_step", [_GP, C.c_double, _D, _D, _D])
    sig("ss_redblack_sor", [_GP, _D, _D, _D, C.c_double, C.c_double, C.c_int, C.c_int,
                            C.POINTER(C.c_int), _D])
    sig("ss_face_coefficients", [_GP, _D, _D, C.c_double, C.c_double, C.c_double, _D])
    sig("ss_heat_smooth", [_GP, _D, C.c_double, C.c_int, C.c_double, C.c_double, C.c_int, _D])
    sig("ss_local_threshold", [_GP, _D, _CP, C.c_int, C.c_double, C.c_double, _D])
    sig("ss_build_initial", [_GP, _CP, C.c_int, C.c_double, C.c_double, C.c_int, _D])
    sig("ss_local_rescale", [_GP, _D, _CP, C.c_int, C.c_double])
    sig("ss_extract_mask", [_GP, _D, C.c_double, C.POINTER(C.c_uint8)])
    sig("ss_apply_dirichlet", [_GP, _D, C.c_double])
    sig("ss_apply_mirror_ghosts", [_GP, _D])
    sig("ss_interior_minmax", [_GP, _D, _D, _D])
    sig("ss_segment", [_GP, _D, _CP, C.c_int, C.POINTER(SegParams), _D, _D, C.POINTER(StepDiag)])
    _IP = C.POINTER(C.c_int)
    sig("ss_label_components", [_GP, C.POINTER(C.c_uint8), _IP, _IP])
    sig("ss_distance_centers", [_GP, _IP, _IP, C.POINTER(CellRecord), C.c_int, _IP])
    sig("ss_backtrack_link", [_GP, _IP, _IP, C.POINTER(CellRecord), C.c_int, _IP, _IP, _IP])
    sig("ss_track", [_GP, _D, C.c_double, C.c_int, C.c_double, C.POINTER(TrackPoint), C.c_int, _IP])
    sig("ss_session_track", [C.c_void_p, C.c_double, C.c_int, C.c_double, C.POINTER(TrackPoint), C.c_int, _IP])

    sig("ss_session_create", [_GP, C.c_int, C.POINTER(C.c_void_p)])
    sig("ss_session_create_group", [_GP, C.c_int, C.c_int, C.POINTER(C.c_void_p)])
    sig("ss_nccl_unique_id", [C.POINTER(C.c_uint8)])
    sig("ss_session_create_dist", [_GP, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_void_p)])
    sig("ss_session_create_dist_host", [_GP, C.c_int, C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)])
    sig("ss_session_slab", [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)])
    sig("ss_session_destroy", [C.c_void_p])
    sig("ss_session_stream", [C.c_void_p], C.c_void_p)
    sig("ss_session_prepare", [C.c_void_p, _D, _CP, C.c_int, C.POINTER(SegParams), _D])
    sig("ss_session_step", [C.c_void_p, C.POINTER(StepDiag)])
    sig("ss_session_set_u", [C.c_void_p, _D])
    sig("ss_session_get_u", [C.c_void_p, _D])
    sig("ss_session_get_mask", [C.c_void_p, C.c_double, C.POINTER(C.c_uint8)])
    sig("ss_session_fixed_sweeps", [C.c_void_p, C.c_int, _D])
    sig("ss_session_step_fixed", [C.c_void_p, C.c_int, C.POINTER(StepDiag)])
    sig("ss_selftest_rsqrt", [_D])
    sig("ss_session_assemble_export", [C.c_void_p, _D])
    sig("ss_session_step_host", [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(StepDiag)])
    sig("ss_session_step_host_async", [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(StepDiag)])
    sig("ss_session_wait", [C.c_void_p])
    sig("ss_session_set_u_interior", [C.c_void_p, C.c_void_p])
    sig("ss_session_get_u_interior", [C.c_void_p, C.c_void_p])
    sig("ss_session_set_loop_mode", [C.c_void_p, C.c_int])
    sig("ss_session_eoc_row", [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_int, _D,
                               C.POINTER(C.c_longlong)])
    sig("ss_session_set_profiling", [C.c_void_p, C.c_int])
    sig("ss_session_set_kernel", [C.c_void_p, C.c_int])
    sig("ss_session_sor_kernel", [C.c_void_p, C.POINTER(C.c_int)])
    sig("ss_session_profile", [C.c_void_p, C.POINTER(Profile)])
    _lib = L
    return L


def _check(status: int, iterations: int = 0, residual: float = 0.0) -> None:
    if status == SS_OK:
        return
    msg = library().ss_last_error().decode(errors="replace")
    if status == SS_ERR_VALIDATION:
        raise ValidationError(msg)
    if status == SS_ERR_NOCONVERGE:
        raise SolverError(msg, residual, iterations)
    if status == SS_ERR_NONFINITE:
        raise NumericalError(msg)
    if status == SS_ERR_STATE:
        raise StateError(msg)
    raise DeviceError(msg)


def launch_count() -> int:
    """Kernels launched by the library so far (process-wide)."""
    return int(library().ss_launch_count())


def device_available() -> bool:
    return bool(library().ss_device_available())


def sor_pass_bytes(g: Grid) -> float:
    return float(library().ss_sor_pass_bytes(C.byref(g)))


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def _field(g: Grid, a, name: str, per_face: bool = False) -> np.ndarray:
    shape = g.shape + ((8,) if per_face else ())
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.shape != shape:
        raise ValidationError(f"{name}: shape {a.shape} does not match grid {shape}")
    return a


def _centers(rows) -> tuple:
    rows = list(rows)
    arr = (Center * max(1, len(rows)))()
    for n, r in enumerate(rows):
        if isinstance(r, Center):
            arr[n] = r
        else:
            arr[n] = Center(int(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]))
    return arr, len(rows)


# ----------------------------------------------------------------------------- reference API
@dataclass
class StepCoefficients:
    """solver.hpp:36-45 (padded indexing; ghost rows zero)."""
    offdiag: np.ndarray
    diag: np.ndarray
    abar: np.ndarray


@dataclass
class SorResult:
    """solver.hpp:57-61"""
    u: np.ndarray
    iterations: int = 0
    residual: float = 0.0


def assemble_step(u_prev, G, tau: float, epsilon: float, g: Grid) -> StepCoefficients:
    u = _field(g, u_prev, "u_prev")
    Gf = None if G is None else _field(g, G, "G", per_face=True)
    off = np.empty(g.shape + (8,))
    dg = np.empty(g.shape)
    ab = np.empty(g.shape)
    _check(library().ss_assemble_step(C.byref(g), _dp(u), _dp(Gf), tau, epsilon, _dp(off), _dp(dg), _dp(ab)))
    return StepCoefficients(off, dg, ab)


def assemble_heat_step(g: Grid, dt: float) -> StepCoefficients:
    off = np.empty(g.shape + (8,))
    dg = np.empty(g.shape)
    ab = np.empty(g.shape)
    _check(library().ss_assemble_heat_step(C.byref(g), dt, _dp(off), _dp(dg), _dp(ab)))
    return StepCoefficients(off, dg, ab)


def redblack_sor(coeff, rhs, u_guess, omega: float, sor_tol: float, sor_max_iter: int, g: Grid,
                 workers: int = 1) -> SorResult:
    off = _field(g, coeff.offdiag if isinstance(coeff, StepCoefficients) else coeff, "offdiag", True)
    r = _field(g, rhs, "rhs")
    u = np.array(_field(g, u_guess, "u_guess"), copy=True)  # u_guess is taken by value
    it = C.c_int(0)
    res = C.c_double(0.0)
    st = library().ss_redblack_sor(C.byref(g), _dp(off), _dp(r), _dp(u), omega, sor_tol,
                                   sor_max_iter, workers, C.byref(it), C.byref(res))
    _check(st, it.value, res.value)
    return SorResult(u, it.value, res.value)


def face_coefficients(I0s, ITs, K: float, delta: float, vartheta: float, g: Grid) -> np.ndarray:
    a = _field(g, I0s, "smoothed_image")
    b = _field(g, ITs, "smoothed_threshold")
    G = np.empty(g.shape + (8,))
    _check(library().ss_face_coefficients(C.byref(g), _dp(a), _dp(b), K, delta, vartheta, _dp(G)))
    return G


def heat_smooth(image, g: Grid, sigma: float, steps: int = 1, omega: float = 1.85,
                sor_tol: float = 1e-10, sor_max_iter: int = 10000) -> np.ndarray:
    a = _field(g, image, "image")
    out = np.empty(g.shape)
    _check(library().ss_heat_smooth(C.byref(g), _dp(a), sigma, steps, omega, sor_tol, sor_max_iter, _dp(out)))
    return out


def local_threshold(image, centers, g: Grid, lam: float = 0.5, background: float = 0.0) -> np.ndarray:
    a = _field(g, image, "image")
    arr, n = _centers(centers)
    out = np.empty(g.shape)
    _check(library().ss_local_threshold(C.byref(g), _dp(a), arr, n, lam, background, _dp(out)))
    return out


def build_initial(centers, g: Grid, v: float = 1.0, R: float = 10.0, profile: int = 0) -> np.ndarray:
    arr, n = _centers(centers)
    out = np.empty(g.shape)
    _check(library().ss_build_initial(C.byref(g), arr, n, v, R, profile, _dp(out)))
    return out


def local_rescale(u, centers, g: Grid, radius: Optional[float] = None) -> np.ndarray:
    """Returns the rescaled copy (the reference rescales in place)."""
    out = np.array(_field(g, u, "u"), copy=True)
    arr, n = _centers(centers)
    _check(library().ss_local_rescale(C.byref(g), _dp(out), arr, n, float("nan") if radius is None else float(radius)))
    return out


def extract_mask(u, g: Grid, level: float = 0.5) -> np.ndarray:
    a = _field(g, u, "u")
    m = np.empty((g.n4, g.n3, g.n2, g.n1), dtype=np.uint8)
    _check(library().ss_extract_mask(C.byref(g), _dp(a), level, m.ctypes.data_as(C.POINTER(C.c_uint8))))
    return m


# ----------------------------------------------------------------------------- tracking
# frames are (n4, n3, n2, n1) arrays, x fastest (MaskFrames / LabelField, tracking.hpp:14-34)
def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def label_components(mask, g: Grid):
    """tracking.cpp:69-127 -> (labels int32 (n4, n3, n2, n1), labels_per_frame list)"""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    if m.shape != (g.n4, g.n3, g.n2, g.n1):
        raise ValidationError(f"mask shape {m.shape} != {(g.n4, g.n3, g.n2, g.n1)}")
    lab = np.empty(m.shape, dtype=np.int32)
    lpf = np.empty(g.n4, dtype=np.int32)
    _check(library().ss_label_components(C.byref(g), m.ctypes.data_as(C.POINTER(C.c_uint8)), _ip(lab), _ip(lpf)))
    return lab, lpf.tolist()


def distance_centers(labels, labels_per_frame, g: Grid):
    """tracking.cpp:189-215 -> list of CellRecord (frame, label order)"""
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    lpf = np.ascontiguousarray(labels_per_frame, dtype=np.int32)
    n = int(lpf.sum())
    out = (CellRecord * max(n, 1))()
    got = C.c_int(0)
    _check(library().ss_distance_centers(C.byref(g), _ip(lab), _ip(lpf), out, n, C.byref(got)))
    return list(out[:got.value])


def backtrack_link(records, labels, labels_per_frame, g: Grid):
    """tracking.cpp:220-296 -> partial trajectories as lists of record indices"""
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    lpf = np.ascontiguousarray(labels_per_frame, dtype=np.int32)
    n = len(records)
    arr = (CellRecord * max(n, 1))(*records)
    idx = np.zeros(max(n, 1), dtype=np.int32)
    starts = np.zeros(n + 2, dtype=np.int32)
    nc = C.c_int(0)
    _check(library().ss_backtrack_link(C.byref(g), _ip(lab), _ip(lpf), arr, n, _ip(idx), _ip(starts), C.byref(nc)))
    return [idx[starts[c]:starts[c + 1]].tolist() for c in range(nc.value)]


def _points(call):
    cap = 4096
    while True:
        out = (TrackPoint * cap)()
        n = C.c_int(0)
        st = call(out, cap, C.byref(n))
        if st == 0:
            return [(p.trajectory_id, p.frame, p.x, p.y, p.z) for p in out[:n.value]]
        if n.value <= cap:
            _check(st)
        cap = n.value


def track(u, g: Grid, level: float = 0.5, window: int = 3, radius: float = 5.0):
    """track() (tracking.cpp:374-401): rows (trajectory_id, frame, x, y, z) in output order"""
    a = _field(g, u, "u")
    return _points(lambda out, cap, n: library().ss_track(C.byref(g), _dp(a), level, window, radius, out, cap, n))


def write_trajectories(points, path: str) -> None:
    """io.cpp:170-177 format: header + "id,frame,x,y,z" rows (C++ ostream default precision)"""
    with open(path, "w") as f:
        f.write("trajectory_id,frame,x,y,z\n")
        for tid, fr, x, y, z in points:
            f.write(f"{tid},{fr},{x:g},{y:g},{z:g}\n")


def apply_dirichlet(f, g: Grid, value: float) -> np.ndarray:
    """grid.cpp:126-136 (returns a copy)."""
    out = np.array(_field(g, f, "field"), copy=True)
    _check(library().ss_apply_dirichlet(C.byref(g), _dp(out), value))
    return out


def apply_mirror_ghosts(f, g: Grid) -> np.ndarray:
    """grid.cpp:138-156 (returns a copy)."""
    out = np.array(_field(g, f, "field"), copy=True)
    _check(library().ss_apply_mirror_ghosts(C.byref(g), _dp(out)))
    return out


def interior_minmax(f, g: Grid):
    """grid.cpp:158-171"""
    a = _field(g, f, "field")
    lo, hi = C.c_double(0.0), C.c_double(0.0)
    _check(library().ss_interior_minmax(C.byref(g), _dp(a), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def segment(image, centers, params: SegParams, g: Grid, u0=None):
    """solver.cpp:405-441. Returns (u, per-step diagnostics)."""
    a = _field(g, image, "image")
    u0a = None if u0 is None else _field(g, u0, "u0")
    arr, n = _centers(centers)
    out = np.empty(g.shape)
    diags = (StepDiag * params.n_steps)()
    _check(library().ss_segment(C.byref(g), _dp(a), arr, n, C.byref(params), _dp(u0a), _dp(out), diags))
    return out, [dict(iterations=d.iterations, residual=d.residual, tol=d.tol, umin=d.umin,
                      umax=d.umax) for d in diags]


def eoc_row(n: int, omega: float = 1.5, sor_tol: float = 1e-8, sor_max_iter: int = 10000,
            n_slabs: int = 1, device: int = 0):
    """run_levelset_row (eoc.cpp:83-137) on the GPU: returns (L2 error, total SOR sweeps)."""
    g = Grid.make((n,) * 4, 2.5 / n)
    with Session(g, device=device, n_slabs=n_slabs) as s:
        err = C.c_double(0.0)
        sw = C.c_longlong(0)
        _check(library().ss_session_eoc_row(s._h, n, omega, sor_tol, sor_max_iter, C.byref(err), C.byref(sw)))
        return err.value, sw.value


# ----------------------------------------------------------------------------- device session
def _nccl_of_torch_first() -> None:
    """The library dlopens "libnccl.so.2" on first NCCL use and gets whichever copy is
    loaded already.  Import torch first (when installed) so that copy is torch's bundled
    NCCL: were the system library loaded first under the same soname, a later
    `import torch` would bind libtorch_cuda to it and fail on symbols the older NCCL lacks."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    _nccl_of_torch_first()
    buf = (C.c_uint8 * 128)()
    _check(library().ss_nccl_unique_id(buf))
    return bytes(buf)


class Session:
    """Device-resident segment() state (the performance boundary).

    ``prepare`` runs segment()'s preamble on the GPU; ``step`` one time step;
    u stays in HBM between steps unless ``get_u`` / ``set_u`` move it.

    ``n_slabs > 1`` splits the grid along l into slabs on the same device (the
    multi-GPU decomposition with device-copy halo exchange); ``dist=(rank,
    world, uid)`` makes this process's slab of an NCCL job, whose host arrays
    are the rank's padded slab (see :mod:`paper_2111_11866_b200.dist`).
    """

    def __init__(self, g: Grid, device: int = 0, n_slabs: int = 1, dist=None):
        self.g = g
        h = C.c_void_p()
        if dist is not None:
            rank, world, uid = dist
            if hasattr(uid, "as_abi"):  # dist.HostComm: exchanges staged through the host
                self._comm = uid
                _check(library().ss_session_create_dist_host(C.byref(g), rank, world, uid.as_abi(), device,
                                                             C.byref(h)))
            else:
                _nccl_of_torch_first()
                ub = (C.c_uint8 * 128).from_buffer_copy(uid)
                _check(library().ss_session_create_dist(C.byref(g), rank, world, ub, device, C.byref(h)))
        else:
            _check(library().ss_session_create_group(C.byref(g), n_slabs, device, C.byref(h)))
        self._h = h
        lb, lc, w = C.c_int(0), C.c_int(0), C.c_int(0)
        _check(library().ss_session_slab(h, C.byref(lb), C.byref(lc), C.byref(w)))
        self.l_begin, self.l_count, self.world = lb.value, lc.value, w.value
        self.distributed = dist is not None
        # host arrays: whole padded grid, or the rank's padded slab
        self.host_shape = (self.l_count + 2,) + g.shape[1:] if self.distributed else g.shape

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            library().ss_session_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def stream(self) -> int:
        return int(library().ss_session_stream(self._h) or 0)

    def _host(self, a, name):
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.shape != self.host_shape:
            raise ValidationError(f"{name}: shape {a.shape} does not match {self.host_shape}")
        return a

    def prepare(self, image, centers, params: SegParams, u0=None):
        a = self._host(image, "image")
        u0a = None if u0 is None else self._host(u0, "u0")
        arr, n = _centers(centers)
        self.params = params
        _check(library().ss_session_prepare(self._h, _dp(a), arr, n, C.byref(params), _dp(u0a)))

    def step(self) -> dict:
        d = StepDiag()
        st = library().ss_session_step(self._h, C.byref(d))
        _check(st, d.iterations, d.residual)  # SolverError carries iterations / last residual
        return dict(iterations=d.iterations, residual=d.residual, tol=d.tol, umin=d.umin, umax=d.umax)

    def step_nodiag(self) -> None:
        _check(library().ss_session_step(self._h, None))

    def step_fixed(self, n_sweeps: int, diag: bool = True):
        """One BASELINE config-4 time step: assemble, exactly n_sweeps sweeps, rescale."""
        d = StepDiag()
        _check(library().ss_session_step_fixed(self._h, n_sweeps, C.byref(d) if diag else None))
        return dict(iterations=d.iterations, residual=d.residual, tol=d.tol, umin=d.umin, umax=d.umax) if diag else None

    @property
    def interior_shape(self):
        g = self.g
        return (self.l_count if self.distributed else g.n4, g.n3, g.n2, g.n1)

    def step_host(self, u_in=None, u_out=None, n_sweeps: int = 0, diag: bool = True):
        """One time step with the host's copy of u as compact interiors (interior_shape):
        u_in (or None) -> u^{n-1}, then step (n_sweeps = 0) or step_fixed(n_sweeps), and u^n
        -> u_out (a new array when None and diag is requested).  numpy arrays or raw
        pointers (int, e.g. a pinned torch tensor's data_ptr())."""
        def ptr(a, name, write):
            if a is None:
                return None
            if isinstance(a, int):
                return C.c_void_p(a)
            if a.shape != self.interior_shape or a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValidationError(f"{name}: expected a C-contiguous float64 array of shape {self.interior_shape}")
            return C.c_void_p(a.ctypes.data)
        d = StepDiag()
        st = library().ss_session_step_host(self._h, ptr(u_in, "u_in", False), ptr(u_out, "u_out", True), n_sweeps,
                                            C.byref(d) if diag else None)
        _check(st, d.iterations, d.residual)
        return dict(iterations=d.iterations, residual=d.residual, tol=d.tol, umin=d.umin, umax=d.umax) if diag else None

    def step_host_async(self, u_in=None, u_out=None, n_sweeps: int = 0, diag: bool = True):
        """step_host with the result's download left in flight (one slab per process, page-locked
        buffers given as pointers; otherwise step_host): u_out is complete after wait().  When
        the next call's u_in is this call's u_out, each upload chunk waits on the device for its
        download chunk -- the D2H of step n and the H2D of step n + 1 overlap."""
        d = StepDiag()
        p_in = None if u_in is None else C.c_void_p(int(u_in))
        p_out = None if u_out is None else C.c_void_p(int(u_out))
        st = library().ss_session_step_host_async(self._h, p_in, p_out, n_sweeps, C.byref(d) if diag else None)
        _check(st, d.iterations, d.residual)
        return dict(iterations=d.iterations, residual=d.residual, tol=d.tol, umin=d.umin, umax=d.umax) if diag else None

    def wait(self) -> None:
        """Every transfer of step_host_async done (and the session's stream idle)."""
        _check(library().ss_session_wait(self._h))

    def assemble_export(self) -> np.ndarray:
        """The off-diagonals the next step would assemble at the session's u (the device
        path's tile kernel), padded (n4+2, n3+2, n2+2, n1+2, 8) fp64."""
        out = np.empty(self.g.shape + (8,))
        _check(library().ss_session_assemble_export(self._h, _dp(out)))
        return out

    def set_u_interior(self, u) -> None:
        a = np.ascontiguousarray(u, dtype=np.float64).reshape(self.interior_shape)
        _check(library().ss_session_set_u_interior(self._h, C.c_void_p(a.ctypes.data)))

    def get_u_interior(self) -> np.ndarray:
        out = np.empty(self.interior_shape)
        _check(library().ss_session_get_u_interior(self._h, C.c_void_p(out.ctypes.data)))
        return out

    def set_u(self, u) -> None:
        a = self._host(u, "u")
        _check(library().ss_session_set_u(self._h, _dp(a)))

    def set_u_ptr(self, ptr: int) -> None:
        _check(library().ss_session_set_u(self._h, C.cast(C.c_void_p(ptr), _D)))

    def get_u(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        out = np.zeros(self.host_shape) if out is None else out
        _check(library().ss_session_get_u(self._h, _dp(out)))
        return out

    def get_u_ptr(self, ptr: int) -> None:
        _check(library().ss_session_get_u(self._h, C.cast(C.c_void_p(ptr), _D)))

    def get_mask(self, level: float = 0.5) -> np.ndarray:
        g = self.g
        m = np.empty((self.l_count if self.distributed else g.n4, g.n3, g.n2, g.n1), dtype=np.uint8)
        _check(library().ss_session_get_mask(self._h, level, m.ctypes.data_as(C.POINTER(C.c_uint8))))
        return m

    def track(self, level: float = 0.5, window: int = 3, radius: float = 5.0):
        """track() on the device-resident u (single-process sessions)"""
        return _points(lambda out, cap, n: library().ss_session_track(self._h, level, window, radius, out, cap, n))

    def fixed_sweeps(self, n: int) -> float:
        r = C.c_double(0.0)
        _check(library().ss_session_fixed_sweeps(self._h, n, C.byref(r)))
        return r.value

    def set_loop_mode(self, mode: int) -> None:
        _check(library().ss_session_set_loop_mode(self._h, mode))

    def set_kernel(self, kernel: str) -> None:
        """'auto' (default): 'resident' when the solve's working set fits L2, else 'tma';
        'tma': TMA-fed two-pass; 'ldg': plain load two-pass; 'resident': the whole solve
        in one cooperative launch (LDG tiles, grid barriers); 'wave': two-iteration TMA
        wavefront through L2 (experimental, measured slower)."""
        _check(library().ss_session_set_kernel(
            self._h, {"ldg": 0, "tma": 1, "wave": 2, "resident": 3, "auto": 4, "tma2d": 5,
                       "kwave": 7}[kernel]))

    def sor_kernel(self) -> str:
        """The SOR kernel the last segmentation solve ran (after the support checks)."""
        k = C.c_int(-1)
        _check(library().ss_session_sor_kernel(self._h, C.byref(k)))
        return {-1: "none", 0: "ldg", 1: "tma", 2: "wave", 3: "resident", 5: "tma2d", 7: "kwave"}[k.value]

    def set_profiling(self, on: bool) -> None:
        _check(library().ss_session_set_profiling(self._h, 1 if on else 0))

    def profile(self) -> dict:
        p = Profile()
        _check(library().ss_session_profile(self._h, C.byref(p)))
        return {k: getattr(p, k) for k, _ in Profile._fields_}
