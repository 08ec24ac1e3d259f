"""CPU: the host half of tracking (include/subsurf_b200/track_link.hpp: prolong_and_merge,
tracking.cpp:312-372) against the unmodified reference on random partial trajectories --
gaps 1..window+1, tangents from 1- and 2-record partials, ties in gap and distance."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tl(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("tl") / "libtl.so")
    subprocess.run(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "track_link_cabi.cpp"), "-o", so], check=True)
    return C.CDLL(so)


def random_partials(rng, n):
    parts = []
    for _ in range(n):
        f0 = int(rng.integers(0, 12))
        length = int(rng.integers(1, 5))
        p = rng.integers(0, 20, size=3)
        v = rng.integers(-2, 3, size=3)
        parts.append([(f0 + t, *(p + t * v + rng.integers(-1, 2, size=3)).tolist()) for t in range(length)])
    return parts


def run(lib, fn, parts, window, radius):
    sizes = np.array([len(p) for p in parts], dtype=np.int32)
    fxyz = np.array([r for p in parts for r in p], dtype=np.int32).reshape(-1)
    out = np.zeros_like(fxyz)
    osz = np.zeros(len(parts) + 1, dtype=np.int32)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))
    if fn == "tl_merge":
        f = lib.tl_merge
        f.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int, C.c_double, C.POINTER(C.c_int),
                      C.POINTER(C.c_int)]
        n = f(len(parts), ip(sizes), ip(fxyz), window, radius, ip(out), ip(osz))
    else:
        f = lib.ref_prolong_and_merge
        f.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int, C.c_double, C.POINTER(C.c_int),
                      C.POINTER(C.c_int), C.POINTER(C.c_int)]
        nn = C.c_int(0)
        assert f(len(parts), ip(sizes), ip(fxyz), window, radius, ip(out), ip(osz), C.byref(nn)) == 0
        n = nn.value
    res, q = [], 0
    for t in range(n):
        res.append([tuple(out[4 * (q + r): 4 * (q + r) + 4]) for r in range(osz[t])])
        q += osz[t]
    return res


@pytest.mark.parametrize("seed", range(8))
def test_merge_matches_reference(tl, ref, seed):
    rng = np.random.default_rng(seed)
    parts = random_partials(rng, int(rng.integers(2, 40)))
    for window, radius in ((3, 5.0), (1, 2.0), (4, 8.5), (2, 0.0)):
        assert run(tl, "tl_merge", parts, window, radius) == run(ref.lib, "ref", parts, window, radius)
