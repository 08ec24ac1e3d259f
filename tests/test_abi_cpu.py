"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, validates parameters before touching the device, and has no
CPU fallback (compute entry points fail with SS_ERR_CUDA without a GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "subsurf_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SS_API\s+[\w\s\*]+?\b(ss_\w+)\s*\(", text)))


def test_header_declares_the_reference_entry_points():
    names = declared_symbols()
    for n in ["ss_assemble_step", "ss_assemble_heat_step", "ss_redblack_sor", "ss_face_coefficients",
              "ss_heat_smooth", "ss_local_threshold", "ss_build_initial", "ss_local_rescale",
              "ss_extract_mask", "ss_segment", "ss_session_create", "ss_session_step",
              "ss_label_components", "ss_distance_centers", "ss_backtrack_link", "ss_track", "ss_session_track",
              "ss_session_step_fixed", "ss_session_step_host", "ss_session_step_host_async", "ss_session_wait"]:
        assert n in names


def test_abi_version(ss):
    """ABI 6: ss_session_step_host_async / ss_session_wait."""
    assert ss.library().ss_abi_version() == 6


def test_library_exports_every_declared_symbol(ss):
    lib = ss.library()
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing


def test_no_cpu_fallback(ss):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except ImportError:
        pass
    assert ss.device_available() is False
    g = ss.Grid.make((4, 4, 4, 4), 0.25)
    u = np.zeros(g.shape)
    with pytest.raises(ss.DeviceError, match="no CPU fallback"):
        ss.assemble_step(u, None, 0.1, 1e-3, g)
    with pytest.raises(ss.DeviceError):
        ss.Session(g)


def test_validation_precedes_device(ss):
    g = ss.Grid.make((4, 4, 4, 4), 0.25)
    u = np.zeros(g.shape)
    with pytest.raises(ss.ValidationError, match="epsilon"):
        ss.assemble_step(u, None, 0.1, 0.0, g)
    with pytest.raises(ss.ValidationError, match="omega"):
        ss.redblack_sor(np.zeros(g.shape + (8,)), u, u, 2.5, 1e-8, 10, g)
    with pytest.raises(ss.ValidationError, match="frame"):
        ss.local_threshold(u, [(7, 1, 1, 1, 1.0)], g)
    with pytest.raises(ss.ValidationError, match="radius"):
        ss.local_rescale(u, [(0, 1, 1, 1, 0.0)], g)
    with pytest.raises(ss.ValidationError, match="sigma"):
        ss.heat_smooth(u, g, -1.0)
    with pytest.raises(ss.ValidationError, match="spacings"):
        ss.assemble_step(u, None, 0.1, 1e-3, ss.Grid.make((4, 4, 4, 4), 0.0))
    with pytest.raises(ss.ValidationError, match="shape"):
        ss.assemble_step(np.zeros((3, 3)), None, 0.1, 1e-3, g)


def test_pass_bytes():
    import paper_2111_11866_b200 as ss
    g = ss.Grid.make((64, 64, 64, 64), 1 / 64)
    # 56 B per doxel per sweep, half per colour pass
    assert ss.sor_pass_bytes(g) == 0.5 * 64 ** 4 * 56


def test_tracking_validation_and_no_fallback(ss):
    """tracking entry points: shape checks before the device; no CPU fallback without one"""
    g = ss.Grid.make((4, 3, 2, 2), 1.0)
    with pytest.raises(ss.ValidationError, match="mask shape"):
        ss.label_components(np.zeros((2, 2, 3, 5), np.uint8), g)
    if ss.device_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(ss.DeviceError):
        ss.label_components(np.zeros((2, 2, 3, 4), np.uint8), g)
    with pytest.raises(ss.DeviceError):
        ss.track(np.zeros(g.shape), g)
