"""The EOC verification harness on the GPU (eoc.cpp:83-137):
Table 1 rows against the reference's values and the paper's."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# paper Table 1; the oracle (= reference) values for n <= 40
PAPER = {10: 1.680403e-2, 20: 4.653133e-3, 40: 1.208771e-3, 80: 3.029600e-4}
ORACLE = {10: 1.684177e-2, 20: 4.668374e-3, 40: 1.213313e-3}


def test_eoc_rows_10_20_match_reference(gpu):
    d = dict(np.load(os.path.join(GOLD, "eoc.npz")))
    e10, _ = gpu.eoc_row(10)
    e20, _ = gpu.eoc_row(20)
    assert e10 == pytest.approx(float(d["e10"]), rel=1e-12)
    assert e20 == pytest.approx(float(d["e20"]), rel=1e-12)


def test_eoc_slabs_match(gpu):
    e1, s1 = gpu.eoc_row(20)
    e4, s4 = gpu.eoc_row(20, n_slabs=4)
    assert s1 == s4 and e1 == pytest.approx(e4, rel=1e-13)


def test_eoc_rows_40_80_table1(gpu):
    """Acceptance criterion 1: errors within 5% of Table 1, EOC trend ~2.
    n = 80 is the paper's 41681 s serial MPI run."""
    e20, _ = gpu.eoc_row(20)
    e40, _ = gpu.eoc_row(40)
    e80, sweeps = gpu.eoc_row(80)
    assert e40 == pytest.approx(ORACLE[40], rel=2e-6)
    for n, e in ((40, e40), (80, e80)):
        assert abs(e - PAPER[n]) / PAPER[n] < 0.05
    assert abs(np.log2(e20 / e40) - 1.944661) < 0.1
    assert abs(np.log2(e40 / e80) - 1.996342) < 0.1
