"""Seeded random segment() cases on the GPU against the oracle restatement, bit for bit:
random extents (odd, 1-wide, wider than a 32-slot segment), anisotropic spacings (powers
of two and not), random solver/edge parameters, u0 given or built, rescale on/off, and
every SOR kernel family (auto, TMA whole rows, TMA 2D-tiled, LDG, resident)."""
import numpy as np
import pytest

import _cases as cs

pytestmark = pytest.mark.gpu

KERNELS = ["auto", "tma", "tma2d", "ldg", "resident"]


def random_case(seed):
    rng = np.random.default_rng(seed)
    dims = (int(rng.choice([1, 3, 7, 16, 33, 70])), int(rng.integers(1, 9)), int(rng.integers(1, 8)),
            int(rng.integers(1, 6)))
    if rng.random() < 0.5:
        h = tuple(float(2.0 ** -int(rng.integers(2, 6))) for _ in range(4))
    else:
        h = tuple(float(rng.uniform(0.05, 0.4)) for _ in range(4))
    img = cs.f32_image(dims, seed, noise=float(rng.uniform(0.0, 0.2)))
    rows = [(int(rng.integers(0, dims[3])), float(rng.uniform(0, dims[0] - 1)), float(rng.uniform(0, dims[1] - 1)),
             float(rng.uniform(0, dims[2] - 1)), float(rng.uniform(1.2, 3.5))) for _ in range(int(rng.integers(1, 5)))]
    kw = dict(tau=float(rng.uniform(0.02, 0.3)), epsilon=float(10 ** rng.uniform(-4, -1)),
              omega=float(rng.uniform(1.1, 1.8)), sor_rel_tol=1e-8, n_steps=int(rng.integers(1, 3)),
              sigma=float(rng.uniform(0.0, 0.3)), K=float(10 ** rng.uniform(0, 3)), delta=float(rng.uniform(0, 1)),
              vartheta=float(rng.uniform(0, 1)), rescale_each_step=int(rng.integers(0, 2)),
              rescale_radius=float(rng.uniform(0, 4)), init_R=float(rng.uniform(2, 6)),
              init_profile=int(rng.integers(0, 2)), lam=float(rng.uniform(0.2, 0.8)))
    u0 = None
    if rng.random() < 0.3:
        u0 = np.zeros(img.shape)
        u0[1:-1, 1:-1, 1:-1, 1:-1] = rng.random(u0[1:-1, 1:-1, 1:-1, 1:-1].shape)
    return dims, h, img, rows, kw, u0


@pytest.mark.parametrize("seed", range(40))
def test_random_segment_cases(gpu, oracle, seed):
    from oracle.oracle_py import Grid, seg_params
    dims, h, img, rows, kw, u0 = random_case(seed)
    okw = {k: v for k, v in kw.items() if k != "lam"}
    okw["lambda_"] = kw["lam"]
    try:
        st, uo, info = oracle.segment(Grid.make(dims, h), img, rows, seg_params(**okw), u0)
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"oracle rejected the case: {e}")
    if st != 0:
        pytest.skip(f"oracle status {st} (case outside the valid parameter space)")
    its_o = [d["iterations"] for d in info["diags"]]
    g = gpu.Grid.make(dims, h)
    for kernel in KERNELS:
        with gpu.Session(g) as s:
            s.set_kernel(kernel)
            s.prepare(img, rows, gpu.seg_params(**kw), u0)
            its = [s.step()["iterations"] for _ in range(kw["n_steps"])]
            u = s.get_u()
        assert its == its_o, (kernel, its, its_o)
        assert np.array_equal(u.view(np.uint64), uo.view(np.uint64)), kernel
