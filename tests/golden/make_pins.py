"""Full-size parity pins of the BASELINE configs, from the UNMODIFIED reference.

Runs the reference (oracle/_ref, compiled in place from /root/reference/proj/src)
through its public calls on the seeded synthetic workloads of bench.py
(workloads.py) and records, per config, what the GPU suite must reproduce:

* sha256 of the inputs (f32-valued image, u0, centres table) -- the GPU box
  regenerates them with the same seeded generators; a mismatch means the host
  produced different inputs and the pin cannot be checked there;
* per time step: SOR iterations, the stopping residual, the tolerance, min/max of u;
* sha256 of the final u's bits and the 0.5-superlevel mask voxel count.

  config0  32^4, all 10 steps of segment() (rel. tol 1e-8 harness loop)
  config1  64^4, all 20 steps
  config2  256x256x64x32, all 30 steps
  config3s 512x512x128x4 (config 3's first 4 frames as a grid), steps 1-5
  config4  256x256x128x16 (N = 1), 10 steps of exactly 50 sweeps each: the reference
           throws SolverError at max_iter; ref_segment_fixed recovers the reference's
           own iterate by re-running with sor_tol = the thrown residual (oracle/ref_shim.cpp)

    python tests/golden/make_pins.py [config0 config1 ...]

Writes tests/golden/pins.json (merged with what is already there; PINS_OUT writes
elsewhere, PINS_STEPS_<config> pins a shorter run).  On 8 host cores config 2's 30 steps
take ~86 min, config 1 6 min, config 4 8 min, config 3's frames 10 min.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle_py as op  # noqa: E402
import workloads  # noqa: E402

OUT = os.environ.get("PINS_OUT", os.path.join(HERE, "pins.json"))  # PINS_OUT: write elsewhere, merge later


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def input_hashes(wl) -> dict:
    return {"image": sha(wl.image), "u0": sha(wl.u0), "rows": sha(np.asarray(wl.rows, dtype=np.float64))}


PLAN = {  # config -> (workload builder, steps, fixed sweeps or None)
    "config0": (lambda: workloads.config0(), 10, None),
    "config1": (lambda: workloads.config1(), 20, None),
    "config2": (lambda: workloads.config2(), 30, None),
    "config4": (lambda: workloads.config4(1), 10, 50),
    "config3s": (lambda: workloads.config3_slab(4), 5, None),  # config 3's 512x512x128 frames
}


def run(name: str) -> dict:
    build, steps, fixed = PLAN[name]
    steps = int(os.environ.get("PINS_STEPS_" + name, steps))  # a shorter pin of the same run
    wl = build()
    R = op.ref()
    g = op.Grid.make(wl.dims, wl.h)
    workers = min(R.lib.ref_hardware_threads(), wl.dims[3])
    p = op.seg_params(**{**wl.params, "n_steps": steps})
    t0 = time.time()
    if fixed:
        st, u, info = R.segment_fixed(g, wl.image, wl.rows, p, wl.u0, workers, fixed, 0)
    else:
        st, u, info = R.segment(g, wl.image, wl.rows, p, wl.u0, workers)
    assert st == 0, (name, st, R.lib.ref_last_error())
    mask = R.extract_mask(g, u, 0.5)
    return {
        "workload": wl.name, "dims": list(wl.dims), "h": wl.h, "steps": steps, "fixed_sweeps": fixed,
        "inputs": input_hashes(wl),
        "iterations": [d["iterations"] for d in info["diags"]],
        "residual": [d["residual"] for d in info["diags"]],
        "tol": [d["tol"] for d in info["diags"]],
        "umin": [d["umin"] for d in info["diags"]],
        "umax": [d["umax"] for d in info["diags"]],
        "u_sha256": sha(u),
        "mask_voxels": int(mask.sum()),
        "reference": f"oracle/_ref (unmodified /root/reference/proj), {workers} workers, "
                     f"{time.time() - t0:.0f} s on the build container",
    }


def main(names):
    names = [n for n in names if n in PLAN]
    pins = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        t = time.time()
        pins[name] = run(name)
        print(name, pins[name]["iterations"], pins[name]["u_sha256"][:16], f"{time.time() - t:.0f} s", flush=True)
        json.dump(pins, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or list(PLAN))
