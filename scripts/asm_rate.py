"""Device time of the coefficient assembly (assemble_kernel, both colours) per time step on
a config's grid, from the session's profiling events: asm_rate.py [config] -> JSON line."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2111_11866_b200 as ss
import workloads
cfg = sys.argv[1] if len(sys.argv) > 1 else "config1"
wl = workloads.CONFIGS[cfg]()
g = ss.Grid.make(wl.dims, wl.h)
s = ss.Session(g)
s.prepare(wl.image, wl.rows, ss.seg_params(**{**wl.params, "n_steps": 6}), wl.u0)
s.step()
s.set_profiling(True)
s.profile()
for _ in range(4):
    s.step()
p = s.profile()
print(json.dumps(dict(config=cfg, lib=os.environ.get("SUBSURF_B200_LIB"),
                      assemble_ms_per_step=p["assemble_ms"] / 4, assemble_launches=p["assemble_n"],
                      rescale_ms_per_step=p["rescale_ms"] / 4)))
