"""EOC verification rows (eoc.cpp:83-137) on one B200:
L2 error, total SOR sweeps, wall time and the kernel-time split per row."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C
import paper_2111_11866_b200 as ss

rows = [int(x) for x in (sys.argv[1:] or ["80", "160"])]
out = []
for n in rows:
    g = ss.Grid.make((n,) * 4, 2.5 / n)
    t0 = time.perf_counter()
    with ss.Session(g) as s:
        t1 = time.perf_counter()
        err, sw = C.c_double(0.0), C.c_longlong(0)
        s.profile()
        ss._check(ss.library().ss_session_eoc_row(s._h, n, 1.5, 1e-8, 10000, C.byref(err), C.byref(sw)))
        t2 = time.perf_counter()
        pr = s.profile()
    out.append({"n": n, "l2_error": err.value, "sweeps": sw.value, "wall_s": t2 - t1, "session_create_s": t1 - t0,
                "us_per_sweep": 1e6 * (t2 - t1) / max(1, sw.value)})
    print(json.dumps(out[-1]), flush=True)
