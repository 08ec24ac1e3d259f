"""bench.py -- SOR voxel-updates/s of the 4D SUBSURF time step on B200.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config config4]

Default workload: BASELINE config 4 -- 256x256x128 x (16 N) frames, weak scaling
along t (one 16-frame slab per GPU; N = 1 is the largest single-GPU config, 134 M
doxels), config-2 data and solver settings, exactly 50 red-black sweeps per time
step.  A *step* = one time step of segment() with that fixed sweep count
(solver.cpp:428-438): assemble_step + 50 sweeps + local_rescale.  --config
config0/1/2 run segment() steps to relative residual 1e-8 instead; config3
(512x512x128x64, strong, N >= 2) likewise.

value = interior doxels x completed red+black sweeps / device time of the K
timed steps (all ranks: max over ranks of the device time), inputs resident in
HBM.  e2e = the same metric through the public session API with the step's input
u copied H2D from pinned host memory and the result u copied D2H inside the timed
region.

--impl reference times the UNMODIFIED reference CPU solver (oracle/_ref, built
from /root/reference/proj/src) through its own public calls on the same workload
(rank 0 only under torchrun), with the same `config` dict.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SOR voxel-updates/s (4D grid, red+black sweep = 1 update/doxel)"
UNIT = "voxel-updates/s"
SURVEY_BYTES_PER_SWEEP = 56.0  # 8 fp32 coeff + rhs + u read + u write
FIXED_SWEEPS = 50              # BASELINE config 4


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        # started (and its first sample read) BEFORE the timed region: nvidia-smi's start-up
        # (NVML init) stalls driver calls for milliseconds and must not land inside it
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.pre = list(self.lines)  # samples before the region: used only if none fall inside
        self.lines = []
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        lines = self.lines or getattr(self, "pre", [])
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            try:
                pw.append(float(parts[7]))
            except ValueError:
                pass
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w": statistics.median(pw) if pw else None}


def workload_config(wl, config: str, world: int) -> dict:
    """The `config` dict of the JSON line -- identical in both arms (same workload)."""
    fixed = wl.notes.get("fixed_sweeps")
    big = wl.n_interior // world * 200 > 1e9
    return {"workload": wl.name, "config": config, "dims": list(wl.dims), "omega": wl.params["omega"],
            "sor": f"fixed {fixed} sweeps/step (no stopping test)" if fixed else "to relative residual 1e-8",
            "l2": "inputs larger than L2 (no flush): state + coefficients + G ~ "
                  f"{wl.n_interior // world * 200 / 1e9:.1f} GB per GPU vs 0.126 GB L2" if big
                  else "working set partly L2-resident (small config)"}


def make_workload(workloads, ssd, config, rank, world):
    """config0: 32^4 (1 GPU); config1: 64^4, weak-scaled along t for N > 1 (one 64^4
    replica per GPU); config2: 256x256x64x32 (strong scaling over N); config3:
    512x512x128x64 (strong, N >= 2); config4: 256x256x128x(16 N) weak, fixed 50 sweeps."""
    if config == "config0":
        if world > 1:
            raise SystemExit("config0 is a single-GPU config")
        return workloads.config0()
    if config == "config1":
        if world == 1:
            return workloads.config1()
        lb, cnt = ssd.partition(64 * world, world)[rank]
        return workloads.config1(replicas=world, planes=(lb - 1, lb + cnt))
    if config == "config3" and world < 2:
        # 2.1e9 doxels x ~130 B of device state = 280 GB: more than one B200 (BASELINE: 2/4/8 GPUs)
        raise SystemExit("config3 needs >= 2 GPUs (280 GB of device state)")
    if config == "tiny":  # bench-path tests only (6 frames per rank)
        lb, cnt = ssd.partition(6 * world, world)[rank]
        return workloads.tiny(world, planes=(lb - 1, lb + cnt) if world > 1 else None)
    n4 = {"config2": 32, "config3": 64, "config4": 16 * world}[config]
    lb, cnt = ssd.partition(n4, world)[rank]
    planes = (lb - 1, lb + cnt) if world > 1 else None
    if config == "config4":
        return workloads.config4(gpus=world, planes=planes)
    return workloads.CONFIGS[config](planes=planes)


def cpu_baseline_sample(wl):
    """The reference's own redblack_sor (oracle/_ref) on the workload's full grid, steady
    state: the system assemble_step(u0, G == 1), then two calls of 2 and 22 sweeps timed on
    the host's threads (the reference parallelises over l only: min(threads, n4) workers);
    the difference of the two wall times / 20 is the per-sweep time without the per-call
    scatter, coefficient packing and thread start-up."""
    from oracle import oracle_py as op
    if not op.ref_available():
        return None
    R = op.ref()
    g = op.Grid.make(wl.dims, wl.h)
    workers = min(R.lib.ref_hardware_threads(), wl.dims[3])
    na, nb = 2, 22
    t0 = time.perf_counter()
    st, (sa, sb) = R.sor_rate(g, wl.u0, wl.params["tau"], wl.params["epsilon"], wl.params["omega"], na, nb, workers)
    if st != 0:
        return {"error": R.lib.ref_last_error().decode() if isinstance(R.lib.ref_last_error(), bytes) else "sor_rate failed"}
    per_sweep = (sb - sa) / (nb - na)
    return {"value": wl.n_interior / per_sweep, "unit": UNIT, "cores": workers, "kind": "reference",
            "sample": f"redblack_sor of the unmodified reference (oracle/_ref) on the full {tuple(wl.dims)} grid, "
                      f"{workers} std::thread workers: calls of {na} and {nb} sweeps ({sa:.2f} s, {sb:.2f} s), "
                      f"per-sweep time = difference / {nb - na} = {per_sweep * 1e3:.1f} ms "
                      f"(system assembled at u0 with G == 1; {time.perf_counter() - t0:.1f} s in all)"}


def run_reference(args, config):
    """The unmodified reference (oracle/_ref) through its public calls on the same
    workload as our arm -- at N > 1 on one GPU's share of the weak-scaled grid (the host's
    cores do not grow with N; the metric is a rate).  Per step: config 4 = assemble_step +
    redblack_sor(max_iter 50, caught SolverError: the reference has no fixed-sweep mode and
    drops the iterate) + local_rescale; configs 0-2 = segment() time steps to rel. 1e-8.
    Bounded: one untimed warm-up step, then min(K, cap) timed steps."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import workloads
    from oracle import oracle_py as op
    if config == "config3":
        print(json.dumps({"impl": "reference", "unavailable": "config3 needs ~530 GB of host RAM for the "
                          "reference (234 B per padded doxel)"}))
        return 0
    if not op.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return 0
    from paper_2111_11866_b200 import dist as ssd
    wl = make_workload(workloads, ssd, config, 0, 1)
    # the config dict names the N-GPU workload (rank 0's slab carries its global dims and
    # name); the timed sample is the N = 1 workload, one GPU's share
    cfg_wl = wl if world == 1 else make_workload(workloads, ssd, config, 0, world)
    R = op.ref()
    g = op.Grid.make(wl.dims, wl.h)
    workers = min(R.lib.ref_hardware_threads(), wl.dims[3])
    cap = {"config0": 50, "config1": 20, "config2": 2, "config4": 4}[config]
    timed = max(1, min(args.steps, cap))
    n = 1 + timed
    fixed = wl.notes.get("fixed_sweeps")
    p = op.seg_params(**{**wl.params, "n_steps": n})
    t0 = time.perf_counter()
    if fixed:
        st, u, info = R.segment_fixed(g, wl.image, wl.rows, p, wl.u0, workers, fixed, 1)
    else:
        st, u, info = R.segment(g, wl.image, wl.rows, p, wl.u0, workers)
    wall = time.perf_counter() - t0
    if st != 0:
        print(json.dumps({"impl": "reference", "unavailable": f"reference run failed: {R.lib.ref_last_error()}"}))
        return 0
    its = [d["iterations"] for d in info["diags"]][1:]
    secs = info["step_seconds"][1:]
    value = wl.n_interior * sum(its) / sum(secs)
    what = (f"assemble_step + redblack_sor({fixed} sweeps, SolverError caught) + local_rescale" if fixed
            else "segment() time steps (assemble_step + redblack_sor to rel. 1e-8 + local_rescale)")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": timed, "warmup": 1, "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True,
        "scaling": "strong" if config in ("config2", "config3") else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": workload_config(cfg_wl, config, world),
        "sor_iterations": its,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "reference",
                         "sample": f"{timed} timed {what} on {tuple(wl.dims)} after 1 untimed step "
                                   f"(setup: threshold, heat_smooth x2, face_coefficients {info['times'][0]:.1f} s untimed; "
                                   f"wall {wall:.1f} s; steps capped at {cap} to bound the run)"
                                   + (f"; at N = {world} one GPU's {tuple(wl.dims)} share of the grid" if world > 1 else "")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config4", choices=["config0", "config1", "config2", "config3", "config4", "tiny"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--loop-mode", type=int, default=1)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    wd = float(os.environ.get("SUBSURF_BENCH_WATCHDOG", 0) or 0)
    if wd > 0:  # a stuck rank dumps every thread's stack and exits instead of idling on the GPU
        import faulthandler
        faulthandler.dump_traceback_later(wd, exit=True)

    if args.impl == "reference":
        return run_reference(args, args.config)

    import workloads
    import torch
    import paper_2111_11866_b200 as ss
    from paper_2111_11866_b200 import dist as ssd

    rank, world, local = env_rank()
    # SUBSURF_DIST_TRANSPORT=host: the ranks exchange through the host (gloo + dist.HostComm),
    # so several ranks may share one GPU -- a functional test of this multi-rank path where
    # only one GPU exists, never a scaling measurement
    host_tr = os.environ.get("SUBSURF_DIST_TRANSPORT") == "host"
    local = local % max(1, torch.cuda.device_count()) if host_tr else local
    torch.cuda.set_device(local)
    uid = None
    force_dist = os.environ.get("SUBSURF_FORCE_DIST") == "1"  # exercise the NCCL path at N=1
    dist_init = world > 1 or force_dist
    if dist_init:
        import torch.distributed as tdist
        if host_tr:
            import datetime
            # a rank that never joins fails the launch within minutes instead of gloo's 30
            tdist.init_process_group("gloo", timeout=datetime.timedelta(seconds=180))
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # each rank builds only its slab (owned planes + one halo/ghost plane per side)
        wl = make_workload(workloads, ssd, args.config, rank, world)
        uid = ssd.HostComm() if host_tr else ssd.broadcast_uid(ss.nccl_unique_id() if rank == 0 else None)
    else:
        wl = make_workload(workloads, ssd, args.config, 0, 1)
    fixed = wl.notes.get("fixed_sweeps")
    scaling = "strong" if args.config in ("config2", "config3") else "weak"

    g = ss.Grid.make(wl.dims, wl.h)
    p = ss.seg_params(**{**wl.params, "n_steps": args.warmup + args.steps})
    sess = ss.Session(g, device=local, dist=(rank, world, uid) if (world > 1 or force_dist) else None)
    sess.set_loop_mode(args.loop_mode)
    stream = torch.cuda.ExternalStream(sess.stream, device=torch.device("cuda", local))

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def do_step():
        if fixed:
            sess.step_fixed(fixed, diag=False)  # config 4: assemble + exactly 50 sweeps + rescale
        else:
            sess.step_nodiag()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if host_tr else "cuda")
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return [float(v) for v in t.tolist()]

    # ---------------- value: device-resident steps
    sess.prepare(wl.image, wl.rows, p, wl.u0)
    for _ in range(args.warmup):
        do_step()
    sess.profile()  # reset counters
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    l0 = ss.launch_count()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            do_step()
        e1.record(stream)
        e1.synchronize()
    launches = ss.launch_count() - l0
    barrier()
    ms = e0.elapsed_time(e1)
    prof = sess.profile()
    sweeps = prof["sweeps"]
    # halo exchange of the timed run (t-slabs, N > 1): the comm stream's exchange time and the
    # part the compute stream waited for after its interior slices
    halo_vals = [prof["halo_ms"] / prof["halo_n"], prof["halo_exposed_ms"] / prof["halo_n"]] if prof.get("halo_n") \
        else [0.0, 0.0]
    ms_max, hx, hexp = max_over_ranks([ms] + halo_vals)
    value = wl.n_interior * sweeps / (ms_max * 1e-3)  # whole grid (all ranks) per second

    # ---------------- e2e: the same steps through the public host-buffer call
    # (ss_session_step_host_async): every step uploads its input u^{n-1} from pinned host
    # memory and reads its result u^n back (compact interiors of this rank's slices; the ghost
    # layer is the session's Dirichlet data), the upload overlapped with the assembly; the
    # result's download is left in flight and the next step's upload of that same host buffer
    # is chained to it chunk by chunk on the device (D2H and H2D overlap; on the ranks of a
    # distributed run the chunked upload precedes the halo exchange and the assembly)
    n_owned = int(np.prod(sess.interior_shape))
    host_in = torch.empty(n_owned, dtype=torch.float64, pin_memory=True)
    host_out = torch.empty(n_owned, dtype=torch.float64, pin_memory=True)
    sess.prepare(wl.image, wl.rows, p, wl.u0)
    for _ in range(args.warmup):
        do_step()
    host_in.copy_(torch.from_numpy(sess.get_u_interior().ravel()))
    sess.profile()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        sess.step_host_async(host_in.data_ptr(), host_out.data_ptr(), fixed or 0, diag=False)
        host_in, host_out = host_out, host_in
    sess.wait()  # the last result is on the host; the stream is ordered after every copy
    f1.record(stream)
    f1.synchronize()
    barrier()
    ms_e2e = f0.elapsed_time(f1)
    sweeps_e2e = sess.profile()["sweeps"]
    (ms_e2e_max,) = max_over_ranks([ms_e2e])
    e2e_value = wl.n_interior * sweeps_e2e / (ms_e2e_max * 1e-3)

    # ---------------- per-kernel split (profiling run, after the timed region)
    sess.prepare(wl.image, wl.rows, p, wl.u0)
    for _ in range(args.warmup):
        do_step()
    sess.set_profiling(True)
    sess.profile()
    for _ in range(2):
        do_step()
    pr = sess.profile()
    sess.set_profiling(False)
    # roofline of the dominant kernel (SOR colour pass): its time measured live in the timed
    # region -- CUDA events around every SOR loop (one CUDA-graph launch per solve; the
    # host-driven loop on slab groups) / the colour passes it ran, launch gaps and the
    # finalize included; the profiling run's per-kernel events are reported beside it
    pass_ms_kernel = (pr["red_ms"] + pr["black_ms"]) / max(1, pr["red_n"] + pr["black_n"])
    pass_ms = prof["loop_ms"] / prof["loop_passes"] if prof.get("loop_passes") else pass_ms_kernel
    n_local = wl.n_interior // world  # doxels of this rank's slab (weak scaling: equal slabs)
    bytes_per_pass = SURVEY_BYTES_PER_SWEEP * n_local / 2.0
    achieved = bytes_per_pass / (pass_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(args.config, {}).get("sor_pass_bytes")
        except Exception:
            traffic = None
    tot = pr["red_ms"] + pr["black_ms"] + pr["assemble_ms"] + pr["rescale_ms"]
    sor_share = (pr["red_ms"] + pr["black_ms"]) / max(1e-9, tot)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(wl, args.config, world),
            "parallelism": (f"t-slabs x{world} (" + ("host-staged gloo exchange, ranks sharing a GPU: "
                                                     "functional test, not a scaling number" if host_tr else
                                                     "NCCL halo exchange per colour pass") + ")") if world > 1 else "1 GPU",
            "sweeps_timed": int(sweeps),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * n_owned * world,
                    "d2h_bytes_per_step": 8 * n_owned * world,
                    "call": "Session.step_host_async (ss_session_step_host_async) + wait(): every step "
                            "u^{n-1} H2D from pinned host memory, the time step, u^n D2H -- compact "
                            "interiors, all inside the CUDA events; step n+1's input is step n's host "
                            "output, each upload chunk device-ordered after its download chunk (the two "
                            "PCIe directions overlap)"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "sor_pass_tma (one colour half-sweep)",
                         "bytes_per_launch": bytes_per_pass, "avg_launch_ms": pass_ms,
                         "avg_launch_ms_source": "timed region: events around each SOR loop / passes run"
                         if prof.get("loop_passes") else "profiling run: per-kernel events",
                         "avg_launch_ms_per_kernel_events": pass_ms_kernel,
                         "peak_source": peak_src, "sor_share_of_step": sor_share,
                         "assemble_ms_per_step": pr["assemble_ms"] / max(1, pr["assemble_n"])},
            "clocks": clk.summary(),
        }
        if world > 1:
            line["halo"] = {"exchanges_timed": int(prof.get("halo_n", 0)), "exchange_ms": hx, "exposed_ms": hexp,
                            "overlapped_ms": max(0.0, hx - hexp),
                            "source": "timed region: events on the comm stream around each colour pass's "
                                      "exchange and on the compute stream after its interior slices "
                                      "(mean per exchange, max over ranks)"}
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline_sample(wl)
            except Exception as e:  # reported, not fatal
                line["cpu_baseline"] = {"error": str(e)}
        print(json.dumps(line))
    sess.close()
    if dist_init:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
