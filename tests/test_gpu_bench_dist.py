"""bench.py's multi-rank path (torchrun, N = 2 and 3) on one GPU: the ranks' halo
exchanges go through the host (SUBSURF_DIST_TRANSPORT=host -> gloo + dist.HostComm),
so the path runs -- per-rank slab workloads, max-over-ranks timing, the halo report
of the timed run, one JSON line from rank 0 -- without a second GPU.  A functional
test only: ranks sharing a GPU measure nothing about scaling."""
import json
import os
import signal
import socket
import subprocess
import sys
import warnings

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_bench(n):
    # a stuck rank dumps its stacks and exits after 240 s (bench.py's watchdog); the launcher and
    # whatever it left behind are killed as a process group, so nothing idles on the GPU
    env = dict(os.environ, SUBSURF_DIST_TRANSPORT="host", SUBSURF_BENCH_WATCHDOG="240")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(n),
           "--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    proc = subprocess.Popen(cmd, cwd=ROOT, env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                            start_new_session=True)
    try:
        out, err = proc.communicate(timeout=420)
        return proc.returncode, out, err
    except subprocess.TimeoutExpired:
        return -1, "", "bench.py ranks did not finish in 420 s"
    finally:
        try:
            os.killpg(proc.pid, signal.SIGKILL)  # launcher, ranks, their nvidia-smi samplers
        except ProcessLookupError:
            pass
        proc.wait()


@pytest.mark.parametrize("n", [2, 3])
def test_bench_multirank_over_host_transport(gpu, n):
    rc, out, err = _run_bench(n)
    if rc != 0:
        # seen once in ~70 runs (a 3-rank launch that never got going on a just-acquired box,
        # not reproduced in 45 back-to-back repeats): report it and try once more; a second
        # failure fails the test with both logs
        warnings.warn(f"bench.py --gpus {n} over the host transport failed once (rc {rc}):\n{err[-3000:]}")
        first = err
        rc, out, err = _run_bench(n)
        assert rc == 0, "first attempt:\n" + first[-3000:] + "\nsecond attempt:\n" + err[-3000:]
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["value"] > 0 and d["config"]["dims"] == [24, 20, 12, 6 * n]
    assert d["halo"]["exchanges_timed"] > 0 and d["halo"]["exchange_ms"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * 24 * 20 * 12 * 6 * n
