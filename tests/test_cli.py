"""The `subsurf-b200` CLI drop-in (paper_2111_11866_b200/host/cli.cpp; reference
cli.cpp:117-262): config keys, file formats (io.cpp:22-223), error behaviour on
CPU, and segment / threshold-preview / eoc output on the GPU against the oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

import _cases as cs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2111_11866_b200", "subsurf-b200")


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2111_11866_b200", "csrc")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2111_11866_b200", "host")], check=True)
    return CLI


def write_case(d, dims, h, image, rows, extra=""):
    n1, n2, n3, n4 = dims
    json.dump({"dims": list(dims), "spacing": [h] * 4, "dtype": "f32le", "order": "i-fastest"},
              open(os.path.join(d, "img.json"), "w"))
    image[1:-1, 1:-1, 1:-1, 1:-1].astype("<f4").tofile(os.path.join(d, "img.raw"))
    with open(os.path.join(d, "centers.csv"), "w") as f:
        f.write("frame,x,y,z,radius\n")
        for r in rows:
            f.write(",".join(str(v) for v in r) + "\n")
    with open(os.path.join(d, "cfg.txt"), "w") as f:
        f.write(f"# test config\ninput_header = {d}/img.json\ninput_data = {d}/img.raw\n"
                f"centers = {d}/centers.csv\noutput = {d}/out\n" + extra)


def read_out(prefix):
    hdr = json.load(open(prefix + ".json"))
    n1, n2, n3, n4 = hdr["dims"]
    return hdr, np.fromfile(prefix + ".raw", dtype="<f4").reshape(n4, n3, n2, n1)


def test_cli_usage_and_errors(cli, tmp_path):
    r = subprocess.run([cli, "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "segment" in r.stdout and "eoc" in r.stdout
    r = subprocess.run([cli, "segment"], capture_output=True, text=True)
    assert r.returncode == 2 and "--config" in r.stderr
    bad = tmp_path / "bad.txt"
    bad.write_text("no equals sign here\n")
    r = subprocess.run([cli, "segment", "--config", str(bad)], capture_output=True, text=True)
    assert r.returncode == 1 and "expected key = value" in r.stderr
    dims = (4, 4, 3, 3)
    write_case(str(tmp_path), dims, 0.25, cs.f32_image(dims, 1), [(0, 1.5, 1.5, 1.0, 1.0)])
    (tmp_path / "img.raw").write_bytes((tmp_path / "img.raw").read_bytes()[:-1])
    r = subprocess.run([cli, "segment", "--config", str(tmp_path / "cfg.txt")], capture_output=True, text=True)
    assert r.returncode == 1 and "payload is" in r.stderr  # io.cpp:83-86 FormatError


@pytest.mark.parametrize("row", ["0 1.5 1.5 1.0 1.0", "0,1.5 1.5,1.0,1.0", "0;1.5;1.5;1.0;1.0", "0,1.5,1.5,1.0"])
def test_cli_centers_grammar(cli, tmp_path, row):
    """read_centers accepts exactly frame,x,y,z,radius with ',' separators (io.cpp:158-163):
    whitespace- or partly comma-separated rows are a FormatError, like the reference's."""
    dims = (4, 4, 3, 3)
    write_case(str(tmp_path), dims, 0.25, cs.f32_image(dims, 1), [(0, 1.5, 1.5, 1.0, 1.0)])
    (tmp_path / "centers.csv").write_text("frame,x,y,z,radius\n" + row + "\n")
    r = subprocess.run([cli, "segment", "--config", str(tmp_path / "cfg.txt")], capture_output=True, text=True)
    assert r.returncode == 1 and "expected frame,x,y,z,radius" in r.stderr, r.stderr


def test_cli_no_cpu_fallback(cli, tmp_path):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is visible")
    except ImportError:
        pass
    dims = (4, 4, 3, 3)
    write_case(str(tmp_path), dims, 0.25, cs.f32_image(dims, 1), [(0, 1.5, 1.5, 1.0, 1.0)])
    r = subprocess.run([cli, "segment", "--config", str(tmp_path / "cfg.txt")], capture_output=True, text=True)
    assert r.returncode == 1 and "no CPU fallback" in r.stderr


@pytest.mark.gpu
def test_cli_segment_matches_oracle(cli, oracle, ref, tmp_path):
    from oracle import oracle_py as op
    dims, h = (10, 8, 7, 6), 0.125
    img = cs.f32_image(dims, 3)
    rows = [(f, 4.5, 3.5, 3.0, 2.0) for f in range(dims[3])]
    extra = ("tau = 0.125\nepsilon = 0.001\nomega = 1.4\nsor_tol = 1e-9\nn_steps = 3\nsigma = 0.17677669529663687\n"
             "K = 200\ndelta = 0.5\nvartheta = 0.5\ninit_R = 3\nrescale_radius = 3\nexport_vtk = true\n")
    write_case(str(tmp_path), dims, h, img, rows, extra)
    r = subprocess.run([cli, "segment", "--config", str(tmp_path / "cfg.txt")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert r.stderr.count("sor_iters=") == 3
    hdr, u = read_out(str(tmp_path / "out"))
    p = op.seg_params(tau=0.125, epsilon=1e-3, omega=1.4, sor_tol=1e-9, n_steps=3, sigma=0.17677669529663687,
                      K=200.0, delta=0.5, vartheta=0.5, init_R=3.0, rescale_radius=3.0)
    st, uo, info = oracle.segment(op.Grid.make(dims, h), img, rows, p)
    assert st == 0
    assert np.array_equal(u, uo[1:-1, 1:-1, 1:-1, 1:-1].astype("<f4"))
    # the output files against the reference's own writers on the same u (io.cpp:99-119,
    # :198-223; cli.cpp:129-133): payload and VTK frames byte for byte; the JSON header's
    # whitespace depends on the (unvendored) nlohmann version, so it is compared parsed
    g = op.Grid.make(dims, h)
    d = str(tmp_path)
    assert ref.write_image4d(g, uo, d + "/ref.json", d + "/ref.raw") == 0
    assert open(d + "/ref.raw", "rb").read() == open(d + "/out.raw", "rb").read()
    assert json.load(open(d + "/ref.json")) == json.load(open(d + "/out.json"))
    for l in range(1, dims[3] + 1):
        assert ref.export_frame_vtk(g, uo, l, f"{d}/ref_f{l - 1}.vtk") == 0
        assert open(f"{d}/ref_f{l - 1}.vtk", "rb").read() == open(f"{d}/out_f{l - 1}.vtk", "rb").read(), l


@pytest.mark.gpu
def test_cli_threshold_and_eoc(cli, oracle, tmp_path):
    from oracle import oracle_py as op
    dims, h = (9, 7, 6, 4), 0.25
    img = cs.f32_image(dims, 4)
    rows = cs.centers_overlapping(dims)
    write_case(str(tmp_path), dims, h, img, rows, "lambda = 0.3\nbackground = -1\n")
    r = subprocess.run([cli, "threshold-preview", "--config", str(tmp_path / "cfg.txt")], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    _, th = read_out(str(tmp_path / "out"))
    st, tho = oracle.local_threshold(op.Grid.make(dims, h), img, rows, 0.3, -1.0)
    assert np.array_equal(th, tho[1:-1, 1:-1, 1:-1, 1:-1].astype("<f4"))
    r = subprocess.run([cli, "eoc", "--max-n", "20"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.rstrip("\n").splitlines()
    assert len(lines) == 3 and float(lines[1].split()[3]) == pytest.approx(1.684177e-2, rel=1e-6)
    assert float(lines[2].split()[4]) == pytest.approx(1.851052, rel=1e-5)
    # print_report's exact layout (eoc.cpp:193-203): header, setw(4)/setw(9)/setw(10) columns,
    # scientific error, fixed EOC from the second row on
    assert lines[0] == "   n          h  final step         error        EOC"
    for q, (n, steps) in enumerate(((10, 1), (20, 4))):
        err = float(lines[q + 1].split()[3])
        want = f"{n:4d}  {2.5 / n:>9g}  {steps:10d}  {err:.6e}"
        if q:
            want += f"   {float(lines[q + 1].split()[4]):.6f}"
        assert lines[q + 1] == want


@pytest.mark.gpu
def test_cli_track_matches_reference(cli, ref, tmp_path):
    """`subsurf-b200 track` (cli.cpp:161-188) == the reference's track() on the same f32 field."""
    from oracle.oracle_py import Grid
    dims = (24, 20, 10, 8)
    u = cs.track_scene(dims, 11)
    u32 = np.zeros_like(u)
    u32[1:-1, 1:-1, 1:-1, 1:-1] = u[1:-1, 1:-1, 1:-1, 1:-1].astype(np.float32)
    d = str(tmp_path)
    json.dump({"dims": list(dims), "spacing": [1.0] * 4, "dtype": "f32le", "order": "i-fastest"},
              open(os.path.join(d, "u.json"), "w"))
    u32[1:-1, 1:-1, 1:-1, 1:-1].astype("<f4").tofile(os.path.join(d, "u.raw"))
    with open(os.path.join(d, "trk.txt"), "w") as f:
        f.write(f"input_header = {d}/u.json\ninput_data = {d}/u.raw\noutput = {d}/traj.csv\n"
                f"level = 0.5\nwindow = 3\nradius = 5\nvtk_prefix = {d}/lab\n")
    r = subprocess.run([cli, "track", "--config", os.path.join(d, "trk.txt")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rows = open(os.path.join(d, "traj.csv")).read().splitlines()
    assert rows[0] == "trajectory_id,frame,x,y,z"
    want = ref.track(Grid.make(dims, 1.0), u32, 0.5, 3, 5.0)
    assert rows[1:] == [f"{a},{b},{x:g},{y:g},{z:g}" for a, b, x, y, z in want]
    # byte for byte against the reference's writers: write_trajectories (io.cpp:170-177) of
    # its track() points, and the label-field VTKs of cli.cpp:174-188
    g = Grid.make(dims, 1.0)
    assert ref.write_trajectories(want, os.path.join(d, "ref.csv")) == 0
    assert open(os.path.join(d, "ref.csv"), "rb").read() == open(os.path.join(d, "traj.csv"), "rb").read()
    assert ref.export_label_vtks(g, u32, 0.5, os.path.join(d, "reflab")) == 0
    for l in range(dims[3]):
        a = open(os.path.join(d, f"reflab_f{l}.vtk"), "rb").read()
        assert a == open(os.path.join(d, f"lab_f{l}.vtk"), "rb").read(), l
