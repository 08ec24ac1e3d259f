"""Build and run the C++ drop-in test (tests/cpp/test_host_mirror.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_cpp_test():
    pkg = os.path.join(ROOT, "paper_2111_11866_b200")
    subprocess.run(["make", "-s", "-C", os.path.join(pkg, "host")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")],
                   check=True)
    exe = os.path.join(ROOT, "tests", "cpp", "test_host_mirror")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ROOT, "oracle"),
                    os.path.join(ROOT, "tests", "cpp", "test_host_mirror.cpp"), "-o", exe,
                    "-L" + pkg, "-lsubsurf_b200_host", "-lsubsurf_b200", "-Wl,-rpath," + pkg,
                    "-L" + os.path.join(ROOT, "oracle"), "-loracle", "-Wl,-rpath," + os.path.join(ROOT, "oracle")],
                   check=True)
    return exe


def test_cpp_dropin_builds():
    """CPU: the C++ mirror and the test link (no device needed to build)."""
    assert os.path.exists(build_cpp_test())


@pytest.mark.gpu
def test_cpp_dropin_matches_oracle():
    exe = build_cpp_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "ALL OK" in r.stdout
