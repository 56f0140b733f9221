"""The 128-bit window conversions used by the fitness kernels' region
pricing (fixed192.cuh: x128_to_double / x128_from_double) agree with the
192-bit fixed-point path bit for bit (host build of the same header)."""

import os
import subprocess

from conftest import ROOT


def test_x128_conversions_match_192_bit_path(tmp_path):
    src = os.path.join(ROOT, "tests", "native", "x128_check.cpp")
    exe = tmp_path / "x128_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-o", str(exe), src], check=True)
    out = subprocess.run([str(exe), "300000"], capture_output=True, text=True, timeout=300)
    iters, bad = map(int, out.stdout.split())
    assert iters == 300000 and bad == 0 and out.returncode == 0
