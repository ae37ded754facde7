"""Randomised sweeps through the C ABI: qdwh_partial_eig / qdwh_partial_svd
(tools/fuzz_partial.py: sizes, spectra, fractions and the randomized-detection switch drawn
from a seeded generator, every case checked against its planted spectrum and the north-star
gates) and the dense entry points (tools/fuzz_dense.py, against LAPACK)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed", [11, 12])
def test_partial_drivers_fuzz(seed):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_partial.py"), str(seed), "30", "24"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert lines[-1] == "FAILS 0", "\n".join(l for l in lines if l.startswith("FAIL"))[-3000:]
    assert sum(l.startswith("ok") for l in lines) >= 40


def test_dense_entry_points_fuzz():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_dense.py"), "21", "12"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert lines[-1] == "FAILS 0", "\n".join(l for l in lines if l.startswith("FAIL"))[-3000:]
    assert sum(l.startswith("ok") for l in lines) == 48
