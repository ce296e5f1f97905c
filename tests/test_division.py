"""The exact division by cluster size used by the K-means kernels (k_kmeans.cu
div_n: Markstein's fma correction from the correctly rounded reciprocal)
gives the bits of IEEE x / n, checked on the host for every non-power-of-two
n up to 1024 (the kernels' table size) on random and few-bit operands."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def test_markstein_division_matches_ieee(tmp_path):
    exe = tmp_path / "div_check"
    # -ffp-contract=off: the C statements are the kernel's operations, one rounding each
    r = subprocess.run(["gcc", "-O2", "-ffp-contract=off", os.path.join(HERE, "cpp", "div_check.c"), "-o", str(exe),
                        "-lm"], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("no C compiler: " + r.stderr[-200:])
    out = subprocess.run([str(exe), "20000"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.startswith("bad 0 of"), out.stdout
