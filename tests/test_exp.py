"""tkv_exp (csrc/tkv_exp.cuh) is the exp() of the reference's CPU build bit for
bit: glibc's exp as selected on this image's FMA + AVX2 hosts.  The table
generator (tools/gen_exp_table.py) is checked against the committed header,
and a host build of the function against the C library over 18M inputs."""
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2510_01290_b200", "csrc")


def test_generated_table_is_committed():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_exp_table
    rows = gen_exp_table.table()
    text = open(os.path.join(CSRC, "tkv_exp_table.h")).read()
    for tb, hb in rows:
        assert f"0x{tb:016x}ull, 0x{hb:016x}ull" in text


def test_host_build_matches_libc_exp_bit_for_bit():
    flags = open("/proc/cpuinfo").read()
    if " fma" not in flags or " avx2" not in flags:
        pytest.skip("glibc selects its FMA exp only on FMA + AVX2 hosts")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "exp_check")
        subprocess.run(["g++", "-std=c++17", "-O2", "-I" + CSRC, os.path.join(ROOT, "tests", "cpp", "exp_check.cpp"),
                        "-o", exe], check=True)
        out = subprocess.run([exe, "2000000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:]
    assert "mismatches 0" in out.stdout
