"""The C++ host side (include/thinkv_b200.hpp) drives the GPU path like a C++
caller of the reference drives ThinkvMethod: the reference's golden
walkthrough (test_sim.cpp:386-489) must come out bit-identical, and pool
exhaustion must surface as an exception with the reference's exit code 4."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
DRIVER = os.path.join(ROOT, "build", "walkthrough_driver")

WALK = {"model": {"num_layers": 1, "head_dim": 4, "num_heads": 1, "embed_dim": 8, "seed": 7},
        "tau": 4, "group_size": 4, "block_size": 4, "budget": 64, "schedule": [2],
        "num_thoughts": 3, "max_gen_len": 16, "seed": 1, "pool_blocks": 16,
        "scripted_trace": ["R", "E", "T", "R"], "dump_positions": [3, 7, 11, 12, 15]}


def test_cpp_driver_is_built_against_the_header():
    if not os.path.exists(DRIVER):
        pytest.skip("build() has not produced build/walkthrough_driver")
    out = subprocess.run(["nm", "-D", "--undefined-only", DRIVER], capture_output=True, text=True).stdout
    for sym in ("tkv_init", "tkv_run_create", "tkv_step", "tkv_finish", "tkv_dump_json"):
        assert sym in out


@pytest.mark.gpu
def test_cpp_walkthrough_golden(tmp_path):
    q, k, v = O.toy_stream(WALK)
    arr = np.stack([np.asarray(q).reshape(16, 4), np.asarray(k).reshape(16, 4), np.asarray(v).reshape(16, 4)])
    f = tmp_path / "walk.f64"
    arr.astype(np.float64).tofile(f)
    p = subprocess.run([DRIVER, str(f)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    golden = json.load(open(os.path.join(HERE, "golden", "walkthrough_dumps.json")))
    assert json.loads(p.stdout) == golden


@pytest.mark.gpu
def test_cpp_oom_exit_code():
    p = subprocess.run([DRIVER, "-", "oom"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    assert json.loads(p.stdout)["oom_exit_code"] == 4
