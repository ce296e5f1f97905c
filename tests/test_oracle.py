"""CPU tests of the oracle itself (no GPU).

The oracle restates the reference's ThinkvMethod over the compiled reference
library (oracle/_ref).  These tests pin it:
  * the reference's own doctest suites pass against oracle/_ref (built from
    /root/reference by oracle/Makefile; skipped where the prebuilt binaries
    are absent);
  * the restatement reproduces thinkv::generation_loop byte for byte
    (metrics, events, block tables, segments, step dumps) on a spread of
    configurations, and the reference's golden walkthrough fixture;
  * the golden wire vectors (quant_vectors.json) decode to the documented
    codes under the restated codec (oracle/codecs.py);
  * the synthetic generator is deterministic and bf16-exact.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
REF_BIN = os.path.join(os.path.dirname(HERE), "oracle", "_ref")

BASE = {"model": {"num_layers": 2, "head_dim": 8, "num_heads": 2, "gqa_group_size": 1,
                  "embed_dim": 16, "seed": 5},
        "tau": 16, "group_size": 8, "block_size": 4, "budget": 512, "schedule": [8, 4, 2],
        "num_thoughts": 3, "max_gen_len": 112, "prompt_len": 0, "seed": 21, "pool_blocks": 256,
        "scripted_trace": ["R", "E", "T", "R", "E", "T", "R"]}
UNSCRIPTED = {k: v for k, v in BASE.items() if k != "scripted_trace"}
CAL = {"layers": [0, 1], "thresholds": [0.3, 0.6], "num_thoughts": 3, "bandwidth_rule": "scott"}

TOY_CONFIGS = {
    "walkthrough": {"model": {"num_layers": 1, "head_dim": 4, "num_heads": 1, "embed_dim": 8, "seed": 7},
                    "tau": 4, "group_size": 4, "block_size": 4, "budget": 64, "schedule": [2],
                    "num_thoughts": 3, "max_gen_len": 16, "seed": 1, "pool_blocks": 16,
                    "scripted_trace": ["R", "E", "T", "R"], "dump_positions": [3, 7, 11, 12, 15]},
    "small": BASE,
    "maxpool_fp8": {**BASE, "model": {**BASE["model"], "num_heads": 4, "gqa_group_size": 2},
                    "precision_map": "R8E4T2", "budget": 24, "dump_positions": [40, 80]},
    "raw16_overflow": {**BASE, "precision_map": "R16E8T2", "budget": 20},
    "prompt_misaligned": {**BASE, "prompt_len": 20, "tau": 12, "budget": 30, "max_gen_len": 90},
    "calibrated": {**UNSCRIPTED, "calibration": CAL, "budget": 30},
    "per_layer": {**UNSCRIPTED, "calibration": {**CAL, "thresholds": [0.2, 0.5]}, "budget": 30,
                  "per_layer_thought": True},
    "big_d": {**BASE, "model": {**BASE["model"], "head_dim": 64, "num_heads": 4, "gqa_group_size": 4},
              "tau": 32, "group_size": 16, "block_size": 16, "budget": 60, "schedule": [16, 8, 4],
              "max_gen_len": 400},
}


@pytest.mark.parametrize("name", sorted(TOY_CONFIGS))
def test_restatement_matches_generation_loop(name):
    r = O.toy_compare(TOY_CONFIGS[name])
    assert "error" not in r, r.get("error")
    for key in ("metrics", "events", "tables", "segments", "step_dumps"):
        assert r["reference"][key] == r["oracle"][key], f"{name}: {key} differs"


def test_walkthrough_golden_fixture():
    r = O.toy_compare(TOY_CONFIGS["walkthrough"])
    golden = json.load(open(os.path.join(HERE, "golden", "walkthrough_dumps.json")))
    assert r["oracle"]["step_dumps"] == golden


@pytest.mark.parametrize("suite", ["test_quant", "test_attention", "test_thought", "test_evictor",
                                   "test_pager", "test_sim"])
def test_reference_suite_passes(suite):
    exe = os.path.join(REF_BIN, suite)
    if not os.path.exists(exe):
        pytest.skip("reference suites are built only where /root/reference exists")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr


def test_quant_wire_vectors():
    import codecs_ref as CR
    for vec in json.load(open(os.path.join(HERE, "golden", "quant_vectors.json"))):
        xs = np.array(vec["values"], dtype=np.float64)
        if vec["format"] == "TERNARY2":
            got = CR.serialize(CR.ternary_group(xs))
        elif vec["format"] == "NVFP4":
            got = CR.serialize(CR.nvfp4_group(xs))
        else:
            got = CR.serialize(CR.fp8_group(xs, np.float32(vec["scale"])))
        assert got.hex() == vec["bytes"], vec["comment"]


def test_e4m3_known_codes():
    import codecs_ref as CR
    # test_quant.cpp:101-116
    assert CR.e4m3_encode(1.0) == 0x38
    assert CR.e4m3_encode(448.0) == 0x7E
    assert CR.e4m3_encode(1e9) == 0x7E
    assert CR.e4m3_encode(2.0 ** -10) == 0x00  # subnormal tie to even
    assert CR.e4m3_encode(3 * 2.0 ** -10) == 0x02
    for c in range(256):
        if c & 0x7F == 0x7F:
            continue
        assert CR.e4m3_encode(CR.e4m3_decode(c)) == (c if c != 0x80 else 0x80)


def test_synth_is_deterministic_and_bf16():
    a = O.synth_step(7, 4, 16, 8, 4, 64, 10)
    b = O.synth_step(7, 4, 16, 8, 4, 64, 10)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    q, k, v = a
    assert q.shape == (8, 4, 64) and k.shape == (8, 64)
    f = O.bf16_to_f64(k)
    assert np.all(np.isfinite(f)) and 0.5 < f.std() < 3.0
    c = O.synth_step(7, 4, 16, 8, 4, 64, 11)
    assert not np.array_equal(c[1], k)


GATHER_CONFIGS = {
    "small": TOY_CONFIGS["small"],
    "maxpool": {**BASE, "model": {**BASE["model"], "num_heads": 4, "gqa_group_size": 4}},
    "prompt_misaligned": TOY_CONFIGS["prompt_misaligned"],
    "big_d": TOY_CONFIGS["big_d"],
}


@pytest.mark.parametrize("name", sorted(GATHER_CONFIGS))
def test_gather_restatement_matches_run_baseline(name):
    """The GatherMethod restatement (external inputs) reproduces the
    reference's run_baseline(config, "gather_compaction") metrics."""
    cfg = dict(GATHER_CONFIGS[name])
    cfg["budget"] = min(cfg["budget"], 24)
    r = O.gather_toy_compare(cfg)
    assert "error" not in r, r.get("error")
    assert r["oracle"] == r["reference"]
    assert r["reference"]["moved_token_slots"] > 0
