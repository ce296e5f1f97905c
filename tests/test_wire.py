"""Wire layout of the compressed-cache export: the package's
host reader (paper_2510_01290_b200.wire) against the reference's golden wire
vectors (tests/golden/quant_vectors.json = proj/tests/fixtures), its
round-trip / error behaviour (test_quant.cpp:360-402), and the oracle's
export stream (built by the compiled reference's serialize_group)."""
import json
import os

import numpy as np
import pytest

import codecs_ref as R
from paper_2510_01290_b200 import wire

HERE = os.path.dirname(os.path.abspath(__file__))
FMT = {"TERNARY2": wire.TERNARY2, "NVFP4": wire.NVFP4, "FP8E4M3": wire.FP8E4M3}


def golden():
    return json.load(open(os.path.join(HERE, "golden", "quant_vectors.json")))


@pytest.mark.parametrize("i", range(3))
def test_golden_vectors_roundtrip(i):
    vec = golden()[i]
    b = bytes.fromhex(vec["bytes"])
    grp, used = wire.deserialize_group(b)
    assert used == len(b)
    assert grp.format == FMT[vec["format"]] and grp.g == len(vec["values"])
    assert wire.serialize_group(grp) == b
    # codes equal the reference encoder restatement's (pinned in test_oracle.py)
    ref = {"TERNARY2": lambda xs: R.ternary_group(xs), "NVFP4": lambda xs: R.nvfp4_group(xs),
           "FP8E4M3": lambda xs: R.fp8_group(xs, vec.get("scale", 1.0))}[vec["format"]](vec["values"])
    assert list(grp.codes) == [int(c) for c in ref.codes]
    dec = [wire.decode_code(grp.format, c, grp.scale()) for c in grp.codes]
    if vec["format"] == "NVFP4":
        assert dec == vec["values"]  # exactly representable on the grid at scale 1.0
    if vec["format"] == "TERNARY2":
        assert dec == [0.8125, 0.0, 0.0, 0.8125]  # test_quant.cpp:214-228 (delta = e4m3(0.8))


def test_deserialize_errors():
    with pytest.raises(wire.WireError):  # truncated header (test_quant.cpp:400)
        wire.deserialize_group(bytes([0x00, 0x10]))
    with pytest.raises(wire.WireError):  # unknown format tag
        wire.deserialize_group(bytes([0x07, 0x01, 0x00, 0x38, 0x00]))
    with pytest.raises(wire.WireError):  # codes truncated
        wire.deserialize_group(bytes([0x01, 0x10, 0x00, 0x38, 0x00]))


def test_roundtrip_property():
    rng = np.random.default_rng(5)
    for fmt, bits in ((wire.TERNARY2, 2), (wire.NVFP4, 4), (wire.FP8E4M3, 8)):
        for g in (1, 2, 3, 7, 16, 33):
            codes = [int(x) for x in rng.integers(0, 1 << bits, g)]
            if fmt == wire.TERNARY2:
                codes = [c if c != 2 else 0 for c in codes]
            grp = wire.QuantizedGroup(fmt, g, int(rng.integers(0, 0x7E)), float(rng.random()), codes)
            back, used = wire.deserialize_group(wire.serialize_group(grp))
            assert back.codes == codes and back.g == g


def test_oracle_export_parses():
    """The oracle's export (reference serialize_group over the reference
    pager) covers every live pager token and parses exactly."""
    import oracle as O
    from harness import synth_inputs
    rng = np.random.default_rng(1)
    script = [[int(x) for x in rng.integers(0, 3, 12)]]
    cfg = O.RunConfig(num_seqs=1, units_per_seq=2, num_q_heads=2, head_dim=32, tau=16, group_size=8,
                      block_size=8, budget=40, levels=(8, 4, 2), psi_bits=(4, 8, 2), max_gen_len=160,
                      script=script)
    orc = O.OracleRun(cfg)
    for t in range(cfg.max_gen_len):
        q, k, v = synth_inputs(cfg, 0x71534B56, t)
        orc.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
    tables = orc.dump(0, "tables")
    for u in range(2):
        b = orc.export(0, u)
        recs, used = wire.parse_unit(b)
        assert used == len(b)
        ids = np.concatenate([r.ids for r in recs])
        assert np.all(np.diff(ids) > 0)
        kinds = {r.kind for r in recs}
        assert kinds <= {wire.TERNARY2, wire.NVFP4, wire.FP8E4M3}
        # live tokens of the reference's own block-table dump (pager.cpp:327-362)
        live = sorted(tok for blk in tables[u]["blocks"]
                      for tok, ev in zip(blk["tokens"], blk["eviction_mask"]) if tok is not None and ev == "0")
        assert ids.tolist() == live
        assert any(r.kind == wire.FP8E4M3 for r in recs) and any(r.kind == wire.TERNARY2 for r in recs)
