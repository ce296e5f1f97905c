"""Shared parity harness: drive the CUDA path (paper_2510_01290_b200) and the
oracle (oracle/, the reference restatement over the compiled reference
library) on identical inputs and compare everything the reference exposes.

Tolerances:
  * cache state (codes implied by dumps, block tables, eviction masks, start
    indices, segment masks, free lists, segment members, events, metrics):
    exact equality of the reference's JSON views;
  * attention outputs: max |gpu - oracle| <= ATOL + RTOL * max|oracle| per
    step, with ATOL = 1e-3 and RTOL = 1e-3 (north_star: "max-abs 1e-3
    relative to the reference"); the CUDA kernel accumulates in fp32 with
    exact dequantised products, so observed errors are ~1e-6.
"""
from __future__ import annotations

import dataclasses

import numpy as np

import oracle as O

ATOL = 1e-3
RTOL = 1e-3


def oracle_config(cfg) -> "O.RunConfig":
    fields = {f.name for f in dataclasses.fields(O.RunConfig)}
    return O.RunConfig(**{k: v for k, v in dataclasses.asdict(cfg).items() if k in fields})


def synth_inputs(cfg, seed, step):
    q, k, v = O.synth_step(seed, cfg.units_per_seq, cfg.tau, cfg.units, cfg.num_q_heads,
                           cfg.head_dim, step)
    return q, k, v


def run_parity(cfg, seed=0x71534B56, steps=None, check_every=1, inputs=None):
    """Returns a dict of comparison results.  inputs: optional callable
    step -> (q, k, v) numpy arrays in cfg.input_dtype's host representation
    (uint16 bf16 bits or float64)."""
    import torch
    from paper_2510_01290_b200 import DecodeRun

    steps = steps if steps is not None else cfg.prompt_len + cfg.max_gen_len
    run = DecodeRun(cfg)
    orc = O.OracleRun(oracle_config(cfg))
    dev = torch.device("cuda:0")
    rows = cfg.out_rows
    out = torch.empty((cfg.units, rows, cfg.head_dim), dtype=torch.float32, device=dev)
    max_err = 0.0
    for t in range(steps):
        if inputs is None:
            q, k, v = synth_inputs(cfg, seed, t)
        else:
            q, k, v = inputs(t)
        if cfg.input_dtype == "bf16":
            qd, kd, vd = O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v)
            tq = torch.from_numpy(q.view(np.int16)).view(torch.bfloat16).to(dev)
            tk = torch.from_numpy(k.view(np.int16)).view(torch.bfloat16).to(dev)
            tv = torch.from_numpy(v.view(np.int16)).view(torch.bfloat16).to(dev)
        else:
            qd, kd, vd = q, k, v
            tt = torch.float64 if cfg.input_dtype == "f64" else torch.float32
            tq, tk, tv = (torch.from_numpy(np.ascontiguousarray(x)).to(dev, tt) for x in (q, k, v))
        ref_out, _ = orc.step(qd, kd, vd)
        run.step(tq, tk, tv, out)
        if t % check_every == 0 or t == steps - 1:
            got = out.double().cpu().numpy()
            err = float(np.max(np.abs(got - ref_out)))
            scale = float(np.max(np.abs(ref_out)))
            assert err <= ATOL + RTOL * scale, f"step {t}: attention error {err} (scale {scale})"
            max_err = max(max_err, err)
    run.synchronize()
    res = {"max_err": max_err, "run": run, "oracle": orc, "steps": steps}
    return res


def compare_export(res, cfg):
    """Compressed-cache export (k_export.cu) == the oracle's export built by
    the reference's serialize_group, byte for byte, for every unit; the
    stream parses with the package's wire reader."""
    from paper_2510_01290_b200 import wire
    run, orc = res["run"], res["oracle"]
    buf, offs = run.export_cache()
    host = buf.cpu().numpy().tobytes()
    ups = cfg.units_per_seq
    for u in range(cfg.units):
        got = host[offs[u]:offs[u + 1]]
        ref = orc.export(u // ups, u % ups)
        assert got == ref, f"unit {u}: export differs ({len(got)} vs {len(ref)} bytes)"
        recs, used = wire.parse_unit(got)
        assert used == len(got)
    return len(host)


def compare_state(res, cfg, finish=True):
    run, orc = res["run"], res["oracle"]
    compare_export(res, cfg)
    compare_bytes(run, [orc])
    if finish:
        run.finish()
        orc.finish()
    for s in range(cfg.num_seqs):
        gt, ot = run.tables(s), orc.dump(s, "tables")
        assert gt == ot, f"seq {s}: block tables differ"
        gs, os_ = run.segments(s), orc.dump(s, "segments")
        assert gs == os_, f"seq {s}: segments differ"
        if cfg.record_events:
            ge, oe = run.events(s), orc.dump(s, "events")
            assert [l for l in ge.splitlines()] == [l for l in oe.splitlines()], f"seq {s}: events differ"
        if cfg.dump_positions:
            assert run.step_dumps(s) == orc.dump(s, "step_dumps"), f"seq {s}: step dumps differ"
        if finish:
            assert run.metrics(s) == orc.dump(s, "metrics"), f"seq {s}: metrics differ"


def unit_subset_config(cfg, units):
    """A run of len(units) one-unit sequences that is, unit for unit, the same
    decode as units `units` of `cfg` (scripted labels are per sequence and
    units are independent): unit u keeps its sequence's script."""
    ups = cfg.units_per_seq
    return dataclasses.replace(cfg, num_seqs=len(units), units_per_seq=1,
                               script=[list(cfg.script[u // ups]) for u in units])


def run_parity_units(cfg, units, seed=0x71534B56, steps=None, check=()):
    """GPU vs oracle over global units `units` of `cfg` (inputs of those
    global units, generated as cfg generates them) for `steps` steps.  The
    oracle decodes each unit on its own thread, concurrently with the GPU.
    Outputs are compared at the positions in `check`; returns the same dict
    as run_parity with one OracleRun per unit under "oracles"."""
    import threading

    import torch
    from paper_2510_01290_b200 import DecodeRun

    steps = steps if steps is not None else cfg.prompt_len + cfg.max_gen_len
    sub = unit_subset_config(cfg, units)
    check = set(check)
    G, D, ups = cfg.num_q_heads, cfg.head_dim, cfg.units_per_seq
    orcs = [O.OracleRun(oracle_config(unit_subset_config(cfg, [u]))) for u in units]
    ref_outs = [dict() for _ in units]
    errs = []

    def worker(i):
        try:
            for t in range(steps):
                q, k, v = O.synth_step(seed, ups, cfg.tau, 1, G, D, t, unit0=units[i])
                out, _ = orcs[i].step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
                if t in check:
                    ref_outs[i][t] = out[0].copy()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(units))]
    for th in threads:
        th.start()
    run = DecodeRun(sub)
    dev = torch.device("cuda:0")
    out = torch.empty((len(units), sub.out_rows, D), dtype=torch.float32, device=dev)
    got = {}
    for t in range(steps):
        parts = [O.synth_step(seed, ups, cfg.tau, 1, G, D, t, unit0=u) for u in units]
        q, k, v = (np.concatenate([p[j] for p in parts]) for j in range(3))
        tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
        run.step(tq, tk, tv, out)
        if t in check:
            got[t] = out.double().cpu().numpy()
    run.synchronize()
    for th in threads:
        th.join()
    if errs:
        raise errs[0]
    max_err = 0.0
    for t, g in got.items():
        for i in range(len(units)):
            ref = ref_outs[i][t]
            err = float(np.max(np.abs(g[i] - ref)))
            scale = float(np.max(np.abs(ref)))
            assert err <= ATOL + RTOL * scale, f"step {t} unit {units[i]}: attention error {err} (scale {scale})"
            max_err = max(max_err, err)
    return {"max_err": max_err, "run": run, "oracles": orcs, "steps": steps, "config": sub}


def compare_units_state(res, finish=True):
    """compare_state for run_parity_units: unit i of the GPU run against its
    own OracleRun (tables, segments, events, export bytes, fragmentation
    byte accounting, metrics)."""
    run, orcs, sub = res["run"], res["oracles"], res["config"]
    buf, offs = run.export_cache()
    host = buf.cpu().numpy().tobytes()
    for i, orc in enumerate(orcs):
        assert host[offs[i]:offs[i + 1]] == orc.export(0, 0), f"unit {i}: export differs"
    compare_bytes(run, orcs)
    if finish:
        run.finish()
        for orc in orcs:
            orc.finish()
    for i, orc in enumerate(orcs):
        assert run.tables(i) == orc.dump(0, "tables"), f"unit {i}: block tables differ"
        assert run.segments(i) == orc.dump(0, "segments"), f"unit {i}: segments differ"
        if sub.record_events:
            assert run.events(i).splitlines() == orc.dump(0, "events").splitlines(), f"unit {i}: events differ"
        if finish:
            assert run.metrics(i) == orc.dump(0, "metrics"), f"unit {i}: metrics differ"


def compare_bytes(run, orcs):
    """Byte accounting (tkv_bytes, the roofline numerator) against the
    reference's BlockPager::fragmentation_stats (pager.cpp:299-325) summed
    over units: live slots, live code bits, live scale bytes."""
    frag = [f for orc in orcs for seq in range(orc.cfg.num_seqs) for f in orc.dump(seq, "frag")]
    b = run.bytes()
    assert b["live_slots"] == sum(f["live_slots"] for f in frag)
    assert b["resident_slots"] == sum(f["live_slots"] + f["masked_slots"] for f in frag)
    # RAW16 passthrough: the reference counts 16 bits per element; the device
    # stores (and K1 reads) the input dtype, so those bits scale by its width.
    in_bytes = {"bf16": 2, "f32": 4, "f64": 8}[run.cfg.input_dtype]
    want_bits = sum(bits * (in_bytes // 2 if fmt == "RAW16" else 1)
                    for f in frag for fmt, bits in f["live_code_bits_by_format"].items())
    assert b["live_code_bytes"] * 8 == want_bits
    assert b["live_scale_bytes"] == sum(f["live_scale_bytes"] for f in frag)
    return b
