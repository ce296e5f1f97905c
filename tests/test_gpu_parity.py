"""GPU parity: the CUDA decode path against the oracle (reference
restatement over the compiled reference library) on identical inputs.

Cache state, eviction decisions, slot placements, free lists, events and
metrics must be bit-identical; attention outputs within harness.ATOL/RTOL.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
from harness import compare_state, oracle_config as harness_oracle_config, run_parity  # noqa: E402
from paper_2510_01290_b200 import DecodeRun, ThinkvConfig, TkvError  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def script(num_seqs, intervals, seed=3, pT=200):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(num_seqs):
        s = []
        for _ in range(intervals):
            s.append(2 if rng.random() < pT / 1000 else int(rng.integers(0, 2)))
        out.append(s)
    return out


def test_walkthrough_golden_fixture_on_gpu():
    """The reference's golden walkthrough (test_sim.cpp:386-489), fed the
    ToyModel stream in fp64, reproduces walkthrough_dumps.json on the GPU."""
    ref_cfg = {"model": {"num_layers": 1, "head_dim": 4, "num_heads": 1, "embed_dim": 8, "seed": 7},
               "tau": 4, "group_size": 4, "block_size": 4, "budget": 64, "schedule": [2],
               "num_thoughts": 3, "max_gen_len": 16, "seed": 1, "pool_blocks": 16,
               "scripted_trace": ["R", "E", "T", "R"], "dump_positions": [3, 7, 11, 12, 15]}
    q, k, v = O.toy_stream(ref_cfg)
    cfg = ThinkvConfig(num_seqs=1, units_per_seq=1, num_q_heads=1, head_dim=4, tau=4, group_size=4,
                       block_size=4, pool_blocks=16, budget=64, levels=(2,), psi_bits=(4, 4, 2),
                       max_gen_len=16, script=[[1, 0, 2, 1]], input_dtype="f64", record_events=True,
                       dump_positions=(3, 7, 11, 12, 15))
    res = run_parity(cfg, inputs=lambda t: (q[t], k[t], v[t]))
    golden = json.load(open(os.path.join(HERE, "golden", "walkthrough_dumps.json")))
    assert res["run"].step_dumps(0) == golden
    compare_state(res, cfg)


CONFIGS = {
    # d=128, G=4 per-head (R1-Llama-8B head shape), block 16, R4E4T2, transitions
    "llama_shape": ThinkvConfig(num_seqs=2, units_per_seq=3, num_q_heads=4, head_dim=128, tau=32,
                                group_size=16, block_size=16, budget=96, levels=(16, 8, 4),
                                max_gen_len=420, script=script(2, 16), record_events=True,
                                dump_positions=(100, 257)),
    # GPT-OSS head shape d=64, G=8, max-pool GQA, FP8 reasoning band, block 8
    "gptoss_maxpool_fp8": ThinkvConfig(num_seqs=2, units_per_seq=2, num_q_heads=8, gqa_maxpool=True,
                                       head_dim=64, tau=32, group_size=16, block_size=8, budget=80,
                                       levels=(16, 8, 4), psi_bits=(4, 8, 2), max_gen_len=360,
                                       script=script(2, 12, seed=5), record_events=True),
    # Qwen-14B G=5, raw 16-bit passthrough band + ternary, prompt prefix, tau % g != 0
    "qwen_raw16_prompt": ThinkvConfig(num_seqs=1, units_per_seq=3, num_q_heads=5, head_dim=128, tau=24,
                                      group_size=16, block_size=8, budget=60, levels=(12, 6, 3),
                                      psi_bits=(8, 16, 2), prompt_len=20, max_gen_len=300,
                                      script=script(1, 14, seed=9, pT=300), record_events=True),
    # per-layer labels (per_layer_thought, sim.cpp:713-716, :728-730): every layer
    # classifies its own sparsity, so layers of a sequence get different bands,
    # Case-1 transitions fire per layer and their segment sizes diverge
    "per_layer_calibrated": ThinkvConfig(num_seqs=2, units_per_seq=4, num_q_heads=4, head_dim=64, tau=32,
                                         group_size=16, block_size=16, budget=90, levels=(16, 8, 4),
                                         max_gen_len=400, scripted=False, thresholds=(0.965, 0.978),
                                         calib_units=(0, 2), per_layer_thought=True, record_events=True,
                                         dump_positions=(127, 255)),
    # calibrated labels from the fp64 sparsity kernel (refresh steps only)
    "calibrated": ThinkvConfig(num_seqs=2, units_per_seq=3, num_q_heads=4, head_dim=64, tau=32,
                               group_size=16, block_size=16, budget=90, levels=(16, 8, 4),
                               max_gen_len=400, scripted=False, thresholds=(0.25, 0.55),
                               calib_units=(0, 2), record_events=True),
}


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_parity_synthetic(name):
    cfg = CONFIGS[name]
    res = run_parity(cfg)
    compare_state(res, cfg)
    if cfg.per_layer_thought:  # the layers really got different labels
        ev = [json.loads(l) for l in res["run"].events(0).splitlines()]
        assert any(len(set(e["bands"])) > 1 for e in ev if e["type"] == "refresh")


def test_parity_full_tau_kmeans():
    """tau = 128 segments: the 128 -> 64 K-means with farthest-first restarts
    and the 8 -> 4 exhaustive-seed path, at the paper's schedule."""
    cfg = ThinkvConfig(num_seqs=1, units_per_seq=2, num_q_heads=4, head_dim=128, tau=128,
                       group_size=16, block_size=16, budget=400, levels=(64, 32, 16, 8, 4),
                       max_gen_len=1300, script=[[1, 0, 1, 0, 2, 1, 0, 1, 0, 1, 2]], record_events=True)
    res = run_parity(cfg, check_every=7)
    compare_state(res, cfg)


KMEANS_STRESS = {
    # many 128 -> 64 -> 32 -> 16 -> 8 -> 4 chains, FP8 band (scaled keys)
    "tau128_fp8": ThinkvConfig(num_seqs=2, units_per_seq=6, num_q_heads=4, head_dim=128, tau=128, group_size=16,
                               block_size=16, budget=300, levels=(64, 32, 16, 8, 4), psi_bits=(8, 4, 2),
                               max_gen_len=1450, script=script(2, 13, seed=21, pT=250), record_events=True),
    # tau = 96: 96 -> 64 -> 32 ... anneals (m not a power of two in the two-CTA class), block 8
    "tau96_m96": ThinkvConfig(num_seqs=2, units_per_seq=3, num_q_heads=4, head_dim=128, tau=96, group_size=16,
                              block_size=8, budget=260, levels=(64, 32, 16, 8, 4), psi_bits=(4, 8, 2),
                              max_gen_len=1100, script=script(2, 13, seed=29, pT=300), record_events=True),
    # d = 64, all bands quantised: the multi-CTA restart classes (means in global memory)
    "tau128_d64": ThinkvConfig(num_seqs=2, units_per_seq=4, num_q_heads=8, head_dim=64, tau=128, group_size=16,
                               block_size=16, budget=300, levels=(64, 32, 16, 8, 4), psi_bits=(4, 4, 2),
                               max_gen_len=1450, script=script(2, 13, seed=23, pT=250), record_events=True),
    # f32 inputs with a raw 16-bit band: f32 key store (fp32 means in global memory), d = 64
    "tau128_f32_raw": ThinkvConfig(num_seqs=1, units_per_seq=6, num_q_heads=8, gqa_maxpool=True, head_dim=64,
                                   tau=128, group_size=16, block_size=8, budget=300, levels=(64, 32, 16, 8, 4),
                                   psi_bits=(16, 4, 2), max_gen_len=1450, script=script(1, 13, seed=22, pT=250),
                                   input_dtype="f32", record_events=True),
}


@pytest.mark.parametrize("name", sorted(KMEANS_STRESS))
def test_parity_kmeans_stress(name):
    """Many full-size K-means chains: the approximate-distance cache with
    exact fallback must reproduce every medoid set of the reference."""
    from harness import synth_inputs
    cfg = KMEANS_STRESS[name]
    inputs = None
    if cfg.input_dtype != "bf16":
        inputs = lambda t: tuple(O.bf16_to_f64(x) for x in synth_inputs(cfg, 0x71534B56, t))  # noqa: E731
    res = run_parity(cfg, check_every=25, inputs=inputs)
    compare_state(res, cfg)


def test_block_start_list_at_capacity():
    """A block whose slots all belong to later segments keeps its implicit
    first segment too: bs + 1 start indices (pager.cpp:190-216).  When one
    more segment reuses a slot there, the reference appends its start and
    mask before pruning the emptied one, so the device arrays hold one extra
    start and mask transiently (TKV_STARTS_PER_BLOCK).  This configuration
    (block size 4, found by an oracle search) reaches bs + 1 starts by step
    275 and keeps churning; the step dumps prove it got there."""
    from paper_2510_01290_b200.synth import band_script
    cfg = ThinkvConfig(num_seqs=2, units_per_seq=2, num_q_heads=2, head_dim=32, tau=32, group_size=16,
                       block_size=4, budget=96, levels=(16, 8, 4), max_gen_len=900,
                       script=band_script(5, 2, 30, 3, 100), record_events=True,
                       dump_positions=tuple(range(250, 900, 5)))
    res = run_parity(cfg, check_every=4)
    dumps = res["run"].step_dumps(0)
    most = max(len(b["start_indices"]) for d in dumps.values() for t in d["block_tables"] for b in t["blocks"])
    assert most >= cfg.block_size + 1
    compare_state(res, cfg)


def test_pool_exhaustion_matches_reference_error():
    cfg = ThinkvConfig(num_seqs=1, units_per_seq=1, num_q_heads=2, head_dim=16, tau=16, group_size=8,
                       block_size=4, pool_blocks=3, budget=4096, levels=(8, 4), max_gen_len=64,
                       script=[[1]])
    with pytest.raises(O.OracleError) as oe:
        run_parity(cfg)
    assert oe.value.code == 4
    run = DecodeRun(cfg)
    dev = torch.device("cuda:0")
    q = torch.zeros((1, 2, 16), dtype=torch.bfloat16, device=dev)
    kv = torch.ones((1, 16), dtype=torch.bfloat16, device=dev)
    out = torch.empty((1, 2, 16), device=dev)
    for _ in range(64):
        run.step(q, kv, kv, out)
    with pytest.raises(TkvError) as ge:
        run.synchronize()
    assert ge.value.code == 4


def test_device_synth_matches_host_generator():
    """tkv_synth_inputs (device) == the oracle's generator for the same global
    units, so sharded runs (unit0 = rank offset) see the 1-GPU inputs."""
    cfg = ThinkvConfig(num_seqs=2, units_per_seq=3, num_q_heads=4, head_dim=64, tau=32, group_size=16,
                       block_size=16, budget=96, levels=(16, 8, 4), max_gen_len=64, script=[[1], [0]])
    run = DecodeRun(cfg)
    dev = torch.device("cuda:0")
    q = torch.empty((6, 4, 64), dtype=torch.bfloat16, device=dev)
    k = torch.empty((6, 64), dtype=torch.bfloat16, device=dev)
    v = torch.empty((6, 64), dtype=torch.bfloat16, device=dev)
    for unit0, step in ((0, 0), (0, 37), (12, 5), (6 * 1000, 129)):
        run.synth_inputs(0x71534B56, step, q, k, v, unit0=unit0)
        hq, hk, hv = O.synth_step(0x71534B56, 3, 32, 6, 4, 64, step, unit0=unit0)
        torch.cuda.synchronize()
        for got, want in ((q, hq), (k, hk), (v, hv)):
            assert np.array_equal(got.cpu().view(torch.int16).numpy().view(np.uint16), want)


def test_host_buffer_steps_match_device_steps():
    """tkv_step_host / tkv_step_host_async (staged uploads on a copy stream)
    produce the same outputs and cache state as device-pointer steps."""
    cfg = ThinkvConfig(num_seqs=2, units_per_seq=2, num_q_heads=4, head_dim=128, tau=32, group_size=16,
                       block_size=16, budget=64, levels=(16, 8, 4), max_gen_len=200, script=script(2, 8),
                       record_events=True)
    dev = torch.device("cuda:0")
    a, b, c = DecodeRun(cfg), DecodeRun(cfg), DecodeRun(cfg)
    out = torch.empty((cfg.units, 4, 128), device=dev)
    outs_b = [torch.empty((cfg.units, 4, 128)).pin_memory() for _ in range(2)]
    out_c = torch.empty((cfg.units, 4, 128)).pin_memory()
    for t in range(cfg.max_gen_len):
        q, k, v = O.synth_step(0x71534B56, cfg.units_per_seq, cfg.tau, cfg.units, 4, 128, t)
        tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16) for x in (q, k, v))
        a.step(tq.to(dev), tk.to(dev), tv.to(dev), out)
        pq, pk, pv = tq.pin_memory(), tk.pin_memory(), tv.pin_memory()
        b.step_host_async(pq, pk, pv, outs_b[t % 2])
        c.step_host(tq.contiguous(), tk.contiguous(), tv.contiguous(), out_c)
        b.synchronize()  # pq/pk/pv are released at the end of the iteration
        ref = out.cpu()
        assert torch.equal(outs_b[t % 2], ref)
        assert torch.equal(out_c, ref)
    for r in (a, b, c):
        r.finish()
    for s in range(2):
        assert b.tables(s) == a.tables(s) and c.tables(s) == a.tables(s)
        assert b.events(s) == a.events(s)


def test_parity_cta_per_unit_attention_variant(monkeypatch):
    """The CTA-per-unit K1 variant (used when slot ids exceed 16 bits) stays
    parity-green: forced here through TKV_K1_V2 on a small configuration."""
    monkeypatch.setenv("TKV_K1_V2", "1")
    cfg = CONFIGS["llama_shape"]
    res = run_parity(cfg, check_every=3)
    compare_state(res, cfg)


def test_parity_generic_kmeans_for_tiny_instances(monkeypatch):
    """Instances with m <= 8 normally run the subset-table kernel; the generic
    restart kernel must give the same (reference) decisions."""
    monkeypatch.setenv("TKV_KM_NO_TINY", "1")
    cfg = CONFIGS["llama_shape"]
    res = run_parity(cfg, check_every=5)
    compare_state(res, cfg)


def test_parity_warp_per_restart_kmeans_for_tiny_instances(monkeypatch):
    """TKV_KM_NO_TABLE: the warp-per-restart m <= 8 kernel (km_tiny) instead
    of the subset-table kernel."""
    monkeypatch.setenv("TKV_KM_NO_TABLE", "1")
    cfg = CONFIGS["llama_shape"]
    res = run_parity(cfg, check_every=5)
    compare_state(res, cfg)


@pytest.mark.parametrize("maxpool", [False, True])
def test_layer_by_layer_stepping_matches_full_steps(maxpool):
    """tkv_step_layer (a model's per-layer decode loop) gives bit-identical
    outputs and cache state to whole-step tkv_step on the same inputs."""
    L, H, S, G, D = 3, 2, 2, 4, 128
    cfg = ThinkvConfig(num_seqs=S, units_per_seq=L * H, num_q_heads=G, gqa_maxpool=maxpool, head_dim=D, tau=32,
                       group_size=16, block_size=16, budget=80, levels=(16, 8, 4), max_gen_len=300,
                       script=script(S, 12, seed=11), record_events=True)
    dev = torch.device("cuda:0")
    a, b = DecodeRun(cfg), DecodeRun(cfg)
    rows = cfg.out_rows
    out_a = torch.empty((cfg.units, rows, D), device=dev)
    out_b = torch.empty((S, L, H, rows, D), device=dev)
    for t in range(cfg.max_gen_len):
        q, k, v = O.synth_step(0x71534B56, cfg.units_per_seq, cfg.tau, cfg.units, G, D, t)
        tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
        a.step(tq, tk, tv, out_a)
        q5, k5, v5 = tq.view(S, L, H, G, D), tk.view(S, L, H, D), tv.view(S, L, H, D)
        for l in range(L):
            ol = torch.empty((S, H, rows, D), device=dev)
            b.step_layer(l, L, q5[:, l].contiguous(), k5[:, l].contiguous(), v5[:, l].contiguous(), ol)
            out_b[:, l] = ol
        assert torch.equal(out_b.reshape(cfg.units, rows, D), out_a), f"step {t}"
    a.finish()
    b.finish()
    for s in range(S):
        assert b.tables(s) == a.tables(s)
        assert b.segments(s) == a.segments(s)
        assert b.events(s) == a.events(s)
        assert b.metrics(s) == a.metrics(s)


def test_sparsity_trace_matches_reference_every_step():
    """record_sparsity_trace: the exact per-unit layer_sparsity_average of
    every decode step (the reference computes it each step, sim.cpp:779),
    exported in calibration-trace JSONL form (thought.cpp:66-75)."""
    cfg = ThinkvConfig(num_seqs=2, units_per_seq=3, num_q_heads=4, head_dim=64, tau=32, group_size=16,
                       block_size=16, budget=90, levels=(16, 8, 4), prompt_len=8, max_gen_len=200,
                       script=script(2, 8, seed=4), record_sparsity_trace=True)
    run = DecodeRun(cfg)
    orc = O.OracleRun(harness_oracle_config(cfg))
    dev = torch.device("cuda:0")
    out = torch.empty((cfg.units, 4, 64), device=dev)
    ref = []
    for t in range(cfg.prompt_len + cfg.max_gen_len):
        q, k, v = O.synth_step(0x71534B56, cfg.units_per_seq, cfg.tau, cfg.units, 4, 64, t)
        _, sp = orc.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
        if t >= cfg.prompt_len:
            ref.append(sp.copy())
        tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
        run.step(tq, tk, tv, out)
    ref = np.array(ref)  # [decode steps, units]
    for s in range(2):
        rec = json.loads(run.sparsity_trace(s))
        assert sorted(rec, key=int) == ["0", "1", "2"]
        for u in range(3):
            got = np.array(rec[str(u)])
            assert got.shape == (cfg.max_gen_len,)
            assert np.array_equal(got, ref[:, s * 3 + u]), f"seq {s} unit {u}"


def test_export_edge_cases():
    """Compressed-cache export: empty cache (before the first emission), a
    unit sub-range, mid-run exports (partial windows, evicted and reused
    slots) byte-equal to the oracle's, and the too-small-buffer error."""
    import ctypes as C
    from paper_2510_01290_b200 import _abi, wire
    cfg = ThinkvConfig(num_seqs=2, units_per_seq=3, num_q_heads=4, head_dim=64, tau=32, group_size=16,
                       block_size=8, budget=40, levels=(16, 8, 4), psi_bits=(8, 4, 2), max_gen_len=200,
                       script=script(2, 8, seed=17, pT=300))
    run = DecodeRun(cfg)
    orc = O.OracleRun(harness_oracle_config(cfg))
    dev = torch.device("cuda:0")
    out = torch.empty((cfg.units, 4, 64), device=dev)
    buf, offs = run.export_cache()
    assert offs.tolist() == [12 * u for u in range(cfg.units + 1)]  # headers only
    for u in range(cfg.units):
        recs, used = wire.parse_unit(buf.cpu().numpy().tobytes()[offs[u]:offs[u + 1]])
        assert recs == [] and used == 12
    for t in range(cfg.max_gen_len):
        q, k, v = O.synth_step(0x71534B56, cfg.units_per_seq, cfg.tau, cfg.units, 4, 64, t)
        orc.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
        tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
        run.step(tq, tk, tv, out)
        if t in (15, 16, 47, 120, 199):
            buf, offs = run.export_cache(unit0=2, nunits=3)
            host = buf.cpu().numpy().tobytes()
            for j, u in enumerate(range(2, 5)):
                assert host[offs[j]:offs[j + 1]] == orc.export(u // 3, u % 3), f"step {t} unit {u}"
    need = C.c_size_t(0)
    small = torch.empty(8, dtype=torch.uint8, device=dev)
    rc = _abi.lib.tkv_export_cache(run._h, 0, cfg.units, small.data_ptr(), 8, None, C.byref(need))
    assert rc == 2 and need.value > 8


@pytest.mark.parametrize("D,maxpool", [(128, False), (64, True)])
def test_immediate_and_runtime_slot_stride_k1_agree(monkeypatch, D, maxpool):
    """K1's immediate slot-row stride instantiation (widest band 4-bit, the
    BASELINE configs 2-4) and its runtime-stride form (TKV_K1_RUNTIME_STRIDE)
    compute bit-identical outputs and leave identical cache state."""
    S, U, G = 2, 3, 8 if maxpool else 4
    cfg = ThinkvConfig(num_seqs=S, units_per_seq=U, num_q_heads=G, gqa_maxpool=maxpool, head_dim=D, tau=32,
                       group_size=16, block_size=16, budget=80, levels=(16, 8, 4), psi_bits=(4, 4, 2),
                       max_gen_len=260, script=script(S, 10, seed=5), record_events=True)
    dev = torch.device("cuda:0")
    a, b = DecodeRun(cfg), DecodeRun(cfg)
    out_a = torch.empty((cfg.units, cfg.out_rows, D), device=dev)
    out_b = torch.empty_like(out_a)
    for t in range(cfg.max_gen_len):
        q, k, v = O.synth_step(0x71534B56, cfg.units_per_seq, cfg.tau, cfg.units, G, D, t)
        tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
        monkeypatch.delenv("TKV_K1_RUNTIME_STRIDE", raising=False)
        a.step(tq, tk, tv, out_a)
        monkeypatch.setenv("TKV_K1_RUNTIME_STRIDE", "1")
        b.step(tq, tk, tv, out_b)
        assert torch.equal(out_a, out_b), f"step {t}"
    a.finish()
    b.finish()
    for s in range(S):
        assert b.tables(s) == a.tables(s)
        assert b.segments(s) == a.segments(s)
