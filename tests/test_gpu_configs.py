"""GPU parity at the BASELINE configurations themselves (BASELINE.json
configs[0] and configs[1]), not just at small shapes: the CUDA decode path
against the oracle (the reference's ThinkvMethod restated over the compiled
reference library, /root/reference/proj/src/sim.cpp:748-843) on identical
inputs, over the full generation length.

Cache state (block tables, segments, events, compressed-cache bytes, byte
accounting, metrics) must be identical; attention within harness.ATOL/RTOL.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
from harness import (compare_state, compare_units_state, run_parity, run_parity_units,  # noqa: E402
                     synth_inputs)
from paper_2510_01290_b200 import DecodeRun, ThinkvConfig  # noqa: E402
from paper_2510_01290_b200.synth import band_script  # noqa: E402

SEED = 0x71534B56


def baseline_config(n):
    """bench.py's PRESETS[n] as a ThinkvConfig (the same script generator)."""
    import bench
    p = bench.PRESETS[n]
    gen = p["max_gen"]
    return ThinkvConfig(num_seqs=p["seqs"], units_per_seq=p["layers"] * p["kv_heads"], num_q_heads=p["q_per_kv"],
                        head_dim=p["head_dim"], tau=128, group_size=16, block_size=p["block_size"],
                        budget=p["budget"], levels=(64, 32, 16, 8, 4), psi_bits=tuple(p["psi"]), max_gen_len=gen,
                        script=band_script(SEED, p["seqs"], gen // 128 + 2, 3, 100), record_events=True)


def test_baseline_config1_full_run():
    """configs[0]: 1 sequence x 8 KV heads, d=128, G=4 per-head, 4096 generated
    tokens, R8E4T2, budget 204 (5%), block 16 -- the CPU-reference run, every
    step, every output compared."""
    cfg = baseline_config(1)
    assert (cfg.units, cfg.max_gen_len, cfg.budget, tuple(cfg.psi_bits)) == (8, 4096, 204, (4, 8, 2))
    res = run_parity(cfg)
    compare_state(res, cfg)


def test_baseline_config2_units_over_the_whole_32k():
    """configs[1] (the benchmarked configuration: bs 32 x 32 layers x 8 KV
    heads, d=128, G=4, 32K generated, budget 1024, R4E4T2, block 16): 16
    units spread over the batch (different sequences, layers and heads),
    decoded over all 32768 steps -- 256 segments per unit, the infeasible
    budget with its 128 -> 64 -> ... -> 4 anneal chain at every boundary.
    Outputs compared every 97th step and over the last 130 steps."""
    cfg = baseline_config(2)
    assert (cfg.units, cfg.max_gen_len, cfg.budget) == (8192, 32768, 1024)
    units = [i * (cfg.units // 16) + (i * 37) % cfg.units_per_seq for i in range(16)]
    check = set(range(0, cfg.max_gen_len, 97)) | set(range(cfg.max_gen_len - 130, cfg.max_gen_len))
    res = run_parity_units(cfg, units, check=check)
    compare_units_state(res)


@pytest.mark.parametrize("n", [3, 4])
def test_baseline_configs_3_and_4_units_over_the_whole_generation(n):
    """configs[2] (GPT-OSS-20B shape: d=64, G=8 per-head, 24 layers, 32K
    generated, budget 1024) and configs[3] (R1-Distill-Qwen-14B shape: G=5,
    48 layers, 16K generated, budget 819 = 5%): 8 units spread over each
    batch decoded over the whole generation against the oracle -- the head
    shapes of the bench lines, at their full lengths and budgets."""
    cfg = baseline_config(n)
    assert (cfg.head_dim, cfg.num_q_heads) == ((64, 8) if n == 3 else (128, 5))
    units = [i * (cfg.units // 8) + (i * 29) % cfg.units_per_seq for i in range(8)]
    check = set(range(0, cfg.max_gen_len, 211)) | set(range(cfg.max_gen_len - 130, cfg.max_gen_len))
    res = run_parity_units(cfg, units, check=check)
    compare_units_state(res)


def test_f64_inputs_with_raw16_band():
    """f64 inputs with a 16-bit passthrough band: the raw fp64 keys take the
    fp64-key anneal kernel (k_evict.cu anneal_kernel) -- the configuration a
    C++ drop-in caller with double vectors uses."""
    cfg = ThinkvConfig(num_seqs=2, units_per_seq=3, num_q_heads=4, head_dim=64, tau=128, group_size=16,
                       block_size=8, budget=300, levels=(64, 32, 16, 8, 4), psi_bits=(4, 16, 2),
                       max_gen_len=1450, script=[[1, 0, 1, 2, 1, 1, 0, 2, 1, 1, 0, 1, 1],
                                                 [1, 1, 2, 1, 0, 1, 1, 1, 2, 0, 1, 1, 1]],
                       input_dtype="f64", record_events=True)

    def inputs(t):
        q, k, v = synth_inputs(cfg, SEED, t)
        rng = np.random.default_rng(t)  # full-width doubles (not bf16-representable)
        return tuple(O.bf16_to_f64(x) * (1 + 1e-6 * rng.standard_normal(x.shape)) for x in (q, k, v))

    res = run_parity(cfg, check_every=9, inputs=inputs)
    compare_state(res, cfg)


def test_device_byte_accounting_matches_host_walk():
    """k_bytes.cu (the bench's per-launch roofline numerator) == tkv_bytes'
    host walk of the same state, field by field, at steps around emissions,
    boundaries and evictions."""
    cfg = ThinkvConfig(num_seqs=2, units_per_seq=3, num_q_heads=4, head_dim=128, tau=32, group_size=16,
                       block_size=16, budget=64, levels=(16, 8, 4), psi_bits=(4, 8, 2), max_gen_len=300,
                       script=band_script(SEED, 2, 12, 3, 300))
    run = DecodeRun(cfg)
    dev = torch.device("cuda:0")
    out = torch.empty((cfg.units, 4, 128), device=dev)
    checked = 0
    for t in range(cfg.max_gen_len):
        q, k, v = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev)
                   for x in synth_inputs(cfg, SEED, t))
        probe = t % 29 == 0 or t % 32 in (0, 1, 15, 16)
        if probe:
            want = run.bytes()
            run.bytes_accounting(True)
        run.step(q, k, v, out)
        if probe:
            got, n = run.bytes_accumulated()
            run.bytes_accounting(False)
            assert n == 1 and got == want, f"step {t}: {got} != {want}"
            checked += 1
    assert checked > 20


def test_device_byte_accounting_over_a_long_window():
    """One accounting window over many steps (emissions, boundaries and
    evictions inside it, runs of launches on unchanged pager state that reuse
    the previous counts, k_bytes.cu) == the sum of the host walk before every
    step; full steps and layer-by-layer launches mixed."""
    cfg = ThinkvConfig(num_seqs=2, units_per_seq=4, num_q_heads=4, head_dim=128, tau=32, group_size=16,
                       block_size=16, budget=64, levels=(16, 8, 4), psi_bits=(4, 8, 2), max_gen_len=260,
                       script=band_script(SEED, 2, 12, 3, 300))
    run = DecodeRun(cfg)
    dev = torch.device("cuda:0")
    L, H = 2, 2  # units_per_seq = layers x kv-heads
    out = torch.empty((cfg.units, 4, 128), device=dev)
    lout = torch.empty((cfg.num_seqs * H, 4, 128), device=dev)
    start = 70
    for t in range(start):
        q, k, v = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev)
                   for x in synth_inputs(cfg, SEED, t))
        run.step(q, k, v, out)
    want = None
    run.bytes_accounting(True)
    for t in range(start, cfg.max_gen_len):
        q, k, v = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev)
                   for x in synth_inputs(cfg, SEED, t))
        b = run.bytes()
        want = b if want is None else {f: want[f] + b[f] for f in want}
        if 150 <= t < 170:  # layer by layer: units [seq][layer][head]
            qv, kv, vv = (x.view(cfg.num_seqs, L, H, *x.shape[1:]) for x in (q, k, v))
            for layer in range(L):
                run.step_layer(layer, L, qv[:, layer].contiguous().view(-1, *q.shape[1:]),
                               kv[:, layer].contiguous().view(-1, *k.shape[1:]),
                               vv[:, layer].contiguous().view(-1, *v.shape[1:]), lout)
        else:
            run.step(q, k, v, out)
    got, n = run.bytes_accumulated()
    run.bytes_accounting(False)
    assert n == cfg.max_gen_len - start
    assert got == want
