"""Small decode runs for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the decode path on tiny configurations,
each run checked against the oracle at the end so a sanitizer-visible fault
that changes results is also caught.

  compute-sanitizer --tool racecheck python tools/sanitize_run.py [names...]

Configurations: smoke (tau 32, levels 16/8/4: K1, K2, K3a, the table K-means,
the 16-point restart class), tau128 (the 128 -> 64 -> ... -> 4 chain: prep,
the two-CTA 128-point class, 64/32/16 classes, table kernel), d64 (d = 64
multi-CTA classes, maxpool), f32raw (f32 key store, single-CTA restart
kernels, raw band), tiny (the warp-per-restart 8 -> 4 kernel), gather
(the gather-compaction comparator).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from harness import compare_state, run_parity, synth_inputs  # noqa: E402
from paper_2510_01290_b200 import ThinkvConfig  # noqa: E402
from paper_2510_01290_b200.synth import band_script  # noqa: E402

CONFIGS = {
    "smoke": ThinkvConfig(num_seqs=1, units_per_seq=2, num_q_heads=4, head_dim=128, tau=32, group_size=16,
                          block_size=16, budget=64, levels=(16, 8, 4), max_gen_len=140,
                          script=[[1, 0, 2, 1, 0]], record_events=True),
    "tau128": ThinkvConfig(num_seqs=1, units_per_seq=2, num_q_heads=4, head_dim=128, tau=128, group_size=16,
                           block_size=16, budget=140, levels=(64, 32, 16, 8, 4), max_gen_len=400,
                           script=[[1, 1, 1, 1, 1]], record_events=True),
    "d64": ThinkvConfig(num_seqs=1, units_per_seq=2, num_q_heads=8, gqa_maxpool=True, head_dim=64, tau=128,
                        group_size=16, block_size=16, budget=140, levels=(64, 32, 16, 8, 4), psi_bits=(4, 4, 2),
                        max_gen_len=400, script=[[1, 0, 1, 1, 1]], record_events=True),
    "f32raw": ThinkvConfig(num_seqs=1, units_per_seq=2, num_q_heads=8, head_dim=64, tau=128, group_size=16,
                           block_size=8, budget=140, levels=(64, 32, 16, 8, 4), psi_bits=(16, 4, 2),
                           max_gen_len=400, script=[[1, 1, 0, 1, 1]], input_dtype="f32", record_events=True),
}


def run_config(name):
    cfg = CONFIGS[name]
    inputs = None
    if cfg.input_dtype != "bf16":
        inputs = lambda t: tuple(O.bf16_to_f64(x) for x in synth_inputs(cfg, 0x71534B56, t))  # noqa: E731
    res = run_parity(cfg, check_every=37, inputs=inputs)
    compare_state(res, cfg)
    print(f"{name}: ok ({res['steps']} steps, max |err| {res['max_err']:.2e})", flush=True)


def run_tiny():
    os.environ["TKV_KM_NO_TABLE"] = "1"  # read at launch: the warp-per-restart m <= 8 kernel
    try:
        run_config("smoke")
    finally:
        del os.environ["TKV_KM_NO_TABLE"]


def run_gather():
    import torch
    from paper_2510_01290_b200 import GatherRun
    units, G, D, budget = 4, 4, 128, 48
    run = GatherRun(units, G, D, budget, exact=True)
    dev = torch.device("cuda:0")
    out = torch.empty((units, G, D), device=dev)
    rng = np.random.default_rng(5)
    for t in range(120):
        q, k, v = (torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(dev, torch.bfloat16)
                   for s in ((units, G, D), (units, D), (units, D)))
        run.step(q, k, v, out)
    torch.cuda.synchronize()
    print("gather: ok", run.stats(), flush=True)


def run_graph():
    """CUDA-graph replay of plain steps (tkv_step_plain / tkv_graph_step_begin),
    2 layers, final state against the oracle."""
    import torch
    from harness import oracle_config
    from paper_2510_01290_b200 import DecodeRun
    cfg = CONFIGS["smoke"]
    L, S, H, G, D = 2, 1, 1, 4, 128
    run = DecodeRun(cfg)
    orc = O.OracleRun(oracle_config(cfg))
    dev = torch.device("cuda:0")
    qs = [torch.empty((S, H, G, D), dtype=torch.bfloat16, device=dev) for _ in range(L)]
    ks = [torch.empty((S, H, D), dtype=torch.bfloat16, device=dev) for _ in range(L)]
    vs = [torch.empty((S, H, D), dtype=torch.bfloat16, device=dev) for _ in range(L)]
    os_ = [torch.empty((S, H, G, D), dtype=torch.float32, device=dev) for _ in range(L)]
    stream, graphs, replays = torch.cuda.Stream(), {}, 0
    with torch.cuda.stream(stream):
        for t in range(cfg.max_gen_len):
            q, k, v = synth_inputs(cfg, 0x71534B56, t)
            orc.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
            tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
            for l in range(L):
                qs[l].copy_(tq.view(S, L, H, G, D)[:, l])
                ks[l].copy_(tk.view(S, L, H, D)[:, l])
                vs[l].copy_(tv.view(S, L, H, D)[:, l])
            kind = run.step_kind()
            if kind:
                if kind not in graphs:
                    graphs[kind] = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graphs[kind]):
                        for l in range(L):
                            run.step_layer(l, L, qs[l], ks[l], vs[l], os_[l])
                run.graph_step_begin()
                graphs[kind].replay()
                replays += 1
            else:
                for l in range(L):
                    run.step_layer(l, L, qs[l], ks[l], vs[l], os_[l])
    torch.cuda.synchronize()
    compare_state({"run": run, "oracle": orc}, cfg)
    print(f"graph: ok ({replays} replayed steps of {cfg.max_gen_len})", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or ["smoke", "tau128", "d64", "f32raw", "tiny", "gather", "graph"]
    for n in names:
        if n == "tiny":
            run_tiny()
        elif n == "gather":
            run_gather()
        elif n == "graph":
            run_graph()
        else:
            run_config(n)
