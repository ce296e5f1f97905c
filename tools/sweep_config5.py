"""BASELINE config 5: eviction-stress sweep -- KV budget 2-20% of a 32K
generation x thought-switch rate -- timing ThinKV slot reuse against the
gather-compaction comparator (GatherMethod, proj/src/sim.cpp:1117-1206) on the
same synthetic inputs at the R1-Llama-8B head shape.

Each point builds the cache to `budget + 2*tau` decode steps (the cache is
full and evicting from then on), then times `--steps` steps of each method
with CUDA events (device time, inputs resident).  Reduced batch (--seqs
sequences x 32 layers x 8 kv heads) keeps the sweep to minutes; the per-unit
work per step is the full-size workload's.  Prints one JSON line per point and
writes profiles/config5_sweep.json when --out is given.

  python sweep_config5.py [--seqs 4] [--steps 64] [--out profiles/r01_config5_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SEED = 0x71534B56


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=4)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--budgets", type=int, nargs="*", default=[655, 1638, 3277, 6554])
    ap.add_argument("--pts", type=int, nargs="*", default=[0, 100, 200, 400], help="p_T in permille")
    ap.add_argument("--exact-gather", action="store_true", help="fp64 victim scores (reference-exact)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    from paper_2510_01290_b200 import DecodeRun, GatherRun, ThinkvConfig
    from paper_2510_01290_b200.synth import band_script
    dev = torch.device("cuda:0")
    U, G, D, tau = args.seqs * args.layers * 8, 4, 128, 128
    q = torch.empty((U, G, D), dtype=torch.bfloat16, device=dev)
    k = torch.empty((U, D), dtype=torch.bfloat16, device=dev)
    v = torch.empty((U, D), dtype=torch.bfloat16, device=dev)
    out = torch.empty((U, G, D), dtype=torch.float32, device=dev)
    results = []

    def timed(step_fn, run_synth, t0, n):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        qs = torch.empty((n, U, G, D), dtype=torch.bfloat16, device=dev)
        ks = torch.empty((n, U, D), dtype=torch.bfloat16, device=dev)
        vs = torch.empty((n, U, D), dtype=torch.bfloat16, device=dev)
        for i in range(n):
            run_synth(SEED, t0 + i, qs[i], ks[i], vs[i])
        torch.cuda.synchronize()
        ev0.record()
        for i in range(n):
            step_fn(qs[i], ks[i], vs[i], out)
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / n

    for budget in args.budgets:
        ctx = budget + 2 * tau
        # gather comparator (independent of p_T: it has no thought types)
        g = GatherRun(U, G, D, budget, exact=args.exact_gather)
        th0 = DecodeRun(ThinkvConfig(num_seqs=args.seqs, units_per_seq=args.layers * 8, num_q_heads=G, head_dim=D,
                                     tau=tau, group_size=16, block_size=16, budget=budget, max_gen_len=ctx + 1024,
                                     script=[[1]] * args.seqs))  # only for its synth kernel
        t0 = time.time()
        for t in range(ctx):
            th0.synth_inputs(SEED, t, q, k, v)
            g.step(q, k, v, out)
        g_ms = timed(lambda a, b, c, o: g.step(a, b, c, o), th0.synth_inputs, ctx, args.steps)
        gstats = g.stats()
        del g
        for pt in args.pts:
            script = band_script(SEED, args.seqs, (ctx + 1024) // tau + 2, 3, pt)
            cfg = ThinkvConfig(num_seqs=args.seqs, units_per_seq=args.layers * 8, num_q_heads=G, head_dim=D, tau=tau,
                               group_size=16, block_size=16, budget=budget, levels=(64, 32, 16, 8, 4),
                               psi_bits=(4, 4, 2), max_gen_len=ctx + 1024, script=script)
            run = DecodeRun(cfg)
            for t in range(ctx):
                run.synth_inputs(SEED, t, q, k, v)
                run.step(q, k, v, out)
            n = max(args.steps, tau)  # whole tau periods: every timed window holds one eviction wave
            th_ms = timed(lambda a, b, c, o: run.step(a, b, c, o), run.synth_inputs, ctx, n)
            line = {"budget": budget, "budget_frac_of_32k": budget / 32768, "p_T": pt / 1000, "units": U,
                    "thinkv_ms_per_step": th_ms, "gather_ms_per_step": g_ms,
                    "thinkv_tokens_per_s": args.seqs / (th_ms / 1e3), "gather_tokens_per_s": args.seqs / (g_ms / 1e3),
                    "speedup": g_ms / th_ms, "gather_exact_scores": args.exact_gather,
                    "gather_moved_slots_per_unit_step": gstats["moved_token_slots"] / max(1, gstats["eviction_steps"]) / U,
                    "build_s": time.time() - t0}
            print(json.dumps(line), flush=True)
            results.append(line)
            del run
        del th0
    if args.out:
        with open(os.path.join(ROOT, args.out), "w") as f:
            json.dump({"what": "BASELINE config 5 sweep (tools/sweep_config5.py)", "points": results}, f, indent=1)


if __name__ == "__main__":
    main()
