"""Large-sample GPU parity at a BASELINE configuration: K units spread over
the batch (different sequences, layers and heads) decoded over the whole
generation on the GPU and, one unit per thread, by the oracle (the
reference's ThinkvMethod over the compiled reference library).  Block
tables, segments, events, exported compressed-cache bytes, byte accounting
and metrics must be identical; outputs within the harness tolerance at the
checked positions.  Prints one JSON line.

  python tools/parity_units.py --config 2 --units 128
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--units", type=int, default=128)
    args = ap.parse_args()
    from harness import compare_units_state, run_parity_units
    from test_gpu_configs import baseline_config
    cfg = baseline_config(args.config)
    n = min(args.units, cfg.units)
    units = sorted({(i * cfg.units) // n + (i * 37) % min(cfg.units_per_seq, max(1, cfg.units // n)) for i in range(n)})
    check = set(range(0, cfg.max_gen_len, 257)) | set(range(cfg.max_gen_len - 64, cfg.max_gen_len))
    t0 = time.time()
    res = run_parity_units(cfg, units, check=check)
    compare_units_state(res)
    boundaries = cfg.max_gen_len // cfg.tau
    print(json.dumps({"config": args.config, "units": len(units), "unit_ids": units, "steps": res["steps"],
                      "refresh_boundaries_per_unit": boundaries, "max_err": res["max_err"],
                      "checked_positions": len(check), "state_bit_exact": True,
                      "compared": "block tables, segments, events, compressed-cache export bytes, byte accounting, "
                                  "metrics (exact); outputs within 1e-3 + 1e-3 max|ref| at the checked positions",
                      "wall_s": time.time() - t0}), flush=True)


if __name__ == "__main__":
    main()
