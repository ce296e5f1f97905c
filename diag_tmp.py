import json, sys, os
sys.path.insert(0, "tests"); sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import numpy as np, torch
import oracle as O
from harness import unit_subset_config, oracle_config
from test_gpu_configs import baseline_config
from paper_2510_01290_b200 import DecodeRun
cfg = baseline_config(2)
u = int(sys.argv[1]) if len(sys.argv) > 1 else 0
dumps = tuple(range(127, 32768, 128))
sub = unit_subset_config(cfg, [u])
import dataclasses
sub = dataclasses.replace(sub, dump_positions=dumps)
run = DecodeRun(sub)
orc = O.OracleRun(oracle_config(sub))
dev = torch.device("cuda:0")
out = torch.empty((1, 4, 128), device=dev)
for t in range(32768):
    q, k, v = O.synth_step(0x71534B56, cfg.units_per_seq, 128, 1, 4, 128, t, unit0=u)
    orc.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
    tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
    run.step(tq, tk, tv, out)
G = run.step_dumps(0); R = orc.dump(0, "step_dumps")
for t in dumps:
    g, o = G[str(t)], R[str(t)]
    if g == o:
        continue
    print("first difference at", t)
    for key in ("block_tables", "segments"):
        if g[key] != o[key]:
            gt, ot = g[key][0], o[key][0]
            if key == "block_tables":
                print("free", gt["free_blocks"] == ot["free_blocks"], len(gt["blocks"]), len(ot["blocks"]))
                n = 0
                for a, b in zip(gt["blocks"], ot["blocks"]):
                    if a != b:
                        print("GPU", json.dumps(a)); print("REF", json.dumps(b)); n += 1
                        if n > 3: break
            else:
                for a, b in zip(gt, ot):
                    if a != b:
                        print("GPU", json.dumps(a)); print("REF", json.dumps(b)); break
    break
ev_g = run.events(0).splitlines(); ev_o = orc.dump(0, "events").splitlines()
for i, (a, b) in enumerate(zip(ev_g, ev_o)):
    if a != b:
        print("event", i); print("GPU", a[:600]); print("REF", b[:600]); break
print("done", t)
