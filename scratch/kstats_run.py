"""K-means phase statistics at the config-2 unit shape (TKV_KSTATS=1):
a reduced batch decoded to `steps`, kstats + per-kernel timing per tau period."""
import os, sys, time
if "nostats" not in sys.argv: os.environ.setdefault("TKV_KSTATS", "1")
sys.path[:0] = ['.']
import torch
from paper_2510_01290_b200 import DecodeRun, ThinkvConfig
from paper_2510_01290_b200.synth import band_script
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nseq = int(sys.argv[2]) if len(sys.argv) > 2 else 4
script = band_script(0x71534B56, nseq, steps // 128 + 2, 3, 100)
cfg = ThinkvConfig(num_seqs=nseq, units_per_seq=256, num_q_heads=4, head_dim=128, tau=128, group_size=16,
                   block_size=16, budget=1024, levels=(64, 32, 16, 8, 4), psi_bits=(4, 4, 2),
                   max_gen_len=32768, script=script)
run = DecodeRun(cfg)
dev = torch.device('cuda')
U = cfg.units
q = torch.empty((U, 4, 128), dtype=torch.bfloat16, device=dev)
k = torch.empty((U, 128), dtype=torch.bfloat16, device=dev)
v = torch.empty((U, 128), dtype=torch.bfloat16, device=dev)
out = torch.empty((U, 4, 128), dtype=torch.float32, device=dev)
run.timing_enable(True)
for t in range(steps):
    run.synth_inputs(0x71534B56, t, q, k, v)
    run.step(q, k, v, out)
    if (t + 1) % 128 == 0 and t >= 1024:
        tm = run.timing_read()
        print(f"steps {t-127}..{t}: " + " ".join(f"{n}={tm[n]:.2f}" for n in ("attend_ms", "score_ms", "flush_ms", "anneal_ms", "apply_ms")) + f" anneal_launches={tm['anneal_launches']}", flush=True)
        run.timing_enable(True)
    elif (t + 1) % 128 == 0:
        run.timing_read(); run.timing_enable(True)
