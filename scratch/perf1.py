import sys, time, numpy as np, torch
sys.path[:0] = ['.', 'oracle', 'tests']
from paper_2510_01290_b200 import DecodeRun, ThinkvConfig

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
nseq = int(sys.argv[2]) if len(sys.argv) > 2 else 32
rng = np.random.default_rng(1)
script = [[2 if rng.random() < 0.1 else int(rng.integers(0, 2)) for _ in range(300)] for _ in range(nseq)]
cfg = ThinkvConfig(num_seqs=nseq, units_per_seq=256, num_q_heads=4, head_dim=128, tau=128, group_size=16,
                   block_size=16, budget=1024, levels=(64, 32, 16, 8, 4), psi_bits=(4, 4, 2),
                   max_gen_len=32768, script=script)
t0 = time.time()
run = DecodeRun(cfg)
print("create", time.time() - t0, flush=True)
dev = torch.device('cuda')
U = cfg.units
q = torch.empty((U, 4, 128), dtype=torch.bfloat16, device=dev)
k = torch.empty((U, 128), dtype=torch.bfloat16, device=dev)
v = torch.empty((U, 128), dtype=torch.bfloat16, device=dev)
out = torch.empty((U, 4, 128), dtype=torch.float32, device=dev)
run.timing_enable(True)
t0 = time.time()
for t in range(steps):
    run.synth_inputs(7, t, q, k, v)
    run.step(q, k, v, out)
    if (t + 1) % 250 == 0:
        tm = run.timing_read()
        torch.cuda.synchronize()
        el = time.time() - t0
        print(f"step {t+1}: wall {el:.2f}s ({el/250*1e3:.2f} ms/step) " +
              " ".join(f"{n}={tm[n]/250:.3f}" for n in ("attend_ms", "score_ms", "flush_ms", "anneal_ms", "apply_ms")) +
              f" anneal_launches={tm['anneal_launches']}", flush=True)
        run.timing_enable(True)
        t0 = time.time()
b = run.bytes()
print(b)
print("live/unit", b['live_slots'] / U, "bytes/live", b['algorithmic_bytes'] / max(1, b['live_slots']))
