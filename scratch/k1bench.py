"""K1 variant microbenchmark at the config-2 shape: decode to `ctx`, then time
the attention kernel per variant (env switches read at launch)."""
import os, sys, time
sys.path[:0] = ['.']
import torch
from paper_2510_01290_b200 import DecodeRun, ThinkvConfig
from paper_2510_01290_b200.synth import band_script
ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 2600
variants = sys.argv[2].split(',') if len(sys.argv) > 2 else ['v2', 'v3']
script = band_script(0x71534B56, 32, 300, 3, 100)
cfg = ThinkvConfig(num_seqs=32, units_per_seq=256, num_q_heads=4, head_dim=128, tau=128, group_size=16,
                   block_size=16, budget=1024, levels=(64, 32, 16, 8, 4), psi_bits=(4, 4, 2),
                   max_gen_len=32768, script=script)
run = DecodeRun(cfg)
dev = torch.device('cuda')
U = cfg.units
q = torch.empty((U, 4, 128), dtype=torch.bfloat16, device=dev)
k = torch.empty((U, 128), dtype=torch.bfloat16, device=dev)
v = torch.empty((U, 128), dtype=torch.bfloat16, device=dev)
out = torch.empty((U, 4, 128), dtype=torch.float32, device=dev)
t0 = time.time()
for t in range(ctx):
    run.synth_inputs(0x71534B56, t, q, k, v)
    run.step(q, k, v, out)
torch.cuda.synchronize()
print(f"ctx {ctx} built in {time.time() - t0:.1f}s; bytes {run.bytes()['algorithmic_bytes']}", flush=True)
pos = ctx
for rep in range(3):
    for var in variants:
        os.environ.pop('TKV_K1_V2', None); os.environ.pop('TKV_K1_MINB', None)
        if var == 'v2': os.environ['TKV_K1_V2'] = '1'
        if var == 'minb4': os.environ['TKV_K1_MINB'] = '4'
        run.timing_enable(True)
        for i in range(20):
            if (pos + 1) % 128 == 0 or pos % 128 == 0:  # keep refresh/eviction steps out of the window
                run.synth_inputs(0x71534B56, pos, q, k, v); run.step(q, k, v, out); pos += 1; continue
            run.synth_inputs(0x71534B56, pos, q, k, v)
            run.step(q, k, v, out)
            pos += 1
        tm = run.timing_read()
        b = run.bytes()['algorithmic_bytes']
        ms = tm['attend_ms'] / tm['attend_launches']
        print(f"variant {var}: {ms:.4f} ms/launch  {b / ms / 1e6:.0f} GB/s", flush=True)
