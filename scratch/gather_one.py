import sys, torch
sys.path[:0] = ['.']
from paper_2510_01290_b200 import GatherRun, DecodeRun, ThinkvConfig
U, G, D, budget = 1024, 4, 128, 655
dev = torch.device('cuda')
g = GatherRun(U, G, D, budget, exact=False)
th = DecodeRun(ThinkvConfig(num_seqs=4, units_per_seq=256, num_q_heads=G, head_dim=D, tau=128, group_size=16,
                            block_size=16, budget=budget, max_gen_len=2000, script=[[1]] * 4))
q = torch.empty((U, G, D), dtype=torch.bfloat16, device=dev); k = torch.empty((U, D), dtype=torch.bfloat16, device=dev)
v = torch.empty((U, D), dtype=torch.bfloat16, device=dev); out = torch.empty((U, G, D), device=dev)
for t in range(700):
    th.synth_inputs(7, t, q, k, v)
    g.step(q, k, v, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for t in range(700, 740):
    g.step(q, k, v, out)
e1.record(); torch.cuda.synchronize()
print("gather ms/step", e0.elapsed_time(e1) / 40)
