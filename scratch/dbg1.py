import sys, numpy as np, torch
sys.path[:0] = ['.', 'oracle', 'tests']
import oracle as O
from harness import synth_inputs, oracle_config
from paper_2510_01290_b200 import DecodeRun, ThinkvConfig
cfg = ThinkvConfig(num_seqs=1, units_per_seq=2, num_q_heads=4, head_dim=128, tau=32, group_size=16, block_size=16, budget=96, levels=(16,8,4), max_gen_len=40, script=[[1]])
run = DecodeRun(cfg); orc = O.OracleRun(oracle_config(cfg))
dev = torch.device('cuda')
out = torch.empty((cfg.units, 4, 128), device=dev)
for t in range(6):
    q,k,v = synth_inputs(cfg, 1, t)
    ro,_ = orc.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
    f = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).to(dev)
    run.step(f(q), f(k), f(v), out)
    g = out.double().cpu().numpy()
    e = np.abs(g-ro)
    print(t, e.max(), [e[u].max() for u in range(cfg.units)], [e[0, r].max() for r in range(4)])
    if e.max() > 1e-3:
        print(' ref', ro[0,0,:6]); print(' got', g[0,0,:6])
