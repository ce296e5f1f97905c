import sys, numpy as np, torch
sys.path[:0] = ['.', 'oracle', 'tests']
import oracle as O
from paper_2510_01290_b200 import GatherRun
units, G, D, budget = 3, 4, 128, 48
dev = torch.device('cuda')
gpu = GatherRun(units, G, D, budget, exact=True)
orc = O.GatherOracle(units, G, D, budget)
out = torch.empty((units, G, D), device=dev)
Ks, Vs = [], []
for t in range(8):
    q, k, v = O.synth_step(0x71534B56, units, 32, units, G, D, t)
    ref, _ = orc.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
    tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
    gpu.step(tq, tk, tv, out)
    torch.cuda.synchronize()
    got = out.double().cpu().numpy()
    Ks.append(O.bf16_to_f64(k)); Vs.append(O.bf16_to_f64(v))
    K = np.stack(Ks, 1); V = np.stack(Vs, 1)  # [units, n, D]
    qd = O.bf16_to_f64(q)
    lg = np.einsum('ugd,und->ugn', qd, K) / np.sqrt(D)
    p = np.exp(lg - lg.max(-1, keepdims=True)); p /= p.sum(-1, keepdims=True)
    mine = np.einsum('ugn,und->ugd', p, V)
    print(t, 'gpu-ref', np.abs(got - ref).max(), 'numpy-ref', np.abs(mine - ref).max(), 'gpu-numpy', np.abs(got-mine).max())
    if np.abs(got - ref).max() > 1e-2:
        print(' per unit/head err', np.abs(got - ref).max(-1))
        print(' gpu ids', gpu.ids(0), 'orc ids', orc.ids(0))
