"""A real-model caller of the decode path: a bf16 decoder with the
R1-Distill-Llama-8B attention shape (hidden 4096, 32 q / 8 kv heads, d=128,
32 layers; random weights, no checkpoint is reachable here) whose attention
runs through tkv_step_layer.  Per layer and decode step:

    x = rmsnorm(h);  q, k, v = x Wq, x Wk, x Wv       (cuBLAS bf16 GEMMs)
    o = tkv_step_layer(layer, q, k, v)                 (K1 on the compressed cache)
    h = h + bf16(o) Wo                                 (+ the MLP with --mlp)

Keys arrive post-RoPE in the reference (apply_rotary is outside the path), so
no rotary is applied.  The decode context is built with the synthetic inputs
(tkv_synth_inputs, the bench's own path) up to --ctx, then the model drives
the run: K steps eagerly (every launch from Python), then K steps where each
plain or emission step replays the CUDA graph of its kind holding the whole
model step (tkv_graph_step_begin + graph.replay()) and boundary / eviction
steps run eagerly.  Both windows open on a refresh boundary and span whole
tau periods.  Prints one JSON line.

    python tools/model_loop.py [--seqs 4] [--ctx 32640] [--steps 128] [--mlp]
"""
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
    ap.add_argument("--ctx", type=int, default=32768 - 3 * 128, help="first model-driven decode position")
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--mlp", action="store_true", help="add the Llama MLP (intermediate 14336) per layer")
    args = ap.parse_args()

    import torch
    from paper_2510_01290_b200 import DecodeRun, ThinkvConfig
    from paper_2510_01290_b200.synth import band_script

    S, L, H, G, D, HID = args.seqs, args.layers, 8, 4, 128, 4096
    tau = 128
    max_gen = args.ctx + 2 * (args.steps + args.warmup + 16 + tau) + 16
    cfg = ThinkvConfig(num_seqs=S, units_per_seq=L * H, num_q_heads=G, head_dim=D, tau=tau, group_size=16,
                       block_size=16, budget=1024, levels=(64, 32, 16, 8, 4), psi_bits=(4, 4, 2),
                       max_gen_len=max_gen, script=band_script(SEED, S, max_gen // tau + 2, 3, 100))
    dev = torch.device("cuda:0")
    run = DecodeRun(cfg)
    U = cfg.units
    # 1. context through the synthetic path (untimed)
    q0 = torch.empty((U, G, D), dtype=torch.bfloat16, device=dev)
    k0 = torch.empty((U, D), dtype=torch.bfloat16, device=dev)
    v0 = torch.empty((U, D), dtype=torch.bfloat16, device=dev)
    o0 = torch.empty((U, G, D), dtype=torch.float32, device=dev)
    t0 = time.time()
    for t in range(args.ctx - args.warmup):
        run.synth_inputs(SEED, t, q0, k0, v0)
        run.step(q0, k0, v0, o0)
    torch.cuda.synchronize()
    ctx_s = time.time() - t0

    # 2. the model: random bf16 weights, static activations (graph-capturable)
    g = torch.Generator(device=dev).manual_seed(7)

    def w(i, o):
        return (torch.randn((i, o), device=dev, generator=g) * (i ** -0.5)).to(torch.bfloat16)
    Wq = [w(HID, H * G * D) for _ in range(L)]
    Wk = [w(HID, H * D) for _ in range(L)]
    Wv = [w(HID, H * D) for _ in range(L)]
    Wo = [w(H * G * D, HID) for _ in range(L)]
    if args.mlp:
        Wg = [w(HID, 14336) for _ in range(L)]
        Wu = [w(HID, 14336) for _ in range(L)]
        Wd = [w(14336, HID) for _ in range(L)]
    emb = torch.randn((64, S, HID), device=dev, generator=g).to(torch.bfloat16)
    h = torch.empty((S, HID), dtype=torch.bfloat16, device=dev)
    x = torch.empty_like(h)
    qb = [torch.empty((S, H, G, D), dtype=torch.bfloat16, device=dev) for _ in range(L)]
    kb = [torch.empty((S, H, D), dtype=torch.bfloat16, device=dev) for _ in range(L)]
    vb = [torch.empty((S, H, D), dtype=torch.bfloat16, device=dev) for _ in range(L)]
    ob = [torch.empty((S, H, G, D), dtype=torch.float32, device=dev) for _ in range(L)]

    def rmsnorm(y):
        yf = y.float()
        return (yf * torch.rsqrt(yf.pow(2).mean(-1, keepdim=True) + 1e-6)).to(torch.bfloat16)

    def model_step():
        for l in range(L):
            x.copy_(rmsnorm(h))
            torch.matmul(x, Wq[l], out=qb[l].view(S, H * G * D))
            torch.matmul(x, Wk[l], out=kb[l].view(S, H * D))
            torch.matmul(x, Wv[l], out=vb[l].view(S, H * D))
            run.step_layer(l, L, qb[l], kb[l], vb[l], ob[l])
            h.add_(torch.matmul(ob[l].view(S, H * G * D).to(torch.bfloat16), Wo[l]))
            if args.mlp:
                y = rmsnorm(h)
                h.add_(torch.matmul(torch.nn.functional.silu(y @ Wg[l]) * (y @ Wu[l]), Wd[l]))

    stream = torch.cuda.Stream()
    graphs = {}  # one per capturable step kind (1 plain, 2 emission)
    res = {}
    with torch.cuda.stream(stream):
        for mode in ("eager", "graph"):
            pos0 = run.position
            # align the window to a refresh boundary; the warmup before it
            # holds at least one emission, so both graphs are captured untimed
            pre = args.warmup + 16
            lead = (-(pos0 + pre)) % tau + pre
            replays = eager = 0
            for i in range(lead + args.steps):
                if i == lead:
                    torch.cuda.synchronize()
                    run.timing_enable(True)
                    ev0 = torch.cuda.Event(enable_timing=True)
                    ev0.record(stream)
                    h0 = time.perf_counter()
                h.copy_(emb[(run.position) % 64])
                kind = run.step_kind() if mode == "graph" else 0
                if kind:
                    if kind not in graphs:
                        graphs[kind] = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(graphs[kind]):
                            model_step()
                    run.graph_step_begin()
                    graphs[kind].replay()
                    replays += i >= lead
                else:
                    model_step()
                    eager += i >= lead
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record(stream)
            host_s = time.perf_counter() - h0
            torch.cuda.synchronize()
            dev_ms = ev0.elapsed_time(ev1)
            tm = run.timing_read()
            res[mode] = {"ms_per_step": dev_ms / args.steps, "tokens_per_s": S * args.steps / (dev_ms / 1e3),
                         "host_enqueue_ms_per_step": host_s * 1e3 / args.steps,
                         "positions": [pos0 + lead, pos0 + lead + args.steps - 1],
                         "graph_replayed_steps": replays, "eager_steps": eager,
                         "tkv_launches": tm["total_launches"]}
    line = {"what": "R1-Distill-Llama-8B-shaped bf16 decoder (random weights) with ThinKV attention via "
                    "tkv_step_layer; eager vs CUDA-graph replay of plain and emission steps",
            "seqs": S, "layers": L, "mlp": args.mlp, "context_build_s": ctx_s, **res,
            "graph_speedup": res["eager"]["ms_per_step"] / res["graph"]["ms_per_step"]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
