"""CUDA-graph replay of plain and emission decode steps (the
real-model caller): a model's per-layer decode step captured once per step
kind with tkv_step_layer inside the capture, replayed for every step of that
kind (tkv_graph_step_begin), eager steps at boundaries / evictions.  Outputs
and the final cache state must equal the oracle's, exactly as the eager path
does."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
from harness import ATOL, RTOL, compare_state, oracle_config  # noqa: E402
from paper_2510_01290_b200 import DecodeRun, ThinkvConfig, TkvError  # noqa: E402

SEED = 0x71534B56


def _script(num_seqs, intervals, seed):
    rng = np.random.default_rng(seed)
    return [[2 if rng.random() < 0.2 else int(rng.integers(0, 2)) for _ in range(intervals)]
            for _ in range(num_seqs)]


@pytest.mark.parametrize("layers,budget", [(1, 64), (2, 80), (4, 10_000)])
def test_graph_replayed_plain_steps_match_the_oracle(layers, budget):
    S, H, G, D = 2, 2, 4, 128
    cfg = ThinkvConfig(num_seqs=S, units_per_seq=layers * H, num_q_heads=G, head_dim=D, tau=32, group_size=16,
                       block_size=16, budget=budget, levels=(16, 8, 4), max_gen_len=230,
                       script=_script(S, 8, seed=layers), record_events=True)
    dev = torch.device("cuda:0")
    run = DecodeRun(cfg)
    orc = O.OracleRun(oracle_config(cfg))
    rows = cfg.out_rows
    # the model's static buffers: one q/k/v/out set per layer
    qs = [torch.empty((S, H, G, D), dtype=torch.bfloat16, device=dev) for _ in range(layers)]
    ks = [torch.empty((S, H, D), dtype=torch.bfloat16, device=dev) for _ in range(layers)]
    vs = [torch.empty((S, H, D), dtype=torch.bfloat16, device=dev) for _ in range(layers)]
    os_ = [torch.empty((S, H, rows, D), dtype=torch.float32, device=dev) for _ in range(layers)]

    def model_step():
        for l in range(layers):
            run.step_layer(l, layers, qs[l], ks[l], vs[l], os_[l])

    stream = torch.cuda.Stream()
    graphs, replays, eager = {}, {1: 0, 2: 0}, 0
    with torch.cuda.stream(stream):
        for t in range(cfg.max_gen_len):
            q, k, v = O.synth_step(SEED, cfg.units_per_seq, cfg.tau, cfg.units, G, D, t)
            tq, tk, tv = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(dev) for x in (q, k, v))
            q5, k5, v5 = tq.view(S, layers, H, G, D), tk.view(S, layers, H, D), tv.view(S, layers, H, D)
            for l in range(layers):
                qs[l].copy_(q5[:, l])
                ks[l].copy_(k5[:, l])
                vs[l].copy_(v5[:, l])
            ref, _ = orc.step(O.bf16_to_f64(q), O.bf16_to_f64(k), O.bf16_to_f64(v))
            kind = run.step_kind()
            if kind:
                if kind not in graphs:
                    pos = run.position
                    graphs[kind] = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graphs[kind]):
                        model_step()  # recorded, not executed
                    assert run.position == pos
                run.graph_step_begin()
                graphs[kind].replay()
                replays[kind] += 1
            else:
                with pytest.raises(TkvError):
                    run.graph_step_begin()  # a non-plain step refuses replay
                model_step()
                eager += 1
            got = torch.stack(os_, dim=1).reshape(cfg.units, rows, D).double().cpu().numpy()
            err = float(np.max(np.abs(got - ref)))
            assert err <= ATOL + RTOL * float(np.max(np.abs(ref))), f"step {t}: error {err}"
    torch.cuda.synchronize()
    # boundaries every 32 steps (and eviction steps) are eager; plain and emission steps replay
    assert replays[1] >= cfg.max_gen_len // 4 and replays[2] >= 1 and eager >= cfg.max_gen_len // 32
    compare_state({"run": run, "oracle": orc}, cfg)
