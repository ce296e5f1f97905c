"""bench.py's reference arm (CPU, no GPU needed): one JSON line in the
driver's contract, timing the compiled reference on the host cores."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--max-gen", "384", "--steps", "2", "--warmup", "1", "--e2e-steps", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "tokens/s" and line["higher_is_better"] is True
    assert line["steps"] == 2 and line["warmup"] == 1 and line["n_gpus"] == 1 and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["global_batch"] == 1 and line["scaling"] == "weak"
    # the GPU arm prints the same config object (bench_config), incl. the L2 statement
    assert line["config"]["l2"].startswith("working set fits in L2")
    assert set(line["config"]) == {"workload", "global_batch", "units_per_gpu", "parallelism", "gqa", "tau",
                                   "timed_positions", "e2e_positions", "tpot_formula", "l2"}


def test_reference_arm_does_not_map_the_cuda_library():
    """The reference arm imports the package only for its configuration types;
    the CUDA library loads lazily, so that process never maps it."""
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', '1', '--max-gen', '300', "
            "'--steps', '2', '--warmup', '1', '--e2e-steps', '1']; import bench; bench.main(); "
            "maps = open('/proc/self/maps').read(); assert 'libthinkv_b200' not in maps, 'mapped'; "
            "assert 'liboracle' in maps")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]


def test_amortised_tpot():
    sys.path.insert(0, ROOT)
    import bench
    # windows of whole tau periods: their mean (a trailing partial period is dropped)
    steps = [10.0, 1.0, 3.0, 1.0] * 2 + [50.0]
    assert bench.amortize(steps, 8, 4)[0] == 15.0 * 2 / 8
    # short window opening on a boundary: the rest of the period at the median plain step
    tpot, bnd, oth = bench.amortize([130.0, 1.0, 1.0, 1.0, 27.0, 1.0], 256, 128)
    assert bnd == [130.0] and len(oth) == 5 and abs(tpot - (161.0 + 122 * 1.0) / 128) < 1e-12
    with pytest.raises(ValueError):
        bench.amortize([1.0, 2.0], 257, 128)

    class A:
        ctx, warmup, steps, e2e_steps = None, 5, 20, 128

    class Cfg:
        max_gen_len, tau = 32768, 128
    assert bench.positions(A, Cfg) == 32512
