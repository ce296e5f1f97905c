"""Drop-in proof: the reference's own unit suites -- test_quant,
test_attention, test_evictor, test_pager, test_sim (/root/reference/proj/
tests, 88 cases incl. the walkthrough golden fixture and generation_loop
runs) -- compiled unchanged and linked against the B200 library instead of
the reference's pager/quantizer/evictor/attention: BlockPager,
quantize_window, kmeans_select, on_transition_end, on_budget_overflow,
gqa_attend, sparsity and layer_sparsity_average come from
libthinkv_dropin.a over libthinkv_b200.so's kernels (oracle/Makefile
`dropin-tests`).  Every case must pass on the GPU."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin")


@pytest.mark.parametrize("suite", ["test_quant", "test_attention", "test_evictor", "test_pager", "test_sim"])
def test_reference_suite_on_the_gpu_library(suite):
    exe = os.path.join(BIN, suite)
    assert os.path.exists(exe), f"{exe} missing: build with `make -C oracle dropin-tests`"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    summary = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out.stdout)
    assert out.returncode == 0 and summary and summary.group(3) == "0", (out.stdout[-3000:] + out.stderr[-3000:])
    # the binary really ran on the CUDA library (its kernels, not a CPU copy)
    maps = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libthinkv_b200.so" in maps
