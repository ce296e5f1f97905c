"""Device build of tkv_exp (K3a sparsity, exact gather scores) == the C
library's exp() -- the one the reference's softmax_row calls -- bit for bit
(Python's math.exp calls it)."""
import ctypes as C
import math
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2510_01290_b200 import Context, _abi  # noqa: E402


def test_device_exp_matches_libc_bit_for_bit():
    flags = open("/proc/cpuinfo").read()
    if " fma" not in flags or " avx2" not in flags:
        pytest.skip("glibc selects its FMA exp only on FMA + AVX2 hosts")
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.uniform(-1, 1, 200000), rng.uniform(-60, 0, 400000), rng.uniform(-800, 800, 200000),
                         rng.uniform(-746, -700, 100000), rng.uniform(-1e-15, 1e-15, 10000),
                         rng.integers(0, 2**63, 100000, dtype=np.int64).view(np.float64),
                         np.array([0.0, -0.0, 512.0, -512.0, 1024.0, -1024.0, np.inf, -np.inf])])
    xs = np.ascontiguousarray(xs[np.isfinite(xs) | np.isinf(xs)])
    ys = np.empty_like(xs)
    ctx = Context.get(0)
    _abi.check(_abi.lib.tkv_exp_f64(ctx._h, xs.ctypes.data, ys.ctypes.data, xs.size))
    bad = 0
    for x, y in zip(xs.tolist(), ys.tolist()):
        try:
            want = math.exp(x)
        except OverflowError:
            want = math.inf
        if struct.pack("<d", want) != struct.pack("<d", y):
            bad += 1
    assert bad == 0, f"{bad} of {xs.size} differ"
