"""The division-free NVFP4 / ternary encoders of the quantize-on-append
kernel (k_append.cu nvfp4_encode_cmp / ternary_encode_cmp, restated here)
against the pinned codec restatement of quant.cpp:114-158 on bf16 inputs:
every E4M3 scale, random values and values within a few ulps of every
decision midpoint (the exactness argument's edge cases)."""
import math

import numpy as np

import codecs_ref as R

MIDS = (0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0)


def nvfp4_cmp(x, s):
    a = abs(x)
    i = (a > s * 0.25) + (a >= s * 0.75) + (a > s * 1.25) + (a >= s * 1.75) + (a > s * 2.5) + (a >= s * 3.5) + \
        (a > s * 5.0)
    if i == 0:
        return 0
    return (0x8 if math.copysign(1.0, x) < 0 else 0) | int(i)


def ternary_cmp(x, d):
    return R.ternary_bits(0 if not abs(x) > d * 0.5 else (1 if x > 0 else -1))


def to_bf16(x):
    b = int(np.array([x], dtype=np.float32).view(np.uint32)[0])
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return float(np.array([b], dtype=np.uint32).view(np.float32)[0])


def samples(rng, s, n, mids):
    for t in range(n):
        if t % 2 == 0:
            x = s * mids[rng.integers(len(mids))] * (1 + rng.choice([-1, 0, 1]) * 2.0 ** -rng.integers(5, 9))
            x *= rng.choice([-1.0, 1.0])
        else:
            x = rng.normal() * s * 4
        x = to_bf16(x)
        if math.isfinite(x):
            yield x


def test_nvfp4_compare_encoder_matches_reference():
    rng = np.random.default_rng(0)
    for code in range(1, 0x7F):
        s = R.e4m3_decode(code)
        for x in samples(rng, s, 200, MIDS):
            assert nvfp4_cmp(x, s) == R.nvfp4_encode_value(x / s), (x, s)


def test_ternary_compare_encoder_matches_reference():
    rng = np.random.default_rng(1)
    for code in range(1, 0x7F):
        d = R.e4m3_decode(code)
        for x in samples(rng, d, 200, (0.5, 1.5)):
            ref = R.ternary_bits(int(min(max(float(np.rint(x / d)), -1.0), 1.0)))
            assert ternary_cmp(x, d) == ref, (x, d)
