"""Pure-Python restatement of the reference codecs (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/proj/src/quant.cpp line by line; pinned by
tests/test_oracle.py against the reference's golden wire vectors
(tests/golden/quant_vectors.json, copied from proj/tests/fixtures) and the
known-answer codes of test_quant.cpp:101-116.  Used by CPU tests that must
not need the compiled oracle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List

import numpy as np

E4M3_MAX = 448.0
NVFP4_GRID = (0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0)  # quant.cpp:106


def _rne(x: float) -> float:
    return float(np.rint(x))  # nearbyint in the default rounding mode


def e4m3_encode(x: float) -> int:  # quant.cpp:67-89
    if math.isnan(x):
        raise ValueError("e4m3: NaN input")
    sign = 0x80 if math.copysign(1.0, x) < 0 else 0
    a = abs(x)
    if a >= E4M3_MAX:
        return sign | 0x7E
    if a < 2.0 ** -6:
        r = _rne(a * 2.0 ** 9)
        if r >= 8.0:
            return sign | 0x08
        return sign | int(r)
    fr, e = math.frexp(a)
    e -= 1
    fr *= 2.0
    m = _rne((fr - 1.0) * 8.0)
    if m >= 8.0:
        e += 1
        m = 0.0
    if e > 8 or (e == 8 and m > 6.0):
        return sign | 0x7E
    return sign | ((e + 7) << 3) | int(m)


def e4m3_decode(code: int) -> float:  # quant.cpp:91-99
    sign = -1.0 if code & 0x80 else 1.0
    e = (code >> 3) & 0xF
    m = code & 0x7
    if e == 15 and m == 7:
        return float("nan")
    v = m * 2.0 ** -9 if e == 0 else (1.0 + m / 8.0) * 2.0 ** (e - 7)
    return sign * v


def nvfp4_encode_value(x: float) -> int:  # quant.cpp:114-130
    if x == 0.0:
        return 0
    sign = 0x8 if math.copysign(1.0, x) < 0 else 0
    a = abs(x)
    best, best_d = 0, abs(a - NVFP4_GRID[0])
    for i in range(1, 8):
        d = abs(a - NVFP4_GRID[i])
        if d < best_d or (d == best_d and i % 2 == 0):
            best, best_d = i, d
    return 0 if best == 0 else sign | best


def ternary_bits(v: int) -> int:  # quant.cpp:219-226
    return {0: 0b00, 1: 0b01, -1: 0b11}[v]


@dataclass
class Group:
    fmt: str
    g: int
    scale_code: int = 0
    scale_f32: float = 0.0
    codes: List[int] = field(default_factory=list)


def ternary_group(xs) -> Group:  # quant.cpp:141-158
    am = max((abs(float(x)) for x in xs), default=0.0)
    sc = e4m3_encode(am)
    delta = e4m3_decode(sc)
    codes = [0] * len(xs)
    if delta > 0.0:
        for i, x in enumerate(xs):
            r = _rne(float(x) / delta)
            codes[i] = ternary_bits(int(min(max(r, -1.0), 1.0)))
    return Group("TERNARY2", len(xs), sc, 0.0, codes)


def nvfp4_group(xs) -> Group:  # quant.cpp:160-174
    am = max((abs(float(x)) for x in xs), default=0.0)
    sc = e4m3_encode(am / 6.0)
    s = e4m3_decode(sc)
    codes = [nvfp4_encode_value(float(x) / s) if s > 0.0 else 0 for x in xs]
    return Group("NVFP4", len(xs), sc, 0.0, codes)


def fp8_group(xs, scale) -> Group:  # quant.cpp:180-193
    scale = float(np.float32(scale))
    codes = [e4m3_encode(float(x) / scale) if scale > 0.0 else 0 for x in xs]
    return Group("FP8E4M3", len(xs), 0, scale, codes)


def serialize(g: Group) -> bytes:  # quant.cpp:274-322
    tag = {"TERNARY2": 0, "NVFP4": 1, "FP8E4M3": 2}[g.fmt]
    out = bytearray([tag, g.g & 0xFF, (g.g >> 8) & 0xFF])
    if g.fmt == "FP8E4M3":
        out += np.float32(g.scale_f32).tobytes()
    else:
        out.append(g.scale_code)
    c = g.codes
    if g.fmt == "TERNARY2":
        cells = [(c[i] & 3) | ((c[i + 1] & 3) << 2 if i + 1 < len(c) else 0) for i in range(0, len(c), 2)]
        for i in range(0, len(cells), 2):
            out.append(cells[i] | ((cells[i + 1] << 4) if i + 1 < len(cells) else 0))
    elif g.fmt == "NVFP4":
        for i in range(0, len(c), 2):
            out.append((c[i] & 0xF) | (((c[i + 1] & 0xF) << 4) if i + 1 < len(c) else 0))
    else:
        out += bytes(c)
    return bytes(out)
