"""Host-side reader for the compressed-cache export.

`DecodeRun.export_cache` writes every live pager token as QuantizedGroups in
the reference's wire layout (serialize_group, proj/src/quant.cpp:274-324,
quant.hpp:104-110); the stream layout is documented in csrc/k_export.cu.
This module mirrors the reference's `deserialize_group`
(quant.cpp:326-376) -- same field order, same truncation / unknown-tag
errors (ErrorKind::kParse -> status 2) -- and walks a unit stream into
per-token codes, scales and decoded key/value vectors (decode_code,
quant.cpp:195-205).  It is pure host code over bytes already downloaded.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field
from typing import List

import numpy as np

TERNARY2, NVFP4, FP8E4M3, RAW = 0, 1, 2, 3
FORMAT_NAMES = {TERNARY2: "TERNARY2", NVFP4: "NVFP4", FP8E4M3: "FP8E4M3", RAW: "RAW16"}
_NVFP4_GRID = (0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0)  # quant.cpp:106


class WireError(ValueError):
    """deserialize_group's ErrorKind::kParse (exit code 2)."""
    code = 2


@dataclass
class QuantizedGroup:  # quant.hpp:60-68
    format: int = NVFP4
    g: int = 16
    scale_code: int = 0
    scale_f32: float = 0.0
    codes: List[int] = field(default_factory=list)

    def scale(self) -> float:
        return self.scale_f32 if self.format == FP8E4M3 else e4m3_decode(self.scale_code)


def e4m3_decode(code: int) -> float:  # quant.cpp:91-99
    sign = -1.0 if code & 0x80 else 1.0
    e, m = (code >> 3) & 0xF, code & 0x7
    if e == 15 and m == 7:
        return math.nan
    v = m * 0.001953125 if e == 0 else (1.0 + m / 8.0) * math.ldexp(1.0, e - 7)
    return sign * v


def decode_code(fmt: int, code: int, scale: float) -> float:  # quant.cpp:195-205
    if fmt == TERNARY2:
        return {0: 0.0, 1: 1.0, 2: 0.0, 3: -1.0}[code & 3] * scale
    if fmt == NVFP4:
        return (-1.0 if code & 0x8 else 1.0) * _NVFP4_GRID[code & 7] * scale
    return e4m3_decode(code) * scale


def serialize_group(g: QuantizedGroup) -> bytes:  # quant.cpp:274-324
    out = bytearray([g.format, g.g & 0xFF, (g.g >> 8) & 0xFF])
    if g.format == FP8E4M3:
        out += struct.pack("<f", g.scale_f32)
    else:
        out.append(g.scale_code)
    c = g.codes
    if g.format == TERNARY2:
        for i in range(0, len(c), 4):
            b = 0
            for e in range(4):
                if i + e < len(c):
                    b |= (c[i + e] & 3) << (2 * e)
            out.append(b)
    elif g.format == NVFP4:
        for i in range(0, len(c), 2):
            out.append((c[i] & 0xF) | ((c[i + 1] & 0xF) << 4 if i + 1 < len(c) else 0))
    else:
        out += bytes(c)
    return bytes(out)


def deserialize_group(b, off: int = 0):
    """(group, bytes consumed) from b[off:] (quant.cpp:326-376)."""
    def need(n):
        if len(b) - off < n:
            raise WireError("group record truncated")
    need(3)
    if b[off] > 2:
        raise WireError(f"unknown format tag {b[off]}")
    grp = QuantizedGroup(format=b[off], g=b[off + 1] | (b[off + 2] << 8))
    p = 3
    if grp.format == FP8E4M3:
        need(p + 4)
        grp.scale_f32 = struct.unpack_from("<f", b, off + p)[0]
        p += 4
    else:
        need(p + 1)
        grp.scale_code = b[off + p]
        p += 1
    n = grp.g
    if grp.format == TERNARY2:
        need(p + (n + 3) // 4)
        grp.codes = [(b[off + p + i // 4] >> (2 * (i % 4))) & 3 for i in range(n)]
        p += (n + 3) // 4
    elif grp.format == NVFP4:
        need(p + (n + 1) // 2)
        grp.codes = [(b[off + p + i // 2] >> (4 * (i % 2))) & 0xF for i in range(n)]
        p += (n + 1) // 2
    else:
        need(p + n)
        grp.codes = list(b[off + p:off + p + n])
        p += n
    return grp, p


@dataclass
class Record:
    kind: int               # TERNARY2 / NVFP4 / FP8E4M3 / RAW
    band: int               # thought band
    ids: np.ndarray         # token ids (ascending)
    keys: np.ndarray        # [n][d] decoded keys (BlockPager::key_of values)
    values: np.ndarray      # [n][d] decoded values
    key_groups: List[QuantizedGroup] = field(default_factory=list)
    value_groups: List[QuantizedGroup] = field(default_factory=list)


def parse_unit(b, off: int = 0):
    """One unit stream -> (list of Record, bytes consumed)."""
    b = memoryview(bytes(b)) if not isinstance(b, (bytes, bytearray, memoryview)) else b
    if len(b) - off < 12:
        raise WireError("unit header truncated")
    nrec, nlive, d, vg = struct.unpack_from("<IIHH", b, off)
    p = off + 12
    recs = []
    total = 0
    for _ in range(nrec):
        if len(b) - p < 4:
            raise WireError("record header truncated")
        kind, band, n = b[p], b[p + 1], b[p + 2] | (b[p + 3] << 8)
        p += 4
        ids = np.frombuffer(bytes(b[p:p + 8 * n]), dtype="<i8").copy()
        if ids.size != n:
            raise WireError("record ids truncated")
        p += 8 * n
        keys = np.zeros((n, d))
        vals = np.zeros((n, d))
        rec = Record(kind, band, ids, keys, vals)
        if kind == RAW:
            raw = np.frombuffer(bytes(b[p:p + 16 * n * d]), dtype="<f8")
            if raw.size != 2 * n * d:
                raise WireError("raw record truncated")
            raw = raw.reshape(n, 2, d)
            keys[:], vals[:] = raw[:, 0], raw[:, 1]
            p += 16 * n * d
        elif kind == FP8E4M3:
            for side, arr in ((0, keys), (1, vals)):
                grp, used = deserialize_group(b, p)
                p += used
                (rec.key_groups if side == 0 else rec.value_groups).append(grp)
                s = grp.scale()
                arr[:] = np.array([decode_code(FP8E4M3, c, s) for c in grp.codes]).reshape(n, d)
        elif kind in (TERNARY2, NVFP4):
            for c in range(d):
                grp, used = deserialize_group(b, p)
                p += used
                rec.key_groups.append(grp)
                s = grp.scale()
                keys[:, c] = [decode_code(kind, x, s) for x in grp.codes]
            chunks = (d + vg - 1) // vg
            for t in range(n):
                for j in range(chunks):
                    grp, used = deserialize_group(b, p)
                    p += used
                    rec.value_groups.append(grp)
                    s = grp.scale()
                    vals[t, j * vg:j * vg + grp.g] = [decode_code(kind, x, s) for x in grp.codes]
        else:
            raise WireError(f"unknown record kind {kind}")
        total += n
        recs.append(rec)
    if total != nlive:
        raise WireError(f"unit header says {nlive} live tokens, records hold {total}")
    return recs, p - off
