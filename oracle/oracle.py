"""ctypes wrapper over oracle/_ref/liboracle.so (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module; the product path never does.  The library restates the
reference's ThinkvMethod (/root/reference/proj/src/sim.cpp:494-958) on top of
the compiled, unmodified reference library -- see oracle_driver.h.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "liboracle.so")


class SynthParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("units_per_seq", C.c_int32), ("tau", C.c_int32),
                ("sink_tokens", C.c_int32), ("reserved", C.c_int32)]


class OrcDesc(C.Structure):
    _fields_ = [
        ("num_seqs", C.c_int32), ("units_per_seq", C.c_int32), ("num_q_heads", C.c_int32),
        ("gqa_maxpool", C.c_int32), ("head_dim", C.c_int32), ("tau", C.c_int32),
        ("group_size", C.c_int32), ("block_size", C.c_int32), ("pool_blocks", C.c_int32),
        ("budget", C.c_int64), ("num_levels", C.c_int32), ("levels", C.c_int64 * 16),
        ("psi_bits", C.c_int32 * 8), ("num_thoughts", C.c_int32),
        ("threshold_fraction", C.c_double), ("prompt_len", C.c_int64),
        ("max_gen_len", C.c_int64), ("scripted", C.c_int32), ("script_len", C.c_int32),
        ("script_bands", C.POINTER(C.c_int32)), ("per_layer_thought", C.c_int32),
        ("num_thresholds", C.c_int32), ("thresholds", C.c_double * 8),
        ("num_calib_units", C.c_int32), ("calib_units", C.c_int32 * 64),
        ("num_dump_positions", C.c_int32), ("dump_positions", C.POINTER(C.c_int64)),
    ]


_lib = None
_lock = threading.Lock()


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"oracle library missing: {LIB_PATH} (run `make -C oracle`)")
            L = C.CDLL(LIB_PATH)
            L.orc_create.restype = C.c_void_p
            L.orc_create.argtypes = [C.POINTER(OrcDesc), C.c_char_p, C.c_int]
            L.orc_destroy.argtypes = [C.c_void_p]
            L.orc_step.argtypes = [C.c_void_p] + [C.c_void_p] * 5
            L.orc_finish.argtypes = [C.c_void_p]
            L.orc_dump.restype = C.c_char_p
            L.orc_dump.argtypes = [C.c_void_p, C.c_int, C.c_char_p]
            L.orc_export.restype = C.c_int64
            L.orc_export.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64]
            L.orc_toy_compare.restype = C.c_char_p
            L.orc_toy_compare.argtypes = [C.c_char_p]
            L.orc_toy_stream.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.orc_synth_step.argtypes = [C.POINTER(SynthParams), C.c_int64, C.c_int32, C.c_int32,
                                         C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
            L.orc_gather_create.restype = C.c_void_p
            L.orc_gather_create.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64]
            L.orc_gather_destroy.argtypes = [C.c_void_p]
            L.orc_gather_step.argtypes = [C.c_void_p, C.c_int32] + [C.c_void_p] * 5
            L.orc_gather_ids.restype = C.c_int64
            L.orc_gather_ids.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64]
            L.orc_gather_stats.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
            L.orc_gather_toy_compare.restype = C.c_char_p
            L.orc_gather_toy_compare.argtypes = [C.c_char_p]
            _lib = L
    return _lib


@dataclass
class RunConfig:
    """Mirror of the reference SimConfig fields that drive the hot path
    (proj/include/thinkv/sim.hpp:38-68), over `num_seqs` independent
    sequences of `units_per_seq` units (one unit = one reference "layer")."""
    num_seqs: int = 1
    units_per_seq: int = 1
    num_q_heads: int = 1
    gqa_maxpool: bool = False
    head_dim: int = 16
    tau: int = 128
    group_size: int = 16
    block_size: int = 8
    pool_blocks: int = 0
    budget: int = 1024
    levels: Sequence[int] = (64, 32, 16, 8, 4)
    psi_bits: Sequence[int] = (4, 4, 2)  # bands E, R, T (R4E4T2)
    num_thoughts: int = 3
    threshold_fraction: float = 0.01
    prompt_len: int = 0
    max_gen_len: int = 1024
    scripted: bool = True
    script: Optional[List[List[int]]] = None  # [num_seqs][intervals]
    per_layer_thought: bool = False
    thresholds: Sequence[float] = ()
    calib_units: Sequence[int] = ()
    dump_positions: Sequence[int] = ()

    def to_desc(self):
        d = OrcDesc()
        d.num_seqs = self.num_seqs
        d.units_per_seq = self.units_per_seq
        d.num_q_heads = self.num_q_heads
        d.gqa_maxpool = int(self.gqa_maxpool)
        d.head_dim = self.head_dim
        d.tau = self.tau
        d.group_size = self.group_size
        d.block_size = self.block_size
        d.pool_blocks = self.pool_blocks
        d.budget = self.budget
        d.num_levels = len(self.levels)
        for i, x in enumerate(self.levels):
            d.levels[i] = x
        for i, b in enumerate(self.psi_bits):
            d.psi_bits[i] = b
        d.num_thoughts = self.num_thoughts
        d.threshold_fraction = self.threshold_fraction
        d.prompt_len = self.prompt_len
        d.max_gen_len = self.max_gen_len
        d.scripted = int(self.scripted)
        keep = []
        if self.scripted:
            script = self.script or [[1]] * self.num_seqs
            n = max(len(s) for s in script)
            arr = np.array([list(s) + [s[-1]] * (n - len(s)) for s in script], dtype=np.int32)
            keep.append(arr)
            d.script_len = n
            d.script_bands = arr.ctypes.data_as(C.POINTER(C.c_int32))
        d.per_layer_thought = int(self.per_layer_thought)
        d.num_thresholds = len(self.thresholds)
        for i, t in enumerate(self.thresholds):
            d.thresholds[i] = t
        d.num_calib_units = len(self.calib_units)
        for i, u in enumerate(self.calib_units):
            d.calib_units[i] = u
        if self.dump_positions:
            dp = np.array(self.dump_positions, dtype=np.int64)
            keep.append(dp)
            d.num_dump_positions = len(dp)
            d.dump_positions = dp.ctypes.data_as(C.POINTER(C.c_int64))
        return d, keep

    @property
    def units(self):
        return self.num_seqs * self.units_per_seq

    @property
    def out_groups(self):
        return 1 if self.gqa_maxpool else self.num_q_heads


class OracleRun:
    def __init__(self, cfg: RunConfig):
        self.cfg = cfg
        desc, self._keep = cfg.to_desc()
        err = C.create_string_buffer(512)
        self._h = lib().orc_create(C.byref(desc), err, 512)
        if not self._h:
            raise ValueError(err.value.decode())

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().orc_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def step(self, q: np.ndarray, k: np.ndarray, v: np.ndarray):
        c = self.cfg
        q = np.ascontiguousarray(q, dtype=np.float64)
        k = np.ascontiguousarray(k, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros((c.units, c.out_groups, c.head_dim), dtype=np.float64)
        sp = np.zeros((c.units,), dtype=np.float64)
        rc = lib().orc_step(self._h, q.ctypes.data, k.ctypes.data, v.ctypes.data,
                            out.ctypes.data, sp.ctypes.data)
        if rc != 0:
            raise OracleError(rc, self.dump(0, "error"))
        return out, sp

    def finish(self):
        rc = lib().orc_finish(self._h)
        if rc != 0:
            raise OracleError(rc, self.dump(0, "error"))

    def export(self, seq: int, unit: int) -> bytes:
        """Unit `unit` of sequence `seq` in the k_export.cu stream layout, built
        by the reference's BlockPager::read_active/group_table + serialize_group."""
        n = lib().orc_export(self._h, seq, unit, None, 0)
        if n < 0:
            raise OracleError(-n, self.dump(0, "error"))
        buf = C.create_string_buffer(max(1, n))
        lib().orc_export(self._h, seq, unit, buf, n)
        return buf.raw[:n]

    def dump(self, seq: int, what: str):
        s = lib().orc_dump(self._h, seq, what.encode()).decode()
        if what in ("error", "events"):
            return s
        return json.loads(s)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class GatherOracle:
    """GatherMethod (sim.cpp:1117-1206) restated for external per-unit inputs:
    attend over every kept token, evict the lowest head-averaged score once
    over budget and shift later tokens down (moved_token_slots)."""

    def __init__(self, units: int, num_q_heads: int, head_dim: int, budget: int, gqa_maxpool: bool = False):
        self.units, self.G, self.D = units, num_q_heads, head_dim
        self.groups = 1 if gqa_maxpool else num_q_heads
        self._h = lib().orc_gather_create(units, num_q_heads, int(gqa_maxpool), head_dim, budget)

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().orc_gather_destroy(self._h)
        except Exception:
            pass

    def step(self, q, k, v, prefill: bool = False):
        q = np.ascontiguousarray(q, dtype=np.float64)
        k = np.ascontiguousarray(k, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros((self.units, self.groups, self.D))
        victims = np.zeros(self.units, dtype=np.int64)
        rc = lib().orc_gather_step(self._h, int(prefill), q.ctypes.data, k.ctypes.data, v.ctypes.data,
                                   out.ctypes.data, victims.ctypes.data)
        if rc:
            raise OracleError(rc, "gather step failed")
        return out, victims

    def ids(self, unit: int) -> np.ndarray:
        n = lib().orc_gather_ids(self._h, unit, None, 0)
        buf = np.zeros(max(n, 1), dtype=np.int64)
        lib().orc_gather_ids(self._h, unit, buf.ctypes.data, n)
        return buf[:n]

    def stats(self):
        moved, ev = C.c_int64(), C.c_int64()
        lib().orc_gather_stats(self._h, C.byref(moved), C.byref(ev))
        return {"moved_token_slots": moved.value, "eviction_steps": ev.value}


def gather_toy_compare(config: dict) -> dict:
    return json.loads(lib().orc_gather_toy_compare(json.dumps(config).encode()).decode())


def toy_compare(config: dict) -> dict:
    return json.loads(lib().orc_toy_compare(json.dumps(config).encode()).decode())


def toy_stream(config: dict):
    """ToyModel q/k/v stream of a reference SimConfig dict (doubles):
    q [steps, layers, heads, d], k/v [steps, layers, d]."""
    m = config["model"]
    steps = config.get("prompt_len", 0) + config["max_gen_len"]
    L, H, D = m["num_layers"], m["num_heads"], m["head_dim"]
    q = np.zeros((steps, L, H, D))
    k = np.zeros((steps, L, D))
    v = np.zeros((steps, L, D))
    rc = lib().orc_toy_stream(json.dumps(config).encode(), q.ctypes.data, k.ctypes.data,
                              v.ctypes.data)
    if rc != 0:
        raise OracleError(rc, "toy stream failed")
    return q, k, v


def synth_step(seed: int, units_per_seq: int, tau: int, units: int, G: int, d: int, step: int,
               unit0: int = 0, sink_tokens: int = 4):
    """bf16 bit patterns (uint16) for one step: q [units,G,d], k/v [units,d]."""
    p = SynthParams(seed, units_per_seq, tau, sink_tokens, 0)
    q = np.empty((units, G, d), dtype=np.uint16)
    k = np.empty((units, d), dtype=np.uint16)
    v = np.empty((units, d), dtype=np.uint16)
    lib().orc_synth_step(C.byref(p), unit0, units, G, d, step, q.ctypes.data, k.ctypes.data,
                         v.ctypes.data)
    return q, k, v


def bf16_to_f64(x: np.ndarray) -> np.ndarray:
    return (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
