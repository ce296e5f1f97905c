"""B200-native ThinKV decode path (arxiv 2510.01290).

Host-side mirror of the reference's per-step interface over the C ABI in
include/thinkv_b200.h:

  reference (proj/src/sim.cpp, proj/include/thinkv/sim.hpp)   here
  --------------------------------------------------------    ---------------------------
  SimConfig (hot-path fields)                                  ThinkvConfig
  ThinkvMethod(cfg)            (sim.cpp:494-508)               DecodeRun(cfg)
  ThinkvMethod::process(sv)    (sim.cpp:748-843)               DecodeRun.step(q, k, v, out)
  ThinkvMethod::finish()       (sim.cpp:871-958)               DecodeRun.finish()
  RunOutput.final_block_tables / final_segments / events_jsonl DecodeRun.tables()/segments()/events()
  RunOutput.metrics / step_dumps                               DecodeRun.metrics()/step_dumps()
  thinkv::Error{kind}.exit_code()                              TkvError.code (same numbers)

Inputs q/k/v are torch CUDA tensors (device memory and streams come from
PyTorch; all compute is in the library's sm_100a kernels).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _abi
from ._abi import TkvError, check, lib

__all__ = ["ThinkvConfig", "DecodeRun", "GatherRun", "TkvError", "Context"]


@dataclass
class ThinkvConfig:
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
    psi_bits: Sequence[int] = (4, 4, 2)  # per band: E, R, T (R4E4T2)
    num_thoughts: int = 3
    threshold_fraction: float = 0.01
    prompt_len: int = 0
    max_gen_len: int = 1024
    scripted: bool = True
    script: Optional[List[List[int]]] = None
    per_layer_thought: bool = False
    thresholds: Sequence[float] = ()
    calib_units: Sequence[int] = ()
    input_dtype: str = "bf16"
    record_events: bool = False
    dump_positions: Sequence[int] = ()
    record_sparsity_trace: bool = False

    @property
    def units(self) -> int:
        return self.num_seqs * self.units_per_seq

    @property
    def out_rows(self) -> int:
        return 1 if self.gqa_maxpool else self.num_q_heads

    def to_desc(self):
        import numpy as np
        d = _abi.RunDesc()
        keep = []
        for name in ("num_seqs", "units_per_seq", "num_q_heads", "head_dim", "tau", "group_size",
                     "block_size", "pool_blocks", "budget", "num_thoughts", "threshold_fraction",
                     "prompt_len", "max_gen_len"):
            setattr(d, name, getattr(self, name))
        d.gqa_maxpool = int(self.gqa_maxpool)
        d.num_levels = len(self.levels)
        for i, x in enumerate(self.levels):
            d.levels[i] = int(x)
        for i, b in enumerate(self.psi_bits):
            d.psi_bits[i] = int(b)
        d.scripted = int(self.scripted)
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
        d.input_dtype = _abi.DTYPES[self.input_dtype]
        d.record_events = int(self.record_events)
        d.record_sparsity_trace = int(self.record_sparsity_trace)
        if self.dump_positions:
            dp = np.array(self.dump_positions, dtype=np.int64)
            keep.append(dp)
            d.num_dump_positions = len(dp)
            d.dump_positions = dp.ctypes.data_as(C.POINTER(C.c_int64))
        return d, keep


class Context:
    """One CUDA device (tkv_init)."""

    _by_device = {}

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.tkv_init(device, C.byref(h)))
        self._h = h
        self.device = device

    @classmethod
    def get(cls, device: int = 0) -> "Context":
        if device not in cls._by_device:
            cls._by_device[device] = cls(device)
        return cls._by_device[device]


class DecodeRun:
    """The ThinKV decode path for a batch of sequences on one GPU."""

    def __init__(self, cfg: ThinkvConfig, device: int = 0):
        self.cfg = cfg
        self.ctx = Context.get(device)
        desc, keep = cfg.to_desc()
        h = C.c_void_p()
        check(lib.tkv_run_create(self.ctx._h, C.byref(desc), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.tkv_run_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # -- stepping ---------------------------------------------------------
    @staticmethod
    def _stream(stream):
        # Default: PyTorch's current stream, so the caller's reads/writes of
        # q/k/v/out are ordered with the run (tkv_step joins the two streams).
        if stream is None:
            import torch
            stream = torch.cuda.current_stream()
        return stream.cuda_stream

    def step(self, q, k, v, out, stream=None):
        """q [units,G,d], k/v [units,d] (input dtype), out [units,rows,d] fp32: CUDA tensors."""
        s = self._stream(stream)
        check(lib.tkv_step(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), s))

    def step_layer(self, layer: int, num_layers: int, q, k, v, out, stream=None):
        """One layer of a step (tkv_step_layer): q [seqs,H,G,d], k/v [seqs,H,d],
        out [seqs,H,rows,d]; call layers 0..num_layers-1 in order."""
        s = self._stream(stream)
        check(lib.tkv_step_layer(self._h, layer, num_layers, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                 out.data_ptr(), s))

    def step_kind(self) -> int:
        """The next step's capturable kind (tkv_step_plain): 1 plain (only the
        attention kernel), 2 emission (attention + the window's quantisation),
        0 neither (boundary / eviction: step eagerly).  Keep one captured CUDA
        graph per kind."""
        r = lib.tkv_step_plain(self._h)
        if r < 0:
            check(-r)
        return r

    def step_plain(self) -> bool:
        return self.step_kind() == 1

    def graph_step_begin(self, stream=None):
        """Before each replay of the captured graph of kind step_kind() on
        `stream` (tkv_graph_step_begin): stages the step's scalars and
        advances the run by one step.  Under stream capture, step() /
        step_layer() record the next step's launches instead of executing
        them."""
        check(lib.tkv_graph_step_begin(self._h, self._stream(stream)))

    def step_host(self, q, k, v, out):
        """Same with host (numpy / pinned CPU tensor) buffers, synchronous."""
        ptr = (lambda a: a.ctypes.data) if hasattr(q, "ctypes") else (lambda a: a.data_ptr())
        check(lib.tkv_step_host(self._h, ptr(q), ptr(k), ptr(v), ptr(out)))

    def step_host_async(self, q, k, v, out):
        """Pipelined host-buffer step (tkv_step_host_async): returns after
        enqueueing; buffers stay owned by the run until synchronize()."""
        ptr = (lambda a: a.ctypes.data) if hasattr(q, "ctypes") else (lambda a: a.data_ptr())
        check(lib.tkv_step_host_async(self._h, ptr(q), ptr(k), ptr(v), ptr(out)))

    def synth_inputs(self, seed: int, step: int, q, k, v, stream=None, unit0: int = 0):
        """Synthetic bf16 inputs of global units unit0.. for `step` (csrc/synth.h)."""
        s = self._stream(stream)
        check(lib.tkv_synth_inputs(self._h, seed, unit0, step, q.data_ptr(), k.data_ptr(), v.data_ptr(), s))

    def finish(self):
        check(lib.tkv_finish(self._h))

    def synchronize(self):
        check(lib.tkv_synchronize(self._h))

    @property
    def position(self) -> int:
        return lib.tkv_position(self._h)

    # -- views in the reference's JSON shapes -------------------------------
    def _dump(self, seq: int, what: str) -> str:
        need = C.c_size_t(0)
        check(lib.tkv_dump_json(self._h, seq, what.encode(), None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(lib.tkv_dump_json(self._h, seq, what.encode(), buf, need.value, C.byref(need)))
        return buf.value.decode()

    def tables(self, seq: int = 0):
        return json.loads(self._dump(seq, "tables"))

    def segments(self, seq: int = 0):
        return json.loads(self._dump(seq, "segments"))

    def events(self, seq: int = 0) -> str:
        return self._dump(seq, "events")

    def metrics(self, seq: int = 0):
        return json.loads(self._dump(seq, "metrics"))

    def step_dumps(self, seq: int = 0):
        return json.loads(self._dump(seq, "step_dumps"))

    def sparsity_trace(self, seq: int = 0) -> str:
        """Calibration-trace JSONL line of a sequence (record_sparsity_trace)."""
        return self._dump(seq, "sparsity_trace")

    def bytes(self) -> dict:
        b = _abi.Bytes()
        check(lib.tkv_bytes(self._h, C.byref(b)))
        return {n: getattr(b, n) for n, _ in _abi.Bytes._fields_}

    def bytes_accounting(self, enable: bool = True):
        """Exact per-launch algorithmic bytes on the device (k_bytes.cu); resets the sums."""
        check(lib.tkv_bytes_accounting(self._h, int(enable)))

    def bytes_accumulated(self):
        """(sums over the accounted attention launches as in bytes(), launches)."""
        b, n = _abi.Bytes(), C.c_int64()
        check(lib.tkv_bytes_accumulated(self._h, C.byref(b), C.byref(n)))
        return {f: getattr(b, f) for f, _ in _abi.Bytes._fields_}, n.value

    def export_cache(self, unit0: int = 0, nunits: int = None):
        """Live pager tokens of units [unit0, unit0 + nunits) in the reference
        wire layout (serialize_group, proj/src/quant.cpp:274-324; stream layout
        in csrc/k_export.cu).  Returns (device uint8 tensor, host int64 offsets
        of the nunits + 1 unit streams).  Parse with paper_2510_01290_b200.wire."""
        import numpy as np
        import torch
        nunits = self.cfg.units - unit0 if nunits is None else nunits
        offs = np.zeros(nunits + 1, dtype=np.int64)
        need = C.c_size_t(0)
        check(lib.tkv_export_cache(self._h, unit0, nunits, None, 0, offs.ctypes.data, C.byref(need)))
        buf = torch.empty(max(1, need.value), dtype=torch.uint8, device=torch.device("cuda", self.ctx.device))
        check(lib.tkv_export_cache(self._h, unit0, nunits, buf.data_ptr(), buf.numel(), offs.ctypes.data,
                                   C.byref(need)))
        return buf[:need.value], offs

    def timing_enable(self, enable: bool = True):
        check(lib.tkv_timing_enable(self._h, int(enable)))

    def timing_read(self) -> dict:
        t = _abi.Timing()
        check(lib.tkv_timing_read(self._h, C.byref(t)))
        return {n: getattr(t, n) for n, _ in _abi.Timing._fields_}

    def unit_sparsity(self):
        import numpy as np
        out = np.zeros(self.cfg.units, dtype=np.float64)
        check(lib.tkv_unit_sparsity(self._h, out.ctypes.data, out.size))
        return out


class GatherRun:
    """Gather-compaction comparator (GatherMethod, proj/src/sim.cpp:1117-1206)
    on the GPU: dense full-precision cache, attention-score eviction of the
    lowest head-averaged score once over budget, physical compaction.
    exact=True reproduces the reference's victims (fp64 scores)."""

    def __init__(self, units: int, num_q_heads: int, head_dim: int, budget: int, gqa_maxpool: bool = False,
                 input_dtype: str = "bf16", exact: bool = True, device: int = 0):
        self.ctx = Context.get(device)
        d = _abi.GatherDesc(units, num_q_heads, int(gqa_maxpool), head_dim, budget, _abi.DTYPES[input_dtype],
                            int(exact))
        h = C.c_void_p()
        check(lib.tkv_gather_create(self.ctx._h, C.byref(d), C.byref(h)))
        self._h = h
        self.units, self.rows = units, 1 if gqa_maxpool else num_q_heads

    def close(self):
        if getattr(self, "_h", None):
            lib.tkv_gather_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def step(self, q, k, v, out, prefill: bool = False, stream=None):
        s = DecodeRun._stream(stream)
        check(lib.tkv_gather_step(self._h, int(prefill), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), s))

    def stats(self) -> dict:
        moved, ev = C.c_int64(), C.c_int64()
        check(lib.tkv_gather_stats(self._h, C.byref(moved), C.byref(ev)))
        return {"moved_token_slots": moved.value, "eviction_steps": ev.value}

    def ids(self, unit: int):
        import numpy as np
        n = C.c_int64()
        check(lib.tkv_gather_ids(self._h, unit, None, 0, C.byref(n)))
        buf = np.zeros(max(1, n.value), dtype=np.int64)
        check(lib.tkv_gather_ids(self._h, unit, buf.ctypes.data, n.value, C.byref(n)))
        return buf[:n.value]
