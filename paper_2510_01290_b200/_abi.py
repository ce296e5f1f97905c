"""ctypes binding of include/thinkv_b200.h (libthinkv_b200.so, built in-tree).

The library is the product: there is no Python or CPU fallback.  The shared
library is loaded on first use (the first `lib.<symbol>` access, e.g. when a
DecodeRun is created) and that use raises if it is missing.  Loading lazily
keeps processes that only need the configuration types -- bench.py's CPU
reference arm -- from mapping the CUDA library at all.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libthinkv_b200.so")

# Every symbol include/thinkv_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "tkv_last_error", "tkv_abi_version", "tkv_init", "tkv_ctx_destroy", "tkv_run_create",
    "tkv_run_destroy", "tkv_step", "tkv_step_layer", "tkv_step_host", "tkv_finish", "tkv_synchronize",
    "tkv_position", "tkv_dump_json", "tkv_bytes", "tkv_unit_sparsity", "tkv_synth_inputs",
    "tkv_timing_enable", "tkv_timing_read", "tkv_bytes_accounting", "tkv_bytes_accumulated", "tkv_exp_f64", "tkv_step_host_async", "tkv_export_cache",
    "tkv_step_plain", "tkv_graph_step_begin",
    "tkv_dropin_quantize_window", "tkv_dropin_decode", "tkv_dropin_gqa_attend", "tkv_dropin_sparsity",
    "tkv_dropin_kmeans_select", "tkv_dropin_pager_place", "tkv_dropin_pager_evict",
    "tkv_gather_create", "tkv_gather_destroy", "tkv_gather_step", "tkv_gather_stats", "tkv_gather_ids",
)

STATUS = {0: "ok", 1: "unexpected", 2: "config", 3: "calibration", 4: "out_of_memory",
          5: "integrity"}

DTYPES = {"bf16": 0, "f32": 1, "f64": 2}


class RunDesc(C.Structure):
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
        ("input_dtype", C.c_int32), ("record_events", C.c_int32),
        ("num_dump_positions", C.c_int32), ("dump_positions", C.POINTER(C.c_int64)),
        ("record_sparsity_trace", C.c_int32),
    ]


class Bytes(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "live_slots", "resident_slots", "live_code_bytes", "live_scale_bytes", "buffer_bytes",
        "qo_bytes", "meta_bytes", "algorithmic_bytes")]


class Timing(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("attend_ms", "score_ms", "flush_ms", "anneal_ms", "apply_ms")] + \
               [(n, C.c_int64) for n in ("attend_launches", "score_launches", "flush_launches",
                                         "anneal_launches", "apply_launches", "total_launches")] + \
               [("host_ms", C.c_double), ("host_wait_ms", C.c_double), ("steps", C.c_int64)]


class GatherDesc(C.Structure):
    _fields_ = [("num_units", C.c_int32), ("num_q_heads", C.c_int32), ("gqa_maxpool", C.c_int32),
                ("head_dim", C.c_int32), ("budget", C.c_int64), ("input_dtype", C.c_int32),
                ("exact_scores", C.c_int32)]


class TkvError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{STATUS.get(code, code)}] {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the ThinKV decode path)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.tkv_last_error.restype = C.c_char_p
    L.tkv_abi_version.restype = C.c_int
    L.tkv_init.argtypes = [C.c_int, C.POINTER(vp)]
    L.tkv_ctx_destroy.argtypes = [vp]
    L.tkv_run_create.argtypes = [vp, C.POINTER(RunDesc), C.POINTER(vp)]
    L.tkv_run_destroy.argtypes = [vp]
    L.tkv_step.argtypes = [vp, vp, vp, vp, vp, vp]
    L.tkv_step_host.argtypes = [vp, vp, vp, vp, vp]
    L.tkv_step_layer.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, vp, vp]
    L.tkv_step_host_async.argtypes = [vp, vp, vp, vp, vp]
    L.tkv_step_plain.argtypes = [vp]
    L.tkv_graph_step_begin.argtypes = [vp, vp]
    L.tkv_finish.argtypes = [vp]
    L.tkv_synchronize.argtypes = [vp]
    L.tkv_position.argtypes = [vp]
    L.tkv_position.restype = C.c_int64
    L.tkv_dump_json.argtypes = [vp, C.c_int, C.c_char_p, C.c_char_p, C.c_size_t,
                                C.POINTER(C.c_size_t)]
    L.tkv_bytes.argtypes = [vp, C.POINTER(Bytes)]
    L.tkv_exp_f64.argtypes = [vp, vp, vp, C.c_int64]
    L.tkv_bytes_accounting.argtypes = [vp, C.c_int]
    L.tkv_bytes_accumulated.argtypes = [vp, C.POINTER(Bytes), C.POINTER(C.c_int64)]
    L.tkv_export_cache.argtypes = [vp, C.c_int64, C.c_int64, vp, C.c_size_t, vp, C.POINTER(C.c_size_t)]
    L.tkv_unit_sparsity.argtypes = [vp, vp, C.c_int64]
    L.tkv_timing_enable.argtypes = [vp, C.c_int]
    L.tkv_timing_read.argtypes = [vp, C.POINTER(Timing)]
    L.tkv_synth_inputs.argtypes = [vp, C.c_uint64, C.c_int64, C.c_int64, vp, vp, vp, vp]
    L.tkv_gather_create.argtypes = [vp, C.POINTER(GatherDesc), C.POINTER(vp)]
    L.tkv_gather_destroy.argtypes = [vp]
    L.tkv_gather_step.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp]
    L.tkv_gather_stats.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.tkv_gather_ids.argtypes = [vp, C.c_int, vp, C.c_int64, C.POINTER(C.c_int64)]
    return L


class _LazyLib:
    """Proxy for the CDLL: resolves it on the first attribute access."""

    def __init__(self):
        self.__dict__["_cdll"] = None

    def __getattr__(self, name):
        cdll = self.__dict__["_cdll"]
        if cdll is None:
            cdll = self.__dict__["_cdll"] = _load()
        return getattr(cdll, name)


lib = _LazyLib()


def check(rc: int):
    if rc != 0:
        raise TkvError(rc, lib.tkv_last_error().decode(errors="replace"))
