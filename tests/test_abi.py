"""CPU checks of the C-ABI boundary (no GPU needed): the in-tree library
loads, exports every symbol include/thinkv_b200.h declares, and rejects
invalid configurations with the reference's error codes before touching a
device."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "thinkv_b200.h")).read()
    return sorted(set(re.findall(r"\b(tkv_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2510_01290_b200 import _abi
    lib = C.CDLL(_abi.LIB_PATH)
    syms = header_symbols()
    assert syms, "no declarations parsed"
    for s in syms:
        assert hasattr(lib, s), f"{s} missing from libthinkv_b200.so"
    assert sorted(_abi.EXPORTS) == syms
    assert lib.tkv_abi_version() == 2


def test_library_is_sm100a():
    from paper_2510_01290_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _desc(**kw):
    from paper_2510_01290_b200 import ThinkvConfig
    return ThinkvConfig(**kw).to_desc()


@pytest.mark.parametrize("bad,msg", [
    (dict(levels=(4, 8)), "strictly descending"),
    (dict(budget=2, levels=(4,)), "budget must be"),
    (dict(block_size=64), "block_size"),
    (dict(psi_bits=(4, 3, 2)), "unsupported precision"),
    (dict(scripted=False), "thresholds"),
    (dict(script=[[7]]), "scripted band out of range"),
    (dict(scripted=False, thresholds=(0.3, 0.6), calib_units=(5,)), "calibration layer index out of range"),
])
def test_config_validation_codes(bad, msg):
    from paper_2510_01290_b200 import _abi
    base = dict(num_seqs=1, units_per_seq=1, num_q_heads=1, head_dim=16, tau=16, group_size=8,
                block_size=4, budget=64, levels=(8, 4), max_gen_len=32, script=[[1]])
    base.update(bad)
    desc, keep = _desc(**base)
    h = C.c_void_p()
    rc = _abi.lib.tkv_run_create(None, C.byref(desc), C.byref(h))
    assert rc == 2  # thinkv::ErrorKind::kConfig -> exit code 2
    assert msg in _abi.lib.tkv_last_error().decode()


def test_valid_config_needs_a_context():
    from paper_2510_01290_b200 import _abi
    desc, keep = _desc(num_seqs=1, units_per_seq=1, num_q_heads=1, head_dim=16, tau=16,
                       group_size=8, block_size=4, budget=64, levels=(8, 4), max_gen_len=32,
                       script=[[1]])
    h = C.c_void_p()
    assert _abi.lib.tkv_run_create(None, C.byref(desc), C.byref(h)) == 2
