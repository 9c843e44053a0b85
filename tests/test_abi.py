"""CPU-side checks of the C ABI boundary (no compute calls: no GPU here)."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

import paper_2205_04702_b200 as sp
from paper_2205_04702_b200 import _binding as B


def test_every_header_symbol_is_exported():
    syms = sp.header_symbols()
    assert {"sp_create", "sp_plan", "sp_forward", "sp_train", "sp_flush", "sp_destroy",
            "sp_end_of_data", "sp_surrogate_grad"} <= set(syms)
    for s in syms:
        assert hasattr(sp.lib, s), s


def test_abi_version_matches_header():
    hdr = open(B.HEADER).read()
    v = int(re.search(r"#define SP_ABI_VERSION (\d+)", hdr).group(1))
    assert sp.lib.sp_abi_version() == v


def test_status_codes_match_header():
    hdr = open(B.HEADER).read()
    for name, code in [("SP_OK", 0), ("SP_ERR_INVALID_ARG", 1), ("SP_ERR_CAPACITY", 2),
                       ("SP_ERR_INDEX_RANGE", 3), ("SP_ERR_STATE", 4), ("SP_ERR_CUDA", 5)]:
        assert re.search(rf"\b{name} = {code}\b", hdr), name
        assert B.STATUS_NAMES[code] == name


def test_desc_struct_layout():
    # offsets of the C struct under the x86-64 SysV ABI
    assert B.SpDesc.rows.offset == 8 and B.SpDesc.host_tables.offset == 16
    assert B.SpDesc.stream.offset == 64 and B.SpDesc.policy.offset == 84
    assert B.SpDesc.policy_seed.offset == 96 and B.SpDesc.world.offset == 104
    assert B.SpDesc.nccl_id.offset == 112 and B.SpDesc.table_ids.offset == 136
    assert ctypes.sizeof(B.SpDesc) == 144


def test_invalid_descriptors_rejected_before_touching_a_device():
    h = ctypes.c_void_p()
    assert sp.lib.sp_create(None, ctypes.byref(h)) == sp.SP_ERR_INVALID_ARG
    rows = (ctypes.c_int64 * 1)(100)
    slots = (ctypes.c_int64 * 1)(10)
    tabs = (ctypes.c_void_p * 1)(1)
    base = dict(num_tables=1, rows=rows, host_tables=tabs, dim=16, slots=slots, window=3, past=-1,
                future=-1, batch_size=4, pooling=2, device=0, stream=None, flags=0, log_factor=0,
                host_threads=0, reserved=0)
    for bad in [dict(dim=6), dict(dim=0), dict(num_tables=0), dict(batch_size=0),
                dict(past=1, future=3), dict(policy=3), dict(policy=-1), dict(reserved=1)]:
        d = B.SpDesc(**{**base, **bad})
        assert sp.lib.sp_create(ctypes.byref(d), ctypes.byref(h)) == sp.SP_ERR_INVALID_ARG, bad
    slots[0] = 101  # more slots than rows
    d = B.SpDesc(**base)
    assert sp.lib.sp_create(ctypes.byref(d), ctypes.byref(h)) == sp.SP_ERR_INVALID_ARG


def test_null_context_calls_fail_cleanly():
    assert sp.lib.sp_plan(None, None) == sp.SP_ERR_INVALID_ARG
    assert sp.lib.sp_flush(None) == sp.SP_ERR_INVALID_ARG
    assert sp.lib.sp_error_string(None) == b"null context"


@pytest.mark.skipif(shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"),
                    reason="cuobjdump not available")
def test_library_holds_sm100a_code_only():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", sp.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_context_needs_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        sp.ScratchPipe([10], [None], 4, [4], 2, 1)
