"""Loads the C-ABI library libnanospec.so (include/nanospec.h) with ctypes.

There is no fallback: if the library is missing or fails to load, importing the
product API raises.  Build it with ``python -m paper_2605_26444_b200.build``
(``__graft_entry__.build()`` does the same).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnanospec.so")

OK, EINVAL, EEMPTY, ECUDA, EDEVICE, EUNSUPPORTED = range(6)

# Every symbol include/nanospec.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "nanospec_abi_version", "nanospec_status_str",
    "nanospec_state_workspace_bytes", "nanospec_state_create", "nanospec_state_destroy",
    "nanospec_state_init", "nanospec_state_update", "nanospec_state_update_batch",
    "nanospec_state_read", "nanospec_state_check", "nanospec_state_ids_ptr", "nanospec_state_n_active_ptr",
    "nanospec_head_scratch_bytes", "nanospec_draft_logits_topk", "nanospec_draft_logits_topk_ex",
    "nanospec_logits_topk_ids", "nanospec_merge_topk", "nanospec_debug_set_trace",
    "nanospec_debug_set_head_mode", "nanospec_step", "nanospec_step_fused", "nanospec_step_debug",
    "nanospec_step_host", "nanospec_step_host_async", "nanospec_step_host_io_bytes", "nanospec_tree_expand", "nanospec_tree_rerank",
    "nanospec_repack", "nanospec_draft_logits_topk_packed",
]


class NanoSpecError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_str(status)} (status {status})")


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2605_26444_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    L.nanospec_abi_version.restype = i32
    L.nanospec_status_str.argtypes = [ctypes.c_int]
    L.nanospec_status_str.restype = ctypes.c_char_p
    L.nanospec_state_workspace_bytes.argtypes = [i32, i32, i32, ctypes.c_int, i32, i32]
    L.nanospec_state_workspace_bytes.restype = sz
    L.nanospec_state_create.argtypes = [ctypes.POINTER(vp), i32, i32, i32, ctypes.c_int, i32, i32, vp, sz, vp]
    L.nanospec_state_destroy.argtypes = [vp]
    L.nanospec_state_init.argtypes = [vp, i32, vp, i64, vp, i32, vp]
    L.nanospec_state_update.argtypes = [vp, i32, vp, i32, vp, i32, vp]
    L.nanospec_state_update_batch.argtypes = [vp, vp, i32, vp, i32, vp]
    L.nanospec_state_read.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp]
    L.nanospec_state_check.argtypes = [vp, vp]
    L.nanospec_state_ids_ptr.argtypes = [vp, i32]
    L.nanospec_state_ids_ptr.restype = vp
    L.nanospec_state_n_active_ptr.argtypes = [vp, i32]
    L.nanospec_state_n_active_ptr.restype = vp
    L.nanospec_head_scratch_bytes.argtypes = [i32, i32, i32]
    L.nanospec_head_scratch_bytes.restype = sz
    L.nanospec_draft_logits_topk.argtypes = [vp, vp, i32, i64, vp, i32, i32, vp, vp, vp, vp, vp, sz, vp]
    L.nanospec_draft_logits_topk_ex.argtypes = [vp, vp, i32, i64, vp, i32, i32, vp, vp, vp, vp, vp, sz,
                                                ctypes.c_int, vp]
    L.nanospec_logits_topk_ids.argtypes = [vp, vp, i32, i32, vp, i32, i64, vp, i32, i32, vp, vp, vp, vp, vp, sz,
                                           ctypes.c_int, vp]
    L.nanospec_merge_topk.argtypes = [vp, vp, vp, i32, i32, i32, vp, vp, vp, vp]
    L.nanospec_debug_set_trace.argtypes = [vp, i32]
    L.nanospec_debug_set_head_mode.argtypes = [i32]
    L.nanospec_step_host_io_bytes.argtypes = [i32, i32, i32, i32, i32, ctypes.POINTER(sz), ctypes.POINTER(sz)]
    L.nanospec_step_host_io_bytes.restype = sz
    L.nanospec_step_host.argtypes = [vp, i32, vp, i32, i32, vp, i32, i64, i32, i32, vp, vp, sz, vp, sz, vp]
    L.nanospec_step_host_async.argtypes = [vp, i32, vp, i32, i32, vp, i32, i64, i32, i32, vp, vp, sz, vp, sz, vp, vp,
                                           vp, vp]
    L.nanospec_step_fused.argtypes = [vp, i32, i32, i32, i32, i32]
    L.nanospec_step.argtypes = [vp, i32, vp, i32, vp, i32, vp, i32, i64, vp, i32, i32, vp, vp, vp, vp, sz, vp]
    L.nanospec_repack.argtypes = [vp, i32, vp, i32, i64, vp, i64, vp, vp]
    L.nanospec_draft_logits_topk_packed.argtypes = [vp, vp, i32, i64, vp, i32, i32, vp, vp, vp, vp, sz, vp]
    L.nanospec_tree_expand.argtypes = [vp, vp, i32, vp, vp, vp, i32, vp, vp, vp, i32, i32, i32, vp, vp, vp]
    L.nanospec_tree_rerank.argtypes = [vp, vp, i32, i32, vp, vp, vp]
    L.nanospec_step_debug.argtypes = [vp, i32, vp, i32, vp, i32, vp, i32, i64, vp, i32, i32, vp, vp, vp, vp, vp, sz,
                                      vp]
    _lib = L
    return L


def status_str(s: int) -> str:
    return lib().nanospec_status_str(int(s)).decode()


def check(status: int, what: str):
    if status != OK:
        raise NanoSpecError(status, what)
