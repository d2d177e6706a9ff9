"""The C-ABI library loads and exports every symbol include/nanospec.h declares;
host-only entry points (sizes, status strings) behave as documented.  No
compute calls: runs without a GPU."""
import ctypes
import json
import os
import re

import pytest

from paper_2605_26444_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nanospec.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nanospec_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    L = N.lib()
    decl = _declared()
    assert len(decl) >= 17
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(N.EXPORTS) == decl


def test_abi_version_and_status_strings():
    L = N.lib()
    assert L.nanospec_abi_version() == 1
    for s in range(6):
        assert N.status_str(s)
    assert N.status_str(N.EEMPTY) == "empty prompt"


def _a(x):
    return (x + 255) // 256 * 256


def test_workspace_layout_and_table6_sizes():
    """Per-sequence state = bitmap ceil(V/32)*4 (the paper's 16 KB `token_ids`,
    T6 P:449) + ids W*4 (12 KB at W=3072) + ring W*4 + cnt V*4 + pos V*4 +
    first V*4 + 16-byte meta; independent of context length."""
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_table6.json")))
    V, W = gold["vocab"], gold["w_max"]
    L = N.lib()
    words = (V + 31) // 32
    assert words * 4 == gold["exact_bytes"]["token_ids"]
    assert W * 4 == gold["exact_bytes"]["tokens_tensor"]
    assert W * gold["d_model"] * 2 == gold["exact_bytes"]["repack_buf"]  # what one head call reads at |I| = W
    got = L.nanospec_state_workspace_bytes(V, W, 1, 0, 0, 1)
    assert got == _a(16) + _a(words * 4) + _a(W * 4) * 2 + _a(V * 4) * 3
    # R2 keeps no cnt / pos arrays
    assert L.nanospec_state_workspace_bytes(V, W, 1, 1, 0, 1) == got - 2 * _a(V * 4)
    # batch scales linearly (one state per sequence)
    assert L.nanospec_state_workspace_bytes(V, W, 64, 0, 0, 1) >= 64 * (words * 4 + W * 8 + V * 12)
    # vocab-parallel shard: bitmap/cnt/pos over V_local, first over V
    vl = (V - 3 + 7) // 8
    assert L.nanospec_state_workspace_bytes(V, W, 1, 0, 3, 8) == \
        _a(16) + _a(((vl + 31) // 32) * 4) + _a(W * 4) * 2 + _a(vl * 4) * 2 + _a(V * 4)


@pytest.mark.parametrize("args", [(0, 10, 1, 0, 0, 1), (10, 0, 1, 0, 0, 1), (10, 10, 0, 0, 0, 1),
                                  (10, 10, 1, 7, 0, 1), (10, 10, 1, 0, 2, 2), (10, 10, 1, 0, -1, 2)])
def test_invalid_geometry_returns_zero(args):
    assert N.lib().nanospec_state_workspace_bytes(*args) == 0


def test_head_scratch_bytes():
    L = N.lib()
    assert L.nanospec_head_scratch_bytes(1, 3072, 60) >= 60 * 3072 * 4
    assert L.nanospec_head_scratch_bytes(1, 3072, 0) == 0
    assert L.nanospec_head_scratch_bytes(1, 3072, 257) == 0
    assert L.nanospec_head_scratch_bytes(0, 3072, 1) == 0


def test_host_validation_without_gpu():
    """Null handles / pointers are rejected before anything is launched."""
    L = N.lib()
    assert L.nanospec_state_init(None, 0, None, 1, None, 0, None) == N.EINVAL
    assert L.nanospec_state_update(None, 0, None, 0, None, 0, None) == N.EINVAL
    h = ctypes.c_void_p()
    assert L.nanospec_state_create(ctypes.byref(h), 10, 10, 1, 0, 0, 1, None, 0, None) == N.EINVAL
    assert L.nanospec_state_create(ctypes.byref(h), 10, 10, 1, 1, 0, 2, None, 1 << 20, None) in (N.EINVAL,
                                                                                                  N.EUNSUPPORTED)
    assert L.nanospec_merge_topk(None, None, None, 1, 1, 1, None, None, None, None) == N.EINVAL
    assert L.nanospec_draft_logits_topk(None, None, 8, 8, None, 1, 1, None, None, None, None, None, 0, None) \
        == N.EINVAL
