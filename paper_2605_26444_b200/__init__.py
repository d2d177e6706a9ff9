"""B200-native NanoSpec hot path: the draft LM head restricted to a per-step,
context-derived active vocabulary (arxiv 2605.26444).

    from paper_2605_26444_b200 import ActiveVocab, draft_logits_topk

The compute lives in libnanospec.so (C ABI, include/nanospec.h); this package
is a thin ctypes binding.  Importing it loads the library and fails loudly if
it is missing -- there is no CPU fallback.
"""
from ._native import lib as _lib

_lib()  # fail loudly at import if the native library is missing

from .nanospec import (  # noqa: E402
    ActiveVocab,
    DraftTree,
    HeadOutputs,
    PackedHead,
    draft_logits_topk,
    head_scratch_bytes,
    logits_topk_ids,
    merge_topk,
    state_workspace_bytes,
    StepHostIO,
    step,
    step_debug,
    step_host,
    step_is_fused,
)

__all__ = [
    "ActiveVocab", "DraftTree", "HeadOutputs", "PackedHead", "draft_logits_topk", "logits_topk_ids", "merge_topk",
    "head_scratch_bytes", "state_workspace_bytes", "step", "step_debug", "step_host", "StepHostIO", "step_is_fused",
]
