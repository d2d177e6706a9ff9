"""A tiny end-to-end pass of every kernel of the path, for compute-sanitizer
(memcheck / synccheck / racecheck / initcheck): state init + update (fast and
general paths, rule R2), the CUDA-core head + select, the tensor-core head
(stream + select kernels; split-K > 1, persistent, list mode + merge), the
fused step (device and pipelined host buffers), the
vocab-parallel merge, the draft-tree expansion / rerank and the repack variant.

    compute-sanitizer --tool memcheck python scripts/sanitize.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26444_b200 as P  # noqa: E402
from synthetic import inputs as SI  # noqa: E402


def t(a):
    return torch.as_tensor(np.asarray(a, np.int32), device="cuda")


def main():
    torch.cuda.set_device(0)
    V, d, n, k = 3000, 128, 8, 10
    W = SI.bf16_weights(V, d, seed=0, device="cuda")
    z = SI.Zipf(V)
    prompt, pre = SI.prompt_and_prefill(z, 2, 300, 3)
    for rule in ("window", "unique_fifo"):
        st = P.ActiveVocab(V, 256, rule=rule)
        st.init(0, t(prompt), t(pre))
        for dd, vv in SI.decode_steps(z, 3, 2, n_draft=8, k_ver=3):
            st.update(0, t(dd), t(vv))
        H = SI.bf16_hidden(n, d, seed=1, device="cuda").reshape(1, n, d)
        for impl in ("simt", "tc"):
            P.draft_logits_topk(st, W, H, k, impl=impl, debug_logits=True)
    st = P.ActiveVocab(V, 1024)
    st.init(0, t(prompt), t(pre))
    out = P.HeadOutputs(1, n, k, 1024, "cuda")
    for dd, vv in SI.decode_steps(z, 5, 2, n_draft=8, k_ver=3):
        H = SI.bf16_hidden(n, d, seed=2, device="cuda")
        P.step(st, 0, t(dd), t(vv), W, H, k, out=out)
        P.step_debug(st, 0, t(dd), t(vv), W, H, k, out=out)
    # persistent tensor-core head (tiles > SMs would be large; a batch of 3 instead)
    stb = P.ActiveVocab(V, 512, batch=3)
    for b in range(3):
        stb.init(b, t(prompt[: 100 + 50 * b]))
    P.draft_logits_topk(stb, W, SI.bf16_hidden(n, d, seed=3, device="cuda", batch=3), k)
    # list mode (more tiles than SMs, split-K 1): the dense head over [0, V2),
    # 313 tiles -> 148 tile-pair units + 17 single-tile units, lists + merge
    V2 = 40000
    W2 = SI.bf16_weights(V2, d, seed=9, device="cuda")
    allids = torch.arange(V2, dtype=torch.int32, device="cuda")
    P.logits_topk_ids(allids, torch.tensor([V2], dtype=torch.int32, device="cuda"), W2,
                      SI.bf16_hidden(n, d, seed=10, device="cuda"), k, debug_logits=True)
    # host-buffer steps, pipelined (copy stream + two staging slots)
    io = P.StepHostIO(n, d, 8, 3, k, 1024, "cuda", slots=2)
    for dd, vv in SI.decode_steps(z, 9, 3, n_draft=8, k_ver=3):
        P.step_host(st, 0, io, io.pack_inputs(SI.bf16_hidden(n, d, seed=11, device="cuda"), dd, vv), W, k)
    torch.cuda.synchronize()
    # vocab-parallel merge of two shards
    v, i, l, _ = P.draft_logits_topk(st, W, SI.bf16_hidden(n, d, seed=4, device="cuda").reshape(1, n, d), k)
    P.merge_topk(torch.stack([v[0], v[0]]), torch.stack([i[0], i[0]]), torch.stack([l[0], l[0]]), k)
    # draft tree
    tree = P.DraftTree(1 + k + 2 * 4 * k, 4, "cuda")
    o1, o4 = P.HeadOutputs(1, 1, k, 1024, "cuda"), P.HeadOutputs(1, 4, k, 1024, "cuda")
    P.draft_logits_topk(st, W, SI.bf16_hidden(1, d, seed=5, device="cuda").reshape(1, 1, d), k, out=o1)
    tree.expand(o1.topk_logit[0], o1.topk_id[0], o1.lse[0], 4)
    for lvl in range(2):
        P.draft_logits_topk(st, W, SI.bf16_hidden(4, d, seed=6 + lvl, device="cuda").reshape(1, 4, d), k, out=o4)
        tree.expand(o4.topk_logit[0], o4.topk_id[0], o4.lse[0], 4)
    tree.rerank(16)
    # repack variant
    ph = P.PackedHead(st, d, "cuda")
    ph.refresh(0, W)
    ph.head(SI.bf16_hidden(n, d, seed=8, device="cuda").reshape(1, n, d), k, P.HeadOutputs(1, n, k, 1024, "cuda"))
    torch.cuda.synchronize()
    assert st.check() == 0
    print("sanitize pass done")


if __name__ == "__main__":
    main()
