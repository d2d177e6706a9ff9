"""Host-side cost of one pipelined host-buffer step call (Python wrapper +
ctypes + the C call's enqueue) vs its GPU time: wall time of issuing E calls
without a sync, then the device time of the same E steps."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_26444_b200 as P  # noqa: E402
from synthetic import inputs as SI  # noqa: E402

dev = torch.device("cuda", 0)
V, d, n, k, Wm, R, E = 128256, 4096, 60, 10, 3072, 8, 64
W = SI.bf16_weights(V, d, seed=0, device=dev)
pools = SI.disjoint_pools(V, Wm + 126, R, seed=3)
states, ups = [], []
for r in range(R):
    prompt, u = SI.cyclic_fresh_updates(pools[r], Wm, 3 * E // R + 4)
    st = P.ActiveVocab(V, Wm, device=dev)
    st.init(0, torch.as_tensor(prompt, device=dev))
    states.append(st)
    ups.append(u)
H = SI.bf16_hidden(n, d, seed=1, device=dev)
for slots in (1, 2):
    io = P.StepHostIO(n, d, 60, 3, k, Wm, dev, slots=slots)
    blocks = [io.pack_inputs(H, ups[s % R][s // R + (slots - 1) * (E // R)][0], ups[s % R][s // R + (slots - 1) * (E // R)][1])
              for s in range(E)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if slots > 1:
        io.copy_stream.wait_event(e0)
    t0 = time.perf_counter()
    for s in range(E):
        P.step_host(states[s % R], 0, io, blocks[s], W, k)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"slots {slots}: host issue {(t1 - t0) / E * 1e6:.1f} us/call, device {e0.elapsed_time(e1) * 1e3 / E:.1f} us/step")
