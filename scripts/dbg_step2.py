import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_26444_b200 as P
from synthetic import inputs as SI
dev = torch.device("cuda", 0)
V, d, Wm, n, k = 128256, 4096, 3072, 60, 10
W = SI.bf16_weights(V, d, seed=0, device=dev)
R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mode = sys.argv[2] if len(sys.argv) > 2 else "eager"
pools = SI.disjoint_pools(V, Wm + 126, R, seed=3)
states, outs, ud, uv = [], [], [], []
Hs = SI.bf16_hidden(n, d, seed=1, device=dev, batch=R)
for r in range(R):
    prompt, ups = SI.cyclic_fresh_updates(pools[r], Wm, 40)
    st = P.ActiveVocab(V, Wm, device=dev); st.init(0, torch.as_tensor(prompt, device=dev)); states.append(st)
    outs.append(P.HeadOutputs(1, n, k, Wm, dev))
    ud.append(torch.as_tensor(np.stack([u[0] for u in ups]), device=dev)); uv.append(torch.as_tensor(np.stack([u[1] for u in ups]), device=dev))
print("fused:", P.step_is_fused(states[0], 60, 3, d, n, k))
cur = [0] * R
def step(s):
    r = s % R; c = cur[r]; cur[r] += 1
    P.step(states[r], 0, ud[r][c], uv[r][c], W, Hs[r], k, out=outs[r])
torch.cuda.synchronize()
stream = torch.cuda.Stream(dev); torch.cuda.set_stream(stream)
if mode == "eager":
    for s in range(8 * R):
        step(s)
        if "sync" in sys.argv: torch.cuda.synchronize()
    torch.cuda.synchronize(); print("eager ok")
else:
    for s in range(2 * R): step(s)
    torch.cuda.synchronize(); print("warm ok")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for s in range(4 * R): step(s)
    g.replay(); torch.cuda.synchronize(); print("graph ok")
