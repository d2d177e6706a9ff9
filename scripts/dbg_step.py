import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2605_26444_b200 as P
from oracle import oracle as O
from synthetic import inputs as SI
t = lambda a: torch.as_tensor(np.asarray(a, np.int32), device="cuda")
W = SI.bf16_weights(128256, 4096, seed=0, device="cuda"); Wb = SI.bf16_bits(W)
V, d = W.shape; Wm, n, k = 256, 16, 10
rng = np.random.default_rng(4)
st = P.ActiveVocab(V, Wm); prompt = rng.integers(0, V, 300); st.init(0, t(prompt))
ref = O.OracleStream(V, Wm).init(prompt)
before = set(ref.active()[0].tolist())
g0 = st.read(0)
dd = rng.integers(0, V, 60); dd[::7] = dd[1]; vv = rng.integers(0, V, 3)
H = SI.bf16_hidden(n, d, seed=300, device="cuda")
v, i, l = P.step(st, 0, t(dd), t(vv), W, H, k)
torch.cuda.synchronize()
ref.update(dd, vv)
ids = ref.active()[0]
after = set(ids.tolist())
print("n_old", g0["n_active"], "n_new", len(ids), "enter", len(after - before), "leave", len(before - after))
z, A = O.logits(Wb, SI.bf16_bits(H), ids)
vr, ir = O.topk(z, ids, k)
for node in range(n):
    if i[0, node, 0].item() != ir[node, 0]:
        g = int(ir[node, 0]); print("node", node, "gpu", i[0, node, :4].tolist(), "ref", ir[node, :4].tolist(), "ref-top in before:", g in before, "entering:", g not in before)
# compare with separate calls on a fresh copy
st2 = P.ActiveVocab(V, Wm); st2.init(0, t(prompt)); st2.update(0, t(dd), t(vv))
v2, i2, l2, _ = P.draft_logits_topk(st2, W, H.reshape(1, n, d), k)
torch.cuda.synchronize()
print("separate == ref top1:", (i2[0, :, 0].cpu().numpy() == ir[:, 0]).all())
print("fused lse", l[0, :4].tolist(), "ref lse", O.lse(z)[:4].tolist())
print("lse diff per node", np.round(l[0].cpu().numpy() - O.lse(z), 4).tolist())
for Wm2, n2 in ((3072, 16), (256, 8), (512, 16), (256, 24)):
    rng = np.random.default_rng(4)
    st = P.ActiveVocab(V, Wm2); prompt = rng.integers(0, V, Wm2 + 44); st.init(0, t(prompt))
    ref = O.OracleStream(V, Wm2).init(prompt)
    dd = rng.integers(0, V, 60); vv = rng.integers(0, V, 3)
    H = SI.bf16_hidden(n2, d, seed=300, device="cuda")
    v, i, l = P.step(st, 0, t(dd), t(vv), W, H, k)
    torch.cuda.synchronize(); ref.update(dd, vv); ids = ref.active()[0]
    z, A = O.logits(Wb, SI.bf16_bits(H), ids); vr, ir = O.topk(z, ids, k)
    bad = [nd for nd in range(n2) if i[0, nd, 0].item() != ir[nd, 0]]
    print("W", Wm2, "n", n2, "bad nodes", bad)
