import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_gpu_layer as L
import oracle as O
from paper_2603_08026_b200 import dyllm
res = {}
_orig = L.unpack_lists
def rec(rows, off, N):
    out = _orig(rows, off, N); res['got'] = out; return out
L.unpack_lists = rec
_ls = dyllm.Cache.layer_step
def ls(self, layer, mode, idx, off, tau, io, oo, sim=None):
    res['tau'] = tau; res['sim'] = sim; res['cache'] = self; res['layer'] = layer
    return _ls(self, layer, mode, idx, off, tau, io, oo, sim)
dyllm.Cache.layer_step = ls
_sl = O.sparse_layer
calls = []
def sl(*a, **k):
    r = _sl(*a, **k); calls.append(r); return r
O.sparse_layer = sl
try:
    L._teacher_forced_layer("small64", 1, "fi")
except AssertionError as e:
    print("assert", e)
b = 2
refs = calls[-b:]
sim = res['sim'].cpu().numpy().reshape(b, -1)
C = res['cache'].export(1, dyllm.CTX).float().cpu().numpy()
print("tau", res['tau'])
for s in range(b):
    r = refs[s]
    got = set(res['got'][s].tolist()); ref = set(r.idx_out.tolist())
    print("seq", s, "diff", sorted(got ^ ref), "max s err", np.abs(sim[s] - r.s).max(), "argmax", np.argmax(np.abs(sim[s]-r.s)))
    for row in sorted(got ^ ref):
        print("  row", row, "s_oracle", r.s[row], "s_gpu", sim[s, row])
        print("  C gpu", C[s,row,:8], "\n  C ref", r.C[row,:8])
        print("  rel", np.abs(C[s,row]-r.C[row]).max()/np.abs(r.C[row]).max())
