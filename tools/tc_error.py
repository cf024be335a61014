import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2307_03738_b200 as q
from oracle import qigen_oracle as orc
K = N = 8192
for M in (16, 64):
    rng = np.random.default_rng(99 + M)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    codes, s, z = orc.quantize_matrix(w, 4, 64)
    cm = q.quantize_matrix(w, q.QuantConfig(4, 64))
    pw = q.PanelWeights.from_codes(cm)
    X = rng.normal(0, 1, (M, K)).astype(np.float32)
    ref = orc.qgemv_reference(codes, s, z, X)
    Y = pw.gemv(torch.from_numpy(X).cuda(), path="tc").cpu().numpy()
    Yg = pw.gemv(torch.from_numpy(X).cuda(), path="gemv").cpu().numpy()
    e = lambda a: np.abs(a - ref).max() / (1 + np.abs(ref).max())
    print(f"M={M}: tcgen05 path rel err {e(Y):.2e}, IMMA path {e(Yg):.2e}")
