import time, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2307_03738_b200 as q
rng = np.random.default_rng(0)
pms = []
for (K, N) in [(4096, 4096), (4096, 11008), (11008, 4096)]:
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    cm = q.quantize_matrix(w, q.QuantConfig(4, 128))
    pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
xs = [rng.normal(0, 1, pm.n).astype(np.float32) for pm in pms]
refs = [q.qgemv_reference(pm, x) for pm, x in zip(pms, xs)]
for _ in range(3):
    ys = [q.qgemv(pm, x) for pm, x in zip(pms, xs)]
for y, r in zip(ys, refs):
    assert np.abs(y - r).max() / (1 + np.abs(r).max()) < 1e-5
t0 = time.perf_counter()
n = 200
for _ in range(n):
    for pm, x in zip(pms, xs):
        q.qgemv(pm, x)
dt = (time.perf_counter() - t0) / (n * len(pms))
print(f"qgemv(pm, x_numpy): {dt * 1e6:.1f} us per call")
x2 = np.stack([xs[0], xs[0]])
y2 = q.qgemv(pms[0], x2)
assert np.abs(y2[1] - refs[0]).max() / (1 + np.abs(refs[0]).max()) < 1e-5
print("ok")
