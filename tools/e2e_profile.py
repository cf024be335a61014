"""Host-side cost breakdown of qgemv_batch over the configs[1] sweep."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import runtime as R  # noqa: E402
SWEEP = [(b, g, shp) for shp in [(4096, 4096), (4096, 11008), (11008, 4096)]
         for b in (2, 3, 4) for g in (32, 64, 128, None)]
pms, xs = [], []
for i, (b, g, (K, N)) in enumerate(SWEEP):
    w = torch.randn(K, N, device="cuda") * 0.02
    cm = q.quantize_matrix(w, q.QuantConfig(b, g))
    pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
    xs.append(np.random.default_rng(i).normal(0, 1, K).astype(np.float32))
q.qgemv_batch(pms, xs)
b = next(iter(R._BATCHES.values()))
torch.cuda.synchronize()
def t(f, n=50):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6
print("full qgemv_batch      %.1f us" % t(lambda: q.qgemv_batch(pms, xs)))
print("concatenate           %.1f us" % t(lambda: np.concatenate(xs, out=b.xh_np)))
print("H2D                   %.1f us" % t(lambda: b.x.copy_(b.xh, non_blocking=True)))
print("group.run             %.1f us" % t(lambda: b.group.run()))
print("D2H                   %.1f us" % t(lambda: b.yh.copy_(b.y, non_blocking=True)))
print("yh copy + split       %.1f us" % t(lambda: np.split(b.yh_np.copy(), b.noff[1:-1])))
print("shape checks          %.1f us" % t(lambda: [tuple(x.shape) for x in xs]))

def manual():
    ts = [time.perf_counter()]
    key = tuple(id(pm) for pm in pms)
    bb = R._BATCHES.pop(key, None); R._BATCHES[key] = bb
    ts.append(time.perf_counter())
    host = all(R._dev.is_host(x) for x in xs)
    for i, (pw, x) in enumerate(zip(bb.pws, xs)):
        shp = tuple(x.shape)
    ts.append(time.perf_counter())
    np.concatenate(xs, out=bb.xh_np, casting="same_kind")
    ts.append(time.perf_counter())
    bb.x.copy_(bb.xh, non_blocking=True)
    ts.append(time.perf_counter())
    bb.group.run()
    ts.append(time.perf_counter())
    bb.yh.copy_(bb.y, non_blocking=True)
    ts.append(time.perf_counter())
    torch.cuda.current_stream().synchronize()
    ts.append(time.perf_counter())
    r = np.split(bb.yh_np.copy(), bb.noff[1:-1])
    ts.append(time.perf_counter())
    return np.diff(ts) * 1e6
acc = np.zeros(8)
for _ in range(50):
    acc += manual()
print("manual phases (us): lookup %.1f checks %.1f concat %.1f h2d-issue %.1f run-issue %.1f d2h-issue %.1f sync %.1f split %.1f" % tuple(acc / 50))
