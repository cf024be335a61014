"""Per-CTA start/end of the grouped GEMV kernel in a replayed graph (imbalance)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402
dev = torch.device("cuda")
SWEEP = [(b, g, shp) for shp in [(4096, 4096), (4096, 11008), (11008, 4096)]
         for b in (2, 3, 4) for g in (32, 64, 128, None)]
ent = []
for i, (b, g, (K, N)) in enumerate(SWEEP):
    pw = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, q.QuantConfig(b, g))
    ent.append((pw, torch.randn(K, device=dev), torch.zeros(N, device=dev)))
grp = q.GemvGroup(ent)
L = _lib.lib()
bufs = [torch.zeros(148 * 4, dtype=torch.int64, device=dev) for _ in range(4)]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    grp.run(); s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for b_ in bufs:
            L.qigen_debug_trace(b_.data_ptr()); grp.run()
        L.qigen_debug_trace(None)
    g.replay(); s.synchronize()
    for b_ in bufs: b_.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s); g.replay(); e1.record(s); e1.synchronize()
print(f"4 runs in {e0.elapsed_time(e1)*1e3:.1f} us")
t = [b_.view(-1, 4).cpu().numpy() for b_ in bufs]
t0 = t[0][:, 0].min()
for i, x in enumerate(t):
    st, en = (x[:, 0] - t0) / 1e3, (x[:, 3] - t0) / 1e3
    if x[:, 1].min() > 0:
        p1, bar = (x[:, 1] - t0) / 1e3, (x[:, 2] - t0) / 1e3
        print(f"   phase1 done {p1.min():7.2f}-{p1.max():7.2f}  barrier out {bar.min():7.2f}-{bar.max():7.2f}")
    d = en - st
    print(f"run {i}: start {st.min():7.2f}-{st.max():7.2f}  end {en.min():7.2f}-{en.max():7.2f}  "
          f"dur min/med/max {d.min():6.1f}/{np.median(d):6.1f}/{d.max():6.1f}")
en = (t[1][:, 3] - t[1][:, 0].min()) / 1e3
print("run 1 CTA end percentiles (us from first start): " +
      " ".join(f"p{p}={np.percentile(en, p):.1f}" for p in (0, 10, 25, 50, 75, 90, 100)))
