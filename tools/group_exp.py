"""Grouped GEMV vs per-GEMV launches over the BASELINE configs[1] sweep:
parity (grouped vs split-K kernel) and CUDA-graph timing."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200.runtime import GemvGroup  # noqa: E402

dev = torch.device("cuda")
SWEEP = [(b, g, shp) for shp in [(4096, 4096), (4096, 11008), (11008, 4096)]
         for b in (2, 3, 4) for g in (32, 64, 128, None)]
pws, xs, ys, yref = [], [], [], []
for i, (b, g, (K, N)) in enumerate(SWEEP):
    torch.manual_seed(i)
    pw = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, q.QuantConfig(b, g))
    x = torch.randn(K, device=dev)
    pws.append(pw); xs.append(x); ys.append(torch.zeros(N, device=dev))
    yref.append(pw.gemv(x))
import os
from paper_2307_03738_b200 import _lib as _L
_L.lib().qigen_debug_group_mode(int(os.environ.get("GMODE", "0"), 0))
grp = GemvGroup(list(zip(pws, xs, ys)))
_L.lib().qigen_debug_group_mode(0)
grp.run(); torch.cuda.synchronize()
worst = 0.0
for (b, g, shp), y, r in zip(SWEEP, ys, yref):
    err = ((y - r).abs().max() / (1 + r.abs().max())).item()
    worst = max(worst, err)
    if err > 1e-5:
        print("MISMATCH", b, g, shp, err)
print("grouped vs split-K worst rel err", worst)
nb = grp.nbytes_algorithmic
s = torch.cuda.Stream()
from paper_2307_03738_b200 import _lib  # noqa: E402
def stream_only():
    _lib.lib().qigen_debug_group_mode(1); grp.run(); _lib.lib().qigen_debug_group_mode(0)
for name, fn in [("grouped", grp.run), ("grouped_stream_only", stream_only),
                 ("chain", lambda: [pw.gemv(x, out=y) for pw, x, y in zip(pws, xs, ys)]),
                 ("chain_xready", lambda: [pw.gemv(x, out=y, x_ready=True) for pw, x, y in zip(pws, xs, ys)])]:
    with torch.cuda.stream(s):
        fn(); s.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=s):
            fn()
        for _ in range(5):
            gph.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(50):
            gph.replay()
        e1.record(s); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 50
    print(f"{name}: {us:.1f} us/step  {nb / us / 1e3:.0f} GB/s")
