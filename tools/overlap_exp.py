"""Step-to-step overlap of the grouped GEMV (configs[1] sweep, 36 GEMVs).

Variants: steps replayed as one CUDA graph each (graph boundaries serialise
steps) vs issued as plain stream launches (the prep kernel of step n+1 is a
programmatic dependent of step n's grouped kernel), with the prep kernel
triggering the grouped launch after (default) or before (mode & 32) its wait.
Checks every variant's y against the split-K kernel."""
import os
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402
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
grp = GemvGroup(list(zip(pws, xs, ys)))
nb = grp.nbytes_algorithmic
s = torch.cuda.Stream()
STEPS = int(os.environ.get("STEPS", "200"))


def check(tag):
    worst = max(((y - r).abs().max() / (1 + r.abs().max())).item() for y, r in zip(ys, yref))
    assert worst < 1e-5, (tag, worst)


for mode in (0, 32):
    _lib.lib().qigen_debug_group_mode(mode)
    with torch.cuda.stream(s):
        grp.run(); s.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=s):
            grp.run()
        for name, fn in [("graph", gph.replay), ("stream", grp.run)]:
            for _ in range(20):
                fn()
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(STEPS):
                fn()
            e1.record(s); e1.synchronize()
            check((mode, name))
            us = e0.elapsed_time(e1) * 1e3 / STEPS
            print(f"mode={mode:2d} {name:6s}: {us:6.1f} us/step  {nb / us / 1e3:5.0f} GB/s", flush=True)
    _lib.lib().qigen_debug_group_mode(0)
