"""Steady-state timeline: a CUDA graph of back-to-back GEMVs (PDL), each
launch tracing its CTAs (globaltimer) into its own buffer."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
L = _lib.lib()
import os
KS = int(os.environ.get("KS", "0"))
L.qigen_debug_early_trigger(int(os.environ.get("EARLY", "0")))
L.qigen_debug_prefetch(int(os.environ.get("PRE", "-1")))
L.qigen_debug_gemv_tuning(*map(int, os.environ.get("TUNE", "0:8:0:0").split(":")))
for shp, b, g in [((4096, 4096), 4, 128), ((4096, 11008), 4, 128), ((11008, 4096), 3, 64)]:
    K, N = shp
    cfg = q.QuantConfig(b, g)
    base = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, cfg)
    R = 16
    pws = [base] + [q.PanelWeights(base.qw.clone(), base.qsz.clone(), K, N, cfg) for _ in range(R - 1)]
    xs = [torch.randn(K, device=dev) for _ in range(R)]
    if os.environ.get("XSAME"):
        xs = [xs[0]] * R
    ys = [torch.empty(N, device=dev) for _ in range(R)]
    bufs = [torch.zeros(4096 * 16, dtype=torch.int64, device=dev) for _ in range(R)]
    cbufs = [torch.zeros(4096 * 16, dtype=torch.int64, device=dev) for _ in range(R)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for pw, x, y in zip(pws, xs, ys):
            pw.gemv(x, out=y, k_splits=KS, x_ready=bool(int(os.environ.get("XREADY", "0"))))
        s.synchronize()
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=s):
            for i, (pw, x, y) in enumerate(zip(pws, xs, ys)):
                L.qigen_debug_trace(bufs[i].data_ptr())
                L.qigen_debug_trace_clk(cbufs[i].data_ptr())
                pw.gemv(x, out=y, k_splits=KS, x_ready=bool(int(os.environ.get("XREADY", "0"))))
            L.qigen_debug_trace(None)
            L.qigen_debug_trace_clk(None)
        for _ in range(3):
            gph.replay()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        gph.replay()
        e1.record(s)
        s.synchronize()
    print(f"K={K} N={N} b={b} g={g}: {R} GEMVs in {e0.elapsed_time(e1)*1e3:.1f} us "
          f"({e0.elapsed_time(e1)*1e3/R:.2f} us each, {base.nbytes_algorithmic()*R/e0.elapsed_time(e1)/1e6:.0f} GB/s)")
    tr = [b_.view(-1, 16).cpu().numpy() for b_ in bufs]
    tc = [b_.view(-1, 16).cpu().numpy() for b_ in cbufs]
    t0 = min(t[t[:, 0] > 0][:, 0].min() for t in tr)
    for i, t in enumerate(tr[:6]):
        t = t[t[:, 0] > 0]
        rel = (t[:, :8] - t0) / 1e3
        print(f"  #{i} ctas {len(t)} entry {rel[:,0].min():6.2f}-{rel[:,0].max():6.2f}  wait {rel[:,1].min():6.2f}-{rel[:,1].max():6.2f}"
              f"  prol {np.median(rel[:,2]):6.2f} stage0 {np.median(rel[:,5]):6.2f} loop {np.median(rel[:,3]):6.2f} (max {rel[:,3].max():6.2f}) push {np.median(rel[:,6]):6.2f} bar {np.median(rel[:,7]):6.2f} exit {rel[:,4].min():6.2f}-{rel[:,4].max():6.2f}")
    # per-phase medians relative to each CTA's own PDL wait (kernels #1..)
    names = {8: "xload", 11: "dig1", 10: "digits", 2: "sync", 5: "stage0", 3: "loop", 6: "cl_wait", 7: "inbox", 4: "exit"}
    rows = []
    for t in tc[1:]:
        t = t[t[:, 0] > 0].astype(np.int64)
        rows.append(t)
    t = np.concatenate(rows)
    print("   phase (SM cycles after wait, median/p90): " + "  ".join(
        f"{n} {np.median(t[:, i] - t[:, 1]):.0f}/{np.percentile(t[:, i] - t[:, 1], 90):.0f}"
        for i, n in names.items()))
