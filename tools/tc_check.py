"""Quick correctness/timing check of the tcgen05 small-batch path."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import runtime as R  # noqa: E402

dev = torch.device("cuda")
for (K, N, T, g) in [(256, 128, 16, 64), (512, 256, 16, 64), (1024, 384, 32, 128), (8192, 8192, 16, 64),
                     (8192, 8192, 64, 64), (4096, 11008, 48, 128)]:
    w = torch.randn(K, N, device=dev) * 0.02
    pw = q.PanelWeights.from_float(w, q.QuantConfig(4, g))
    cm = q.quantize_matrix(w, q.QuantConfig(4, g))
    wd = q.dequantize_matrix(cm).double()
    x = torch.randn(T, K, device=dev)
    y = pw.gemv(x)
    torch.cuda.synchronize()
    yref = x.double() @ wd
    err = ((y.double() - yref).abs().max() / (1 + yref.abs().max())).item()
    y2 = pw.gemv(x, path="gemv")
    err2 = ((y2.double() - yref).abs().max() / (1 + yref.abs().max())).item()
    # timing
    reps = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g_ = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pw.gemv(x, out=y)
        s.synchronize()
        with torch.cuda.graph(g_, stream=s):
            for _ in range(10):
                pw.gemv(x, out=y)
        g_.replay()
        e0.record(s)
        for _ in range(reps):
            g_.replay()
        e1.record(s)
        s.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * 10)
    print(f"K={K} N={N} T={T} g={g}: tc err {err:.2e}  gemv err {err2:.2e}  tc {us:.1f} us "
          f"({pw.nbytes_algorithmic() / us / 1e3:.0f} GB/s, L2-warm)", flush=True)
