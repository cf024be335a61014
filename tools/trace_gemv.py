"""Per-CTA timeline of one GEMV launch (globaltimer stamps, qigen_debug_trace)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
pre = int(sys.argv[1]) if len(sys.argv) > 1 else -1
_lib.lib().qigen_debug_prefetch(pre)
print("stages before PDL wait:", pre)
for shp, b, g in [((4096, 4096), 4, 128), ((11008, 4096), 4, 128), ((4096, 11008), 4, 128),
                  ((4096, 4096), 2, 32)]:
    K, N = shp
    pw = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, q.QuantConfig(b, g))
    x = torch.randn(K, device=dev)
    y = torch.empty(N, device=dev)
    buf = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)
    for rep in range(3):
        flush.zero_()  # evict L2
        buf.zero_()
        torch.cuda.synchronize()
        _lib.lib().qigen_debug_trace(buf.data_ptr())
        pw.gemv(x, out=y)
        torch.cuda.synchronize()
        _lib.lib().qigen_debug_trace(None)
    t = buf.view(-1, 16).cpu().numpy()
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    rel = (t[:, :5] - base) / 1e3
    print(f"K={K} N={N} b={b} g={g} ctas={len(t)} bytes={pw.nbytes_algorithmic()/1e6:.1f}MB")
    for i, name in enumerate(["entry", "after_wait", "after_prologue", "after_loop", "exit"]):
        col = rel[:, i]
        print(f"  {name:15s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us")
    print(f"  prologue  med {np.median(rel[:,2]-rel[:,1]):.2f} us; loop med {np.median(rel[:,3]-rel[:,2]):.2f} max {np.max(rel[:,3]-rel[:,2]):.2f}; epi med {np.median(rel[:,4]-rel[:,3]):.2f} us")
