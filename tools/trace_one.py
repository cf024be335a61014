"""Per-CTA timeline of one GEMV launch: python tools/trace_one.py K N bits g tokens [splits]."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402

K, N, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = None if sys.argv[4] == "fc" else int(sys.argv[4])
T = int(sys.argv[5])
S = int(sys.argv[6]) if len(sys.argv) > 6 else 0
dev = torch.device("cuda")
pw = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, q.QuantConfig(b, g))
x = torch.randn(T, K, device=dev)
y = torch.empty(T, N, device=dev)
buf = torch.zeros(8192 * 16, dtype=torch.int64, device=dev)
for rep in range(3):
    buf.zero_()
    torch.cuda.synchronize()
    _lib.lib().qigen_debug_trace(buf.data_ptr())
    pw.gemv(x, out=y, k_splits=S)
    torch.cuda.synchronize()
    _lib.lib().qigen_debug_trace(None)
t = buf.view(-1, 16).cpu().numpy()
t = t[t[:, 0] > 0]
rel = (t - t[:, 0].min()) / 1e3
print(f"K={K} N={N} b={b} g={g} tokens={T} ctas={len(t)}")
names = ["entry", "after_wait", "after_prologue", "after_loop", "exit", "stage0", "pushed",
         "owner_in", "loads_issued", "loads_landed", "rounds_done"]
for i, name in enumerate(names):
    col = rel[:, i][t[:, i] > 0]
    if len(col):
        print(f"  {name:15s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us")
