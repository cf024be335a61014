"""Prologue timing vs weight stages issued before the PDL wait (qigen_debug_prefetch)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402
K, N = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda")
pw = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, q.QuantConfig(4, 128))
x = torch.randn(1, K, device=dev)
y = torch.empty(1, N, device=dev)
buf = torch.zeros(8192 * 16, dtype=torch.int64, device=dev)
for pre in (-1, 0, 1):
    _lib.lib().qigen_debug_prefetch(pre)
    for rep in range(3):
        buf.zero_(); torch.cuda.synchronize()
        _lib.lib().qigen_debug_trace(buf.data_ptr()); pw.gemv(x, out=y); torch.cuda.synchronize()
        _lib.lib().qigen_debug_trace(None)
    t = buf.view(-1, 16).cpu().numpy(); t = t[t[:, 0] > 0]
    rel = (t - t[:, 0].min()) / 1e3
    med = lambda i: np.median(rel[:, i][t[:, i] > 0])
    print(f"pre={pre:2d}: wait {med(1):5.2f} loads {med(8):5.2f} rounds {med(10):5.2f} prol {med(2):5.2f} "
          f"stage0 {med(5):5.2f} loop {med(3):5.2f} exit {med(4):5.2f}  cyc issue {np.median(t[:,11]):.0f} "
          f"firstdig {np.median(t[:,12]):.0f} rest {np.median(t[:,13]):.0f}")
_lib.lib().qigen_debug_prefetch(-1)
