import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402
K, N, T, g = (int(v) for v in sys.argv[1:5])
mode = int(sys.argv[5]) if len(sys.argv) > 5 else 0
_lib.lib().qigen_debug_tc_mode(mode)
dev = torch.device("cuda")
pw = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, q.QuantConfig(4, g))
x = torch.randn(T, K, device=dev)
y = torch.empty(T, N, device=dev)
buf = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
for _ in range(3):
    buf.zero_(); torch.cuda.synchronize()
    _lib.lib().qigen_debug_trace(buf.data_ptr()); pw.gemv(x, out=y); torch.cuda.synchronize()
    _lib.lib().qigen_debug_trace(None)
t = buf.view(-1, 16).cpu().numpy(); t = t[t[:, 0] > 0]
rel = (t - t[:, 0].min()) / 1e3
print(f"K={K} N={N} T={T} mode={mode} ctas={len(t)}")
for i, n in enumerate(["start", "after_wait", "dequant_done(w0)", "mma_issued", "accdone", "end"]):
    c = rel[:, i][t[:, i] > 0]
    if len(c): print(f"  {n:18s} min {c.min():7.2f} med {np.median(c):7.2f} max {c.max():7.2f}")
names = {6: "dq0 wfull", 7: "dq0 aempty", 8: "dq8 wfull", 9: "dq8 aempty", 10: "mma xfull",
         11: "mma afull", 12: "W wempty", 13: "X xempty", 14: "dq0 loop", 15: "mma issue"}
for i, n in names.items():
    c = t[:, i] / 1.9e3
    print(f"  {n:18s} us@1.9GHz med {np.median(c):7.2f} max {c.max():7.2f}")
