import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
K, N, T, g = (int(v) for v in sys.argv[1:5])
pw = q.PanelWeights.from_float(torch.randn(K, N, device="cuda") * 0.02, q.QuantConfig(4, g))
x = torch.randn(T, K, device="cuda")
for _ in range(3):
    y = pw.gemv(x)
torch.cuda.synchronize()
print("ok")
