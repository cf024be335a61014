"""One decode-attention launch at the 65B B=8 shape (for ncu)."""
import math, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200.decode import GpuBackend  # noqa: E402
B, H, ctx, hd = 8, 64, 1025, 128
qkv = torch.randn(B, 3 * H * hd, device="cuda")
cos, sin = torch.ones(hd // 2, device="cuda"), torch.zeros(hd // 2, device="cuda")
kc = torch.randn(B, H, ctx, hd, device="cuda").half()
vc = torch.randn(B, H, ctx, hd, device="cuda").half()
out = torch.empty(B, H * hd, device="cuda")
for _ in range(3):
    GpuBackend.attention(qkv, cos, sin, kc, vc, ctx - 1, 1 / math.sqrt(hd), out, torch.empty(0))
torch.cuda.synchronize()
