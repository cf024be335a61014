"""Standalone check of qigen_attn_decode against torch SDPA over (B, H, ctx, pos)."""
import math, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200.decode import GpuBackend  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from decode_backends import OracleBackend  # noqa: E402

for (B, H, ctx, pos) in [(1, 32, 513, 512), (1, 64, 513, 512), (1, 32, 1025, 1024), (1, 64, 1025, 1024),
                         (2, 8, 100, 70), (1, 64, 1025, 500)]:
    hd = 128
    qkv = torch.randn(B, 3 * H * hd, device="cuda")
    ang = torch.rand(hd // 2, device="cuda") * 6
    cos, sin = ang.cos(), ang.sin()
    kc = (torch.randn(B, H, ctx, hd, device="cuda")).half()
    vc = (torch.randn(B, H, ctx, hd, device="cuda")).half()
    kc2, vc2 = kc.clone(), vc.clone()
    out = torch.empty(B, H * hd, device="cuda")
    ref = torch.empty(B, H * hd, device="cuda")
    ws = GpuBackend.attention_workspace(B, H, hd, ctx, "cuda")
    try:
        GpuBackend.attention(qkv, cos, sin, kc, vc, pos, 1 / math.sqrt(hd), out, ws)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print("FAIL", (B, H, ctx, pos), str(e)[:80]); break
    OracleBackend.attention(qkv, cos, sin, kc2, vc2, pos, 1 / math.sqrt(hd), ref, None)
    err = ((out - ref).abs().max() / (1 + ref.abs().max())).item()
    print((B, H, ctx, pos), "rel err", err, "cache equal", torch.equal(kc, kc2) and torch.equal(vc, vc2), flush=True)
