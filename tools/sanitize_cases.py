"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): quantize + pack + panels, the
split-K GEMV (fused prologues, prep kernel, K splits, g = 16), the grouped GEMV,
the tcgen05 GEMM, decode attention, the fused LM head and the emulated TP push
all-reduce.  Exits nonzero on a numerical mismatch."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib, decode as D  # noqa: E402
from paper_2307_03738_b200.runtime import GemvGroup  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda")
rng = np.random.default_rng(0)
fails = []


def check(name, y, ref, tol=1e-5):
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    err = np.abs(y - ref).max() / (1 + np.abs(ref).max())
    print(f"{name}: rel err {err:.2e}", flush=True)
    if not err <= tol:
        fails.append(name)


for bits, g, (K, N) in [(4, 128, (1024, 320)), (3, 64, (768, 200)), (2, None, (512, 96)),
                        (4, 16, (512, 64)), (3, 32, (2304, 130))]:
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    cm = q.quantize_matrix(w, q.QuantConfig(bits, g))
    pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N)))
    wd = q.dequantize_matrix(cm).double().cpu().numpy()
    for T in (1, 3):
        X = rng.normal(0, 1, (T, K)).astype(np.float32)
        check(f"qgemv b{bits} g{g} {K}x{N} T{T}", q.qgemv(pm, X), X.astype(np.float64) @ wd)
    pw = q.runtime.exec_layout(pm)
    x = torch.from_numpy(rng.normal(0, 1, (2, K)).astype(np.float32)).cuda()
    for ks in (1, 2, 3):
        check(f"gemv ks{ks} b{bits} g{g}", pw.gemv(x, k_splits=ks).cpu(), x.double().cpu().numpy() @ wd)
    _lib.lib().qigen_debug_force_prep(1)
    check(f"gemv prep b{bits} g{g}", pw.gemv(x).cpu(), x.double().cpu().numpy() @ wd)
    _lib.lib().qigen_debug_force_prep(0)
    nw = torch.rand(K, device=dev) + 0.5
    xn = (x / torch.sqrt(x.pow(2).mean(-1, keepdim=True) + 1e-5) * nw).double().cpu().numpy()
    check(f"gemv rmsnorm b{bits} g{g}", pw.gemv(x, prologue="rmsnorm", norm_weight=nw).cpu(), xn @ wd)

# grouped
specs = [(1024, 512, 4, 128), (768, 100, 3, None), (2048, 256, 2, 32), (512, 64, 4, 256)]
ents, refs = [], []
for K, N, b, g in specs:
    w = torch.randn(K, N, device=dev) * 0.02
    pw = q.PanelWeights.from_float(w, q.QuantConfig(b, g))
    x = torch.randn(K, device=dev)
    ents.append((pw, x, torch.empty(N, device=dev)))
    refs.append(pw.gemv(x).cpu())
grp = GemvGroup(ents)
for _ in range(2):
    grp.run()
torch.cuda.synchronize()
for (_, _, y), r in zip(ents, refs):
    check("grouped", y.cpu(), r, 2e-6)

# tcgen05 GEMM
K, N = 1024, 272
w = torch.randn(K, N, device=dev) * 0.02
pw = q.PanelWeights.from_float(w, q.QuantConfig(4, 64))
X = torch.randn(20, K, device=dev)
check("tcgen05 gemm", pw.gemv(X, path="tc").cpu(), pw.gemv(X, path="gemv").cpu(), 2e-3)

# decode attention
B, H, hd, ctx, pos = 1, 4, 128, 80, 70
qkv = torch.randn(B, 3 * H * hd, device=dev)
ang = torch.rand(hd // 2, device=dev)
kc = torch.randn(B, H, ctx, hd, device=dev).half()
vc = torch.randn(B, H, ctx, hd, device=dev).half()
out = torch.empty(B, H * hd, device=dev)
ws = D.GpuBackend.attention_workspace(B, H, hd, ctx, dev)
D.GpuBackend.attention(qkv, ang.cos(), ang.sin(), kc, vc, pos, 1 / math.sqrt(hd), out, ws)
torch.cuda.synchronize()
print("attention ok", flush=True)

# LM head
V, d, B = 600, 1024, 2
h = torch.randn(B, d, device=dev)
nw = torch.ones(d, device=dev)
W = (torch.randn(V, d, device=dev) * 0.02).half()
wsl = D.GpuBackend.lm_head_workspace(V, d, B, dev)
lg = torch.empty(B, V, device=dev)
mx = torch.empty(B, device=dev)
ix = torch.empty(B, dtype=torch.int64, device=dev)
D.GpuBackend.lm_head(h, nw, 1e-5, W, 0, lg, mx, ix, wsl)
torch.cuda.synchronize()
if not torch.equal(ix, lg.argmax(-1)):
    fails.append("lm_head argmax")

# emulated TP push all-reduce
cfg = D.LlamaConfig(n_layers=2, d_model=512, n_heads=4, head_dim=128, ffn=1024, vocab=512,
                    bits=4, group=128)
ref = D.LlamaTP(cfg, batch=1, max_ctx=40, seed=1)
ms = D.emulated_tp(cfg, 2, batch=1, max_ctx=40, seed=1)
tok = torch.tensor([7], device=dev)
t1 = ref.step(tok, 30)
t2 = D.emulated_step(ms, tok, 30)
torch.cuda.synchronize()
check("emulated tp2 logits", ms[0].last_logits.cpu(), ref.last_logits.cpu(), 5e-4)
if not torch.equal(t1, t2):
    fails.append("tp tokens")
print("FAILS:", fails)
sys.exit(1 if fails else 0)
