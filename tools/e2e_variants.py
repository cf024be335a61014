"""A/B of host-path variants for qgemv_batch over the configs[1] sweep (same box)."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import runtime as R  # noqa: E402
SWEEP = [(b, g, shp) for shp in [(4096, 4096), (4096, 11008), (11008, 4096)]
         for b in (2, 3, 4) for g in (32, 64, 128, None)]
pms, xs = [], []
for i, (b, g, (K, N)) in enumerate(SWEEP):
    w = torch.randn(K, N, device="cuda") * 0.02
    cm = q.quantize_matrix(w, q.QuantConfig(b, g))
    pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
    xs.append(np.random.default_rng(i).normal(0, 1, K).astype(np.float32))
ref = q.qgemv_batch(pms, xs)
b = next(iter(R._BATCHES.values()))
torch.cuda.synchronize()

def t(f, n=400):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6

def fresh_out():
    np.concatenate(xs, out=b.xh_np)
    b.x.copy_(b.xh, non_blocking=True)
    b.group.run()
    yh = torch.empty(b.y.numel(), pin_memory=True)
    yh.copy_(b.y, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return np.split(yh.numpy(), b.noff[1:-1])

s = torch.cuda.current_stream()
def torch_copies():  # the previous qgemv_batch host path: torch copies, slices
    np.concatenate(xs, out=b.xh_np, casting="same_kind")
    b.x.copy_(b.xh, non_blocking=True)
    b.group.run()
    yh = torch.empty(b.y.numel(), pin_memory=True)
    yh.copy_(b.y, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    yv = yh.numpy()
    return [yv[sl] for sl in b.yslices]

def fresh_out_lean():
    np.concatenate(xs, out=b.xh_np)
    b.x.copy_(b.xh, non_blocking=True)
    R.lib().qigen_gemv_group_run(b.group._h, s.cuda_stream)
    yh = torch.empty(b.y.numel(), pin_memory=True)
    yh.copy_(b.y, non_blocking=True)
    s.synchronize()
    return np.split(yh.numpy(), b.noff[1:-1])

yh_shared = torch.empty(b.y.numel(), pin_memory=True)
def shared_copy_out():  # the previous host path: shared staging buffer + copy-out
    np.concatenate(xs, out=b.xh_np)
    b.x.copy_(b.xh, non_blocking=True)
    b.group.run()
    yh_shared.copy_(b.y, non_blocking=True)
    s.synchronize()
    return np.split(yh_shared.numpy().copy(), b.noff[1:-1])

def copies_and_kernels():
    b.x.copy_(b.xh, non_blocking=True)
    b.group.run()
    yh_shared.copy_(b.y, non_blocking=True)

def kern_only():
    b.group.run()

for name, f in [("qgemv_batch", lambda: q.qgemv_batch(pms, xs)), ("fresh_out", fresh_out),
                ("fresh_out_lean", fresh_out_lean), ("shared_copy_out", shared_copy_out),
                ("gpu_side_only", copies_and_kernels), ("kernels_only", kern_only),
                ("qgemv_batch", lambda: q.qgemv_batch(pms, xs)), ("torch_copies", torch_copies),
                ("qgemv_batch", lambda: q.qgemv_batch(pms, xs)), ("torch_copies", torch_copies)]:
    us = t(f)
    print("%-16s %7.1f us" % (name, us))
for f in (fresh_out, fresh_out_lean, shared_copy_out, torch_copies):
    out = f()
    assert all(np.array_equal(a, r) for a, r in zip(out, ref)), f.__name__
print("outputs identical")
