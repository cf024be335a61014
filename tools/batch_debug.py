import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from oracle import qigen_oracle as orc  # noqa: E402
pms, xs, refs = [], [], []
for i, (K, N, b, g) in enumerate([(1024, 512, 4, 128), (2048, 300, 3, 32), (512, 1024, 2, None)]):
    rng = np.random.default_rng(40 + i)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    cm = q.quantize_matrix(w, q.QuantConfig(b, g))
    codes, s, z = cm.numpy()
    pms.append(q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cm.config, (K, N))))
    xs.append(rng.normal(0, 1, K).astype(np.float32))
    refs.append(orc.qgemv_reference(codes, s, z, xs[-1]))
for call in range(3):
    ys = q.qgemv_batch(pms, xs)
    print(call, [float(np.abs(y - r).max() / (1 + np.abs(r).max())) for y, r in zip(ys, refs)])
