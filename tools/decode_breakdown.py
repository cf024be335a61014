"""Run a few eager decode steps of a shrunk LLaMA (for ncu launch lists)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_03738_b200 import decode as D  # noqa: E402

cfg = D.shrink(D.LLAMA_7B, n_layers=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
m = D.LlamaTP(cfg, batch=1, max_ctx=513, seed=0)
tok = torch.zeros(1, dtype=torch.long, device="cuda")
for _ in range(3):
    m.step(tok, 512)
torch.cuda.synchronize()
print("ok")
