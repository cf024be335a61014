"""Chain timing (graph of 16 back-to-back GEMVs, PDL) for every K split."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402

dev = torch.device("cuda")
shapes = [(4096, 4096), (4096, 11008), (11008, 4096)]
cases = [(b, g) for b in (2, 3, 4) for g in (32, 128, None)]
if len(sys.argv) > 1:
    cases = [(4, 128)]
for K, N in shapes:
    for b, g in cases:
        cfg = q.QuantConfig(b, g)
        base = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, cfg)
        R = 16
        pws = [base] + [q.PanelWeights(base.qw.clone(), base.qsz.clone(), K, N, cfg) for _ in range(R - 1)]
        xs = [torch.randn(K, device=dev) for _ in range(R)]
        ys = [torch.empty(N, device=dev) for _ in range(R)]
        res = {}
        for S in [0] + list(range(1, 17)):
            if S > (K + 255) // 256:
                break
            try:
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    for pw, x, y in zip(pws, xs, ys):
                        pw.gemv(x, out=y, k_splits=S)
                    st.synchronize()
                    gph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gph, stream=st):
                        for pw, x, y in zip(pws, xs, ys):
                            pw.gemv(x, out=y, k_splits=S)
                    for _ in range(3):
                        gph.replay()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    for _ in range(10):
                        gph.replay()
                    e1.record(st)
                    st.synchronize()
                res[S] = round(e0.elapsed_time(e1) * 1e3 / (10 * R), 2)
            except Exception as ex:  # noqa: BLE001
                res[S] = str(ex)[:40]
        best = min((v, k) for k, v in res.items() if isinstance(v, float) and k > 0)
        print(json.dumps({"K": K, "N": N, "b": b, "g": g, "auto": res.get(0), "best_S": best[1],
                          "best_us": best[0], "all": res}), flush=True)
        del pws, base
        torch.cuda.empty_cache()
