"""Dependent-chain experiment: CUDA graph of back-to-back GEMVs over R rotating
weight copies (PDL), sweeping the K split and the PDL trigger point."""
import argparse, json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2307_03738_b200 as q  # noqa: E402
from paper_2307_03738_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="4096x4096:4:128,4096x11008:4:128,11008x4096:3:64,4096x4096:2:fc")
ap.add_argument("--variants", default="0:0:8:0:0:0",
                help="comma list of early:policy:wpc:ring_kb:max_ctas:splits")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--x-ready", type=int, default=0)
ap.add_argument("--carveout", type=int, default=-1)
args = ap.parse_args()
L = _lib.lib()
dev = torch.device("cuda")
for case in args.cases.split(","):
    shp, b, gs = case.split(":")
    K, N = map(int, shp.split("x")); b = int(b); g = None if gs == "fc" else int(gs)
    cfg = q.QuantConfig(b, g)
    pw0 = q.PanelWeights.from_float(torch.randn(K, N, device=dev) * 0.02, cfg)
    nb = pw0.nbytes_algorithmic()
    R = max(8, int(4 * 126e6 // nb) + 1)
    pws = [pw0] + [q.PanelWeights(pw0.qw.clone(), pw0.qsz.clone(), K, N, cfg) for _ in range(R - 1)]
    xs = [torch.randn(K, device=dev) for _ in range(R)]
    ys = [torch.empty(N, device=dev) for _ in range(R)]
    for var in args.variants.split(","):
        early, pol, wpc, ring, mx, ks = map(int, var.split(":"))
        L.qigen_debug_early_trigger(early)
        L.qigen_debug_gemv_tuning(pol, wpc, ring, mx)
        if True:
            s = torch.cuda.Stream()
            try:
                with torch.cuda.stream(s):
                    for pw, x, y in zip(pws, xs, ys):
                        pw.gemv(x, out=y, k_splits=ks, x_ready=bool(args.x_ready))
                    s.synchronize()
                    gph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gph, stream=s):
                        for pw, x, y in zip(pws, xs, ys):
                            pw.gemv(x, out=y, k_splits=ks, x_ready=bool(args.x_ready))
                    for _ in range(3):
                        gph.replay()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    for _ in range(args.reps):
                        gph.replay()
                    e1.record(s)
                    e1.synchronize()
            except Exception as e:  # noqa: BLE001
                print(json.dumps(dict(case=case, var=var, err=str(e)[:100])), flush=True)
                continue
            us = e0.elapsed_time(e1) * 1e3 / (args.reps * R)
            print(json.dumps(dict(case=case, var=var, us=round(us, 2),
                                  gbs=round(nb / us / 1e3, 1))), flush=True)
    L.qigen_debug_early_trigger(0)
    L.qigen_debug_gemv_tuning(0, 8, 0, 0)
