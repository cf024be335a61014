#!/usr/bin/env python3
"""Benchmark of the quantized-GEMV hot path (BASELINE.json metric, configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (one "step"): one batch-1 qGEMV over each of the 36 distinct weight
matrices of BASELINE configs[1] — b in {2,3,4} x g in {32,64,128,FC} x KxN in
{4096x4096, 4096x11008, 11008x4096} — W ~ N(0, 0.02^2) quantized on the GPU
(bit-exact with the reference), x ~ N(0,1) f32, seeded.  The step reads
~622 MB of packed weights + scales/zeros, i.e. inputs larger than the 126 MB
L2, so no L2 flush is needed between steps.

value  = algorithmic bytes (packed codes + f32 scale + f32 zero) of all ranks
         / device time of the timed steps (max over ranks), GB/s.  The step is
         a CUDA graph of the activation-prep kernel + ONE persistent grouped
         GEMV kernel over the 36 independent GEMVs (GemvGroup); inputs are
         resident in HBM.  config.chain_gbs reports the same GEMVs as 36
         dependent single-GEMV launches.
e2e    = same metric through the public API `qgemv_batch(pms, xs_host)`: host
         activations in, host results out, every step (zero-copy over PCIe).
decode = BASELINE configs[3]/[4]: LLaMA-7B (B=1) and LLaMA-65B (B=1, B=8) decode
         steps, tensor-parallel over the N ranks (NCCL), tokens/s and roofline.
N > 1  = `--gpus N` re-executes itself under torch.distributed.run (one process
         per GPU).  The sweep runs as independent replicas on every rank (weak
         scaling, no data-path collective: GEMVs of distinct matrices are
         independent); the decode steps are tensor-parallel across the ranks.
cpu_baseline / --impl reference = the reference's CPU path on the box's host
         cores: the C port of its generated kernel (oracle/qgemv_port.c, bit-
         identical to the reference's numba kernel) on all 36 matrices at all
         threads and at 1 thread, plus the reference's own numba kernel
         (baseline/_ref, oracle/ref_numba.py) on configs[0].
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SWEEP = [(b, g, shp) for shp in [(4096, 4096), (4096, 11008), (11008, 4096)]
         for b in (2, 3, 4) for g in (32, 64, 128, None)]
WORKLOAD = ("BASELINE configs[1] sweep: b{2,3,4} x g{32,64,128,full} x KxN"
            "{4096x4096,4096x11008,11008x4096}, batch 1, f32 activations")


def algo_bytes(K, N, bits, g):
    G = 1 if g is None else K // g
    return K * N * bits // 8 + G * N * 8


STEP_BYTES = sum(algo_bytes(K, N, b, g) for b, g, (K, N) in SWEEP)


def graph_kernel_counts(graph) -> tuple[int, int]:
    """(kernel nodes, kernel nodes that are this package's own kernels) of a
    captured CUDA graph (built with keep_graph=True), read back through the CUDA
    driver API: the per-step launch count the bench reports."""
    from cuda.bindings import driver as cu
    g = cu.CUgraph(graph.raw_cuda_graph())
    _, _, n = cu.cuGraphGetNodes(g, 0)
    _, nodes, n = cu.cuGraphGetNodes(g, n)
    total = ours = 0
    for nd in nodes[:n]:
        _, typ = cu.cuGraphNodeGetType(nd)
        if typ != cu.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
            continue
        total += 1
        _, prm = cu.cuGraphKernelNodeGetParams(nd)
        err, name = cu.cuFuncGetName(prm.func)
        if err != cu.CUresult.CUDA_SUCCESS:
            err, name = cu.cuKernelGetName(prm.kern)
        name = name.decode() if isinstance(name, bytes) else str(name)
        ours += "qigen" in name
    return total, ours


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:  # noqa: BLE001
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi-equivalent sampling via NVML in a thread (SM clock, reasons)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.max = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()

    def report(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU side: the reference path restated by the oracle (C port, exec layout)
# ---------------------------------------------------------------------------

def _cpu_case(args):
    i, b, g, K, N = args
    from oracle import qigen_oracle as orc
    rng = np.random.default_rng(1000 + i)
    w = rng.normal(0, 0.02, (K, N)).astype(np.float32)
    codes, s, z = orc.quantize_matrix(w, b, g)
    mu, tu, m_b, t_b = orc.plan(b, g, (K, N))
    ex = orc.ExecLayout(orc.pack_rowseq(codes, b), s, z, K, N, b, g, m_b, t_b)
    x = rng.normal(0, 1, K).astype(np.float32)
    return ex, x, algo_bytes(K, N, b, g), (b, g, K, N), (mu, tu, m_b, t_b)


def build_cpu_cases(subset):
    """Seeded sweep matrices quantized and laid out by the oracle's restatement
    of the reference (quant.py / packing.py / Appendix B exec layout), built in
    a process pool (untimed setup)."""
    import multiprocessing as mp
    jobs = [(i, b, g, K, N) for i, (b, g, (K, N)) in enumerate(subset)]
    procs = max(1, min(len(jobs), len(os.sched_getaffinity(0)), 16))
    if procs == 1:
        return [_cpu_case(j) for j in jobs]
    with mp.get_context("spawn").Pool(procs) as pool:
        return pool.map(_cpu_case, jobs)


def time_cpu(cases, reps, threads):
    from oracle import qigen_oracle as orc
    for ex, x, *_ in cases:  # warm-up (2 warm-ups)
        orc.qgemv_port(ex, x, threads=threads)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for ex, x, *_ in cases:
            orc.qgemv_port(ex, x, threads=threads)
        times.append(time.perf_counter() - t0)
    nbytes = sum(c[2] for c in cases)
    return nbytes / statistics.median(times) / 1e9, statistics.median(times)


def cpu_threads() -> int:
    return len(os.sched_getaffinity(0))


REF_NUMBA_CONFIGS = [(4, 128, (4096, 4096)), (2, 32, (4096, 4096))]  # configs[0] + a 2-bit one


def time_ref_numba(cases, threads, reps=5):
    """The reference's own numba-compiled kernel (oracle/ref_numba.py) on the
    REF_NUMBA_CONFIGS matrices: compile (untimed), 2 warm-ups, median of reps,
    at 1 thread and at `threads`.  None if the reference is not installed."""
    from oracle import ref_numba
    if ref_numba.available() is None:
        return {"unavailable": "reference package not installed in baseline/_ref"}
    out = {}
    for c in cases:
        ex, x, nbytes, (b, g, K, N), plan = c
        if (b, g, (K, N)) not in REF_NUMBA_CONFIGS:
            continue
        t0 = time.perf_counter()
        k = ref_numba.RefKernel(ex, b, g, plan)
        k(x, 1)
        compile_s = time.perf_counter() - t0
        res = {"compile_s": round(compile_s, 1)}
        for th in sorted({1, threads}):
            for _ in range(2):
                k(x, th)
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                k(x, th)
                ts.append(time.perf_counter() - t0)
            res[f"gbs_{th}t"] = round(nbytes / statistics.median(ts) / 1e9, 4)
            res[f"ms_{th}t"] = round(1e3 * statistics.median(ts), 3)
        out[f"b{b} g{g} {K}x{N}"] = res
    return out


def cpu_baseline_block(cases, steps_all=3, steps_one=1):
    """cpu_baseline: the C port on all 36 matrices at all threads and at 1
    thread, plus the reference's numba kernel on REF_NUMBA_CONFIGS."""
    threads = cpu_threads()
    gbs, t_all = time_cpu(cases, steps_all, threads)
    gbs1, t_one = time_cpu(cases, steps_one, 1)
    nbytes = sum(c[2] for c in cases)
    return {
        "value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "port",
        "value_1thread": round(gbs1, 4),
        "sample": (f"all {len(cases)} sweep matrices ({nbytes / 1e6:.0f} MB per pass; the GPU "
                   f"arm's workload), C port of the reference's generated kernel "
                   f"(oracle/qgemv_port.c, bit-identical to the reference's numba kernel) on its "
                   f"exec layout; median of {steps_all} passes at {threads} threads "
                   f"({1e3 * t_all:.1f} ms per pass), {steps_one} pass at 1 thread "
                   f"({1e3 * t_one:.0f} ms)"),
        "reference_numba": time_ref_numba(cases, threads),
    }


def run_reference(args):
    """--impl reference: the reference's CPU path on the host cores, same
    workload (all 36 sweep matrices), metric and unit as our arm."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = cpu_threads()
    t0 = time.perf_counter()
    cases = build_cpu_cases(SWEEP)
    setup = time.perf_counter() - t0
    for _ in range(args.warmup):
        time_cpu(cases, 1, threads)
    times = []
    for _ in range(args.steps):
        _, t = time_cpu(cases, 1, threads)
        times.append(t)
    nbytes = sum(c[2] for c in cases)
    value = nbytes * len(times) / sum(times) / 1e9
    gbs1, t1 = time_cpu(cases, 1, 1)
    sample = (f"all {len(cases)} sweep matrices (b x g x shape), {nbytes / 1e6:.1f} MB per step; "
              f"C port of the reference's generated kernel (bit-identical to its numba kernel) "
              f"on its exec layout, {threads} threads; 1 thread: {gbs1:.3f} GB/s "
              f"({1e3 * t1:.0f} ms per step); setup {setup:.1f} s untimed")
    line = {"metric": "quantized GEMV effective HBM GB/s", "value": round(value, 4), "unit": "GB/s",
            "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "matrices": len(cases), "bytes_per_step": nbytes},
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads,
                             "kind": "port", "value_1thread": round(gbs1, 4), "sample": sample,
                             "reference_numba": time_ref_numba(cases, threads)},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = init_dist()
    import paper_2307_03738_b200 as q
    from paper_2307_03738_b200.runtime import PanelWeights

    dev = torch.device("cuda", local)
    mats, xs, ys, pms = [], [], [], []
    gen = torch.Generator(device=dev)
    for i, (b, g, (K, N)) in enumerate(SWEEP):
        gen.manual_seed(1000 + i + 7919 * rank)
        w = torch.randn((K, N), generator=gen, device=dev) * 0.02
        cfg = q.QuantConfig(b, g)
        cm = q.quantize_matrix(w, cfg)
        # the reference-format object a user holds, and its GPU layout cache
        pm = q.lay_out_blocks(cm, q.plan(q.DEFAULT_HARDWARE, cfg, (K, N)))
        pw = q.runtime.exec_layout(pm)
        del w, cm
        mats.append(pw)
        pms.append(pm)
        xs.append(torch.randn(K, generator=gen, device=dev))
        ys.append(torch.empty(N, device=dev))
    torch.cuda.synchronize()

    stream = torch.cuda.Stream(device=dev)
    # the step: the 36 independent GEMVs as one grouped persistent launch
    # (activation prep kernel + gemv_group_kernel), replayed as a CUDA graph
    group = q.GemvGroup(list(zip(mats, xs, ys)))

    def capture(fn):
        with torch.cuda.stream(stream):
            fn()
            stream.synchronize()
            g = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(g, stream=stream):
                fn()
            g.instantiate()
        stream.synchronize()
        return g

    graph = capture(group.run)
    try:
        k_total, k_ours = graph_kernel_counts(graph)
    except Exception as e:  # noqa: BLE001 (reported, not fatal)
        print(f"kernel count unavailable: {e}", file=sys.stderr)
        k_total = k_ours = 2

    def chain():  # the same GEMVs as 36 dependent single-GEMV launches (PDL)
        for pw, x, y in zip(mats, xs, ys):
            pw.gemv(x, out=y)
    chain_graph = capture(chain)

    def timed(g, steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                g.replay()
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    sampler = ClockSampler(local)
    with sampler:
        with torch.cuda.stream(stream):
            # warm-up (+ a short soak so the clock sampler sees the GPU under load)
            soak_end = time.perf_counter() + 0.5
            w_done = 0
            while w_done < args.warmup or time.perf_counter() < soak_end:
                graph.replay()
                w_done += 1
                if w_done % 50 == 0:
                    stream.synchronize()
            stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms = timed(graph, args.steps)
        torch.cuda.synchronize()
    chain_ms = timed(chain_graph, max(3, min(args.steps, 50)))
    chain_steps = max(3, min(args.steps, 50))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_per_step = ms / args.steps
    value = STEP_BYTES * world * args.steps / (ms / 1e3) / 1e9
    kernel_gbs = STEP_BYTES / (ms_per_step / 1e3) / 1e9
    chain_gbs = STEP_BYTES * chain_steps / (chain_ms / 1e3) / 1e9

    # --- e2e through the public API with host buffers --------------------------
    # qgemv_batch(pms, xs): host x gathered into pinned memory, the grouped launch
    # reads it and stores y into a fresh pinned block over PCIe (zero-copy), sync
    xs_host = [x.cpu().numpy() for x in xs]
    e2e_steps = max(1, min(args.steps, 200))
    # (a) inputs in pageable numpy arrays: the call gathers them into pinned memory first
    for _ in range(max(3, args.warmup)):  # warm-up (plan, staging and pinned result blocks cached)
        q.qgemv_batch(pms, xs_host)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        q.qgemv_batch(pms, xs_host)
    torch.cuda.synchronize()
    e2e_pageable = STEP_BYTES * e2e_steps / (time.perf_counter() - t0) / 1e9
    # (b) the headline: inputs in page-locked host memory (numpy views handed out by
    # qgemv_batch_inputs, filled in place), read by the kernel over PCIe every step
    xs_pin = q.qgemv_batch_inputs(pms)
    for dst, src in zip(xs_pin, xs_host):
        np.copyto(dst, src)
    for _ in range(max(3, args.warmup)):
        q.qgemv_batch(pms, xs_pin)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        q.qgemv_batch(pms, xs_pin)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = STEP_BYTES * world * e2e_steps / e2e_s / 1e9
    # the reference's own seam, one blocking qgemv(pm, x_host) per matrix:
    # numpy in, numpy out, a host round trip per call (reported next to the batched form)
    seam_steps = max(1, min(args.steps, 10))
    for pm, xh in zip(pms, xs_host):
        q.qgemv(pm, xh)
    t0 = time.perf_counter()
    for _ in range(seam_steps):
        for pm, xh in zip(pms, xs_host):
            q.qgemv(pm, xh)
    seam_s = time.perf_counter() - t0
    seam_gbs = STEP_BYTES * seam_steps / seam_s / 1e9
    seam_us = seam_s / (seam_steps * len(pms)) * 1e6
    h2d = sum(K * 4 for _, _, (K, N) in SWEEP)
    d2h = sum(N * 4 for _, _, (K, N) in SWEEP)
    del group, graph, chain_graph
    torch.cuda.synchronize()

    # --- decode steps (configs[3]/[4]), tensor parallel over the ranks ----------
    decode = {}
    if not args.no_decode:
        dsteps = max(3, min(args.steps, 50))
        for wl, B in DECODE_DEFAULT:
            try:
                decode[f"{wl} B={B}"] = measure_decode(wl, B, 0, 0, dsteps, args.warmup)
            except Exception as e:  # noqa: BLE001 (reported in the line, not fatal)
                decode[f"{wl} B={B}"] = {"error": f"{type(e).__name__}: {e}"[:300]}

    if rank == 0:
        peak, peak_src = measured_peak()
        line = {
            "metric": "quantized GEMV effective HBM GB/s",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8 x s8 -> s32 (IMMA), f32 epilogue",
            "data": "synthetic (seeded N(0,0.02^2) weights, N(0,1) activations)",
            "config": {"workload": WORKLOAD, "matrices": len(SWEEP),
                       "bytes_per_step": STEP_BYTES,
                       "l2": "inputs larger than L2 (%.0f MB per step vs 126 MB)" % (STEP_BYTES / 1e6),
                       "launch": "CUDA graph: activation prep + one persistent grouped GEMV kernel "
                                 "(gemv_group_kernel, 148 CTAs) over the 36 independent GEMVs",
                       "chain_gbs": round(chain_gbs, 1),
                       "chain": "the same 36 GEMVs as dependent single-GEMV launches (PDL), GB/s",
                       "parallelism": f"replicas x{world}"},
            "roofline": {"bound": "hbm", "achieved": round(kernel_gbs, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s",
                         "frac": round(kernel_gbs / peak, 4), "traffic": _traffic()},
            "e2e": {"value": round(e2e, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "api": "qgemv_batch(pms, xs): xs = numpy vectors in page-locked host memory (qgemv_batch_inputs), read by the grouped launch over PCIe; y stored into a fresh pinned block (zero-copy both ways), sync; numpy results",
                    "pageable_inputs_gbs": round(e2e_pageable, 1),
                    "pageable_inputs": "the same call on pageable numpy inputs (gathered into the pinned buffer first)",
                    "seam_gbs": round(seam_gbs, 1), "seam_us_per_call": round(seam_us, 1),
                    "seam": "the same 36 matrices as 36 blocking qgemv(pm, x_host) calls (numpy in / numpy out, the reference's per-matrix seam)"},
            "gpu_launches": k_ours * args.steps,
            "kernels_per_step": {"ours": k_ours, "all": k_total},
            "clocks": sampler.report(),
            "decode": decode,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_block(build_cpu_cases(SWEEP))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def measure_decode(workload, B, ctx, layers, steps, warmup, tp_shard=0):
    """One decode step of a random-init LLaMA shard per GPU (tensor parallel
    over the ranks of the process group), replayed as a CUDA graph: device
    tokens/s (max over ranks), roofline on bytes/step, e2e with token ids from
    and to pinned host memory.  Returns a dict (identical on every rank)."""
    import torch
    import torch.distributed as dist
    from paper_2307_03738_b200 import decode as D

    rank, world, local = dist_env()
    cfg = D.LLAMA_7B if workload == "llama7b" else D.LLAMA_65B
    if layers:
        cfg = D.shrink(cfg, n_layers=layers)
    ctx = ctx or (512 if workload == "llama7b" else 1024)
    t0 = time.perf_counter()
    tp = D.ShardTP(tp_shard) if tp_shard > 1 else D.TP()
    model = D.LlamaTP(cfg, batch=B, max_ctx=ctx + 1, seed=0, tp=tp)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    tok = torch.zeros(B, dtype=torch.long, device="cuda")
    pos = ctx  # ctx past tokens in the cache, this step writes position ctx
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for _ in range(2):
            model.step(tok, pos)
        stream.synchronize()
        if world > 1 and getattr(model, "comm", None) is not None:
            # the push all-reduce over peer memory has only ever been verified with ranks
            # emulated on one GPU: check it here (no wait timed out, every rank got the same
            # greedy tokens) and fall back to NCCL otherwise
            bad = torch.tensor([1 if model.comm.error() else 0], device="cuda")
            toks = [torch.empty_like(model.next_tokens) for _ in range(world)]
            dist.all_gather(toks, model.next_tokens.contiguous())
            if any(not torch.equal(t, toks[0]) for t in toks):
                bad.fill_(1)
            dist.all_reduce(bad, op=dist.ReduceOp.MAX)
            if int(bad.item()):
                del model
                torch.cuda.empty_cache()
                model = D.LlamaTP(cfg, batch=B, max_ctx=ctx + 1, seed=0, tp=tp, comm="nccl")
                model.comm_kind = "nccl (the push all-reduce failed its check on this box)"
                for _ in range(2):
                    model.step(tok, pos)
                stream.synchronize()
        if world > 1:
            dist.barrier()
        graph = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(graph, stream=stream):
            nxt = model.step(tok, pos)
        graph.instantiate()
        try:
            k_total, k_ours = graph_kernel_counts(graph)
        except Exception as e:  # noqa: BLE001 (reported, not fatal)
            print(f"kernel count unavailable: {e}", file=sys.stderr)
            k_total = k_ours = None
        sampler = ClockSampler(local)
        with sampler:
            for _ in range(warmup):
                graph.replay()
            stream.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                graph.replay()
            e1.record(stream)
            e1.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / steps
    # e2e: token ids in from pinned host memory, next ids back, every step
    tok_h = torch.zeros(B, dtype=torch.long).pin_memory()
    out_h = torch.zeros(B, dtype=torch.long).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n_e2e = min(steps, 50)
    w0 = time.perf_counter()
    with torch.cuda.stream(stream):
        for _ in range(n_e2e):
            tok.copy_(tok_h, non_blocking=True)
            graph.replay()
            out_h.copy_(nxt, non_blocking=True)
            stream.synchronize()
    e2e_s = (time.perf_counter() - w0) / n_e2e
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    nbytes = model.bytes_per_step(pos)
    if world > 1:
        t = torch.tensor([float(nbytes)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nbytes = int(t.item())
    peak, peak_src = measured_peak()
    gbs = nbytes / (ms_step / 1e3) / 1e9
    comm = getattr(model, "comm_kind", None)
    if getattr(model, "stack", None) is not None:
        if model.stack_error():
            raise RuntimeError("decode stack: a wait inside the persistent kernel timed out")
        engine = ("persistent decode stack: all layers in one cooperative launch "
                  "(csrc/decode_stack.cu)")
    else:
        engine = ("per-op kernel chain (digit epilogues)" if getattr(model, "chained", False)
                  else "per-op kernels")
    res = {
        "value": round(B / (ms_step / 1e3), 2), "unit": "tokens/s",
        "ms_per_step": round(ms_step, 4), "steps": steps,
        "config": {"workload": f"{workload} decode step", "layers": cfg.n_layers,
                   "d_model": cfg.d_model, "bits": cfg.bits, "group": cfg.group, "batch": B,
                   "ctx": ctx, "setup_s": round(setup_s, 1),
                   "parallelism": (f"tp{tp_shard} shard of rank 0 on one GPU, collectives "
                                   f"skipped (per-GPU compute only)") if tp_shard > 1
                   else f"tp{world}", "allreduce": comm, "engine": engine},
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": round(gbs / peak, 4),
                     "bytes_per_step_per_gpu": nbytes, "traffic": None},
        "e2e": {"value": round(B / e2e_s, 2), "unit": "tokens/s", "h2d_bytes_per_step": 8 * B,
                "d2h_bytes_per_step": 8 * B},
        "gpu_launches": None if k_ours is None else k_ours * steps,
        "kernels_per_step": {"ours": k_ours, "all": k_total},
        "clocks": sampler.report(),
    }
    del graph, model
    torch.cuda.empty_cache()
    return res


def init_dist():
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines show the N ranks
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def run_decode(args):
    """BASELINE configs[3]/[4] as the line's own metric (--workload)."""
    import torch.distributed as dist
    rank, world, local = init_dist()
    r = measure_decode(args.workload, args.batch, args.ctx, args.layers, args.steps,
                       args.warmup, args.tp_shard)
    if rank == 0:
        line = {"metric": "decode tokens/s", "value": r["value"], "unit": "tokens/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u8 x s8 -> s32 (IMMA) linears, f16 KV/lm_head",
                "data": "synthetic (random-init weights, random fp16 KV cache)"}
        line.update({k: r[k] for k in ("config", "roofline", "e2e", "gpu_launches",
                                        "kernels_per_step", "clocks")})
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


DECODE_DEFAULT = [("llama7b", 1), ("llama65b", 1), ("llama65b", 8)]


def _kernel_sources_sha16() -> str:
    import hashlib
    h = hashlib.sha256()
    for name in ("gemv_grouped.cu", "gemv_common.cuh", "common.cuh"):
        h.update((ROOT / "paper_2307_03738_b200" / "csrc" / name).read_bytes())
    return h.hexdigest()[:16]


def _traffic():
    """DRAM bytes per step from the committed ncu capture, only if it was taken
    on the current kernel sources (profiles/traffic.json records their hash);
    otherwise None (never a stale number)."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            if d.get("kernel_sources_sha16") == _kernel_sources_sha16():
                return d.get("dram_bytes_per_step")
        except Exception:  # noqa: BLE001
            return None
    return None


def relaunch_distributed(n: int) -> int:
    """`--gpus N` outside torchrun: re-execute under torch.distributed.run, one
    process per GPU (127.0.0.1 rendezvous)."""
    import socket
    import subprocess
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-decode", action="store_true",
                    help="skip the decode measurements (configs[3]/[4]) of the default line")
    ap.add_argument("--workload", choices=["sweep", "llama7b", "llama65b"], default="sweep")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ctx", type=int, default=0)
    ap.add_argument("--layers", type=int, default=0, help="override the layer count (smoke runs)")
    ap.add_argument("--tp-shard", type=int, default=0,
                    help="decode: time rank 0's shard of a TP group of this size on one GPU "
                         "(collectives skipped: per-GPU compute only)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload != "sweep":
        return run_decode(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
