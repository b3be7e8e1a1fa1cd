#!/usr/bin/env python
"""Benchmark of the Flash PD-SSM fwd+bwd scan on B200 (BASELINE.json metric:
"PD-SSM fwd+bwd scan tokens/s at L=2048, d=1024; HBM GB/s vs peak; 1/2/4/8 GPU").

A step = pdssm_scan_fwd (h_t + chunk_state) followed by pdssm_scan_bwd (db, dD, g)
over one batch of the headline workload (config 2: B=16, L=2048, H=8, N=128,
K=32, complex fp32, per-step D), inputs resident in HBM (>= 1.3 GB per step, larger
than the 126 MB L2, so no flush is needed).  Multi-GPU: one process per GPU,
batch x head sharding with no data-path collective -- every rank runs its own
full batch (weak scaling); value = all ranks' tokens / max-over-ranks time.

--impl reference times the float64 CPU oracle (oracle/, the only reference this
paper-only tier has) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PD-SSM fwd+bwd scan tokens/s at L=2048,d=1024; HBM GB/s vs peak; 1/2/4/8 GPU"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--complex", type=int, default=2, choices=[1, 2])
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--state", type=int, default=128)
    ap.add_argument("--tau", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-layer", action="store_true")
    ap.add_argument("--seed", type=int, default=2000)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def peak_tflops(dtype):
    """Dense tensor peak for the layer GEMMs: measured cuBLAS bf16 burst; fp32 runs use the
    3xTF32 split (3 tf32 MMAs per product, tf32 = 1/2 bf16 nominal) -> bf16/6 useful."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    bf = 1645.9
    if os.path.exists(p):
        with open(p) as f:
            bf = float(json.load(f).get("bf16_tflops", bf))
    return bf if dtype == "bf16" else bf / 6.0


def traffic_of(kernel):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "traffic_latest.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f).get(kernel)


def count_launches(fn):
    """Kernels one call of fn launches (CUPTI via torch.profiler), counted outside the timed region."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA" and "pdssm" in e.name]
    return len(names), sorted(set(n.split("(")[0][:80] for n in names))


def algo_bytes_per_seq_step(N, c, p):
    """fwd reads D, b, k*, writes h -> 3cNp + 1;
    bwd reads dh, D, h_{t-1}, k*, writes db, dD, g -> 5cNp + 5."""
    return 3 * c * N * p + 1, 5 * c * N * p + 5


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, idx):
        self.idx = idx
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{idx}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_sample(L, N, K, c, seed, seqs=1):
    """Oracle (O5 + O8, float64 NumPy) on `seqs` (b,h) sequences of the workload."""
    import oracle as O
    import synth
    inp = synth.scan_inputs(1, seqs, L, N, K, c, seed=seed, dh=True)
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    Dz, bz, ez = (O.planes_to_complex(inp[k]) for k in ("diag", "bias", "dh"))
    t0 = time.perf_counter()
    h = O.scan_forward(Pm, Dz, bz)
    O.scan_backward(Pm, Dz, h, ez)
    return time.perf_counter() - t0


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    B, L, H, N, K, c = 16, 2048, a.heads, a.state, 32, a.complex
    Lh = 512                                    # bounded sample: one (b,h) sequence, 512 steps
    cpu_oracle_sample(64, N, K, c, a.seed)     # warm numpy
    for _ in range(a.warmup):
        pass
    times = [cpu_oracle_sample(Lh, N, K, c, a.seed + i) for i in range(a.steps)]
    t = float(np.sum(times))
    tokens = a.steps * Lh / H                   # one head of Lh tokens = Lh/H token-equivalents
    v = tokens / t
    cores = 1
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * t / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config2 fig1-shape scan fwd+bwd (oracle sample)", "batch": B, "seq_len": L,
                       "heads": H, "state": N, "dict": K, "complex": c == 2},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"1 (b,h) sequence x {Lh} steps per step, N={N}, complex={c == 2}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def layer_kernels(P, torch, dev, adt, dtype, B, L, H, N, K, c, stream):
    """Time select (a2/a3), projection (a5) and readout (a8) at the config-2 layer shape
    (d_in = d = H*N, readout rows P = d/H) with CUDA events on the launching stream."""
    d_in, Pp = H * N, N
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn((B, L, d_in), device=dev, generator=g).to(adt)
    S = ((torch.rand((H, K, d_in), device=dev, generator=g) * 2 - 1) / d_in ** 0.5).to(adt)
    Bw = ((torch.rand((H, c, N, d_in), device=dev, generator=g) * 2 - 1) / d_in ** 0.5).to(adt)
    Cw = (torch.rand((H, c, Pp, N), device=dev, generator=g) * 2 - 1) / N ** 0.5
    bout = torch.empty((B, H, L, c, N), device=dev, dtype=adt)
    y = torch.empty((B, L, H, Pp), device=dev, dtype=adt)
    k_sel = torch.empty((B, H, L), device=dev, dtype=torch.uint8)
    dims = P.make_dims(B, H, L, N, 1, c=c, dtype=P.BF16 if dtype == "bf16" else P.F32, p_out=Pp)
    wsr = torch.empty(max(P.workspace_bytes(dims, P.OP_READOUT), 256), dtype=torch.uint8, device=dev)

    def t(fn, n=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3   # us

    # NEXT-2 layer-level forward (select -> b = Bx -> scan -> y), PER_DICT diagonals D_k
    di = torch.randint(0, N, (H, K, N), device=dev, generator=g).to(torch.int16)
    Dk = (torch.rand((H, K, c, N), device=dev, generator=g) * 2 - 1) * 0.7
    lo = {"kstar": torch.empty((B, H, L), device=dev, dtype=torch.uint8), "h": bout, "y": y}
    tl = t(lambda: P.layer_fwd(x, S, di, Dk, Bw, C=Cw, per_dict=True, out=lo))
    Dout = torch.empty((B, H, L, c, N), device=dev, dtype=adt)
    bmag = torch.randn((H, N), device=dev, generator=g) + 2.0
    tg_ = t(lambda: P.diag_gen(x, Bw, bmag, out=Dout))   # NEXT-2 D_t generator (fused sigmoid/sincos epilogue)
    # NEXT-3 PD-SSM soft generator (Eqs. 2-4) as the comparison baseline of the hard selection
    lg = torch.randn((B, H, L, K), device=dev, generator=g)
    Md = (torch.rand((H, K, N, N), device=dev, generator=g) * 2 - 1) / N ** 0.5
    Pso = torch.empty((B, H, L, N), device=dev, dtype=torch.int16)
    dso = P.make_dims(B, H, L, N, K, dtype=P.BF16 if dtype == "bf16" else P.F32)
    wso = torch.empty(P.workspace_bytes(dso, P.OP_SOFT), dtype=torch.uint8, device=dev)
    tso = t(lambda: P.soft_select(lg, Md, bf16=dtype == "bf16", out=Pso, ws=wso))
    ts = t(lambda: P.select(x, S))
    tp = t(lambda: P.project(x, Bw, out=bout))
    tr = t(lambda: P.readout(bout, Cw, out=y, ws=wsr))
    peak = peak_tflops(dtype)
    f_sel = 2.0 * B * L * H * K * d_in
    f_prj = 2.0 * B * L * H * c * N * d_in
    f_rd = 2.0 * B * L * H * c * N * Pp
    out = {"dtype": dtype, "tensor_peak_tflops": peak,
           "tensor_peak_kind": "measured bf16 burst" + (" / 6 (3xTF32)" if dtype != "bf16" else ""),
           "shape": {"d_in": d_in, "P": Pp, "K": K}}
    for name, us, fl in (("select", ts, f_sel), ("project", tp, f_prj), ("readout", tr, f_rd), ("diag_gen", tg_, f_prj)):
        tf = fl / (us * 1e-6) / 1e12
        out[name] = {"us": us, "tflops": tf, "frac": tf / peak}
    f_soft = 2.0 * B * L * H * K * N * N
    out["soft_select_baseline"] = {"us": tso, "tflops": f_soft / (tso * 1e-6) / 1e12,
                                   "frac": f_soft / (tso * 1e-6) / 1e12 / peak,
                                   "vs_hard_select": tso / ts,
                                   "what": "PD-SSM generator (Eqs. 2-4): mixture GEMM + column hardmax epilogue"}
    out["layer_fwd"] = {"us": tl, "tokens_per_s": B * L / (tl * 1e-6), "diag": "per_dict",
                        "chain": "pdssm_layer_fwd = select + project + scan_fwd + readout"}
    return out


def surrogate_kernels(P, torch, dev, d, fo, bo, dims, dtype, B, L, H, N, K, c, p, stream):
    """NEXT-1 (Prop. 2): selector dlogits and the dense dictionary gradient,
    timed alone on the bench's own backward outputs (lambda = dbias, the saved h, D).
    dict_grad algorithmic bytes per (b,h,t): read lambda, D, h_{t-1} (3cNp) + k* (1 per CTA scan,
    counted once); flops 2 c N^2 per (b,h,t) (the grouped outer-product GEMM)."""
    g = torch.Generator(device=dev).manual_seed(11)
    M = (torch.rand((H, K, N, N), device=dev, generator=g) * 2 - 1) / N ** 0.5
    logits = torch.randn((B, H, L, K), device=dev, generator=g)
    dM = torch.empty_like(M)
    dl = torch.empty_like(logits)

    def t(fn, n=10):
        """n calls captured in one CUDA graph (the calls are graph-safe), so host-side
        argument marshalling does not pad the device time of these short kernels."""
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs), torch.cuda.graph(graph, stream=gs):
            for _ in range(n):
                fn()
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3   # us

    td = t(lambda: P.dict_grad(M, d["kstar"], d["diag"], fo["h"], bo["dbias"], 1.0, dims, out=dM))
    tsg = t(lambda: P.select_grad(logits, d["kstar"], bo["gsel"], 1.0, out=dl))
    peak, _ = peaks()
    dbytes = (3 * c * N * p + 1) * B * H * L + 2 * H * K * N * N * 4
    dflops = 2.0 * c * N * N * B * H * L
    sbytes = (8 * K + 5) * B * H * L
    tpk = peak_tflops(dtype) if dtype == "bf16" else peak_tflops("f32")
    return {"dict_grad": {"us": td, "gbs": dbytes / (td * 1e-6) / 1e9, "hbm_frac": dbytes / (td * 1e-6) / 1e9 / peak,
                          "tflops": dflops / (td * 1e-6) / 1e12, "tensor_frac": dflops / (td * 1e-6) / 1e12 / tpk,
                          "algo_bytes": dbytes, "flops": dflops,
                          "path": "tcgen05 kind::tf32 3xTF32" if N == 128 else "simt"},
            "select_grad": {"us": tsg, "gbs": sbytes / (tsg * 1e-6) / 1e9, "hbm_frac": sbytes / (tsg * 1e-6) / 1e9 / peak,
                            "algo_bytes": sbytes}}


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    import paper_2605_19150_b200 as P
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    B, L, H, N, K, c = 16, 2048, a.heads, a.state, 32, a.complex
    bf16 = a.dtype == "bf16"
    p = 2 if bf16 else 4
    adt = torch.bfloat16 if bf16 else torch.float32
    # global inputs are generated per rank-shard (batch x head sharding: rank r owns batch block r)
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=a.seed + 17 * rank, dh=True, bf16=bf16)
    host = {k: torch.from_numpy(v) for k, v in inp.items()}
    d = {k: v.to(dev) for k, v in host.items()}
    d["dict_idx"] = d["dict_idx"].to(torch.int16)
    for k in ("diag", "bias", "dh"):
        d[k] = d[k].to(adt)
    # outputs / workspaces preallocated once (calls are allocation-free)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], tau=a.tau)
    dims = f["dims"]
    fo = {"h": f["h"], "chunk_state": f["chunk_state"],
          "ws": torch.empty(P.workspace_bytes(dims, P.OP_FWD), dtype=torch.uint8, device=dev)}
    bo = {"ws": torch.empty(P.workspace_bytes(dims, P.OP_BWD), dtype=torch.uint8, device=dev),
          "dbias": torch.empty_like(f["h"]), "ddiag": torch.empty_like(f["h"]),
          "gsel": torch.empty((B, H, L), dtype=torch.float32, device=dev)}
    stream = torch.cuda.current_stream()

    def step_fwd():
        return P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], tau=a.tau, out=fo)

    def step_bwd(fr):
        return P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], fr["h"], fr["chunk_state"], dims, dh=d["dh"],
                          want_dh0=False, out=bo)

    for _ in range(max(a.warmup, 3)):
        step_bwd(step_fwd())
    torch.cuda.synchronize()
    try:
        launches_per_step, kernel_names = count_launches(lambda: step_bwd(step_fwd()))
    except Exception as ex:   # profiler unavailable: the fused path's documented count
        launches_per_step, kernel_names = 4, [f"profiler failed: {ex}"[:80]]

    # ---- timed region: K steps, per-call CUDA events on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    clk = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(a.steps):
        ev[i][0].record(stream)
        fr = step_fwd()
        ev[i][1].record(stream)
        step_bwd(fr)
        ev[i][2].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    if world > 1:
        dist.barrier()
    elapsed = t_start.elapsed_time(t_end) / 1e3
    fwd_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    bwd_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))
    if world > 1:
        tt = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = float(tt.item())
    tokens_per_rank = B * L
    value = world * tokens_per_rank * a.steps / elapsed

    fb, bb = algo_bytes_per_seq_step(N, c, p)
    S = B * H
    fwd_bytes = fb * S * L
    bwd_bytes = bb * S * L
    peak, peak_kind = peaks()
    dominant = "scan_bwd" if bwd_ms >= fwd_ms else "scan_fwd"
    dom_bytes, dom_ms = (bwd_bytes, bwd_ms) if dominant == "scan_bwd" else (fwd_bytes, fwd_ms)
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    step_gbs = (fwd_bytes + bwd_bytes) / (elapsed / a.steps) / 1e9

    # ---- end-to-end through the public API with pinned host buffers
    e2e = None
    if not a.no_e2e:
        pin = {k: host[k].pin_memory() for k in ("kstar", "diag", "bias", "dh")}
        if bf16:
            pin = {k: (v.to(adt).pin_memory() if k in ("diag", "bias", "dh") else v) for k, v in pin.items()}
        g_host = torch.empty((B, H, L), dtype=torch.float32).pin_memory()
        h2d = sum(v.numel() * v.element_size() for v in pin.values())
        d2h = g_host.numel() * 4
        e_steps = max(3, min(a.steps, 10))

        def e2e_step():
            for k, v in pin.items():
                d[k].copy_(v, non_blocking=True)
            fr = step_fwd()
            step_bwd(fr)
            g_host.copy_(bo["gsel"], non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(e_steps):
            e2e_step()
        s1.record(stream)
        torch.cuda.synchronize()
        et = s0.elapsed_time(s1) / 1e3
        if world > 1:
            tt = torch.tensor([et], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            et = float(tt.item())
        e2e = {"value": world * tokens_per_rank * e_steps / et, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h)}

    # ---- CPU oracle baseline on a bounded sample (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        Lh = 512
        cpu_oracle_sample(64, N, K, c, a.seed)
        reps = 3
        t = sum(cpu_oracle_sample(Lh, N, K, c, a.seed + i) for i in range(reps))
        cpu = {"value": reps * Lh / H / t, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{reps} x one (b,h) sequence of {Lh} steps (N={N}, complex={c == 2}), fwd O5 + bwd O8, "
                         "float64 NumPy, single thread; tokens = steps/H"}

    # ---- layer-level kernels of the path (a2/a3 select, a5 projection, a8 readout), timed alone
    layer = None
    if not a.no_layer:
        layer = layer_kernels(P, torch, dev, adt, a.dtype, B, L, H, N, K, c, stream)
        layer["surrogate_grads"] = surrogate_kernels(P, torch, dev, d, fo, bo, dims, a.dtype, B, L, H, N, K, c, p,
                                                     stream)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
                "ms_per_step": 1e3 * elapsed / a.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": a.dtype, "data": "synthetic",
                "config": {"workload": "config2: paper Fig.1 shape, fwd+bwd scan", "batch_per_gpu": B, "seq_len": L,
                           "heads": H, "state": N, "d": H * N, "dict": K, "complex": c == 2, "diag": "per_step",
                           "tau": int(f["tau"]), "parallelism": f"dp{world} (batch x head shards, no collective)",
                           "l2": "inputs larger than L2 (>=1.3 GB per step), no flush"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic_of(dominant), "kernel": dominant,
                             "algo_bytes_per_launch": dom_bytes, "peak_kind": peak_kind,
                             "traffic_source": "profiles/traffic_latest.json (ncu --set full, dram read+write per launch)"},
                "step_hbm": {"achieved_gbs": step_gbs, "frac": step_gbs / peak, "fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
                             "algo_bytes_fwd": fwd_bytes, "algo_bytes_bwd": bwd_bytes},
                "clocks": clocks, "e2e": e2e, "gpu_launches": launches_per_step * a.steps,
                "launches_per_step": {"count": launches_per_step, "kernels": kernel_names},
                "layer_kernels": layer, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
