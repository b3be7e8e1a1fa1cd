#!/usr/bin/env python
"""Benchmark of the Flash PD-SSM fwd+bwd scan on B200 (BASELINE.json metric:
"PD-SSM fwd+bwd scan tokens/s at L=2048, d=1024; HBM GB/s vs peak; 1/2/4/8 GPU").

A step = pdssm_scan_fwd (h_t + chunk_state) followed by pdssm_scan_bwd (db, dD, g) over one
batch of the chosen workload, inputs resident in HBM (every config moves >= 0.5 GB per step,
more than the 126 MB L2, so no flush is needed).  Workloads (BASELINE.json configs):

  --config 2 (default, the headline): B=16 per GPU, L=2048, H=8, N=128 (d = 1024), K=32, complex,
             PER_STEP D; batch x head, weak scaling: the global batch is 16*G rows generated once
             (row-wise seeded streams) and rank r takes rows [16r, 16r+16) -- no collective.
  --config 4: hybrid-LLM layer, B=32, H=32, L=4096, N=64, K=48, real, bf16; batch x head, STRONG
             scaling: the 1024 (b, h) sequences are split over the G ranks.
  --config 3: long time series, B=4, H=8, L=17984, N=128, K=32, real fp32, temporally persistent
             k*; sequence parallel (strong): rank g owns steps [gL/G, (g+1)L/G) of every sequence,
             one all-gather of segment summaries per direction over NCCL.
  --config 5: S_5 word problem, B=4, H=4, L=65536, N=64, K=16, PER_DICT D = 1, b = 0,
             h0 = arange; sequence parallel (strong).
  --dtype f32|bf16, --mode bh|sp override the config's natural choice; --recompute runs the
  backward in recompute mode (no saved states; chunk 64).

Multi-GPU: one process per GPU (torchrun), barrier + synchronize around exactly K timed steps,
max over ranks; value = all ranks' tokens / that time.  --impl reference times the float64 CPU
oracle (oracle/, the only reference this paper-only tier has) on a bounded sample of the same
workload.
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

# name, B, H, L, N, K, c, dtype, mode, scaling, extras
BENCH_CONFIGS = {
    2: dict(workload="config2: paper Fig.1 shape, fwd+bwd scan", B=16, H=8, L=2048, N=128, K=32, c=2,
            dtype="f32", mode="bh", scaling="weak", seed=2000),
    3: dict(workload="config3: long time series (EigenWorms-like), fwd+bwd scan", B=4, H=8, L=17984, N=128, K=32,
            c=1, dtype="f32", mode="sp", scaling="strong", seed=3000, sticky=0.9),
    4: dict(workload="config4: hybrid-LLM layer, fwd+bwd scan", B=32, H=32, L=4096, N=64, K=48, c=1,
            dtype="bf16", mode="bh", scaling="strong", seed=4000),
    5: dict(workload="config5: S_5 word problem stress, fwd+bwd scan", B=4, H=4, L=65536, N=64, K=16, c=1,
            dtype="f32", mode="sp", scaling="strong", seed=5000, s5=True),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(BENCH_CONFIGS))
    ap.add_argument("--dtype", default=None, choices=["f32", "bf16"])
    ap.add_argument("--mode", default=None, choices=["bh", "sp"])
    ap.add_argument("--recompute", action="store_true", help="backward without saved states (chunk 64)")
    ap.add_argument("--tau", type=int, default=0)
    ap.add_argument("--seeds", type=int, default=3, help="seeds 0..n-1 timed (value from seed 0; min/max reported)")
    ap.add_argument("--stat-steps", type=int, default=50, help="extra steps for the per-step median")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-layer", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional test of the multi-rank paths with several ranks sharing one GPU")
    ap.add_argument("--profile", action="store_true",
                    help="under ncu: one seed, no clock block, no per-step statistics, no CPU / e2e / layer legs")
    a = ap.parse_args()
    if a.profile:
        a.seeds, a.stat_steps, a.no_cpu_baseline, a.no_e2e, a.no_layer = 1, 1, True, True, True
    return a


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
    bf = 1590.0
    if os.path.exists(p):
        with open(p) as f:
            bf = float(json.load(f).get("bf16_tflops", bf))
    return bf if dtype == "bf16" else bf / 6.0


def traffic_of(kernel, config, dsuffix=""):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "traffic_latest.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        j = json.load(f)
    return j.get(f"config{config}{dsuffix}:{kernel}", j.get(kernel) if (config == 2 and not dsuffix) else None)


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


def algo_bytes_per_seq_step(N, c, p, per_dict=False, recompute=False):
    """fwd reads D, b, k*, writes h -> 3cNp + 1;
    bwd reads dh, D, h_{t-1}, k*, writes db, dD, g -> 5cNp + 5.  PER_DICT drops the D stream
    (2cNp + 1, 4cNp + 5).  Recompute mode reads b instead of h_{t-1} (same count)."""
    d = 0 if per_dict else 1
    return (2 + d) * c * N * p + 1, (4 + d) * c * N * p + 5


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


# ---------------------------------------------------------------- CPU oracle baseline
def _cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return model, cores


def _oracle_task(args):
    """Oracle O5 + O8 (float64 NumPy, sequential; one thread) on the (b, h) sequences `rows` x all
    heads of the workload's global inputs; returns (compute start, compute end) wall times."""
    os.environ["OMP_NUM_THREADS"] = "1"
    cfg, seed, b, L = args
    import oracle as O
    import synth
    H, N, K, c = cfg["H"], cfg["N"], cfg["K"], cfg["c"]
    if cfg.get("s5"):
        dict5, _, _ = synth.s5_dictionary(N, K, seed=5000)
        inp = synth.scan_inputs_rows(cfg["B"], H, L, N, K, c, seed, rows=(b, b + 1), dh=True, per_dict=True)
        inp["dict_idx"] = np.tile(dict5[None], (H, 1, 1))
        Dz = np.ones((1, H, L, N), np.complex128)
        bz = np.zeros((1, H, L, N), np.complex128)
    else:
        inp = synth.scan_inputs_rows(cfg["B"], H, L, N, K, c, seed, rows=(b, b + 1), dh=True,
                                     sticky=cfg.get("sticky", 0.0))
        Dz, bz = (O.planes_to_complex(inp[k]) for k in ("diag", "bias"))
    Pm = O.gather_P(inp["dict_idx"], inp["kstar"])
    ez = O.planes_to_complex(inp["dh"])
    t0 = time.time()
    h = O.scan_forward(Pm, Dz, bz)
    O.scan_backward(Pm, Dz, h, ez)
    return t0, time.time()


def cpu_oracle_baseline(cfg, budget_s=8.0):
    """The oracle as it stands on the host cores, on the workload's own shape (full L, its global
    inputs): batch rows (each = H head sequences) on 1 core in turn, and on all affinity cores as a
    process pool (one row per task).  Rows are added until ~budget_s of single-core work; the all-core
    leg runs up to cores x that many rows.  tokens = rows x L; throughput = tokens / compute wall span."""
    import multiprocessing as mp
    model, cores = _cpu_info()
    L = cfg["L"]
    t0, t1 = _oracle_task((cfg, cfg["seed"], 0, L))
    per_row = t1 - t0
    n1 = int(max(1, min(cfg["B"], budget_s // max(per_row, 1e-3))))
    spans = [_oracle_task((cfg, cfg["seed"], b, L)) for b in range(n1)]
    one = n1 * L / sum(e - s for s, e in spans)
    nall = int(max(1, min(cfg["B"] * 8, cores * max(1, budget_s // max(per_row, 1e-3)))))
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        spans = pool.map(_oracle_task, [(cfg, cfg["seed"] + 1 + b // cfg["B"], b % cfg["B"], L) for b in range(nall)])
    wall = max(e for _, e in spans) - min(s for s, _ in spans)
    allc = nall * L / wall
    return {"value": allc, "unit": UNIT, "cores": cores, "kind": "oracle", "value_1core": one, "cpu_model": model,
            "sample": f"{cfg['workload'].split(':')[0]} at full shape (L={L}, H={cfg['H']}, N={cfg['N']}, K={cfg['K']}, "
                      f"c={cfg['c']}): 1 core {n1} batch rows in turn, all {cores} affinity cores {nall} rows as a "
                      f"process pool; fwd O5 + bwd O8, float64 NumPy, one thread per process; tokens = rows x L"}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = BENCH_CONFIGS[a.config]
    cb = cpu_oracle_baseline(cfg)
    v = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": cfg["scaling"],
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"] + " (oracle sample)", "batch": cfg["B"], "seq_len": cfg["L"],
                       "heads": cfg["H"], "state": cfg["N"], "dict": cfg["K"], "complex": cfg["c"] == 2},
            "cpu_baseline": cb,
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
    # NEXT-2 layer forward with D_t generated in the same GEMM as the selector and the projection
    Wd = ((torch.rand((H, c, N, d_in), device=dev, generator=g) * 2 - 1) / d_in ** 0.5).to(adt)
    lo2 = {"kstar": torch.empty((B, H, L), device=dev, dtype=torch.uint8), "h": bout, "y": y}
    tgen = t(lambda: P.layer_fwd(x, S, di, None, Bw, C=Cw, Wd=Wd, bias_mag=bmag, out=lo2))
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
                        "chain": "pdssm_layer_fwd = fused (select + project) GEMM + scan_fwd + readout"}
    out["layer_fwd_gen"] = {"us": tgen, "tokens_per_s": B * L / (tgen * 1e-6), "diag": "per_step, generated",
                            "chain": "pdssm_layer_fwd_gen = fused (select + project + D_t generator) GEMM + scan_fwd + readout",
                            "unfused_sum_us": ts + tp + tg_ + tr,
                            "unfused_parts": "select + project + diag_gen + readout timed alone (scan excluded)"}
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


def make_inputs(cfg, a, seed, world, rank, bf16):
    """Host inputs of this rank: generated globally (row-wise streams), then sliced.
    Returns (inp dict of numpy arrays, B_local, L_local, description of the shard)."""
    import synth
    from paper_2605_19150_b200.parallel import shard_range
    B, H, L, N, K, c = cfg["B"], cfg["H"], cfg["L"], cfg["N"], cfg["K"], cfg["c"]
    mode = a.mode or cfg["mode"]
    if mode == "bh" and cfg["scaling"] == "weak":
        Bg, rows, t0, t1 = B * world, (B * rank, B * rank + B), 0, L
        shard = f"dp{world}: rows [{rows[0]}, {rows[1]}) of a global batch of {Bg} (weak scaling, no collective)"
    elif mode == "bh":
        Bg, rows, t0, t1 = B, shard_range(B, world, rank), 0, L
        shard = f"dp{world}: batch rows [{rows[0]}, {rows[1]}) x {H} heads of {B * H} sequences (strong, no collective)"
    else:
        Bg, rows = B, (0, B)
        t0, t1 = shard_range(L, world, rank)
        shard = f"sp{world}: steps [{t0}, {t1}) of L = {L} (strong; one all-gather of segment summaries per direction)"
    if cfg.get("s5"):
        dict5, _, _ = synth.s5_dictionary(N, K, seed=5000)
        inp = synth.scan_inputs_rows(Bg, H, L, N, K, c, seed, rows=rows, dh=True, per_dict=True)
        inp["dict_idx"] = np.tile(dict5[None], (H, 1, 1))
        inp["diag"] = np.ones((H, K, c, N), np.float32)
        inp["bias"] = np.zeros_like(inp["bias"])
        inp["h0"] = np.tile(np.arange(N, dtype=np.float32).reshape(1, 1, 1, N), (rows[1] - rows[0], H, c, 1))
    else:
        inp = synth.scan_inputs_rows(Bg, H, L, N, K, c, seed, rows=rows, dh=True, sticky=cfg.get("sticky", 0.0),
                                     bf16=bf16)
    if (t0, t1) != (0, L):
        for k in ("kstar", "diag", "bias", "dh"):
            if k in inp and not (k == "diag" and cfg.get("s5")):
                inp[k] = np.ascontiguousarray(inp[k][:, :, t0:t1])
    return inp, rows[1] - rows[0], t1 - t0, shard, Bg


class Step:
    """One fwd+bwd scan step through the public API on this rank's shard."""

    def __init__(self, P, torch, dev, cfg, a, inp, bf16, world):
        self.P, self.torch = P, torch
        adt = torch.bfloat16 if bf16 else torch.float32
        self.pd = bool(cfg.get("s5"))
        self.host = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in inp.items()}
        d = {k: v.to(dev) for k, v in self.host.items()}
        d["dict_idx"] = d["dict_idx"].to(torch.int16)
        for k in ("diag", "bias", "dh"):
            if not (k == "diag" and self.pd):
                d[k] = d[k].to(adt)
        self.d = d
        self.adt = adt
        self.world = world
        self.mode = a.mode or cfg["mode"]
        self.recompute = a.recompute
        self.tau = a.tau if a.tau else (64 if a.recompute else 0)
        self.h0 = d.get("h0")
        f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=self.h0, tau=self.tau, per_dict=self.pd)
        self.dims = f["dims"]
        self.tau_eff = int(f["tau"])
        self.fo = {"h": f["h"], "chunk_state": f["chunk_state"],
                   "ws": torch.empty(P.workspace_bytes(self.dims, P.OP_FWD), dtype=torch.uint8, device=dev)}
        self.bo = {"ws": torch.empty(P.workspace_bytes(self.dims, P.OP_BWD), dtype=torch.uint8, device=dev),
                   "dbias": torch.empty_like(f["h"]),
                   "ddiag": torch.empty(d["diag"].shape, dtype=torch.float32 if self.pd else adt, device=dev),
                   "gsel": torch.empty(d["kstar"].shape, dtype=torch.float32, device=dev)}
        self.sp = None
        if self.mode == "sp" and world > 1:
            from paper_2605_19150_b200.parallel import CudaOps, SequenceParallelScan
            self.sp = SequenceParallelScan(CudaOps(cfg["N"], cfg["K"], cfg["c"], tau=self.tau, per_dict=self.pd))

    def fwd(self):
        d = self.d
        if self.sp is not None:
            out, ctx = self.sp.forward(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=self.h0)
            return (out, ctx)
        return self.P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=self.h0, tau=self.tau,
                               per_dict=self.pd, out=self.fo)

    def bwd(self, fr):
        d = self.d
        if self.sp is not None:
            out, ctx = fr
            return self.sp.backward(d["kstar"], d["dict_idx"], d["diag"], out, ctx, d["dh"])
        hs = None if self.recompute else fr["h"]
        return self.P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], hs, fr["chunk_state"], self.dims, dh=d["dh"],
                               h0=self.h0, want_dh0=False, out=self.bo, bias=d["bias"] if self.recompute else None)

    def step(self):
        return self.bwd(self.fwd())


def timed(torch, dist, st, stream, steps, world, dev, per_step=True):
    """Exactly `steps` steps between a barrier + synchronize on both sides; CUDA events on the
    launching stream; returns (elapsed s max over ranks, [fwd ms], [bwd ms])."""
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)] if per_step else []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(steps):
        if per_step:
            ev[i][0].record(stream)
            fr = st.fwd()
            ev[i][1].record(stream)
            st.bwd(fr)
            ev[i][2].record(stream)
        else:
            st.step()
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    el = t_start.elapsed_time(t_end) / 1e3
    if world > 1:
        tt = torch.tensor([el], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = float(tt.item())
    fw = [e[0].elapsed_time(e[1]) for e in ev]
    bw = [e[1].elapsed_time(e[2]) for e in ev]
    return el, fw, bw


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist

    import paper_2605_19150_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(torch.cuda.device_count(), 1)   # (gloo tests: several ranks may share one GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if a.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    cfg = BENCH_CONFIGS[a.config]
    dtype = a.dtype or cfg["dtype"]
    bf16 = dtype == "bf16"
    p = 2 if bf16 else 4
    B, H, L, N, K, c = cfg["B"], cfg["H"], cfg["L"], cfg["N"], cfg["K"], cfg["c"]
    mode = a.mode or cfg["mode"]
    scaling = cfg["scaling"] if mode == cfg["mode"] else ("strong" if mode == "sp" else "weak")
    stream = torch.cuda.current_stream()

    seed_vals = []
    main_res = None
    for si in range(max(1, a.seeds)):
        inp, B_loc, L_loc, shard, Bg = make_inputs(cfg, a, cfg["seed"] + si, world, rank, bf16)
        st = Step(P, torch, dev, cfg, a, inp, bf16, world)
        for _ in range(max(a.warmup, 3)):
            st.step()
        torch.cuda.synchronize()
        if si == 0 and not a.profile:   # nvidia-smi sampling spans the timed region of the reported value
            clk = Clocks(local)
            clk.start()
            time.sleep(0.3)
        el, fw, bw = timed(torch, dist, st, stream, a.steps, world, dev)
        if si == 0 and not a.profile:
            timed(torch, dist, st, stream, max(a.steps, 200), world, dev, per_step=False)
            clocks = clk.stop()
        elif si == 0:
            clocks = None
        tokens_all = (Bg if cfg["scaling"] == "weak" and mode == "bh" else B) * L   # whole-job tokens per step
        v = tokens_all * a.steps / el
        seed_vals.append(v)
        if si == 0:
            main_res = (st, inp, B_loc, L_loc, shard, Bg, el, fw, bw, tokens_all)
        else:
            del st
    st, inp, B_loc, L_loc, shard, Bg, elapsed, fw, bw, tokens_all = main_res
    value = seed_vals[0]
    try:
        if a.profile:
            raise RuntimeError("not counted under --profile")
        launches_per_step, kernel_names = count_launches(st.step)
    except Exception as ex:
        launches_per_step, kernel_names = None, [f"profiler failed: {ex}"[:80]]
    # per-step median over --stat-steps further steps (seed 0)
    _, sfw, sbw = timed(torch, dist, st, stream, max(a.stat_steps, 1), world, dev)
    step_ms = [f_ + b_ for f_, b_ in zip(sfw, sbw)]
    fwd_ms, bwd_ms = float(np.median(sfw)), float(np.median(sbw))


    fb, bb = algo_bytes_per_seq_step(N, c, p, per_dict=bool(cfg.get("s5")))
    S_loc = B_loc * H
    fwd_bytes, bwd_bytes = fb * S_loc * L_loc, bb * S_loc * L_loc
    peak, peak_kind = peaks()
    dominant = "scan_bwd" if bwd_ms >= fwd_ms else "scan_fwd"
    dom_bytes, dom_ms = (bwd_bytes, bwd_ms) if dominant == "scan_bwd" else (fwd_bytes, fwd_ms)
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    step_gbs = (fwd_bytes + bwd_bytes) / (np.median(step_ms) / 1e3) / 1e9

    # ---- end to end through the public API: H2D of the step's inputs from pinned host memory,
    #      fwd + bwd, D2H of the gradients (db, dD, g) into pinned host memory, every step
    e2e = None
    if not a.no_e2e and st.sp is None:
        keys = ["kstar", "diag", "bias", "dh"] if not st.pd else ["kstar", "bias", "dh"]
        pin = {}
        for k in keys:
            t = st.host[k]
            if bf16 and k in ("diag", "bias", "dh"):
                t = t.to(torch.bfloat16)
            pin[k] = t.pin_memory()
        outs = {k: torch.empty(st.bo[k].shape, dtype=st.bo[k].dtype).pin_memory() for k in ("dbias", "ddiag", "gsel")}
        h2d = sum(v.numel() * v.element_size() for v in pin.values())
        d2h = sum(v.numel() * v.element_size() for v in outs.values())
        e_steps = max(3, min(a.steps, 5))
        # Pipelined over three streams: the H2D of step i+1 and the D2H of step i-1 run on the copy
        # engines while step i computes (device inputs and outputs double-buffered, the pinned host
        # buffers shared); every step still moves its inputs in and its gradients out inside the
        # timed region, which ends when the last D2H has landed.
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        d_sets = [st.d, dict(st.d)]
        o_sets = [st.bo, dict(st.bo)]
        for k in keys:
            d_sets[1][k] = torch.empty_like(st.d[k])
        for k in outs:
            o_sets[1][k] = torch.empty_like(st.bo[k])
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_c = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        d0, bo0 = st.d, st.bo

        def e2e_run(n, s_end):
            for i in range(n):
                j = i % 2
                with torch.cuda.stream(s_in):
                    if i >= 2:
                        s_in.wait_event(ev_c[j])           # step i-2 has finished reading these inputs
                    for k, v in pin.items():
                        d_sets[j][k].copy_(v, non_blocking=True)
                    ev_in[j].record(s_in)
                stream.wait_event(ev_in[j])
                if i >= 2:
                    stream.wait_event(ev_out[j])           # the D2H of step i-2 has read these outputs
                st.d, st.bo = d_sets[j], o_sets[j]
                st.step()
                ev_c[j].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_c[j])
                    for k, v in outs.items():
                        v.copy_(o_sets[j][k], non_blocking=True)
                    ev_out[j].record(s_out)
            stream.wait_stream(s_in)
            stream.wait_stream(s_out)
            if s_end is not None:
                s_end.record(stream)

        e2e_run(2, None)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        e2e_run(e_steps, s1)
        torch.cuda.synchronize()
        st.d, st.bo = d0, bo0
        et = s0.elapsed_time(s1) / 1e3
        if world > 1:
            tt = torch.tensor([et], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            et = float(tt.item())
        e2e = {"value": tokens_all * e_steps / et, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "copies": "H2D " + ", ".join(keys) + "; D2H db, dD, g",
               "pipelined": "H2D of step i+1 and D2H of step i-1 overlap step i (copy streams, double buffers)"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_oracle_baseline(cfg)

    layer = None
    if a.config == 2 and world == 1 and not a.no_layer and not a.recompute:
        layer = layer_kernels(P, torch, dev, st.adt, dtype, B, L, H, N, K, c, stream)
        layer["surrogate_grads"] = surrogate_kernels(P, torch, dev, st.d, st.fo, st.bo, st.dims, dtype, B, L, H, N,
                                                     K, c, p, stream)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": 1e3 * elapsed / a.steps, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": {"workload": cfg["workload"], "config_id": a.config, "batch": Bg,
                           "batch_per_gpu": B_loc if mode == "bh" else Bg, "seq_len": L, "seq_len_per_gpu": L_loc,
                           "heads": H, "state": N, "d": H * N, "dict": K, "complex": c == 2,
                           "diag": "per_dict (D = 1)" if cfg.get("s5") else "per_step", "tau": st.tau_eff,
                           "backward": "recompute (no saved states)" if a.recompute else "saved states",
                           "parallelism": shard,
                           "l2": "inputs larger than L2 (>= 0.5 GB per step), no flush"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic_of(dominant, a.config, "" if dtype == BENCH_CONFIGS[a.config]["dtype"] else "_" + dtype), "kernel": dominant,
                             "algo_bytes_per_launch": dom_bytes, "peak_kind": peak_kind,
                             "traffic_source": "profiles/traffic_latest.json (ncu --set full, dram read+write per launch)"},
                "step_hbm": {"achieved_gbs": step_gbs, "frac": step_gbs / peak, "fwd_ms_median": fwd_ms,
                             "bwd_ms_median": bwd_ms, "step_ms_median": float(np.median(step_ms)),
                             "stat_steps": len(step_ms), "algo_bytes_fwd": fwd_bytes, "algo_bytes_bwd": bwd_bytes,
                             "per_rank": world > 1},
                "seeds": {"values": seed_vals, "min": min(seed_vals), "max": max(seed_vals),
                          "seeds": [cfg["seed"] + i for i in range(len(seed_vals))]},
                "clocks": clocks, "e2e": e2e,
                "gpu_launches": None if launches_per_step is None else launches_per_step * a.steps,
                "launches_per_step": {"count": launches_per_step, "kernels": kernel_names},
                "layer_kernels": layer, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
