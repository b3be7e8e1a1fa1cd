"""Small invocations of every kernel family, run under compute-sanitizer by
tests/test_gpu_sanitizer.py (racecheck / synccheck / memcheck).  Not a test module itself.
usage: python tests/sanitize_driver.py <family>"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2605_19150_b200 as P  # noqa: E402
import synth  # noqa: E402


def dev(inp, bf16=False):
    d = {}
    for k, v in inp.items():
        t = torch.from_numpy(np.ascontiguousarray(v)).cuda()
        if k == "dict_idx":
            t = t.to(torch.int16)
        elif bf16 and k in ("diag", "bias", "dh"):
            t = t.to(torch.bfloat16)
        d[k] = t
    return d


def scan(path, B, H, L, N, K, c, tau, bf16=False, per_dict=False, recompute=False, maps=False):
    os.environ["PDSSM_PATH"] = path
    inp = synth.scan_inputs(B, H, L, N, K, c, seed=L + N, h0=True, dh=True, bf16=bf16, per_dict=per_dict)
    d = dev(inp, bf16 and not per_dict)
    if per_dict and bf16:
        for k in ("bias", "dh"):
            d[k] = d[k].to(torch.bfloat16)
    f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"], h0=d["h0"], tau=tau, per_dict=per_dict,
                   export_maps=maps)
    P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], None if recompute else f["h"], f["chunk_state"], f["dims"],
               dh=d["dh"], h0=d["h0"], bias=d["bias"] if recompute else None)
    torch.cuda.synchronize()


def main(family):
    if family == "seq":
        scan("seq", 2, 2, 70, 128, 8, 2, 0)
        scan("seq", 2, 2, 70, 64, 8, 1, 0, bf16=True)
        scan("seq", 1, 2, 40, 64, 5, 2, 0, per_dict=True, maps=True)
    elif family == "seq_paired":
        os.environ.pop("PDSSM_PATH", None)
        os.environ["PDSSM_SEQ_PAIR_BWD"] = "1"
        scan("", 2, 160, 40, 64, 8, 1, 0)
    elif family == "fused":
        scan("fused", 2, 2, 150, 128, 8, 2, 32)
        scan("fused", 1, 2, 100, 64, 8, 1, 16, bf16=True)
        scan("fused", 1, 2, 100, 32, 5, 2, 16, per_dict=True)
    elif family == "generic":
        scan("generic", 1, 2, 60, 40, 6, 2, 16)
        scan("generic", 1, 2, 60, 16, 6, 1, 7, recompute=True)
        scan("generic", 1, 1, 40, 8, 3, 2, 8, per_dict=True)
    elif family == "gemm":
        os.environ.pop("PDSSM_PATH", None)
        B, L, H, K, N, d_in = 1, 160, 2, 16, 32, 64
        x = torch.randn(B, L, d_in, device="cuda")
        S = torch.randn(H, K, d_in, device="cuda")
        di = torch.from_numpy(synth.random_maps(H, K, N, seed=1).astype(np.int16)).cuda()
        P.select(x, S, di, want_P=True, want_logits=True)
        P.select(x.bfloat16(), S.bfloat16(), di)
        Bw = torch.randn(H, 2, N, d_in, device="cuda")
        b = P.project(x, Bw)
        Cw = torch.randn(H, 2, 16, N, device="cuda")
        P.readout(b, Cw)
        torch.cuda.synchronize()
    elif family == "surrogate":
        os.environ.pop("PDSSM_PATH", None)
        B, H, L, N, K, c = 1, 2, 64, 128, 4, 2
        inp = synth.scan_inputs(B, H, L, N, K, c, seed=5, dh=True)
        d = dev(inp)
        f = P.scan_fwd(d["kstar"], d["dict_idx"], d["diag"], d["bias"])
        db, _, g, _ = P.scan_bwd(d["kstar"], d["dict_idx"], d["diag"], f["h"], f["chunk_state"], f["dims"], dh=d["dh"])
        M = torch.from_numpy(synth.dictionary(H, K, N, 6)).cuda()
        P.dict_grad(M, d["kstar"], d["diag"], f["h"], db, 1.0, f["dims"])
        logits = torch.randn(B, H, L, K, device="cuda")
        P.select_grad(logits, d["kstar"], g, 1.0)
        torch.cuda.synchronize()
    else:
        raise SystemExit(f"unknown family {family}")
    print("done", family)


if __name__ == "__main__":
    main(sys.argv[1])
