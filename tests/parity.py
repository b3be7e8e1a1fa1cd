"""Parity measures shared by the GPU tests (reading R19 / SURVEY A19).

`rel`      max|gpu - oracle| / max|oracle| over the whole tensor;
`rel_bh`   the same ratio inside every (b, h) sequence (its own maximum as the scale), maximised
           over the sequences, so an error in a low-magnitude head cannot hide under another
           head's maximum;
`check`    asserts both against one bar and, when $PDSSM_PARITY_LOG names a file, appends the
           measured values as a JSON line (tests/parity_report.py tabulates them).

Bars: 1e-4 for fp32 inputs, 2e-2 for bf16 inputs (BASELINE.json north_star).  DESIGN.md R19 derives
why the bf16 values stay well inside 2e-2 (one RNE rounding of each stored output, plus one-ulp
differences of bf16-stored intermediates the backward consumes)."""
import json
import os

import numpy as np

TOL = {"f32": 1e-4, "bf16": 2e-2}


def _arr(a, like):
    cplx = np.iscomplexobj(a) or np.iscomplexobj(like)
    return np.asarray(a, dtype=np.complex128 if cplx else np.float64)


def rel(a, b):
    a = _arr(a, b)
    b = _arr(b, a)
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-30))


def rel_bh(a, b, axes=(0, 1)):
    """max over the (b, h) sequences (the two `axes`) of the per-sequence relative error."""
    a = _arr(a, b)
    b = _arr(b, a)
    if b.size == 0:
        return 0.0
    a = np.moveaxis(a, axes, (0, 1))
    b = np.moveaxis(b, axes, (0, 1))
    B, H = b.shape[:2]
    err = np.abs(a - b).reshape(B, H, -1).max(axis=-1)
    scale = np.maximum(np.abs(b).reshape(B, H, -1).max(axis=-1), 1e-30)
    # a sequence whose reference is exactly zero must be reproduced exactly
    return float(np.max(err / scale))


def check(name, got, ref, tol, bh_axes=(0, 1)):
    r = rel(got, ref)
    rb = rel_bh(got, ref, bh_axes) if bh_axes is not None else None
    log = os.environ.get("PDSSM_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"name": name, "tol": tol, "rel": r, "rel_bh": rb,
                                "test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]}) + "\n")
    assert r <= tol, f"{name}: per-tensor relative error {r:.3e} > {tol:.1e}"
    if rb is not None:
        assert rb <= tol, f"{name}: per-(b,h) relative error {rb:.3e} > {tol:.1e}"
    return r, rb
