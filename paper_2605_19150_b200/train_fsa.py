"""NEXT-4: desk-scale state-tracking training (a Table 1 analogue).

Two Flash PD-SSM blocks (d_model 128, 4 heads, complex state 32 per head, K = sqrt(D) ~ 11),
Adam at lr 2e-3 with linear warm-up and cosine decay, batch 256, train lengths up to 40,
validation on lengths 40..256 (length generalisation), the setup of PAPER.md:785-787 -- but
for a few thousand steps instead of 100,000.  The straight-through temperature is annealed
exponentially from 1 to 0.1 (PAPER.md:201-203 gives no schedule: reading R26).

usage: python -m paper_2605_19150_b200.train_fsa [--tasks parity,cycle_nav,...] [--steps 2000]
prints one JSON line per task."""
from __future__ import annotations

import argparse
import json
import math
import time

import numpy as np
import torch

from paper_2605_19150_b200 import fsa_tasks
from paper_2605_19150_b200.block import FSAClassifier

EVAL_LENGTHS = (40, 64, 100, 128, 160, 200, 256)


def train_task(task, steps=2000, batch=256, max_len=40, lr=2e-3, seed=0, device="cuda", log_every=0, t0=1.0,
               t1=0.1, bmag=2.0, dict_size=None):
    spec = fsa_tasks.TASKS[task]
    torch.manual_seed(seed)
    rng = np.random.default_rng(seed)
    model = FSAClassifier(spec["vocab"], spec["classes"], dict_size=dict_size).to(device)
    with torch.no_grad():
        for b in model.blocks:
            b.mixer.b_mag.fill_(bmag)
    opt = torch.optim.Adam(model.parameters(), lr=lr)
    warm = max(1, steps // 20)
    sched = torch.optim.lr_scheduler.LambdaLR(
        opt, lambda s: (s + 1) / warm if s < warm else 0.5 * (1 + math.cos(math.pi * (s - warm) / max(1, steps - warm))))
    tic = time.time()
    losses = []
    for step in range(steps):
        model.set_temperature(t0 * (t1 / t0) ** (step / max(1, steps - 1)))   # exponential t0 -> t1
        L = int(rng.integers(2, max_len + 1))
        x, y = fsa_tasks.sample(task, batch, L, rng)
        x = torch.from_numpy(x).to(device)
        y = torch.from_numpy(y).to(device)
        loss = torch.nn.functional.cross_entropy(model(x), y)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        torch.nn.utils.clip_grad_norm_(model.parameters(), 1.0)
        opt.step()
        sched.step()
        losses.append(float(loss.detach()))
        if log_every and step % log_every == 0:
            print(f"{task} step {step} loss {np.mean(losses[-log_every:]):.4f}", flush=True)
    torch.cuda.synchronize()
    train_s = time.time() - tic
    model.eval()
    accs = {}
    with torch.no_grad():
        for L in EVAL_LENGTHS:
            x, y = fsa_tasks.sample(task, 512, L, np.random.default_rng(10_000 + L))
            pred = model(torch.from_numpy(x).to(device)).argmax(-1).cpu().numpy()
            accs[L] = float((pred == y).mean())
    return {"task": task, "steps": steps, "batch": batch, "train_max_len": max_len, "seed": seed, "lr": lr,
            "temperature": [t0, t1], "b_mag_init": bmag, "dict_size": model.blocks[0].mixer.K,
            "final_train_loss": float(np.mean(losses[-50:])), "val_acc_by_len": accs,
            "val_acc_mean": float(np.mean(list(accs.values()))), "train_seconds": train_s,
            "ms_per_step": 1e3 * train_s / steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tasks", default="parity,cycle_nav,even_pairs,mod_arith")
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--seeds", type=int, default=1)
    ap.add_argument("--log-every", type=int, default=0)
    ap.add_argument("--lr", type=float, default=2e-3)
    ap.add_argument("--t0", type=float, default=1.0)
    ap.add_argument("--t1", type=float, default=0.1)
    ap.add_argument("--bmag", type=float, default=2.0)
    ap.add_argument("--dict", type=int, default=0, help="dictionary size K (0: round(sqrt(d_model)))")
    a = ap.parse_args()
    for task in a.tasks.split(","):
        for seed in range(a.seeds):
            print(json.dumps(train_task(task, a.steps, a.batch, lr=a.lr, seed=seed, log_every=a.log_every, t0=a.t0,
                                        t1=a.t1, bmag=a.bmag,
                                        dict_size=a.dict or None)), flush=True)


if __name__ == "__main__":
    main()
