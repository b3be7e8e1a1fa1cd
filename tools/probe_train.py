"""Short parity-training runs (the GPU test's smoke setting and variants): final train loss per setting."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_19150_b200 import train_fsa

for steps, lr in ((300, 2e-3), (300, 5e-4), (600, 2e-3), (600, 5e-4)):
    for seed in (0, 1, 2):
        r = train_fsa.train_task("parity", steps=steps, batch=64, max_len=16, seed=seed, lr=lr)
        print(f"steps {steps} lr {lr} seed {seed}: final_train_loss {r['final_train_loss']:.4f}", flush=True)
