"""Synthetic state-tracking tasks of the paper's Table 1 (generated as in
Deletang et al., the setup of PAPER.md:785-787): a random sequence of input symbols, the label is
the automaton's final state (no intermediate supervision).

  parity       symbols {0, 1};          label = number of 1s mod 2
  cycle_nav    symbols {+1, -1, stay};  label = position on a 5-cycle after the moves (start 0)
  even_pairs   symbols {a, b};          label = 1 iff the numbers of "ab" and "ba" pairs are equal,
                                        i.e. the first and the last symbol agree
  mod_arith    symbols {0..4, +, -, *}; alternating operand / operator, operands first and last;
                                        label = left-to-right evaluation mod 5 (SPEC.md:493 leaves
                                        precedence unstated: reading R31, no precedence)

Data generation only (test/training harness of NEXT-4); the labels are computed by the task
definitions directly, not by the model."""
from __future__ import annotations

import numpy as np

TASKS = {
    "parity": dict(vocab=2, classes=2),
    "cycle_nav": dict(vocab=3, classes=5),
    "even_pairs": dict(vocab=2, classes=2),
    "mod_arith": dict(vocab=8, classes=5),
}


def sample(task, batch, length, rng):
    """(tokens int64 [batch][length], labels int64 [batch])."""
    if task == "parity":
        x = rng.integers(0, 2, size=(batch, length))
        return x, x.sum(axis=1) % 2
    if task == "cycle_nav":
        x = rng.integers(0, 3, size=(batch, length))
        step = np.where(x == 0, 1, np.where(x == 1, -1, 0))
        return x, step.sum(axis=1) % 5
    if task == "even_pairs":
        x = rng.integers(0, 2, size=(batch, length))
        return x, (x[:, 0] == x[:, -1]).astype(np.int64)
    if task == "mod_arith":
        n = length if length % 2 == 1 else length - 1   # operand (op operand)*
        n = max(n, 1)
        operands = rng.integers(0, 5, size=(batch, (n + 1) // 2))
        ops = rng.integers(0, 3, size=(batch, n // 2))   # 0 +, 1 -, 2 *
        x = np.empty((batch, n), np.int64)
        x[:, 0::2] = operands
        x[:, 1::2] = 5 + ops
        val = operands[:, 0].copy()
        for i in range(ops.shape[1]):
            o, v = ops[:, i], operands[:, i + 1]
            val = np.where(o == 0, val + v, np.where(o == 1, val - v, val * v)) % 5
        return x, val
    raise KeyError(task)
