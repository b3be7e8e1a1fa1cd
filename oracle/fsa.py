"""Deterministic FSAs and the Prop. 1 construction (App. D
PAPER.md:849-858).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

An automaton is (n_states, n_symbols, delta[sigma][q], q_init, label[q]).  The
Prop. 1 map to a Flash PD-SSM is

    A(sigma) = sum_q enc(delta(q, sigma)) enc(q)^T

i.e. dictionary entry k = sigma has the column-one-hot index map
dict_idx[sigma][q] = delta(q, sigma), diagonal 1, B = 0, h0 = enc(q_init)
(reading R5) and one readout row per label class (reading R23).
"""
from __future__ import annotations

import numpy as np


class Automaton:
    def __init__(self, name, delta, q_init, label):
        self.name = name
        self.delta = np.asarray(delta, dtype=np.int64)      # [K][N]
        self.K, self.N = self.delta.shape
        self.q_init = int(q_init)
        self.label = np.asarray(label, dtype=np.int64)      # [N]
        assert (self.delta >= 0).all() and (self.delta < self.N).all()

    def run(self, tokens):
        """left fold of delta from q_init; returns the state after each token."""
        q = self.q_init
        out = []
        for s in tokens:
            q = int(self.delta[s, q])
            out.append(q)
        return out

    def compile(self):
        """Prop. 1: (dict_idx [1][K][N] uint16, diag [1][K][N] (=1), h0 [N], C [n_cls][N])."""
        dict_idx = self.delta.astype(np.uint16)[None]
        diag = np.ones((1, self.K, self.N))
        h0 = np.zeros(self.N)
        h0[self.q_init] = 1.0
        n_cls = int(self.label.max()) + 1
        C = np.zeros((n_cls, self.N))
        for q in range(self.N):
            C[self.label[q], q] = 1.0
        return dict_idx, diag, h0, C


def parity():
    """alphabet {0,1}; flip on 1."""
    return Automaton("parity", [[0, 1], [1, 0]], 0, [0, 1])


def cyclic_z5():
    """Z_5 word problem: symbol s rotates the state by s (K=5)."""
    return Automaton("z5", [[(q + s) % 5 for q in range(5)] for s in range(5)], 0, list(range(5)))


def cycle_nav():
    """cycle navigation: symbols {+1, -1, 0} on 5 positions."""
    moves = [1, -1, 0]
    return Automaton("cycle_nav", [[(q + m) % 5 for q in range(5)] for m in moves], 0, list(range(5)))


def even_pairs():
    """even pairs: label = (first symbol == last symbol).
    states: 0 = start, 1+2*f+l for first f, last l in {a=0, b=1}."""
    N = 5
    delta = np.zeros((2, N), dtype=np.int64)
    for s in range(2):
        delta[s, 0] = 1 + 2 * s + s
        for f in range(2):
            for l in range(2):
                delta[s, 1 + 2 * f + l] = 1 + 2 * f + s
    label = [1, 1, 0, 0, 1]          # empty string counts as "equal"
    return Automaton("even_pairs", delta, 0, label)


MOD_OPS = ["none", "+", "-", "*"]


def mod_arith():
    """mod-5 arithmetic evaluated left to right (no precedence, SPEC.md:493 leaves
    it unstated).  symbols 0..4 = digits, 5,6,7 = '+','-','*'.  state = value*4+op
    with op in (none,+,-,*); start = (0,'+').  Digit after a digit restarts the
    value; operator after operator replaces it (totalisation, ours).  '*0'
    collapses every value to 0, so the maps are non-injective."""
    N, K = 20, 8
    delta = np.zeros((K, N), dtype=np.int64)
    for v in range(5):
        for op in range(4):
            q = v * 4 + op
            for d in range(5):
                if op == 0:
                    nv = d
                elif op == 1:
                    nv = (v + d) % 5
                elif op == 2:
                    nv = (v - d) % 5
                else:
                    nv = (v * d) % 5
                delta[d, q] = nv * 4 + 0
            for o in range(3):
                delta[5 + o, q] = v * 4 + (o + 1)
    label = [q // 4 for q in range(N)]
    return Automaton("mod_arith", delta, 0 * 4 + 1, label)


# independent interpreters (no delta table) used to pin the tables above
def interp_parity(tokens):
    return sum(tokens) % 2


def interp_z5(tokens):
    return sum(tokens) % 5


def interp_cycle_nav(tokens):
    return sum({0: 1, 1: -1, 2: 0}[s] for s in tokens) % 5


def interp_even_pairs(tokens):
    if not tokens:
        return 1
    return int(tokens[0] == tokens[-1])


def interp_mod_arith(tokens):
    value, pending = 0, "+"
    for s in tokens:
        if s < 5:
            if pending is None:
                value = s
            elif pending == "+":
                value = (value + s) % 5
            elif pending == "-":
                value = (value - s) % 5
            else:
                value = (value * s) % 5
            pending = None
        else:
            pending = "+-*"[s - 5]
    return value
