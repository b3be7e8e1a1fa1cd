"""NEXT-4 task data (paper_2605_19150_b200/fsa_tasks.py) against the automata of oracle/fsa.py
(themselves pinned against independent interpreters in test_oracle_pins.py): every generated label
is the automaton's final state label (Prop. 1's FSAs; tasks PAPER.md:303-313)."""
import numpy as np
import pytest

from oracle import fsa
from paper_2605_19150_b200 import fsa_tasks

AUTOMATA = {"parity": fsa.parity, "cycle_nav": fsa.cycle_nav, "even_pairs": fsa.even_pairs, "mod_arith": fsa.mod_arith}


@pytest.mark.parametrize("task", sorted(fsa_tasks.TASKS))
@pytest.mark.parametrize("length", [1, 2, 7, 40, 41])
def test_labels_are_automaton_runs(task, length):
    A = AUTOMATA[task]()
    x, y = fsa_tasks.sample(task, 64, length, np.random.default_rng(length))
    assert x.max() < fsa_tasks.TASKS[task]["vocab"] and y.max() < fsa_tasks.TASKS[task]["classes"]
    for row, lab in zip(x, y):
        assert A.label[A.run(list(row))[-1]] == lab
