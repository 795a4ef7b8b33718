"""The oracle (reference compiled into oracle/_ref) is pinned against the
golden vectors recorded in SURVEY §8(c) and the reference's own known-answer
tests, before anything is compared against it."""
import math

import numpy as np
import pytest

import ref


def test_threefry_golden():
    assert ref.threefry([0, 0, 0, 0], [0, 0, 0, 0]) == [
        0x0068c71d9376b741, 0x400933a14e65d6c4, 0xeae334bacaeedb8e, 0x4e8fdcfaedb0c1bb]
    assert ref.threefry([1, 2, 3, 4], [7, 0, 0, 0]) == [
        0x61f1b2de62009234, 0xe652b7d18dd8e838, 0xf52db324729c9eff, 0x3b6400e0f244207a]


def test_normal_uniform_golden():
    assert [ref.normal_for([9, 9, 9, 9], n) for n in range(4)] == [
        -0.6440914772193016, 0.01829712429490133, -0.034442890301287318, 0.87464058382000676]
    assert [ref.uniform_for([1, 2, 3, 4], n) for n in range(4)] == [
        0.42215537193592678, 0.66898891201998423, 0.83606679467008072, 0.4723881525473691]


def test_stc_protocol_golden():
    h, z, p = ref.run_stc_protocol(0, 0)  # STET trial 0
    assert (h, z, p) == (4.5449467093946359, 0.75323495592946443, 0.24731552999708523)


def test_solve_tree_two_compartment_closed_form():
    # test_solver.cpp:39-65 analogue: symmetric two-compartment relaxation
    cap, a = 2.0, 0.5
    v = ref.solve_tree([-1, 0], [cap, cap], [0.0, 0.0], [0.0, a], [0.0, 0.0], [-40.0, -80.0])
    d = (-40.0 + 80.0) * cap / (cap + 2 * a)
    assert abs((v[0] - v[1]) - d) < 1e-12 * abs(d)
    assert abs(0.5 * (v[0] + v[1]) + 60.0) < 1e-12


def test_worker_invariance_small_net():
    # test_engine.cpp:287-309: results never depend on the worker count
    cfg = ref.default_consolidation(n_cells=50, n_exc=40, pattern=10, t_learn_ms=500.0, seed=11)
    rr = ref.RefRecipe.consolidation(cfg)
    runs = []
    for w in (1, 3):
        e = ref.RefEngine(rr.view, 0.5, 11, w)
        e.advance_to(800.0)
        runs.append(e.spike_arrays())
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])
    assert len(runs[0][0]) > 50


def test_er_density():
    n, p = 300, 0.1
    c = sum(ref.er_connected(3, i, j, n, p) for i in range(n) for j in range(n))
    mean = p * n * (n - 1)
    assert abs(c - mean) < 3 * math.sqrt(mean * (1 - p))
