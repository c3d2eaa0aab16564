"""Pins for the oracle's schedule driver and dynamic
update: the round structure is checked against a hand-written
decision trace of the paper's rules on top of the (pinned) oracle sweep."""
from __future__ import annotations

import numpy as np

import oracle
from tests import helpers as H
from workloads import configs, dynamic, graphs


def test_alpha_sequence_clamped():
    """1, 0.3, 0.09, 0.027, 0.0081, then 0.008 (reading R2)."""
    a, seq = 1.0, []
    while True:
        seq.append(a)
        if a <= 0.008:
            break
        a = max(a * 0.3, 0.008)
    np.testing.assert_allclose(seq, [1, 0.3, 0.09, 0.027, 0.0081, 0.008], rtol=1e-12)


def _schedule_by_hand(S, x, q, sch):
    """The paper's rules re-stated literally around oracle.sweep_exact."""
    alpha, trace = sch.alpha0, []
    while True:
        final = alpha <= sch.alpha_min
        for _ in range(sch.max_final_iters if final else sch.a):
            y = oracle.sweep_exact(S, x, alpha, q)
            rel = np.linalg.norm(y - x) / np.linalg.norm(x)
            trace.append(alpha)
            x = y
            if rel < sch.eps:
                break
        if final:
            return x, trace
        alpha = max(alpha * sch.factor, sch.alpha_min)


def test_single_level_schedule_matches_literal_rules():
    w = configs.make("cfg2_rgg1024")
    sch = oracle.paper_schedule(max_final_iters=30)
    x0 = w.x0.astype(np.float64)
    x, e, nl, sw = oracle.layout_schedule(w.graph, w.S, 2, 0.0, 0, sch, w.seed, multilevel=False, x_init=x0)
    xr, trace = _schedule_by_hand(w.S, x0, 0.0, sch)
    assert nl == 1 and sw[0] == len(trace)
    np.testing.assert_array_equal(x, xr)
    np.testing.assert_allclose(e, oracle.energy(w.S, xr, 0.008, 0.0), rtol=0)


def test_converged_path_stops_after_one_sweep_per_round():
    """A fixed point of every alpha is impossible, but a K2 at distance d with no
    non-S pairs is a fixed point for all alpha: each round stops after 1 sweep."""
    g = H.path(2)
    S = H.sset_with(g, np.ones(2))
    x0 = np.array([[0.0, 0.0], [1.0, 0.0]])
    x, e, nl, sw = oracle.layout_schedule(g, S, 2, 0.0, 0, oracle.paper_schedule(), 1, multilevel=False, x_init=x0)
    assert sw[0] == 6  # six rounds (R2), one sweep each
    np.testing.assert_array_equal(x, x0)


def test_multilevel_schedule_levels_and_sweeps():
    w = configs.make("cfg3_mesh32")
    sch = oracle.paper_schedule(max_final_iters=20)
    x, e, nl, sw = oracle.layout_schedule(w.graph, w.S, 2, 0.0, 2, sch, w.seed, n_stop=100)
    assert nl >= 3 and np.all(sw >= 6) and np.all(sw <= 5 * 2 + 20)
    assert np.all(np.isfinite(x))


def test_dynamic_update_runs_finest_level_only():
    w = configs.make("cfg3_mesh32")
    sch = oracle.paper_schedule(max_final_iters=15)
    x, _, _, _ = oracle.layout_schedule(w.graph, w.S, 2, 0.0, 2, sch, w.seed, n_stop=100)
    gq = dynamic.perturb(w.graph, 5.0, 2, seed=3)
    from workloads import sset
    Sq = sset.hop2_sset(gq)
    y, e, nl, sw = oracle.layout_schedule(gq, Sq, 2, 0.0, 2, sch, w.seed, dynamic=True, x_init=x)
    assert nl == 3 and sw[0] >= 1 and np.all(sw[1:] == 0) and sw[0] <= sch.max_final_iters
    # alpha_min from the start: the first sweep equals a plain Eq.(3) sweep at 0.008
    lv = oracle.build_hierarchy(gq, seed=w.seed, n_stop=1, max_levels=3)
    anc = oracle.ancestor(lv, 0, 2)
    y1 = oracle.sweep_approx(Sq, x, 0.008, 0.0, lv[0].parent, anc, lv[2].n)
    y1b, _, _, sw1 = oracle.layout_schedule(gq, Sq, 2, 0.0, 2, oracle.paper_schedule(max_final_iters=1), w.seed,
                                            dynamic=True, x_init=x)
    assert sw1[0] == 1
    np.testing.assert_array_equal(y1, y1b)


def test_perturbation_model():
    g = graphs.grid2d(20, 20)
    q = dynamic.perturb(g, 5.0, 2, seed=1)
    assert q.n == g.n
    from scipy.sparse.csgraph import connected_components
    assert connected_components(q.to_scipy(), directed=False)[0] == 1
    assert abs(q.m - g.m) <= 2


# ---------------------------------------------------------------- full stress (f4)
def test_full_stress_worked_examples():
    """SPEC S:325-326 examples re-derived: path-3 at 0,1,2 -> F = 0 (the pair
    (0,2) has length 2 = d); K2 at distance 3 -> F = (3-1)^2 = 4."""
    g = H.path(3)
    F, s, Fs, P = oracle.full_stress(g, np.array([[0.0, 0], [1, 0], [2, 0]]))
    assert F == 0.0 and P == 3 and s == 1.0
    F, s, Fs, P = oracle.full_stress(H.path(2), np.array([[0.0, 0], [3, 0]]))
    assert F == 4.0 and abs(s - 1 / 3) < 1e-15 and Fs == 0.0


def test_full_stress_against_scipy_and_numeric_min():
    """Distances from scipy's shortest_path (library routine); F(s) minimised
    numerically (bounded scalar search) agrees with the closed form."""
    from scipy.optimize import minimize_scalar
    from scipy.sparse.csgraph import shortest_path

    g = H.random_connected(60, 40, seed=9)
    x = np.random.default_rng(10).normal(size=(g.n, 2)) * 3
    D = shortest_path(g.to_scipy(), unweighted=True, directed=False)
    iu = np.triu_indices(g.n, 1)
    d = D[iu]
    l = np.linalg.norm(x[iu[0]] - x[iu[1]], axis=1)
    F_ref = np.sum((l - d) ** 2 / d ** 2)
    F, s, Fs, P = oracle.full_stress(g, x)
    np.testing.assert_allclose(F, F_ref, rtol=1e-12)
    assert P == iu[0].shape[0]
    res = minimize_scalar(lambda t: np.sum((t * l - d) ** 2 / d ** 2), bounds=(1e-3, 1e3), method="bounded",
                          options={"xatol": 1e-12})
    np.testing.assert_allclose(s, res.x, rtol=1e-6)
    np.testing.assert_allclose(Fs, res.fun, rtol=1e-9)


def test_full_stress_scale_and_rigid_invariance():
    g = H.random_connected(40, 30, seed=11)
    x = np.random.default_rng(12).normal(size=(g.n, 3))
    F, s, Fs, _ = oracle.full_stress(g, x)
    c, sn = np.cos(0.7), np.sin(0.7)
    Q = np.array([[c, -sn, 0], [sn, c, 0], [0, 0, 1.0]])
    F2, s2, Fs2, _ = oracle.full_stress(g, 2.5 * x @ Q.T + 1.0)
    np.testing.assert_allclose(Fs2, Fs, rtol=1e-10)
    np.testing.assert_allclose(s2, s / 2.5, rtol=1e-10)
