"""Pins for oracle/br.py, oracle/egt.py, oracle/cfr.py, oracle/lp.py (no GPU)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import br, cfr, dgf, egt, games, lp, seqform

from .test_oracle_dgf import interior_point
from .test_oracle_games import random_treeplex

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def kuhn():
    return seqform.build(games.kuhn())


def pennies():
    return seqform.build(games.matrix_game([[1, -1], [-1, 1]]))


# ----------------------------------------------------------------- best response / gap
@pytest.mark.parametrize("seed", range(10))
def test_best_response_vs_vertex_enumeration(seed):
    rng = np.random.default_rng(seed)
    tp = random_treeplex(rng, int(rng.integers(2, 7)))
    g = rng.standard_normal(tp.n_seq)
    for sense in ("min", "max"):
        v, q = br.best_response(tp, g, sense)
        assert math.isclose(v, q @ g, rel_tol=1e-12, abs_tol=1e-12)
        assert math.isclose(v, br.brute_force_best_response(tp, g, sense), rel_tol=1e-12, abs_tol=1e-12)


def test_gap_examples_matching_pennies():
    sf = pennies()
    u = sf.X.uniform()
    assert abs(br.saddle_gap(sf, u, sf.Y.uniform())) < 1e-15
    x = np.array([1.0, 1.0, 0.0])
    assert math.isclose(br.saddle_gap(sf, x, sf.Y.uniform()), 1.0)


def test_gap_nonnegative_random():
    sf = kuhn()
    rng = np.random.default_rng(0)
    for _ in range(200):
        assert br.saddle_gap(sf, interior_point(sf.X, rng), interior_point(sf.Y, rng)) >= -1e-12


# ----------------------------------------------------------------- LP values (pins for A + treeplex)
def test_kuhn_value_lp():
    g = json.load(open(os.path.join(GOLD, "kuhn.json")))
    v, _ = lp.game_value(kuhn())
    assert abs(-v - g["value_to_player1"]) < 1e-9


def test_leduc_value_lp():
    g = json.load(open(os.path.join(GOLD, "leduc.json")))
    v, _ = lp.game_value(seqform.build(games.leduc()))
    assert abs(-v - g["value_to_player1"]) < g["tolerance"]


# ----------------------------------------------------------------- EGT
@pytest.mark.parametrize("game", ["kuhn", "pennies"])
def test_egt_theory_egc_and_bounds(game):
    """With mu_x mu_y = ||A||^2/(phi_X phi_Y) the EGC holds at every
    iterate, eps_sad <= mu_x Omega_X + mu_y Omega_Y and
    eps_sad(x^T, y^T) <= 4||A||/(T+1) sqrt(Omega_X Omega_Y / (phi_X phi_Y))."""
    sf = kuhn() if game == "kuhn" else pennies()
    X, Y = sf.X, sf.Y
    An = sf.max_abs_A()
    bound_c = 4 * An * math.sqrt(X.Omega * Y.Omega / (X.phi * Y.phi))
    prob = egt.Problem(sf)
    mu = egt.theory_mu(sf)
    x, y = egt.initialize(prob, mu, mu)
    st = egt.EGTState(x, y, mu, mu)
    scale = mu * (X.Omega + Y.Omega)
    assert egt.excessive_gap(prob, st.x, st.y, st.mu_x, st.mu_y) >= -1e-9 * scale
    for T in range(1, 301):
        egt.egt_iteration(prob, st, "theory")
        assert X.check_feasible(st.x) and Y.check_feasible(st.y)
        egv = egt.excessive_gap(prob, st.x, st.y, st.mu_x, st.mu_y)
        assert egv >= -1e-9 * (st.mu_x * X.Omega + st.mu_y * Y.Omega)
        gap = br.saddle_gap(sf, st.x, st.y)
        assert gap <= st.mu_x * X.Omega + st.mu_y * Y.Omega + 1e-12
        assert gap <= bound_c / (T + 1) + 1e-12


def test_egt_as_backtracks_and_keeps_egc():
    sf = kuhn()
    prob = egt.Problem(sf)
    mu = 0.05 * egt.theory_mu(sf)
    x, y = egt.initialize(prob, mu, mu)
    st = egt.EGTState(x, y, mu, mu, tau=0.99)      # forced failure: tau far too large
    mu_prev = (st.mu_x, st.mu_y)
    for _ in range(60):
        tau_before = st.tau
        focus_x = st.mu_x > st.mu_y
        egt.egt_iteration(prob, st, "as")
        assert egt.excessive_gap(prob, st.x, st.y, st.mu_x, st.mu_y) >= 0
        # the focused player's mu shrinks by exactly (1 - tau_accepted)
        if focus_x:
            assert math.isclose(st.mu_x, mu_prev[0] * (1 - st.tau), rel_tol=1e-14) and st.mu_y == mu_prev[1]
        else:
            assert math.isclose(st.mu_y, mu_prev[1] * (1 - st.tau), rel_tol=1e-14) and st.mu_x == mu_prev[0]
        assert st.tau <= tau_before
        mu_prev = (st.mu_x, st.mu_y)
    assert st.backtracks >= 1


@pytest.mark.parametrize("variant,iters", [("balanced", 600), ("as", 300)])
def test_egt_practical_converges_on_kuhn(variant, iters):
    sf = kuhn()
    st, prob = egt.run(sf, variant, iters, mu=0.05 * egt.theory_mu(sf))
    gap = br.saddle_gap(sf, st.x, st.y)
    assert gap < 5e-3
    val = st.x @ (sf.A @ st.y)
    assert abs(-val - (-1 / 18)) < 5e-3


def test_egt_symmetric_fixed_point_pennies():
    sf = pennies()
    st, _ = egt.run(sf, "theory", 5)
    assert np.allclose(st.x[1:], 0.5) and np.allclose(st.y[1:], 0.5)


# ----------------------------------------------------------------- RM / RM+ / CFR
def test_rm_examples():
    z0 = np.array([0.5, 0.5])
    r, z = cfr.regret_update("rm", np.zeros(2), z0, np.array([1.0, 0.0]))
    assert np.allclose(r, [0.5, -0.5]) and np.allclose(z, [1.0, 0.0])
    r, z = cfr.regret_update("rmp", np.zeros(2), z0, np.array([-1.0, 0.0]))
    assert np.allclose(r, [0.0, 0.5]) and np.allclose(z, [0.0, 1.0])
    # all regrets negative -> uniform (PAPER.md:64 comment)
    r, z = cfr.regret_update("rm", np.array([-1.0, -2.0]), z0, np.array([0.0, 0.0]))
    assert np.allclose(z, 0.5)


def test_regret_minimisers_shift_invariant():
    rng = np.random.default_rng(0)
    for kind in ("rm", "rmp"):
        r = rng.standard_normal(4) if kind == "rm" else np.abs(rng.standard_normal(4))
        z = rng.random(4)
        z /= z.sum()
        g = rng.standard_normal(4)
        a = cfr.regret_update(kind, r, z, g)
        b = cfr.regret_update(kind, r, z, g + 3.7)
        assert np.allclose(a[0], b[0], atol=1e-13) and np.allclose(a[1], b[1], atol=1e-13)


def test_alpha_schedules():
    assert cfr.alpha("uniform", 1) == 1 and cfr.alpha("uniform", 4) == 0.25
    assert cfr.alpha("linear", 1) == 1 and math.isclose(cfr.alpha("linear", 3), 0.5)
    # uniform averaging of iterates is the arithmetic mean
    rng = np.random.default_rng(0)
    xs = rng.random((10, 3))
    avg = np.zeros(3)
    for t, x in enumerate(xs, 1):
        a = cfr.alpha("uniform", t)
        avg = a * x + (1 - a) * avg
    assert np.allclose(avg, xs.mean(0), atol=1e-14)


def test_cfr_rock_paper_scissors():
    sf = seqform.build(games.matrix_game([[0, -1, 1], [1, 0, -1], [-1, 1, 0]]))
    for v in ("cfr_rm", "cfr_rmp", "cfr_plus"):
        st = cfr.run(sf, v, 3000)
        assert br.saddle_gap(sf, st.xbar, st.ybar) < 2e-2
        assert np.allclose(st.xbar[1:], 1 / 3, atol=2e-2)


@pytest.mark.parametrize("variant", ["cfr_rm", "cfr_rmp", "cfr_plus"])
def test_cfr_kuhn(variant):
    sf = kuhn()
    st = cfr.run(sf, variant, 2000)
    L = 4.0  # maximum payoff difference for player 1 in Kuhn: +2 .. -2
    assert br.saddle_gap(sf, st.xbar, st.ybar) <= 1e-2
    assert abs(-(st.xbar @ (sf.A @ st.ybar)) - (-1 / 18)) < 5e-3
    assert st.grads == 2 * 2000
    assert sf.X.check_feasible(st.xbar) and sf.Y.check_feasible(st.ybar)
    del L


def test_cfr_plus_bound():
    """eps_sad(xbar, ybar) is the sum of both players' regrets; each is bounded by
    2|S|L sqrt(max n_j)/sqrt(T)."""
    sf = kuhn()
    st = cfr.CFRState(sf, "cfr_plus")
    L = 4.0
    for T in range(1, 1001):
        cfr.cfr_iteration(st)
        if T in (1, 3, 10, 30, 100, 300, 1000):
            gap = br.saddle_gap(sf, st.xbar, st.ybar)
            assert gap <= 2 * cfr.cfr_plus_regret_bound(sf, T, L)


# ----------------------------------------------------------------- practical mu (reading R14)
@pytest.mark.parametrize("name", ["kuhn", "leduc", "pennies"])
def test_practical_mu_scan(name):
    """The scan returns the last k before the EGC at the initial point first fails: the EGC
    holds at mu_theory * 2^-j for every j <= k (Nesterov's theorem covers j = 0,
    PAPER.md:363-371) and fails at k + 1 (unless k is the cap)."""
    sf = {"kuhn": kuhn, "pennies": pennies, "leduc": lambda: seqform.build(games.leduc())}[name]()
    k, mu = egt.practical_mu(sf, kmax=30)
    mu_th = egt.theory_mu(sf)
    assert mu == mu_th * 2.0 ** -k
    prob = egt.Problem(sf)
    for j in range(k + 2):
        if j > 30:
            break
        m = mu_th * 2.0 ** -j
        x0, y0 = egt.initialize(prob, m, m)
        assert sf.X.check_feasible(x0) and sf.Y.check_feasible(y0)
        egv = egt.excessive_gap(prob, x0, y0, m, m)
        assert (egv >= 0) == (j <= k), (j, egv)


def test_egt_as_from_practical_mu_keeps_egc_and_converges():
    """EGT/as (Alg. 3-4) from the practical mu on Kuhn: every accepted iterate satisfies the
    EGC, eps_sad <= mu_x Omega_X + mu_y Omega_Y, and it approaches -1/18."""
    sf = kuhn()
    k, mu = egt.practical_mu(sf)
    assert k >= 1
    prob = egt.Problem(sf)
    x, y = egt.initialize(prob, mu, mu)
    st = egt.EGTState(x, y, mu, mu)
    for _ in range(400):
        egt.egt_iteration(prob, st, "as")
        assert egt.excessive_gap(prob, st.x, st.y, st.mu_x, st.mu_y) >= 0
        gap = br.saddle_gap(sf, st.x, st.y)
        assert -1e-12 <= gap <= st.mu_x * sf.X.Omega + st.mu_y * sf.Y.Omega + 1e-12
    assert br.saddle_gap(sf, st.x, st.y) < 2e-3
    assert abs(-(st.x @ (sf.A @ st.y)) - (-1 / 18)) < 2e-3
