"""Pins for oracle/dgf.py: dilated entropy, smoothed best response, prox (no GPU)."""
import math

import numpy as np
import pytest
from scipy.optimize import minimize

from oracle import dgf, games, seqform
from oracle.treeplex import Treeplex

from .test_oracle_games import fig1, random_treeplex


def interior_point(tp, rng, spread=2.0):
    b = tp.uniform_behavioral()
    for j in range(tp.n_simplex):
        s, n = tp.start[j], tp.size[j]
        w = np.exp(spread * rng.standard_normal(n))
        b[s:s + n] = w / w.sum()
    return tp.behavioral_to_sequence(b)


def kuhn_X():
    return seqform.build(games.kuhn()).X


def test_single_simplex_values():
    tp = Treeplex(3, [(1, 2, 0)])
    assert tp.beta[0] == 2
    assert math.isclose(dgf.dgf_value(tp, np.array([1, 1.0, 0.0])), 2 * math.log(2))
    want = 2 * (0.25 * math.log(0.25) + 0.75 * math.log(0.75) + math.log(2))
    assert math.isclose(dgf.dgf_value(tp, np.array([1, 0.25, 0.75])), want)
    assert abs(dgf.dgf_value(tp, tp.uniform())) < 1e-15


@pytest.mark.parametrize("tpf", [lambda: fig1()[0], kuhn_X])
def test_dgf_nonnegative_zero_at_centre(tpf):
    tp = tpf()
    rng = np.random.default_rng(0)
    assert abs(dgf.dgf_value(tp, tp.uniform())) < 1e-12
    for _ in range(100):
        assert dgf.dgf_value(tp, interior_point(tp, rng)) >= -1e-12


@pytest.mark.parametrize("tpf", [lambda: fig1()[0], kuhn_X, lambda: random_treeplex(np.random.default_rng(5), 8)])
def test_gradient_finite_differences(tpf):
    """Appendix gradient vs central differences of d in the free coordinates
    (the appendix formula uses sum_{i'} q_{i'} = q_i, valid at feasible q)."""
    tp = tpf()
    rng = np.random.default_rng(1)
    for _ in range(20):
        q = interior_point(tp, rng, 1.0)
        g = dgf.dgf_gradient(tp, q)
        for i in range(1, tp.n_seq):
            h = 1e-6 * q[i]
            qp, qm = q.copy(), q.copy()
            qp[i] += h
            qm[i] -= h
            fd = (dgf.dgf_value(tp, qp) - dgf.dgf_value(tp, qm)) / (2 * h)
            assert abs(fd - g[i]) <= 1e-5 * max(1.0, abs(g[i]))


def test_gradient_requires_interior():
    tp = Treeplex(3, [(1, 2, 0)])
    with pytest.raises(ValueError):
        dgf.dgf_gradient(tp, np.array([1.0, 1.0, 0.0]))


def test_prox_shift_identity():
    """PAPER.md:876 closed form on >= 1000 random interior points (Fig. 1, Kuhn, Leduc)."""
    tps = [fig1()[0], kuhn_X(), seqform.build(games.leduc()).X]
    rng = np.random.default_rng(2)
    n = 0
    for tp, count in zip(tps, (500, 450, 60)):
        cf = dgf.prox_shift_closed_form(tp)
        for _ in range(count):
            q = interior_point(tp, rng)
            direct = -dgf.dgf_value(tp, q) + dgf.dgf_gradient(tp, q) @ q
            assert abs(direct - cf) <= 1e-9 * max(1.0, abs(cf))
            n += 1
    assert n >= 1000
    assert math.isclose(dgf.prox_shift_closed_form(Treeplex(3, [(1, 2, 0)])), -2 * (math.log(2) - 1))
    assert math.isclose(dgf.prox_shift_closed_form(Treeplex(4, [(1, 3, 0)])), -2 * (math.log(3) - 1))


# ----------------------------------------------------------------- smoothed best response
def test_sbr_single_simplex_closed_form():
    tp = Treeplex(3, [(1, 2, 0)])
    q, v = dgf.smoothed_best_response(tp, np.array([0.0, 0.0, 0.0]), 1.0)
    assert np.allclose(q[1:], 0.5) and abs(v) < 1e-15
    q, v = dgf.smoothed_best_response(tp, np.array([0.0, -1.0, 0.0]), 1.0)
    e = math.exp(0.5)
    want = np.array([e, 1.0]) / (e + 1)             # qbar_i ~ exp(-g_i / beta), beta = 2
    assert np.allclose(q[1:], want, atol=1e-15)
    assert math.isclose(v, -want[0] + 2 * (want @ np.log(want) + math.log(2)), rel_tol=1e-14)


def _softmax_param(tp, theta):
    b = np.zeros(tp.n_seq)
    b[0] = 1
    for j in range(tp.n_simplex):
        s, n = tp.start[j], tp.size[j]
        t = theta[s:s + n] - theta[s:s + n].max()
        e = np.exp(t)
        b[s:s + n] = e / e.sum()
    return tp.behavioral_to_sequence(b)


def _generic_min(tp, obj, q0):
    """Generic optimiser over the treeplex (softmax logits, L-BFGS) - independent of
    the closed form."""
    theta0 = np.log(np.maximum(tp.sequence_to_behavioral(q0), 1e-300))
    res = minimize(lambda th: obj(_softmax_param(tp, th)), theta0, method="L-BFGS-B",
                   options={"maxiter": 20000, "ftol": 1e-15, "gtol": 1e-12})
    return _softmax_param(tp, res.x), res.fun


@pytest.mark.parametrize("seed", range(12))
def test_sbr_matches_generic_optimiser(seed):
    rng = np.random.default_rng(seed)
    tp = random_treeplex(rng, int(rng.integers(2, 7)))
    g = rng.standard_normal(tp.n_seq)
    mu = float(np.exp(rng.uniform(-1, 1)))
    q, v = dgf.smoothed_best_response(tp, g, mu)
    assert tp.check_feasible(q, 1e-12)
    # the value is the objective at the returned point
    assert math.isclose(v, q @ g + mu * dgf.dgf_value(tp, q), rel_tol=1e-10, abs_tol=1e-12)
    q2, v2 = _generic_min(tp, lambda p: p @ g + mu * dgf.dgf_value(tp, p), tp.uniform())
    assert v <= v2 + 1e-10
    assert abs(v - v2) <= 1e-6 * max(1.0, abs(v))
    assert np.abs(q - q2).max() <= 1e-4
    # no random feasible point does better
    for _ in range(50):
        p = interior_point(tp, rng)
        assert p @ g + mu * dgf.dgf_value(tp, p) >= v - 1e-12


def test_sbr_large_gradients_stable():
    tp = fig1()[0]
    g = np.zeros(tp.n_seq)
    g[1:] = 1e4 * np.random.default_rng(0).standard_normal(tp.n_seq - 1)
    q, v = dgf.smoothed_best_response(tp, g, 1e-3)
    assert np.isfinite(q).all() and np.isfinite(v) and tp.check_feasible(q, 1e-9)


def test_conjugate_sign():
    tp = Treeplex(3, [(1, 2, 0)])
    q = dgf.conjugate_gradient(tp, np.array([0.0, 1.0, 0.0]))
    e = math.exp(0.5)
    assert np.allclose(q[1:], [e / (e + 1), 1 / (e + 1)])


# ----------------------------------------------------------------- prox mapping
def _bregman(tp, q, qp):
    return dgf.dgf_value(tp, q) - dgf.dgf_value(tp, qp) - dgf.dgf_gradient(tp, qp) @ (q - qp)


def test_prox_zero_gradient_returns_centre():
    tp = fig1()[0]
    rng = np.random.default_rng(3)
    for _ in range(10):
        qp = interior_point(tp, rng)
        assert np.abs(dgf.prox_mapping(tp, np.zeros(tp.n_seq), qp) - qp).max() < 1e-12


def test_prox_single_simplex_at_uniform():
    """At the uniform centre the shift is constant on the simplex, so prox = SBR (mu = 1)."""
    tp = Treeplex(3, [(1, 2, 0)])
    q = dgf.prox_mapping(tp, np.array([0.0, -1.0, 0.0]), tp.uniform())
    e = math.exp(0.5)
    assert np.allclose(q[1:], [e / (e + 1), 1 / (e + 1)])


@pytest.mark.parametrize("seed", range(8))
def test_prox_matches_generic_optimiser(seed):
    rng = np.random.default_rng(100 + seed)
    tp = random_treeplex(rng, int(rng.integers(2, 6)))
    g = rng.standard_normal(tp.n_seq)
    qp = interior_point(tp, rng)
    q = dgf.prox_mapping(tp, g, qp)
    obj = lambda p: p @ g + _bregman(tp, p, qp)
    q2, v2 = _generic_min(tp, obj, qp)
    assert obj(q) <= v2 + 1e-9
    assert np.abs(q - q2).max() <= 1e-4
