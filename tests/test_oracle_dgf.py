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


# ----------------------------------------------------------------- prox at boundary centres
# The EGT prox centre is a smoothed best response (Alg. 2 line 3); the oracle
# takes it by its behavioural log-probabilities (reading R16), which stay finite where the
# behavioural probabilities underflow -- the bench's operating point.  The pins below check
# that form against an independent statement of the same problem: the Bregman divergence of
# the dilated entropy written per simplex, D(q || q') = sum_j beta_j q_{p_j} KL(qbar^j || qbar'^j)
# (itself pinned against d(q) - d(q') - <grad d(q'), q - q'> at interior points), minimised by a
# generic optimiser over the centre's support.
def _kl_form(tp, q, lb_c):
    """sum_j beta_j q_{p_j} sum_{i: qbar_i > 0} qbar_i (log qbar_i - lb_c_i)."""
    tot = 0.0
    for j in range(tp.n_simplex):
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        if q[p] <= 0:
            continue
        qb = q[s:s + n] / q[p]
        nz = qb > 0
        tot += tp.beta[j] * q[p] * float(np.sum(qb[nz] * (np.log(qb[nz]) - lb_c[s:s + n][nz])))
    return tot


def _support_min(tp, obj, support, rng):
    """Generic optimiser over the face {qbar_i = 0 off the support}: softmax logits on the
    support only, L-BFGS from a random start (independent of the closed form)."""
    idx = np.flatnonzero(support)

    def point(theta):
        b = tp.uniform_behavioral()
        full = np.full(tp.n_seq, -np.inf)
        full[idx] = theta
        for j in range(tp.n_simplex):
            s, n = tp.start[j], tp.size[j]
            t = full[s:s + n]
            e = np.exp(t - t.max())
            b[s:s + n] = e / e.sum()
        return tp.behavioral_to_sequence(b)

    res = minimize(lambda th: obj(point(th)), 0.1 * rng.standard_normal(len(idx)), method="L-BFGS-B",
                   options={"maxiter": 50000, "ftol": 1e-15, "gtol": 1e-12})
    return point(res.x), res.fun


def _random_log_centre(tp, rng, spread=2.0, drop=0.0, far=0.0):
    """Behavioural log-probabilities: random softmax per simplex; with `drop`, entries
    excluded (-inf, never a whole simplex); with `far`, entries pushed to log qbar ~ -800
    (qbar underflows to 0 in fp64 while log qbar stays finite)."""
    lb = np.zeros(tp.n_seq)
    for j in range(tp.n_simplex):
        s, n = tp.start[j], tp.size[j]
        t = spread * rng.standard_normal(n)
        if n > 1:
            for i in range(n):
                if i != int(np.argmax(t)):
                    if rng.random() < drop:
                        t[i] = -np.inf
                    elif rng.random() < far:
                        t[i] = -800.0 + t[i]
        m = t.max()
        lb[s:s + n] = t - (m + math.log(np.exp(t - m).sum()))
    return lb


def test_kl_form_is_the_bregman_divergence():
    rng = np.random.default_rng(41)
    for _ in range(10):
        tp = random_treeplex(rng, int(rng.integers(2, 7)))
        qc = interior_point(tp, rng)
        lb_c = np.log(np.maximum(tp.sequence_to_behavioral(qc), 1e-300))
        q = interior_point(tp, rng)
        assert math.isclose(_kl_form(tp, q, lb_c), _bregman(tp, q, qc), rel_tol=1e-9, abs_tol=1e-12)


def test_prox_log_centre_equals_sequence_centre_in_the_interior():
    rng = np.random.default_rng(42)
    for _ in range(10):
        tp = random_treeplex(rng, int(rng.integers(2, 7)))
        qc = interior_point(tp, rng)
        lb_c = np.log(tp.sequence_to_behavioral(qc))
        g = rng.standard_normal(tp.n_seq)
        a = dgf.prox_mapping(tp, g, qc)
        b = dgf.prox_mapping(tp, g, lb_prev=lb_c)
        assert np.abs(a - b).max() <= 1e-12


def test_prox_log_centre_single_simplex_closed_form():
    """One simplex (beta = 2): qbar_i ~ qbar'_i exp(-g_i / beta) = exp(lb_i - g_i / 2); the
    -800 entry is exp(-800) ~ 0 relative to the others, written out by hand."""
    tp = Treeplex(4, [(1, 3, 0)])
    lb_c = np.array([0.0, math.log(0.25), math.log(0.75), -800.0])
    g = np.array([0.0, 1.0, -0.5, -1500.0])
    q = dgf.prox_mapping(tp, g, lb_prev=lb_c)
    e = np.array([0.25 * math.exp(-0.5), 0.75 * math.exp(0.25), math.exp(-800.0 + 750.0)])
    assert np.allclose(q[1:], e / e.sum(), rtol=1e-13, atol=0)


@pytest.mark.parametrize("seed", range(8))
def test_prox_on_the_support_matches_generic_optimiser(seed):
    """Centres with excluded entries (qbar' = 0 exactly): the oracle's prox keeps them at 0
    and minimises <q, g> + D(q || q') over the rest."""
    rng = np.random.default_rng(300 + seed)
    tp = random_treeplex(rng, int(rng.integers(3, 7)))
    lb_c = _random_log_centre(tp, rng, drop=0.4)
    g = rng.standard_normal(tp.n_seq)
    q = dgf.prox_mapping(tp, g, lb_prev=lb_c)
    assert tp.check_feasible(q, 1e-12)
    assert np.all(q[1:][np.isneginf(lb_c[1:])] == 0.0)
    obj = lambda p: p @ g + _kl_form(tp, p, lb_c)  # noqa: E731
    q2, v2 = _support_min(tp, obj, ~np.isneginf(lb_c) & (np.arange(tp.n_seq) > 0), rng)
    assert obj(q) <= v2 + 1e-9
    assert np.abs(q - q2).max() <= 1e-4


@pytest.mark.parametrize("seed", range(6))
def test_prox_at_underflowing_centres_matches_generic_optimiser(seed):
    """Centres whose behavioural probabilities underflow (log qbar' ~ -800, qbar' = 0 in fp64)
    while the gradient pulls toward them (g ~ -1500 there): the log form keeps the exact
    Bregman geometry, and the optimiser over the full face agrees."""
    rng = np.random.default_rng(400 + seed)
    tp = random_treeplex(rng, int(rng.integers(3, 6)))
    lb_c = _random_log_centre(tp, rng, far=0.5)
    g = rng.standard_normal(tp.n_seq)
    far = lb_c < -500
    g[far] = -1500.0 - 50.0 * rng.random(int(far.sum()))  # -g/beta competes with lb there
    q = dgf.prox_mapping(tp, g, lb_prev=lb_c)
    assert tp.check_feasible(q, 1e-12) and np.isfinite(q).all()
    obj = lambda p: p @ g + _kl_form(tp, p, lb_c)  # noqa: E731
    q2, v2 = _support_min(tp, obj, np.arange(tp.n_seq) > 0, rng)
    assert obj(q) <= v2 + 1e-8 * max(1.0, abs(v2))
    assert np.abs(q - q2).max() <= 1e-4


def test_prox_excluded_entry_is_the_limit_of_vanishing_centres():
    rng = np.random.default_rng(7)
    tp = random_treeplex(rng, 5)
    lb_c = _random_log_centre(tp, rng, drop=0.5)
    g = rng.standard_normal(tp.n_seq)
    q_inf = dgf.prox_mapping(tp, g, lb_prev=lb_c)
    lb_far = np.where(np.isneginf(lb_c), -1e4, lb_c)
    q_far = dgf.prox_mapping(tp, g, lb_prev=lb_far)
    assert np.abs(q_inf - q_far).max() <= 1e-300 + 1e-15


def test_sbr_log_behavioural_closed_form():
    """log qbar from the SBR equals log of its qbar where that is representable, and stays
    finite (and exact in the closed form) where qbar underflows."""
    tp = Treeplex(4, [(1, 3, 0)])
    g = np.array([0.0, 0.0, 2.0, 3000.0])
    q, v, b, lb = dgf.smoothed_best_response(tp, g, 1.0, behavioral=True)
    # w = beta = 2: t = -(g - 0) / 2 = (0, -1, -1500); S = 1 + e^-1 (+ e^-1500 = 0)
    S = 1.0 + math.exp(-1.0)
    assert np.allclose(lb[1:], [-math.log(S), -1.0 - math.log(S), -1500.0 - math.log(S)], rtol=1e-15, atol=0)
    assert b[3] == 0.0 and np.allclose(np.exp(lb[1:3]), b[1:3], rtol=1e-15)
