"""Pins for the parts of oracle/cfr.py that a floating-point run cannot pin by itself.

* Reading R15: RM / RM+ switch to the uniform strategy "if r^t = 0"
  (PAPER.md:64, 85).  The oracle decides that in fp64 with a noise threshold (SNAP, and the
  per-hand scale M_h of ``hand_scales``).  The reference here is the same Gen-CFR run in
  exact rational arithmetic (``fractions.Fraction``), written out below from PAPER.md:21-45,
  55-69, 76-90, 92-95 -- on games built so that the exact regrets are 0 while fp64 leaves
  rounding noise, the snapped oracle must equal the exact run and the unsnapped one must not.
* Alternating updates (Gen-CFR line 35): y^t responds to x^t, not
  x^{t-1}; a hand-computed one-iteration example where the two differ.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

from oracle import cfr, games, seqform
from oracle.games import Chance, Decision, Terminal


# ----------------------------------------------------------------- exact Gen-CFR
def _exact_A(sf):
    """The game's payoff matrix in exact rationals (entries are multiples of 1/60 here;
    fp64 accumulation noise ~1e-17 is removed by limit_denominator)."""
    return [[Fr(v).limit_denominator(10 ** 4) for v in row] for row in sf.A.toarray()]


def _seq(tp, b):
    q = [Fr(0)] * tp.n_seq
    q[0] = Fr(1)
    for j in range(tp.n_simplex):
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        for i in range(s, s + n):
            q[i] = q[p] * b[i]
    return q


def _uniform(tp):
    b = [Fr(0)] * tp.n_seq
    b[0] = Fr(1)
    for j in range(tp.n_simplex):
        s, n = tp.start[j], tp.size[j]
        for i in range(s, s + n):
            b[i] = Fr(1, int(n))
    return b


def _exact_pass(tp, g, z, r, kind):
    """Gen-CFR lines 30-33: bottom-up, g_{p_j} += <g^j, z^{j,t-1}>, then R(g^j): RM line 63-64
    or RM+ line 84-85 with the literal "if r^t = 0 use uniform" (no positive part left)."""
    g, z, r = list(g), list(z), list(r)
    for j in reversed(range(tp.n_simplex)):
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        gj = g[s:s + n]
        v = sum(a * b for a, b in zip(gj, z[s:s + n]))
        g[p] += v
        rn = [r[s + i] + gj[i] - v for i in range(n)]
        if kind == "rmp":
            rn = [max(x, Fr(0)) for x in rn]
        pos = [max(x, Fr(0)) for x in rn]
        tot = sum(pos)
        r[s:s + n] = rn
        z[s:s + n] = [x / tot for x in pos] if tot > 0 else [Fr(1, int(n))] * n
    return z, r


def exact_run(sf, variant, T):
    kind, scheme = cfr.VARIANTS[variant]
    A = _exact_A(sf)
    X, Y = sf.X, sf.Y
    nx, ny = X.n_seq, Y.n_seq
    zx, zy = _uniform(X), _uniform(Y)
    rx, ry = [Fr(0)] * nx, [Fr(0)] * ny
    xb, yb = [Fr(0)] * nx, [Fr(0)] * ny
    y = _seq(Y, zy)
    for t in range(1, T + 1):
        g = [-sum(A[i][k] * y[k] for k in range(ny)) for i in range(nx)]        # line 29
        zx, rx = _exact_pass(X, g, zx, rx, kind)
        x = _seq(X, zx)
        a = Fr(1, t) if scheme == "uniform" else Fr(2 * t, t * t + t)
        xb = [a * x[i] + (1 - a) * xb[i] for i in range(nx)]                    # line 34
        g = [sum(A[k][i] * x[k] for k in range(nx)) for i in range(ny)]         # line 35
        zy, ry = _exact_pass(Y, g, zy, ry, kind)
        y = _seq(Y, zy)
        yb = [a * y[i] + (1 - a) * yb[i] for i in range(ny)]                    # line 41 (R9)
    f = lambda v: np.array([float(e) for e in v])  # noqa: E731
    return f(zx), f(zy), f(xb), f(yb)


def _close(st, ex, tol=1e-15):
    zx, zy, xb, yb = ex
    return all(np.abs(a - b).max() <= tol for a, b in ((st.zx, zx), (st.zy, zy), (st.xbar, xb), (st.ybar, yb)))


# ----------------------------------------------------------------- games with exact zero regrets
def tied_gains_game():
    """Player 2 picks one of three columns without seeing a fair coin; per coin side the
    columns pay player 2 (0.1, 0.5), (0.2, 0.4), (0.3, 0.3): every column's expected payoff is
    exactly 3/10, so every regret is exactly 0 and RM stays uniform; fp64 accumulates the
    three gains with different rounding."""
    cols = ((0.1, 0.5), (0.2, 0.4), (0.3, 0.3))
    outs = []
    for side in range(2):
        y = Decision(1, "", "", [("a%d" % i, Terminal(-c[side])) for i, c in enumerate(cols)])
        outs.append((0.5, y))
    return seqform.build(Decision(0, "", "", [("x", Chance(outs))]))


def cancelling_subtree_game():
    """Player 1 chooses L or R; after L (never chosen: R is strictly better) a second
    decision {a, b} whose gains are the coin average of (0.1, 0.2, -0.3) for a and 0 for b --
    exactly 0 for both, while fp64 leaves ~1e-17 on a, far below the rounding noise of the
    same hand's other gains (R's are O(1)), the scale M_h of reading R15."""
    outs = []
    for v in (0.1, 0.2, -0.3):
        dL = Decision(0, "", "L", [("a", Terminal(v)), ("b", Terminal(0.0))])
        dR = Decision(1, "", "R", [("c", Terminal(1.0)), ("d", Terminal(0.5))])
        outs.append((1.0 / 3.0, Decision(0, "", "", [("L", dL), ("R", dR)])))
    return seqform.build(Chance(outs))


@pytest.mark.parametrize("variant", ["cfr_rm", "cfr_rmp", "cfr_plus"])
def test_snap_reproduces_exact_arithmetic(variant):
    sf = tied_gains_game()
    ex = exact_run(sf, variant, 6)
    assert np.allclose(ex[1][1:], 1.0 / 3.0)      # exact: every regret 0 -> uniform
    assert _close(cfr.run(sf, variant, 6), ex)
    old = cfr.SNAP
    try:
        cfr.SNAP = 0.0                            # the literal fp64 "r = 0" test decides on noise
        assert not _close(cfr.run(sf, variant, 6), ex)
    finally:
        cfr.SNAP = old


@pytest.mark.parametrize("variant", ["cfr_rm", "cfr_rmp", "cfr_plus"])
def test_hand_scale_reproduces_exact_arithmetic(variant):
    sf = cancelling_subtree_game()
    ex = exact_run(sf, variant, 6)
    assert np.allclose(ex[0][3:], 0.5)            # the L/a, L/b simplex stays uniform
    assert _close(cfr.run(sf, variant, 6), ex)
    old = cfr.hand_scales
    try:
        cfr.hand_scales = lambda labels, g: np.zeros(len(g))  # noqa: E731  (M_h dropped)
        assert not _close(cfr.run(sf, variant, 6), ex)
    finally:
        cfr.hand_scales = old


@pytest.mark.parametrize("variant", ["cfr_rm", "cfr_rmp", "cfr_plus"])
def test_kuhn_first_iterations_exact(variant):
    sf = seqform.build(games.kuhn())
    assert _close(cfr.run(sf, variant, 8), exact_run(sf, variant, 8), tol=1e-14)


@pytest.mark.parametrize("name,T", [("kuhn", 300), ("leduc", 25)])
def test_noise_threshold_inert_on_kuhn_and_leduc(name, T):
    """Where no regret is 0 up to rounding, the threshold changes nothing: trajectories with
    SNAP = 0 and without M_h are bit-identical to the oracle's."""
    sf = seqform.build(games.kuhn() if name == "kuhn" else games.leduc())
    old_snap, old_hs = cfr.SNAP, cfr.hand_scales
    for variant in ("cfr_rm", "cfr_rmp", "cfr_plus"):
        ref = cfr.run(sf, variant, T)
        try:
            cfr.SNAP = 0.0
            cfr.hand_scales = lambda labels, g: np.zeros(len(g))  # noqa: E731
            alt = cfr.run(sf, variant, T)
        finally:
            cfr.SNAP, cfr.hand_scales = old_snap, old_hs
        for a, b in ((ref.xbar, alt.xbar), (ref.ybar, alt.ybar), (ref.zx, alt.zx), (ref.zy, alt.zy)):
            assert np.array_equal(a, b)


# ----------------------------------------------------------------- alternating updates
def test_alternating_updates_hand_example():
    """A = [[1, 0], [0, 0]] (payoff to player 2; x minimises <x, A y>), x^0 = y^0 = (1/2, 1/2).
    Iteration 1 by hand (RM):
      x: g = -A y^0 = (-1/2, 0), <z, g> = -1/4, r = (-1/4, 1/4) -> x^1 = (0, 1)
      y (alternating, Gen-CFR line 35: g = A^T x^1) : g = (0, 0), r = (0, 0) -> y^1 = (1/2, 1/2)
      y (simultaneous, g = A^T x^0 = (1/2, 0)): r = (1/4, -1/4) -> y^1 = (1, 0)."""
    sf = seqform.build(games.matrix_game([[-1.0, 0.0], [0.0, 0.0]]))
    assert np.array_equal(sf.A.toarray()[1:, 1:], [[1.0, 0.0], [0.0, 0.0]])
    st = cfr.CFRState(sf, "cfr_rm")
    cfr.cfr_iteration(st)
    assert np.array_equal(st.zx[1:], [0.0, 1.0])
    assert np.array_equal(st.zy[1:], [0.5, 0.5])      # not (1, 0): y^1 answers x^1
    assert np.array_equal(st.xbar[1:], [0.0, 1.0]) and np.array_equal(st.ybar[1:], [0.5, 0.5])
