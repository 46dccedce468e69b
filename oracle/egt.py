"""Excessive Gap Technique with the dilated entropy DGF (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:280-372 (EGT, Algorithms 1-2) and PAPER.md:541-611 (practical EGT:
mu balancing, EGT/as with aggressive mu reduction, Algorithms 3-4).

Player x minimises <x, A y>, player y maximises it.  Smoothed functions
(PAPER.md:286-287):
  f_{mu_y}(x)  = max_y <x, A y> - mu_y d_Y(y)
  phi_{mu_x}(y) = min_x <x, A y> + mu_x d_X(x)
with smoothed best responses y_{mu_y}(x), x_{mu_x}(y).  A step focused on y is
the x step applied to the mirrored problem min_y max_x <y, (-A^T) x>
(reading R5), so one ``_step`` serves both players.
"""
import math

import numpy as np

from .dgf import smoothed_best_response, prox_mapping


class Counter:
    def __init__(self):
        self.n = 0


class Problem:
    """The two mirrored views of the BSPP: view 0 = x minimises <x, A y>;
    view 1 = y minimises <y, -A^T x>."""

    def __init__(self, sf):
        self.sf = sf
        self.tp = (sf.X, sf.Y)
        self.grads = Counter()

    def grad(self, v, other):
        """Gradient of the view-v player's objective at the other player's point."""
        self.grads.n += 1
        return self.sf.Ay(other) if v == 0 else -self.sf.ATx(other)

    def sbr(self, v, other, mu, behavioral=False):
        """(response, value) = argmin/min over own treeplex of <q, grad> + mu d(q)
        (behavioral=True: also its behavioural strategy and log, see dgf)."""
        return smoothed_best_response(self.tp[v], self.grad(v, other), mu, behavioral)


def smoothed_f(prob, x, mu_y):
    """f_{mu_y}(x) and y_{mu_y}(x)."""
    y, val = prob.sbr(1, x, mu_y)
    return -val, y


def smoothed_phi(prob, y, mu_x):
    """phi_{mu_x}(y) and x_{mu_x}(y)."""
    x, val = prob.sbr(0, y, mu_x)
    return val, x


def excessive_gap(prob, x, y, mu_x, mu_y):
    """EGV(x, y) = phi_{mu_x}(y) - f_{mu_y}(x)."""
    return smoothed_phi(prob, y, mu_x)[0] - smoothed_f(prob, x, mu_y)[0]


def theory_mu(sf):
    """mu_x = mu_y = ||A|| / sqrt(phi_X phi_Y): the symmetric solution of
    mu_x = phi_X / L_1(f_{mu_y}), L_1 = ||A||^2 / (phi_Y mu_y)."""
    return sf.max_abs_A() / math.sqrt(sf.X.phi * sf.Y.phi)


def practical_mu(sf, kmax=30):
    """Reading R14, "practically-tuned initial choice for the initial smoothing parameters"
    (PAPER.md:545-547): mu_x = mu_y = theory_mu * 2^-k where k is the last of 0, 1, ..., kmax
    before the excessive gap condition at the initial point (Alg. 1 / Alg. 3 lines 1-2,
    PAPER.md:576-578) first fails -- a plain scan, every k evaluated until the first failure.
    Returns (k, mu)."""
    mu_th = theory_mu(sf)
    prob = Problem(sf)
    k_ok = 0
    for k in range(kmax + 1):
        mu = mu_th * 2.0 ** -k
        x0, y0 = initialize(prob, mu, mu)
        if excessive_gap(prob, x0, y0, mu, mu) < 0:
            break
        k_ok = k
    return k_ok, mu_th * 2.0 ** -k_ok


def initialize(prob, mu_x, mu_y):
    """Algorithm 1 lines 1-2, reading R4:
    x_omega = the DGF centre (uniform behavioural strategy, d = 0);
    y^0 = y_{mu_y}(x_omega);
    x^0 = grad d_X^*(-mu_x^{-1} grad f_{mu_y}(x_omega)), grad f(x_omega) = A y^0
        = argmin_x <x, A y^0> + mu_x d_X(x) = x_{mu_x}(y^0)."""
    x_omega = prob.tp[0].uniform()
    _, y0 = smoothed_f(prob, x_omega, mu_y)
    _, x0 = smoothed_phi(prob, y0, mu_x)
    return x0, y0


def _step(prob, v, mu, mu_other, p, o, tau):
    """Algorithm 2 for the view-v player (own point p, other o):
      p_hat  = (1 - tau) p + tau p_mu(o)
      o_plus = (1 - tau) o + tau o_mu(p_hat)
      p_til  = grad d^*(grad d(p_mu(o)) - tau / ((1 - tau) mu) grad f(p_hat))
             = prox at centre p_mu(o) of the gradient  s * grad f(p_hat),  s = tau / ((1 - tau) mu)
      p_plus = (1 - tau) p + tau p_til
      mu_plus = (1 - tau) mu
    grad f(p_hat) = (view-v gradient at o_mu(p_hat)).  The prox centre p_mu(o) enters
    through its behavioural log-probabilities (reading R16)."""
    w = 1 - v
    p_mu, _, _, p_mu_lb = prob.sbr(v, o, mu, behavioral=True)
    p_hat = (1 - tau) * p + tau * p_mu
    o_mu_hat, _ = prob.sbr(w, p_hat, mu_other)
    o_plus = (1 - tau) * o + tau * o_mu_hat
    grad_f = prob.grad(v, o_mu_hat)
    s = tau / ((1 - tau) * mu)
    p_til = prox_mapping(prob.tp[v], s * grad_f, lb_prev=p_mu_lb)
    p_plus = (1 - tau) * p + tau * p_til
    return (1 - tau) * mu, p_plus, o_plus


class EGTState:
    def __init__(self, x, y, mu_x, mu_y, tau=0.5):
        self.x, self.y = x, y
        self.mu_x, self.mu_y = mu_x, mu_y
        self.tau = tau
        self.t = 0
        self.backtracks = 0


def step_xy(prob, st, focus, tau):
    """Step focused on 'x' or 'y'; returns the candidate (mu_x, mu_y, x, y)."""
    if focus == "x":
        mu_x, x, y = _step(prob, 0, st.mu_x, st.mu_y, st.x, st.y, tau)
        return mu_x, st.mu_y, x, y
    mu_y, y, x = _step(prob, 1, st.mu_y, st.mu_x, st.y, st.x, tau)
    return st.mu_x, mu_y, x, y


def egt_iteration(prob, st, variant):
    """One iteration of EGT (theory, Algorithm 1), EGT with mu balancing
     or EGT/as (Algorithms 3-4)."""
    if variant == "theory":
        focus = "x" if st.t % 2 == 0 else "y"           # Alg. 1 lines 6-9
        tau = 2.0 / (st.t + 3)                           # Alg. 1 line 5
        st.mu_x, st.mu_y, st.x, st.y = step_xy(prob, st, focus, tau)
    elif variant == "balanced":
        focus = "x" if st.mu_x > st.mu_y else "y"
        tau = 2.0 / (st.t + 3)                           # reading R6
        st.mu_x, st.mu_y, st.x, st.y = step_xy(prob, st, focus, tau)
    elif variant == "as":
        focus = "x" if st.mu_x > st.mu_y else "y"        # Alg. 3 lines 6-10
        while True:                                      # Alg. 4 (Decr), reading R8
            mu_x, mu_y, x, y = step_xy(prob, st, focus, st.tau)
            if excessive_gap(prob, x, y, mu_x, mu_y) >= 0:
                break
            st.tau *= 0.5
            st.backtracks += 1
            if st.tau < 1e-12:
                raise RuntimeError("EGT/as: tau underflow")
        st.mu_x, st.mu_y, st.x, st.y = mu_x, mu_y, x, y
    else:
        raise ValueError(variant)
    st.t += 1
    return st


def run(sf, variant, iters, mu=None, record=None):
    prob = Problem(sf)
    if mu is None:
        mu = theory_mu(sf)
    elif isinstance(mu, str) and mu == "practical":
        mu = practical_mu(sf)[1]
    mu_x, mu_y = (mu, mu) if np.isscalar(mu) else mu
    x, y = initialize(prob, mu_x, mu_y)
    st = EGTState(x, y, mu_x, mu_y)
    for _ in range(iters):
        egt_iteration(prob, st, variant)
        if record is not None:
            record(st, prob)
    return st, prob
