"""Dilated entropy DGF, smoothed best response and prox mapping (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:448-537 (Section "Smoothed Best Responses") and the appendix
"Prox shift".  Vectors follow oracle/treeplex.py: entry 0 is
the empty sequence (value 1); a gradient's entry 0 carries the terms that do
not depend on the player's own sequences (leaves reached before the player's
first move), so after the bottom-up pass it holds the objective value.
"""
import math

import numpy as np


def d_simplex(xbar):
    """d_j(x) = sum_i x_i log x_i + log n, with 0 log 0 = 0."""
    xbar = np.asarray(xbar, dtype=float)
    nz = xbar > 0
    return float(np.sum(xbar[nz] * np.log(xbar[nz])) + math.log(len(xbar)))


def dgf_value(tp, q):
    """d(q) = sum_j beta_j q_{p_j} d_j(q^j / q_{p_j}).
    Simplexes with zero parent weight contribute 0."""
    total = 0.0
    for j in range(tp.n_simplex):
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        qp = q[p]
        if qp > 0:
            total += tp.beta[j] * qp * d_simplex(q[s:s + n] / qp)
    return total


def dgf_gradient(tp, q):
    """Appendix formula, for interior q:
    grad_{ji} d(q) = beta_j (log(q_i / q_{p_j}) + 1) + sum_{k in D_j^i} beta_k (log n_k - 1).
    Entry 0 (the empty sequence, not a variable) is 0."""
    q = np.asarray(q, dtype=float)
    if (q[1:] <= 0).any():
        raise ValueError("dgf_gradient requires an interior point (all q_i > 0)")
    g = np.zeros(tp.n_seq)
    for j in range(tp.n_simplex):
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        g[s:s + n] = tp.beta[j] * (np.log(q[s:s + n] / q[p]) + 1.0)
    for j in range(tp.n_simplex):
        p = tp.parent[j]
        if p != 0:
            g[p] += tp.beta[j] * (math.log(tp.size[j]) - 1.0)
    return g


def prox_shift_closed_form(tp):
    """-d(q) + <grad d(q), q> = -sum_{j: b_Q^j = 0} beta_j q_{p_j} (log n_j - 1)
    (PAPER.md:876), with q_{p_j} = 1 at root simplexes."""
    return -sum(tp.beta[j] * (math.log(tp.size[j]) - 1.0) for j in tp.roots)


def smoothed_best_response(tp, g, mu, behavioral=False):
    """argmin_{q in Q} <q, g> + mu d(q) and its value, by the paper's closed form.

    PAPER.md:467-512.  Bottom-up over the simplexes; at simplex j (after the
    values of the simplexes below have been added to g):
      qbar_i  proportional to  exp(-g_i / (mu beta_j))
    computed with the smallest g_i subtracted (overflow safety), then the value
      g_{i*} + mu beta_j log qbar_{i*} + mu beta_j log n,  i* = argmax qbar_i
     is added to the parent entry g_{p_j}.  mu scales every
    beta_j (mu d(q) in Eq. (4)).  Returns (q, value): q in
    sequence form, value = final g[0] = <q, g> + mu d(q) at the minimiser.

    behavioral=True also returns the behavioural strategy b (b^j = qbar^j at every
    simplex, also where the parent weight is 0) and its logarithm lb, in the closed form
    of PAPER.md:494: log qbar_i = -(g_i - min g) / w - log sum_k exp(-(g_k - min g) / w)
    (finite even where qbar_i underflows to 0; the prox centres of reading R16).
    An entry g_i = +inf (excluded from the support, see prox_mapping) gets qbar_i = 0.
    """
    G = np.array(g, dtype=float)
    b = np.zeros(tp.n_seq)
    b[0] = 1.0
    lb = np.zeros(tp.n_seq)
    for j in tp.bottom_up():
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        w = mu * tp.beta[j]
        Gj = G[s:s + n]
        t = -(Gj - Gj.min()) / w
        e = np.exp(t)
        S = e.sum()
        qbar = e / S
        i_star = int(np.argmax(qbar))
        G[p] += Gj[i_star] + w * math.log(qbar[i_star]) + w * math.log(n)
        b[s:s + n] = qbar
        lb[s:s + n] = t - math.log(S)
    q = tp.behavioral_to_sequence(b)
    if behavioral:
        return q, float(G[0]), b, lb
    return q, float(G[0])


def conjugate_gradient(tp, g, mu=1.0):
    """grad d*(g) = argmax_q <g, q> - mu d(q)."""
    q, _ = smoothed_best_response(tp, -np.asarray(g, dtype=float), mu)
    return q


def dgf_gradient_behavioral(tp, lb):
    """The appendix gradient of the point whose behavioural strategy has
    logarithm lb, with log(q_i / q_{p_j}) = log qbar_i = lb_i (reading R16):
      grad_{ji} d = beta_j (lb_i + 1) + sum_{k in D_j^i} beta_k (log n_k - 1).
    Defined at every point an SBR returns, including where qbar_i underflows or the parent
    weight q_{p_j} is 0.  lb_i = -inf (qbar_i = 0 exactly) gives -inf."""
    lb = np.asarray(lb, dtype=float)
    g = np.zeros(tp.n_seq)
    for j in range(tp.n_simplex):
        s, n = tp.start[j], tp.size[j]
        g[s:s + n] = tp.beta[j] * (lb[s:s + n] + 1.0)
    for j in range(tp.n_simplex):
        p = tp.parent[j]
        if p != 0:
            g[p] += tp.beta[j] * (math.log(tp.size[j]) - 1.0)
    return g


def prox_mapping(tp, g, q_prev=None, lb_prev=None):
    """argmin_{q in Q} <q, g> + D(q || q_prev), D the Bregman divergence of d
    (PAPER.md:514-528): solved as a smoothed best response (mu = 1) on the
    shifted gradient g - grad d(q_prev).

    The centre is given either in sequence form (q_prev, interior points only: the
    gradient takes log(q_i / q_{p_j}), the pitfall PAPER.md:529-537 names) or by its
    behavioural log-probabilities lb_prev (reading R16: the EGT prox centre is a smoothed
    best response, whose log qbar is known in closed form, so grad d is exact everywhere).
    An entry with qbar'_i = 0 (lb_prev_i = -inf) has an infinite shifted gradient and
    stays 0: the prox restricted to the centre's support, the limit PAPER.md:535-537
    describes ("setting bad actions too close to zero")."""
    if lb_prev is None:
        shifted = np.asarray(g, dtype=float) - dgf_gradient(tp, q_prev)
    else:
        shifted = np.asarray(g, dtype=float) - dgf_gradient_behavioral(tp, lb_prev)
    q, _ = smoothed_best_response(tp, shifted, 1.0)
    return q
