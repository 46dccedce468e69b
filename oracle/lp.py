"""Sequence-form linear program for the game value (oracle side; a pin, not the method).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The value of min_{x in X} max_{y in Y} <x, A y> by the
classical LP ("taking the dual of the optimization problem
faced by one player ... and injecting the primal x-player constraints"):
for fixed x, max_y <A^T x, y> s.t. F y = f, y >= 0 has dual min_v f^T v s.t.
F^T v >= A^T x; so  min_{x, v} f^T v  s.t.  F^T v - A^T x >= 0,  E x = e,  x >= 0.
E/F are the treeplex constraints: entry 0 = 1, and for every simplex j
sum_{i in I_j} q_i - q_{p_j} = 0.
"""
import numpy as np
import scipy.sparse as sp
from scipy.optimize import linprog


def constraint_matrix(tp):
    rows, cols, vals = [0], [0], [1.0]
    for j in range(tp.n_simplex):
        r = j + 1
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        rows += [r] * n + [r]
        cols += list(range(s, s + n)) + [p]
        vals += [1.0] * n + [-1.0]
    E = sp.coo_matrix((vals, (rows, cols)), shape=(tp.n_simplex + 1, tp.n_seq)).tocsr()
    e = np.zeros(tp.n_simplex + 1)
    e[0] = 1.0
    return E, e


def game_value(sf):
    E, e = constraint_matrix(sf.X)
    F, f = constraint_matrix(sf.Y)
    nx, nv = sf.X.n_seq, F.shape[0]
    c = np.concatenate([np.zeros(nx), f])
    # A^T x - F^T v <= 0
    A_ub = sp.hstack([sf.A.T, -F.T]).tocsr()
    b_ub = np.zeros(sf.Y.n_seq)
    A_eq = sp.hstack([E, sp.csr_matrix((E.shape[0], nv))]).tocsr()
    bounds = [(0, None)] * nx + [(None, None)] * nv
    res = linprog(c, A_ub=A_ub, b_ub=b_ub, A_eq=A_eq, b_eq=e, bounds=bounds, method="highs")
    if res.status != 0:
        raise RuntimeError(res.message)
    return res.fun, res.x[:nx]
