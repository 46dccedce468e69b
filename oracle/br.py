"""Best responses and the saddle-point residual (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:308-312: eps_sad(x, y) = max_{y'} x^T A y' - min_{x'} x'^T A y, the sum
of the players' regrets.  A best response over a treeplex is the bottom-up
dynamic programme (best action per simplex after adding the values of the
simplexes below, the mu -> 0 limit of the smoothed best response,
PAPER.md:497-500).
"""
import numpy as np


def best_response(tp, g, sense):
    """Optimum of <q, g> over Q for sense 'min' or 'max': (value, pure q).
    Ties go to the lowest action index."""
    G = np.array(g, dtype=float)
    b = np.zeros(tp.n_seq)
    b[0] = 1.0
    for j in tp.bottom_up():
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        Gj = G[s:s + n]
        i = int(np.argmin(Gj) if sense == "min" else np.argmax(Gj))
        G[p] += Gj[i]
        b[s + i] = 1.0
    return float(G[0]), tp.behavioral_to_sequence(b)


def saddle_gap(sf, x, y):
    """eps_sad(x, y) = max_y' <x, A y'> - min_x' <x', A y>."""
    vy, _ = best_response(sf.Y, sf.ATx(x), "max")
    vx, _ = best_response(sf.X, sf.Ay(y), "min")
    return vy - vx


def brute_force_best_response(tp, g, sense):
    """Enumerate every pure strategy (vertex of Q) -- tiny treeplexes only."""
    best = None
    choices = []

    def rec(j_list, b):
        nonlocal best
        if not j_list:
            q = tp.behavioral_to_sequence(b)
            v = float(q @ g)
            if best is None or (v < best if sense == "min" else v > best):
                best = v
            return
        j, rest = j_list[0], j_list[1:]
        s, n = tp.start[j], tp.size[j]
        for i in range(n):
            b2 = b.copy()
            b2[s:s + n] = 0.0
            b2[s + i] = 1.0
            rec(rest, b2)

    b0 = tp.uniform_behavioral()
    rec(list(range(tp.n_simplex)), b0)
    del choices
    return best
