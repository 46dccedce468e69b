"""Sequence form of a literal extensive-form game (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:151-158 / 247-253: the Nash equilibrium of a two-player zero-sum
perfect-recall EFG solves min_{x in X} max_{y in Y} <x, A y> where X, Y are the
players' sequence-form treeplexes and A the sequence-form payoff matrix.  Here
x is player 1 (minimises), y is player 2, and A[i, j] = sum over leaves z whose
player-1 sequence is i and player-2 sequence is j of chance(z) * payoff to
player 2 at z.  Index 0 of each vector is the empty sequence (R1), so
leaves reached before a player's first move contribute to row/column 0 (the
paper's a_1, a_2 linear terms).
"""
import numpy as np
import scipy.sparse as sp

from .games import Chance, Decision, Terminal
from .treeplex import Treeplex


class SeqForm:
    def __init__(self, X, Y, A, labels_x, labels_y, big_blind=None):
        self.X, self.Y, self.A = X, Y, A
        self.labels_x, self.labels_y = labels_x, labels_y
        self.big_blind = big_blind

    def Ay(self, y):
        return self.A @ y

    def ATx(self, x):
        return self.A.T @ x

    def max_abs_A(self):
        """||A|| read as max |A_ij| (R7)."""
        return float(np.abs(self.A.data).max()) if self.A.nnz else 0.0


def build(root, big_blind=None):
    """Enumerate the tree once: create a simplex per information set (checking
    perfect recall), and accumulate A over the leaves."""
    simplexes = [[], []]        # per player: list of [start, n, parent]
    labels = [["∅"], ["∅"]]
    infoset_id = [{}, {}]       # key -> (simplex id, first seq)
    n_seq = [1, 1]
    entries = {}

    def seq_block(p, node, cur_seq):
        key = (node.hand, node.history)
        if key in infoset_id[p]:
            j, first = infoset_id[p][key]
            if simplexes[p][j][2] != cur_seq:
                raise ValueError("imperfect recall: infoset reached from two parent sequences")
            if simplexes[p][j][1] != len(node.actions):
                raise ValueError("inconsistent action counts within an information set")
            return first
        first = n_seq[p]
        infoset_id[p][key] = (len(simplexes[p]), first)
        simplexes[p].append([first, len(node.actions), cur_seq])
        n_seq[p] += len(node.actions)
        for tok, _ in node.actions:
            h = tok if not node.history else node.history + "/" + tok
            labels[p].append(node.hand + "|" + h)
        return first

    stack = [(root, 0, 0, 1.0)]
    while stack:
        node, s1, s2, reach = stack.pop()
        if isinstance(node, Terminal):
            if reach != 0.0:
                entries[(s1, s2)] = entries.get((s1, s2), 0.0) + reach * (-node.payoff1)
        elif isinstance(node, Chance):
            for p, ch in reversed(node.outcomes):
                stack.append((ch, s1, s2, reach * p))
        else:
            p = node.player
            first = seq_block(p, node, s1 if p == 0 else s2)
            for i in reversed(range(len(node.actions))):
                ch = node.actions[i][1]
                if p == 0:
                    stack.append((ch, first + i, s2, reach))
                else:
                    stack.append((ch, s1, first + i, reach))

    # DFS creates simplexes parent-first: top-down order holds
    X = Treeplex(n_seq[0], [tuple(s) for s in simplexes[0]], labels[0])
    Y = Treeplex(n_seq[1], [tuple(s) for s in simplexes[1]], labels[1])
    if entries:
        keys = list(entries)
        A = sp.coo_matrix(([entries[k] for k in keys], ([k[0] for k in keys], [k[1] for k in keys])),
                          shape=(n_seq[0], n_seq[1])).tocsr()
    else:
        A = sp.csr_matrix((n_seq[0], n_seq[1]))
    return SeqForm(X, Y, A, labels[0], labels[1], big_blind)
