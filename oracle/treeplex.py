"""Treeplex (oracle side).  PAPER.md:374-421 (Section "Treeplexes").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Index convention (reading R1): a sequence-form vector has
``n_seq`` entries; entry 0 is the empty sequence, fixed to 1, playing the role
of the paper's convention "q_{p_j} = 1 if no branching operation precedes
Delta^j".  Every other entry belongs to exactly one simplex.

A simplex j is (start, n, parent): its index set I_j = [start, start+n)
(PAPER.md:406-407), p_j = parent.  Simplexes are listed in
top-down order (a simplex after the simplex owning its parent sequence).
"""
import math

import numpy as np


class Treeplex:
    def __init__(self, n_seq, simplexes, seq_labels=None):
        self.n_seq = int(n_seq)
        self.start = np.array([s[0] for s in simplexes], dtype=np.int64)
        self.size = np.array([s[1] for s in simplexes], dtype=np.int64)
        self.parent = np.array([s[2] for s in simplexes], dtype=np.int64)
        self.n_simplex = len(simplexes)
        self.seq_labels = seq_labels
        self._validate()
        self._derive()

    # ------------------------------------------------------------------ structure
    def _validate(self):
        owner = np.full(self.n_seq, -1, dtype=np.int64)
        for j in range(self.n_simplex):
            s, n = self.start[j], self.size[j]
            if n < 1:
                raise ValueError("simplex dimension must be >= 1")
            if (owner[s:s + n] != -1).any():
                raise ValueError("index sets overlap")
            owner[s:s + n] = j
        if owner[0] != -1:
            raise ValueError("entry 0 is the empty sequence, not a simplex entry")
        if (owner[1:] == -1).any():
            raise ValueError("index sets must partition 1..n_seq-1")
        for j in range(self.n_simplex):
            p = self.parent[j]
            if not (0 <= p < self.n_seq):
                raise ValueError("parent index out of range")
            if p != 0 and owner[p] >= j:
                raise ValueError("simplexes must be in top-down order (parent first); cycle?")
        self.owner = owner  # simplex owning each sequence (-1 for the empty sequence)

    def _derive(self):
        n_seq, J = self.n_seq, self.n_simplex
        # D_j^i: simplexes reached immediately after taking branch i
        self.children_of_seq = [[] for _ in range(n_seq)]
        for j in range(J):
            self.children_of_seq[self.parent[j]].append(j)
        self.roots = [j for j in range(J) if self.parent[j] == 0]
        # b_Q^j: number of branching operations preceding simplex j
        self.b = np.zeros(J, dtype=np.int64)
        for j in range(J):
            p = self.parent[j]
            self.b[j] = 0 if p == 0 else self.b[self.owner[p]] + 1
        # d_j: maximum depth below j counted in branching operations; leaves 0
        # (reading R2, consistent with Fig. 1's d_1 = 2, d_2 = 1, b^8 = 2)
        self.d = np.zeros(J, dtype=np.int64)
        # beta_j = 2 + sum_{k in D^j} 2 beta_k
        self.beta = np.zeros(J)
        # M: max l1 norm over Q: f(j) = 1 + max_i sum_{k in D_j^i} f(k)
        f = np.zeros(J)
        # Omega = max d - min d; d >= 0 with min 0 at the uniform centre, so
        # Omega(j) = beta_j log n_j + max_i sum_{k in D_j^i} Omega(k)
        om = np.zeros(J)
        for j in reversed(range(J)):
            s, n = self.start[j], self.size[j]
            kids = [k for i in range(s, s + n) for k in self.children_of_seq[i]]
            self.d[j] = 0 if not kids else 1 + max(self.d[k] for k in kids)
            self.beta[j] = 2.0 + sum(2.0 * self.beta[k] for k in kids)
            f[j] = 1.0 + max(sum(f[k] for k in self.children_of_seq[i]) for i in range(s, s + n))
            om[j] = self.beta[j] * math.log(n) + max(
                sum(om[k] for k in self.children_of_seq[i]) for i in range(s, s + n))
        self.M = float(sum(f[j] for j in self.roots))
        self.Omega = float(sum(om[j] for j in self.roots))
        self.phi = 1.0 / self.M  # strong convexity modulus of the dilated entropy
        self.depth = int(max(self.d)) if J else 0

    def top_down(self):
        return range(self.n_simplex)

    def bottom_up(self):
        return range(self.n_simplex - 1, -1, -1)

    # ------------------------------------------------------------------ vectors
    def uniform(self):
        """Uniform strategy at every simplex in sequence form (Gen-CFR line 1)."""
        return self.behavioral_to_sequence(self.uniform_behavioral())

    def uniform_behavioral(self):
        b = np.zeros(self.n_seq)
        b[0] = 1.0
        for j in range(self.n_simplex):
            s, n = self.start[j], self.size[j]
            b[s:s + n] = 1.0 / n
        return b

    def behavioral_to_sequence(self, b):
        """q_i = q_{p_j} * b_i top-down (each simplex scaled by its parent)."""
        q = np.zeros(self.n_seq)
        q[0] = 1.0
        for j in self.top_down():
            s, n = self.start[j], self.size[j]
            q[s:s + n] = q[self.parent[j]] * b[s:s + n]
        return q

    def sequence_to_behavioral(self, q):
        """b^j = q^j / q_{p_j}; uniform where q_{p_j} = 0 (reading R3)."""
        b = np.zeros(self.n_seq)
        b[0] = 1.0
        for j in range(self.n_simplex):
            s, n = self.start[j], self.size[j]
            qp = q[self.parent[j]]
            b[s:s + n] = q[s:s + n] / qp if qp > 0 else 1.0 / n
        return b

    def check_feasible(self, q, tol=1e-9):
        """q >= 0 and sum_{i in I_j} q_i = q_{p_j} for every simplex."""
        if abs(q[0] - 1.0) > tol or (q < -tol).any():
            return False
        for j in range(self.n_simplex):
            s, n = self.start[j], self.size[j]
            if abs(q[s:s + n].sum() - q[self.parent[j]]) > tol * max(1.0, abs(q[self.parent[j]])):
                return False
        return True
