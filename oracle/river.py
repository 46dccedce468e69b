"""River endgame (oracle side): betting rules and a hand-vectorised sequence form.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Betting rules: PAPER.md:670-688.  Chance deals each player a private 2-card
hand; player 1 (x, "Libratus") moves first and may fold, check or bet
multipliers of the pot; the game ends on a fold, a call, or check-check; the
better hand wins a showdown and ties split.  Readings (R10-R13):

* bet-size context by (player, number of bets/raises so far in the street n):
  P1: n=0 P1_OPEN, n=1 P1_VS_BET ("checks and the other player bets"),
      n=2 P1_VS_RAISE ("bets and the other player raises"), n>=3 P1_SUBSEQ;
  P2: n=0 P2_VS_CHECK, n=1 P2_VS_BET, n>=2 P2_SUBSEQ.
* a pot-fraction f bet/raise first matches the outstanding amount `toc`, then adds
  inc = round_half_up(f * (pot + toc)) chips, pot = starting pot + all chips
  committed this street; f is an exact rational so the rounding is exact integer
  arithmetic.  Sizes whose total reaches the stack are dropped; "all-in"
  (total = stack) is added when the context lists it; duplicates are merged.
* fold is offered facing no bet only when ``open_fold`` (the paper lists it).
* payoffs are net chips for the whole hand: both players put pot/2 in before
  the river.  Fold by P1: -(pot/2 + c1) to P1; fold by P2: +(pot/2 + c2);
  showdown: +-(pot/2 + c) to the winner, 0 on a tie.
"""
from fractions import Fraction

import numpy as np
import scipy.sparse as sp

from .cards import hand_label
from .treeplex import Treeplex

CONTEXTS = ("P1_OPEN", "P1_VS_BET", "P1_VS_RAISE", "P1_SUBSEQ",
            "P2_VS_CHECK", "P2_VS_BET", "P2_SUBSEQ")


class RiverParams:
    def __init__(self, pot, stack, fracs, allin, raise_cap=1000, open_fold=True, big_blind=100):
        self.pot = int(pot)
        self.stack = int(stack)
        self.fracs = {k: [Fraction(f) for f in fracs.get(k, ())] for k in CONTEXTS}
        self.allin = {k: bool(allin.get(k, False)) for k in CONTEXTS}
        self.raise_cap = int(raise_cap)
        self.open_fold = bool(open_fold)
        self.big_blind = big_blind


def context(player, n_bets):
    if player == 0:
        return ("P1_OPEN", "P1_VS_BET", "P1_VS_RAISE")[n_bets] if n_bets < 3 else "P1_SUBSEQ"
    return ("P2_VS_CHECK", "P2_VS_BET")[n_bets] if n_bets < 2 else "P2_SUBSEQ"


class PubNode:
    __slots__ = ("kind", "player", "history", "children", "fold_by",
                 "payoff_fold_to_p1", "showdown_amount")

    def __init__(self, kind, player=None, history="", children=None):
        self.kind = kind
        self.player = player
        self.history = history
        self.children = children or []
        self.fold_by = None
        self.payoff_fold_to_p1 = None
        self.showdown_amount = None


def _join(h, t):
    return t if not h else h + "/" + t


def betting_tree(rp):
    """Public betting tree of the river endgame."""
    half = rp.pot / 2.0

    def fold_terminal(p, c, hist):
        t = PubNode("terminal", history=hist)
        t.fold_by = p
        t.payoff_fold_to_p1 = -(half + c[0]) if p == 0 else (half + c[1])
        return t

    def showdown_terminal(c, hist):
        assert c[0] == c[1]
        t = PubNode("terminal", history=hist)
        t.showdown_amount = half + c[0]
        return t

    def rec(p, c, n_bets, hist):
        me, opp = c[p], c[1 - p]
        toc = opp - me
        pot = rp.pot + c[0] + c[1]
        node = PubNode("decision", player=p, history=hist)
        if toc > 0 or rp.open_fold:
            node.children.append(("f", fold_terminal(p, c, _join(hist, "f"))))
        if toc > 0:
            cc = list(c)
            cc[p] = opp
            node.children.append(("c", showdown_terminal(cc, _join(hist, "c"))))
        elif p == 0:
            node.children.append(("k", rec(1, c, n_bets, _join(hist, "k"))))
        else:
            node.children.append(("k", showdown_terminal(c, _join(hist, "k"))))
        if n_bets < rp.raise_cap and opp < rp.stack:
            ctx = context(p, n_bets)
            totals = set()
            for f in rp.fracs[ctx]:
                X = pot + toc
                inc = (2 * f.numerator * X + f.denominator) // (2 * f.denominator)
                tot = me + toc + inc
                if inc >= 1 and tot < rp.stack:
                    totals.add(tot)
            if rp.allin[ctx]:
                totals.add(rp.stack)
            for tot in sorted(totals):
                cc = list(c)
                cc[p] = tot
                tok = "b%d" % tot
                node.children.append((tok, rec(1 - p, cc, n_bets + 1, _join(hist, tok))))
        return node

    return rec(0, [0, 0], 0, "")


class PublicSeqs:
    """Per-player public decision nodes (top-down) and public sequences (node, action)."""

    def __init__(self, tree, player):
        self.nodes = []          # decision nodes of `player`, top-down
        self.node_first = []     # first public sequence of each node
        self.node_parent = []    # parent public sequence (-1 = empty sequence)
        self.seq_token_hist = []  # history string including the action
        seq_of = {}

        def rec(node, last_seq):
            if node.kind == "terminal":
                node_last[id(node)] = last_seq
                return
            if node.player == player:
                m = len(self.nodes)
                self.nodes.append(node)
                self.node_first.append(len(self.seq_token_hist))
                self.node_parent.append(last_seq)
                firsts = []
                for tok, ch in node.children:
                    firsts.append(len(self.seq_token_hist))
                    self.seq_token_hist.append(_join(node.history, tok))
                for (tok, ch), s in zip(node.children, firsts):
                    rec(ch, s)
                seq_of[m] = firsts
            else:
                for tok, ch in node.children:
                    rec(ch, last_seq)

        node_last = {}
        rec(tree, -1)
        self.n_pub = len(self.seq_token_hist)
        self.terminal_last = node_last  # id(terminal) -> last public seq of `player` (-1 = empty)


def terminals(tree):
    out = []

    def rec(n):
        if n.kind == "terminal":
            out.append(n)
        else:
            for _, ch in n.children:
                rec(ch)
    rec(tree)
    return out


class RiverSeqForm:
    """Sequence form of a river endgame, vectorised over hands.

    Sequence index for player p, hand a (position in ``hands``), public seq k:
    1 + a * n_pub[p] + k; index 0 is the empty sequence.  A[i, j] = sum over
    leaves z with seq1(z)=i, seq2(z)=j of chance(z) * payoff-to-player-2(z)
    ("A is the sequence-form payoff matrix"; x minimises <x, Ay>).
    Chance(h1, h2) = prior1[h1] prior2[h2] [h1, h2 disjoint] / Z.
    """

    def __init__(self, params, deck, board, prior1, prior2, build_sparse=True):
        from .handeval import holdem_strengths
        self.params = params
        self.deck = deck
        self.board = tuple(board)
        self.tree = betting_tree(params)
        self.hands = [h for h in deck.combos() if not set(h) & set(board)]
        H = len(self.hands)
        self.H = H
        self.pi1 = np.array([prior1.get(h, 0.0) for h in self.hands])
        self.pi2 = np.array([prior2.get(h, 0.0) for h in self.hands])
        cards = np.array(self.hands)
        share = ((cards[:, None, 0] == cards[None, :, 0]) | (cards[:, None, 0] == cards[None, :, 1]) |
                 (cards[:, None, 1] == cards[None, :, 0]) | (cards[:, None, 1] == cards[None, :, 1]))
        compat = ~share
        C = np.outer(self.pi1, self.pi2) * compat
        self.Z = C.sum()
        self.C = C / self.Z
        st = holdem_strengths(deck, board, self.hands)
        self.strength = st
        # sign of player 2's showdown payoff: +1 when h2 beats h1
        self.Sgn = np.sign(st[None, :] - st[:, None]).astype(float)
        self.pub = [PublicSeqs(self.tree, 0), PublicSeqs(self.tree, 1)]
        self.terms = terminals(self.tree)
        self.X = self._treeplex(0)
        self.Y = self._treeplex(1)
        self.labels_x = self._labels(0)
        self.labels_y = self._labels(1)
        self.A = self._sparse_A() if build_sparse else None
        self.big_blind = params.big_blind

    # --------------------------------------------------------------- structure
    def seq_index(self, p, a, k):
        return 0 if k < 0 else 1 + a * self.pub[p].n_pub + k

    def _treeplex(self, p):
        pub = self.pub[p]
        simplexes = []
        for a in range(self.H):
            for m, node in enumerate(pub.nodes):
                simplexes.append((self.seq_index(p, a, pub.node_first[m]), len(node.children),
                                  self.seq_index(p, a, pub.node_parent[m])))
        return Treeplex(1 + self.H * pub.n_pub, simplexes)

    def _labels(self, p):
        pub = self.pub[p]
        labels = ["∅"]
        for h in self.hands:
            hl = hand_label(h)
            labels.extend(hl + "|" + s for s in pub.seq_token_hist)
        return labels

    def block(self, t):
        """Dense H x H block of A contributed by terminal t (rows h1, cols h2)."""
        if t.fold_by is not None:
            return self.C * (-t.payoff_fold_to_p1)
        return self.C * self.Sgn * t.showdown_amount

    def _sparse_A(self):
        rows, cols, vals = [], [], []
        a1 = np.repeat(np.arange(self.H), self.H)
        a2 = np.tile(np.arange(self.H), self.H)
        nz = self.C.reshape(-1) != 0
        for t in self.terms:
            k1 = self.pub[0].terminal_last[id(t)]
            k2 = self.pub[1].terminal_last[id(t)]
            r = np.where(k1 < 0, 0, 1 + a1 * self.pub[0].n_pub + k1)
            c = np.where(k2 < 0, 0, 1 + a2 * self.pub[1].n_pub + k2)
            v = self.block(t).reshape(-1)
            rows.append(r[nz])
            cols.append(c[nz])
            vals.append(v[nz])
        A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(self.X.n_seq, self.Y.n_seq)).tocsr()
        A.sum_duplicates()
        return A

    # --------------------------------------------------------------- products without A
    def Ay(self, y):
        """A @ y accumulated terminal block by terminal block (A never stored)."""
        g = np.zeros(self.X.n_seq)
        n1, n2 = self.pub[0].n_pub, self.pub[1].n_pub
        for t in self.terms:
            k1 = self.pub[0].terminal_last[id(t)]
            k2 = self.pub[1].terminal_last[id(t)]
            ys = np.ones(self.H) if k2 < 0 else y[1 + np.arange(self.H) * n2 + k2]
            v = self.block(t) @ ys
            if k1 < 0:
                g[0] += v.sum()
            else:
                g[1 + np.arange(self.H) * n1 + k1] += v
        return g

    def ATx(self, x):
        g = np.zeros(self.Y.n_seq)
        n1, n2 = self.pub[0].n_pub, self.pub[1].n_pub
        for t in self.terms:
            k1 = self.pub[0].terminal_last[id(t)]
            k2 = self.pub[1].terminal_last[id(t)]
            xs = np.ones(self.H) if k1 < 0 else x[1 + np.arange(self.H) * n1 + k1]
            v = self.block(t).T @ xs
            if k2 < 0:
                g[0] += v.sum()
            else:
                g[1 + np.arange(self.H) * n2 + k2] += v
        return g

    def max_abs_A(self):
        """||A|| as the largest |A_ij| (reading R7).  Terminals map to distinct
        public sequence pairs in this game; a terminal whose player-1 (player-2)
        sequence is empty puts the column (row) sums of its block in row (column) 0."""
        pairs = {(self.pub[0].terminal_last[id(t)], self.pub[1].terminal_last[id(t)]) for t in self.terms}
        assert len(pairs) == len(self.terms)
        best = 0.0
        for t in self.terms:
            k1 = self.pub[0].terminal_last[id(t)]
            k2 = self.pub[1].terminal_last[id(t)]
            B = self.block(t)
            if k1 < 0 and k2 < 0:
                B = np.array([[B.sum()]])
            elif k1 < 0:
                B = B.sum(axis=0, keepdims=True)
            elif k2 < 0:
                B = B.sum(axis=1, keepdims=True)
            best = max(best, float(np.abs(B).max()))
        return best
