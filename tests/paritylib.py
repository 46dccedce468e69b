"""Test infrastructure: build the same game on both sides and align index spaces.

The CUDA path stores a player's vector per game as [n_pub][H_pad]; the oracle
uses its own sequence numbering.  Both emit canonical labels
``"<hand cards>|<public history through the action>"`` ("∅" for the empty
sequence), so the alignment is a label join -- no arithmetic is shared.
"""
import numpy as np

from oracle import games, river, seqform
from oracle.cards import Deck, hand_label
from paper_1810_03063_b200 import workloads


class Pair:
    """Product game (batch) + one oracle sequence form per game."""

    def __init__(self, kind, n_games=1, spec=None, seed=0, n_ranks=13, n_suits=4, build_sparse=True,
                 sample=None, boards=None, priors=None):
        """``sample``: games that get an oracle sequence form (default: all); ``boards`` /
        ``priors`` override the seeded river inputs."""
        import paper_1810_03063_b200 as P
        self.kind = kind
        self.n_games = n_games
        if kind == "kuhn":
            self.game = P.Game(P.KUHN, n_games=n_games)
            sf = seqform.build(games.kuhn())
            self.sf = [sf] * n_games
        elif kind == "leduc":
            self.game = P.Game(P.LEDUC, n_games=n_games)
            sf = seqform.build(games.leduc())
            self.sf = [sf] * n_games
        else:
            spec = spec or workloads.river_spec("tiny", pot=2, stack=6, raise_cap=2)
            if boards is None:
                boards = workloads.random_boards(n_games, seed, n_ranks, n_suits)
            if priors is None:
                priors = workloads.random_priors(boards, seed, n_ranks, n_suits)
            p1, p2 = priors
            self.boards, self.priors = boards, (p1, p2)
            self.game = P.Game(P.RIVER, n_games=n_games, river=spec, boards=boards, prior1=p1, prior2=p2,
                               n_ranks=n_ranks, n_suits=n_suits)
            deck = Deck(n_ranks, n_suits)
            rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap",
                                                           "open_fold")})
            which = range(n_games) if sample is None else sample
            self.sf = {g: river.RiverSeqForm(rp, deck, boards[g], workloads.prior_dict(p1[g], deck.n_cards),
                                             workloads.prior_dict(p2[g], deck.n_cards), build_sparse=build_sparse)
                       for g in which}
        self._maps = {}

    def tp(self, g, p):
        return self.sf[g].X if p == 0 else self.sf[g].Y

    def labels(self, g, p):
        return self.sf[g].labels_x if p == 0 else self.sf[g].labels_y

    def index_map(self, g, p):
        """oracle sequence index i >= 1  ->  flat product index s*H_pad + h."""
        key = (g, p)
        if key in self._maps:
            return self._maps[key]
        G = self.game
        cards = G.hand_cards(g)
        hl = [hand_label([c for c in row if c >= 0]) for row in cards]
        hist = [G.pub_history(p, s) for s in range(G.n_pub[p])]
        where = {}
        for s in range(1, G.n_pub[p]):
            for h in range(G.H):
                where[hl[h] + "|" + hist[s]] = s * G.H_pad + h
        labels = self.labels(g, p)
        idx = np.array([where[lab] for lab in labels[1:]], dtype=np.int64)
        self._maps[key] = idx
        return idx

    # oracle vector (n_seq) <-> product block [n_pub * H_pad]
    def to_product(self, g, p, v, row0=None):
        G = self.game
        out = np.zeros(G.n_pub[p] * G.H_pad)
        out[self.index_map(g, p)] = v[1:]
        if row0 is not None:
            out[:G.H] = row0
        return out

    def from_product(self, g, p, block):
        v = np.zeros(self.tp(g, p).n_seq)
        v[1:] = block[self.index_map(g, p)]
        return v

    def valid_mask(self, g, p):
        G = self.game
        m = np.zeros(G.n_pub[p] * G.H_pad, dtype=bool)
        m[self.index_map(g, p)] = True
        return m


def random_behavioral(tp, rng, spread=1.0):
    b = tp.uniform_behavioral()
    for j in range(tp.n_simplex):
        s, n = tp.start[j], tp.size[j]
        w = np.exp(spread * rng.standard_normal(n))
        b[s:s + n] = w / w.sum()
    return b


def rel_err(got, want):
    scale = max(np.abs(want).max(), 1e-300)
    return np.abs(got - want).max() / scale
