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


# Worst per-element relative errors seen by assert_parity / assert_scalar, by check name, and
# the worst error as a fraction of the bound the check allowed (<= 1: passed; printed at the
# end of the session by tests/conftest.py).  A check whose bound includes a measured sensitivity
# of the oracle (practical mu, fp32 CFR+) can show a relative error above its rtol on entries
# that the sensitivity floor covers; the fraction-of-bound column is the verdict.
REPORT = {}
BOUND = {}

FLOOR64, FLOOR32 = 1e-13, 1e-5


def assert_parity(got, want, rtol, what, floor=None, mask=None):
    """BASELINE.json north_star's bar, per element: |got - want| <= rtol * |want|, with an
    absolute floor of floor * max|want| for entries that cancel to ~0 (a showdown entry is a
    difference of prefix sums as large as the largest entry, so its rounding is ~ulp of the
    largest entry, not of itself): floor = 1e-13 in fp64 (~450 ulp of the largest entry),
    1e-5 in fp32 (the north star's fp32 bar itself: with a 24-bit mantissa an entry that cancels
    to 1e-3 of the largest cannot be 1e-5-accurate relative to itself).  Records the worst relative error among entries >= 1e-6 max|want|."""
    got = np.asarray(got, dtype=float).ravel()
    want = np.asarray(want, dtype=float).ravel()
    if mask is not None:
        got, want = got[np.asarray(mask).ravel()], want[np.asarray(mask).ravel()]
    assert got.shape == want.shape
    if floor is None:
        floor = FLOOR64 if rtol < 1e-7 else FLOOR32
    scale = np.abs(want).max() if want.size else 0.0
    err = np.abs(got - want)
    bad = ~(err <= rtol * np.abs(want) + floor * scale)
    if bad.any():
        i = int(np.argmax(np.where(bad, err / np.maximum(np.abs(want), 1e-300), -1.0)))
        raise AssertionError("%s: %d of %d entries off (worst: got %r want %r, |want|max %g)"
                             % (what, int(bad.sum()), got.size, got[i], want[i], scale))
    big = np.abs(want) >= 1e-6 * scale
    worst = float((err[big] / np.abs(want[big])).max()) if big.any() and scale > 0 else 0.0
    key = what.split("[")[0]
    REPORT[key] = max(REPORT.get(key, 0.0), worst)
    allowed = rtol * np.abs(want) + floor * scale
    frac = float((err / np.maximum(allowed, 1e-300)).max()) if err.size else 0.0
    BOUND[key] = max(BOUND.get(key, 0.0), frac)
    return worst


def assert_scalar(got, want, rtol, what, floor=1e-12):
    """Per-game values / eps_sad: |got - want| <= rtol * |want| + floor (payoff units)."""
    got, want = float(got), float(want)
    if not abs(got - want) <= rtol * abs(want) + floor:
        raise AssertionError("%s: got %r want %r" % (what, got, want))
    key = what.split("[")[0]
    if want != 0:
        REPORT[key] = max(REPORT.get(key, 0.0), abs(got - want) / abs(want))
    allowed = rtol * abs(want) + floor
    BOUND[key] = max(BOUND.get(key, 0.0), abs(got - want) / allowed if allowed > 0 else 0.0)
