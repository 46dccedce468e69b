"""Cards, decks and canonical hole-card combos (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

A deck has ``n_ranks`` ranks (the TOP ``n_ranks`` of 2..A, so the ace is always
rank value 12) and ``n_suits`` suits.  Card id = rank_pos * n_suits + suit with
rank_pos in [0, n_ranks).  The standard 52-card deck is n_ranks=13, n_suits=4,
so card id = rank*4 + suit with rank 0 = '2'.

The canonical hole-card order (used by the C-ABI and workloads for priors) is
all pairs (c1, c2), c1 < c2, in lexicographic order: 1326 combos for 52 cards.
PAPER.md:670-675 (the river subgame deals each player a private hand).
"""
import itertools

RANK_CHARS = "23456789TJQKA"
SUIT_CHARS = "cdhs"


class Deck:
    def __init__(self, n_ranks=13, n_suits=4):
        assert 1 <= n_ranks <= 13 and 1 <= n_suits <= 4
        self.n_ranks = n_ranks
        self.n_suits = n_suits
        self.n_cards = n_ranks * n_suits

    def rank_value(self, card):
        """Rank value in 0..12 (12 = ace)."""
        return 13 - self.n_ranks + card // self.n_suits

    def suit(self, card):
        return card % self.n_suits

    def name(self, card):
        return RANK_CHARS[self.rank_value(card)] + SUIT_CHARS[self.suit(card)]

    def combos(self):
        """Canonical 2-card hole-card combos (c1 < c2), lexicographic."""
        return list(itertools.combinations(range(self.n_cards), 2))


def hand_label(cards):
    """Canonical hand label used to align oracle and CUDA index spaces:
    ascending card ids joined by ','."""
    return ",".join(str(c) for c in sorted(cards))
