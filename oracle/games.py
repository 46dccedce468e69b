"""Literal extensive-form game trees (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Nodes are plain Python objects; ``seqform.build`` turns a tree into the
sequence form.  Games:

* ``kuhn()``          3-card Kuhn poker (ante 1, bet 1); game value -1/18 to player 1.
* ``leduc()``         Leduc hold'em: 6 cards (J,Q,K x 2 suits), ante 1, bets 2 then 4,
                      at most 2 bets per round, board card dealt between rounds
                      (BASELINE.json configs[1]; PAPER.md:719-721 names the game).
* ``river_literal()`` the river endgame of PAPER.md:670-688 with an explicit chance
                      node over every hand pair (small decks only; the full deck
                      uses the hand-vectorised builder in ``river.py``).
* ``matrix_game()``   a one-shot game with payoff matrix (both players one simplex).

Payoffs are to player 1 (the x / first-moving player).  Public-history labels:
tokens joined by '/': 'k' check, 'c' call, 'f' fold, 'b<n>' bet/raise to a total
of n chips committed in the current round by the actor, 'd<card>' a public card.
"""
import itertools

import numpy as np

from .cards import hand_label


class Chance:
    __slots__ = ("outcomes",)

    def __init__(self, outcomes):
        self.outcomes = outcomes  # list of (prob, child)


class Decision:
    __slots__ = ("player", "hand", "history", "actions")

    def __init__(self, player, hand, history, actions):
        self.player = player      # 0 = x (player 1), 1 = y (player 2)
        self.hand = hand          # hand label of the acting player (private information)
        self.history = history    # public history string before the action
        self.actions = actions    # list of (token, child)

    @property
    def infoset(self):
        return (self.player, self.hand, self.history)


class Terminal:
    __slots__ = ("payoff1",)

    def __init__(self, payoff1):
        self.payoff1 = float(payoff1)


def _join(hist, tok):
    return tok if not hist else hist + "/" + tok


# ---------------------------------------------------------------------- matrix game
def matrix_game(M):
    """One-shot game: player 1 picks row i, player 2 (not seeing it) picks column j,
    player 1 receives M[i][j].  Sequence-form A is then -M (A is player 2's payoff)."""
    M = np.asarray(M, dtype=float)
    rows = []
    for i in range(M.shape[0]):
        cols = [("a%d" % j, Terminal(M[i, j])) for j in range(M.shape[1])]
        rows.append(("a%d" % i, Decision(1, "", "", cols)))
    return Decision(0, "", "", rows)


# ---------------------------------------------------------------------- Kuhn
def kuhn():
    """Kuhn poker: cards J<Q<K (ids 0,1,2), ante 1, one bet of 1."""
    def showdown(c1, c2, amount):
        return amount if c1 > c2 else -amount

    outcomes = []
    for c1, c2 in itertools.permutations(range(3), 2):
        h1, h2 = hand_label([c1]), hand_label([c2])
        # P1 checks
        p2_after_check = Decision(1, h2, "k", [
            ("k", Terminal(showdown(c1, c2, 1))),
            ("b1", Decision(0, h1, "k/b1", [
                ("f", Terminal(-1)),
                ("c", Terminal(showdown(c1, c2, 2))),
            ])),
        ])
        p2_after_bet = Decision(1, h2, "b1", [
            ("f", Terminal(+1)),
            ("c", Terminal(showdown(c1, c2, 2))),
        ])
        root = Decision(0, h1, "", [("k", p2_after_check), ("b1", p2_after_bet)])
        outcomes.append((1.0 / 6.0, root))
    return Chance(outcomes)


# ---------------------------------------------------------------------- Leduc
LEDUC_CARDS = 6  # id = rank*2 + suit, ranks J,Q,K


def leduc_strength(card, board):
    """Pair with the board beats any unpaired hand; otherwise the higher rank."""
    r, b = card // 2, board // 2
    return 10 + r if r == b else r


def leduc(bets=(2, 4), max_bets=2, ante=1):
    def betting(c1, c2, board, rnd, committed, to_act, n_bets, hist, round_commit):
        """committed: total chips put in by each player; round_commit: chips this round."""
        hands = (hand_label([c1]), hand_label([c2]))
        me, opp = to_act, 1 - to_act
        toc = committed[opp] - committed[me]
        acts = []
        if toc > 0:
            # fold: the folder loses everything committed
            pay = -committed[0] if me == 0 else committed[1]
            acts.append(("f", Terminal(pay)))
            # call ends the round
            newc = list(committed)
            newc[me] += toc
            acts.append(("c", end_round(c1, c2, board, rnd, newc, _join(hist, "c"))))
        else:
            if me == 0:
                acts.append(("k", betting(c1, c2, board, rnd, committed, 1, n_bets,
                                          _join(hist, "k"), round_commit)))
            else:
                acts.append(("k", end_round(c1, c2, board, rnd, committed, _join(hist, "k"))))
        if n_bets < max_bets:
            newc = list(committed)
            newrc = list(round_commit)
            add = toc + bets[rnd]
            newc[me] += add
            newrc[me] += add
            tok = "b%d" % newrc[me]
            acts.append((tok, betting(c1, c2, board, rnd, newc, opp, n_bets + 1,
                                      _join(hist, tok), newrc)))
        return Decision(me, hands[me], hist, acts)

    def end_round(c1, c2, board, rnd, committed, hist):
        if rnd == 0:
            rest = [c for c in range(LEDUC_CARDS) if c not in (c1, c2)]
            outs = []
            for b in rest:
                outs.append((1.0 / len(rest),
                             betting(c1, c2, b, 1, committed, 0, 0, _join(hist, "d%d" % b), [0, 0])))
            return Chance(outs)
        s1, s2 = leduc_strength(c1, board), leduc_strength(c2, board)
        w = committed[1]  # equal to committed[0] at a showdown
        return Terminal(w if s1 > s2 else (-w if s1 < s2 else 0.0))

    outcomes = []
    for c1, c2 in itertools.permutations(range(LEDUC_CARDS), 2):
        root = betting(c1, c2, None, 0, [ante, ante], 0, 0, "", [0, 0])
        outcomes.append((1.0 / 30.0, root))
    return Chance(outcomes)


# ---------------------------------------------------------------------- river (literal)
def river_literal(params, deck, board, prior1, prior2):
    """River endgame as a literal tree: chance deals (h1, h2) with
    probability prior1[h1] prior2[h2] / Z over disjoint pairs of hands that avoid
    the board ("a Chance node deal[s] out hands according to this
    conditional distribution"), then the public betting tree of ``river.betting_tree``.

    prior1/prior2: dict hand(tuple c1<c2) -> weight.  Small decks only.
    """
    from .handeval import holdem_strengths
    from . import river

    tree = river.betting_tree(params)
    hands = [h for h in deck.combos() if not set(h) & set(board)]
    strength = dict(zip(hands, holdem_strengths(deck, board, hands)))
    pairs = [(a, b) for a in hands for b in hands if not set(a) & set(b)]
    w = np.array([prior1.get(a, 0.0) * prior2.get(b, 0.0) for a, b in pairs])
    Z = w.sum()

    def instantiate(node, h1, h2):
        if node.kind == "terminal":
            if node.fold_by is not None:
                return Terminal(node.payoff_fold_to_p1)
            s1, s2 = strength[h1], strength[h2]
            W = node.showdown_amount
            return Terminal(W if s1 > s2 else (-W if s1 < s2 else 0.0))
        hand = hand_label(h1 if node.player == 0 else h2)
        return Decision(node.player, hand, node.history,
                        [(tok, instantiate(ch, h1, h2)) for tok, ch in node.children])

    outcomes = [(wi / Z, instantiate(tree, a, b)) for (a, b), wi in zip(pairs, w) if wi > 0]
    return Chance(outcomes)


# ---------------------------------------------------------------------- tree walk
def expected_payoff1(node, strat):
    """Expected payoff to player 1 by walking the tree with behavioural strategies.

    strat(player, hand, history) -> probability vector over the node's actions.
    Independent of the sequence form: pins A via x^T A y = -E[u1]."""
    if isinstance(node, Terminal):
        return node.payoff1
    if isinstance(node, Chance):
        return sum(p * expected_payoff1(ch, strat) for p, ch in node.outcomes)
    probs = strat(node.player, node.hand, node.history)
    return sum(pr * expected_payoff1(ch, strat)
               for pr, (_, ch) in zip(probs, node.actions) if pr != 0.0)
