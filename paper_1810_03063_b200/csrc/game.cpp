// Host-side game construction: public trees (Kuhn, Leduc, river endgame), the
// per-player treeplex layout, hand strength order and card-removal tables.
// Independent of the oracle (separate implementation of the same game rules).
#include "game.h"

#include <algorithm>
#include <array>
#include <stdexcept>
#include <cmath>
#include <functional>
#include <numeric>
#include <set>
#include <thread>

namespace egt {

static std::string join(const std::string& h, const std::string& t) { return h.empty() ? t : h + "/" + t; }

// ------------------------------------------------------------------ hand strength
// Standard poker ranking; ranks 0..12 (12 = ace), suits any ints.
static int64_t eval5(const int* r, const int* s) {
    int cnt[13] = {0};
    for (int i = 0; i < 5; ++i) cnt[r[i]]++;
    bool flush = true;
    for (int i = 1; i < 5; ++i) flush = flush && (s[i] == s[0]);
    int top = -1;
    for (int hi = 12; hi >= 4 && top < 0; --hi) {
        bool ok = true;
        for (int k = 0; k < 5; ++k) ok = ok && cnt[hi - k] > 0;
        if (ok) top = hi;
    }
    if (top < 0 && cnt[12] && cnt[0] && cnt[1] && cnt[2] && cnt[3]) top = 3;  // wheel
    // groups ordered by (count desc, rank desc)
    int grp[5], ng = 0;
    for (int c = 4; c >= 1; --c)
        for (int rk = 12; rk >= 0; --rk)
            if (cnt[rk] == c) grp[ng++] = rk;
    int c0 = cnt[grp[0]], c1 = ng > 1 ? cnt[grp[1]] : 0;
    int cat;
    if (top >= 0 && flush) cat = 8;
    else if (c0 == 4) cat = 7;
    else if (c0 == 3 && c1 == 2) cat = 6;
    else if (flush) cat = 5;
    else if (top >= 0) cat = 4;
    else if (c0 == 3) cat = 3;
    else if (c0 == 2 && c1 == 2) cat = 2;
    else if (c0 == 2) cat = 1;
    else cat = 0;
    int64_t key = cat;
    if (cat == 8 || cat == 4) {
        key = key * 13 + top;
        for (int i = 1; i < 5; ++i) key *= 13;
    } else {
        for (int i = 0; i < 5; ++i) key = key * 13 + (i < ng ? grp[i] : 0);
    }
    return key;
}

// The best 5 of n <= 7 cards directly (rank counts, suit counts, rank masks) -- the same key
// as the maximum of eval5 over all 5-subsets (hand_strength_subsets), which it replaces on
// the load path: category, then the group ranks ordered by (count desc, rank desc).
int64_t hand_strength(const int* ranks, const int* suits, int n) {
    if (n < 5 || n > 7) return hand_strength_subsets(ranks, suits, n);
    int cnt[13] = {0}, scnt[8] = {0};
    unsigned mask = 0, smask[8] = {0};
    for (int i = 0; i < n; ++i) {
        cnt[ranks[i]]++;
        mask |= 1u << ranks[i];
        const int su = suits[i] & 7;
        scnt[su]++;
        smask[su] |= 1u << ranks[i];
    }
    auto top_straight = [](unsigned m) {
        for (int hi = 12; hi >= 4; --hi)
            if (((m >> (hi - 4)) & 0x1Fu) == 0x1Fu) return hi;
        if ((m & 0x100Fu) == 0x100Fu) return 3;  // wheel A-2-3-4-5
        return -1;
    };
    auto key_of = [](int cat, const int* g, int ng) {
        int64_t key = cat;
        for (int i = 0; i < 5; ++i) key = key * 13 + (i < ng ? g[i] : 0);
        return key;
    };
    auto straight_key = [](int cat, int top) {
        int64_t key = (int64_t)cat * 13 + top;
        for (int i = 1; i < 5; ++i) key *= 13;
        return key;
    };
    int fs = -1;
    for (int su = 0; su < 8; ++su)
        if (scnt[su] >= 5) fs = su;
    if (fs >= 0) {
        const int t = top_straight(smask[fs]);
        if (t >= 0) return straight_key(8, t);
    }
    // ranks by count, descending rank
    int quads = -1, trips[2] = {-1, -1}, pairs[3] = {-1, -1, -1}, nt = 0, np = 0;
    for (int rk = 12; rk >= 0; --rk) {
        if (cnt[rk] == 4 && quads < 0) quads = rk;
        else if (cnt[rk] == 3 && nt < 2) trips[nt++] = rk;
        else if (cnt[rk] == 2 && np < 3) pairs[np++] = rk;
    }
    auto kickers = [&](int* out, int want, int ex1, int ex2) {  // highest ranks not ex1/ex2
        int k = 0;
        for (int rk = 12; rk >= 0 && k < want; --rk)
            if (cnt[rk] > 0 && rk != ex1 && rk != ex2) out[k++] = rk;
        return k;
    };
    int g[5];
    if (quads >= 0) {
        g[0] = quads;
        const int k = kickers(g + 1, 1, quads, -1);
        return key_of(7, g, 1 + k);
    }
    if (nt >= 1 && (nt >= 2 || np >= 1)) {  // full house: best trips + best other pair
        g[0] = trips[0];
        g[1] = nt >= 2 ? (np >= 1 ? std::max(trips[1], pairs[0]) : trips[1]) : pairs[0];
        return key_of(6, g, 2);
    }
    if (fs >= 0) {
        int k = 0;
        for (int rk = 12; rk >= 0 && k < 5; --rk)
            if (smask[fs] >> rk & 1u) g[k++] = rk;
        return key_of(5, g, 5);
    }
    {
        const int t = top_straight(mask);
        if (t >= 0) return straight_key(4, t);
    }
    if (nt >= 1) {
        g[0] = trips[0];
        const int k = kickers(g + 1, 2, trips[0], -1);
        return key_of(3, g, 1 + k);
    }
    if (np >= 2) {
        g[0] = pairs[0];
        g[1] = pairs[1];
        const int k = kickers(g + 2, 1, pairs[0], pairs[1]);
        return key_of(2, g, 2 + k);
    }
    if (np == 1) {
        g[0] = pairs[0];
        const int k = kickers(g + 1, 3, pairs[0], -1);
        return key_of(1, g, 1 + k);
    }
    const int k = kickers(g, 5, -1, -1);
    return key_of(0, g, k);
}

int64_t hand_strength_subsets(const int* ranks, const int* suits, int n) {
    int64_t best = -1;
    int idx[5];
    // all 5-subsets of n <= 7 cards
    for (idx[0] = 0; idx[0] < n; ++idx[0])
        for (idx[1] = idx[0] + 1; idx[1] < n; ++idx[1])
            for (idx[2] = idx[1] + 1; idx[2] < n; ++idx[2])
                for (idx[3] = idx[2] + 1; idx[3] < n; ++idx[3])
                    for (idx[4] = idx[3] + 1; idx[4] < n; ++idx[4]) {
                        int r[5], s[5];
                        for (int k = 0; k < 5; ++k) { r[k] = ranks[idx[k]]; s[k] = suits[idx[k]]; }
                        best = std::max(best, eval5(r, s));
                    }
    return best;
}

// ------------------------------------------------------------------ public trees
static int add_node(PublicTree& T, PNode n) {
    T.nodes.push_back(std::move(n));
    return (int)T.nodes.size() - 1;
}

static int terminal(PublicTree& T, int kind, double amount, double kappa, int bs, const std::string& hist) {
    PNode n;
    n.kind = ND_TERMINAL;
    n.term_kind = kind;
    n.amount = amount;
    n.kappa = kappa;
    n.board_state = bs;
    n.hist = hist;
    return add_node(T, n);
}

static int decision(PublicTree& T, int player, int bs, const std::string& hist) {
    PNode n;
    n.kind = ND_DECISION;
    n.player = player;
    n.board_state = bs;
    n.hist = hist;
    return add_node(T, n);
}

static void link(PublicTree& T, int parent, const std::string& tok, int child) {
    T.nodes[parent].tok.push_back(tok);
    T.nodes[parent].child.push_back(child);
}

// Kuhn: cards J<Q<K, ante 1, bet 1; every deal (c1,c2) has probability 1/6.
static void build_kuhn(PublicTree& T) {
    const double k = 1.0 / 6.0;
    T.n_board_states = 1;
    T.board_cards = {{}};
    int root = decision(T, 0, 0, "");
    int p2k = decision(T, 1, 0, "k");
    link(T, root, "k", p2k);
    link(T, p2k, "k", terminal(T, T_SHOWDOWN, 1, k, 0, "k/k"));
    int p1kb = decision(T, 0, 0, "k/b1");
    link(T, p2k, "b1", p1kb);
    link(T, p1kb, "f", terminal(T, T_FOLD_P1, +1, k, 0, "k/b1/f"));
    link(T, p1kb, "c", terminal(T, T_SHOWDOWN, 2, k, 0, "k/b1/c"));
    int p2b = decision(T, 1, 0, "b1");
    link(T, root, "b1", p2b);
    link(T, p2b, "f", terminal(T, T_FOLD_P2, -1, k, 0, "b1/f"));
    link(T, p2b, "c", terminal(T, T_SHOWDOWN, 2, k, 0, "b1/c"));
}

// Leduc: 6 cards (id = rank*2 + suit), ante 1, bets 2 then 4, at most 2 bets per round,
// board card dealt between the rounds (board state 1 + card).  Deal probability of an
// ordered (c1, c2) is 1/30; with the board card 1/120.
static void build_leduc(PublicTree& T) {
    const int bets[2] = {2, 4};
    T.n_board_states = 7;
    T.board_cards.assign(7, {});
    for (int b = 0; b < 6; ++b) T.board_cards[1 + b] = {b};
    std::function<int(int, int, int, int, int, int, int, int, const std::string&)> rec;
    std::function<int(int, int, int, int, const std::string&)> end_round;
    end_round = [&](int rnd, int c0, int c1, int bs, const std::string& hist) -> int {
        if (rnd == 0) {
            PNode ch;
            ch.kind = ND_CHANCE;
            ch.hist = hist;
            int cn = add_node(T, ch);
            for (int b = 0; b < 6; ++b) {
                std::string h = join(hist, "d" + std::to_string(b));
                int child = rec(1, c0, c1, 0, 0, 0, 0, 1 + b, h);
                link(T, cn, "d" + std::to_string(b), child);
            }
            return cn;
        }
        return terminal(T, T_SHOWDOWN, (double)c1, 1.0 / 120.0, bs, hist);
    };
    rec = [&](int rnd, int c0, int c1, int rc0, int rc1, int p, int nb, int bs, const std::string& hist) -> int {
        int n = decision(T, p, bs, hist);
        int me = p == 0 ? c0 : c1, opp = p == 0 ? c1 : c0;
        int toc = opp - me;
        double kap = rnd == 0 ? 1.0 / 30.0 : 1.0 / 120.0;
        if (toc > 0) {
            int t = p == 0 ? terminal(T, T_FOLD_P1, +(double)c0, kap, bs, join(hist, "f"))
                           : terminal(T, T_FOLD_P2, -(double)c1, kap, bs, join(hist, "f"));
            link(T, n, "f", t);
            int child = end_round(rnd, opp, opp, bs, join(hist, "c"));
            link(T, n, "c", child);
        } else {
            int child = p == 0 ? rec(rnd, c0, c1, rc0, rc1, 1, nb, bs, join(hist, "k"))
                               : end_round(rnd, c0, c1, bs, join(hist, "k"));
            link(T, n, "k", child);
        }
        if (nb < 2) {
            int add = toc + bets[rnd];
            int nc0 = c0, nc1 = c1, nrc0 = rc0, nrc1 = rc1;
            std::string tok;
            if (p == 0) { nc0 += add; nrc0 += add; tok = "b" + std::to_string(nrc0); }
            else { nc1 += add; nrc1 += add; tok = "b" + std::to_string(nrc1); }
            int child = rec(rnd, nc0, nc1, nrc0, nrc1, 1 - p, nb + 1, bs, join(hist, tok));
            link(T, n, tok, child);
        }
        return n;
    };
    rec(0, 1, 1, 0, 0, 0, 0, 0, "");
}

// River endgame, PAPER.md:670-688 with DESIGN.md readings R10-R13.
struct RiverRules {
    int pot, stack, cap;
    bool open_fold;
    std::vector<std::pair<int64_t, int64_t>> fr[EGT_N_CTX];
    bool allin[EGT_N_CTX];
};

static int river_ctx(int p, int nb) {
    if (p == 0) return nb < 3 ? nb : 3;
    return 4 + (nb < 2 ? nb : 2);
}

static int build_river_rec(PublicTree& T, const RiverRules& R, int p, int64_t c0, int64_t c1, int nb,
                           const std::string& hist) {
    const double half = R.pot / 2.0;
    int n = decision(T, p, 0, hist);
    int64_t me = p == 0 ? c0 : c1, opp = p == 0 ? c1 : c0;
    int64_t toc = opp - me;
    int64_t pot = R.pot + c0 + c1;
    if (toc > 0 || R.open_fold) {
        int t = p == 0 ? terminal(T, T_FOLD_P1, +(half + (double)c0), 1.0, 0, join(hist, "f"))
                       : terminal(T, T_FOLD_P2, -(half + (double)c1), 1.0, 0, join(hist, "f"));
        link(T, n, "f", t);
    }
    if (toc > 0) {
        link(T, n, "c", terminal(T, T_SHOWDOWN, half + (double)opp, 1.0, 0, join(hist, "c")));
    } else if (p == 0) {
        link(T, n, "k", build_river_rec(T, R, 1, c0, c1, nb, join(hist, "k")));
    } else {
        link(T, n, "k", terminal(T, T_SHOWDOWN, half + (double)c0, 1.0, 0, join(hist, "k")));
    }
    if ((R.cap <= 0 || nb < R.cap) && opp < R.stack) {
        int ctx = river_ctx(p, nb);
        std::set<int64_t> totals;
        for (auto& f : R.fr[ctx]) {
            int64_t X = pot + toc;
            int64_t inc = (2 * f.first * X + f.second) / (2 * f.second);  // round half up, exact
            int64_t tot = me + toc + inc;
            if (inc >= 1 && tot < R.stack) totals.insert(tot);
        }
        if (R.allin[ctx]) totals.insert(R.stack);
        for (int64_t tot : totals) {
            std::string tok = "b" + std::to_string(tot);
            int child = p == 0 ? build_river_rec(T, R, 1, tot, c1, nb + 1, join(hist, tok))
                               : build_river_rec(T, R, 0, c0, tot, nb + 1, join(hist, tok));
            link(T, n, tok, child);
        }
    }
    return n;
}

// ------------------------------------------------------------------ layout
static void build_layout(HostGame& G) {
    PublicTree& T = G.tree;
    for (int p = 0; p < 2; ++p) {
        G.pl[p] = PlayerLayout();
        G.pl[p].seq_hist = {""};
        G.pl[p].seq_owner = {-1};
    }
    G.terms.clear();
    std::function<void(int, int, int, int, int)> visit = [&](int n, int s0, int s1, int l0, int l1) {
        const PNode& N = T.nodes[n];
        if (N.kind == ND_TERMINAL) {
            Terminal t;
            t.kind = N.term_kind;
            t.amount = N.amount;
            t.kappa = N.kappa;
            t.board_state = N.board_state;
            t.last_seq[0] = s0;
            t.last_seq[1] = s1;
            G.terms.push_back(t);
            return;
        }
        if (N.kind == ND_CHANCE) {
            for (int c : N.child) visit(c, s0, s1, l0, l1);
            return;
        }
        int p = N.player;
        PlayerLayout& L = G.pl[p];
        int m = (int)L.node_pub.size();
        int first = L.n_pub;
        L.node_pub.push_back(n);
        L.first.push_back(first);
        L.nact.push_back((int)N.child.size());
        L.parent_seq.push_back(p == 0 ? s0 : s1);
        L.board_state.push_back(N.board_state);
        L.level.push_back(p == 0 ? l0 : l1);
        for (size_t a = 0; a < N.child.size(); ++a) {
            L.seq_hist.push_back(join(N.hist, N.tok[a]));
            L.seq_owner.push_back(m);
        }
        L.n_pub += (int)N.child.size();
        for (size_t a = 0; a < N.child.size(); ++a) {
            int s = first + (int)a;
            if (p == 0) visit(N.child[a], s, s1, l0 + 1, l1);
            else visit(N.child[a], s0, s, l0, l1 + 1);
        }
    };
    visit(0, 0, 0, 0, 0);
    for (int p = 0; p < 2; ++p) {
        PlayerLayout& L = G.pl[p];
        L.depth = 0;
        for (int l : L.level) L.depth = std::max(L.depth, l + 1);
        std::vector<std::vector<int>> by(L.n_pub);
        for (size_t t = 0; t < G.terms.size(); ++t) by[G.terms[t].last_seq[p]].push_back((int)t);
        L.term_off.assign(L.n_pub + 1, 0);
        L.term_idx.clear();
        for (int s = 0; s < L.n_pub; ++s) {
            L.term_off[s] = (int)L.term_idx.size();
            for (int t : by[s]) L.term_idx.push_back(t);
        }
        L.term_off[L.n_pub] = (int)L.term_idx.size();
        // Order for the card-domain gradient kernel (which reuses an opponent row's totals for a
        // fold that follows a terminal on the same opponent row, and recomputes for a
        // showdown): inside a row showdowns first; and where a row ends with a fold and the
        // next starts with a showdown on the same opponent row, the two rows swap (row order
        // is free: each row is written when its last terminal is done).  pair_next[r] marks a
        // swapped pair (r, r + 1), which a shard boundary never splits.
        for (int s = 0; s < L.n_pub; ++s)
            std::stable_sort(L.term_idx.begin() + L.term_off[s], L.term_idx.begin() + L.term_off[s + 1],
                             [&](int a, int b) { return (G.terms[a].kind == T_SHOWDOWN) > (G.terms[b].kind == T_SHOWDOWN); });
        L.rows_term.clear();
        for (int s = 0; s < L.n_pub; ++s)
            if (L.term_off[s + 1] > L.term_off[s]) L.rows_term.push_back(s);
        L.pair_next.assign(L.rows_term.size(), 0);
        for (size_t r = 0; r + 1 < L.rows_term.size(); ++r) {
            const int a = L.rows_term[r], b = L.rows_term[r + 1];
            const Terminal& last = G.terms[L.term_idx[L.term_off[a + 1] - 1]];
            const Terminal& first = G.terms[L.term_idx[L.term_off[b]]];
            const int oa = last.last_seq[1 - p], ob = first.last_seq[1 - p];
            if (last.kind != T_SHOWDOWN && first.kind == T_SHOWDOWN && oa == ob && oa != 0) {
                std::swap(L.rows_term[r], L.rows_term[r + 1]);
                L.pair_next[r] = 1;
                ++r;
            }
        }
        L.chunk_off.assign(1, 0);
        // a tree with at most two chunks' worth of terminals keeps them in one CTA (staging the
        // tables twice costs more than the second CTA gains); GRAD_CHUNK_MAX_TERMS still bounds it
        int chunk = grad_chunk_terms(G.n_games);
        const int n_terms = (int)L.term_idx.size();
        if (n_terms <= 2 * chunk && n_terms <= GRAD_CHUNK_MAX_TERMS) chunk = n_terms;
        for (int r = 0, n = 0; r < (int)L.rows_term.size(); ++r) {
            const int s = L.rows_term[r];
            n += L.term_off[s + 1] - L.term_off[s];
            if ((n >= chunk && !L.pair_next[r]) || r + 1 == (int)L.rows_term.size()) {
                L.chunk_off.push_back(r + 1);
                n = 0;
            }
        }
        const int nn = (int)L.first.size();
        L.lvl_off.assign(L.depth + 1, 0);
        L.lvl_nodes.clear();
        for (int l = 0; l < L.depth; ++l) {
            L.lvl_off[l] = (int)L.lvl_nodes.size();
            for (int m = 0; m < nn; ++m)
                if (L.level[m] == l) L.lvl_nodes.push_back(m);
        }
        L.lvl_off[L.depth] = (int)L.lvl_nodes.size();
        std::vector<std::vector<int>> kid(L.n_pub);
        for (int m = 0; m < nn; ++m) kid[L.parent_seq[m]].push_back(m);
        L.kid_off.assign(L.n_pub + 1, 0);
        L.kids.clear();
        for (int s = 0; s < L.n_pub; ++s) {
            L.kid_off[s] = (int)L.kids.size();
            for (int m : kid[s]) L.kids.push_back(m);
        }
        L.kid_off[L.n_pub] = (int)L.kids.size();
        // warp schedule per level: groups of nodes with a common (non-empty) parent sequence,
        // largest first onto the least-loaded warp (load = actions)
        L.sched_off.assign((size_t)L.depth * TREE_WARPS + 1, 0);
        L.sched_nodes.clear();
        L.root_slot.assign(nn, -1);
        L.n_root = 0;
        for (int m = 0; m < nn; ++m)
            if (L.parent_seq[m] == 0) L.root_slot[m] = L.n_root++;
        for (int l = 0; l < L.depth; ++l) {
            std::vector<std::vector<int>> groups;
            std::vector<int> gid(L.n_pub, -1);
            for (int idx = L.lvl_off[l]; idx < L.lvl_off[l + 1]; ++idx) {
                const int m = L.lvl_nodes[idx], par = L.parent_seq[m];
                if (par == 0) {
                    groups.push_back({m});
                } else {
                    if (gid[par] < 0) {
                        gid[par] = (int)groups.size();
                        groups.push_back({});
                    }
                    groups[gid[par]].push_back(m);
                }
            }
            auto load = [&](const std::vector<int>& gr) {
                int a = 0;
                for (int m : gr) a += L.nact[m];
                return a;
            };
            std::stable_sort(groups.begin(), groups.end(),
                             [&](const std::vector<int>& a, const std::vector<int>& b) { return load(a) > load(b); });
            std::vector<std::vector<int>> per(TREE_WARPS);
            std::vector<int> wl(TREE_WARPS, 0);
            for (const auto& gr : groups) {
                const int w = (int)(std::min_element(wl.begin(), wl.end()) - wl.begin());
                wl[w] += load(gr);
                for (int m : gr) per[w].push_back(m);
            }
            for (int w = 0; w < TREE_WARPS; ++w) {
                L.sched_off[(size_t)l * TREE_WARPS + w] = (int)L.sched_nodes.size();
                for (int m : per[w]) L.sched_nodes.push_back(m);
            }
        }
        L.sched_off[(size_t)L.depth * TREE_WARPS] = (int)L.sched_nodes.size();
        L.seq_slot.assign(L.n_pub, -1);
        L.n_int = 0;
        for (int s = 0; s < L.n_pub; ++s)
            if (L.kid_off[s + 1] > L.kid_off[s]) L.seq_slot[s] = L.n_int++;
    }
}

static int combo_index(int c1, int c2, int n) {
    // canonical order of (c1 < c2) pairs, lexicographic
    return c1 * (2 * n - c1 - 1) / 2 + (c2 - c1 - 1);
}

// strength key of internal hand h for board state bs of game g (only for valid hands)
static int64_t strength_of(const HostGame& G, int g, int bs, int h, const std::vector<int>& board) {
    const int* hc = &G.hand_cards[((size_t)g * G.H + h) * 2];
    if (G.kind == EGT_GAME_KUHN) return hc[0];
    if (G.kind == EGT_GAME_LEDUC) {
        if (board.empty()) return hc[0] / 2;
        int r = hc[0] / 2, b = board[0] / 2;
        return r == b ? 10 + r : r;
    }
    (void)board;
    return G.strength[(size_t)g * G.H + h];  // river: computed once while ordering the hands
}

static std::vector<int> board_of(const HostGame& G, const std::vector<std::vector<int>>& game_boards, int g, int bs) {
    if (G.kind == EGT_GAME_RIVER) return game_boards[g];
    return G.tree.board_cards[bs];
}

static void build_card_plan(const HostGame& G, const std::vector<std::vector<int>>& by_card,
                            const std::vector<int16_t>& lo, const std::vector<std::array<int, 2>>& cards_of_pos,
                            int nv, CardPlan& plan);

static void build_table(const HostGame& G, int g, int bs, const std::vector<int>& board, BoardTable& tb) {
    const int H = G.H, Hp = G.H_pad, hs = G.hand_size;
    tb.valid.assign(Hp, 0);
    std::vector<std::pair<int64_t, int>> v;
    for (int h = 0; h < H; ++h) {
        const int* hc = &G.hand_cards[((size_t)g * H + h) * 2];
        bool ok = true;
        for (int k = 0; k < hs; ++k)
            for (int c : board) ok = ok && hc[k] != c;
        if (!ok) continue;
        tb.valid[h] = 1;
        v.push_back({strength_of(G, g, bs, h, board), h});
    }
    std::sort(v.begin(), v.end());  // (strength, hand) ascending: ties by hand index
    int nv = (int)v.size();
    tb.nvalid = nv;
    tb.order.assign(Hp, 0);
    tb.lo.assign(Hp, 0);
    tb.hi.assign(Hp, 0);
    tb.lohi.assign(Hp, 0);
    for (int i = 0; i < nv; ++i) tb.order[i] = (int16_t)v[i].second;
    for (int h = 0, i = nv; h < H; ++h)
        if (!tb.valid[h]) tb.order[i++] = (int16_t)h;  // blocked hands after the valid ones
    for (int i = 0; i < nv;) {
        int j = i;
        while (j < nv && v[j].first == v[i].first) ++j;
        for (int k = i; k < j; ++k) {
            tb.lo[k] = (int16_t)i;
            tb.hi[k] = (int16_t)j;
            tb.lohi[k] = (uint32_t)i | ((uint32_t)j << 16);
        }
        i = j;
    }
    // card array: for each card, the sorted positions of the valid hands holding it + an end slot
    std::vector<std::vector<int>> by_card(G.n_cards);
    for (int i = 0; i < nv; ++i) {
        const int* hc = &G.hand_cards[((size_t)g * H + v[i].second) * 2];
        for (int k = 0; k < hs; ++k) by_card[hc[k]].push_back(i);
    }
    // uniform segments: card c owns slots [c * seg_w, (c + 1) * seg_w); its hands first, then
    // padding, the end slot last
    const int W = G.seg_w;
    tb.cent.assign((size_t)G.n_ce, (uint16_t)CE_END);
    tb.pcard.assign(2 * (size_t)Hp, 0);
    for (int c = 0; c < G.n_cards; ++c) {
        const std::vector<int>& L = by_card[c];
        const int start = c * W, len = (int)L.size();
        for (int j = 0; j < len; ++j) {
            const int i = L[j];
            tb.cent[start + j] = (uint16_t)i;
            const int relo = (int)(std::lower_bound(L.begin(), L.end(), (int)tb.lo[i]) - L.begin());
            const int rehi = (int)(std::lower_bound(L.begin(), L.end(), (int)tb.hi[i]) - L.begin());
            const int* hc = &G.hand_cards[((size_t)g * H + v[i].second) * 2];
            const int k = (hs == 2 && hc[1] == c) ? 1 : 0;
            tb.pcard[2 * (size_t)i + k] = PC_PACK(start, relo, rehi, W - 1);
        }
        tb.cent[start] |= (uint16_t)CE_FIRST;
    }
    // river boards: the card-domain gradient kernel's conflict-free exchange plan
    if (hs == 2 && G.n_cards <= CARD_NT / CARD_GL && G.n_cards - 6 <= CARD_GL * CARD_CH && nv <= CARD_NP &&
        G.kind == EGT_GAME_RIVER) {
        std::vector<std::array<int, 2>> cp(nv);
        for (int i = 0; i < nv; ++i) {
            const int* hc = &G.hand_cards[((size_t)g * H + v[i].second) * 2];
            cp[i] = {std::min(hc[0], hc[1]), std::max(hc[0], hc[1])};
        }
        build_card_plan(G, by_card, tb.lo, cp, nv, tb.plan);
        CardPlan& pl = tb.plan;
        pl.tab.assign(CARD_TAB_WORDS, 0u);
        std::copy(pl.pw.begin(), pl.pw.end(), pl.tab.begin() + CARD_TAB_PW);
        std::copy(pl.pr.begin(), pl.pr.end(), pl.tab.begin() + CARD_TAB_PR);
        for (int i = 0; i < nv; ++i) pl.tab[CARD_TAB_LOHI + i] = tb.lohi[i];
        std::copy(pl.lane.begin(), pl.lane.end(), pl.tab.begin() + CARD_TAB_LANE);
    }
}

// Proper edge colouring of a bipartite multigraph with max degree <= 16 in 16 colours
// (alternating-path method; exists by Koenig's theorem).  edges[k] = (left, right).
static std::vector<int> colour_edges16(int n_left, int n_right, const std::vector<std::pair<int, int>>& edges) {
    constexpr int C = 16;
    std::vector<int> at_l((size_t)n_left * C, -1), at_r((size_t)n_right * C, -1), col(edges.size(), -1);
    std::vector<uint32_t> used_l(n_left, 0u), used_r(n_right, 0u);  // colours in use at a vertex
    std::vector<int> path;
    auto set = [&](int e, int c) {
        col[e] = c;
        at_l[(size_t)edges[e].first * C + c] = e;
        at_r[(size_t)edges[e].second * C + c] = e;
        used_l[edges[e].first] |= 1u << c;
        used_r[edges[e].second] |= 1u << c;
    };
    for (size_t k = 0; k < edges.size(); ++k) {
        const int u = edges[k].first, v = edges[k].second;
        const uint32_t both = ~(used_l[u] | used_r[v]) & 0xFFFFu;
        if (both) {  // a colour free at both ends: no recolouring
            set((int)k, __builtin_ctz(both));
            continue;
        }
        const uint32_t fl = ~used_l[u] & 0xFFFFu, fr = ~used_r[v] & 0xFFFFu;
        if (!fl || !fr) throw std::runtime_error("edge colouring: degree above 16");
        const int a = __builtin_ctz(fl), b = __builtin_ctz(fr);
        // a is taken at v: swap a and b along the alternating path that starts at v with colour
        // a (it cannot reach u, where a is free), freeing a at v
        path.clear();
        int x = v, side = 1, c = a;
        while (true) {
            const int e = side ? at_r[(size_t)x * C + c] : at_l[(size_t)x * C + c];
            if (e < 0) break;
            path.push_back(e);
            x = side ? edges[e].first : edges[e].second;
            side ^= 1;
            c = c == a ? b : a;
        }
        for (int e : path) {
            at_l[(size_t)edges[e].first * C + col[e]] = -1;
            at_r[(size_t)edges[e].second * C + col[e]] = -1;
            used_l[edges[e].first] &= ~(1u << col[e]);
            used_r[edges[e].second] &= ~(1u << col[e]);
        }
        for (int e : path) set(e, col[e] == a ? b : a);
        set((int)k, a);
    }
    return col;
}

// addresses of a colouring: colour c, m-th edge of that colour -> 16 m + c
static std::vector<int> colour_addresses(const std::vector<int>& col) {
    std::vector<int> cnt(16, 0), addr(col.size());
    for (size_t k = 0; k < col.size(); ++k) addr[k] = 16 * cnt[col[k]]++ + col[k];
    return addr;
}

// The conflict-free plan of grad_card_kernel for one river board (see CardPlan in game.h).
// by_card[c]: positions holding card c in strength order; lo[i]: tie group start of position i.
static void build_card_plan(const HostGame& G, const std::vector<std::vector<int>>& by_card,
                            const std::vector<int16_t>& lo, const std::vector<std::array<int, 2>>& cards_of_pos,
                            int nv, CardPlan& plan) {
    const int NT = CARD_NT, K = CARD_K, GLN = CARD_GL, CH = CARD_CH, NP = CARD_NP;
    // slot (c, k) -> thread, slot index; the card index (0: lower card of its hand)
    struct Slot { int c, k, pos, which, thread, s; };
    std::vector<Slot> slots;
    std::vector<std::array<int, 2>> slot_of_pos(nv, {-1, -1});
    for (int c = 0; c < G.n_cards; ++c)
        for (int k = 0; k < (int)by_card[c].size(); ++k) {
            const int i = by_card[c][k];
            const int which = cards_of_pos[i][0] == c ? 0 : 1;
            slot_of_pos[i][which] = (int)slots.size();
            slots.push_back({c, k, i, which, c * GLN + k / CH, k % CH});
        }
    // w1 / w2: left = position-lane write groups (array, half-warp, j), right = slot-lane read
    // groups (half-warp, s) -- one colouring for both arrays, since a read group mixes them
    const int n_wg = (NT / 16) * K, n_rg = (NT / 16) * CH;
    std::vector<int> waddr[2];
    {
        std::vector<std::pair<int, int>> e(2 * (size_t)nv);
        for (int a = 0; a < 2; ++a)
            for (int i = 0; i < nv; ++i) {
                const Slot& sl = slots[slot_of_pos[i][a]];
                e[(size_t)a * nv + i] = {a * n_wg + (i / K / 16) * K + i % K, (sl.thread / 16) * CH + sl.s};
            }
        const std::vector<int> col = colour_edges16(2 * n_wg, n_rg, e);
        for (int a = 0; a < 2; ++a)
            waddr[a] = colour_addresses(std::vector<int>(col.begin() + (size_t)a * nv, col.begin() + (size_t)(a + 1) * nv));
    }
    // ex: left = slot-lane write groups (half-warp, s), right = position-lane read groups (half-warp, j, card)
    std::vector<std::pair<int, int>> e(slots.size());
    for (size_t q = 0; q < slots.size(); ++q) {
        const int i = slots[q].pos;
        e[q] = {(slots[q].thread / 16) * CH + slots[q].s, ((i / K / 16) * K + i % K) * 2 + slots[q].which};
    }
    const std::vector<int> xcol = colour_edges16(n_rg, n_wg * 2, e);
    const std::vector<int> xaddr = colour_addresses(xcol);
    // padding slots also store (unconditionally): each gets a colour free in its write group and
    // a fresh address of that colour, never read
    std::vector<int> ccount(16, 0);
    for (size_t q = 0; q < slots.size(); ++q) ccount[xcol[q]] = std::max(ccount[xcol[q]], xaddr[q] / 16 + 1);
    std::vector<std::vector<char>> used((size_t)n_rg, std::vector<char>(16, 0));
    for (size_t q = 0; q < slots.size(); ++q) used[(slots[q].thread / 16) * CH + slots[q].s][xcol[q]] = 1;
    std::vector<int> pad_addr((size_t)NT * CH, -1);
    for (int t = 0; t < NT; ++t)
        for (int s2 = 0; s2 < CH; ++s2) {
            const int c = t / GLN, k = (t % GLN) * CH + s2;
            if (c < G.n_cards && k < (int)by_card[c].size()) continue;
            std::vector<char>& u = used[(t / 16) * CH + s2];
            int col = 0;
            while (col < 16 && u[col]) ++col;
            if (col == 16) throw std::runtime_error("card plan: no free colour for a padding slot");
            u[col] = 1;
            pad_addr[(size_t)t * CH + s2] = 16 * ccount[col]++ + col;
        }
    for (int col = 0; col < 16; ++col)
        if (16 * ccount[col] > CARD_EX) throw std::runtime_error("card plan: ex exchange region too small");
    // w region: w1 [0, NP), w2 [NP, 2 NP), then 16 zero cells, one per bank pair (2 NP is a
    // multiple of 16): the padding slots of a read group gather from the zero cell of a bank
    // pair no real slot of the group reads, so they never conflict (padding lanes of one group
    // share that cell: a broadcast)
    const int zero_cell = 2 * NP;
    std::vector<uint32_t> group_used((size_t)n_rg, 0u);
    for (size_t q = 0; q < slots.size(); ++q)
        group_used[(size_t)(slots[q].thread / 16) * CH + slots[q].s] |=
            1u << ((waddr[slots[q].which][slots[q].pos] + slots[q].which * NP) % 16);
    plan.pw.assign(NP, 0u);
    plan.pr.assign(NP, 0u);
    for (int i = 0; i < nv; ++i) {
        plan.pw[i] = (uint32_t)(waddr[0][i] * 8) | ((uint32_t)((NP + waddr[1][i]) * 8) << 16);
        plan.pr[i] = (uint32_t)xaddr[slot_of_pos[i][0]] | ((uint32_t)xaddr[slot_of_pos[i][1]] << 16);
    }
    plan.lane.assign((size_t)NT * 8, 0u);
    for (int t = 0; t < NT; ++t) {
        uint32_t* L = &plan.lane[(size_t)t * 8];
        for (int s = 0; s < CH; ++s) {
            const uint32_t used = group_used[(size_t)(t / 16) * CH + s];
            int free_col = 0;
            while (free_col < 16 && ((used >> free_col) & 1u)) ++free_col;
            const uint32_t z = (uint32_t)((zero_cell + (free_col & 15)) * 8);
            L[s / 2] |= (s & 1) ? z << 16 : z;
            const int pa = pad_addr[(size_t)t * CH + s];
            if (pa >= 0) L[3 + s / 2] |= (s & 1) ? (uint32_t)pa << 16 : (uint32_t)pa;
        }
    }
    // per segment: run heads / tails (tie-group changes inside the card's strength-ordered
    // list) and, per lane, the lanes that hold the run open at its chunk's start / end
    for (int c = 0; c < G.n_cards; ++c) {
        const std::vector<int>& Lc = by_card[c];
        const int len = (int)Lc.size();
        std::vector<int> head(len), tail(len);
        for (int k = 0; k < len; ++k) {
            head[k] = k == 0 || lo[Lc[k]] != lo[Lc[k - 1]];
            tail[k] = k == len - 1 || lo[Lc[k]] != lo[Lc[k + 1]];
        }
        for (int part = 0; part < GLN; ++part) {
            const int t = c * GLN + part;
            uint32_t* L = &plan.lane[(size_t)t * 8];
            uint32_t flags = 0;
            for (int s = 0; s < CH; ++s) {
                const int k = part * CH + s;
                if (k >= len) continue;
                const int q = slot_of_pos[Lc[k]][cards_of_pos[Lc[k]][0] == c ? 0 : 1];
                const uint32_t g = (uint32_t)(waddr[slots[q].which][Lc[k]] + slots[q].which * NP) * 8;
                L[s / 2] = (s & 1) ? ((L[s / 2] & 0xFFFFu) | (g << 16)) : ((L[s / 2] & 0xFFFF0000u) | g);
                L[3 + s / 2] |= (s & 1) ? (uint32_t)xaddr[q] << 16 : (uint32_t)xaddr[q];
                flags |= 1u << s;
                if (head[k]) flags |= 1u << (6 + s);
                if (tail[k]) flags |= 1u << (12 + s);
            }
            L[6] = flags;
            // src_lo: the nearest lane before this one (same segment) with a run head; src_hi:
            // the nearest lane after it with a run tail (absolute lane indices in the warp)
            int src_lo = t, src_hi = t;
            for (int q = part - 1; q >= 0 && src_lo == t; --q)
                for (int s = 0; s < CH; ++s)
                    if (q * CH + s < len && head[q * CH + s]) src_lo = c * GLN + q;
            for (int q = part + 1; q < GLN && src_hi == t; ++q)
                for (int s = 0; s < CH; ++s)
                    if (q * CH + s < len && tail[q * CH + s]) { src_hi = c * GLN + q; break; }
            L[7] = (uint32_t)(src_lo & 31) | ((uint32_t)(src_hi & 31) << 8);
        }
    }
}

// Runs f(g) for every game on the host's cores (games are independent); first error wins.
template <class F>
static std::string parallel_games(int n, F&& f) {
    const int nt = std::max(1, std::min<int>(n, (int)std::thread::hardware_concurrency()));
    std::vector<std::string> errs(nt);
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int g = t; g < n; g += nt) {
                std::string e = f(g);
                if (!e.empty() && errs[t].empty()) errs[t] = e;
            }
        });
    for (auto& x : th) x.join();
    for (auto& e : errs)
        if (!e.empty()) return e;
    return "";
}

std::string build_host_game(const egt_game_spec& spec, HostGame& G) {
    G = HostGame();
    if (spec.n_games < 1) return "n_games must be >= 1";
    G.kind = spec.kind;
    G.n_games = spec.n_games;
    std::vector<std::vector<int>> game_boards;
    if (spec.kind == EGT_GAME_KUHN) {
        build_kuhn(G.tree);
        G.H = 3; G.hand_size = 1; G.n_cards = 3; G.n_combos = 3;
    } else if (spec.kind == EGT_GAME_LEDUC) {
        build_leduc(G.tree);
        G.H = 6; G.hand_size = 1; G.n_cards = 6; G.n_combos = 6;
    } else if (spec.kind == EGT_GAME_RIVER) {
        if (spec.n_ranks < 2 || spec.n_ranks > 13 || spec.n_suits < 1 || spec.n_suits > 4)
            return "invalid deck";
        G.n_ranks = spec.n_ranks; G.n_suits = spec.n_suits;
        G.n_cards = spec.n_ranks * spec.n_suits;
        if (G.n_cards < 9) return "deck too small for a 5-card board and two hands";
        if (!spec.boards) return "river games need boards";
        if (spec.pot < 2 || spec.stack < 1) return "invalid pot/stack";
        RiverRules R;
        R.pot = spec.pot; R.stack = spec.stack; R.cap = spec.raise_cap; R.open_fold = spec.open_fold != 0;
        for (int c = 0; c < EGT_N_CTX; ++c) {
            if (spec.n_fracs[c] < 0 || spec.n_fracs[c] > EGT_MAX_FRACS) return "invalid n_fracs";
            for (int i = 0; i < spec.n_fracs[c]; ++i) {
                if (spec.frac_num[c][i] <= 0 || spec.frac_den[c][i] <= 0) return "fractions must be positive";
                R.fr[c].push_back({spec.frac_num[c][i], spec.frac_den[c][i]});
            }
            R.allin[c] = spec.allin[c] != 0;
        }
        G.tree.n_board_states = 1;
        G.tree.board_cards = {{}};
        build_river_rec(G.tree, R, 0, 0, 0, 0, "");
        game_boards.resize(spec.n_games);
        for (int g = 0; g < spec.n_games; ++g) {
            std::set<int> seen;
            for (int k = 0; k < 5; ++k) {
                int c = spec.boards[g * 5 + k];
                if (c < 0 || c >= G.n_cards || seen.count(c)) return "invalid board";
                seen.insert(c);
                game_boards[g].push_back(c);
            }
        }
        G.hand_size = 2;
        G.n_combos = G.n_cards * (G.n_cards - 1) / 2;
        G.H = G.n_combos - (5 * (G.n_cards - 5) + 10);  // combos avoiding 5 board cards
    } else {
        return "unknown game kind";
    }
    G.H_pad = (G.H + 31) / 32 * 32;
    if (G.H > EGT_MAX_HANDS) return "too many private hands for the gradient kernel";
    // card segments: at most (n_cards - 6) valid river hands hold a card; one hand per card otherwise
    G.seg_w = (G.hand_size == 2 ? G.n_cards - 6 : 1) + 1;
    G.n_ce = (G.n_cards * G.seg_w + 7) / 8 * 8;
    if (G.n_cards - 5 - 1 > 63 && G.kind == EGT_GAME_RIVER) return "deck too large (card segments > 63)";
    build_layout(G);
    const int Gn = G.n_games, H = G.H, Hp = G.H_pad;

    // hands (internal order) and priors
    G.hand_cards.assign((size_t)Gn * H * 2, -1);
    G.hand_combo.assign((size_t)Gn * H, 0);
    G.strength.assign((size_t)Gn * H, 0);
    for (int p = 0; p < 2; ++p) G.prior[p].assign((size_t)Gn * Hp, 0.0);
    G.kappa_game.assign(Gn, 1.0);
    auto per_game = [&](int g) -> std::string {
        if (G.kind != EGT_GAME_RIVER) {
            for (int h = 0; h < H; ++h) {
                G.hand_cards[((size_t)g * H + h) * 2] = h;
                G.hand_combo[(size_t)g * H + h] = h;
                G.prior[0][(size_t)g * Hp + h] = 1.0;
                G.prior[1][(size_t)g * Hp + h] = 1.0;
            }
            return "";
        }
        const std::vector<int>& bd = game_boards[g];
        std::vector<std::pair<int64_t, int>> hv;  // (strength, combo)
        std::vector<std::pair<int, int>> cards;
        // A hand's strength depends only on its two ranks and on whether each hole card has the
        // board's flush suit (the one suit with >= 3 board cards; with none, no flush exists):
        // one evaluation per such key, shared by every hand that has it.
        int fs = -1, scnt[4] = {0, 0, 0, 0};
        for (int c : bd) scnt[c % G.n_suits]++;
        for (int su = 0; su < G.n_suits; ++su)
            if (scnt[su] >= 3) fs = su;
        std::vector<int64_t> memo(13 * 13 * 4, -1);
        for (int c1 = 0; c1 < G.n_cards; ++c1)
            for (int c2 = c1 + 1; c2 < G.n_cards; ++c2) {
                if (std::find(bd.begin(), bd.end(), c1) != bd.end() ||
                    std::find(bd.begin(), bd.end(), c2) != bd.end()) continue;
                int ranks[7], suits[7], n = 0;
                ranks[n] = 13 - G.n_ranks + c1 / G.n_suits; suits[n++] = c1 % G.n_suits;
                ranks[n] = 13 - G.n_ranks + c2 / G.n_suits; suits[n++] = c2 % G.n_suits;
                const int key = ((ranks[0] * 13 + ranks[1]) * 2 + (suits[0] == fs)) * 2 + (suits[1] == fs);
                if (memo[key] < 0) {
                    for (int c : bd) { ranks[n] = 13 - G.n_ranks + c / G.n_suits; suits[n++] = c % G.n_suits; }
                    memo[key] = hand_strength(ranks, suits, n);
                }
                hv.push_back({memo[key], combo_index(c1, c2, G.n_cards)});
            }
        if ((int)hv.size() != H) return "internal: hand count";
        std::sort(hv.begin(), hv.end());
        std::vector<std::pair<int, int>> combo_cards(G.n_combos);
        for (int c1 = 0, k = 0; c1 < G.n_cards; ++c1)
            for (int c2 = c1 + 1; c2 < G.n_cards; ++c2, ++k) combo_cards[k] = {c1, c2};
        for (int h = 0; h < H; ++h) {
            int ci = hv[h].second;
            G.strength[(size_t)g * H + h] = hv[h].first;
            G.hand_combo[(size_t)g * H + h] = ci;
            G.hand_cards[((size_t)g * H + h) * 2] = combo_cards[ci].first;
            G.hand_cards[((size_t)g * H + h) * 2 + 1] = combo_cards[ci].second;
            for (int p = 0; p < 2; ++p) {
                const double* pr = p == 0 ? spec.prior1 : spec.prior2;
                double w = pr ? pr[(size_t)g * G.n_combos + ci] : 1.0;
                if (!(w >= 0) || !std::isfinite(w)) return "priors must be finite and >= 0";
                G.prior[p][(size_t)g * Hp + h] = w;
            }
        }
        // Z = sum over disjoint (h1, h2) of prior1 prior2 (inclusion-exclusion over shared cards)
        std::vector<double> card_sum(G.n_cards, 0.0);
        double T2 = 0;
        for (int h = 0; h < H; ++h) {
            double w = G.prior[1][(size_t)g * Hp + h];
            T2 += w;
            card_sum[G.hand_cards[((size_t)g * H + h) * 2]] += w;
            card_sum[G.hand_cards[((size_t)g * H + h) * 2 + 1]] += w;
        }
        double Z = 0;
        for (int h = 0; h < H; ++h) {
            const int* hc = &G.hand_cards[((size_t)g * H + h) * 2];
            double compat = T2 - card_sum[hc[0]] - card_sum[hc[1]] + G.prior[1][(size_t)g * Hp + h];
            Z += G.prior[0][(size_t)g * Hp + h] * compat;
        }
        if (!(Z > 0)) return "priors leave no compatible hand pair";
        G.kappa_game[g] = 1.0 / Z;
        return "";
    };
    std::string err = parallel_games(Gn, per_game);
    if (!err.empty()) return err;

    // tables per (game, board state)
    const int nbs = G.tree.n_board_states;
    G.tables.resize((size_t)Gn * nbs);
    parallel_games(Gn, [&](int g) -> std::string {
        for (int bs = 0; bs < nbs; ++bs)
            build_table(G, g, bs, board_of(G, game_boards, g, bs), G.tables[(size_t)g * nbs + bs]);
        return "";
    });
    G.all_valid = 1;
    for (const BoardTable& tb : G.tables)
        if (tb.nvalid != H) G.all_valid = 0;

    // beta and M per (node, hand), validity of game 0
    // (identical across games: river hands all avoid their board; Kuhn/Leduc games are equal)
    for (int p = 0; p < 2; ++p) {
        const PlayerLayout& L = G.pl[p];
        int nn = (int)L.first.size();
        std::vector<std::vector<int>> kids(L.n_pub);
        for (int m = 0; m < nn; ++m) kids[L.parent_seq[m]].push_back(m);
        G.beta[p].assign((size_t)nn * Hp, 0.0);
        std::vector<double> f((size_t)nn * Hp, 0.0);
        G.M[p].assign(Gn, 0.0);
        for (int m = nn - 1; m >= 0; --m) {
            const BoardTable& tb = G.tables[L.board_state[m]];
            for (int h = 0; h < H; ++h) {
                if (!tb.valid[h]) continue;
                double b = 2.0, fbest = 0.0;
                for (int a = 0; a < L.nact[m]; ++a) {
                    double fs = 0.0;
                    for (int c : kids[L.first[m] + a]) {
                        if (!G.tables[L.board_state[c]].valid[h]) continue;
                        b += 2.0 * G.beta[p][(size_t)c * Hp + h];
                        fs += f[(size_t)c * Hp + h];
                    }
                    fbest = std::max(fbest, fs);
                }
                G.beta[p][(size_t)m * Hp + h] = b;
                f[(size_t)m * Hp + h] = 1.0 + fbest;
            }
        }
        double M = 0;
        for (int m : kids[0])
            for (int h = 0; h < H; ++h) M += f[(size_t)m * Hp + h];
        for (int g = 0; g < Gn; ++g) G.M[p][g] = M;
    }

    return "";
}


// ||A|| = max |A_ij| of game g (R7); only the theory mu needs it.
// Per board state: the largest prior product over compatible pairs (fold blocks) and over
// compatible non-tied pairs (showdown blocks) -- for each hand a, the player-2 hands in
// descending prior order are scanned until the first admissible partner (a hand blocks at
// most 2 * 46 others, so the scan is short); terminals whose player-1 (-2) sequence is
// empty aggregate their block's columns (rows) into row (column) 0, computed with the
// same card-removal sums as the gradient (O(H) per terminal).
std::vector<double> compute_max_abs_A_all(const HostGame& G) {
    std::vector<double> out(G.n_games, 0.0);
    parallel_games(G.n_games, [&](int g) -> std::string {
        out[g] = compute_max_abs_A(G, g);
        return "";
    });
    return out;
}

double compute_max_abs_A(const HostGame& G, int g) {
    const int H = G.H, Hp = G.H_pad, nbs = G.tree.n_board_states, hs = G.hand_size;
    const double* pr[2] = {&G.prior[0][(size_t)g * Hp], &G.prior[1][(size_t)g * Hp]};
    const int* hc = &G.hand_cards[(size_t)g * H * 2];
    auto compat = [&](int a, int b) {
        for (int i = 0; i < hs; ++i)
            for (int j = 0; j < hs; ++j)
                if (hc[2 * a + i] == hc[2 * b + j]) return false;
        return true;
    };
    std::vector<int> desc2(H);
    std::iota(desc2.begin(), desc2.end(), 0);
    std::sort(desc2.begin(), desc2.end(), [&](int x, int y) { return pr[1][x] > pr[1][y]; });
    double best = 0.0;
    for (int bs = 0; bs < nbs; ++bs) {
        const BoardTable& tb = G.tables[(size_t)g * nbs + bs];
        std::vector<int> grp(H, -1);
        for (int i = 0; i < tb.nvalid; ++i) grp[tb.order[i]] = tb.lo[i];
        // max prior products over admissible pairs
        double pmax_fold = 0.0, pmax_sd = 0.0;
        for (int a = 0; a < H; ++a) {
            if (!tb.valid[a] || pr[0][a] == 0.0) continue;
            bool got_f = false, got_s = false;
            for (int k = 0; k < H && !(got_f && got_s); ++k) {
                const int b = desc2[k];
                if (!tb.valid[b] || !compat(a, b)) continue;
                if (!got_f) {
                    pmax_fold = std::max(pmax_fold, pr[0][a] * pr[1][b]);
                    got_f = true;
                }
                if (!got_s && grp[b] != grp[a]) {
                    pmax_sd = std::max(pmax_sd, pr[0][a] * pr[1][b]);
                    got_s = true;
                }
            }
        }
        // aggregated rows / columns: for each hand of the non-empty side, the signed sum over
        // the compatible hands of the empty side (fold: all, showdown: stronger - weaker)
        auto agg_max = [&](int side, bool sd) {
            // side = the player whose sequence is non-empty (its hands index the aggregate)
            const double* ps = pr[side];
            const double* po = pr[1 - side];
            std::vector<double> w(tb.nvalid), P(tb.nvalid + 1, 0.0);
            std::vector<std::vector<double>> cardP(G.n_cards);  // prefix sums per card, strength order
            std::vector<std::vector<int>> cardPos(G.n_cards);
            for (int i = 0; i < tb.nvalid; ++i) {
                const int h = tb.order[i];
                w[i] = po[h];
                P[i + 1] = P[i] + w[i];
                for (int k = 0; k < hs; ++k) cardPos[hc[2 * h + k]].push_back(i);
            }
            for (int c = 0; c < G.n_cards; ++c) {
                cardP[c].assign(cardPos[c].size() + 1, 0.0);
                for (size_t j = 0; j < cardPos[c].size(); ++j) cardP[c][j + 1] = cardP[c][j] + w[cardPos[c][j]];
            }
            auto cprefix = [&](int c, int pos) {  // sum of w over hands holding c at positions < pos
                const auto& L = cardPos[c];
                return cardP[c][std::lower_bound(L.begin(), L.end(), pos) - L.begin()];
            };
            double m = 0.0, tot = 0.0;
            const double T = P[tb.nvalid];
            std::vector<double> rowsum(tb.nvalid);
            for (int i = 0; i < tb.nvalid; ++i) {
                const int h = tb.order[i];
                double v;
                if (!sd) {
                    v = T + (hs == 2 ? w[i] : 0.0);
                    for (int k = 0; k < hs; ++k) v -= cardP[hc[2 * h + k]].back();
                } else {
                    const int lo = tb.lo[i], hi = tb.hi[i];
                    double weaker = P[lo], stronger = T - P[hi];
                    for (int k = 0; k < hs; ++k) {
                        const int c = hc[2 * h + k];
                        weaker -= cprefix(c, lo);
                        stronger -= cardP[c].back() - cprefix(c, hi);
                    }
                    // sign of player 2's payoff: + when player 2's hand is stronger
                    v = side == 0 ? stronger - weaker : weaker - stronger;
                }
                rowsum[i] = ps[h] * v;
                m = std::max(m, std::fabs(rowsum[i]));
                tot += rowsum[i];
            }
            return std::make_pair(m, std::fabs(tot));
        };
        for (const Terminal& t : G.terms) {
            if (t.board_state != bs) continue;
            const bool sd = t.kind == T_SHOWDOWN;
            const double scale = t.kappa * G.kappa_game[g] * std::fabs(t.amount);
            const bool e0 = t.last_seq[0] == 0, e1 = t.last_seq[1] == 0;
            double m;
            if (!e0 && !e1) m = sd ? pmax_sd : pmax_fold;
            else if (e0 && e1) m = agg_max(0, sd).second;
            else m = agg_max(e1 ? 0 : 1, sd).first;
            best = std::max(best, scale * m);
        }
    }
    return best;
}

}  // namespace egt
