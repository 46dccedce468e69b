// The card-domain gradient kernel's host plan (game.cpp build_card_plan) on random river boards:
//  * every shared-memory exchange is bank-conflict free per half-warp (distinct 8-byte bank
//    pairs among the lanes of a half-warp in each instruction),
//  * the exchanges deliver the right values (each slot reads its hand's weight, each position
//    reads the card parts of its own two slots),
//  * the run heads / tails and source lanes reproduce the segment prefixes at the start and end
//    of every slot's tie run (computed here by brute force).
// Prints "violations N"; exit 1 on any.
#include "game.h"
#include <array>
#include <cstdio>
#include <cstring>
#include <map>
#include <random>
#include <set>
using namespace egt;
static long long viol = 0;
static void fail(const char* what, int g, int a, int b) {
    if (viol++ < 10) std::printf("violation: %s (game %d, %d, %d)\n", what, g, a, b);
}
int main(int argc, char** argv) {
    const int n_games = argc > 1 ? std::atoi(argv[1]) : 24;
    std::mt19937 rng(12345);
    std::vector<int32_t> boards;
    for (int g = 0; g < n_games; ++g) {
        std::set<int> b;
        while ((int)b.size() < 5) b.insert((int)(rng() % 52));
        if (g == 0) b = {48, 44, 40, 36, 32};  // royal flush board: every hand ties
        for (int c : b) boards.push_back(c);
    }
    egt_game_spec sp;
    std::memset(&sp, 0, sizeof(sp));
    sp.kind = EGT_GAME_RIVER;
    sp.n_games = n_games;
    sp.pot = 2100;
    sp.stack = 18950;
    sp.open_fold = 1;
    for (int c = 0; c < EGT_N_CTX; ++c) {
        sp.n_fracs[c] = 1;
        sp.frac_num[c][0] = 1;
        sp.frac_den[c][0] = 1;
        sp.allin[c] = 1;
    }
    sp.n_ranks = 13;
    sp.n_suits = 4;
    sp.boards = boards.data();
    HostGame G;
    std::string err = build_host_game(sp, G);
    if (!err.empty()) {
        std::printf("build error: %s\n", err.c_str());
        return 1;
    }
    const int NT = CARD_NT, K = CARD_K, CH = CARD_CH, NP = CARD_NP;
    for (int g = 0; g < n_games; ++g) {
        const BoardTable& tb = G.tables[g];
        const CardPlan& pl = tb.plan;
        if (pl.pw.size() != (size_t)NP || pl.lane.size() != (size_t)NT * 8 || pl.tab.size() != (size_t)CARD_TAB_WORDS) {
            fail("no plan", g, 0, 0);
            continue;
        }
        for (int i = 0; i < NP; ++i)
            if (pl.tab[CARD_TAB_PW + i] != pl.pw[i] || pl.tab[CARD_TAB_PR + i] != pl.pr[i] ||
                (i < G.H && pl.tab[CARD_TAB_LOHI + i] != tb.lohi[i]))
                fail("flat table", g, i, 0);
        for (int i = 0; i < NT * 8; ++i)
            if (pl.tab[CARD_TAB_LANE + i] != pl.lane[i]) fail("flat lane table", g, i, 0);
        const int H = G.H;
        // positions -> cards (lower, higher)
        std::vector<std::array<int, 2>> cards(H);
        for (int i = 0; i < H; ++i) {
            const int* hc = &G.hand_cards[((size_t)g * H + tb.order[i]) * 2];
            cards[i] = {std::min(hc[0], hc[1]), std::max(hc[0], hc[1])};
        }
        // w exchange: writes (position lanes), per (half-warp, j) distinct banks per array
        std::vector<double> w(CARD_WREGION, 0.0);
        for (int hw = 0; hw < NT / 16; ++hw)
            for (int j = 0; j < K; ++j)
                for (int a = 0; a < 2; ++a) {
                    std::set<int> banks;
                    for (int l = 0; l < 16; ++l) {
                        const int i = (hw * 16 + l) * K + j;
                        if (i >= H) continue;
                        const unsigned off = a ? pl.pw[i] >> 16 : pl.pw[i] & 0xFFFFu;
                        if (off % 8 || off / 8 >= (unsigned)(2 * NP)) fail("w offset", g, i, a);
                        if (!banks.insert((off / 8) % 16).second) fail("w write conflict", g, hw, j);
                        w[off / 8] = 1.0 + i;
                    }
                }
        // card lanes: gathers, flags, run values
        std::vector<double> wt(H);
        for (int i = 0; i < H; ++i) wt[i] = 0.5 + (double)(rng() % 1000);
        std::vector<int> ex_slot_pos(CARD_EX, -1), ex_slot_card(CARD_EX, -1);
        for (int hw = 0; hw < NT / 16; ++hw)
            for (int s = 0; s < CH; ++s) {
                std::set<int> rbanks, xbanks;
                std::set<unsigned> pad_cell;
                for (int l = 0; l < 16; ++l) {
                    const int t = hw * 16 + l;
                    const uint32_t* L = &pl.lane[(size_t)t * 8];
                    const unsigned cg = (s & 1) ? L[s / 2] >> 16 : L[s / 2] & 0xFFFFu;
                    const bool valid = (L[6] >> s) & 1u;
                    const int c = t / CARD_GL, k = (t % CARD_GL) * CH + s;
                    std::vector<int> hold;
                    for (int i = 0; i < H; ++i)
                        if (c < G.n_cards && (cards[i][0] == c || cards[i][1] == c)) hold.push_back(i);
                    if (valid != (k < (int)hold.size())) { fail("valid flag", g, t, s); continue; }
                    const unsigned px = (s & 1) ? L[3 + s / 2] >> 16 : L[3 + s / 2] & 0xFFFFu;
                    if (px >= (unsigned)CARD_EX) { fail("ex offset", g, t, s); continue; }
                    if (!xbanks.insert(px % 16).second) fail("ex write conflict", g, hw, s);
                    if (ex_slot_pos[px] != -1) fail("ex address shared", g, t, s);
                    if (!valid) {
                        if (cg / 8 < (unsigned)(2 * NP) || cg / 8 >= (unsigned)CARD_WREGION)
                            fail("padding slot not on a zero cell", g, t, s);
                        // padding lanes of a group may share their zero cell (a broadcast), but
                        // no real lane of the group may use its bank pair
                        if (pad_cell.insert(cg / 8).second && !rbanks.insert((cg / 8) % 16).second)
                            fail("w read conflict (zero cell)", g, hw, s);
                        ex_slot_pos[px] = -2;  // a padding slot's private address (never read)
                        continue;
                    }
                    const int i = hold[k];
                    if (w[cg / 8] != 1.0 + i) fail("gather delivers the wrong weight", g, t, s);
                    if (!rbanks.insert((cg / 8) % 16).second) fail("w read conflict", g, hw, s);
                    ex_slot_pos[px] = i;
                    ex_slot_card[px] = c;
                }
            }
        // ex exchange: reads (position lanes), per (half-warp, j, card) distinct banks, own slots
        for (int hw = 0; hw < NT / 16; ++hw)
            for (int j = 0; j < K; ++j)
                for (int a = 0; a < 2; ++a) {
                    std::set<int> banks;
                    for (int l = 0; l < 16; ++l) {
                        const int i = (hw * 16 + l) * K + j;
                        if (i >= H) continue;
                        const unsigned e = a ? pl.pr[i] >> 16 : pl.pr[i] & 0xFFFFu;
                        if (e >= (unsigned)CARD_EX || ex_slot_pos[e] != i || ex_slot_card[e] != cards[i][a])
                            fail("ex read of a wrong slot", g, i, a);
                        if (!banks.insert(e % 16).second) fail("ex read conflict", g, hw, j);
                    }
                }
        // run values: emulate the kernel's register / shuffle computation for every segment
        for (int c = 0; c < G.n_cards; ++c) {
            std::vector<int> hold;
            for (int i = 0; i < H; ++i)
                if (cards[i][0] == c || cards[i][1] == c) hold.push_back(i);
            const int len = (int)hold.size();
            std::vector<double> pre(len + 1, 0.0);
            for (int k = 0; k < len; ++k) pre[k + 1] = pre[k] + wt[hold[k]];
            std::vector<double> ex(CARD_GL * CH), y(CARD_GL * CH, 0.0);
            for (int k = 0; k < len; ++k) y[k] = wt[hold[k]];
            for (int k = 0; k < CARD_GL * CH; ++k) ex[k] = k <= len ? pre[std::min(k, len)] : pre[len];
            std::vector<double> lh(32, 0.0), ft(32, 0.0);
            for (int part = 0; part < CARD_GL; ++part) {
                const int t = c * CARD_GL + part;
                const uint32_t fl = pl.lane[(size_t)t * 8 + 6];
                for (int s = 0; s < CH; ++s)
                    if ((fl >> (6 + s)) & 1u) lh[t & 31] = ex[part * CH + s];
                for (int s = CH - 1; s >= 0; --s)
                    if ((fl >> (12 + s)) & 1u) ft[t & 31] = ex[part * CH + s] + y[part * CH + s];
            }
            for (int part = 0; part < CARD_GL; ++part) {
                const int t = c * CARD_GL + part;
                const uint32_t fl = pl.lane[(size_t)t * 8 + 6], src = pl.lane[(size_t)t * 8 + 7];
                double cur = lh[src & 31u];
                double lo_v[CH], hi_v[CH];
                for (int s = 0; s < CH; ++s) {
                    if ((fl >> (6 + s)) & 1u) cur = ex[part * CH + s];
                    lo_v[s] = cur;
                }
                cur = ft[(src >> 8) & 31u];
                for (int s = CH - 1; s >= 0; --s) {
                    if ((fl >> (12 + s)) & 1u) cur = ex[part * CH + s] + y[part * CH + s];
                    hi_v[s] = cur;
                }
                for (int s = 0; s < CH; ++s) {
                    const int k = part * CH + s;
                    if (k >= len) continue;
                    const int i = hold[k];
                    // brute force: prefix over the segment's hands with position < lo(i) / < hi(i)
                    double want_lo = 0, want_hi = 0;
                    for (int m = 0; m < len; ++m) {
                        if (hold[m] < tb.lo[i]) want_lo += wt[hold[m]];
                        if (hold[m] < tb.hi[i]) want_hi += wt[hold[m]];
                    }
                    if (lo_v[s] != want_lo) fail("run start prefix", g, c, k);
                    if (hi_v[s] != want_hi) fail("run end prefix", g, c, k);
                }
            }
        }
    }
    std::printf("checked %d boards, violations %lld\n", n_games, viol);
    return viol ? 1 : 0;
}
