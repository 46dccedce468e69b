// The load path's direct 7-card evaluator (hand_strength) against the brute-force maximum of
// the 5-card evaluation over all 5-subsets (hand_strength_subsets): exhaustive on reduced
// decks, seeded random hands on the full deck.  Prints the mismatch count; exit 1 on any.
#include "game.h"
#include <cstdio>
#include <random>
using namespace egt;
static long long bad = 0, total = 0;
static void check(const int* cards, int n, int n_ranks, int n_suits) {
    int r[7], s[7];
    for (int i = 0; i < n; ++i) { r[i] = 13 - n_ranks + cards[i] / n_suits; s[i] = cards[i] % n_suits; }
    const long long a = hand_strength(r, s, n), b = hand_strength_subsets(r, s, n);
    ++total;
    if (a != b && bad++ < 5) std::printf("mismatch: fast %lld brute %lld\n", a, b);
}
static void exhaustive(int n_ranks, int n_suits, int n) {
    const int N = n_ranks * n_suits;
    int c[7];
    for (int i = 0; i < n; ++i) c[i] = i;
    for (;;) {
        check(c, n, n_ranks, n_suits);
        int i = n - 1;
        while (i >= 0 && c[i] == N - n + i) --i;
        if (i < 0) break;
        ++c[i];
        for (int j = i + 1; j < n; ++j) c[j] = c[j - 1] + 1;
    }
}
int main() {
    exhaustive(6, 4, 7);   // 24 cards: every 7-card hand (flushes, full houses, quads, wheels)
    exhaustive(7, 2, 7);   // two suits: straights and full houses without flushes of five
    std::mt19937_64 rng(7);
    for (int t = 0; t < 200000; ++t) {
        int c[7], k = 0;
        unsigned long long used = 0;
        while (k < 7) {
            const int x = (int)(rng() % 52);
            if (!(used >> x & 1)) { used |= 1ull << x; c[k++] = x; }
        }
        check(c, 7, 13, 4);
    }
    std::printf("checked %lld mismatches %lld\n", total, bad);
    return bad != 0;
}
