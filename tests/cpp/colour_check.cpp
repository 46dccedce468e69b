// The card plan's bipartite edge colouring (game.cpp colour_edges16) on random multigraphs:
// every vertex of degree <= 16 gets its edges coloured with 16 colours, no two edges at one
// vertex share a colour (Koenig's theorem says this always exists; the colouring must find it
// also on the worst cases: 16-regular multigraphs with repeated edges).  Prints "violations N".
#include "../../paper_1810_03063_b200/csrc/game.cpp"
#include <cstdio>
#include <random>
int main(int argc, char** argv) {
    const int trials = argc > 1 ? std::atoi(argv[1]) : 200;
    std::mt19937 rng(2468);
    long long viol = 0, edges_total = 0;
    for (int t = 0; t < trials; ++t) {
        const int nl = 8 + (int)(rng() % 120), nr = nl;
        // a d-regular bipartite multigraph as the union of d random perfect matchings
        // (d = 16 on most trials), then some edges dropped
        const int d = t % 4 ? 16 : 1 + (int)(rng() % 16);
        std::vector<std::pair<int, int>> e;
        std::vector<int> perm(nr);
        for (int k = 0; k < d; ++k) {
            for (int i = 0; i < nr; ++i) perm[i] = i;
            std::shuffle(perm.begin(), perm.end(), rng);
            for (int i = 0; i < nl; ++i) e.push_back({i, perm[i]});
        }
        if (t % 3 == 0) {
            std::shuffle(e.begin(), e.end(), rng);
            e.resize(e.size() * 3 / 4);
        }
        std::shuffle(e.begin(), e.end(), rng);
        const std::vector<int> col = egt::colour_edges16(nl, nr, e);
        std::vector<int> at_l((size_t)nl * 16, 0), at_r((size_t)nr * 16, 0);
        for (size_t k = 0; k < e.size(); ++k) {
            if (col[k] < 0 || col[k] >= 16) { ++viol; continue; }
            if (at_l[(size_t)e[k].first * 16 + col[k]]++) ++viol;
            if (at_r[(size_t)e[k].second * 16 + col[k]]++) ++viol;
        }
        edges_total += (long long)e.size();
    }
    std::printf("%d graphs, %lld edges, violations %lld\n", trials, edges_total, viol);
    return viol ? 1 : 0;
}
