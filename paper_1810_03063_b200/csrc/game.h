// Host-side game model and GPU layout (no CUDA here).
//
// A game of the batch is a public tree (shared by all games) times private hands
// (per game).  The treeplex of player p is the Cartesian product
// over hands of the player's public decision tree: simplex
// (node m, hand h) has index set {(first[m] + a, h)} and parent (parent_seq[m], h).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/egt_b200.h"

namespace egt {

// private hands per game the gradient kernel handles (256 threads x 5 positions)
constexpr int EGT_MAX_HANDS = 1280;
// warps of the treeplex kernel; each level's nodes are scheduled onto them on the host
#ifndef TREE_WARPS_DEF
#define TREE_WARPS_DEF 8
#endif
constexpr int TREE_WARPS = TREE_WARPS_DEF;
// terminals per CTA of the staged river gradient kernel (rows are never split)
#ifndef EGT_GRAD_CHUNK_TERMS
#define EGT_GRAD_CHUNK_TERMS 16
#endif
constexpr int GRAD_CHUNK_TERMS = EGT_GRAD_CHUNK_TERMS;
// Terminals per gradient CTA for a batch of n_games: GRAD_CHUNK_TERMS from half a game per SM
// up, fewer for small batches so that a launch still spreads over the SMs
inline int grad_chunk_terms(int n_games) {
    const int t = (GRAD_CHUNK_TERMS * n_games + 73) / 74;
    return t < 4 ? 4 : (t > GRAD_CHUNK_TERMS ? GRAD_CHUNK_TERMS : t);
}
constexpr int GRAD_CHUNK_MAX_TERMS = 64;  // a chunk never exceeds this (rows are small)

enum NodeKind { ND_DECISION = 0, ND_CHANCE = 1, ND_TERMINAL = 2 };
enum TermKind { T_FOLD_P1 = 0, T_FOLD_P2 = 1, T_SHOWDOWN = 2 };

struct PNode {
    int kind = ND_DECISION;
    int player = -1;
    int board_state = 0;
    std::string hist;
    std::vector<int> child;
    std::vector<std::string> tok;
    int term_kind = -1;
    double amount = 0;  // fold: payoff to player 2; showdown: amount W won by the better hand
    double kappa = 1;   // public chance weight of the path (Kuhn/Leduc deal probabilities)
};

struct PublicTree {
    std::vector<PNode> nodes;  // nodes[0] = root
    int n_board_states = 1;
    std::vector<std::vector<int>> board_cards;  // per board state (shared part; river: per game)
};

// Per-player treeplex layout over public sequences.
struct PlayerLayout {
    int n_pub = 1;                 // incl. row 0 = empty sequence
    std::vector<int> node_pub;     // public tree node id of each decision node (top-down order)
    std::vector<int> first, nact, parent_seq, board_state, level;
    std::vector<std::string> seq_hist;  // [n_pub], "" for row 0
    std::vector<int> seq_owner;    // decision node owning the sequence (-1 for row 0)
    std::vector<int> term_off, term_idx;  // terminals grouped by this player's last sequence
    std::vector<int> rows_term;           // sequences that end at least one terminal (processing order)
    std::vector<char> pair_next;          // rows_term[r], rows_term[r + 1] were swapped (kept together)
    std::vector<int> chunk_off;           // rows_term split into chunks of ~GRAD_CHUNK_TERMS terminals
    std::vector<int> lvl_off, lvl_nodes;  // decision nodes grouped by level
    std::vector<int> kid_off, kids;       // child decision nodes of each sequence
    // treeplex-kernel schedule: nodes of level l run on warp w in the order
    // sched_nodes[sched_off[l * TREE_WARPS + w] .. sched_off[l * TREE_WARPS + w + 1]); all
    // nodes sharing a parent sequence (other than the empty one) run on one warp, so their
    // values can be added into the parent entry without races; root nodes (parent = empty
    // sequence) keep their values in root_slot[m] >= 0
    std::vector<int> sched_off, sched_nodes, root_slot, seq_slot;
    int n_root = 0, n_int = 0;
    int depth = 0;
};

struct Terminal {
    int kind;
    double amount;
    double kappa;
    int board_state;
    int last_seq[2];
};

// Card-removal / strength-order tables of one (game, board state).
// Positions 0..nvalid-1 are the valid hands in ascending showdown strength; positions
// nvalid..H-1 hold the hands blocked by the board (their gradient entries are 0).
// Card array: card c owns the seg_w slots [c * seg_w, (c + 1) * seg_w): the valid hands
// holding c in strength order (<= 63), then padding, then one end slot; a slot holds the
// hand's position (CE_END for padding and the end slot), CE_FIRST marks slot 0 of every
// segment, so the segmented exclusive scan of the card array leaves each segment's total
// in its end slot.
// Per position and card slot k (the hand's k-th card), pcard packs the card's segment
// start in the card array, the segment indices of the hand's tie group [relo, rehi)
// and the segment length (PC_* below).
// Plan of the card-domain river gradient kernel (kernels.cu grad_card_kernel) for one board:
// CARD_NT threads; thread t owns positions 3t..3t+2 (position domain) and slots
// 6*(t%8)..6*(t%8)+5 of card t/8's segment (card domain).  Every shared-memory exchange
// between the two domains goes through addresses chosen on the host so that no two lanes of a
// half-warp touch the same 8-byte bank pair in one instruction (a proper 16-edge-colouring of
// a bipartite graph of lane groups, which exists by Koenig's theorem):
//   w1 / w2  position -> card:  position i writes its weight to w1 (read by the slot of its
//            lower card) and w2 (higher card);
//   ex       card -> position:  at a row end slot e writes its accumulated card term, and
//            position i reads the slots of its two cards.
constexpr int CARD_NT = 416, CARD_K = 3, CARD_GL = 8, CARD_CH = 6;
constexpr int CARD_NP = CARD_NT * CARD_K;            // positions (>= H_pad)
constexpr int CARD_WREGION = 2 * CARD_NP + 16;       // doubles: w1, w2, 16 zero cells (one per bank pair)
constexpr int CARD_EX = 16 * 192;                    // doubles of the ex exchange (every slot, padding
                                                     // included, has its own conflict-free address)
// one board's plan as one word array (the kernel keeps one pointer): pw, pr, lohi, lane
constexpr int CARD_TAB_PW = 0, CARD_TAB_PR = CARD_NP, CARD_TAB_LOHI = 2 * CARD_NP, CARD_TAB_LANE = 3 * CARD_NP;
constexpr int CARD_TAB_WORDS = 3 * CARD_NP + 8 * CARD_NT;
struct CardPlan {
    std::vector<uint32_t> pw;    // [CARD_NP] byte offsets into the w region: w1 | w2 << 16
    std::vector<uint32_t> pr;    // [CARD_NP] ex element index of the lower-card slot | higher << 16
    std::vector<uint32_t> lane;  // [CARD_NT][8] per thread: cg[3] (gather byte offsets, 2 x 16 bit),
                                 // px[3] (ex element index, 2 x 16 bit), flags (valid 0-5, run head
                                 // 6-11, run tail 12-17), src lanes (lo 0-4, hi 8-12)
    std::vector<uint32_t> tab;   // [CARD_TAB_WORDS] pw | pr | tie group lo | hi << 16 per position | lane
};

struct BoardTable {
    int nvalid = 0;
    CardPlan plan;               // river boards (hand_size 2, identity order) only
    std::vector<int16_t> order;  // [H_pad] position -> hand
    std::vector<int16_t> lo, hi; // [H_pad] per position: tie-group bounds [lo, hi)
    std::vector<uint32_t> lohi;  // [H_pad] lo | hi << 16
    std::vector<uint16_t> cent;  // [n_ce] card array
    std::vector<uint32_t> pcard; // [H_pad][2]
    std::vector<uint8_t> valid;  // [H_pad] per hand
};
#define CE_END 0x0FFFu
#define CE_FIRST 0x1000u
#define PC_START(v) ((int)((v) & 0xFFFu))
#define PC_RELO(v) ((int)(((v) >> 12) & 0x3Fu))
#define PC_REHI(v) ((int)(((v) >> 18) & 0x7Fu))
#define PC_LEN(v) ((int)(((v) >> 25) & 0x7Fu))
#define PC_PACK(start, relo, rehi, len) \
    ((uint32_t)(start) | ((uint32_t)(relo) << 12) | ((uint32_t)(rehi) << 18) | ((uint32_t)(len) << 25))

struct HostGame {
    int kind = 0, n_games = 0;
    int all_valid = 1;  // every hand valid at every board state
    int seg_w = 0, n_ce = 0;  // card-array segment width (incl. end slot) and slots per table
    int H = 0, H_pad = 0, hand_size = 1, n_cards = 0, n_combos = 0;
    int n_ranks = 13, n_suits = 4;
    PublicTree tree;
    PlayerLayout pl[2];
    std::vector<Terminal> terms;
    std::vector<int> hand_cards;       // [G][H][2]
    std::vector<int> hand_combo;       // [G][H] canonical combo index of internal hand
    std::vector<int64_t> strength;     // [G][H] river: showdown strength of internal hand
    std::vector<double> prior[2];      // [G][H_pad]
    std::vector<double> kappa_game;    // [G]
    std::vector<BoardTable> tables;    // [G * n_board_states]
    std::vector<double> beta[2];       // [n_nodes][H_pad]
    std::vector<double> M[2];          // [G]: max l1 norm of the treeplex
    double big_blind = 100;
};

// Builds everything from the spec; returns an error string ("" on success).
std::string build_host_game(const egt_game_spec& spec, HostGame& out);

// ||A|| = max |A_ij| of game g (R7), O(H^2) per board state.
double compute_max_abs_A(const HostGame& G, int g);
// compute_max_abs_A of every game, games spread over the host's cores
std::vector<double> compute_max_abs_A_all(const HostGame& G);

// 5..7-card poker hand strength (larger is better, equal = tie).
int64_t hand_strength(const int* ranks, const int* suits, int n);
// the same key by brute force: max of the 5-card evaluation over all 5-subsets
int64_t hand_strength_subsets(const int* ranks, const int* suits, int n);

}  // namespace egt
