// Device-side data structures and kernel launchers (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace egt {

// A per-game vector, optionally double-buffered (slot chosen per game on device).
struct VecRef {
    double* base = nullptr;         // slot 0 of game 0
    long long game_stride = 0;      // doubles between games
    long long slot_stride = 0;      // doubles between slot 0 and slot 1
    const int* slot_sel = nullptr;  // per-game current slot (nullptr: slot 0)
    int slot_xor = 0;               // 0: current slot, 1: the other one
    __host__ __device__ bool ok() const { return base != nullptr; }
#ifdef __CUDACC__
    // strides count elements of the game's precision T (base only carries the address)
    template <class T = double>
    __device__ __forceinline__ T* at(int g) const {
        long long off = (long long)g * game_stride;
        if (slot_sel) off += (long long)((slot_sel[g] ^ slot_xor) & 1) * slot_stride;
        return reinterpret_cast<T*>(base) + off;
    }
#endif
};

struct DevTerm {
    double amount;  // fold: payoff to player 2; showdown: amount W
    double kappa;   // public chance weight
    int kind;       // 0 fold by P1, 1 fold by P2, 2 showdown
    int bs;         // board state
    int seq[2];     // last public sequence of each player (0 = empty)
};

struct DevGame {
    int n_games, H, H_pad, hand_size, n_bs, n_cards;
    int esz;                  // bytes per vector element: 8 (fp64) or 4 (fp32 mode)
    int all_valid;            // 1: every hand is valid at every board state (river endgames)
    int ident;                // 1: position order = hand order at every board state (river endgames)
    int n_ce;                 // card-array slots per table (n_cards * seg_w, padded to 8)
    int seg_w;                // card-array slots per card (incl. the end slot)
    const int* tab_nvalid;    // [G*n_bs]
    const int16_t* tab_order; // [G*n_bs][H_pad]   position -> hand (valid hands first, strength order)
    const uint32_t* tab_lohi; // [G*n_bs][H_pad]   tie group [lo, hi) of each position
    const uint16_t* tab_cent; // [G*n_bs][n_ce]      card array (CE_* packing, game.h)
    const uint2* tab_pcard;   // [G*n_bs][H_pad]     per position, per card: segment info (PC_*)
    const uint8_t* tab_valid; // [G*n_bs][H_pad]
    // card-domain river gradient plan (game.h CardPlan), one per game; card_plan = 0: none
    int card_plan;
    const uint32_t* card_tab;   // [G][CARD_TAB_WORDS]
    const void* prior[2];     // [G][H_pad] in the game's precision
    const double* kappa_game; // [G]
    const DevTerm* terms;
};

struct DevPlayer {
    int n_pub, n_nodes, n_levels;
    int n_rows_term;         // public sequences that end at least one terminal
    const int* node_first;   // [n_nodes], top-down order
    const int* node_nact;
    const int* node_parent;  // parent public sequence (0 = empty)
    const int* node_bs;
    const int* lvl_off;      // [n_levels+1] nodes grouped by level (treeplex depth b_Q^j)
    const int* lvl_nodes;    // [n_nodes]
    const int* kid_off;      // [n_pub+1] child nodes of each sequence (D_j^i)
    const int* kids;         // [n_nodes]
    const int* sched_off;    // [n_levels * TREE_WARPS + 1] treeplex-kernel warp schedule (game.h)
    const int* sched_nodes;  // [n_nodes]
    const int* root_slot;    // [n_nodes] slot of a root node's value, -1 otherwise
    int n_root;
    const int* seq_slot;     // [n_pub] slot of a sequence with child nodes, -1 otherwise
    int n_int;
    const double* beta;      // [n_nodes][H_pad]
    const int* term_off;     // [n_pub+1] terminals grouped by this player's last sequence
    const int* term_idx;
    const int* rows_term;    // [n_rows_term]
    int n_chunks;
    const int* chunk_off;    // [n_chunks+1] ranges of rows_term, one CTA each (staged gradient kernel)
    int max_chunk_terms;     // most terminals in one chunk (the staged kernel takes <= GRAD_CHUNK_MAX_TERMS)
};

// Fused compute + all-gather of a sharded gradient: every output row a shard computes is
// stored straight into each listed buffer (its own and its peers' gradient buffers, mapped
// over NVLink); rows are disjoint across shards, so no reduction is needed.
constexpr int EGT_MAX_PEERS = 8;
struct DevPeers {
    int n = 0;                          // 0: write gout only
    void* base[EGT_MAX_PEERS] = {};     // game 0, row 0 of each destination (the layout of gout)
};

enum TreeMode { TM_SBR = 0, TM_PROX = 1, TM_BR = 2, TM_CFR = 3, TM_UNIFORM = 4, TM_COMBINE = 5 };

struct TreeArgs {
    int mode = TM_SBR;
    VecRef g;                  // gradient input (SBR/PROX/BR/CFR)
    double gsign = 1.0;        // objective uses gsign * g (min form; CFR: utility)
    const double* mu = nullptr;     // SBR: per-game mu; PROX: per-game step s
    VecRef center;             // PROX: centre (behavioural logs); CFR: current z (in/out); COMBINE: behavioural logs
    VecRef regret;             // CFR
    VecRef avg;                // CFR: running average (sequence form, in/out)
    const int* iter = nullptr; // CFR: per-game t (1-based)
    int cfr_plus = 0;          // CFR: 1 = RM+ threshold
    int avg_linear = 0;        // CFR: 1 = alpha_t = 2t/(t^2+t), else 1/t
    VecRef out_b;              // behavioural output
    VecRef out_lb;             // SBR: log of the behavioural output (prox centres, R16)
    VecRef out_q;              // sequence-form output
    VecRef comb_in, comb_out;  // comb_out = (1 - tau) comb_in + tau q
    const double* tau = nullptr;
    double* value = nullptr;   // per-game value (SBR/BR)
    double* partial = nullptr; // [G][n_tiles] scratch
    unsigned* counter = nullptr; // [G] zero-initialised
    // SBR only: also the best-response value of the same gradient (min <q, gsign g>), fused
    double* br_value = nullptr;
    double* br_partial = nullptr;
    unsigned* br_counter = nullptr;
    const int* mask = nullptr; // run game g only if mask[g] == want
    int want = 0;
};

struct DevScalars {
    double* mu;       // [2][G]
    double* mu_cand;  // [2][G]
    double* tau;      // [G]
    double* step;     // [G]
    double* val;      // [2][G]
    double* egv;      // [G]
    int* focus;       // [G]
    int* cur;         // [G]
    int* t;           // [G]
    int* attempts;    // [G]
    int* backtracks;  // [G]
    int* fail;        // [G]
    const double* brval;  // [2][G] best-response values at the EGT/as candidate (gap)
    double* gap;      // [G] eps_sad of the current iterate (EGT/as maintains it)
    int* live;        // [G] 1 while the game iterates; 0 once its gap reached its target
    const double* target;  // [G] per-game eps_sad target (<= 0: none), egt_set_target
};

// A gradient whose input is the convex combination (1 - tau_g) a + tau_g b of two vectors of the
// other player, formed on the rows the kernel reads (Alg. 2 line 1: x_hat = (1 - tau) x +
// tau x_mu(y)) -- the solver's x_hat never exists as a vector.
struct GradComb {
    VecRef b;
    const double* tau = nullptr;  // [G]
};

// Launchers (return cudaGetLastError()).
// all_rows = 1 writes every row of gout (rows without terminals get 0); 0 writes only the
// rows that end a terminal (the solver's gradient buffers are zeroed once at allocation).
cudaError_t launch_gradient(const DevGame& G, const DevPlayer& P, int player, VecRef vin, VecRef gout,
                            const int* mask, int want, int all_rows, cudaStream_t st,
                            const DevPeers* peers = nullptr, const GradComb* comb = nullptr);
cudaError_t launch_tree(const DevGame& G, const DevPlayer& P, int player, const TreeArgs& A, cudaStream_t st);
cudaError_t kernels_prepare();
size_t tree_smem_bytes(const DevPlayer& P, int esz);

cudaError_t launch_egt_prepare(int variant, int n_games, DevScalars S, cudaStream_t st);
cudaError_t launch_egt_accept(int variant, int n_games, DevScalars S, cudaStream_t st);
cudaError_t launch_tick(int n_games, int* t, const int* live, cudaStream_t st);  // live: nullptr = all
cudaError_t launch_stop_at_target(int n_games, const double* gap, const double* target, int* live, cudaStream_t st);
cudaError_t launch_gap_combine(int n, const double* val, double* out, cudaStream_t st);
constexpr int EGT_MU_SCAN_KMAX = 30;  // the practical-mu scan tries mu_theory * 2^-k, k = 0..30
cudaError_t launch_mu_scan(int n, int k, int phase, const double* mu_th, double* mu, int* scan, int* kbest,
                           const double* val, cudaStream_t st);
cudaError_t launch_emu_allreduce(double* const* bufs, int world, size_t n, int esz, cudaStream_t st);

}  // namespace egt
