/*
 * egt_b200.h — C ABI of the B200-native EGT / CFR solver for poker endgames.
 *
 * Method: arXiv:1810.03063 (reference text at PAPER.md, cited as PAPER.md:<line>).
 * The library solves  min_{x in X} max_{y in Y} <x, A y>
 * over the players' sequence-form treeplexes, for a BATCH of independent games
 * that share one public betting tree (same pot/stack/abstraction; each game has
 * its own board and hand priors).  x is player 1 (moves first, "Libratus",
 * minimises), y is player 2.  A is player 2's payoff.  A is never materialised.
 *
 * Vector layout (device; elements fp64, or fp32 for games loaded with precision EGT_F32 --
 * every device vector argument below is then a float buffer, while per-game scalars such
 * as mu, step sizes and values stay fp64): for player p, a vector holds, per game g, a
 * row-major [n_pub[p]][H_pad] block; row 0 is the empty sequence (value 1 in a
 * strategy, the value/constant term in a gradient; R1), row s >= 1 is
 * public sequence s (a decision node of p and one of its actions) for every
 * private hand h < H (columns H..H_pad-1 are padding, kept 0).  Game g's block
 * starts at g * vec_stride[p] doubles.  Hands are in the library's internal
 * order (for river games: ascending showdown strength on that game's board);
 * egt_hand_cards() gives each internal hand's cards.
 *
 * Ownership: the library allocates and frees all of its device memory; pointers
 * passed in (host or device, as stated per call) stay owned by the caller and are
 * only read/written during the call (device writes are stream-ordered: complete
 * when the stream set by egt_set_stream, default the legacy default stream, syncs).
 *
 * Errors: every int-returning call returns 0 on success and a negative EGT_E_*
 * code on failure; egt_last_error() returns a message for the calling thread.
 * No call falls back to a CPU implementation: without a usable CUDA device every
 * call that touches the device fails with EGT_E_CUDA.
 */
#ifndef EGT_B200_H
#define EGT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EGT_OK 0
#define EGT_E_ARG (-1)     /* invalid argument */
#define EGT_E_CUDA (-2)    /* CUDA runtime error (or no device) */
#define EGT_E_STATE (-3)   /* call out of order (e.g. egt_step before egt_init) */
#define EGT_E_NUMERIC (-4) /* numerical failure (e.g. EGT/as tau underflow) */

/* Game kinds */
#define EGT_GAME_KUHN 1  /* 3-card Kuhn poker, ante 1, bet 1 */
#define EGT_GAME_LEDUC 2 /* Leduc hold'em: 6 cards, bets 2/4, 2 bets per round */
#define EGT_GAME_RIVER 3 /* NLHE river endgame */

/* River bet-size contexts (R10), index into the spec arrays */
#define EGT_CTX_P1_OPEN 0
#define EGT_CTX_P1_VS_BET 1
#define EGT_CTX_P1_VS_RAISE 2
#define EGT_CTX_P1_SUBSEQ 3
#define EGT_CTX_P2_VS_CHECK 4
#define EGT_CTX_P2_VS_BET 5
#define EGT_CTX_P2_SUBSEQ 6
#define EGT_N_CTX 7
#define EGT_MAX_FRACS 16

typedef struct {
    int32_t kind;    /* EGT_GAME_* */
    int32_t n_games; /* batch size B >= 1 */
    /* --- river only (ignored for Kuhn/Leduc) --- */
    int32_t pot;       /* chips in the pot at the start of the river; each player put pot/2 */
    int32_t stack;     /* chips behind per player at the start of the river */
    int32_t raise_cap; /* max bets+raises in the street (<= 0: unlimited) */
    int32_t open_fold; /* 1: fold is offered facing no bet */
    int32_t n_fracs[EGT_N_CTX];                 /* pot multipliers per context ...  */
    int32_t frac_num[EGT_N_CTX][EGT_MAX_FRACS]; /* ... as exact rationals num/den  */
    int32_t frac_den[EGT_N_CTX][EGT_MAX_FRACS];
    int32_t allin[EGT_N_CTX]; /* 1: all-in offered in the context */
    int32_t n_ranks;          /* deck: top n_ranks ranks (13 = standard) */
    int32_t n_suits;          /* deck: suits (4 = standard) */
    const int32_t* boards;    /* HOST [n_games][5] card ids (rank_pos*n_suits + suit) */
    const double* prior1;     /* HOST [n_games][n_combos] canonical combos (c1<c2 lexicographic), >= 0; NULL = uniform */
    const double* prior2;     /* as prior1, for player 2 */
    int32_t precision;        /* EGT_F64 (0, default) or EGT_F32: element type of every vector */
} egt_game_spec;

#define EGT_F64 0 /* fp64 vectors and arithmetic (parity 1e-9 with the oracle) */
#define EGT_F32 1 /* optional fp32 mode: fp32 vectors and arithmetic, fp64 per-game scalars (1e-5) */

typedef struct egt_game egt_game; /* opaque */

typedef struct {
    int32_t n_games;
    int32_t H;          /* private hands per game (river: combos avoiding the board) */
    int32_t H_pad;      /* row length in doubles (H rounded up to 32) */
    int32_t n_combos;   /* canonical hole-card combos of the deck (river) / cards (Kuhn, Leduc) */
    int32_t n_pub[2];   /* public sequences per player, including row 0 (empty sequence) */
    int32_t n_nodes[2]; /* public decision nodes per player */
    int32_t n_terminals;
    int32_t depth[2];   /* levels of decision nodes per player */
    int64_t vec_stride[2]; /* doubles per game in a player's vector (= n_pub * H_pad) */
    double max_abs_A[1];   /* reserved: ||A|| of game 0 (max |A_ij|, R7) */
    int64_t h2d_bytes;     /* bytes egt_load_game copied host -> device (layout, tables, priors) */
    /* gradient of player p: rows (public sequences) of the other player's vector it reads
     * (the distinct sequences terminals end on) and rows of its own output that can be
     * nonzero (sequences that end a terminal) -- the compulsory traffic */
    int32_t grad_rows_read[2];
    int32_t grad_rows_written[2];
    int32_t precision;     /* EGT_F64 or EGT_F32 */
} egt_game_info;

/* ---- game ---------------------------------------------------------------- */

/* Build the public tree, the per-player treeplex layout, the
 * per-board hand-strength order and card-removal tables, and upload them.
 * spec: host struct, read only during the call.  *out receives the handle.
 * Errors: EGT_E_ARG on an invalid spec (bad kind/deck/board/fractions), EGT_E_CUDA. */
int egt_load_game(const egt_game_spec* spec, egt_game** out);

/* Free everything owned by the handle (NULL is a no-op).  Defined by: the game built by
 * egt_load_game; plumbing (ownership), no arithmetic.  Device buffers are allocated from
 * the library's per-device memory pool and return to it: the memory stays reserved for the
 * next game the process loads (the pool is never trimmed; processes that need it back for
 * other allocators should exit or load no further games). */
void egt_free_game(egt_game* game);

/* Stream for every subsequent call on this game (cudaStream_t as void*; NULL = legacy default).
 * Defined by: the GPU implementation of the paper's operations; plumbing,
 * no arithmetic.  Errors: EGT_E_ARG on a NULL game. */
int egt_set_stream(egt_game* game, void* stream);

/* Sizes of the loaded batch into HOST *out: hands H (the root Cartesian product over private
 * hands), public sequences per player (the treeplex index sets,
 * PAPER.md:402-411), terminals, vector strides, the gradient's compulsory rows (DESIGN.md
 * §8(d)).  Errors: EGT_E_ARG on NULL arguments. */
int egt_game_info_get(const egt_game* game, egt_game_info* out);

/* Internal hand h of game g -> its cards: HOST out[2*h+0], out[2*h+1] (second -1 for
 * one-card hands), for h < H.  out: int32 [2*H].  Defined by: "Chance deals out hands"
 * -- the hands of the root Cartesian product.
 * Errors: EGT_E_ARG on a bad game index or NULL out. */
int egt_hand_cards(const egt_game* game, int32_t g, int32_t* out);

/* Public history string of public sequence s >= 1 of `player` (tokens joined by
 * '/': k check, c call, f fold, b<n> bet/raise to n chips this round, d<card> a
 * public card), NUL-terminated into buf[buflen].  s = 0 gives "" (empty sequence).
 * Defined by: the betting rules of PAPER.md:670-688 (readings R10-R12).  Errors: EGT_E_ARG
 * on a bad player / sequence or a buffer too small. */
int egt_pub_history(const egt_game* game, int32_t player, int32_t s, char* buf, int32_t buflen);

/* ---- kernel-level calls (device pointers, all games of the batch) ------------ */

/* Gradient of the bilinear form (Gen-CFR lines 29/35):
 *   player 0: out = A y   (in: y, player-1 layout; out: player-0 layout)
 *   player 1: out = A^T x (in: x, player-0 layout; out: player-1 layout)
 * evaluated per terminal without materialising A: fold payoffs by inclusion-exclusion
 * over blocked cards, showdowns by strength-sorted prefix sums with card-removal
 * correction.  Row 0 of `in` is ignored (the empty sequence is 1); row 0 of `out`
 * receives the terms of leaves where `player` has not acted yet.
 * dev_in/dev_out: DEVICE fp64, n_games * vec_stride[.] each. */
int egt_gradient(egt_game* game, int32_t player, const double* dev_in, double* dev_out);

/* Smoothed best response: per game, q = argmin_{q in Q_player}
 * <q, gsign*g> + mu_g d(q) with d the dilated entropy.
 * dev_g: DEVICE gradient (player layout); dev_mu: DEVICE [n_games];
 * dev_q: DEVICE out, sequence form (may be NULL); dev_b: DEVICE out, behavioural
 * (row 0 = 1; may be NULL); dev_lb: DEVICE out, the behavioural strategy's natural log
 * log qbar_i = -(g_i - min g) / (mu beta_j) - log sum exp(...) (finite where
 * qbar_i underflows; row 0 and blocked hands 0; may be NULL) -- the form egt_prox takes its
 * centre in (R16); dev_value: DEVICE out [n_games], min value (may be NULL). */
int egt_smoothed_br(egt_game* game, int32_t player, const double* dev_g, double gsign,
                    const double* dev_mu, double* dev_q, double* dev_b, double* dev_lb, double* dev_value);

/* Prox mapping: q = argmin_q <q, s_g * gsign * g> + D(q || z), z given
 * by its behavioural strategy's log dev_center_lb (DEVICE, player layout, e.g. egt_smoothed_br's
 * dev_lb; -inf entries are excluded from the support and stay 0), s_g = dev_step[g].
 * Computed as the SBR of the shifted gradient in the centre's log form,
 * qbar_i ~ exp(lb_i - gsign s_g (g_i + values below) / beta_j) (R16).
 * dev_q: DEVICE out, sequence form. */
int egt_prox(egt_game* game, int32_t player, const double* dev_g, double gsign,
             const double* dev_step, const double* dev_center_lb, double* dev_q);

/* Best response value per game: min_{q in Q} <q, gsign*g>  (dev_value DEVICE [n_games]): the
 * bottom-up pass of PAPER.md:497-500 with the best action per simplex (the mu -> 0 limit of
 * the smoothed best response), the two halves of eps_sad.  dev_g: DEVICE
 * gradient (player layout).  Errors: EGT_E_ARG on NULL pointers or a bad player. */
int egt_best_response(egt_game* game, int32_t player, const double* dev_g, double gsign,
                      double* dev_value);

/* ---- solvers --------------------------------------------------------------- */

#define EGT_THEORY 0   /* Alg. 1: tau_t = 2/(t+3), alternate x/y, theory mu */
#define EGT_BALANCED 1 /* "EGT": mu balancing, tau_t = 2/(t+3) */
#define EGT_AS 2       /* "EGT/as": Alg. 3-4, aggressive mu reduction with EGC check */

/* Initialise EGT (Alg. 1 / Alg. 3 lines 1-2; R4) for
 * every game.  mu_x, mu_y > 0: initial smoothing; <= 0: EGT_THEORY uses the theory value
 * ||A||/sqrt(phi_X phi_Y); EGT_BALANCED / EGT_AS take the
 * "practically-tuned initial" mu (R14): mu_theory * 2^-k with k
 * the last of 0, 1, ..., 30 before the excessive gap condition at the initial point first
 * fails, scanned per game on the device.  Errors: EGT_E_ARG on a bad variant, EGT_E_CUDA. */
int egt_init(egt_game* game, int32_t variant, double mu_x, double mu_y);

/* Run n_iters iterations for every game: Alg. 1 for EGT_THEORY, its mu
 * balanced form for EGT_BALANCED, Alg. 3 with Alg. 4
 * for EGT_AS -- each built from Step, Alg. 2.  For EGT_AS one iteration
 * is one Step attempt (+ EGC check): a failed attempt halves tau and leaves the iterate
 * unchanged, so Alg. 4's inner loop unrolls into consecutive iterations.  The iteration is
 * one CUDA graph launch on the game's stream.  Errors: EGT_E_STATE before egt_init. */
int egt_step(egt_game* game, int32_t n_iters);

/* Per-game stopping target for EGT_AS, Alg. 3's "while eps_sad(x, y) > eps"
 * decided on the device: before each iteration a game whose maintained eps_sad is <= its
 * target stops (every launch of the iteration skips it; its iterate, mu, tau and gap stay),
 * so a batch spends no work on games already solved.  host_eps: HOST [n_games] targets in
 * the game's payoff unit, <= 0 = none; NULL clears every target.  Every game is made live
 * again (a lowered target resumes it).  CFR: a game stops when a saddle_gap /
 * saddle_gap_device evaluation of its average (which = 1) finds eps_sad <= its target.
 * Ignored by EGT_THEORY / EGT_BALANCED (they keep no gap).  Persists across egt_init /
 * cfr_init. */
int egt_set_target(egt_game* game, const double* host_eps);

#define CFR_RM 0   /* CFR(RM):  RM,  alpha_t = 1/t */
#define CFR_RMP 1  /* CFR(RM+): RM+, alpha_t = 1/t */
#define CFR_PLUS 2 /* CFR+:     RM+, alpha_t = 2t/(t^2+t) */

/* Initialise Gen-CFR with the variant's regret minimiser (RM PAPER.md:55-69,
 * RM+ PAPER.md:76-90) and stepsizes: x^0, y^0 uniform at every simplex
 * (line 26), zero regrets and averages, t = 1.  Errors: EGT_E_ARG on a bad variant. */
int cfr_init(egt_game* game, int32_t variant);
/* n_iters iterations of Gen-CFR's loop body for every game, with alternating
 * updates (y's gradient A^T x^t); the regret update is fused into the
 * bottom-up treeplex pass and the averaging (lines 34, 41) into its top-down pass.  One CUDA
 * graph launch per iteration.  Errors: EGT_E_STATE before cfr_init. */
int cfr_step(egt_game* game, int32_t n_iters);

/* Saddle-point residual eps_sad per game, written to HOST out[n_games].
 * which = 0: the solver's current iterate (EGT x^t, y^t; CFR x^t, y^t);
 * which = 1: the CFR averages (xbar, ybar); for EGT the same as 0. */
int saddle_gap(egt_game* game, int32_t which, double* host_out);

/* As saddle_gap (eps_sad), but the per-game eps_sad goes to DEVICE
 * dev_out[n_games], stream-ordered (no host synchronisation; complete when the stream set by
 * egt_set_stream syncs).  Errors: EGT_E_STATE without a solver. */
int saddle_gap_device(egt_game* game, int32_t which, double* dev_out);

/* Strategy of `player` in sequence form, HOST out [n_games][n_pub][n_combos]: the EGT
 * iterate (Alg. 1 / 3 return x^t, y^t), or the CFR average xbar / ybar
 * (Gen-CFR line 43); canonical combo/card order; hands blocked by the board are
 * 0; row 0 = 1.  Errors: EGT_E_STATE without a solver, EGT_E_ARG on a bad player. */
int get_avg_strategy(egt_game* game, int32_t player, double* host_out);

/* Solver vectors in the internal DEVICE layout (copies into dev_out, vec_stride doubles/game):
 * which = 0 current iterate (sequence form; EGT x^t / y^t), 1 CFR average
 * (Gen-CFR line 43; EGT: current), 2 CFR cumulative regrets r^t (PAPER.md:63,
 * 84), 3 CFR current behavioural strategy z^t.  Errors: EGT_E_STATE. */
int get_strategy_device(egt_game* game, int32_t player, int32_t which, double* dev_out);

/* Per-game solver scalars to HOST out[n_games][8]:
 * mu_x, mu_y, tau, t (accepted steps / CFR
 * iterations), attempts, backtracks (Alg. 4 line 3), last EGV,
 * gradient evaluations (A y or A^T x, per game).  Errors: EGT_E_ARG. */
int egt_scalars(egt_game* game, double* host_out);

/* ---- sharding one game over ranks (DESIGN.md row 8) -----------------------------
 * Every rank loads the SAME game(s).  egt_shard gives rank `rank` of `world` a contiguous
 * range of the sequences that end terminals (balanced by terminal count); every gradient
 * the library evaluates (egt_gradient, the EGT / CFR solvers, saddle_gap) then computes only
 * those rows and sums the other ranks' rows in with one in-place NCCL all-reduce on the
 * game's stream (inside the solver's CUDA graph).  The rows are disjoint, so the sum is exact
 * and every rank holds the full gradient and the same (replicated) iterates.
 * id: HOST EGT_NCCL_ID_BYTES bytes from egt_nccl_unique_id on rank 0, distributed by the
 * caller; NULL only for world == 1 (no communicator; with an id a 1-rank communicator is
 * built and used).  Call before egt_init / cfr_init (EGT_E_STATE otherwise).
 * NCCL is opened at run time (libnccl.so.2); EGT_E_CUDA if it cannot be. */
#define EGT_NCCL_ID_BYTES 128
/* HOST out[EGT_NCCL_ID_BYTES]: a fresh NCCL unique id for egt_shard (plumbing for the
 * gradient's collective, PAPER.md:299 / DESIGN.md row 8).  Errors: EGT_E_CUDA without NCCL. */
int egt_nccl_unique_id(uint8_t* out);
/* Shard every gradient of this game over `world` ranks as described above. */
int egt_shard(egt_game* game, int32_t rank, int32_t world, const uint8_t* id);

/* Fused compute + all-gather over NVLink (replaces the all-reduce of egt_shard): every rank's
 * gradient kernels store the rows they compute straight into every rank's gradient buffer
 * (peer memory), then a one-element NCCL all-reduce orders the ranks.  Rows are disjoint, so
 * no reduction is needed and each gradient crosses NVLink once (an all-reduce moves it twice).
 * egt_ipc_handles: HOST out[2 * EGT_IPC_HANDLE_BYTES], this rank's gradient buffers (player 0,
 * player 1) as CUDA IPC handles (the first call moves those buffers from the library's memory
 * pool, which has no IPC export, to plain device allocations; call it before egt_init /
 * cfr_init).  egt_shard_peers: HOST handles[world][2][EGT_IPC_HANDLE_BYTES]
 * gathered from every rank (own entry ignored); after egt_shard with an NCCL id, before
 * egt_init / cfr_init; world <= 8.  Applies to the solvers' gradients (egt_gradient keeps the
 * all-reduce, its output buffer being the caller's). */
#define EGT_IPC_HANDLE_BYTES 64
/* (see above) this rank's gradient buffers (PAPER.md:299 outputs) as CUDA IPC handles. */
int egt_ipc_handles(egt_game* game, uint8_t* out);
/* (see above) open every rank's gradient buffers: each gradient of the
 * solvers is then stored row by row into all of them by the kernel that computes it. */
int egt_shard_peers(egt_game* game, const uint8_t* handles);

/* The fused kernel's stores (the gradient) for shard `rank` of `world` into n_dst
 * DEVICE buffers dsts[] (each
 * laid out like a gradient of `player`, zeroed by the caller), synchronous, no communication:
 * several "ranks" emulated on one device must leave every buffer equal to egt_gradient's result. */
int egt_gradient_rows_to(egt_game* game, int32_t player, int32_t rank, int32_t world, const double* dev_in,
                         const uint64_t* dsts, int32_t n_dst);

/* Emulate `world` ranks on this device (tests; world <= 8, 1 = off): every solver gradient
 * runs
 * each rank's slice kernel (exactly as egt_shard's rank would) into that rank's own buffer --
 * fused = 0: rows outside the slice zeroed first, then an elementwise sum of the `world`
 * buffers into each stands in for the NCCL all-reduce; fused = 1: each slice kernel stores
 * its rows into every rank's buffer (egt_shard_peers' stores).  The solver reads rank 0's
 * buffer.  Before egt_init / cfr_init, on a game without egt_shard.  EGT_E_STATE otherwise. */
int egt_shard_emulate(egt_game* game, int32_t world, int32_t fused);

/* Rows of the gradient that shard `rank` of `world` computes, without
 * communication:
 * DEVICE dout receives those rows, every other row 0 (the sum over all ranks is
 * egt_gradient's result).  Synchronous.  For tests and inspection. */
int egt_gradient_rows(egt_game* game, int32_t player, int32_t rank, int32_t world, const double* dev_in,
                      double* dev_out);

/* ---- kernel timing (measurement only) -------------------------------------------
 * egt_timing(game, 1) switches egt_step / cfr_step / saddle_gap* to eager launches,
 * each bracketed by a pair of CUDA events on the library's stream (the stream the
 * kernels run on), and clears the accumulators; egt_timing(game, 0) switches back to
 * CUDA-graph replay.  egt_timing_get writes HOST out[EGT_N_KERNEL_KINDS][4]:
 * total device ms, launches, game-launches that did work (a masked EGT launch only works
 * on the games whose step focuses on that player), and the compulsory HBM bytes of that
 * work, per kernel kind. */
#define EGT_KERNEL_GRAD_AY 0  /* gradient kernel, player 0: A y        */
#define EGT_KERNEL_GRAD_ATX 1 /* gradient kernel, player 1: A^T x      */
#define EGT_KERNEL_TREE 2     /* treeplex kernel (SBR / prox / BR / CFR / combine) */
#define EGT_KERNEL_SCALAR 3   /* per-game scalar kernels (EGT stepsizes, EGC accept, gap) */
#define EGT_KERNEL_COMM 4     /* NCCL all-reduce of a sharded gradient (egt_shard) */
#define EGT_N_KERNEL_KINDS 5
/* Measurement of the paper's per-iteration work (gradients and treeplex passes, PAPER.md:613-625,
 * 726-731); plumbing, no arithmetic.  Errors: EGT_E_ARG on NULL arguments. */
int egt_timing(egt_game* game, int32_t enable);
/* (see egt_timing) the accumulated per-kind times of the gradients / treeplex passes
 * (PAPER.md:726-731 counts) into HOST out[EGT_N_KERNEL_KINDS][4]. */
int egt_timing_get(egt_game* game, double* host_out);

/* Message of the calling thread's last failed call (plumbing for the error codes above; no
 * passage of PAPER.md defines it beyond the operations it reports on). */
const char* egt_last_error(void);

/* Release the memory the current device's library pool keeps reserved from freed games
 * (cudaMemPoolTrimTo(pool, 0)); memory of live games is untouched.  EGT_E_CUDA on failure.
 * Plumbing: device memory of the games of PAPER.md:670-695, no arithmetic. */
int egt_pool_trim(void);

#ifdef __cplusplus
}
#endif
#endif /* EGT_B200_H */
