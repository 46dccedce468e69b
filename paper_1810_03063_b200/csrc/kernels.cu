// sm_100a kernels of the EGT / CFR hot path (fp64, or fp32 in the optional fp32 mode).
//
//  grad_kernel  : g = A y (player 0) or g = A^T x (player 1) without materialising A
//                 (PAPER.md:299 gradient operators; Gen-CFR lines 29/35).
//  tree_kernel  : one pass over a player's treeplex per (game, tile of hands):
//                 bottom-up per simplex (smoothed best response PAPER.md:467-512,
//                 prox mapping PAPER.md:514-537, best response, or the CFR regret
//                 update PAPER.md:30-39/63-64/84-85), then top-down rescale by the
//                 parent sequence with the EGT convex combinations fused.
#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <cmath>

#include "kernels.cuh"
#include "game.h"  // CE_* / PC_* packing of the card tables

namespace egt {

// ------------------------------------------------------------------ warp helpers
template <class T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// inclusive scan that is exact for lanes < LIM (a power of two <= 32)
template <int LIM, typename T>
__device__ __forceinline__ T warp_incl_scan_lim(T v, int lane) {
#pragma unroll
    for (int o = 1; o < LIM; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// exp(x) for x <= 0 to ~1 ulp: x = (64 k + j) ln2 / 64 + r, |r| <= ln2 / 128,
// exp(x) = 2^k' * tab[j] * (1 + r + ... + r^5/120) (truncation < 4e-17 relative).
// tab[j] = 2^(j/64) lives in shared memory.  2^k' is applied as 2^(k'+600) * 2^-600, two exact
// scalings for normal results and one rounding where the result is subnormal, so the result
// underflows gradually and reaches 0 below -745.2 as IEEE exp does -- no floor, no branch (the
// oracle's numpy exp underflows the same way); -inf (and anything below -800) gives 0.
__device__ __forceinline__ double exp_nonpos(double x, const double* __restrict__ tab) {
    x = fmax(x, -800.0);
    const double magic = 6755399441055744.0;  // 1.5 * 2^52: round to nearest integer
    const double big = fma(x, 92.332482616893656877, magic);
    const int k = __double2loint(big);
    const double kd = big - magic;
    double r = fma(kd, -0.010830424696223417, x);
    r = fma(kd, -2.572804622327669e-14, r);
    double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const double v = tab[k & 63] * p;
    const double scale = __hiloint2double(((k >> 6) + 600 + 1023) << 20, 0);  // 2^(k'+600), normal
    return (v * scale) * 0x1p-600;
}

// fp32 mode: the library exp on non-positive arguments (<= 2 ulp)
__device__ __forceinline__ float exp_nonpos(float x, const double* __restrict__) { return expf(x); }

// log(S) for S >= 1 (a softmax normaliser): fp32 hardware log as the start, one Newton step
// y <- y - 1 + S exp(-y) (error ~1e-14 relative; two steps would be exact to rounding)
__device__ __forceinline__ double log_ge1(double S, const double* __restrict__ tab) {
    const double y0 = (double)__logf((float)S);
    return y0 - 1.0 + S * exp_nonpos(-y0, tab);
}
__device__ __forceinline__ float log_ge1(float S, const double* __restrict__) { return logf(S); }

// 1/x for x > 0 normal: hardware approximation + two Newton steps (~1 ulp)
__device__ __forceinline__ double rcp_pos(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ float rcp_pos(float x) { return __frcp_rn(x); }

// Per-game value: the CTA's sum v (valid in thread 0) goes to partial[g][tile]; the last
// CTA of the game sums the tiles in order (deterministic) into value[g].  Contains a barrier.
__device__ __forceinline__ void game_value_reduce(double v, double* partial, unsigned* counter, double* value, int g) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partial[(size_t)g * gridDim.x + blockIdx.x] = v;
        __threadfence();
        const unsigned ticket = atomicAdd(&counter[g], 1u);
        last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double s = 0.0;
        const volatile double* pp = partial + (size_t)g * gridDim.x;
        for (unsigned i = 0; i < gridDim.x; ++i) s += pp[i];
        value[g] = s;
        counter[g] = 0;
    }
}

template <class T>
__device__ __forceinline__ T big_value() { return sizeof(T) == 8 ? (T)DBL_MAX : (T)FLT_MAX; }

// DESIGN.md R15: a regret at the rounding-noise level of its own update counts as 0
template <class T>
__device__ __forceinline__ T cfr_noise() { return sizeof(T) == 8 ? (T)1e-13 : (T)2e-6f; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ gradient
// One CTA per (public sequence s of `player` that ends a terminal, game g).  For every
// terminal t whose last `player` sequence is s (hands of `player`: "self", of the other
// player: "opp"), with the hands in ascending showdown strength (positions i):
//   w[i] = prior_opp(h_i) * v_opp[seq_opp(t), h_i],  P = exclusive prefix sums of w, T = sum w,
//   for every card c: Pc = exclusive prefix sums of w over the hands holding c (in strength
//   order, the card array's segment of c), S_c = their total.
//   fold:     v(h) = sum_{opp h' disjoint from h} w(h') = T - sum_{c in h} S_c + [|h|=2] w(h)
//   showdown: v(h) = sign * (stronger(h) - weaker(h)) over disjoint opp hands, with
//             weaker   = P[lo] - sum_c Pc[lo],  stronger = (T - P[hi]) - sum_c (S_c - Pc[hi])
//             ([lo, hi) = h's tie group), i.e.  v = T - P[hi] - P[lo] + sum_c (Pc[lo] + Pc[hi] - S_c).
//   g[s, h] += kappa_t * kappa_game * amount_t * prior_self(h) * v(h)
// sign = +1 for player 0 (A y: player 2 wins with the stronger hand), -1 for player 1.
// P: block scan over register-resident chunks of K consecutive positions per thread.
// Pc: one segmented block scan over the card array (EPT consecutive slots per thread,
// reset at each segment's first slot); each segment's end slot receives its total S_c.
// Hands that do not share their tie group read their own P / Pc from registers.
template <int NT, int KMAX, int EMAX, typename T>
__global__ void __launch_bounds__(NT, 2) grad_kernel(DevGame G, DevPlayer P, int player, VecRef vin, VecRef gout,
                                                     const int* __restrict__ mask, int want, DevPeers peers,
                                                     VecRef vin2, const double* __restrict__ ctau) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    T* sm = reinterpret_cast<T*>(sm_raw);
    constexpr int NW = NT / 32;
    __shared__ T wtot[NW];
    __shared__ T segv[NW];
    __shared__ int segf[NW];
    const int g = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (mask && mask[g] != want) return;
    const int s = P.rows_term[blockIdx.x];
    const int Hp = G.H_pad, hs = G.hand_size, H = G.H, n_ce = G.n_ce;
    const bool fast = G.ident && G.all_valid;  // positions are hands and every hand is valid
    T* w = sm;               // [Hp]   by position
    T* Pf = w + Hp;          // [Hp+1] by position
    T* Ex = Pf + Hp + 1;     // [n_ce] card array
    T* acc = Ex + n_ce;      // [Hp]   by hand (general path only)
    if (!fast)
        for (int i = tid; i < Hp; i += NT) acc[i] = T(0);
    T racc[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) racc[j] = T(0);
    const int t0 = P.term_off[s], t1 = P.term_off[s + 1];
    const T* __restrict__ popp = static_cast<const T*>(player ? G.prior[0] : G.prior[1]) + (size_t)g * Hp;
    const T* __restrict__ vo = vin.at<T>(g);
    const T* __restrict__ vo2 = ctau ? vin2.at<T>(g) : nullptr;  // x_hat = (1 - tau) vin + tau vin2
    const T ct = ctau ? (T)ctau[g] : T(0), ct1 = T(1) - ct;
    const T kg = (T)G.kappa_game[g];
    const T sd_sign = player == 0 ? T(1) : T(-1);
    const int EPT = (n_ce + NT - 1) / NT;
    const int ebase = tid * EPT;
    for (int ti = t0; ti < t1; ++ti) {
        const DevTerm tm = G.terms[P.term_idx[ti]];
        const int k = g * G.n_bs + tm.bs;
        const int nv = G.tab_nvalid[k];
        const int16_t* __restrict__ order = G.tab_order + (size_t)k * Hp;
        const uint32_t* __restrict__ lohi = G.tab_lohi + (size_t)k * Hp;
        const uint16_t* __restrict__ cent = G.tab_cent + (size_t)k * n_ce;
        const uint2* __restrict__ pcard = G.tab_pcard + (size_t)k * Hp;
        const int so = player ? tm.seq[0] : tm.seq[1];
        const T* __restrict__ vrow = vo + (size_t)so * Hp;
        const T* __restrict__ vrow2 = vo2 ? vo2 + (size_t)so * Hp : nullptr;
        const bool sd = tm.kind == 2;
        const int K = (nv + NT - 1) / NT;
        const int base = tid * K;
        __syncthreads();  // the previous terminal is done with w / Pf / Ex
        // ---- phase A: w (coalesced), then per-thread chunks of K positions, block scan
        for (int i = tid; i < nv; i += NT) {
            const int h = fast ? i : order[i];
            w[i] = popp[h] * (so ? (vrow2 ? ct1 * vrow[h] + ct * vrow2[h] : vrow[h]) : T(1));
        }
        __syncthreads();
        T x[KMAX];
        T run = T(0);
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            const int i = base + j;
            x[j] = (j < K && i < nv) ? w[i] : T(0);
            run += x[j];
        }
        const T incl = warp_incl_scan(run, lane);
        if (lane == 31) wtot[wid] = incl;
        // ---- phase B (local part): card-array chunk, segmented scan inside the thread
        T ex[EMAX];
        T srun = T(0);
        bool sflag = false;
        int first_flag = EMAX;
        unsigned endmask = 0u;
#pragma unroll
        for (int j = 0; j < EMAX; ++j) {
            const int e = ebase + j;
            const bool in = j < EPT && e < n_ce;
            const unsigned c = in ? cent[e] : CE_END;
            if (in && (c & CE_FIRST)) {
                srun = T(0);
                if (!sflag) first_flag = j;
                sflag = true;
            }
            const unsigned pos = c & CE_END;
            if (pos == CE_END) endmask |= 1u << j;
            const T y = pos != CE_END ? w[pos] : T(0);
            ex[j] = srun;
            srun += y;
        }
        // segmented inclusive scan of (srun, sflag) over the warp
        T sv = srun;
        int sf = sflag;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T uv = __shfl_up_sync(0xffffffffu, sv, o);
            const int uf = __shfl_up_sync(0xffffffffu, sf, o);
            if (lane >= o) {
                if (!sf) sv += uv;
                sf |= uf;
            }
        }
        if (lane == 31) {
            segv[wid] = sv;
            segf[wid] = sf;
        }
        __syncthreads();
        // block prefix of P
        T wpre = T(0), total = T(0);
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            const T v = wtot[q];
            wpre += q < wid ? v : T(0);
            total += v;
        }
        const T pbase = wpre + incl - run;
        if (sd) {
            T p = pbase;
#pragma unroll
            for (int j = 0; j < KMAX; ++j) {
                const int i = base + j;
                if (j < K && i < nv) Pf[i] = p;
                p += x[j];
            }
            if (tid == 0) Pf[nv] = total;
        }
        // carry into this thread's first segment: segmented exclusive prefix over threads
        {
            T carry = T(0);
            for (int q = 0; q < wid; ++q) carry = segf[q] ? segv[q] : carry + segv[q];
            const T pv = __shfl_up_sync(0xffffffffu, sv, 1);
            const int pf = __shfl_up_sync(0xffffffffu, sf, 1);
            if (lane > 0) carry = pf ? pv : carry + pv;
#pragma unroll
            for (int j = 0; j < EMAX; ++j) {
                const int e = ebase + j;
                if (j < EPT && e < n_ce) {
                    const T v = j < first_flag ? carry + ex[j] : ex[j];
                    if (sd || ((endmask >> j) & 1u)) Ex[e] = v;
                }
            }
        }
        __syncthreads();
        // ---- phase C: per position
        const T scale = (T)(tm.kappa * G.kappa_game[g] * tm.amount);
        T pre = pbase;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            const int i = base + j;
            if (j < K && i < nv) {
                const uint2 pc = pcard[i];
                T v = total - Ex[PC_START(pc.x) + PC_LEN(pc.x)];
                if (hs == 2) v -= Ex[PC_START(pc.y) + PC_LEN(pc.y)];
                if (sd) {
                    const uint32_t lh = lohi[i];
                    const int lo = lh & 0xFFFFu, hi = lh >> 16;
                    if (lo == i && hi == i + 1) {
                        // alone in its tie group: its own prefixes
                        const T ca = Ex[PC_START(pc.x) + PC_RELO(pc.x)];
                        v += -(pre + (pre + x[j])) + (ca + (ca + x[j]));
                        if (hs == 2) {
                            const T cb = Ex[PC_START(pc.y) + PC_RELO(pc.y)];
                            v += cb + (cb + x[j]);
                        }
                    } else {
                        v += -(Pf[lo] + Pf[hi]) + Ex[PC_START(pc.x) + PC_RELO(pc.x)] +
                             Ex[PC_START(pc.x) + PC_REHI(pc.x)];
                        if (hs == 2) v += Ex[PC_START(pc.y) + PC_RELO(pc.y)] + Ex[PC_START(pc.y) + PC_REHI(pc.y)];
                    }
                    v *= sd_sign;
                } else if (hs == 2) {
                    v += x[j];
                }
                if (fast) racc[j] += scale * v;
                else acc[order[i]] += scale * v;
            }
            pre += x[j];
        }
    }
    const T* __restrict__ pself = static_cast<const T*>(player ? G.prior[1] : G.prior[0]) + (size_t)g * Hp;
    const long long row_off = (long long)g * gout.game_stride + (long long)s * Hp;
    __syncthreads();
    if (fast) {
        const int K = (H + NT - 1) / NT;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            const int i = tid * K + j;
            if (j < K && i < H) w[i] = racc[j];
        }
        __syncthreads();
        for (int i = tid; i < Hp; i += NT) acc[i] = i < H ? pself[i] * w[i] : T(0);
    } else {
        for (int i = tid; i < Hp; i += NT) acc[i] *= pself[i];
    }
    if (peers.n == 0) {
        T* __restrict__ out = gout.at<T>(g) + (size_t)s * Hp;
        for (int i = tid; i < Hp; i += NT) out[i] = acc[i];
    } else {
#pragma unroll
        for (int d = 0; d < EGT_MAX_PEERS; ++d) {  // this shard's row into every shard's buffer
            if (d < peers.n) {
                T* __restrict__ out = reinterpret_cast<T*>(peers.base[d]) + row_off;
                for (int i = tid; i < Hp; i += NT) out[i] = acc[i];
            }
        }
    }
}

// ------------------------------------------------------------------ card-domain river gradient
// River endgames (every hand valid, positions = hands in strength order, two cards per hand):
// one CTA per (chunk of consecutive rows, game), persistent over the chunk's terminals, CARD_NT
// threads playing two roles (game.h CardPlan):
//  * position domain -- thread t holds positions 3t..3t+2: w = prior_opp * v_opp, its block
//    prefix P, the position part of every hand's value (T - P[hi] - P[lo] for a showdown,
//    T + w(h) for a fold), accumulated per position over the row's terminals;
//  * card domain -- the 8 lanes of card c hold the hands holding c in strength order (6 slots
//    each): their weights, the segment prefix Pc and total S_c, and each slot's card part
//    (Pc[lo] + Pc[hi] - S_c for a showdown, -S_c for a fold) accumulated per slot over the
//    row's terminals, never leaving registers until the row ends.
// Pc[lo] / Pc[hi] are the segment prefixes at the start / end of the slot's tie run inside the
// segment: in registers within a lane's 6 slots, and one shuffle from a host-planned source
// lane (the run's head / tail lane) when the run crosses lanes.  A hand's value is its position
// part plus the card parts of its two slots (PAPER.md:299 gradient, reading R13 payoffs):
//   showdown  sign * [(T - P[hi] - P[lo]) + sum_{c in h} (Pc[lo] + Pc[hi] - S_c)]
//   fold      T - S_c1 - S_c2 + w(h)            (inclusion-exclusion over the blocked cards)
// Only two shared-memory exchanges cross the domains, both at host-planned addresses that are
// bank-conflict free per half-warp: the weights (position -> card, once per opponent row) and
// the card parts (card -> position, once per row).  The game's priors and each terminal's
// opponent row arrive by bulk async copies (TMA engine, mbarrier); the next terminal's row is
// in flight while this one is processed.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ unsigned half16(unsigned v, int hi) { return hi ? v >> 16 : v & 0xFFFFu; }
// the plan's w-region byte offsets are for 8-byte elements; fp32 elements sit at half of them
template <class T>
__device__ __forceinline__ unsigned woff(unsigned v, int hi) { return half16(v, hi) >> (sizeof(T) == 4 ? 1 : 0); }

#ifndef CARD_MINB
#define CARD_MINB 2
#endif
template <typename T, bool COMB>
__global__ void __launch_bounds__(CARD_NT, CARD_MINB) grad_card_kernel(DevGame G, DevPlayer P, int player, VecRef vin,
                                                               VecRef gout, const int* __restrict__ mask, int want,
                                                               DevPeers peers, VecRef vin2,
                                                               const double* __restrict__ ctau) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    constexpr int NT = CARD_NT, K = CARD_K, CH = CARD_CH, NW = NT / 32, NP = CARD_NP, MT = GRAD_CHUNK_MAX_TERMS;
    __shared__ T wtot[NW];
    __shared__ __align__(8) uint64_t bar[3];
    // the chunk's terminals in processing order: opponent row, kind, weight, the row each one
    // completes (-1: more terminals of its row follow), its row buffer and whether it is fetched
    __shared__ int t_so[MT], t_kind[MT], t_end[MT], t_idx[MT];
    __shared__ uint32_t t_meta[MT];  // so | (row + 1) << 12 | flags << 24 (one load per terminal)
    __shared__ double t_w[MT];
    __shared__ int s_nT;
    const int g = blockIdx.y, tid = threadIdx.x;
    if (mask && mask[g] != want) return;
    const int Hp = G.H_pad, H = G.H;
    T* popp = reinterpret_cast<T*>(sm_raw);  // [NP] (0 beyond H)
    T* vb = popp + NP;                       // [2][NP] opponent rows (0 beyond Hp)
    T* vb2 = vb + 2 * NP;                    // COMB: [2][NP] the second input's rows
    T* wreg = vb2 + (COMB ? 2 * NP : 0);     // [CARD_WREGION] w1 | w2 | zero cell
    T* Pf = wreg + CARD_WREGION;             // [NP + 4] exclusive prefixes of w by position
    T* Ex = Pf + NP + 4;                     // [CARD_EX] card parts at a row end
    const int r0 = P.chunk_off[blockIdx.x], r1 = P.chunk_off[blockIdx.x + 1];
    const T* __restrict__ vo = vin.at<T>(g);
    const T* __restrict__ vo2 = COMB ? vin2.at<T>(g) : nullptr;
    if (tid == 0) {
        // the chunk's terminals in processing order: its rows in rows_term order (game.cpp
        // build_layout orders rows and terminals so that a terminal sharing the previous one's
        // opponent row is a fold), each row's terminals in term_idx order
        int n = 0;
        for (int r = r0; r < r1; ++r) {
            const int srow = P.rows_term[r];
            for (int k = P.term_off[srow]; k < P.term_off[srow + 1]; ++k) {
                t_idx[n] = P.term_idx[k];
                t_end[n] = k + 1 == P.term_off[srow + 1] ? srow : -1;
                ++n;
            }
        }
        s_nT = n;
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = Hp + tid; i < NP; i += NT) {  // padding the bulk copies never write
        popp[i] = T(0);
        vb[i] = T(0);
        vb[NP + i] = T(0);
        if (COMB) {
            vb2[i] = T(0);
            vb2[NP + i] = T(0);
        }
    }
    if (tid < CARD_WREGION - 2 * NP) wreg[2 * NP + tid] = T(0);  // the zero cell padding slots read
    if (tid < 4) Pf[NP + tid] = T(0);
    __syncthreads();
    const int nT = s_nT;
    for (int i = tid; i < nT; i += NT) {
        const DevTerm tm = G.terms[t_idx[i]];
        t_so[i] = player ? tm.seq[0] : tm.seq[1];
        t_kind[i] = tm.kind;
        t_w[i] = tm.kappa * G.kappa_game[g] * tm.amount * (tm.kind == 2 && player ? -1.0 : 1.0);  // + showdown sign
    }
    __syncthreads();
    // per terminal: its opponent row, the row it completes, and the decisions every thread
    // would otherwise recompute: showdown, new opponent row, fold reusing the previous totals,
    // the next terminal needs a new row (prefetch)
    for (int i = tid; i < nT; i += NT) {
        const int so = t_so[i];
        const bool sd = t_kind[i] == 2;
        const bool new_row = so != 0 && (i == 0 || so != t_so[i - 1]);
        const bool reuse = i > 0 && !sd && so == t_so[i - 1];
        const bool next_new = i + 1 < nT && t_so[i + 1] != 0 && t_so[i + 1] != so;
        t_meta[i] = (uint32_t)so | ((uint32_t)(t_end[i] + 1) << 12) |
                    ((uint32_t)sd << 24) | ((uint32_t)new_row << 25) | ((uint32_t)reuse << 26) | ((uint32_t)next_new << 27);
    }
    __syncthreads();
    if (tid == 0) {
        const unsigned bD = Hp * sizeof(T);
        mbar_expect_tx(&bar[0], bD);
        bulk_g2s(popp, static_cast<const T*>(player ? G.prior[0] : G.prior[1]) + (size_t)g * Hp, bD, &bar[0]);
        // the first two new opponent rows, into buffers 0 and 1 (the loop prefetches the rest,
        // a new row always into the buffer the current row is not in)
        int b = 1, fetched = 0;
        for (int q = 0; q < nT && fetched < 2; ++q) {
            if (t_so[q] != 0 && (q == 0 || t_so[q] != t_so[q - 1])) {
                b ^= 1;
                if (q <= 1) {
                    mbar_expect_tx(&bar[1 + b], COMB ? 2 * bD : bD);
                    bulk_g2s(vb + b * NP, vo + (size_t)t_so[q] * Hp, bD, &bar[1 + b]);
                    if (COMB) bulk_g2s(vb2 + b * NP, vo2 + (size_t)t_so[q] * Hp, bD, &bar[1 + b]);
                }
                ++fetched;
            }
            if (q >= 1) break;
        }
    }
    // the board's plan, in registers for the whole chunk (game.h CardPlan)
    const int lane = tid & 31, wid = tid >> 5;
    const int base = tid * K, part = tid & (CARD_GL - 1);
    // the board's plan (one pointer; the words used once per opponent row / row stay in L1)
    const uint32_t* __restrict__ tab = G.card_tab + (size_t)g * CARD_TAB_WORDS;
    const uint4* __restrict__ lane_g = reinterpret_cast<const uint4*>(tab + CARD_TAB_LANE) + tid * 2;
    const uint4 la = __ldg(lane_g), lb = __ldg(lane_g + 1);
    uint32_t cg[3] = {la.x, la.y, la.z};
    uint32_t flags = lb.z, srcs = lb.w;
    // per position: its w1 / w2 addresses and its tie group's bounds as byte offsets into Pf
    uint32_t pwr[K], plh[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int i = base + j;
        pwr[j] = i < H ? __ldg(tab + CARD_TAB_PW + i) : 0u;
        const uint32_t lh = i < H ? __ldg(tab + CARD_TAB_LOHI + i) : 0u;
        plh[j] = (lh & 0xFFFFu) * sizeof(T) | ((lh >> 16) * sizeof(T)) << 16;
    }
    const unsigned char* const pfb = reinterpret_cast<const unsigned char*>(Pf);
    T* const gdst = gout.at<T>(g);
    const long long goff = (long long)g * gout.game_stride;
    const T ct = COMB ? (T)ctau[g] : T(0), ct1 = T(1) - ct;  // Alg. 2 line 1
    const T* __restrict__ pself_g = static_cast<const T*>(player ? G.prior[1] : G.prior[0]) + (size_t)g * Hp;
    unsigned char* const wbytes = reinterpret_cast<unsigned char*>(wreg);
    T racc[K], rc[CH], x[K];
#pragma unroll
    for (int j = 0; j < K; ++j) racc[j] = x[j] = T(0);
#pragma unroll
    for (int s = 0; s < CH; ++s) rc[s] = T(0);
    T total = T(0), pbase = T(0), segS = T(0);
    unsigned par = 0u;  // mbarrier phase bit of each opponent-row buffer
    bool ex_dirty = false;  // the last row end's Ex reads are not yet behind a barrier
    mbar_wait(&bar[0], 0);
    __syncthreads();  // the processing order
    int q = 1;  // the buffer holding the current opponent row
    for (int li = 0; li < nT; ++li) {
        // per-thread words re-enter the loop opaque (decoded where used; see grad_staged_kernel)
#pragma unroll
        for (int j = 0; j < K; ++j) asm volatile("" : "+r"(pwr[j]), "+r"(plh[j]));
        asm volatile("" : "+r"(cg[0]), "+r"(cg[1]), "+r"(cg[2]), "+r"(flags), "+r"(srcs));
        const int src_lo = (int)(srcs & 31u), src_hi = (int)((srcs >> 8) & 31u);
        const uint32_t meta = t_meta[li];
        const int so = (int)(meta & 0xFFFu);
        const bool sd = (meta >> 24) & 1u;
        const bool new_row = (meta >> 25) & 1u;
        // a fold on the previous terminal's opponent row reuses its totals (w, T, S_c); a
        // showdown always recomputes (its per-slot terms do not survive a terminal)
        const bool reuse = (meta >> 26) & 1u;
        if (new_row) q ^= 1;
        if (tid == 0 && li > 0 && ((meta >> 27) & 1u)) {
            fence_proxy_async();  // the next new row, into the other buffer
            mbar_expect_tx(&bar[2 - q], (COMB ? 2 : 1) * Hp * sizeof(T));
            bulk_g2s(vb + (q ^ 1) * NP, vo + (size_t)t_so[li + 1] * Hp, Hp * sizeof(T), &bar[2 - q]);
            if (COMB) bulk_g2s(vb2 + (q ^ 1) * NP, vo2 + (size_t)t_so[li + 1] * Hp, Hp * sizeof(T), &bar[2 - q]);
        }
        if (new_row) {
            mbar_wait(&bar[1 + q], (par >> q) & 1u);
            par ^= 1u << q;
        }
        const T scale = (T)t_w[li];
        if (!reuse) {  // CTA-uniform
            // ---- position domain: w, its two conflict-free copies for the card lanes, warp scan
            const T* vrow = vb + q * NP;
            const T* vrow2 = vb2 + q * NP;
            T run = T(0);
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const T v = COMB ? ct1 * vrow[base + j] + ct * vrow2[base + j] : vrow[base + j];
                x[j] = so ? popp[base + j] * v : popp[base + j];
                run += x[j];
                if (base + j < H) {
                    *reinterpret_cast<T*>(wbytes + woff<T>(pwr[j], 0)) = x[j];
                    *reinterpret_cast<T*>(wbytes + woff<T>(pwr[j], 1)) = x[j];
                }
            }
            const T incl = warp_incl_scan(run, lane);
            if (lane == 31) wtot[wid] = incl;
            __syncthreads();
            // ---- card domain: the segment's weights, prefix (8-lane group scan) and total
            T y[CH], ssum = T(0);
#pragma unroll
            for (int s = 0; s < CH; ++s) {
                y[s] = *reinterpret_cast<const T*>(wbytes + woff<T>(cg[s / 2], s & 1));
                ssum += y[s];
            }
            T inc = ssum;
#pragma unroll
            for (int o = 1; o < CARD_GL; o <<= 1) {
                const T u = __shfl_up_sync(0xffffffffu, inc, o, CARD_GL);
                if (part >= o) inc += u;
            }
            segS = __shfl_sync(0xffffffffu, inc, lane | (CARD_GL - 1));
            if (sd) {
                T ex[CH];
                T r = inc - ssum;
#pragma unroll
                for (int s = 0; s < CH; ++s) {
                    ex[s] = r;
                    r += y[s];
                }
                // this lane's last run head / first run tail, for lanes whose runs cross into it
                T lh = T(0), ft = T(0);
#pragma unroll
                for (int s = 0; s < CH; ++s)
                    if ((flags >> (6 + s)) & 1u) lh = ex[s];
#pragma unroll
                for (int s = CH - 1; s >= 0; --s)
                    if ((flags >> (12 + s)) & 1u) ft = ex[s] + y[s];
                const T clo = __shfl_sync(0xffffffffu, lh, src_lo);
                const T chi = __shfl_sync(0xffffffffu, ft, src_hi);
                // the slot's card part of this terminal, accumulated at once (nothing per slot
                // stays live across the barrier): Pc at the run's start + Pc at its end - S_c
                T dsd[CH];
                T cur = clo;
#pragma unroll
                for (int s = 0; s < CH; ++s) {
                    if ((flags >> (6 + s)) & 1u) cur = ex[s];
                    dsd[s] = cur;
                }
                cur = chi;
#pragma unroll
                for (int s = CH - 1; s >= 0; --s) {
                    if ((flags >> (12 + s)) & 1u) cur = ex[s] + y[s];
                    rc[s] += scale * (dsd[s] + (cur - segS));
                }
            }
            // ---- position domain: block prefix of w
            const T wsc = warp_incl_scan_lim<(NW <= 16 ? 16 : 32)>(lane < NW ? wtot[lane] : T(0), lane);
            const T wpre_incl = __shfl_sync(0xffffffffu, wsc, (wid + 31) & 31);
            const T wpre = wid ? wpre_incl : T(0);
            total = __shfl_sync(0xffffffffu, wsc, NW - 1);
            pbase = wpre + incl - run;
            if (sd) {
                T pp = pbase;
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    Pf[base + j] = pp;
                    pp += x[j];
                }
                if (tid == 0) Pf[NP] = total;
            }
            __syncthreads();
            ex_dirty = false;
        }
        // ---- this terminal's contribution: position parts (and a fold's card parts)
        if (sd) {
#pragma unroll
            for (int j = 0; j < K; ++j) {  // P at the tie group's bounds (a group's lanes share the address)
                const T phi = *reinterpret_cast<const T*>(pfb + (plh[j] >> 16));
                const T plo = *reinterpret_cast<const T*>(pfb + (plh[j] & 0xFFFFu));
                racc[j] += scale * (total - phi - plo);
            }
        } else {
#pragma unroll
            for (int j = 0; j < K; ++j)  // w(h) back from the position's own w1 cell
                racc[j] += scale * (total + *reinterpret_cast<const T*>(wbytes + woff<T>(pwr[j], 0)));
            const T sS = scale * segS;
#pragma unroll
            for (int s = 0; s < CH; ++s) rc[s] -= sS;
        }
        // ---- row end: card parts to the positions of their hands, then the output row
        const int srow = (int)((meta >> 12) & 0xFFFu) - 1;
        if (srow >= 0) {
            if (ex_dirty) __syncthreads();
            {
                const uint4 lx = __ldg(lane_g), ly = __ldg(lane_g + 1);
                const uint32_t px[3] = {lx.w, ly.x, ly.y};
#pragma unroll
                for (int s = 0; s < CH; ++s) {  // (padding slots own never-read addresses)
                    Ex[half16(px[s / 2], s & 1)] = rc[s];
                    rc[s] = T(0);
                }
            }
            __syncthreads();
            T outv[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const int i = base + j;
                const uint32_t pr = i < H ? __ldg(tab + CARD_TAB_PR + i) : 0u;
                outv[j] = i < H ? __ldg(pself_g + i) * (racc[j] + Ex[half16(pr, 0)] + Ex[half16(pr, 1)]) : T(0);
                racc[j] = T(0);
            }
            ex_dirty = true;
            if (peers.n == 0) {
                T* __restrict__ dst = gdst + (size_t)srow * Hp;
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (base + j < Hp) dst[base + j] = outv[j];
            } else {
                // fused all-gather: the finished row goes straight into every shard's gradient
                // buffer (peer memory over NVLink), overlapping the next terminals
                const long long off = goff + (long long)srow * Hp;
#pragma unroll
                for (int d = 0; d < EGT_MAX_PEERS; ++d) {  // constant indices: no local copy of peers
                    if (d < peers.n) {
                        T* __restrict__ dst = reinterpret_cast<T*>(peers.base[d]) + off;
#pragma unroll
                        for (int j = 0; j < K; ++j)
                            if (base + j < Hp) dst[base + j] = outv[j];
                    }
                }
            }
        }
    }
}

// ------------------------------------------------------------------ staged river gradient
// The same gradient with the card parts read per position instead of accumulated per slot
// (round 1's design): every card's segment of the card array (its hands in strength order,
// padding, an end slot) is scanned by 8 lanes and its exclusive prefixes are stored; phase C
// reads, per position, the segment totals S_c and the prefixes at its tie group's bounds
// Pc[lo], Pc[hi] (PC_* offsets), and the position prefixes P[lo], P[hi].  The position ->
// card gather of phase B goes through the card plan's conflict-free w1 / w2 exchange (game.h
// CardPlan); chunk terminal order, opponent-row double buffering and the fused x_hat input
// (COMB) as in grad_card_kernel.  Measured faster than the card-domain kernel on the bench
// workload, so it is the one the library launches.
template <typename T, bool COMB>
__global__ void __launch_bounds__(CARD_NT, 2) grad_staged_kernel(DevGame G, DevPlayer P, int player, VecRef vin,
                                                                 VecRef gout, const int* __restrict__ mask, int want,
                                                                 DevPeers peers, VecRef vin2,
                                                                 const double* __restrict__ ctau) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    constexpr int NT = CARD_NT, K = CARD_K, CH = CARD_CH, NW = NT / 32, NP = CARD_NP, MT = GRAD_CHUNK_MAX_TERMS;
    __shared__ T wtot[NW];
    __shared__ __align__(8) uint64_t bar[3];
    __shared__ int t_so[MT], t_kind[MT], t_end[MT], t_idx[MT];
    __shared__ uint32_t t_meta[MT];  // so | (row + 1) << 12 | flags << 24
    __shared__ double t_w[MT];
    __shared__ int s_nT;
    const int g = blockIdx.y, tid = threadIdx.x;
    if (mask && mask[g] != want) return;
    const int Hp = G.H_pad, H = G.H, W = G.seg_w;
    T* popp = reinterpret_cast<T*>(sm_raw);  // [NP] (0 beyond H)
    T* vb = popp + NP;                       // [2][NP] opponent rows (0 beyond Hp)
    T* vb2 = vb + 2 * NP;                    // COMB: [2][NP] the second input's rows
    T* wreg = vb2 + (COMB ? 2 * NP : 0);     // [CARD_WREGION] w1 | w2 | zero cell
    T* Pf = wreg + CARD_WREGION;             // [NP + 4] exclusive prefixes of w by position
    T* Ex = Pf + NP + 4;                     // [n_ce] card array: exclusive prefixes per segment
    const int r0 = P.chunk_off[blockIdx.x], r1 = P.chunk_off[blockIdx.x + 1];
    const T* __restrict__ vo = vin.at<T>(g);
    const T* __restrict__ vo2 = COMB ? vin2.at<T>(g) : nullptr;
    if (tid == 0) {
        int n = 0;
        for (int r = r0; r < r1; ++r) {
            const int srow = P.rows_term[r];
            for (int k = P.term_off[srow]; k < P.term_off[srow + 1]; ++k) {
                t_idx[n] = P.term_idx[k];
                t_end[n] = k + 1 == P.term_off[srow + 1] ? srow : -1;
                ++n;
            }
        }
        s_nT = n;
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = Hp + tid; i < NP; i += NT) {
        popp[i] = T(0);
        vb[i] = T(0);
        vb[NP + i] = T(0);
        if (COMB) {
            vb2[i] = T(0);
            vb2[NP + i] = T(0);
        }
    }
    if (tid < CARD_WREGION - 2 * NP) wreg[2 * NP + tid] = T(0);
    if (tid < 4) Pf[NP + tid] = T(0);
    __syncthreads();
    const int nT = s_nT;
    for (int i = tid; i < nT; i += NT) {
        const DevTerm tm = G.terms[t_idx[i]];
        t_so[i] = player ? tm.seq[0] : tm.seq[1];
        t_kind[i] = tm.kind;
        // the showdown sign (+ for A y: player 2 wins with the stronger hand) goes into the weight
        t_w[i] = tm.kappa * G.kappa_game[g] * tm.amount * (tm.kind == 2 && player ? -1.0 : 1.0);
    }
    __syncthreads();
    for (int i = tid; i < nT; i += NT) {
        const int so = t_so[i];
        const bool sd = t_kind[i] == 2;
        const bool new_row = so != 0 && (i == 0 || so != t_so[i - 1]);
        const bool reuse = i > 0 && so == t_so[i - 1];
        // the card-array prefixes and P are needed by a showdown, also one that follows on the
        // same opponent row (then the first of the pair writes them)
        const bool full = sd || (i + 1 < nT && t_so[i + 1] == so && t_kind[i + 1] == 2);
        const bool next_new = i + 1 < nT && t_so[i + 1] != 0 && t_so[i + 1] != so;
        t_meta[i] = (uint32_t)so | ((uint32_t)(t_end[i] + 1) << 12) | ((uint32_t)sd << 24) |
                    ((uint32_t)new_row << 25) | ((uint32_t)reuse << 26) | ((uint32_t)next_new << 27) |
                    ((uint32_t)full << 28);
    }
    __syncthreads();
    if (tid == 0) {
        const unsigned bD = Hp * sizeof(T);
        mbar_expect_tx(&bar[0], bD);
        bulk_g2s(popp, static_cast<const T*>(player ? G.prior[0] : G.prior[1]) + (size_t)g * Hp, bD, &bar[0]);
        int b = 1;
        for (int q = 0; q < 2 && q < nT; ++q)
            if (t_so[q] != 0 && (q == 0 || t_so[q] != t_so[q - 1])) {
                b ^= 1;
                mbar_expect_tx(&bar[1 + b], COMB ? 2 * bD : bD);
                bulk_g2s(vb + b * NP, vo + (size_t)t_so[q] * Hp, bD, &bar[1 + b]);
                if (COMB) bulk_g2s(vb2 + b * NP, vo2 + (size_t)t_so[q] * Hp, bD, &bar[1 + b]);
            }
    }
    const int lane = tid & 31, wid = tid >> 5;
    const int base = tid * K, part = tid & (CARD_GL - 1), sgi = tid / CARD_GL;
    const bool has_seg = sgi < G.n_cards;
    const uint32_t* __restrict__ tab = G.card_tab + (size_t)g * CARD_TAB_WORDS;
    const uint4 la = __ldg(reinterpret_cast<const uint4*>(tab + CARD_TAB_LANE) + tid * 2);
    uint32_t cg[3] = {la.x, la.y, la.z};
    // the card-array slots this thread writes: all of them (bits 0-5) or only its segment's
    // end slot (bits 8-13)
    unsigned masks = 0u;
#pragma unroll
    for (int j = 0; j < CH; ++j) {
        const int e = part * CH + j;
        if (has_seg && e < W) {
            masks |= 1u << j;
            if (e == W - 1) masks |= 1u << (8 + j);
        }
    }
    T* const exs = Ex + sgi * W + part * CH;
    // phase C's shared-memory operands as byte offsets from Pf, two per word: [0] the segment
    // ends of the hand's two cards (S_c), [1] / [2] card x's / card y's prefixes at the tie
    // group's bounds, [3] the position prefixes at them
    uint32_t pa[K][4], pwr[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int i = base + j;
        const uint2 pc = i < Hp ? G.tab_pcard[(size_t)g * Hp + i] : make_uint2(0u, 0u);
        const uint32_t lh = i < Hp ? G.tab_lohi[(size_t)g * Hp + i] : 0u;
        const uint32_t e0 = (NP + 4) * sizeof(T);
        const uint32_t sx = e0 + PC_START(pc.x) * sizeof(T), sy = e0 + PC_START(pc.y) * sizeof(T);
        pa[j][0] = (sx + PC_LEN(pc.x) * sizeof(T)) | (sy + PC_LEN(pc.y) * sizeof(T)) << 16;
        pa[j][1] = (sx + PC_RELO(pc.x) * sizeof(T)) | (sx + PC_REHI(pc.x) * sizeof(T)) << 16;
        pa[j][2] = (sy + PC_RELO(pc.y) * sizeof(T)) | (sy + PC_REHI(pc.y) * sizeof(T)) << 16;
        pa[j][3] = (lh & 0xFFFFu) * sizeof(T) | ((lh >> 16) * sizeof(T)) << 16;
        pwr[j] = i < H ? __ldg(tab + CARD_TAB_PW + i) : 0u;
    }
    const unsigned char* const pfb = reinterpret_cast<const unsigned char*>(Pf);
    auto ldo = [pfb](uint32_t v, int hi) { return *reinterpret_cast<const T*>(pfb + (hi ? v >> 16 : v & 0xFFFFu)); };
    const T* __restrict__ pself_g = static_cast<const T*>(player ? G.prior[1] : G.prior[0]) + (size_t)g * Hp;
    unsigned char* const wbytes = reinterpret_cast<unsigned char*>(wreg);
    const T ct = COMB ? (T)ctau[g] : T(0), ct1 = T(1) - ct;  // Alg. 2 line 1
    T* const gdst = gout.at<T>(g);
    const long long goff = (long long)g * gout.game_stride;
    T racc[K], x[K];
#pragma unroll
    for (int j = 0; j < K; ++j) racc[j] = x[j] = T(0);
    T total = T(0), pbase = T(0);
    unsigned par = 0u;
    int q = 1;
    mbar_wait(&bar[0], 0);
    __syncthreads();
    for (int li = 0; li < nT; ++li) {
        // the per-thread address words re-enter the loop as opaque values every terminal, so
        // the compiler decodes each 16-bit field where it is used (one instruction) instead of
        // keeping ~30 decoded addresses live across the loop (72 registers: spills and
        // rematerialised index arithmetic otherwise, ~9 % slower)
#pragma unroll
        for (int j = 0; j < K; ++j) {
#pragma unroll
            for (int k = 0; k < 4; ++k) asm volatile("" : "+r"(pa[j][k]));
            asm volatile("" : "+r"(pwr[j]));
        }
        asm volatile("" : "+r"(cg[0]), "+r"(cg[1]), "+r"(cg[2]));
        const uint32_t meta = t_meta[li];
        const int so = (int)(meta & 0xFFFu);
        const bool sd = (meta >> 24) & 1u, new_row = (meta >> 25) & 1u, reuse = (meta >> 26) & 1u;
        const bool full = (meta >> 28) & 1u;
        if (new_row) q ^= 1;
        if (tid == 0 && li > 0 && ((meta >> 27) & 1u)) {
            fence_proxy_async();
            mbar_expect_tx(&bar[2 - q], (COMB ? 2 : 1) * Hp * sizeof(T));
            bulk_g2s(vb + (q ^ 1) * NP, vo + (size_t)t_so[li + 1] * Hp, Hp * sizeof(T), &bar[2 - q]);
            if (COMB) bulk_g2s(vb2 + (q ^ 1) * NP, vo2 + (size_t)t_so[li + 1] * Hp, Hp * sizeof(T), &bar[2 - q]);
        }
        if (new_row) {
            mbar_wait(&bar[1 + q], (par >> q) & 1u);
            par ^= 1u << q;
        }
        if (!reuse) {  // CTA-uniform
            // ---- phase A: w = prior_opp * v_opp (COMB: v = x_hat), its conflict-free copies
            const T* vrow = vb + q * NP;
            const T* vrow2 = vb2 + q * NP;
            T run = T(0);
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const T v = COMB ? ct1 * vrow[base + j] + ct * vrow2[base + j] : vrow[base + j];
                x[j] = so ? popp[base + j] * v : popp[base + j];
                run += x[j];
                if (base + j < H) {
                    *reinterpret_cast<T*>(wbytes + woff<T>(pwr[j], 0)) = x[j];
                    *reinterpret_cast<T*>(wbytes + woff<T>(pwr[j], 1)) = x[j];
                }
            }
            const T incl = warp_incl_scan(run, lane);
            if (lane == 31) wtot[wid] = incl;
            __syncthreads();
            // ---- phase B: card sums (segment scans inside lane groups) and the block prefix of w
            {
                T y[CH], ssum = T(0);
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    y[j] = *reinterpret_cast<const T*>(wbytes + woff<T>(cg[j / 2], j & 1));
                    ssum += y[j];
                }
                T inc = ssum;
#pragma unroll
                for (int o = 1; o < CARD_GL; o <<= 1) {
                    const T u = __shfl_up_sync(0xffffffffu, inc, o, CARD_GL);
                    if (part >= o) inc += u;
                }
                // the same accumulation order in both cases, so a segment total never depends on
                // whether the terminal needs the full prefixes (folds: end slot only)
                const unsigned wm = full ? masks : masks >> 8;
                T run2 = inc - ssum;
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    if (wm & (1u << j)) exs[j] = run2;
                    run2 += y[j];
                }
            }
            const T wsc = warp_incl_scan_lim<(NW <= 16 ? 16 : 32)>(lane < NW ? wtot[lane] : T(0), lane);
            const T wpre_incl = __shfl_sync(0xffffffffu, wsc, (wid + 31) & 31);
            const T wpre = wid ? wpre_incl : T(0);
            total = __shfl_sync(0xffffffffu, wsc, NW - 1);
            pbase = wpre + incl - run;
            if (full) {
                T pp = pbase;
#pragma unroll
                for (int j = 0; j < K; ++j) {
                    Pf[base + j] = pp;
                    pp += x[j];
                }
                if (tid == 0) Pf[NP] = total;
            }
            __syncthreads();
        }
        // ---- phase C (positions beyond H compute on padding and are never stored)
        const T scale = (T)t_w[li];
        T pg = T(0);  // P[lo] + P[hi] of the previous position's tie group
#pragma unroll
        for (int j = 0; j < K; ++j) {
            T v = total - ldo(pa[j][0], 0) - ldo(pa[j][0], 1);
            if (sd) {
                // a position in the same tie group as the thread's previous one reuses its P
                // bounds (predicated-off lanes issue no shared-memory wavefronts)
                if (j == 0 || pa[j][3] != pa[j - 1][3]) pg = ldo(pa[j][3], 0) + ldo(pa[j][3], 1);
                v += -pg + ldo(pa[j][1], 0) + ldo(pa[j][1], 1) + ldo(pa[j][2], 0) + ldo(pa[j][2], 1);
            } else {
                v += *reinterpret_cast<const T*>(wbytes + woff<T>(pwr[j], 0));
            }
            racc[j] += scale * v;
        }
        // ---- row end: prior_self * acc straight from registers to the output row(s)
        const int srow = (int)((meta >> 12) & 0xFFFu) - 1;
        if (srow >= 0) {
            T outv[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                const int i = base + j;
                outv[j] = i < H ? __ldg(pself_g + i) * racc[j] : T(0);
                racc[j] = T(0);
            }
            if (peers.n == 0) {
                T* __restrict__ dst = gdst + (size_t)srow * Hp;
#pragma unroll
                for (int j = 0; j < K; ++j)
                    if (base + j < Hp) dst[base + j] = outv[j];
            } else {
                const long long off = goff + (long long)srow * Hp;
#pragma unroll
                for (int d = 0; d < EGT_MAX_PEERS; ++d) {
                    if (d < peers.n) {
                        T* __restrict__ dst = reinterpret_cast<T*>(peers.base[d]) + off;
#pragma unroll
                        for (int j = 0; j < K; ++j)
                            if (base + j < Hp) dst[base + j] = outv[j];
                    }
                }
            }
        }
    }
}

static constexpr int GRAD_NT = 512, GRAD_KMAX = 3, GRAD_EMAX = 6;  // H <= 1536, card array <= 3072

static size_t grad_smem_bytes(const DevGame& G) {
    return (size_t)G.esz * (size_t)(3 * G.H_pad + 1 + G.n_ce);
}

static size_t card_smem_bytes(const DevGame& G, bool comb) {
    return (size_t)G.esz * ((comb ? 5 : 3) * (size_t)CARD_NP + CARD_WREGION + CARD_NP + 4 + CARD_EX);
}

static size_t staged_smem_bytes(const DevGame& G, bool comb) {
    return (size_t)G.esz * ((comb ? 5 : 3) * (size_t)CARD_NP + CARD_WREGION + CARD_NP + 4 + G.n_ce);
}

// EGT_GRAD_KERNEL=card selects the card-domain kernel (measurement); default: the staged one
static bool use_card_kernel() {
    static const bool card = [] {
        const char* v = std::getenv("EGT_GRAD_KERNEL");
        return v && std::strcmp(v, "card") == 0;
    }();
    return card;
}

static bool card_ok(const DevGame& G, const DevPlayer& P) {
    // (terminal metadata packs sequence indices in 12 bits)
    return G.card_plan && G.ident && G.all_valid && G.n_bs == 1 && G.hand_size == 2 && G.H_pad <= CARD_NP &&
           P.n_pub < 4095;
}

template <class T>
static cudaError_t launch_gradient_t(const DevGame& G, const DevPlayer& P, int player, VecRef vin, VecRef gout,
                                     const int* mask, int want, cudaStream_t st, const DevPeers& peers,
                                     const GradComb* comb) {
    const VecRef b = comb ? comb->b : VecRef();
    const double* tau = comb ? comb->tau : nullptr;
    if (card_ok(G, P) && P.max_chunk_terms <= GRAD_CHUNK_MAX_TERMS && !use_card_kernel()) {
        if (P.n_chunks == 0) return cudaSuccess;
        dim3 grid(P.n_chunks, G.n_games);
        if (comb)
            grad_staged_kernel<T, true><<<grid, CARD_NT, staged_smem_bytes(G, true), st>>>(G, P, player, vin, gout,
                                                                                           mask, want, peers, b, tau);
        else
            grad_staged_kernel<T, false><<<grid, CARD_NT, staged_smem_bytes(G, false), st>>>(G, P, player, vin, gout,
                                                                                             mask, want, peers, b, tau);
        return cudaGetLastError();
    }
    if (card_ok(G, P) && P.max_chunk_terms <= GRAD_CHUNK_MAX_TERMS) {
        if (P.n_chunks == 0) return cudaSuccess;
        dim3 grid(P.n_chunks, G.n_games);
        if (comb)
            grad_card_kernel<T, true><<<grid, CARD_NT, card_smem_bytes(G, true), st>>>(G, P, player, vin, gout, mask,
                                                                                       want, peers, b, tau);
        else
            grad_card_kernel<T, false><<<grid, CARD_NT, card_smem_bytes(G, false), st>>>(G, P, player, vin, gout,
                                                                                         mask, want, peers, b, tau);
        return cudaGetLastError();
    }
    dim3 grid(P.n_rows_term, G.n_games);
    grad_kernel<GRAD_NT, GRAD_KMAX, GRAD_EMAX, T>
        <<<grid, GRAD_NT, grad_smem_bytes(G), st>>>(G, P, player, vin, gout, mask, want, peers, b, tau);
    return cudaGetLastError();
}

cudaError_t launch_gradient(const DevGame& G, const DevPlayer& P, int player, VecRef vin, VecRef gout,
                            const int* mask, int want, int all_rows, cudaStream_t st, const DevPeers* peers,
                            const GradComb* comb) {
    const DevPeers none;
    const DevPeers& pr = peers ? *peers : none;
    if (pr.n && gout.slot_sel) return cudaErrorInvalidValue;
    if (all_rows) {
        // rows that end no terminal (or that another shard computes) are 0
        if (gout.slot_sel) return cudaErrorInvalidValue;
        cudaError_t e = cudaSuccess;
        const size_t row_block = (size_t)G.esz * (size_t)P.n_pub * G.H_pad;
        char* base = reinterpret_cast<char*>(gout.base);
        if (gout.game_stride == (long long)P.n_pub * G.H_pad)
            e = cudaMemsetAsync(base, 0, row_block * G.n_games, st);
        else
            for (int g = 0; g < G.n_games && e == cudaSuccess; ++g)
                e = cudaMemsetAsync(base + (size_t)g * gout.game_stride * G.esz, 0, row_block, st);
        if (e != cudaSuccess) return e;
    }
    if (P.n_rows_term == 0) return cudaSuccess;
    return G.esz == 4 ? launch_gradient_t<float>(G, P, player, vin, gout, mask, want, st, pr, comb)
                      : launch_gradient_t<double>(G, P, player, vin, gout, mask, want, st, pr, comb);
}

// ------------------------------------------------------------------ treeplex pass
// CTA = (TH_HANDS = 64 hands, game), TREE_WARPS warps; lane l handles hands l and l + 32 of
// the tile.  The player's whole gradient tile [n_pub][64] is staged in shared memory by
// asynchronous 16-byte copies and scaled once.  Bottom-up, level by level (deepest first),
// every warp runs the nodes the host scheduled for it (game.h): each simplex j = (node,
// hand) solves its local problem (softmax / prox / argmin / regret
// matching) on its entries -- which already hold the values of the simplexes below --,
// overwrites them with the behavioural strategy and adds its value into the parent entry
// (nodes sharing a parent run on one warp, in a fixed order: no races, deterministic);
// root simplexes keep their values apart.  Top-down (shallowest first) each entry becomes
// q_i = q_{p_j} * qbar_i in place and the requested outputs (behavioural, sequence form,
// EGT convex combinations, CFR average) are written row by row.
#ifndef TREE_HPL
#define TREE_HPL 1
#endif
static constexpr int TH_HPL = TREE_HPL, TH_HANDS = 32 * TH_HPL, TH_WARPS = TREE_WARPS, TH_NT = 32 * TH_WARPS;
#ifndef TREE_MIN_CTAS
#define TREE_MIN_CTAS 4
#endif
#ifndef TREE_MIN_CTAS_LB
#define TREE_MIN_CTAS_LB 4
#endif

size_t tree_smem_bytes(const DevPlayer& P, int esz) {
    return sizeof(double) * 64 + (size_t)esz * ((size_t)TH_HANDS * (P.n_pub + 2 * P.n_root + P.n_int) + 3 * P.n_nodes) +
           sizeof(int) * (size_t)P.n_pub +
           sizeof(int) * (size_t)(6 * P.n_nodes + P.n_levels * TH_WARPS + 1);
}

template <class T>
struct TreeNodeCtx {
    int cfr_plus;
    T mu;
    const double* __restrict__ exptab;
    T cfr_scale;  // CFR: max |g| over the hand's sequences (the noise floor of reading R15)
    T* __restrict__ lbo;  // SBR: behavioural log-probabilities output (nullptr: none)
};

// Bottom-up work of simplex (node m, hand h) on its column; returns the simplex value.
template <int MODE, class T>
__device__ __forceinline__ T tree_node_up(const TreeNodeCtx<T>& C, const DevPlayer& P, T* col, int first,
                                               int n, int m, int h, int Hp, T logn, T* __restrict__ cz,
                                               T* __restrict__ rg, T sc, T wgt, T iw) {
    constexpr int mode = MODE;
    for (int a = 0; a < n; ++a) col[a * TH_HANDS] *= sc;  // the objective's scale (see tree_kernel)
    if (mode == TM_SBR) {
        // qbar_i ~ exp(-g_i / w), value = g_{i*} + w log qbar_{i*} + w log n with
        // i* = argmax qbar, w = mu beta_j; log qbar_i = arg_i - log S
        T mn = big_value<T>();
        for (int a = 0; a < n; ++a) mn = fmin(mn, col[a * TH_HANDS]);
        T S = T(0);
        for (int a = 0; a < n; ++a) {
            const T arg = (mn - col[a * TH_HANDS]) * iw;
            col[a * TH_HANDS] = arg;
            S += exp_nonpos(arg, C.exptab);
        }
        const T inv = T(1) / S, lS = log(S);
        for (int a = 0; a < n; ++a) {
            const T arg = col[a * TH_HANDS];
            if (C.lbo) C.lbo[(size_t)(first + a) * Hp + h] = arg - lS;
            col[a * TH_HANDS] = exp_nonpos(arg, C.exptab) * inv;
        }
        return mn - wgt * (lS - logn);
    }
    if (mode == TM_PROX) {
        // shifted-gradient SBR with the centre's behavioural logs
        // (R16): qbar_i ~ exp(lb_i - g_i / beta), value = -beta log sum_i exp(lb_i - g_i / beta)
        const T beta = wgt, ib = iw;
        const T* __restrict__ zr = cz + (size_t)first * Hp + h;
        T m = -big_value<T>();
        for (int a = 0; a < n; ++a) {
            const T e = zr[(size_t)a * Hp] - col[a * TH_HANDS] * ib;
            col[a * TH_HANDS] = e;
            m = fmax(m, e);
        }
        T S = T(0);
        for (int a = 0; a < n; ++a) {
            const T e = exp_nonpos(col[a * TH_HANDS] - m, C.exptab);
            col[a * TH_HANDS] = e;
            S += e;
        }
        const T inv = T(1) / S;
        for (int a = 0; a < n; ++a) col[a * TH_HANDS] *= inv;
        return -beta * (m + log(S));
    }
    if (mode == TM_BR) {
        int best = 0;
        T mn = col[0];
        for (int a = 1; a < n; ++a) {
            const T v = col[a * TH_HANDS];
            if (v < mn) {
                mn = v;
                best = a;
            }
        }
        for (int a = 0; a < n; ++a) col[a * TH_HANDS] = a == best ? T(1) : T(0);
        return mn;
    }
    // TM_CFR: utility u = gsign * g, current strategy z, regrets r
    T v = T(0);
    for (int a = 0; a < n; ++a) v += col[a * TH_HANDS] * cz[(size_t)(first + a) * Hp + h];
    T S = T(0);
    for (int a = 0; a < n; ++a) {
        const size_t ix = (size_t)(first + a) * Hp + h;
        const T u = col[a * TH_HANDS], r0 = rg[ix];
        T r = r0 + u - v;
        if (C.cfr_plus) r = fmax(r, T(0));
        rg[ix] = r;
        // DESIGN.md R15: regrets at the rounding-noise level of their own update count as 0
        const T tol = cfr_noise<T>() * (fabs(r0) + fabs(u) + fabs(v) + C.cfr_scale);
        const T pr = r > tol ? r : T(0);
        col[a * TH_HANDS] = pr;
        S += pr;
    }
    for (int a = 0; a < n; ++a) {
        const T z = S > T(0) ? col[a * TH_HANDS] / S : T(1) / n;
        col[a * TH_HANDS] = z;
        cz[(size_t)(first + a) * Hp + h] = z;
    }
    return v;
}

// The same bottom-up work for a node with a compile-time number of actions N: the N
// entries are read once into registers and written once.
template <int N, int MODE, class T, int LB>
__device__ __forceinline__ T tree_node_up_n(const TreeNodeCtx<T>& C, const DevPlayer& P, T* col, int first,
                                                 int m, int h, int Hp, T logn, T* __restrict__ cz,
                                                 T* __restrict__ rg, T sc, T wgt, T iw) {
    T x[N];
#pragma unroll
    for (int a = 0; a < N; ++a) x[a] = sc * col[a * TH_HANDS];
    constexpr int mode = MODE;
    T value;
    if (mode == TM_SBR && LB == 0) {  // no log output: the exponentials overwrite x in place
        T mn = x[0];
#pragma unroll
        for (int a = 1; a < N; ++a) mn = fmin(mn, x[a]);
        T S = T(0);
#pragma unroll
        for (int a = 0; a < N; ++a) {
            x[a] = exp_nonpos((mn - x[a]) * iw, C.exptab);
            S += x[a];
        }
        const T inv = rcp_pos(S);
#pragma unroll
        for (int a = 0; a < N; ++a) x[a] *= inv;
        value = mn - wgt * (log_ge1(S, C.exptab) - logn);
    } else if (mode == TM_SBR) {
        T mn = x[0];
#pragma unroll
        for (int a = 1; a < N; ++a) mn = fmin(mn, x[a]);
        T S = T(0), e[N];
#pragma unroll
        for (int a = 0; a < N; ++a) {
            x[a] = (mn - x[a]) * iw;  // log qbar_a + log S
            e[a] = exp_nonpos(x[a], C.exptab);
            S += e[a];
        }
        const T inv = rcp_pos(S), lS = log_ge1(S, C.exptab);
        if (LB == 1 || C.lbo) {
#pragma unroll
            for (int a = 0; a < N; ++a) C.lbo[(size_t)(first + a) * Hp + h] = x[a] - lS;
        }
#pragma unroll
        for (int a = 0; a < N; ++a) x[a] = e[a] * inv;
        value = mn - wgt * (lS - logn);
    } else if (mode == TM_PROX) {
        // centre by its behavioural logs (R16): qbar_a ~ exp(lb_a - g_a / beta)
        const T beta = wgt, ib = iw;
        const T* __restrict__ zr = cz + (size_t)first * Hp + h;
        T m = -big_value<T>();
#pragma unroll
        for (int a = 0; a < N; ++a) {
            x[a] = zr[(size_t)a * Hp] - x[a] * ib;
            m = fmax(m, x[a]);
        }
        T S = T(0);
#pragma unroll
        for (int a = 0; a < N; ++a) {
            x[a] = exp_nonpos(x[a] - m, C.exptab);
            S += x[a];
        }
        const T inv = rcp_pos(S);
#pragma unroll
        for (int a = 0; a < N; ++a) x[a] *= inv;
        value = -beta * (m + log_ge1(S, C.exptab));
    } else if (mode == TM_BR) {
        int best = 0;
        T mn = x[0];
#pragma unroll
        for (int a = 1; a < N; ++a)
            if (x[a] < mn) {
                mn = x[a];
                best = a;
            }
#pragma unroll
        for (int a = 0; a < N; ++a) x[a] = a == best ? T(1) : T(0);
        value = mn;
    } else {
        T z[N], r[N];
        const size_t ix0 = (size_t)first * Hp + h;
#pragma unroll
        for (int a = 0; a < N; ++a) {
            z[a] = cz[ix0 + (size_t)a * Hp];
            r[a] = rg[ix0 + (size_t)a * Hp];
        }
        T v = T(0);
#pragma unroll
        for (int a = 0; a < N; ++a) v += x[a] * z[a];
        T S = T(0);
#pragma unroll
        for (int a = 0; a < N; ++a) {
            const T u = x[a], r0 = r[a];
            T rr = r0 + u - v;
            if (C.cfr_plus) rr = fmax(rr, T(0));
            rg[ix0 + (size_t)a * Hp] = rr;
            const T tol = cfr_noise<T>() * (fabs(r0) + fabs(u) + fabs(v) + C.cfr_scale);  // DESIGN.md R15
            x[a] = rr > tol ? rr : T(0);
            S += x[a];
        }
#pragma unroll
        for (int a = 0; a < N; ++a) {
            x[a] = S > T(0) ? x[a] / S : T(1) / N;
            cz[ix0 + (size_t)a * Hp] = x[a];
        }
        value = v;
    }
#pragma unroll
    for (int a = 0; a < N; ++a) col[a * TH_HANDS] = x[a];
    return value;
}

template <int MODE, class T, int LB>
__device__ __forceinline__ T tree_node_up_any(const TreeNodeCtx<T>& C, const DevPlayer& P, T* col, int first,
                                                   int n, int m, int h, int Hp, T logn, T* __restrict__ cz,
                                                   T* __restrict__ rg, T sc, T wgt, T iw) {
    // register-resident widths: up to 9 actions for SBR / BR (one array), fewer for the modes
    // that also hold the centre or the regrets
    constexpr int NMAX = (MODE == TM_SBR || MODE == TM_BR) ? 9 : (MODE == TM_PROX ? 6 : 4);
    switch (n) {  // warp-uniform: every lane works on the same node
#define EGT_NODE_CASE(K) \
    case K:              \
        if (K <= NMAX) return tree_node_up_n<(K <= NMAX ? K : 1), MODE, T, LB>(C, P, col, first, m, h, Hp, logn, cz, rg, sc, wgt, iw); \
        break;
        EGT_NODE_CASE(1) EGT_NODE_CASE(2) EGT_NODE_CASE(3) EGT_NODE_CASE(4) EGT_NODE_CASE(5) EGT_NODE_CASE(6)
        EGT_NODE_CASE(7) EGT_NODE_CASE(8) EGT_NODE_CASE(9)
#undef EGT_NODE_CASE
        default: break;
    }
    return tree_node_up<MODE, T>(C, P, col, first, n, m, h, Hp, logn, cz, rg, sc, wgt, iw);
}

// Top-down work of simplex (node, hand): q_i = q_{p_j} * qbar_i and the requested output rows.
// All global reads of the node are issued before any use (one round trip per node).
template <class T>
struct TreeDownCtx {
    T tau, alpha;
    const double* __restrict__ exptab;
    const T* __restrict__ bin;
    const T* __restrict__ ci;
    T* __restrict__ ob;
    T* __restrict__ oq;
    T* __restrict__ co;
    T* __restrict__ av;
};

// OUTS: the set of output rows (TO_* bits) fixed at compile time, or 0 = decided at run time
enum TreeOuts { TO_B = 1, TO_Q = 2, TO_COMB = 4, TO_AVG = 8, TO_FUSEBR = 16, TO_LB = 32, TO_VAL = 64 };

template <int N, int MODE, int OUTS, class T>
__device__ __forceinline__ void tree_node_down_n(const TreeDownCtx<T>& D, bool ok, T qp, T unif, int first,
                                                 T* col, int h, int Hp) {
    const bool wb = OUTS ? (OUTS & TO_B) != 0 : D.ob != nullptr;  // (TO_FUSEBR, TO_LB: bottom-up flags)
    const bool wq = OUTS ? (OUTS & TO_Q) != 0 : D.oq != nullptr;
    const bool wc = OUTS ? (OUTS & TO_COMB) != 0 : D.co != nullptr;
    const bool wa = OUTS ? (OUTS & TO_AVG) != 0 : D.av != nullptr;
    const size_t ix0 = (size_t)first * Hp + h;
    T b[N], cv[N], avv[N];
#pragma unroll
    for (int a = 0; a < N; ++a) {
        if (!ok) b[a] = T(0);
        else if (MODE == TM_UNIFORM) b[a] = unif;
        else if (MODE == TM_COMBINE) b[a] = exp_nonpos(D.bin[ix0 + (size_t)a * Hp], D.exptab);  // centre: log qbar
        else b[a] = col[a * TH_HANDS];
        cv[a] = wc ? D.ci[ix0 + (size_t)a * Hp] : T(0);
        avv[a] = wa ? D.av[ix0 + (size_t)a * Hp] : T(0);
    }
#pragma unroll
    for (int a = 0; a < N; ++a) {
        const T q = qp * b[a];
        col[a * TH_HANDS] = q;
        const size_t ix = ix0 + (size_t)a * Hp;
        if (wb) D.ob[ix] = b[a];
        if (wq) D.oq[ix] = q;
        if (wc) D.co[ix] = (T(1) - D.tau) * cv[a] + D.tau * q;
        if (wa) D.av[ix] = D.alpha * q + (T(1) - D.alpha) * avv[a];
    }
}

template <int MODE, int OUTS, class T>
__device__ __forceinline__ void tree_node_down_any(const TreeDownCtx<T>& D, bool ok, T qp, int first, int n,
                                                   T* col, int h, int Hp) {
    const T unif = T(1) / n;
    switch (n) {
        case 1: tree_node_down_n<1, MODE, OUTS, T>(D, ok, qp, unif, first, col, h, Hp); return;
        case 2: tree_node_down_n<2, MODE, OUTS, T>(D, ok, qp, unif, first, col, h, Hp); return;
        case 3: tree_node_down_n<3, MODE, OUTS, T>(D, ok, qp, unif, first, col, h, Hp); return;
        case 4: tree_node_down_n<4, MODE, OUTS, T>(D, ok, qp, unif, first, col, h, Hp); return;
        default: break;
    }
    for (int a0 = 0; a0 < n; a0 += 4) {  // wider nodes: four actions per round trip
        const int k = min(4, n - a0);
        T* c0 = col + a0 * TH_HANDS;
        if (k == 4) tree_node_down_n<4, MODE, OUTS, T>(D, ok, qp, unif, first + a0, c0, h, Hp);
        else if (k == 3) tree_node_down_n<3, MODE, OUTS, T>(D, ok, qp, unif, first + a0, c0, h, Hp);
        else if (k == 2) tree_node_down_n<2, MODE, OUTS, T>(D, ok, qp, unif, first + a0, c0, h, Hp);
        else tree_node_down_n<1, MODE, OUTS, T>(D, ok, qp, unif, first + a0, c0, h, Hp);
    }
}

template <class T, int MODE, int OUTS>
__global__ void __launch_bounds__(TH_NT, (OUTS & TO_LB) ? TREE_MIN_CTAS_LB : TREE_MIN_CTAS)
    tree_kernel(DevGame G, DevPlayer P, int player, TreeArgs A) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    double* s_exptab = reinterpret_cast<double*>(sm_raw);        // [64] 2^(j/64) (fp64 exp only)
    T* tile = reinterpret_cast<T*>(s_exptab + 64);                // [n_pub][TH_HANDS]
    const int g = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (A.mask && A.mask[g] != A.want) return;
    const int Hp = G.H_pad, n_pub = P.n_pub, n_nodes = P.n_nodes, n_lv = P.n_levels;
    const int h0 = blockIdx.x * TH_HANDS;
    constexpr int mode = MODE;
    const bool has_grad = mode == TM_SBR || mode == TM_PROX || mode == TM_BR || mode == TM_CFR;
    T* rootv = tile + (size_t)n_pub * TH_HANDS;                   // [n_root][TH_HANDS]
    T* s_logn = rootv + (size_t)P.n_root * TH_HANDS;              // [n_nodes]
    T* s_wgt = s_logn + n_nodes;                                  // [n_nodes] (mu) beta_j (all-valid games)
    T* s_iw = s_wgt + n_nodes;                                    // [n_nodes] its reciprocal
    T* brv = s_iw + n_nodes;                                      // [n_int][TH_HANDS] fused BR: child values
    T* brroot = brv + (size_t)P.n_int * TH_HANDS;                 // [n_root][TH_HANDS] fused BR: root values
    int* s_first = reinterpret_cast<int*>(brroot + (size_t)P.n_root * TH_HANDS);
    int* s_nact = s_first + n_nodes;
    int* s_par = s_nact + n_nodes;
    int* s_bs = s_par + n_nodes;
    int* s_rslot = s_bs + n_nodes;
    int* s_sn = s_rslot + n_nodes;                                // [n_nodes]
    int* s_so = s_sn + n_nodes;                                   // [n_lv * TH_WARPS + 1]
    int* s_slot = s_so + n_lv * TH_WARPS + 1;                     // [n_pub]
    for (int i = tid; i < n_nodes; i += TH_NT) {
        s_first[i] = P.node_first[i];
        s_nact[i] = P.node_nact[i];
        s_par[i] = P.node_parent[i];
        s_bs[i] = P.node_bs[i];
        s_rslot[i] = P.root_slot[i];
        s_sn[i] = P.sched_nodes[i];
        s_logn[i] = log((T)P.node_nact[i]);
    }
    for (int i = tid; i <= n_lv * TH_WARPS; i += TH_NT) s_so[i] = P.sched_off[i];
    if (OUTS & TO_FUSEBR) {
        for (int i = tid; i < n_pub; i += TH_NT) s_slot[i] = P.seq_slot[i];
        for (int i = tid; i < P.n_int * TH_HANDS; i += TH_NT) brv[i] = T(0);
    }
    for (int i = tid; i < 64; i += TH_NT) s_exptab[i] = exp2((double)i / 64.0);
    const uint8_t* __restrict__ valid_g = G.tab_valid + (size_t)g * G.n_bs * Hp;
    const bool all_valid = G.all_valid != 0;
    // simplex weights: w_j = mu beta_j (SBR) or beta_j (prox); beta_j depends on the hand only
    // through board validity, so for all-valid games one value per node serves every hand
    const double wmu = mode == TM_SBR ? A.mu[g] : 1.0;
    if (all_valid)
        for (int i = tid; i < n_nodes; i += TH_NT) {
            const double w = wmu * P.beta[(size_t)i * Hp];
            s_wgt[i] = (T)w;
            s_iw[i] = (T)(1.0 / w);
        }

    // ---- gradient tile: asynchronous 16-byte copies (LDGSTS), all rows in flight.  The tile
    // keeps the raw gradient; the objective's scale sc = gsign (* step for prox) multiplies an
    // entry when a node reads it, and child values are pushed divided by sc.
    const double scd = mode == TM_PROX ? A.gsign * A.mu[g] : A.gsign;
    const T sc = (T)scd, inv_sc = (T)(1.0 / scd);
    if (has_grad) {
        const T* __restrict__ gp = A.g.at<T>(g) + h0;
        constexpr int EPC = 16 / sizeof(T);  // elements per 16-byte chunk
        constexpr int per_row = TH_HANDS / EPC;
        const int n_chunks = n_pub * per_row;
        for (int c = tid; c < n_chunks; c += TH_NT) {
            const int r = c / per_row, k = c % per_row;
            if (h0 + EPC * k < Hp) {
                const unsigned dst = smem_u32(tile + r * TH_HANDS + EPC * k);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gp + (size_t)r * Hp + EPC * k)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();

    // ---- fused best response (stopping test on the same gradient): min_q <q, sc g> bottom-up
    // on the untouched tile, children's values kept in brv (before the SBR pass edits the tile)
    if (OUTS & TO_FUSEBR) {
        for (int L = n_lv - 1; L >= 0; --L) {
            const int i0 = s_so[L * TH_WARPS + wid], i1 = s_so[L * TH_WARPS + wid + 1];
            for (int idx = i0; idx < i1; ++idx) {
                const int m = s_sn[idx];
                const int first = s_first[m], n = s_nact[m], par = s_par[m], rs = s_rslot[m];
#pragma unroll
                for (int j = 0; j < TH_HPL; ++j) {
                    const int c = lane + 32 * j, h = h0 + c;
                    T mn = T(0);
                    if (h < G.H && (all_valid || valid_g[(size_t)s_bs[m] * Hp + h])) {
                        mn = big_value<T>();
                        for (int a = 0; a < n; ++a) {
                            const int sq = first + a, sl = s_slot[sq];
                            const T x = sc * tile[sq * TH_HANDS + c] + (sl >= 0 ? brv[sl * TH_HANDS + c] : T(0));
                            mn = fmin(mn, x);
                        }
                    }
                    if (rs >= 0) brroot[rs * TH_HANDS + c] = mn;
                    else brv[s_slot[par] * TH_HANDS + c] += mn;
                }
            }
            __syncthreads();
        }
        double v = 0.0;
        if (wid == 0) {
#pragma unroll
            for (int j = 0; j < TH_HPL; ++j) {
                const int c = lane + 32 * j;
                if (h0 + c < G.H) {
                    v += scd * (double)tile[c];
                    for (int r = 0; r < P.n_root; ++r) v += (double)brroot[r * TH_HANDS + c];
                }
            }
        }
        v = warp_sum(v);
        game_value_reduce(v, A.br_partial, A.br_counter, A.br_value, g);
    }

    // ---- bottom-up, deepest level first
    TreeNodeCtx<T> C;
    C.cfr_plus = A.cfr_plus;
    C.cfr_scale = T(0);
    // CFR (reading R15): each hand's noise floor, the largest |g| over its sequences (the raw
    // tile; |gsign| = 1), taken before the bottom-up folds child values in
    T cfr_scale[TH_HPL];
#pragma unroll
    for (int j = 0; j < TH_HPL; ++j) {
        cfr_scale[j] = T(0);
        if (MODE == TM_CFR)
            for (int r = 1; r < n_pub; ++r) cfr_scale[j] = fmax(cfr_scale[j], fabs(tile[r * TH_HANDS + lane + 32 * j]));
    }
    C.mu = (mode == TM_SBR) ? (T)A.mu[g] : T(1);
    C.exptab = s_exptab;
    // the smoothed response's behavioural logs (R16), written during the bottom-up
    T* __restrict__ lbo = nullptr;
    if (mode == TM_SBR && (OUTS ? (OUTS & TO_LB) != 0 : A.out_lb.ok())) lbo = A.out_lb.at<T>(g);
    C.lbo = lbo;
    T* __restrict__ cz = A.center.ok() ? A.center.at<T>(g) : nullptr;
    T* __restrict__ rg = A.regret.ok() ? A.regret.at<T>(g) : nullptr;
    // CFR: the global rows a node's bottom-up work reads (current strategy and regrets): the next
    // node's are requested into L1 while this one is processed (-5 % on the CFR passes; the prox
    // centre's rows gained nothing from it and are left alone)
    auto prefetch_up = [&](int m2) {
        if (MODE != TM_CFR) return;
        const int f2 = s_first[m2], n2 = s_nact[m2];
        for (int a = 0; a < n2; ++a) {
            if (cz) asm volatile("prefetch.global.L1 [%0];" ::"l"(cz + (size_t)(f2 + a) * Hp + h0 + lane));
            if (rg) asm volatile("prefetch.global.L1 [%0];" ::"l"(rg + (size_t)(f2 + a) * Hp + h0 + lane));
        }
    };
    if (has_grad) {
        for (int L = n_lv - 1; L >= 0; --L) {
            const int i0 = s_so[L * TH_WARPS + wid], i1 = s_so[L * TH_WARPS + wid + 1];
            if (i0 < i1) prefetch_up(s_sn[i0]);
            for (int idx = i0; idx < i1; ++idx) {
                const int m = s_sn[idx];
                const int first = s_first[m], n = s_nact[m], par = s_par[m], rs = s_rslot[m];
                const T logn = s_logn[m];
                if (idx + 1 < i1) prefetch_up(s_sn[idx + 1]);
#pragma unroll
                for (int j = 0; j < TH_HPL; ++j) {
                    const int c = lane + 32 * j, h = h0 + c;
                    T* col = tile + (size_t)first * TH_HANDS + c;
                    T value = T(0);
                    if (h < G.H && (all_valid || valid_g[(size_t)s_bs[m] * Hp + h])) {
                        T wgt, iw;
                        if (all_valid) {
                            wgt = s_wgt[m];
                            iw = s_iw[m];
                        } else {
                            wgt = (T)(wmu * P.beta[(size_t)m * Hp + h]);
                            iw = T(1) / wgt;
                        }
                        if (MODE == TM_CFR) C.cfr_scale = cfr_scale[j];
                        // the log output is known at compile time for the hot (mode, outputs) kernels
                        constexpr int LB = OUTS ? ((OUTS & TO_LB) ? 1 : 0) : 2;
                        value = tree_node_up_any<MODE, T, LB>(C, P, col, first, n, m, h, Hp, logn, cz, rg, sc, wgt, iw);
                    } else {
                        for (int a = 0; a < n; ++a) col[a * TH_HANDS] = T(0);
                        if (lbo && h < Hp)
                            for (int a = 0; a < n; ++a) lbo[(size_t)(first + a) * Hp + h] = T(0);
                    }
                    if (rs >= 0) rootv[rs * TH_HANDS + c] = value;
                    else tile[par * TH_HANDS + c] += value * inv_sc;
                }
            }
            __syncthreads();
        }
    }

    // ---- per-game value: root entry + root simplexes' values, deterministic reductions
    if (A.value) {
        double v = 0.0;
        if (wid == 0) {
#pragma unroll
            for (int j = 0; j < TH_HPL; ++j) {
                const int c = lane + 32 * j;
                if (h0 + c < G.H) {
                    double u = scd * (double)tile[c];
                    for (int r = 0; r < P.n_root; ++r) u += (double)rootv[r * TH_HANDS + c];
                    v += u;
                }
            }
        }
        v = warp_sum(v);
        game_value_reduce(v, A.partial, A.counter, A.value, g);
    }

    // ---- top-down, shallowest level first
    const bool want_td = OUTS ? (OUTS & ~(TO_FUSEBR | TO_LB | TO_VAL)) != 0
                              : (A.out_b.ok() || A.out_q.ok() || A.comb_out.ok() || mode == TM_CFR);
    if (!want_td) return;
    T* __restrict__ ob = A.out_b.ok() ? A.out_b.at<T>(g) : nullptr;
    if ((OUTS & ~(TO_FUSEBR | TO_LB)) == TO_B && has_grad) {
        // behavioural output only: after the bottom-up every action column of the tile holds its
        // b (0 where the hand is blocked or past H), so no level-by-level descent is needed --
        // one coalesced row-by-row copy, row 0 = 1 for live hands.
        for (int i = tid; i < n_pub * TH_HANDS; i += TH_NT) {
            const int r = i / TH_HANDS, c = i % TH_HANDS, h = h0 + c;
            if (h < Hp) ob[(size_t)r * Hp + h] = r == 0 ? (h < G.H ? T(1) : T(0)) : tile[i];
        }
        return;
    }
    T* __restrict__ oq = A.out_q.ok() ? A.out_q.at<T>(g) : nullptr;
    const T* __restrict__ ci = A.comb_in.ok() ? A.comb_in.at<T>(g) : nullptr;
    T* __restrict__ co = A.comb_out.ok() ? A.comb_out.at<T>(g) : nullptr;
    T* __restrict__ av = A.avg.ok() ? A.avg.at<T>(g) : nullptr;
    const T tau = A.tau ? (T)A.tau[g] : T(0);
    T alpha = T(0);
    if (av) {
        const double t = (double)A.iter[g];
        alpha = (T)(A.avg_linear ? 2.0 * t / (t * t + t) : 1.0 / t);
    }
    const T* __restrict__ bin = (mode == TM_COMBINE) ? cz : nullptr;
    TreeDownCtx<T> Dn;
    Dn.tau = tau;
    Dn.alpha = alpha;
    Dn.exptab = s_exptab;
    Dn.bin = bin;
    Dn.ci = ci;
    Dn.ob = ob;
    Dn.oq = oq;
    Dn.co = co;
    Dn.av = av;
    if (wid == 0) {
#pragma unroll
        for (int j = 0; j < TH_HPL; ++j) {
            const int h = h0 + lane + 32 * j;
            if (h < Hp) {
                const bool live = h < G.H;
                const T q0 = live ? T(1) : T(0);
                if (ob) ob[h] = q0;
                if (oq) oq[h] = q0;
                if (co) co[h] = live ? (T(1) - tau) * ci[h] + tau : T(0);
                if (av) av[h] = q0;
            }
        }
    }
    // the global rows a node's descent reads (convex-combination input, behavioural input,
    // running average): the next node's are requested into L1 while this one is processed
    const T* pf_src[3] = {ci, bin, av};
    auto prefetch_node = [&](int m2) {
        const int f2 = s_first[m2], n2 = s_nact[m2];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (pf_src[k])
                for (int a = 0; a < n2; ++a)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(pf_src[k] + (size_t)(f2 + a) * Hp + h0 + lane));
    };
    for (int L = 0; L < n_lv; ++L) {
        const int i0 = s_so[L * TH_WARPS + wid], i1 = s_so[L * TH_WARPS + wid + 1];
        if (i0 < i1) prefetch_node(s_sn[i0]);
        for (int idx = i0; idx < i1; ++idx) {
            const int m = s_sn[idx];
            const int first = s_first[m], n = s_nact[m], par = s_par[m];
            if (idx + 1 < i1) prefetch_node(s_sn[idx + 1]);
#pragma unroll
            for (int j = 0; j < TH_HPL; ++j) {
                const int c = lane + 32 * j, h = h0 + c;
                const bool ok = h < G.H && (all_valid || valid_g[(size_t)s_bs[m] * Hp + h]);
                const T qp = par == 0 ? (ok ? T(1) : T(0)) : tile[par * TH_HANDS + c];
                tree_node_down_any<MODE, OUTS, T>(Dn, ok, qp, first, n, tile + (size_t)first * TH_HANDS + c, h, Hp);
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_tree(const DevGame& G, const DevPlayer& P, int player, const TreeArgs& A, cudaStream_t st) {
    dim3 grid((G.H_pad + TH_HANDS - 1) / TH_HANDS, G.n_games);
    const size_t sm = tree_smem_bytes(P, G.esz);
    const int outs = (A.out_b.ok() ? TO_B : 0) | (A.out_q.ok() ? TO_Q : 0) | (A.comb_out.ok() ? TO_COMB : 0) |
                     (A.avg.ok() ? TO_AVG : 0) | (A.out_lb.ok() ? TO_LB : 0);
    if (A.out_lb.ok() && A.mode != TM_SBR) return cudaErrorInvalidValue;
#define EGT_TREE_GO(M, O)                                                                       \
    {                                                                                           \
        if (G.esz == 4) tree_kernel<float, M, O><<<grid, TH_NT, sm, st>>>(G, P, player, A);     \
        else tree_kernel<double, M, O><<<grid, TH_NT, sm, st>>>(G, P, player, A);               \
        return cudaGetLastError();                                                              \
    }
    if (A.br_value) {  // the fused stopping test exists for the excessive-gap check's SBR only
        if (A.mode != TM_SBR || outs != (TO_LB | TO_Q)) return cudaErrorInvalidValue;
        EGT_TREE_GO(TM_SBR, TO_LB | TO_Q | TO_FUSEBR)
    }
    // the solver's hot (mode, outputs) combinations get fully specialised kernels
    if (A.mode == TM_SBR && outs == (TO_LB | TO_Q)) EGT_TREE_GO(TM_SBR, TO_LB | TO_Q)
    if (A.mode == TM_SBR && outs == TO_Q) EGT_TREE_GO(TM_SBR, TO_Q)
    if (A.mode == TM_SBR && outs == 0 && A.value) EGT_TREE_GO(TM_SBR, TO_VAL)  // value only: no descent
    if (A.mode == TM_SBR && outs == (TO_Q | TO_COMB)) EGT_TREE_GO(TM_SBR, TO_Q | TO_COMB)
    if (A.mode == TM_PROX && outs == TO_COMB) EGT_TREE_GO(TM_PROX, TO_COMB)
    if (A.mode == TM_COMBINE && outs == TO_COMB) EGT_TREE_GO(TM_COMBINE, TO_COMB)
    if (A.mode == TM_CFR && outs == (TO_Q | TO_AVG)) EGT_TREE_GO(TM_CFR, TO_Q | TO_AVG)
#define EGT_TREE_LAUNCH(M)                                                                            \
    case M:                                                                                           \
        if (G.esz == 4) tree_kernel<float, M, 0><<<grid, TH_NT, sm, st>>>(G, P, player, A);           \
        else tree_kernel<double, M, 0><<<grid, TH_NT, sm, st>>>(G, P, player, A);                     \
        break;
    switch (A.mode) {  // otherwise one kernel per mode, outputs decided at run time
        EGT_TREE_LAUNCH(TM_SBR)
        EGT_TREE_LAUNCH(TM_PROX)
        EGT_TREE_LAUNCH(TM_BR)
        EGT_TREE_LAUNCH(TM_CFR)
        EGT_TREE_LAUNCH(TM_UNIFORM)
        EGT_TREE_LAUNCH(TM_COMBINE)
        default: return cudaErrorInvalidValue;
    }
#undef EGT_TREE_GO
#undef EGT_TREE_LAUNCH
    return cudaGetLastError();
}

template <class T>
static cudaError_t prepare_t() {
    const int lim = 200 * 1024;
    cudaError_t e = cudaFuncSetAttribute(grad_kernel<GRAD_NT, GRAD_KMAX, GRAD_EMAX, T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grad_staged_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grad_staged_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grad_card_kernel<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(grad_card_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    const void* tk[] = {(const void*)tree_kernel<T, TM_SBR, 0>,     (const void*)tree_kernel<T, TM_PROX, 0>,
                        (const void*)tree_kernel<T, TM_BR, 0>,      (const void*)tree_kernel<T, TM_CFR, 0>,
                        (const void*)tree_kernel<T, TM_UNIFORM, 0>, (const void*)tree_kernel<T, TM_COMBINE, 0>,
                        (const void*)tree_kernel<T, TM_SBR, TO_LB | TO_Q>, (const void*)tree_kernel<T, TM_SBR, TO_Q | TO_COMB>,
                        (const void*)tree_kernel<T, TM_SBR, TO_Q>, (const void*)tree_kernel<T, TM_SBR, TO_VAL>,
                        (const void*)tree_kernel<T, TM_PROX, TO_COMB>, (const void*)tree_kernel<T, TM_COMBINE, TO_COMB>,
                        (const void*)tree_kernel<T, TM_CFR, TO_Q | TO_AVG>,
                        (const void*)tree_kernel<T, TM_SBR, TO_LB | TO_Q | TO_FUSEBR>};
    for (const void* f : tk)
        if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    return e;
}

cudaError_t kernels_prepare() {
    cudaError_t e = prepare_t<double>();
    return e == cudaSuccess ? prepare_t<float>() : e;
}

// ------------------------------------------------------------------ per-game scalars
// variant 0 theory (Alg. 1), 1 mu-balanced, 2 EGT/as (Alg. 3-4).
__global__ void egt_prepare_kernel(int variant, int n, DevScalars S) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    // Alg. 3's "while eps_sad > eps" per game: a game whose maintained gap
    // reached its target stops -- focus -1 and live 0 mask every launch of the iteration
    if (variant == 2 && S.target[g] > 0.0 && S.gap[g] <= S.target[g]) S.live[g] = 0;
    if (!S.live[g]) {
        S.focus[g] = -1;
        return;
    }
    const double mx = S.mu[g], my = S.mu[n + g];
    int focus;
    if (variant == 0) focus = (S.t[g] & 1);           // even t: x (Alg. 1 lines 6-9)
    else focus = mx > my ? 0 : 1;                     // PAPER.md:548-549, Alg. 3 line 6
    double tau = variant == 2 ? S.tau[g] : 2.0 / (S.t[g] + 3.0);   // Alg. 1 line 5 / Alg. 3 line 4
    S.tau[g] = tau;
    S.focus[g] = focus;
    const double muf = focus == 0 ? mx : my;
    S.mu_cand[g] = focus == 0 ? (1.0 - tau) * mx : mx;             // Alg. 2 line 5
    S.mu_cand[n + g] = focus == 1 ? (1.0 - tau) * my : my;
    S.step[g] = tau / ((1.0 - tau) * muf);                          // Alg. 2 line 3
}

__global__ void egt_accept_kernel(int variant, int n, DevScalars S) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n || !S.live[g]) return;
    S.attempts[g] += 1;
    bool accept = true;
    if (variant == 2) {
        const double egv = S.val[g] + S.val[n + g];   // phi_{mu_x}(y+) - f_{mu_y}(x+)
        S.egv[g] = egv;
        accept = egv >= 0.0;                          // Alg. 4 line 2 (R8)
    }
    if (accept) {
        S.cur[g] ^= 1;
        S.mu[g] = S.mu_cand[g];
        S.mu[n + g] = S.mu_cand[n + g];
        S.t[g] += 1;
        // eps_sad of the accepted candidate from the best responses to the check's gradients
        // (PAPER.md:311); a rejected attempt leaves the iterate, and its gap, unchanged
        if (variant == 2) S.gap[g] = -S.brval[n + g] - S.brval[g];
    } else {
        S.tau[g] *= 0.5;                              // Alg. 4 line 3
        S.backtracks[g] += 1;
        if (S.tau[g] < 1e-12) S.fail[g] = 1;
    }
}

__global__ void tick_kernel(int n, int* t, const int* live) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n && (!live || live[g])) t[g] += 1;
}

// A CFR game whose evaluated eps_sad (of its average) reached its target stops (egt_set_target)
__global__ void stop_at_target_kernel(int n, const double* __restrict__ gap, const double* __restrict__ target,
                                      int* live) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n && target[g] > 0.0 && gap[g] <= target[g]) live[g] = 0;
}

cudaError_t launch_stop_at_target(int n, const double* gap, const double* target, int* live, cudaStream_t st) {
    stop_at_target_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, gap, target, live);
    return cudaGetLastError();
}


// eps_sad per game from the two best-response values:
// val[g] = min_x <x, A y>, val[n+g] = min_y <y, -A^T x> = -max_y <x, A y>.
__global__ void gap_combine_kernel(int n, const double* __restrict__ val, double* __restrict__ out) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) out[g] = -val[n + g] - val[g];
}

cudaError_t launch_gap_combine(int n, const double* val, double* out, cudaStream_t st) {
    gap_combine_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, val, out);
    return cudaGetLastError();
}

// The practical-mu scan of egt_init (R14), one thread per game.  phase 0: before
// trial k, the trial mu = mu_theory * 2^-k of the games still scanning; phase 1: after it, the
// EGC at the trial's initial point (EGV = val[g] + val[n + g] >= 0) keeps k, else the scan of
// that game ends; phase 2: mu = mu_theory * 2^-k for the last k that kept it.
__global__ void mu_scan_kernel(int n, int k, int phase, const double* __restrict__ mu_th, double* mu, int* scan,
                               int* kbest, const double* __restrict__ val) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    if (phase == 0) {
        if (scan[g]) {
            mu[g] = mu_th[g] * ldexp(1.0, -k);
            mu[n + g] = mu_th[n + g] * ldexp(1.0, -k);
        }
    } else if (phase == 1) {
        if (scan[g]) {
            if (val[g] + val[n + g] >= 0.0) kbest[g] = k;  // Alg. 4's test, EGV >= 0 (R8)
            else scan[g] = 0;
        }
    } else {
        mu[g] = mu_th[g] * ldexp(1.0, -kbest[g]);
        mu[n + g] = mu_th[n + g] * ldexp(1.0, -kbest[g]);
    }
}

cudaError_t launch_mu_scan(int n, int k, int phase, const double* mu_th, double* mu, int* scan, int* kbest,
                           const double* val, cudaStream_t st) {
    mu_scan_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, k, phase, mu_th, mu, scan, kbest, val);
    return cudaGetLastError();
}

// Emulated all-reduce (egt_shard_emulate): every buffer becomes the elementwise sum of the
// `world` buffers, in rank order.
template <class T>
__global__ void emu_allreduce_kernel(double* const* __restrict__ bufs, int world, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        T s = T(0);
        for (int r = 0; r < world; ++r) s += reinterpret_cast<const T*>(bufs[r])[i];
        for (int r = 0; r < world; ++r) reinterpret_cast<T*>(bufs[r])[i] = s;
    }
}

cudaError_t launch_emu_allreduce(double* const* bufs, int world, size_t n, int esz, cudaStream_t st) {
    if (esz == 4) emu_allreduce_kernel<float><<<148 * 8, 256, 0, st>>>(bufs, world, n);
    else emu_allreduce_kernel<double><<<148 * 8, 256, 0, st>>>(bufs, world, n);
    return cudaGetLastError();
}

cudaError_t launch_egt_prepare(int variant, int n, DevScalars S, cudaStream_t st) {
    egt_prepare_kernel<<<(n + 127) / 128, 128, 0, st>>>(variant, n, S);
    return cudaGetLastError();
}
cudaError_t launch_egt_accept(int variant, int n, DevScalars S, cudaStream_t st) {
    egt_accept_kernel<<<(n + 127) / 128, 128, 0, st>>>(variant, n, S);
    return cudaGetLastError();
}
cudaError_t launch_tick(int n, int* t, const int* live, cudaStream_t st) {
    tick_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, t, live);
    return cudaGetLastError();
}

}  // namespace egt
