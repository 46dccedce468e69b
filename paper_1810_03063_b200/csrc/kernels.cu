// sm_100a kernels of the EGT / CFR hot path (fp64).
//
//  grad_kernel  : g = A y (player 0) or g = A^T x (player 1) without materialising A
//                 (PAPER.md:299 gradient operators; Gen-CFR lines 29/35).
//  tree_kernel  : one pass over a player's treeplex per (game, tile of hands):
//                 bottom-up per simplex (smoothed best response PAPER.md:467-512,
//                 prox mapping PAPER.md:514-537, best response, or the CFR regret
//                 update PAPER.md:30-39/63-64/84-85), then top-down rescale by the
//                 parent sequence with the EGT convex combinations fused.
#include <cfloat>
#include <cmath>

#include "kernels.cuh"
#include "game.h"  // ENT_* packing of the card-array entries

namespace egt {

// ------------------------------------------------------------------ warp helpers
__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// exclusive prefix at index r in [0, 64] of a 64-entry segment held as (ex0 at lane r,
// ex1 at lane r - 32); r = 64 gives the total.  Every lane must call it.
__device__ __forceinline__ double seg_prefix(double ex0, double ex1, double tot, int r) {
    const double u = __shfl_sync(0xffffffffu, ex0, r & 31);
    const double v = __shfl_sync(0xffffffffu, ex1, r & 31);
    return r < 32 ? u : (r < 64 ? v : tot);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ gradient
// One CTA per (public sequence s of `player` that ends a terminal, game g).  For every
// terminal t whose last `player` sequence is s (hands of `player`: "self", of the other
// player: "opp"), with hands in ascending showdown strength (positions i):
//   w[i] = prior_opp(h_i) * v_opp[seq_opp(t), h_i],  P = exclusive prefix sums of w,
//   for every card c: the entries of w over the hands holding c, in strength order, and
//   their exclusive prefix sums Pc; S_c their total.
//   fold:     v(h) = u2 * sum_{opp h' disjoint from h} w(h') = T - sum_{c in h} S_c + [|h|=2] w(h)
//   showdown: v(h) = sign * W * (stronger(h) - weaker(h)) over disjoint opp hands, with
//             weaker   = P[lo] - sum_c Pc[lo],  stronger = (T - P[hi]) - sum_c (S_c - Pc[hi])
//             ([lo, hi) = h's tie group), i.e.  v = T - P[hi] - P[lo] + sum_c (Pc[lo] + Pc[hi] - S_c).
//   g[s, h] += kappa_t * kappa_game * prior_self(h) * v(h)
// sign = +1 for player 0 (A y: player 2 wins with the stronger hand), -1 for player 1.
// P is a block scan over register-resident chunks (K consecutive positions per thread);
// the card sums are one warp per card (segments <= 64 entries, two per lane).
template <int NT, int KMAX>
__global__ void __launch_bounds__(NT, 4) grad_kernel(DevGame G, DevPlayer P, int player, VecRef vin, VecRef gout,
                                                  const int* __restrict__ mask, int want, int all_rows) {
    extern __shared__ double sm[];
    __shared__ double wtot[NT / 32];
    constexpr int NW = NT / 32;
    const int g = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (mask && mask[g] != want) return;
    const int s = all_rows ? (int)blockIdx.x : P.rows_term[blockIdx.x];
    const int Hp = G.H_pad, hs = G.hand_size;
    double* w = sm;                // [Hp]   by position
    double* Pf = w + Hp;           // [Hp+1] by position
    double* corr = Pf + Hp + 1;    // [2][Hp] by position
    double* acc = corr + 2 * Hp;   // [Hp]   by hand
    for (int i = tid; i < Hp; i += NT) acc[i] = 0.0;
    const int t0 = P.term_off[s], t1 = P.term_off[s + 1];
    const double* __restrict__ popp = (player ? G.prior[0] : G.prior[1]) + (size_t)g * Hp;
    const double* __restrict__ vo = vin.at(g);
    const double kg = G.kappa_game[g];
    const double sd_sign = player == 0 ? 1.0 : -1.0;
    for (int ti = t0; ti < t1; ++ti) {
        const DevTerm T = G.terms[P.term_idx[ti]];
        const int k = g * G.n_bs + T.bs;
        const int nv = G.tab_nvalid[k];
        const int16_t* __restrict__ order = G.tab_order + (size_t)k * Hp;
        const uint32_t* __restrict__ lohi = G.tab_lohi + (size_t)k * Hp;
        const int16_t* __restrict__ seg = G.tab_seg + (size_t)k * (G.n_cards + 1);
        const uint32_t* __restrict__ ent = G.tab_ent + (size_t)k * 2 * Hp;
        const int so = player ? T.seq[0] : T.seq[1];
        const double* __restrict__ vrow = vo + (size_t)so * Hp;
        const int K = (nv + NT - 1) / NT;
        const int base = tid * K;
        // ---- phase A: w in registers (K consecutive positions per thread), block exclusive scan
        double x[KMAX];
        double run = 0.0;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            x[j] = 0.0;
            const int i = base + j;
            if (j < K && i < nv) {
                const int h = order[i];
                x[j] = popp[h] * (so ? vrow[h] : 1.0);
                w[i] = x[j];
                run += x[j];
            }
        }
        __syncthreads();  // previous terminal done with Pf / corr; acc writes ordered
        const double incl = warp_incl_scan(run, lane);
        if (lane == 31) wtot[wid] = incl;
        __syncthreads();
        double wpre = 0.0, total = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            const double v = wtot[q];
            wpre += q < wid ? v : 0.0;
            total += v;
        }
        double pre = wpre + incl - run;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            const int i = base + j;
            if (j < K && i < nv) {
                Pf[i] = pre;
                pre += x[j];
            }
        }
        if (tid == 0) Pf[nv] = total;
        __syncthreads();
        // ---- phase B: per-card sums, one warp per card
        const bool sd = T.kind == 2;
        for (int c = wid; c < G.n_cards; c += NW) {
            const int a = seg[c], len = seg[c + 1] - a;
            if (len == 0) continue;
            const uint32_t e0 = lane < len ? ent[a + lane] : 0u;
            const uint32_t e1 = lane + 32 < len ? ent[a + lane + 32] : 0u;
            const double x0 = lane < len ? w[ENT_POS(e0)] : 0.0;
            const double x1 = lane + 32 < len ? w[ENT_POS(e1)] : 0.0;
            const double s0 = warp_incl_scan(x0, lane);
            const double s1 = warp_incl_scan(x1, lane);
            const double tot0 = __shfl_sync(0xffffffffu, s0, 31);
            const double Sc = tot0 + __shfl_sync(0xffffffffu, s1, 31);
            const double ex0 = s0 - x0, ex1 = tot0 + s1 - x1;
            // lanes beyond len hold 0, so index len gives the total
            double d0 = -Sc, d1 = -Sc;
            if (sd) {
                d0 += seg_prefix(ex0, ex1, Sc, ENT_RELO(e0)) + seg_prefix(ex0, ex1, Sc, ENT_REHI(e0));
                d1 += seg_prefix(ex0, ex1, Sc, ENT_RELO(e1)) + seg_prefix(ex0, ex1, Sc, ENT_REHI(e1));
            }
            if (lane < len) corr[ENT_SLOT(e0) * Hp + ENT_POS(e0)] = d0;
            if (lane + 32 < len) corr[ENT_SLOT(e1) * Hp + ENT_POS(e1)] = d1;
        }
        __syncthreads();
        // ---- phase C: per hand
        const double scale = T.kappa * kg * T.amount;
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            const int i = base + j;
            if (j < K && i < nv) {
                double v = total + corr[i];
                if (hs == 2) v += corr[Hp + i];
                if (sd) {
                    const uint32_t lh = lohi[i];
                    v = sd_sign * (v - Pf[lh & 0xFFFFu] - Pf[lh >> 16]);
                } else if (hs == 2) {
                    v += x[j];
                }
                acc[order[i]] += scale * v;
            }
        }
    }
    __syncthreads();
    const double* __restrict__ pself = (player ? G.prior[1] : G.prior[0]) + (size_t)g * Hp;
    double* __restrict__ out = gout.at(g) + (size_t)s * Hp;
    for (int i = tid; i < Hp; i += NT) out[i] = pself[i] * acc[i];
}

static constexpr int GRAD_NT = 256, GRAD_KMAX = 5;

static size_t grad_smem_bytes(int Hp) { return sizeof(double) * (size_t)(5 * Hp + 1); }

cudaError_t launch_gradient(const DevGame& G, const DevPlayer& P, int player, VecRef vin, VecRef gout,
                            const int* mask, int want, int all_rows, cudaStream_t st) {
    const int rows = all_rows ? P.n_pub : P.n_rows_term;
    if (rows == 0) return cudaSuccess;
    dim3 grid(rows, G.n_games);
    grad_kernel<GRAD_NT, GRAD_KMAX><<<grid, GRAD_NT, grad_smem_bytes(G.H_pad), st>>>(G, P, player, vin, gout, mask,
                                                                                    want, all_rows);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ treeplex pass
// CTA = (TH_HANDS hands, game); TH_WARPS warps.  The player's whole gradient tile
// [n_pub][TH_HANDS] is staged in shared memory (lane = hand).  Bottom-up, level by level
// (deepest first; nodes of a level are independent and spread over the warps), each
// simplex j = (node m, hand) pulls the values of its child simplexes (D_j^i) into its
// entries, solves its local problem (softmax / prox / argmin / regret
// matching), overwrites its entries with the behavioural strategy and stores its value in
// val[m].  Top-down (shallowest first) each entry becomes q_i = q_{p_j} * qbar_i in place,
// and the requested outputs (behavioural, sequence form, EGT convex combinations, CFR
// average) are written row by row (coalesced, 32 hands per row).
static constexpr int TH_HANDS = 32, TH_WARPS = 8, TH_NT = TH_HANDS * TH_WARPS;

size_t tree_smem_bytes(const DevPlayer& P) {
    return sizeof(double) * (size_t)TH_HANDS * (P.n_pub + P.n_nodes) +
           sizeof(int) * (size_t)(6 * P.n_nodes + P.n_pub + 1 + P.n_levels + 1);
}

__global__ void __launch_bounds__(TH_NT, 4) tree_kernel(DevGame G, DevPlayer P, int player, TreeArgs A) {
    extern __shared__ double tile[];
    const int g = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (A.mask && A.mask[g] != A.want) return;
    const int Hp = G.H_pad, n_pub = P.n_pub, n_nodes = P.n_nodes, n_lv = P.n_levels;
    const int h = blockIdx.x * TH_HANDS + lane;
    const bool live = h < G.H;
    const int mode = A.mode;
    const bool has_grad = mode == TM_SBR || mode == TM_PROX || mode == TM_BR || mode == TM_CFR;
    double* val = tile + (size_t)n_pub * TH_HANDS;  // [n_nodes][TH_HANDS]
    int* s_first = reinterpret_cast<int*>(val + (size_t)n_nodes * TH_HANDS);
    int* s_nact = s_first + n_nodes;
    int* s_par = s_nact + n_nodes;
    int* s_bs = s_par + n_nodes;
    int* s_lvn = s_bs + n_nodes;       // [n_nodes]
    int* s_kidoff = s_lvn + n_nodes;   // [n_pub+1]
    int* s_kids = s_kidoff + n_pub + 1; // [n_nodes]
    int* s_lvoff = s_kids + n_nodes;   // [n_lv+1]
    for (int i = tid; i < n_nodes; i += TH_NT) {
        s_first[i] = P.node_first[i];
        s_nact[i] = P.node_nact[i];
        s_par[i] = P.node_parent[i];
        s_bs[i] = P.node_bs[i];
        s_lvn[i] = P.lvl_nodes[i];
        s_kids[i] = P.kids[i];
    }
    for (int i = tid; i <= n_pub; i += TH_NT) s_kidoff[i] = P.kid_off[i];
    for (int i = tid; i <= n_lv; i += TH_NT) s_lvoff[i] = P.lvl_off[i];
    const uint8_t* __restrict__ valid_g = G.tab_valid + (size_t)g * G.n_bs * Hp;
    const bool all_valid = G.all_valid != 0;

    // ---- load the gradient tile (one 32-hand row per warp instruction)
    if (has_grad) {
        const double* __restrict__ gp = A.g.at(g);
        double sc = A.gsign;
        if (mode == TM_PROX) sc *= A.mu[g];
        for (int r = wid; r < n_pub; r += TH_WARPS)
            tile[r * TH_HANDS + lane] = live ? sc * gp[(size_t)r * Hp + h] : 0.0;
    }
    __syncthreads();

    // ---- bottom-up, deepest level first
    const double mu = (mode == TM_SBR) ? A.mu[g] : 1.0;
    double* __restrict__ cz = A.center.ok() ? A.center.at(g) : nullptr;
    double* __restrict__ rg = A.regret.ok() ? A.regret.at(g) : nullptr;
    if (has_grad) {
        for (int L = n_lv - 1; L >= 0; --L) {
            for (int idx = s_lvoff[L] + wid; idx < s_lvoff[L + 1]; idx += TH_WARPS) {
                const int m = s_lvn[idx];
                const int first = s_first[m], n = s_nact[m];
                double* col = tile + (size_t)first * TH_HANDS + lane;
                const bool ok = live && (all_valid || valid_g[(size_t)s_bs[m] * Hp + h]);
                if (!ok) {
                    for (int a = 0; a < n; ++a) col[a * TH_HANDS] = 0.0;
                    val[m * TH_HANDS + lane] = 0.0;
                    continue;
                }
                // pull the child simplexes' values into this simplex's entries (D_j^i)
                for (int a = 0; a < n; ++a) {
                    const int s = first + a;
                    double x = col[a * TH_HANDS];
                    for (int c = s_kidoff[s]; c < s_kidoff[s + 1]; ++c) x += val[s_kids[c] * TH_HANDS + lane];
                    col[a * TH_HANDS] = x;
                }
                double value;
                if (mode == TM_SBR) {
                    // qbar_i ~ exp(-g_i / w), value = g_{i*} + w log qbar_{i*} + w log n with
                    // i* = argmax qbar, w = mu beta_j
                    const double wgt = mu * P.beta[(size_t)m * Hp + h];
                    double mn = DBL_MAX;
                    for (int a = 0; a < n; ++a) mn = fmin(mn, col[a * TH_HANDS]);
                    double S = 0.0;
                    for (int a = 0; a < n; ++a) {
                        const double e = exp(-(col[a * TH_HANDS] - mn) / wgt);
                        col[a * TH_HANDS] = e;
                        S += e;
                    }
                    const double inv = 1.0 / S;
                    for (int a = 0; a < n; ++a) col[a * TH_HANDS] *= inv;
                    value = mn - wgt * log(S) + wgt * log((double)n);
                } else if (mode == TM_PROX) {
                    // shifted-gradient SBR in multiplicative form:
                    // qbar_i ~ zbar_i exp(-g_i / beta), value = -beta log sum_i zbar_i exp(-g_i / beta)
                    const double beta = P.beta[(size_t)m * Hp + h];
                    const double* __restrict__ zr = cz + (size_t)first * Hp + h;
                    double mn = DBL_MAX;
                    for (int a = 0; a < n; ++a)
                        if (zr[(size_t)a * Hp] > 0.0) mn = fmin(mn, col[a * TH_HANDS]);
                    double S = 0.0;
                    for (int a = 0; a < n; ++a) {
                        const double za = zr[(size_t)a * Hp];
                        const double e = za > 0.0 ? za * exp(-(col[a * TH_HANDS] - mn) / beta) : 0.0;
                        col[a * TH_HANDS] = e;
                        S += e;
                    }
                    const double inv = 1.0 / S;
                    for (int a = 0; a < n; ++a) col[a * TH_HANDS] *= inv;
                    value = mn - beta * log(S);
                } else if (mode == TM_BR) {
                    int best = 0;
                    double mn = col[0];
                    for (int a = 1; a < n; ++a) {
                        const double v = col[a * TH_HANDS];
                        if (v < mn) {
                            mn = v;
                            best = a;
                        }
                    }
                    for (int a = 0; a < n; ++a) col[a * TH_HANDS] = a == best ? 1.0 : 0.0;
                    value = mn;
                } else {  // TM_CFR: utility u = gsign * g, current strategy z, regrets r
                    double v = 0.0;
                    for (int a = 0; a < n; ++a) v += col[a * TH_HANDS] * cz[(size_t)(first + a) * Hp + h];
                    double S = 0.0;
                    for (int a = 0; a < n; ++a) {
                        const size_t ix = (size_t)(first + a) * Hp + h;
                        const double u = col[a * TH_HANDS], r0 = rg[ix];
                        double r = r0 + u - v;
                        if (A.cfr_plus) r = fmax(r, 0.0);
                        rg[ix] = r;
                        // DESIGN.md R15: regrets at the rounding-noise level of their own update count as 0
                        const double tol = 1e-13 * (fabs(r0) + fabs(u) + fabs(v));
                        const double pr = r > tol ? r : 0.0;
                        col[a * TH_HANDS] = pr;
                        S += pr;
                    }
                    for (int a = 0; a < n; ++a) {
                        const double z = S > 0.0 ? col[a * TH_HANDS] / S : 1.0 / n;
                        col[a * TH_HANDS] = z;
                        cz[(size_t)(first + a) * Hp + h] = z;
                    }
                    value = v;
                }
                val[m * TH_HANDS + lane] = value;
            }
            __syncthreads();
        }
    }

    // ---- per-game value: root entry + root simplexes' values, deterministic reductions
    if (A.value) {
        double v = 0.0;
        if (wid == 0 && live) {
            v = tile[lane];
            for (int c = s_kidoff[0]; c < s_kidoff[1]; ++c) v += val[s_kids[c] * TH_HANDS + lane];
        }
        v = warp_sum(v);
        __shared__ bool last;
        if (tid == 0) {
            A.partial[(size_t)g * gridDim.x + blockIdx.x] = v;
            __threadfence();
            const unsigned ticket = atomicAdd(&A.counter[g], 1u);
            last = ticket == gridDim.x - 1;
        }
        __syncthreads();
        if (last && tid == 0) {
            __threadfence();
            double s = 0.0;
            const volatile double* pp = A.partial + (size_t)g * gridDim.x;
            for (unsigned i = 0; i < gridDim.x; ++i) s += pp[i];
            A.value[g] = s;
            A.counter[g] = 0;
        }
    }

    // ---- top-down, shallowest level first
    const bool want_td = A.out_b.ok() || A.out_q.ok() || A.comb_out.ok() || mode == TM_CFR;
    if (!want_td) return;
    double* __restrict__ ob = A.out_b.ok() ? A.out_b.at(g) : nullptr;
    double* __restrict__ oq = A.out_q.ok() ? A.out_q.at(g) : nullptr;
    const double* __restrict__ ci = A.comb_in.ok() ? A.comb_in.at(g) : nullptr;
    double* __restrict__ co = A.comb_out.ok() ? A.comb_out.at(g) : nullptr;
    double* __restrict__ av = A.avg.ok() ? A.avg.at(g) : nullptr;
    const double tau = A.tau ? A.tau[g] : 0.0;
    double alpha = 0.0;
    if (av) {
        const double t = (double)A.iter[g];
        alpha = A.avg_linear ? 2.0 * t / (t * t + t) : 1.0 / t;
    }
    const double* __restrict__ bin = (mode == TM_COMBINE) ? cz : nullptr;
    const bool hvalid = h < Hp;
    if (wid == 0 && hvalid) {
        const double q0 = live ? 1.0 : 0.0;
        if (ob) ob[h] = q0;
        if (oq) oq[h] = q0;
        if (co) co[h] = live ? (1.0 - tau) * ci[h] + tau : 0.0;
        if (av) av[h] = q0;
    }
    for (int L = 0; L < n_lv; ++L) {
        for (int idx = s_lvoff[L] + wid; idx < s_lvoff[L + 1]; idx += TH_WARPS) {
            const int m = s_lvn[idx];
            const int first = s_first[m], n = s_nact[m], par = s_par[m];
            const bool ok = live && (all_valid || valid_g[(size_t)s_bs[m] * Hp + h]);
            const double qp = par == 0 ? (live ? 1.0 : 0.0) : tile[par * TH_HANDS + lane];
            for (int a = 0; a < n; ++a) {
                const int s = first + a;
                double b;
                if (!ok) b = 0.0;
                else if (mode == TM_UNIFORM) b = 1.0 / n;
                else if (mode == TM_COMBINE) b = bin[(size_t)s * Hp + h];
                else b = tile[s * TH_HANDS + lane];
                const double q = qp * b;
                tile[s * TH_HANDS + lane] = q;
                if (hvalid) {
                    const size_t ix = (size_t)s * Hp + h;
                    if (ob) ob[ix] = b;
                    if (oq) oq[ix] = q;
                    if (co) co[ix] = (1.0 - tau) * ci[ix] + tau * q;
                    if (av) av[ix] = alpha * q + (1.0 - alpha) * av[ix];
                }
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_tree(const DevGame& G, const DevPlayer& P, int player, const TreeArgs& A, cudaStream_t st) {
    dim3 grid((G.H_pad + TH_HANDS - 1) / TH_HANDS, G.n_games);
    tree_kernel<<<grid, TH_NT, tree_smem_bytes(P), st>>>(G, P, player, A);
    return cudaGetLastError();
}

cudaError_t kernels_prepare() {
    cudaError_t e = cudaFuncSetAttribute(grad_kernel<GRAD_NT, GRAD_KMAX>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

// ------------------------------------------------------------------ per-game scalars
// variant 0 theory (Alg. 1), 1 mu-balanced, 2 EGT/as (Alg. 3-4).
__global__ void egt_prepare_kernel(int variant, int n, DevScalars S) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
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
    if (g >= n) return;
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
    } else {
        S.tau[g] *= 0.5;                              // Alg. 4 line 3
        S.backtracks[g] += 1;
        if (S.tau[g] < 1e-12) S.fail[g] = 1;
    }
}

__global__ void tick_kernel(int n, int* t) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) t[g] += 1;
}

__global__ void set_mu_scale_kernel(int n, DevScalars S, const double* base, double scale, const int* mask) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n || (mask && !mask[g])) return;
    S.mu[g] = base[g] * scale;
    S.mu[n + g] = base[n + g] * scale;
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

cudaError_t launch_egt_prepare(int variant, int n, DevScalars S, cudaStream_t st) {
    egt_prepare_kernel<<<(n + 127) / 128, 128, 0, st>>>(variant, n, S);
    return cudaGetLastError();
}
cudaError_t launch_egt_accept(int variant, int n, DevScalars S, cudaStream_t st) {
    egt_accept_kernel<<<(n + 127) / 128, 128, 0, st>>>(variant, n, S);
    return cudaGetLastError();
}
cudaError_t launch_tick(int n, int* t, cudaStream_t st) {
    tick_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, t);
    return cudaGetLastError();
}
cudaError_t launch_set_mu_scale(int n, DevScalars S, const double* base, double scale, const int* mask,
                                cudaStream_t st) {
    set_mu_scale_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, S, base, scale, mask);
    return cudaGetLastError();
}

}  // namespace egt
