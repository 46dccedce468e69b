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

namespace egt {

// ------------------------------------------------------------------ block scan
// Exclusive scan of data[0, n) in shared memory, in place; returns the total.
// Deterministic (fixed association order).  Contains __syncthreads().
template <int NT>
__device__ double block_exscan(double* data, int n, double* wtot) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = NT / 32;
    const int per = (n + NT - 1) / NT;
    const int beg = min(tid * per, n), end = min(beg + per, n);
    double s = 0.0;
    for (int i = beg; i < end; ++i) s += data[i];
    double incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wtot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        double t = lane < NW ? wtot[lane] : 0.0;
        double it = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            double v = __shfl_up_sync(0xffffffffu, it, o);
            if (lane >= o) it += v;
        }
        if (lane < NW) wtot[lane] = it - t;
        if (lane == NW - 1) wtot[NW] = it;
    }
    __syncthreads();
    double run = wtot[wid] + (incl - s);
    for (int i = beg; i < end; ++i) {
        double v = data[i];
        data[i] = run;
        run += v;
    }
    double total = wtot[NW];
    __syncthreads();
    return total;
}

// ------------------------------------------------------------------ gradient
// One CTA per (output public sequence s, game g).  For every terminal t whose last
// sequence of `player` is s (hands of the player: "self"; of the other: "opp"):
//   w[i]      = prior_opp(h_i) * v_opp[seq_opp(t), h_i]   (opp hands in strength order)
//   fold:     v(h) = u2 * sum_{opp hands h' disjoint from h} w(h')
//                  = u2 * (T - sum_{c in h} S_c + [|h| = 2] w(h))      (inclusion-exclusion)
//   showdown: v(h) = sign * W * (stronger(h) - weaker(h)) over disjoint opp hands, with
//                  weaker(h) = P[lo] - sum_{c in h} Pc[lo],  stronger = (T - P[hi]) - sum_c (S_c - Pc[hi])
//             P: prefix sums in strength order; Pc: prefix sums over the hands holding card c
//             (segments of the expanded card array E).  sign = +1 for player 0 (A y: player 2
//             wins with the stronger hand), -1 for player 1 (A^T x).
//   g[s, h] += kappa_t * kappa_game * prior_self(h) * v(h)
template <int NT>
__global__ void __launch_bounds__(NT) grad_kernel(DevGame G, DevPlayer P, int player, VecRef vin, VecRef gout,
                                                  const int* __restrict__ mask, int want) {
    extern __shared__ double sm[];
    __shared__ double wtot[NT / 32 + 1];
    const int s = blockIdx.x, g = blockIdx.y, tid = threadIdx.x;
    if (mask && mask[g] != want) return;
    const int Hp = G.H_pad, hs = G.hand_size;
    double* w = sm;
    double* Pf = w + Hp;
    double* E = Pf + Hp + 1;
    double* acc = E + 2 * Hp + 2;
    for (int i = tid; i < Hp; i += NT) acc[i] = 0.0;
    const int t0 = P.term_off[s], t1 = P.term_off[s + 1];
    const double* __restrict__ pself = G.prior[player] + (size_t)g * Hp;
    const double* __restrict__ popp = G.prior[1 - player] + (size_t)g * Hp;
    const double* __restrict__ vo = vin.at(g);
    const double kg = G.kappa_game[g];
    const double sd_sign = player == 0 ? 1.0 : -1.0;
    for (int ti = t0; ti < t1; ++ti) {
        const DevTerm T = G.terms[P.term_idx[ti]];
        const int k = g * G.n_bs + T.bs;
        const int nv = G.tab_nvalid[k];
        const int16_t* __restrict__ order = G.tab_order + (size_t)k * Hp;
        const int16_t* __restrict__ lo = G.tab_lo + (size_t)k * Hp;
        const int16_t* __restrict__ hi = G.tab_hi + (size_t)k * Hp;
        const int4* __restrict__ pos = G.tab_pos + (size_t)k * Hp;
        const int16_t* __restrict__ src = G.tab_src + (size_t)k * (2 * Hp + 2);
        const int so = T.seq[1 - player];
        __syncthreads();  // previous terminal finished with w / Pf / E / acc
        for (int i = tid; i < nv; i += NT) {
            const int h = order[i];
            const double yv = so ? vo[(size_t)so * Hp + h] : 1.0;
            const double wv = popp[h] * yv;
            w[i] = wv;
            Pf[i] = wv;
        }
        __syncthreads();
        const int ne = nv * hs;
        for (int e = tid; e < ne; e += NT) E[e] = w[src[e]];
        __syncthreads();
        const double Ttot = block_exscan<NT>(Pf, nv, wtot);
        const double Etot = block_exscan<NT>(E, ne, wtot);
        if (tid == 0) {
            Pf[nv] = Ttot;
            E[ne] = Etot;
        }
        __syncthreads();
        const double scale = T.kappa * kg * T.amount;
        for (int i = tid; i < nv; i += NT) {
            const int h = order[i];
            const int4 pr = pos[i];
            const int16_t* pd = reinterpret_cast<const int16_t*>(&pr);
            double v;
            if (T.kind == 2) {
                double weaker = Pf[lo[i]];
                double stronger = Ttot - Pf[hi[i]];
                for (int c = 0; c < hs; ++c) {
                    const double est = E[pd[c * 4 + 2]];
                    weaker -= E[pd[c * 4 + 0]] - est;
                    stronger -= E[pd[c * 4 + 3]] - E[pd[c * 4 + 1]];
                }
                v = sd_sign * (stronger - weaker);
            } else {
                double comp = Ttot;
                for (int c = 0; c < hs; ++c) comp -= E[pd[c * 4 + 3]] - E[pd[c * 4 + 2]];
                if (hs == 2) comp += w[i];
                v = comp;
            }
            acc[h] += scale * pself[h] * v;
        }
    }
    __syncthreads();
    double* __restrict__ out = gout.at(g) + (size_t)s * Hp;
    for (int i = tid; i < Hp; i += NT) out[i] = acc[i];
}

static constexpr int GRAD_NT = 256;

cudaError_t launch_gradient(const DevGame& G, const DevPlayer& P, int player, VecRef vin, VecRef gout,
                            const int* mask, int want, cudaStream_t st) {
    const size_t smem = sizeof(double) * (size_t)(G.H_pad + (G.H_pad + 1) + (2 * G.H_pad + 2) + G.H_pad);
    dim3 grid(P.n_pub, G.n_games);
    grad_kernel<GRAD_NT><<<grid, GRAD_NT, smem, st>>>(G, P, player, vin, gout, mask, want);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ treeplex pass
// One thread per private hand, HT hands per CTA; the gradient tile [n_pub][HT] is
// staged in shared memory; the bottom-up pass overwrites each simplex's entries
// with its behavioural strategy and adds the simplex value into the parent entry;
// the top-down pass turns behavioural into sequence form in place.
template <int HT>
__global__ void __launch_bounds__(HT) tree_kernel(DevGame G, DevPlayer P, int player, TreeArgs A) {
    extern __shared__ double tile[];
    __shared__ double red[HT / 32];
    const int g = blockIdx.y, tid = threadIdx.x;
    if (A.mask && A.mask[g] != A.want) return;
    const int Hp = G.H_pad;
    const int h = blockIdx.x * HT + tid;
    const bool live = h < G.H;
    const int n_pub = P.n_pub;
    const int mode = A.mode;
    const bool has_grad = mode == TM_SBR || mode == TM_PROX || mode == TM_BR || mode == TM_CFR;
    double* col = tile + tid;  // column of this hand: col[s * HT]
    const uint8_t* __restrict__ valid_g = G.tab_valid + (size_t)g * G.n_bs * Hp;

    // ---- load
    if (has_grad) {
        const double* __restrict__ gp = A.g.at(g);
        double sc = A.gsign;
        if (mode == TM_PROX) sc *= A.mu[g];
        for (int s = 0; s < n_pub; ++s) col[s * HT] = live ? sc * gp[(size_t)s * Hp + h] : 0.0;
    }

    // ---- bottom-up
    const double mu = (mode == TM_SBR) ? A.mu[g] : 1.0;
    double* __restrict__ cz = A.center.ok() ? A.center.at(g) : nullptr;
    double* __restrict__ rg = A.regret.ok() ? A.regret.at(g) : nullptr;
    if (live && mode != TM_UNIFORM && mode != TM_COMBINE) {
        for (int m = P.n_nodes - 1; m >= 0; --m) {
            const int first = P.node_first[m], n = P.node_nact[m], par = P.node_parent[m];
            if (!valid_g[(size_t)P.node_bs[m] * Hp + h]) {
                for (int a = 0; a < n; ++a) col[(first + a) * HT] = 0.0;
                continue;
            }
            if (mode == TM_SBR) {
                const double wgt = mu * P.beta[(size_t)m * Hp + h];
                double mn = DBL_MAX;
                for (int a = 0; a < n; ++a) mn = fmin(mn, col[(first + a) * HT]);
                double S = 0.0;
                for (int a = 0; a < n; ++a) {
                    const double e = exp(-(col[(first + a) * HT] - mn) / wgt);
                    col[(first + a) * HT] = e;
                    S += e;
                }
                const double inv = 1.0 / S;
                for (int a = 0; a < n; ++a) col[(first + a) * HT] *= inv;
                // value = g_{i*} + w log qbar_{i*} + w log n, i* = argmax qbar
                col[par * HT] += mn - wgt * log(S) + wgt * log((double)n);
            } else if (mode == TM_PROX) {
                // multiplicative form of the shifted-gradient SBR:
                // qbar_i ~ zbar_i exp(-H_i / beta), U = -beta log sum_i zbar_i exp(-H_i / beta)
                const double beta = P.beta[(size_t)m * Hp + h];
                double mn = DBL_MAX;
                for (int a = 0; a < n; ++a)
                    if (cz[(size_t)(first + a) * Hp + h] > 0.0) mn = fmin(mn, col[(first + a) * HT]);
                double S = 0.0;
                for (int a = 0; a < n; ++a) {
                    const double z = cz[(size_t)(first + a) * Hp + h];
                    const double e = z > 0.0 ? z * exp(-(col[(first + a) * HT] - mn) / beta) : 0.0;
                    col[(first + a) * HT] = e;
                    S += e;
                }
                const double inv = 1.0 / S;
                for (int a = 0; a < n; ++a) col[(first + a) * HT] *= inv;
                col[par * HT] += mn - beta * log(S);
            } else if (mode == TM_BR) {
                int best = 0;
                double mn = col[first * HT];
                for (int a = 1; a < n; ++a) {
                    const double v = col[(first + a) * HT];
                    if (v < mn) { mn = v; best = a; }
                }
                for (int a = 0; a < n; ++a) col[(first + a) * HT] = a == best ? 1.0 : 0.0;
                col[par * HT] += mn;
            } else {  // TM_CFR: utility u = gsign * g, current strategy z, regrets r
                double val = 0.0;
                for (int a = 0; a < n; ++a) val += col[(first + a) * HT] * cz[(size_t)(first + a) * Hp + h];
                double S = 0.0;
                for (int a = 0; a < n; ++a) {
                    const size_t idx = (size_t)(first + a) * Hp + h;
                    const double u = col[(first + a) * HT], r0 = rg[idx];
                    double r = r0 + u - val;
                    if (A.cfr_plus) r = fmax(r, 0.0);
                    rg[idx] = r;
                    // DESIGN.md R15: regrets at the rounding-noise level of their own update count as 0
                    const double tol = 1e-13 * (fabs(r0) + fabs(u) + fabs(val));
                    const double pr = r > tol ? r : 0.0;
                    col[(first + a) * HT] = pr;
                    S += pr;
                }
                for (int a = 0; a < n; ++a) {
                    const double z = S > 0.0 ? col[(first + a) * HT] / S : 1.0 / n;
                    col[(first + a) * HT] = z;
                    cz[(size_t)(first + a) * Hp + h] = z;
                }
                col[par * HT] += val;
            }
        }
    }
    const double myval = live ? col[0] : 0.0;

    // ---- top-down
    const bool want_td = A.out_b.ok() || A.out_q.ok() || A.comb_out.ok() || mode == TM_CFR;
    if (want_td) {
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
        col[0] = live ? 1.0 : 0.0;
        if (h < Hp) {
            const double q0 = live ? 1.0 : 0.0;
            if (ob) ob[h] = q0;
            if (oq) oq[h] = q0;
            if (co) co[h] = live ? (1.0 - tau) * ci[h] + tau : 0.0;
            if (av) av[h] = q0;
        }
        for (int m = 0; m < P.n_nodes; ++m) {
            const int first = P.node_first[m], n = P.node_nact[m], par = P.node_parent[m];
            const bool ok = live && valid_g[(size_t)P.node_bs[m] * Hp + h];
            const double qp = col[par * HT];
            for (int a = 0; a < n; ++a) {
                const int s = first + a;
                double b;
                if (!ok) b = 0.0;
                else if (mode == TM_UNIFORM) b = 1.0 / n;
                else if (mode == TM_COMBINE) b = bin[(size_t)s * Hp + h];
                else b = col[s * HT];
                const double q = qp * b;
                col[s * HT] = q;
                if (h < Hp) {
                    const size_t idx = (size_t)s * Hp + h;
                    if (ob) ob[idx] = b;
                    if (oq) oq[idx] = q;
                    if (co) co[idx] = (1.0 - tau) * ci[idx] + tau * q;
                    if (av) av[idx] = alpha * q + (1.0 - alpha) * av[idx];
                }
            }
        }
    }

    // ---- per-game value: deterministic block sum, then the last CTA sums the tiles in order
    if (A.value) {
        double v = myval;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((tid & 31) == 0) red[tid >> 5] = v;
        __syncthreads();
        __shared__ bool last;
        if (tid == 0) {
            double b = 0.0;
            for (int i = 0; i < HT / 32; ++i) b += red[i];
            A.partial[(size_t)g * gridDim.x + blockIdx.x] = b;
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
}

template <int HT>
static cudaError_t launch_tree_ht(const DevGame& G, const DevPlayer& P, int player, const TreeArgs& A,
                                  cudaStream_t st) {
    const size_t smem = sizeof(double) * (size_t)P.n_pub * HT;
    dim3 grid((G.H + HT - 1) / HT, G.n_games);
    tree_kernel<HT><<<grid, HT, smem, st>>>(G, P, player, A);
    return cudaGetLastError();
}

int tree_tile_width(const DevGame& G, const DevPlayer& P) {
    const size_t per_hand = sizeof(double) * (size_t)P.n_pub;
    if (G.H >= 128 && per_hand * 128 <= 64 * 1024) return 128;
    if (G.H >= 64 && per_hand * 64 <= 64 * 1024) return 64;
    return 32;
}

cudaError_t tree_prepare(int max_n_pub) {
    (void)max_n_pub;
    cudaError_t e = cudaSuccess;
    e = cudaFuncSetAttribute(grad_kernel<GRAD_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(tree_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(tree_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(tree_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

cudaError_t launch_tree(const DevGame& G, const DevPlayer& P, int player, const TreeArgs& A, cudaStream_t st) {
    switch (tree_tile_width(G, P)) {
        case 128: return launch_tree_ht<128>(G, P, player, A, st);
        case 64: return launch_tree_ht<64>(G, P, player, A, st);
        default: return launch_tree_ht<32>(G, P, player, A, st);
    }
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
