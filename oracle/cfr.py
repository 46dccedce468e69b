"""Gen-CFR with RM / RM+ and the CFR(RM), CFR(RM+), CFR+ variants (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:1-106: Algorithm Gen-CFR (alternating updates), RM (Algorithm RM),
RM+ (Algorithm RM+), stepsizes alpha^t = 1/t (CFR(RM), CFR(RM+)) and
alpha^t = 2t/(t^2+t) (CFR+).  Strategies are kept per simplex in behavioural
form z^j (the regret minimiser's output), so Gen-CFR's ratio
x^{j,t-1} / x^{t-1}_{p_j} is z^{j,t-1} (reading R3 for zero parent weight).
"""
import numpy as np

VARIANTS = {
    "cfr_rm": ("rm", "uniform"),
    "cfr_rmp": ("rmp", "uniform"),
    "cfr_plus": ("rmp", "linear"),
}


def alpha(scheme, t):
    """1/t, or 2t/(t^2+t)."""
    return 1.0 / t if scheme == "uniform" else 2.0 * t / (t * t + t)


SNAP = 1e-13


def regret_update(kind, r, z, g, scale=0.0):
    """One call of RM or RM+  on one simplex.
    g is the gain (utility) vector; returns (r^t, z^t).

    Reading R15: "if r^t = 0 use uniform strategy" is decided robustly -- a regret
    entry no larger than SNAP * (|r^{t-1}_a| + |g_a| + |<z^{t-1}, g>| + scale) (the rounding
    noise of its own update; `scale` = the largest |gradient entry| among the player's
    sequences of the same private hand, the noise floor of gains that cancel to ~0 where
    the opponent's reach is ~0) counts as 0 in [r^t]^+."""
    val = float(np.dot(z, g))
    r_new = r + g - val
    if kind == "rmp":
        r_new = np.maximum(r_new, 0.0)
    tol = SNAP * (np.abs(r) + np.abs(g) + abs(val) + scale)
    pos = np.where(r_new > tol, r_new, 0.0)
    tot = pos.sum()
    z_new = pos / tot if tot > 0 else np.full(len(r), 1.0 / len(r))
    return r_new, z_new


class CFRState:
    def __init__(self, sf, variant):
        self.kind, self.scheme = VARIANTS[variant]
        self.sf = sf
        self.zx = sf.X.uniform_behavioral()     # x^0 uniform
        self.zy = sf.Y.uniform_behavioral()
        self.rx = np.zeros(sf.X.n_seq)
        self.ry = np.zeros(sf.Y.n_seq)
        self.x = sf.X.behavioral_to_sequence(self.zx)
        self.y = sf.Y.behavioral_to_sequence(self.zy)
        self.xbar = np.zeros(sf.X.n_seq)
        self.ybar = np.zeros(sf.Y.n_seq)
        self.t = 1
        self.grads = 0


def hand_scales(labels, g):
    """Per sequence: max |g| over the player's sequences of the same private hand (labels
    "<hand>|<history>"; the empty sequence gets 0) -- the scale of reading R15."""
    groups = {}
    for i, lab in enumerate(labels):
        if i > 0:
            groups.setdefault(lab.split("|")[0], []).append(i)
    sc = np.zeros(len(g))
    for idx in groups.values():
        sc[idx] = np.abs(np.asarray(g)[idx]).max()
    return sc


def _pass(tp, g, z, r, kind, labels=None, trace=None):
    """Bottom-up pass of Gen-CFR lines 30-33 / 36-39: fold <g^j, z^{j,t-1}> into
    g_{p_j}, then z^{j,t} = R(g^j).  trace(j, m, sj): observation only (tests) -- per simplex,
    m = the smallest |r^t_a| before RM+'s threshold (how close the "[r]^+ / r = 0" decisions of
    this call came to flipping), sj = max |g^j| (the gains with the values below folded in)."""
    g = np.array(g, dtype=float)
    sc = hand_scales(labels, g) if labels is not None else np.zeros(len(g))
    z = z.copy()
    r = r.copy()
    for j in tp.bottom_up():
        s, n, p = tp.start[j], tp.size[j], tp.parent[j]
        gj = g[s:s + n]
        g[p] += np.dot(gj, z[s:s + n])
        if trace is not None:
            pre = r[s:s + n] + gj - float(np.dot(z[s:s + n], gj))
            trace(j, float(np.min(np.abs(pre))), float(np.abs(gj).max()))
        r[s:s + n], z[s:s + n] = regret_update(kind, r[s:s + n], z[s:s + n], gj, sc[s])
    return z, r


def cfr_iteration(st, trace=None):
    """trace(player, j, m, sj): see _pass (observation only)."""
    sf = st.sf
    tx = None if trace is None else (lambda j, m, gm: trace(0, j, m, gm))
    ty = None if trace is None else (lambda j, m, gm: trace(1, j, m, gm))
    g = -sf.Ay(st.y)                                   # line 29: g = -A y^{t-1}
    st.grads += 1
    st.zx, st.rx = _pass(sf.X, g, st.zx, st.rx, st.kind, sf.labels_x, tx)
    st.x = sf.X.behavioral_to_sequence(st.zx)
    a = alpha(st.scheme, st.t)
    st.xbar = a * st.x + (1 - a) * st.xbar            # line 34
    g = sf.ATx(st.x)                                   # line 35: g = A^T x^t (alternating)
    st.grads += 1
    st.zy, st.ry = _pass(sf.Y, g, st.zy, st.ry, st.kind, sf.labels_y, ty)
    st.y = sf.Y.behavioral_to_sequence(st.zy)
    st.ybar = a * st.y + (1 - a) * st.ybar            # line 41, same alpha^t (reading R9)
    st.t += 1
    return st


def run(sf, variant, iters, trace=None):
    st = CFRState(sf, variant)
    for _ in range(iters):
        cfr_iteration(st, trace)
    return st


def cfr_plus_regret_bound(sf, T, L):
    """2 |S_X| L sqrt(max_j |Delta_j|) / sqrt(T)."""
    return 2.0 * sf.X.n_simplex * L * np.sqrt(sf.X.size.max()) / np.sqrt(T)
