#!/usr/bin/env python
"""bench.py — gradient evaluations/sec of EGT/as (dilated entropy) on HUNL river endgames.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W [--impl reference]``;
for N > 1 it is launched under torchrun, one rank per GPU (RANK/LOCAL_RANK/WORLD_SIZE).

Workload: every rank solves its own batch of ``--batch``
independent synthetic Libratus-scale river endgames (the paper's
full bet abstraction, pot 2100, 200-big-blind stacks, 1081 private hands per player,
152 public sequences per player, 203 terminals -> 237M leaf-hand pairs per endgame;
boards and hand priors seeded per rank).  Units are shared out across ranks with no
data-path collective ("scaling": "weak").

One step = one pass of the whole hot path for every game of the batch: one EGT/as
iteration (Alg. 3 body with Alg. 4's excessive-gap check: 4 gradient evaluations, the
count PAPER.md:726-731 uses) including the stopping test eps_sad(x^t, y^t) (Alg. 3 line 5),
which the library takes from the excessive-gap check's gradients (2 best-response passes,
no extra gradient), read back with ``saddle_gap_device``.
``value`` = gradient evaluations of all games on all ranks / max-over-ranks device time.

``--impl reference`` times the CPU oracle (``oracle/``) as it stands on the host cores,
on one endgame of the same workload per step (a bounded sample), same metric.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = ("EGT/as gradient evaluations/sec (4 per iteration as PAPER.md:726-731 counts them; "
          "eps_sad stopping test inside the timed step), HUNL river endgames")
UNIT = "grad_evals/s"
GRADS_PER_STEP = 4  # EGT/as: y_mu(x_hat), the prox gradient, the two excessive-gap responses (R17)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=296, help="endgames per GPU")
    ap.add_argument("--workload", default="libratus", choices=["libratus", "simple"])
    ap.add_argument("--seed", type=int, default=2100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--timing-steps", type=int, default=3, help="steps of the per-kernel event-timing pass")
    ap.add_argument("--converge-games", type=int, default=16,
                    help="also time EGT/as and CFR+ to eps_sad <= --eps-mbb on this many endgames (0: skip)")
    ap.add_argument("--eps-mbb", type=float, nargs="+", default=[100.0, 10.0, 1.0],
                    help="saddle-gap targets in milli-big-blinds (time to each, median game)")
    ap.add_argument("--converge-max-steps", type=int, default=20000)
    ap.add_argument("--no-f32", action="store_true", help="skip the extra fp32-mode measurement")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"],
                    help="f32: the optional fp32 mode (fp32 vectors and arithmetic, DESIGN.md row 9)")
    ap.add_argument("--allreduce", action="store_true",
                    help="with --shard: one in-place NCCL all-reduce per gradient instead of the fused "
                         "compute + all-gather over peer memory")
    ap.add_argument("--shard", action="store_true",
                    help="strong scaling: every rank holds the same batch and computes a slice of each "
                         "gradient's rows; each row is stored into every rank's buffer over NVLink by the "
                         "kernel that finishes it (fused all-gather, DESIGN.md row 8)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def workload(args, rank):
    from paper_1810_03063_b200 import workloads as W
    spec = W.river_spec(args.workload)
    seed = args.seed + 100003 * rank
    boards = W.random_boards(args.batch, seed)
    p1, p2 = W.random_priors(boards, seed)
    return spec, boards, p1, p2


def max_over_ranks(x, world, device="cpu"):
    """Max of a per-rank scalar over all ranks (the contract's max-over-ranks timing)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def throughput(games_per_rank, world, steps, ms, shard=False):
    """Whole-job gradient evaluations per second: every rank's games, every step (sharded:
    the ranks share one batch, so its games count once)."""
    return GRADS_PER_STEP * games_per_rank * (1 if shard else world) * steps / (ms / 1e3)


def time_to_gap(P, spec, boards, p1, p2, solver, eps_mbb, max_steps, check_every=10, precision="f64"):
    """Device time (CUDA events) until the median game of the batch reaches eps_sad <= each
    target in eps_mbb (sum of regrets in milli-big-blinds, 1 mbb = big blind
    / 1000 chips): graph-launched solver steps; every `check_every` steps eps_sad is evaluated
    on the device and read back.  Both solvers are checked the same way and the check is timed
    apart from the solver: "seconds" is the solver's own device time (events around each block
    of steps), "seconds_with_checks" adds the eps_sad evaluations (EGT/as keeps its gap
    current at no gradient cost; CFR+'s average needs 2 gradients + 2 best responses).
    grad_evals_per_game counts each solver's own gradients: 4 per EGT/as attempt, 2 per CFR+
    iteration, not the checks."""
    import torch
    n = len(boards)
    game = P.Game(P.RIVER, n_games=n, river=spec, boards=boards, prior1=p1, prior2=p2, precision=precision)
    st = torch.cuda.current_stream()
    game.set_stream(st)
    gap = torch.zeros(n, dtype=torch.float64, device="cuda")
    if solver == "egt_as":
        game.egt_init(P.EGT_AS)
        step = game.egt_step
        which, per_step = 0, 4
    else:
        game.cfr_init(P.CFR_PLUS)
        step = game.cfr_step
        which, per_step = 1, 2
    mbb = spec["big_blind"] / 1000.0
    targets = sorted(eps_mbb, reverse=True)
    torch.cuda.synchronize()
    checks = []  # (steps, solver seconds so far, solver+check seconds so far, median gap, max gap)
    solver_s = total_s = 0.0
    steps = 0
    while steps < max_steps:
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        step(check_every)
        steps += check_every
        e1.record(st)
        game.saddle_gap_device(which, gap)
        e2.record(st)
        g = gap.cpu().numpy()
        solver_s += e0.elapsed_time(e1) / 1e3
        total_s += e0.elapsed_time(e2) / 1e3
        checks.append((steps, solver_s, total_s, float(np.median(g)), float(np.max(g))))
        if checks[-1][3] <= targets[-1] * mbb:  # the median game reached the last target
            break
    game.close()
    last = checks[-1]
    out = {"solver": solver, "games": n, "precision": precision, "steps_run": steps,
           "seconds_run": last[1], "seconds_run_with_checks": last[2], "check_every": check_every,
           "final_gap_mbb": {"median": last[3] / mbb, "max": last[4] / mbb},
           "grad_evals_per_game": per_step * steps, "to_eps": []}
    for e in targets:
        hit = next((c for c in checks if c[3] <= e * mbb), None)
        out["to_eps"].append({"eps_mbb": e, "median_game_steps": hit[0] if hit else None,
                              "grad_evals_per_game": per_step * hit[0] if hit else None,
                              "seconds": hit[1] if hit else None,
                              "seconds_with_checks": hit[2] if hit else None})
    return out


def workload_config(args, game=None, world=1):
    cfg = {"workload": "%s_river_endgame_batch" % args.workload,
           "games_per_gpu": args.batch, "global_games": args.batch * world,
           "solver": "EGT/as (dilated entropy) + eps_sad per step", "pot": 2100, "stack": 18950,
           "bet_abstraction": "PAPER.md:673-685" if args.workload == "libratus" else "{0.5,1,all-in}",
           "parallelism": ("shard%d (one batch; each gradient's terminal rows split over ranks, %s)"
                           % (world, "NCCL all-reduce per gradient" if getattr(args, "allreduce", False)
                              else "rows stored into every rank's buffer by the kernel (fused all-gather)"))
                          if getattr(args, "shard", False) else
                          "dp%d (independent endgames per rank)" % world}
    if game is not None:
        cfg.update({"hands_per_player": game.H, "pub_seqs": list(game.n_pub),
                    "terminals": game.n_terminals,
                    "leaf_hand_pairs_per_game": game.n_terminals * game.H * game.H,
                    "seq_dims": [game.n_pub[0] * game.H, game.n_pub[1] * game.H]})
    return cfg


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region (B200_PROFILING.md clocks
    line): NVML every 10 ms (nvidia-smi every 200 ms if NVML is unavailable)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    BITS = [0x8, 0x40, 0x20, 0x4]  # nvmlClocksEventReason{HwSlowdown,HwThermalSlowdown,SwThermalSlowdown,SwPowerCap}

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, set of reason names)
        self.source = None
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def sample():
                r = get_reasons(h)
                return (float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)), float(mx),
                        {n for n, b in zip(self.NAMES, self.BITS) if r & b})
            sample()
            return sample
        except Exception:
            return None

    def _smi(self):
        def sample():
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            r = [c.strip() for c in out.split(",")]
            return (float(r[1]), float(r[2]), {n for n, v in zip(self.NAMES, r[5:9]) if v.lower() == "active"})
        return sample

    def start(self):
        sample = self._nvml()
        self.source, period = ("nvml", 0.01) if sample else ("nvidia-smi", 0.2)
        sample = sample or self._smi()

        def run():
            while True:
                try:
                    self.rows.append(sample())
                except Exception:
                    pass
                if self._stop.wait(period):
                    break
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(set().union(*(r[2] for r in self.rows))), "samples": len(self.rows),
                "source": self.source}


# ----------------------------------------------------------------------------- roofline
def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_entry(kind, workload_name):
    """The committed ncu capture's record for the dominant kernel (profiles/ncu_traffic.json)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload_name, {}).get(kind)
    except Exception:
        return None


def ncu_traffic(kind, workload_name):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture, if any."""
    e = ncu_entry(kind, workload_name)
    return None if e is None else float(e["dram_bytes_per_game_launch"])


# ----------------------------------------------------------------------------- CPU oracle leg
def oracle_sample(args, boards, p1, p2, budget_s=20.0, max_iters=None):
    """Time the CPU oracle (as it stands) on game 0 of the workload: EGT/as initial point,
    then EGT/as iterations each followed by eps_sad, until ~budget_s.  Returns
    (grad evals, seconds, iterations)."""
    from oracle import br, egt, river
    from oracle.cards import Deck
    from paper_1810_03063_b200 import workloads as W
    spec = W.river_spec(args.workload)
    deck = Deck(13, 4)
    rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap", "open_fold")})
    sf = river.RiverSeqForm(rp, deck, boards[0], W.prior_dict(p1[0], deck.n_cards),
                            W.prior_dict(p2[0], deck.n_cards), build_sparse=False)
    prob = egt.Problem(sf)
    mu = egt.theory_mu(sf) * 2.0 ** -8
    t0 = time.perf_counter()
    x, y = egt.initialize(prob, mu, mu)
    st = egt.EGTState(x, y, mu, mu)
    grads = prob.grads.n
    iters = 0
    while True:
        egt.egt_iteration(prob, st, "as")
        br.saddle_gap(sf, st.x, st.y)
        iters += 1
        grads = prob.grads.n + 2 * iters
        el = time.perf_counter() - t0
        if el >= budget_s or (max_iters and iters >= max_iters):
            break
    return grads, time.perf_counter() - t0, iters


def host_cores():
    """Cores this process may run on (the oracle's host threads can use at most these)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def host_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info()]
        return max(n) if n else 1
    except Exception:
        return 1


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    spec, boards, p1, p2 = workload(args, 0)
    from oracle import br, egt, river
    from oracle.cards import Deck
    from paper_1810_03063_b200 import workloads as W
    deck = Deck(13, 4)
    rp = river.RiverParams(**{k: spec[k] for k in ("pot", "stack", "fracs", "allin", "raise_cap", "open_fold")})
    sf = river.RiverSeqForm(rp, deck, boards[0], W.prior_dict(p1[0], deck.n_cards),
                            W.prior_dict(p2[0], deck.n_cards), build_sparse=False)
    prob = egt.Problem(sf)
    mu = egt.theory_mu(sf) * 2.0 ** -8
    x, y = egt.initialize(prob, mu, mu)
    st = egt.EGTState(x, y, mu, mu)

    def step():
        egt.egt_iteration(prob, st, "as")
        br.saddle_gap(sf, st.x, st.y)
        prob.grads.n += 2

    for _ in range(args.warmup):
        step()
    g0 = prob.grads.n
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    grads = prob.grads.n - g0
    v = grads / el
    cores = host_cores()
    sample = ("1 endgame (game 0 of rank 0's %d-game batch) per step: %d EGT/as iterations + eps_sad, fp64 numpy "
              "(BLAS threads %d)" % (args.batch, args.steps, host_threads()))
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": dict(workload_config(args, None, 1),
                                                reference_sample="1 of the %d endgames per step (bounded CPU sample)"
                                                                 % args.batch),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_1810_03063_b200 as P
    from paper_1810_03063_b200 import build as B

    rank, local, world = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        B.build()
    if world > 1:
        dist.barrier()
    P.load_library()

    spec, boards, p1, p2 = workload(args, 0 if args.shard else rank)
    game = P.Game(P.RIVER, n_games=args.batch, river=spec, boards=boards, prior1=p1, prior2=p2,
                  precision=args.precision)
    stream = torch.cuda.current_stream()
    game.set_stream(stream)
    if args.shard:
        if not args.allreduce and world > 1:
            game.shard_fused(rank, world)
        else:
            game.shard(rank, world)
    game.egt_init(P.EGT_AS)  # practical mu (R14)
    gap = torch.zeros(args.batch, dtype=torch.float64, device="cuda")

    def step():
        game.egt_step(1)
        game.saddle_gap_device(0, gap)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = Clocks(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ck = clocks.stop()
    ms = max_over_ranks(ev0.elapsed_time(ev1), world, "cuda")
    value = throughput(args.batch, world, args.steps, ms, args.shard)
    gaps = gap.cpu().numpy()

    # per-kernel event timing (same kernels, eager launches, events on the library stream)
    game.timing(True)
    for _ in range(args.timing_steps):
        step()
    kt = game.timing_get()
    game.timing(False)
    torch.cuda.synchronize()
    launches_per_step = sum(v[1] for k, v in kt.items() if k != "comm") / args.timing_steps  # our kernels only
    step_ms_eager = sum(v[0] for v in kt.values()) / args.timing_steps
    tot_ms = sum(v[0] for v in kt.values())
    peak, peak_src = measured_peak()
    # the dominant kernel (the gradient counts both players' launches): the library's
    # algorithmic bytes of the work done / the event-timed kernel time
    groups = {"grad_kernel (A y and A^T x)": ("grad_Ay", "grad_ATx"), "tree_kernel": ("tree",)}
    dom = max(groups, key=lambda n: sum(kt[k][0] for k in groups[n]))
    ks = groups[dom]
    ms_k = sum(kt[k][0] for k in ks)
    nl = sum(kt[k][1] for k in ks)
    byts = sum(kt[k][3] for k in ks)
    achieved = byts / (ms_k / 1e3) / 1e9
    tr = ncu_traffic("grad" if dom.startswith("grad") else "tree", args.workload)
    active = sum(kt[k][2] for k in ks)
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None if tr is None else tr * active / nl,
            "peak_source": peak_src, "algorithmic_bytes_per_launch": byts / nl,
            "avg_launch_ms": ms_k / nl, "share_of_step": ms_k / tot_ms}
    lim = (ncu_entry("grad" if dom.startswith("grad") else "tree", args.workload) or {}).get("limiter")
    if lim:
        roof["limiter"] = lim  # what ncu shows the kernel actually waits on (not DRAM)
    other = [n for n in groups if n != dom][0]
    ko = groups[other]
    ms_o = sum(kt[k][0] for k in ko)
    roof["other_kernel"] = {"kernel": other, "achieved": sum(kt[k][3] for k in ko) / (ms_o / 1e3) / 1e9,
                            "frac": sum(kt[k][3] for k in ko) / (ms_o / 1e3) / 1e9 / peak,
                            "share_of_step": ms_o / tot_ms}
    lim_o = (ncu_entry("grad" if other.startswith("grad") else "tree", args.workload) or {}).get("limiter")
    if lim_o:
        roof["other_kernel"]["limiter"] = lim_o
    kernel_split = {k: {"ms_per_step": v[0] / args.timing_steps, "launches_per_step": v[1] / args.timing_steps,
                        "gbs": (v[3] / (v[0] / 1e3) / 1e9) if v[0] > 0 else None}
                    for k, v in kt.items()}

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if args.shard else "weak", "vs_baseline": None, "dtype": args.precision,
                "data": "synthetic",
                "config": dict(workload_config(args, game, world),
                               l2="no flush: per-step working set %.0f MB > 126 MB L2" %
                               (args.batch * 2 * 7 * 8 * game.H_pad * max(game.n_pub) / 1e6)),
                "roofline": roof, "kernels": kernel_split, "eager_step_ms": step_ms_eager,
                "gpu_launches": int(round(launches_per_step * args.steps)),
                "clocks": ck, "gap_after": {"median": float(np.median(gaps)), "max": float(np.max(gaps)),
                                            "unit": "chips"}}

    # e2e: the same metric through the public API from host buffers -- load the batch from
    # host arrays (H2D inside egt_load_game), init, K steps each reading eps_sad back to host.
    if not args.no_e2e:
        game.close()
        del game
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        pinned = torch.zeros(args.batch, dtype=torch.float64).pin_memory()
        t0 = time.perf_counter()
        g2 = P.Game(P.RIVER, n_games=args.batch, river=spec, boards=boards, prior1=p1, prior2=p2,
                    precision=args.precision)
        t_load = time.perf_counter()
        if args.shard:
            if not args.allreduce and world > 1:
                g2.shard_fused(rank, world)
            else:
                g2.shard(rank, world)
        g2.egt_init(P.EGT_AS)
        torch.cuda.synchronize()
        t_init = time.perf_counter()
        for _ in range(args.steps):
            g2.egt_step(1)
            g2.saddle_gap(0, out=pinned)
        el = time.perf_counter() - t0
        el = max_over_ranks(el, world, "cuda")
        if rank == 0:
            # the same count as `value` (4 per EGT/as iteration); loading, table building and
            # the practical-mu search are overhead inside the wall time
            line["e2e"] = {"value": throughput(args.batch, world, args.steps, el * 1e3, args.shard), "unit": UNIT,
                           "h2d_bytes_per_step": int(g2.h2d_bytes / args.steps),
                           "d2h_bytes_per_step": 8 * args.batch,
                           "what": "wall clock of a whole job through the public API: egt_load_game from host "
                                   "arrays (tables built on the host, copied in) + egt_init (practical-mu search) "
                                   "+ K x (egt_step + saddle_gap into pinned host memory); the K iterations' "
                                   "gradient evaluations over the whole time", "seconds": el,
                           "breakdown_s": {"load": t_load - t0, "init": t_init - t_load,
                                           "steps": el - (t_init - t0) if world == 1 else None}}
        g2.close()

    if rank == 0 and world == 1 and args.precision == "f64" and not args.no_f32 and not args.shard:
        # the optional fp32 mode (DESIGN.md row 9) on the same workload, device-timed the same way
        g32 = P.Game(P.RIVER, n_games=args.batch, river=spec, boards=boards, prior1=p1, prior2=p2, precision="f32")
        g32.set_stream(stream)
        g32.egt_init(P.EGT_AS)
        gap32 = torch.zeros(args.batch, dtype=torch.float64, device="cuda")
        for _ in range(args.warmup):
            g32.egt_step(1)
            g32.saddle_gap_device(0, gap32)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            g32.egt_step(1)
            g32.saddle_gap_device(0, gap32)
        e1.record(stream)
        torch.cuda.synchronize()
        ms32 = e0.elapsed_time(e1)
        line["fp32_mode"] = {"value": throughput(args.batch, 1, args.steps, ms32), "unit": UNIT,
                             "ms_per_step": ms32 / args.steps, "dtype": "f32",
                             "what": "same workload and timing with precision EGT_F32 (parity 1e-5 vs the oracle)"}
        g32.close()

    if rank == 0 and world == 1 and args.workload == "libratus" and not args.no_f32 and not args.shard:
        # BASELINE.json configs[2]: the {1/2, 1, all-in} abstraction on the same boards and
        # ranges, same step and timing (a smaller tree: 90 public sequences per player)
        from paper_1810_03063_b200 import workloads as W
        gs = P.Game(P.RIVER, n_games=args.batch, river=W.river_spec("simple"), boards=boards, prior1=p1,
                    prior2=p2, precision=args.precision)
        gs.set_stream(stream)
        gs.egt_init(P.EGT_AS)
        gaps_s = torch.zeros(args.batch, dtype=torch.float64, device="cuda")
        for _ in range(args.warmup):
            gs.egt_step(1)
            gs.saddle_gap_device(0, gaps_s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            gs.egt_step(1)
            gs.saddle_gap_device(0, gaps_s)
        e1.record(stream)
        torch.cuda.synchronize()
        mss = e0.elapsed_time(e1)
        line["simple_abstraction"] = {"value": throughput(args.batch, 1, args.steps, mss), "unit": UNIT,
                                      "ms_per_step": mss / args.steps, "pub_seqs": list(gs.n_pub),
                                      "terminals": gs.n_terminals,
                                      "what": "BASELINE.json configs[2]: {1/2, 1, all-in} bet abstraction, same "
                                              "boards, ranges, batch and timing"}
        gs.close()

    if args.converge_games > 0:
        n = args.converge_games
        conv = [time_to_gap(P, spec, boards[:n], p1[:n], p2[:n], sv, args.eps_mbb, args.converge_max_steps,
                            precision=args.precision) for sv in ("egt_as", "cfr_plus")]
        if rank == 0:
            line["time_to_gap"] = conv
        # the whole batch to 10 mbb through solve(): every game until its own eps_sad <= 10 mbb,
        # solved games stopped on the device (egt_set_target); wall clock of the call
        # Each solver runs twice on fresh games: the first call of a process after the batch runs
        # above has shown host-side stalls of up to ~1.5 s (not in a process that only solves:
        # scratch runs of 2026-10-19, 0.52 s for both solvers), so both calls are reported.
        solved = {}
        for sv in ("egt_as", "cfr_plus"):
            secs = []
            for _ in range(2):
                gs = P.Game(P.RIVER, n_games=n, river=spec, boards=boards[:n], prior1=p1[:n], prior2=p2[:n],
                            precision=args.precision)
                gs.set_stream(torch.cuda.current_stream())
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = P.solve(gs, sv, eps_mbb=10.0, max_iters=args.converge_max_steps)
                torch.cuda.synchronize()
                secs.append(time.perf_counter() - t0)
                gs.close()
            solved[sv] = {"seconds": secs[1], "seconds_first_call": secs[0], "iterations": int(res["iters"]),
                          "max_gap_mbb": float(np.max(res["gap"])) / (spec["big_blind"] / 1000.0)}
        if rank == 0:
            line["solve_batch_to_10mbb"] = dict(solved, games=n, what="P.solve(..., eps_mbb=10) on the same "
                                                "games from a cold start (incl. init and mu search): every game "
                                                "to 10 mbb, solved ones stopped on the device")

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        grads, secs, iters = oracle_sample(args, boards, p1, p2)
        line["cpu_baseline"] = {"value": grads / secs, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
                                "blas_threads": host_threads(),
                                "sample": "1 endgame (game 0), oracle EGT/as initial point + %d iterations "
                                          "each with eps_sad (%d gradient evals, %.1f s)" % (iters, grads, secs)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
