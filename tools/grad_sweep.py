"""Gradient-only throughput sweep over river bet abstractions (BASELINE.json configs[4]).

For river endgame batches of growing bet-abstraction size (one fraction, {1/2, 1}, the paper's
Libratus abstraction PAPER.md:673-685, and a wider one), the solver's own gradient launches
(A y and A^T x, as EGT/as issues them) are timed on the device by the library's timing mode
(egt_timing: every kernel bracketed by CUDA events on the game's stream) and reported against
the HBM roofline: achieved = algorithmic bytes / kernel time.  Synthetic
boards and priors, seeded; fp64 unless --precision f32.  One JSON line per abstraction and a
markdown table (--md).

N GPUs (configs[4] "at 1/2/4/8 GPUs"): launch under torchrun, one rank per GPU.  --mode dp
gives every rank its own seeded batch (weak scaling, no data-path collective); --mode shard
gives every rank the same batch and splits each gradient's rows over the ranks, every row
stored into all ranks' buffers by the kernel that computes it (the fused all-gather of
DESIGN.md row 8).  Gradient evaluations of all ranks / the max over ranks of the device time
of the gradient launches (and, sharded, their peer barriers).

    python tools/grad_sweep.py --batch 296 --steps 5 --md profiles/r02_grad_sweep.md
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/grad_sweep.py --mode shard
"""
import argparse
import json
from fractions import Fraction
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def specs():
    from paper_1810_03063_b200 import workloads as W

    def wider(ctxs, extra=("3/4", "3/2", "3")):
        sp = W.river_spec("libratus")
        for k in ctxs:
            sp["fracs"][k] = sorted(set(sp["fracs"][k]) | set(extra), key=Fraction)
        return sp
    return [("one fraction {1}", W.river_spec("tiny")),
            ("simple {1/2,1}", W.river_spec("simple")),
            ("libratus (PAPER.md:673-685)", W.river_spec("libratus")),
            ("libratus + {3/4,3/2,3} at the first bet", wider(["P1_OPEN", "P2_VS_CHECK"])),
            ("libratus + {3/4,3/2,3} at the first bet and raise", wider(["P1_OPEN", "P1_VS_BET", "P2_VS_CHECK",
                                                                         "P2_VS_BET"]))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=296)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--seed", type=int, default=2100)
    ap.add_argument("--md", default=None)
    ap.add_argument("--mode", default="dp", choices=["dp", "shard"])
    a = ap.parse_args()
    import torch
    import paper_1810_03063_b200 as P
    from paper_1810_03063_b200 import workloads as W
    rank, local, world = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("LOCAL_RANK", 0), ("WORLD_SIZE", 1)))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak = float(peaks.get("hbm_gbs", 6650.0))
    except Exception:
        peak = 6650.0  # B200_PROFILING.md fallback
    seed = a.seed + (100003 * rank if a.mode == "dp" else 0)
    boards = W.random_boards(a.batch, seed)
    p1, p2 = W.random_priors(boards, seed)
    rows = []

    def over_ranks(x, op):
        if world == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    for name, spec in specs():
        G = P.Game(P.RIVER, n_games=a.batch, river=spec, boards=boards, prior1=p1, prior2=p2, precision=a.precision)
        if a.mode == "shard" and world > 1:
            G.shard_fused(rank, world)
        mu = 50.0
        G.egt_init(P.EGT_AS, mu, mu)
        G.egt_step(a.warmup)
        G.timing(True)
        G.egt_step(a.steps)
        kt = G.timing_get()
        torch.cuda.synchronize()
        out = {"abstraction": name, "pub_seqs": list(G.n_pub), "terminals": G.n_terminals, "hands": G.H,
               "games": a.batch, "precision": a.precision, "n_gpus": world, "mode": a.mode}
        tot_ms = tot_bytes = tot_active = 0.0
        for k in ("grad_Ay", "grad_ATx"):
            ms, launches, active, byts = kt[k]
            out[k] = {"ms": ms / a.steps, "launches_per_step": launches / a.steps,
                      "gbs": byts / (ms * 1e6) if ms > 0 else None}
            tot_ms += ms
            tot_bytes += byts
            tot_active += active
        comm_ms = kt["comm"][0] if a.mode == "shard" else 0.0
        import torch.distributed as _d
        op_max = _d.ReduceOp.MAX if world > 1 else None
        op_sum = _d.ReduceOp.SUM if world > 1 else None
        t_max = over_ranks(tot_ms + comm_ms, op_max)
        games_done = over_ranks(tot_active, op_sum) if a.mode == "dp" else tot_active
        out["grad_evals_per_s"] = games_done / (t_max / 1e3)
        # per-GPU roofline of the gradient kernel itself (sharded: each rank's slice bytes)
        out["achieved_gbs"] = tot_bytes / world ** (a.mode == "shard") / (tot_ms * 1e6) if a.mode == "shard" else \
            tot_bytes / (tot_ms * 1e6)
        out["roofline_frac"] = out["achieved_gbs"] / peak
        out["algorithmic_bytes_per_game_gradient"] = tot_bytes / tot_active
        out["comm_ms_per_step"] = comm_ms / a.steps
        if rank == 0:
            print(json.dumps(out), flush=True)
        rows.append(out)
        G.close()
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return
    if a.md:
        lines = ["| abstraction | public seqs | terminals | MB per game-gradient | gradient evals/s | achieved GB/s | HBM roofline |",
                 "|---|---|---|---|---|---|---|"]
        for r in rows:
            lines.append("| %s | %d / %d | %d | %.2f | %.0f | %.0f | %.1f %% |" % (
                r["abstraction"], r["pub_seqs"][0], r["pub_seqs"][1], r["terminals"],
                r["algorithmic_bytes_per_game_gradient"] / 1e6, r["grad_evals_per_s"], r["achieved_gbs"],
                100 * r["roofline_frac"]))
        with open(a.md, "w") as f:
            f.write("# Gradient-only sweep over bet abstractions (BASELINE.json configs[4]), one B200\n\n")
            f.write("`python tools/grad_sweep.py --batch %d --steps %d --precision %s` -- the solver's own gradient "
                    "launches (EGT/as, both players, masked launches excluded from the game count) timed by "
                    "egt_timing; achieved = algorithmic bytes / kernel time; peak = MEASURED_PEAKS.json hbm_gbs "
                    "(%.0f GB/s).\n\n" % (a.batch, a.steps, a.precision, peak))
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
