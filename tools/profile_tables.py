"""Summaries under profiles/ from a gpurun capture (run here, on the host, with ncu -i):

  python tools/profile_tables.py launches <launches.csv> <out.md>   # ncu launch list -> per-kernel table
  python tools/profile_tables.py full <capture.ncu-rep> <out.md>    # ncu --set full of one EGT/as iteration

The `full` capture is `ncu --set full --import-source on --clock-control none -k regex:"grad_staged|tree_kernel"
--launch-skip 11 --launch-count 12 python tools/profile_step.py --batch 148 --steps 1` (148 Libratus-scale games,
explicit mu: one focus chain is empty); the `launches` list is `ncu --metrics gpu__time_duration.sum
--clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1 --converge-games 0 --no-cpu-baseline
--no-e2e --no-f32`."""
import collections
import csv
import re
import subprocess
import sys

COLS = [('gpu__time_duration.sum', 'µs', 1), ('dram__bytes_read.sum', 'DRAM rd MB', 1),
        ('dram__bytes_write.sum', 'DRAM wr MB', 1), ('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'DRAM %', 1),
        ('smsp__issue_active.avg.pct_of_peak_sustained_active', 'issue active %', 1),
        ('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed', 'shared pipe %', 1),
        ('smsp__inst_executed.sum', 'M inst', 1e-6), ('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'bank conflicts (M)', 1e-6),
        ('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'shared wavefronts (M)', 1e-6),
        ('launch__registers_per_thread', 'regs', 1), ('sm__warps_active.avg.pct_of_peak_sustained_active', 'warps active %', 1),
        ('smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio', 'barrier', 1),
        ('smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio', 'short sb', 1),
        ('smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio', 'long sb', 1)]
LABELS = ['(empty chain) grad, x̂ input', '(empty chain) SBR', '(empty chain) grad', '(empty chain) prox',
          'grad Aᵀx̂ (x̂ formed from x and x_μ(y) rows, COMB)', 'SBR y⁺ (TO_Q + TO_COMB)', 'grad A y_μ(x̂)',
          'prox x⁺ (TO_COMB)', 'check grad A y⁺', 'check SBR + fused BR (TO_LB + TO_Q)', 'check grad Aᵀ x⁺',
          'check SBR + fused BR (TO_LB + TO_Q)']


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    kn, mv, mn = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
    agg, n = {}, collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) < len(h) or r[mn] != 'gpu__time_duration.sum':
            continue
        name = re.sub(r'\s+', ' ', r[kn].split('(')[0].replace('void ', ''))
        agg[name] = agg.get(name, 0.0) + float(r[mv].replace(',', '')) / 1e3
        n[name] += 1
    tot = sum(agg.values())
    lines = ["# ncu launch list (`gpu__time_duration.sum`, cold-cache, serialised)", "",
             "Source: `%s`.  Covers game load, `egt_init` with the practical-μ scan (masked rounds of the initial point:" % path,
             "`tree_kernel<0,2>` SBR sequence form, `<0,64>` SBR value only, `grad_staged_kernel<0>`, `mu_scan_kernel`; the",
             "final initial point writes the caches with `<0,34>`) and two EGT/as steps (`grad_staged_kernel<1>` = the",
             "x̂-fed gradient, `tree_kernel<0,6>` SBR y⁺, `<1,4>` prox, `<0,50>` the excessive-gap check with the fused best",
             "response).", "", "| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        lines.append("| `%s` | %d | %.1f | %.1f %% |" % (k, n[k], v, 100 * v / tot))
    open(out, 'w').write("\n".join(lines) + "\n")


def full(rep, out):
    metrics = ",".join(c[0] for c in COLS)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metrics],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h = r[0]
    lines = ["# ncu --set full of one EGT/as iteration (148 Libratus-scale endgames)", "",
             "Source: `%s` (see tools/profile_tables.py for the command).  Stall columns are cycles per issued" % rep,
             "instruction.", "", "| launch | kernel | " + " | ".join(c[1] for c in COLS) + " |",
             "|" + "---|" * (len(COLS) + 2)]
    vals = {}
    for lab, row in zip(LABELS, r[2:]):
        v = [float(row[h.index(c[0])]) * c[2] for c in COLS]
        vals.setdefault(lab, v)
        name = row[h.index('Kernel Name')].split('(')[0].replace('void egt::', '')
        lines.append("| %s | `%s` | " % (lab, name) + " | ".join("%.1f" % x for x in v) + " |")
    g = vals['grad A y_μ(x̂)']
    us, wf, bc = g[0], g[8] * 1e6, g[7] * 1e6
    floor, floor_nc, hbm = wf / 148 / 1.965e3, (wf - bc) / 148 / 1.965e3, 2.65e6 * 148 / 6542e3
    lines += ["", "Gradient (`grad_A y_μ(x̂)` launch): %.0f µs for 148 game-gradients, %.1f M instructions, issue active %.0f %%, "
              "shared pipe %.0f %%; %.1f M shared wavefronts (%.1f M bank conflicts) = %.0f µs at one wavefront per SM-cycle "
              "(%.0f µs conflict free) against %.0f µs of compulsory DRAM traffic at 6.54 TB/s: HBM ceiling %.0f %% (%.0f %% "
              "conflict free), the kernel at %.0f %% of its shared-memory floor." %
              (us, g[6], g[4], g[5], g[8], g[7], floor, floor_nc, hbm, 100 * hbm / floor, 100 * hbm / floor_nc, 100 * floor / us)]
    open(out, 'w').write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
