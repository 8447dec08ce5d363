"""Summaries of ncu captures for profiles/ (run here, on the files gpurun brings back).

  python tools/ncu_summary.py launches gpurun_out/launches_X.csv profiles/X_launches_summary.txt
      per-kernel totals over the 256^3 energy step before the last (launch list
      of `ncu --metrics gpu__time_duration.sum --csv`; steps are delimited by the
      first K-stage launch of each step)
  python tools/ncu_summary.py metrics gpurun_out/X.ncu-rep profiles/X_metrics.json
      selected `--set full` metrics of every captured launch
"""
import csv
import json
import re
import subprocess
import sys
from collections import OrderedDict

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block",
    "launch__grid_size",
    "launch__block_size",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def _name(s):
    s = s.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    s = re.sub(r"\(.*", "", s).replace("void ", "").strip()
    head, _, rest = s.partition("<")
    return head.split("::")[-1] + ("<" + rest if rest else "")


def launches(src, dst):
    rows = list(csv.reader(l for l in open(src) if not l.startswith("==")))
    hdr = rows[0]
    iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    ks = [(_name(r[iN]), float(r[iV].replace(",", "")) * scale[r[iU]]) for r in rows[1:]]
    # a step starts at the stage-0 K-stage launch (kstage_kernel<3, *, 0, *>, 3 active axes)
    starts = [i for i, (n, _) in enumerate(ks) if re.match(r"kstage_kernel<3, \d+, 0", n)]
    if len(starts) < 2:
        raise SystemExit("need at least two 256^3 steps in the launch list")
    a, b = starts[-2], starts[-1]
    step = ks[a - 3:b - 3]  # the 3 launches before stage 0 (M, bcat) belong to the step
    agg = OrderedDict()
    for n, v in step:
        c = agg.setdefault(n, [0, 0.0])
        c[0] += 1
        c[1] += v
    tot = sum(v for _, v in step)
    out = [f"one 256^3 energy step (launches {a - 3}..{b - 4} of {len(ks)}): "
           f"{len(step)} launches, {tot:.3f} ms kernel time (serialised, cold-cache ncu replay)"]
    for n, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{n[:60]:60s} n={c:4d} t={v:9.3f} ms ({100 * v / tot:5.1f}%)")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def metrics(rep, dst):
    res = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True, check=True)
    rows = list(csv.reader(res.stdout.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = OrderedDict(kernel=_name(r[hdr.index("Kernel Name")]))
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = [r[i], units[i]]
        out.append(d)
    json.dump(out, open(dst, "w"), indent=1)
    for d in out:
        print(d["kernel"], d.get("gpu__time_duration.sum"))


if __name__ == "__main__":
    {"launches": launches, "metrics": metrics}[sys.argv[1]](sys.argv[2], sys.argv[3])
