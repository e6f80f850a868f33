"""Summarise ncu artefacts for profiles/: the launch list (per-kernel ms and
share of one step) and key --set full metrics of a capture.

    python scripts/ncu_summary.py launches gpurun_out/launches.csv
    python scripts/ncu_summary.py full gpurun_out/prof_tc.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "derived__lts__lts2xbar_bytes.sum.per_second",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:]]
    ours = [(n, v / 1e6) for n, v in data if "bsa::" in n or "tc::" in n]
    # the profiled step is the second half of our launches (warm-up step first)
    step = ours[len(ours) // 2:]
    tot = sum(v for _, v in step)
    print("| kernel | ms (cold, serialised) | share of step |\n|---|---|---|")
    for n, v in step:
        short = n.split("(")[0].replace("void ", "")
        print(f"| `{short}` | {v:.3f} | {100 * v / tot:.1f}% |")
    print(f"| **total ({len(step)} launches)** | {tot:.2f} | |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    print("| kernel | " + " | ".join(KEYS) + " |")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        vals = [f"{r[h.index(k)]} {u[h.index(k)]}" if k in h else "-" for k in KEYS]
        print(f"| `{name}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
