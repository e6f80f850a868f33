"""Per-source-line totals of an ncu capture: joins the SASS page of the
report (instructions executed, stall samples per address) with nvdisasm's
line table of the kernel in libbsa.so.

    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTRING [top]
"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line_table(mangled_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2509_07120_b200", "libbsa.so")],
                   cwd=tmp, capture_output=True)
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        dis = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
        funcs = re.split(r"//-+ \.text\.", dis)
        for f in funcs[1:]:
            name = f.split(" ", 1)[0]
            if mangled_sub not in name:
                continue
            cur = None
            table = {}
            for ln in f.splitlines():
                m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
                if m:
                    cur = (os.path.basename(m.group(1)), int(m.group(2)))
                    continue
                m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
                if m and cur:
                    table[int(m.group(1), 16)] = cur
            return name, table
    raise SystemExit(f"no function matching {mangled_sub}")


def main():
    rep, sub = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    name, table = line_table(sub)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    ai, ii = h.index("Address"), h.index("Instructions Executed")
    si = h.index("Warp Stall Sampling (All Samples)")
    agg = defaultdict(lambda: [0, 0])
    tot_i = tot_s = 0
    base = None
    for r in rows[hi + 1:]:
        if len(r) <= max(ai, ii, si) or not r[ai].strip():
            continue
        try:
            addr = int(r[ai], 16)
        except ValueError:
            continue
        # absolute load address: offsets from the function's first instruction
        if base is None:
            base = addr
        addr -= base
        ins = float(r[ii] or 0)
        st = float(r[si] or 0)
        key = table.get(addr, ("?", 0))
        agg[key][0] += ins
        agg[key][1] += st
        tot_i += ins
        tot_s += st
    srcs = {}
    print(f"{name}: {tot_i:.3e} warp instructions, {tot_s:.0f} stall samples")
    print(f"{'file:line':32s} {'inst%':>6s} {'stall%':>6s}  source")
    for (f, l), (ins, st) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        if f not in srcs:
            p = glob.glob(os.path.join(ROOT, "paper_2509_07120_b200", "csrc", f))
            srcs[f] = open(p[0]).read().splitlines() if p else []
        text = srcs[f][l - 1].strip() if 0 < l <= len(srcs[f]) else ""
        print(f"{f + ':' + str(l):32s} {100 * ins / tot_i:6.2f} {100 * st / max(tot_s, 1):6.2f}  {text[:90]}")


if __name__ == "__main__":
    main()
