"""Aggregate ncu warp-stall samples per CUDA source line from a --set full report captured with
--import-source on (kernels built with -lineinfo).

    python tools/ncu_lines.py report.ncu-rep [top_n]
"""
import collections
import csv
import io
import subprocess
import sys

STALLS = ["stall_barrier", "stall_branch_resolving", "stall_dispatch", "stall_drain", "stall_lg", "stall_long_sb",
          "stall_math", "stall_membar", "stall_mio", "stall_misc", "stall_no_inst", "stall_not_selected",
          "stall_selected", "stall_short_sb", "stall_sleep", "stall_tex", "stall_wait"]


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname = "?"
    header = None
    agg = collections.defaultdict(lambda: collections.Counter())
    text = {}
    total = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            header = r
            continue
        if header is None or r[0] in ("", "Function Name"):
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        key = (fname, line)
        text[key] = r[1].strip()[:90]
        h = {n: i for i, n in enumerate(header)}
        try:
            s = int(r[h["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, IndexError):
            continue  # source text with unescaped quotes breaks the CSV row
        if s == 0:
            continue
        total += s
        agg[key]["all"] += s
        for st in STALLS:
            if st in h and r[h[st]] not in ("", "-"):
                agg[key][st] += int(r[h[st]])
    print(f"total samples {total}")
    for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["all"])[:top]:
        reasons = ", ".join(f"{k[6:]}={v}" for k, v in c.most_common(4) if k != "all")
        print(f"{c['all'] / total:6.1%} {key[0]}:{key[1]:<5d} {text[key]:<90s} | {reasons}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
