"""Aggregate ncu warp-stall samples and executed instructions per SASS opcode for one kernel of a
--set full report: python tools/ncu_ops.py report.ncu-rep kernel_regex [top_n]"""
import collections, csv, io, subprocess, sys


def main(path, kern, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg = collections.defaultdict(collections.Counter)
    h = None
    for r in rows:
        if r and r[0] in ("Address", "# Address"):
            h = {n: i for i, n in enumerate(r)}
            continue
        if h is None or len(r) < len(h):
            continue
        src = r[h["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0] + ("." + op.split(".")[1] if op.startswith(("F2F", "DFMA", "DMMA")) and "." in op else "")
        c = agg[op]
        def num(k):
            try:
                return int(float(r[h[k]] or 0))
            except (ValueError, KeyError):
                return 0
        c["samples"] += num("Warp Stall Sampling (All Samples)")
        c["inst"] += num("Instructions Executed")
        for k in h:
            if k.startswith("stall_") and "Not Issued" not in k:
                c[k] += num(k)
    tot = sum(c["samples"] for c in agg.values()) or 1
    ti = sum(c["inst"] for c in agg.values()) or 1
    print(f"total samples {tot}, warp instructions {ti}")
    for op, c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        rs = ", ".join(f"{k[6:]}={v}" for k, v in c.most_common(6) if k.startswith("stall_"))[:100]
        print(f"{c['samples'] / tot:6.1%} inst {c['inst'] / ti:6.1%} {op:<14s} | {rs}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
