"""DRAM traffic and key counters per launch from `ncu --set full` reports -> profiles/r02_traffic.json.

    python tools/ncu_traffic.py out.json rep1.ncu-rep [rep2.ncu-rep ...]

Each report holds launches of tools/sinr_real.py C4 32 1 1 (32 groups x 256 subcarriers per launch); the per-step
figures scale them by (512 x 3276) / (32 x 256). Kernels missing from the reports keep their previous entry."""
import csv, io, json, os, subprocess, sys

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__inst_executed.avg.per_cycle_active", "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(out, reps):
    prev = json.load(open(out)) if os.path.exists(out) else {"per_launch_bytes": {}, "counters": {}}
    per, counters = dict(prev.get("per_launch_bytes", {})), dict(prev.get("counters", {}))
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[h.index("Kernel Name")].split("(")[0]
            short = name.replace("void ", "").split("<")[0]
            c = {k: r[h.index(k)] for k in KEEP if k in h}
            c["dram_units"] = [units[h.index("dram__bytes_read.sum")], units[h.index("gpu__time_duration.sum")]]
            b = sum(float(r[h.index(k)].replace(",", "")) * UNIT[units[h.index(k)]]
                    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            per[short] = int(b)
            counters = {k: v for k, v in counters.items() if k.replace("void ", "").split("<")[0] != short}
            counters[name] = c
    scale = (512 * 3276) / (32 * 256)
    doc = {"config": "C4",
           "source": "ncu --set full, tools/sinr_real.py C4 32 1 1 (one launch each = 32 groups x 256 subcarriers), "
                     "scaled by (512 x 3276)/(32 x 256) to one C4 step",
           "bytes_per_step": {"rgram": int((per.get("k_esplit", 0) + per.get("k_rgram", 0)) * scale),
                              "solve": int(per.get("k_sinr_users", 0) * scale)},
           "per_launch_bytes": per, "counters": counters}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc["bytes_per_step"]), json.dumps(per))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
