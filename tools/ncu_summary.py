"""Summarise ncu raw CSV exports (tools/gpu_profile_r01b.sh) into profiles/<tag>_summary.txt and
profiles/traffic.json (per-launch DRAM traffic of each bench workload's dominant kernel).

    python tools/ncu_summary.py <round-tag> gpurun_out/r01b_*_raw.csv
"""
import csv
import json
import os
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_write.sum", "dram__bytes_read.sum",
    "dram__bytes_write.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "sm__cycles_elapsed.avg.per_second",
    # store coalescing: sectors per L1 store request (16 = one 512-byte row burst per
    # instruction) and per L2 write request (4 = full 128-byte lines)
    "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "lts__t_requests_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum.pct_of_peak_sustained_elapsed",
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"
# workload -> (bench store label, algorithmic bytes per launch)
WORK = {"cfg3": ("ROW", 8 << 30), "cfg4": ("ROW", 32 << 30), "cfg5": ("ROW", 16 << 30),
        "mrg26": ("ROW", 8 << 30), "cfg1": ("SEG", 8 << 20), "cfg2": ("JUMP", 32 << 20)}


def load(path):
    rows = list(csv.reader(open(path)))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def main():
    tag, paths = sys.argv[1], sys.argv[2:]
    out, traffic = [], []
    for p in paths:
        d = load(p)
        name = os.path.basename(p).replace("_raw.csv", "")
        wl = name.split("_")[1]
        out.append(f"== {name}: {d.get('Kernel Name', ('', '?'))[1]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:66s} {d[k][1]:>20s} {d[k][0]}")
        st = sorted(((k[len(STALLS):], float(v[1] or 0)) for k, v in d.items()
                     if k.startswith(STALLS) and not k.endswith("not_issued")), key=lambda t: -t[1])
        tot = sum(v for _, v in st) or 1.0
        out.append("  stall samples (share): " + ", ".join(f"{k} {v / tot:.1%}" for k, v in st[:8]))

        def val(k, scale={"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}):
            u, v = d[k]
            return float(v) * scale.get(u, 1)
        wr, rd = val("dram__bytes_write.sum"), val("dram__bytes_read.sum")
        if wl in WORK:
            kind = "consume" if "consume" in name else "generate"
            traffic.append({"workload": wl, "kind": kind,
                            "store": "SEG" if (kind == "consume" and wl == "cfg5") else WORK[wl][0],
                            "kernel": d.get("Kernel Name", ("", "?"))[1],
                            "dram_bytes_per_launch": int(wr + rd), "dram_bytes_write": int(wr),
                            "dram_bytes_read": int(rd),
                            "algorithmic_bytes_per_launch": WORK[wl][1],
                            "source": f"profiles/{tag}_summary.txt ({name}, ncu --set full "
                                      f"--clock-control none, one launch)"})
    with open(f"profiles/{tag}_summary.txt", "w") as f:
        f.write("\n".join(out) + "\n")
    try:  # merge: a capture updates its workloads' entries and keeps the others
        with open("profiles/traffic.json") as f:
            prev = json.load(f).get("entries", [])
    except (OSError, ValueError):
        prev = []
    key = lambda e: (e["workload"], e.get("kind", "generate"))  # noqa: E731
    fresh = {key(e): e for e in traffic}
    traffic = [fresh.pop(key(e), e) for e in prev] + list(fresh.values())
    with open("profiles/traffic.json", "w") as f:
        json.dump({"entries": traffic,
                   "note": "write bytes sit slightly below the algorithmic bytes: dirty lines "
                           "still in the 126 MB L2 when the kernel ends"}, f, indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main()
