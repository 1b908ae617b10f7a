"""Summarise an .ncu-rep (raw page) into the handful of metrics we track."""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
        "smsp__sass_inst_executed_op_shared_st.sum", "smsp__sass_inst_executed_op_global_st.sum",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__func_cache_config"]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        rec = {"kernel": d.get("Kernel Name", ("?",))[0]}
        for w in WANT:
            if w in d:
                rec[w] = d[w][0] + (" " + d[w][1] if d[w][1] else "")
        stalls = []
        for h, (v, u) in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1
        rec["stall_top"] = {k: round(v / tot, 3) for v, k in sorted(stalls, reverse=True)[:8]}
        out.append(rec)
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps({"report": p, "launches": summarise(p)}, indent=1))
