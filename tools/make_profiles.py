"""Turn gpurun_out/ ncu artefacts into the committed profiles/ summaries.

    python tools/make_profiles.py <round-tag>

Reads gpurun_out/prof_*.ncu-rep (ncu --set full of the top kernels),
gpurun_out/launches.csv (ncu launch list of the bench command) and
gpurun_out/bench*.json, writes profiles/<tag>_*.json|md and
profiles/ncu_traffic.json (per-launch DRAM bytes that bench.py reports as
roofline.traffic).
"""
import collections
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summarise  # noqa: E402

WORKLOAD_OF = {"prof_kron2_f32_n16": "kron2-f32-n16", "prof_kron3_f32_n16": "kron3-f32-n16",
               "prof_kron3_f64_n16": "kron3-f64-n16", "prof_kron3tc_f32_n16": "kron3-f32-n16-tf32",
               "prof_kron3_f32_n10": "kron3-f32-n10", "prof_kron2_f32_n10": "kron2-f32-n10"}


def num(v):
    try:
        return float(str(v).split()[0].replace(",", ""))
    except Exception:
        return None


def to_bytes(v):
    parts = str(v).split()
    x = num(v)
    unit = parts[1] if len(parts) > 1 else "byte"
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")
        per[short][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
    total = sum(sum(m.get("gpu__time_duration.sum", [])) for m in per.values()) or 1
    out = []
    for k, m in sorted(per.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", []))):
        t = m.get("gpu__time_duration.sum", [])
        rd = m.get("dram__bytes_read.sum", [])
        wr = m.get("dram__bytes_write.sum", [])
        out.append({"kernel": k, "launches": len(t), "total_ns": sum(t), "share": round(sum(t) / total, 4),
                    "mean_ns": round(sum(t) / max(1, len(t)), 1),
                    "mean_dram_bytes": round((sum(rd) + sum(wr)) / max(1, len(t)), 1) if rd else None})
    return out


def main(tag):
    out_dir = os.path.join(ROOT, "profiles")
    os.makedirs(out_dir, exist_ok=True)
    traffic_path = os.path.join(out_dir, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "prof_*.ncu-rep"))):
        base = os.path.basename(rep)[:-len(".ncu-rep")]
        summ = summarise(rep)
        with open(os.path.join(out_dir, f"{tag}_{base}.json"), "w") as f:
            json.dump({"report": base, "launches": summ}, f, indent=1)
        src = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_source.py"), rep, "20"],
                             capture_output=True, text=True).stdout
        with open(os.path.join(out_dir, f"{tag}_{base}_stalls.txt"), "w") as f:
            f.write(src)
        wl = WORKLOAD_OF.get(base)
        if wl and summ:
            s = summ[0]
            b = to_bytes(s.get("dram__bytes_read.sum", 0)) + to_bytes(s.get("dram__bytes_write.sum", 0))
            traffic[wl] = {"dram_bytes_per_launch": int(b), "kernel": s["kernel"],
                           "duration": s.get("gpu__time_duration.sum"), "source": f"profiles/{tag}_{base}.json"}
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1)
    lp = os.path.join(ROOT, "gpurun_out", "launches.csv")
    if os.path.exists(lp):
        with open(os.path.join(out_dir, f"{tag}_launches.json"), "w") as f:
            json.dump({"command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                                  "--clock-control none -c 400 python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu",
                       "kernels": launches(lp)}, f, indent=1)
    for b in ("bench.json", "bench_ref.json"):
        p = os.path.join(ROOT, "gpurun_out", b)
        if os.path.exists(p):
            lines = [ln for ln in open(p) if ln.startswith("{")]
            if lines:
                with open(os.path.join(out_dir, f"{tag}_{b}"), "w") as f:
                    f.write(lines[-1])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
