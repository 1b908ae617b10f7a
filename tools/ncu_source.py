"""Aggregate the SASS source page of an .ncu-rep: warp-stall samples by opcode
and by reason, and the hottest instructions (development aid).

    python tools/ncu_source.py gpurun_out/prof.ncu-rep [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def load(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))
    return rows


def main(path, top=25):
    rows = load(path)
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    by_op = collections.defaultdict(lambda: collections.Counter())
    tot = collections.Counter()
    execd = collections.Counter()
    for r in rows:
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_]+)*)", r["Source"])
        op = m.group(1).split(".")[0] if m else "?"
        execd[op] += int(r["Instructions Executed"] or 0)
        for c in stall_cols:
            v = int(r[c] or 0)
            by_op[op][c[6:]] += v
            tot[c[6:]] += v
    allsamp = sum(tot.values()) or 1
    print(f"{path}: {allsamp} samples")
    print("reasons:", ", ".join(f"{k} {v / allsamp:.1%}" for k, v in tot.most_common(10)))
    print(f"{'opcode':12s} {'executed':>12s} {'samples':>8s}  top reasons")
    for op, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:20]:
        s = sum(c.values())
        print(f"{op:12s} {execd[op]:12d} {s / allsamp:8.1%}  " + ", ".join(f"{k} {v / allsamp:.1%}" for k, v in c.most_common(3)))
    print("hottest instructions:")
    rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:top]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        reasons = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"  {r['Address'][-5:]} {s / allsamp:6.2%} {r['Source'].strip()[:60]:60s} " + ", ".join(f"{k} {v}" for v, k in reasons))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
