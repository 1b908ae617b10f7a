"""Print registers / spills per kernel of a .cu compile unit (ptxas -v)."""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xptxas", "-v",
                      "-c", src, "-o", "/tmp/_regs.o"], capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", cur)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and flt in cur:
        print(f"{cur:60s} regs {m.group(1):>4s}  spill {spill[0]}/{spill[1]}")
