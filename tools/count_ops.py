"""Count FP64 SASS instructions (DADD, DMUL, DFMA) per arithmetic-core operation.
flops = DADD + DMUL + 2*DFMA.  Output is the table DESIGN.md / op_flops() use."""
import os
import re
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
src = os.path.join(HERE, "count_ops.cu")
with tempfile.TemporaryDirectory() as d:
    obj = os.path.join(d, "ops.cubin")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-cubin", "-o", obj, src],
                   check=True)
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
cur = None
counts = {}
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = re.sub(r"^_Z\d+", "", m.group(1)).split("PKdPd")[0]
        counts[cur] = {"DADD": 0, "DMUL": 0, "DFMA": 0}
        continue
    if cur:
        for op in ("DADD", "DMUL", "DFMA"):
            if re.search(rf"\b{op}\b", line):
                counts[cur][op] += 1
print(f"{'op':18s} {'DADD':>5s} {'DMUL':>5s} {'DFMA':>5s} {'instr':>6s} {'flops':>6s}")
for k, c in sorted(counts.items()):
    print(f"{k:18s} {c['DADD']:5d} {c['DMUL']:5d} {c['DFMA']:5d} {c['DADD'] + c['DMUL'] + c['DFMA']:6d} "
          f"{c['DADD'] + c['DMUL'] + 2 * c['DFMA']:6d}")
