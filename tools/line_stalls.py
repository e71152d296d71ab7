"""Warp-stall samples and executed instructions per kernels.cu source line
from one ncu report (SASS offsets mapped through `nvdisasm -gi` line info).

Usage: python tools/line_stalls.py REPORT KERNEL_SUBSTRING [TOP]
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1205_4883_b200", "libsieve.so")
SRC = os.path.join(ROOT, "paper_1205_4883_b200", "csrc", "kernels.cu")
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}
base = int(data[0][0], 16)

with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.startswith("kernels") and f.endswith(".cubin")]
    dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, sorted(cub)[-1])],
                         capture_output=True, text=True).stdout
inside, chain, line, off2l = False, [], None, {}
for L in dis.split("\n"):
    if L.startswith("//----") and ".text." in L:
        inside = kname in L
        continue
    if not inside:
        continue
    if L.strip().startswith("//## File"):
        # the lines before an instruction, innermost first
        chain += [int(x) for f, x in re.findall(r'"([^"]+)", line (\d+)', L) if f.endswith("kernels.cu")]
        continue
    m2 = re.match(r"\s+/\*([0-9a-f]{4,})\*/", L)
    if m2:
        if chain:
            line = chain[0]
        off2l[int(m2.group(1), 16)] = line
        chain = []

agg = defaultdict(lambda: [0.0, 0.0])
for r in data:
    l = off2l.get(int(r[0], 16) - base)
    agg[l][0] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    agg[l][1] += float(r[ix["Instructions Executed"]] or 0)
src = open(SRC).read().split("\n")
tot = sum(a[0] for a in agg.values()) or 1.0
for l, (s, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    txt = src[l - 1].strip()[:88] if l else "(no line)"
    print(f"{s:6.0f} {100 * s / tot:5.1f}%  inst {ie:10.0f}  L{l}: {txt}")
