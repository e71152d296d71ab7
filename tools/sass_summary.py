"""SASS evidence of libsieve.so (cuobjdump -sass): per kernel, the count of
the mnemonics that show what the kernel is built from -- shared-memory
atomics (ATOMS), the TMA bulk copy (UBLKCP), distributed-shared-memory
atomics (red.shared::cluster after mapa compiles to ATOM.E.OR on the
mapped address; cluster barriers UCGABAR_ARV/WAIT), popcounts, warp votes and shuffles, tcgen05 (UTC*MMA: none, no
contraction on this path).  Usage: python tools/sass_summary.py [lib]"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1205_4883_b200/libsieve.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
keys = ["ATOMS.OR", "ATOMS.ADD", "ATOM.E.OR", "RED", "ATOMG", "UBLKCP", "POPC", "VOTE", "SHFL", "BAR.SYNC",
        "UCGABAR_ARV", "UCGABAR_WAIT", "LDS", "STS", "LDG", "STG", "UTCHMMA", "UTCQMMA", "HMMA"]
cur, per = None, {}
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and cur:
        op = m.group(1)
        for k in keys:
            if op == k or op.startswith(k + "."):
                per[cur][k] += 1
for fn in sorted(per):
    if "k_sieve" not in fn and "k_base" not in fn and "k_plan" not in fn:
        continue
    c = per[fn]
    print(fn, " ".join(f"{k}={c[k]}" for k in keys if c[k]))
