"""Per-source-line summary of an ncu report (cuda,sass source view): warp-stall
samples, instructions executed and shared-memory wavefronts (actual / ideal)
for the hottest lines.  Usage: python tools/ncu_lines.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        d = dict(zip(hdr[2:], r[2:]))  # metric columns follow "Line No","Source"
        def g(k):
            try:
                return float(d.get(k, "0") or 0)
            except ValueError:
                return 0.0
        lines.append((int(r[0]), r[1][:70], g("Warp Stall Sampling (All Samples)"),
                      g("Instructions Executed"), g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Ideal")))
tot_s = sum(x[2] for x in lines) or 1
tot_i = sum(x[3] for x in lines) or 1
print(f"total samples {tot_s:.0f}  instructions {tot_i:.3e}  smem wavefronts {sum(x[4] for x in lines):.3e}"
      f" (ideal {sum(x[5] for x in lines):.3e})")
for ln, src, s, i, wf, wi in sorted(lines, key=lambda x: -x[2])[:n]:
    print(f"{ln:5d} samp {100*s/tot_s:5.1f}%  inst {100*i/tot_i:5.1f}%  wf {wf:11.0f} ideal {wi:11.0f}  {src}")
