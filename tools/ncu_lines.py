"""Summarise an ncu source page (cuda,sass view) per CUDA source line:
warp-stall samples, executed warp instructions and shared wavefronts."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, fname, res = None, "", []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or not r[0]:
        continue
    def g(k):
        i = hdr.index(k)
        try:
            return int(r[i])
        except ValueError:
            return 0
    s, ie = g("Warp Stall Sampling (All Samples)"), g("Instructions Executed")
    if s or ie:
        res.append((s, ie, fname, r[0], r[1].strip()[:80], g("L1 Wavefronts Shared"),
                    g("L1 Wavefronts Shared Ideal")))
tot = sum(x[0] for x in res) or 1
toti = sum(x[1] for x in res) or 1
print(f"total samples {tot}, warp instructions {toti}")
for s, ie, f, ln, src, wf, wfi in sorted(res, reverse=True)[:n]:
    print(f"{100*s/tot:5.1f}% {100*ie/toti:5.1f}%i {f}:{ln:>4} wf={wf}/{wfi} {src}")
