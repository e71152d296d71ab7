"""Turn one profiling pass (tools/gpurun_profile.sh output in gpurun_out/)
into the committed evidence under profiles/:

  profiles/<tag>_bench.json          the bench.py JSON line
  profiles/<tag>_modes.jsonl         tools/bench_modes.py lines (configs 1, 2, 4, 5)
  profiles/<tag>_k0_peaks.json       shared-memory / HBM microbenchmarks
  profiles/<tag>_launches.csv        ncu launch list (gpu__time_duration.sum)
  profiles/<tag>_ncu_sieve.txt       key counters of one `ncu --set full` capture
  profiles/<tag>_ncu_*regions.txt    per-region breakdowns (config 3, 5, 4 captures)
  profiles/ncu_sieve_summary.json    per-launch DRAM traffic of the sieve kernel
                                     (read by bench.py for roofline.traffic)
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out")
DST = os.environ.get("PROFILE_DST", os.path.join(ROOT, "profiles"))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rep = os.path.join(SRC, sys.argv[2] if len(sys.argv) > 2 else "prof_sieve.ncu-rep")
os.makedirs(DST, exist_ok=True)

for src, dst in [("bench.json", f"{tag}_bench.json"), ("modes.jsonl", f"{tag}_modes.jsonl"),
                 ("k0.json", f"{tag}_k0_peaks.json"), ("report.json", f"{tag}_report.json"),
                 ("rank_blocks.txt", f"{tag}_rank_blocks.txt"), ("f3_ab.jsonl", f"{tag}_f3_cluster_ab.jsonl"),
                 ("phase.json", f"{tag}_phase_counters.json"), ("pytest_gpu.log", f"{tag}_pytest_gpu.log")]:
    if os.path.exists(os.path.join(SRC, src)):
        shutil.copy(os.path.join(SRC, src), os.path.join(DST, dst))

# launch list: keep only the CSV rows, summarise shares per kernel
lp = os.path.join(SRC, "launches.csv")
lines = [l for l in open(lp) if l.startswith('"')] if os.path.exists(lp) else []
with open(os.path.join(DST, f"{tag}_launches.csv"), "w") as f:
    f.writelines(lines)
rows = list(csv.DictReader(lines))
tot = {}
for r in rows:
    k = r["Kernel Name"].split("(")[0]
    tot.setdefault(k, [0, 0])
    tot[k][0] += 1
    tot[k][1] += float(r["Metric Value"])
all_ns = sum(v[1] for v in tot.values())

# full capture: raw counters of the sieve kernel
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hdr, val = rr[0], rr[2]
m = dict(zip(hdr, val))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
        "smsp__inst_executed_op_shared_atom.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
units = dict(zip(hdr, rr[1]))


def num(k):
    try:
        return float(m.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


def to_bytes(k):
    u = units.get(k, "byte")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return num(k) * mult


dram = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")

# lane-level shared atomics (predicated-on thread instructions of the ATOMS
# SASS lines, from the source page): the hardware view of the roofline
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(src.splitlines()))
lane_atoms = 0
if len(srows) > 2:
    sh = srows[1]
    i_src, i_th = sh.index("Source"), sh.index("Predicated-On Thread Instructions Executed")
    for r in srows[2:]:
        if len(r) > i_th and "ATOMS" in r[i_src]:
            lane_atoms += int(r[i_th].replace(",", "") or 0)
cycles = num("sm__cycles_elapsed.avg")
nsm = 148
atom = num("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum")
conf = num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum")
with open(os.path.join(DST, "ncu_sieve_summary.json"), "w") as f:
    json.dump({"tag": tag, "kernel": m.get("Kernel Name"), "dram_bytes_per_launch": dram,
               "lane_atomics_per_launch": lane_atoms,
               "atomic_lane_util": lane_atoms / (nsm * 32 * cycles) if cycles == cycles and cycles else None,
               "smem_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
               "atomic_wavefronts_per_instr": atom / max(atom - conf, 1),
               "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
               "sm_cycles": cycles,
               "source": "ncu --set full --clock-control none, one launch of bench.py config 3; "
                         "atomic_lane_util = predicated-on ATOMS thread instructions / "
                         "(148 SMs x 32 lanes x SM cycles)"}, f, indent=1)

with open(os.path.join(DST, f"{tag}_ncu_sieve.txt"), "w") as f:
    f.write(f"# ncu --set full capture of the sieve kernel ({tag}); bench.py --steps 1 --warmup 0\n")
    for k in keys:
        f.write(f"{k} = {m.get(k)} {units.get(k, '')}\n")
    f.write(f"atomic wavefronts per atomic instruction = {atom / max(atom - conf, 1):.3f}\n")
    f.write(f"lane atomics (predicated-on ATOMS thread instructions) = {lane_atoms}\n")
    f.write(f"atomic lane utilisation = {lane_atoms / (nsm * 32 * cycles):.3f} of 148 x 32 lanes x cycles\n")
    f.write(f"dram bytes per launch = {dram:.0f}\n")
    f.write("\n# launch list shares (ncu, cold-cache, serialised)\n")
    step_ns = sum(ns for k, (n, ns) in tot.items() if "k_k0_atomics" not in k)
    for k, (n, ns) in sorted(tot.items(), key=lambda x: -x[1][1]):
        diag = "k_k0_atomics" in k
        f.write(f"{k}: launches={n} total_us={ns / 1e3:.1f} share={ns / all_ns:.3f}"
                + ("  (K0 microbenchmark, outside the timed steps)" if diag
                   else f" share_without_K0={ns / step_ns:.3f}") + "\n")
print(open(os.path.join(DST, f"{tag}_ncu_sieve.txt")).read())

# per-region breakdowns (tools/sass_regions.py) of the captures present
for cap, name, what in [("prof_sieve.ncu-rep", "ncu_regions", "config 3, bench.py step"),
                        ("prof_batch.ncu-rep", "ncu_batch_regions", "config 5, sieve_batch_async"),
                        ("prof_config4.ncu-rep", "ncu_config4_regions", "config 4, count kernel")]:
    cp = os.path.join(SRC, cap)
    if os.path.exists(cp):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_regions.py"), cp],
                             capture_output=True, text=True).stdout
        with open(os.path.join(DST, f"{tag}_{name}.txt"), "w") as f:
            f.write(f"# tools/sass_regions.py on the ncu --set full capture of {what} ({tag})\n{out}")
        print(out)
