"""Key counters of one `ncu --set full` report (first kernel in it), for
profiles/: duration, DRAM bytes, instructions, issue activity, shared-memory
wavefronts and atomics, and the sampled warp-stall reasons.

Usage: python tools/ncu_summary.py REPORT TITLE
"""
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed_op_shared_atom.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"]
print(f"# {title}")
for k in want:
    if k in h:
        i = h.index(k)
        print(f"{k} = {v[i]} {units[i]}".rstrip())
st = [(float(v[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, k in enumerate(h)
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
      and v[i] not in ("", "0")]
tot = sum(x for x, _ in st) or 1.0
print("stall samples: " + ", ".join(f"{k} {100 * x / tot:.0f}%" for x, k in sorted(st, reverse=True)[:8]))
