"""Per-region cost breakdown of the sieve kernel from one `ncu --set full`
capture: instructions by pipe class, shared-memory wavefronts (actual and
ideal) and warp-stall samples, attributed to the marking regions (A1, A2, B,
C; the plain pass of the batch / kPlain kernels), the wheel init, the epilogue and the rest, through the inlined-line
annotations of `nvdisasm -gi` (the library is built with -lineinfo).

Usage: python tools/sass_regions.py REPORT [KERNEL_MANGLED]
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
SRC = os.path.join(ROOT, "paper_1205_4883_b200", "csrc", "kernels.cu")
LIB = os.path.join(ROOT, "paper_1205_4883_b200", "libsieve.so")
rep = sys.argv[1]

def _captured_kernel(report):
    """Mangled name of the k_sieve<NG, MODE> instantiation in the report."""
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    name = rows[2][rows[0].index("Kernel Name")]
    m = re.search(r"k_sieve<(\d+), (\d+)(?:, (\d+|true|false))?>", name)
    if not m:
        raise SystemExit(f"not a k_sieve capture: {name}")
    if m.group(3) is None:  # round-1 kernels: two template parameters
        return f"_ZN2sv7k_sieveILi{m.group(1)}ELi{m.group(2)}EEEvNS_11SieveParamsE"
    b = 1 if m.group(3) in ("1", "true") else 0
    return f"_ZN2sv7k_sieveILi{m.group(1)}ELi{m.group(2)}ELb{b}EEEvNS_11SieveParamsE"


fn = sys.argv[2] if len(sys.argv) > 2 else _captured_kernel(rep)

# ---- region line ranges from markers in the source
src = open(SRC).read().split("\n")


def line_of(pat, start=0):
    for i in range(start, len(src)):
        if re.search(pat, src[i]):
            return i + 1
    raise SystemExit(f"marker {pat!r} not found")


ms = line_of(r"^__device__ __forceinline__ void mark_segment")
regions = [
    ("wheel", line_of(r"^struct WheelGroup"), line_of(r"^struct PrimeRegions")),
    ("A1", line_of(r"// \(A1\) units", ms), line_of(r"// \(A2\) ", ms)),
    ("A2", line_of(r"// \(A2\) ", ms), line_of(r"// \(B\) one prime per warp", ms)),
    ("B", line_of(r"// \(B\) one prime per warp", ms), line_of(r"// \(C\) large primes", ms)),
    ("C", line_of(r"// \(C\) large primes", ms), line_of(r"// The plain primes \(batch kernel\)", ms)),
    ("plain", line_of(r"// The plain primes \(batch kernel\)", ms), line_of(r"if \(prof\) \{  // per-warp busy cycles", ms)),
    ("bucket", line_of(r"^__device__ __forceinline__ uint2 \*bucket_at"), line_of(r"^// In-place 32x32")),
    ("untranspose", line_of(r"^// In-place 32x32"), line_of(r"^// A6/A7: count, sum")),
    ("epilogue", line_of(r"^// A6/A7: count, sum"), line_of(r"^constexpr uint64_t kFlagAgg")),
    ("list", line_of(r"^constexpr uint64_t kFlagAgg"), line_of(r"^// block-wide sum of two u64")),
]


def region_of(chain):
    for ln in chain:  # innermost first
        for name, a, b in regions:
            if a <= ln < b:
                return name
    return "other"


# ---- offset -> region from nvdisasm -gi
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.startswith("kernels") and f.endswith(".cubin")]
    dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, sorted(cub)[-1])],
                         capture_output=True, text=True).stdout
off2reg = {}
inside = False
chain = []
for line in dis.split("\n"):
    if line.startswith("//----") and ".text." in line:
        inside = line.strip().endswith(".text." + fn + " --------------------------") or (".text." + fn) in line
        continue
    if not inside:
        continue
    if line.strip().startswith("//## File"):
        # (file, line) pairs, innermost first; only kernels.cu lines matter
        chain += [int(ln) for fname, ln in re.findall(r'"([^"]+)", line (\d+)', line)
                  if fname.endswith("kernels.cu")]
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", line)
    if m:
        if chain:
            off2reg[int(m.group(1), 16)] = region_of(chain)
            last = off2reg[int(m.group(1), 16)]
        else:
            off2reg[int(m.group(1), 16)] = off2reg.get(int(m.group(1), 16) - 16, "other")
        chain = []

# ---- ncu per-instruction metrics
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ix = {k: h.index(k) for k in h}


def f(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError):
        return 0.0


base = int(data[0][0], 16)
ALU = re.compile(r"^(LOP3|SHF|ISETP|IADD3|VIMNMX|VIADDMNMX|SEL|PRMT|FLO|LEA|IMNMX|PLOP3|VIADD|BMSK|SGXT|IABS)")
FMA = re.compile(r"^(IMAD|FFMA|FMUL|FADD|MOV|IADD\b)")
LSU = re.compile(r"^(LDS|STS|ATOMS|LDG|STG|LD|ST|RED|ATOM|LDC|SHFL)")
agg = defaultdict(lambda: defaultdict(float))
for r in data:
    off = int(r[0], 16) - base
    reg = off2reg.get(off, "other")
    op = r[1].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", op).split()[0] if op else ""
    cls = "alu" if ALU.match(op) else "fma" if FMA.match(op) else "lsu" if LSU.match(op) else "other"
    a = agg[reg]
    ie = f(r, "Instructions Executed")
    a["inst"] += ie
    a[cls] += ie
    a["atoms"] += ie if op.startswith("ATOMS") else 0
    a["wf"] += f(r, "L1 Wavefronts Shared")
    a["wfi"] += f(r, "L1 Wavefronts Shared Ideal")
    a["samp"] += f(r, "Warp Stall Sampling (All Samples)")
tot = {k: sum(a[k] for a in agg.values()) for k in ("inst", "wf", "samp")}
print(f"{'region':12s} {'samp%':>6s} {'inst M':>8s} {'alu M':>7s} {'fma M':>7s} {'lsu M':>7s} "
      f"{'atoms M':>8s} {'wf M':>7s} {'wf/ideal':>8s}")
for reg in ["wheel", "A1", "A2", "B", "C", "plain", "bucket", "untranspose", "epilogue", "list", "other"]:
    a = agg.get(reg)
    if not a:
        continue
    print(f"{reg:12s} {100 * a['samp'] / tot['samp']:6.1f} {a['inst'] / 1e6:8.1f} {a['alu'] / 1e6:7.1f} "
          f"{a['fma'] / 1e6:7.1f} {a['lsu'] / 1e6:7.1f} {a['atoms'] / 1e6:8.1f} {a['wf'] / 1e6:7.1f} "
          f"{(a['wf'] / a['wfi'] if a['wfi'] else 0):8.2f}")
print(f"{'total':12s} {100.0:6.1f} {tot['inst'] / 1e6:8.1f} {'':7s} {'':7s} {'':7s} {'':8s} {tot['wf'] / 1e6:7.1f}")

# SASS_DUMP=<region>: the region's instructions with their counts and samples
if os.environ.get("SASS_DUMP"):
    print(f"\n# {os.environ['SASS_DUMP']}: offset, executed (M warp instr), stall samples, SASS")
    for r in data:
        off = int(r[0], 16) - base
        if off2reg.get(off, "other") == os.environ["SASS_DUMP"]:
            print(f"{off:6x} {f(r, 'Instructions Executed') / 1e6:8.2f} {f(r, 'Warp Stall Sampling (All Samples)'):7.0f}  {r[1].strip()[:90]}")
