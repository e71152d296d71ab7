#!/usr/bin/env python
"""Headline benchmark: sieved integers/s for pi(N), N = 1e10 (BASELINE.json
configs[2], "config 3"), count + prime sum, on 1/2/4/8 B200 (one process per
GPU under torchrun).

One step = one pass of the whole hot path:
  A2 base primes -> A3-A6 segmented sieve of the rank's block (count + sum)
  -> A9 all-reduce (N>1).  By default ONE kernel launch per rank does all of
  it: the base primes of the rank's block are computed inside the sieve
  kernel (fused A2, cooperative launch), and the all-reduce runs in its last
  CTA over NVLink peer memory (F4, csrc/peer.cuh).  --broadcast: K1 on rank 0
  + NCCL broadcast instead; --allreduce nccl: a separate NCCL all-reduce.

Timing: W untimed warm-up steps; then K steps bracketed by barrier +
synchronize on both sides; every step is timed with CUDA events on the
library stream (the stream the kernels launch on) and L2 is flushed between
steps outside the events; max over ranks.  `value` = integers of the whole
range / device seconds per step.  `e2e` = the same metric through the public
host API (sieve_stats with host outputs, or dist.stats for N>1), host clock.

`--impl reference` times the CPU oracle (the reference arm of this tier) on
a bounded sample of the same workload on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sieved integers/sec (π(N), N=1e10) at 1/2/4/8 B200; % of roofline"
UNIT = "integers/s"
CONFIG3 = (2, 10**10 + 1)
PI_1E10 = 455052511                  # BASELINE.json north_star
SUM_1E10 = 2220822432581729238       # SURVEY.md 8(c) C3 (Lucy-Hedgehog)
WHEEL_BASELINE_MD = 19               # BASELINE.md 4 quotes M_alg with wheel bound 19 (secondary field)
SMEM_LANES_PER_CLK_NOMINAL = 32      # one shared-memory wavefront / clk / SM (fallback if K0 fails)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--seg-kb", type=int, default=0)
    ap.add_argument("--wheel", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--ctas-per-sm", type=int, default=0)
    ap.add_argument("--broadcast", action="store_true",
                    help="rank 0 computes the base primes and NCCL-broadcasts them (default: every "
                         "rank recomputes them, 18 us for config 3 -- no collective on the path)")
    ap.add_argument("--split", choices=["equal", "cost"], default="equal",
                    help="N>1 block split: equal contiguous blocks (config 3, default) or "
                         "cost-weighted blocks (dist.block_of split='cost')")
    ap.add_argument("--allreduce", choices=["fused", "nccl"], default="fused",
                    help="N>1: the (count, sum) all-reduce inside the sieve kernel over NVLink peer "
                         "memory (F4, csrc/peer.cuh; falls back to nccl on every rank if any rank "
                         "cannot attach or verify it) or a separate NCCL all-reduce")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=10**10 - 1,
                    help="integers of config 3 the oracle sieves for cpu_baseline (default: all)")
    ap.add_argument("--cpu-sample-t1", type=int, default=10**9,
                    help="integers of config 3 the single-thread oracle run sieves")
    ap.add_argument("--ref-budget-s", type=float, default=200.0,
                    help="--impl reference: the K timed steps take about this long in all; each step "
                         "is the whole config-3 range when that fits, else an equal prefix sample")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """pynvml sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, index: int, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def sample_now(self):
        """One sample from the calling thread (the timed loop calls it after
        enqueuing its steps, while the GPU still runs them)."""
        if self.ok:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


# ----------------------------------------------------------------- roofline
def algorithmic_marks(lo: int, hi: int, wheel: int) -> int:
    """M_alg: number of (odd prime p, odd multiple m) pairs with wheel < p <=
    isqrt(hi-1) and max(lo, p^2) <= m < hi -- the marks the method must make
    beyond the wheel bound the build uses ("M_alg is the
    exact mark count ... for the wheel bound the build uses")."""
    import numpy as np
    if hi <= lo or hi < 10:
        return 0
    r = math.isqrt(hi - 1)
    s = np.ones(r + 1, dtype=bool)
    s[:2] = False
    for q in range(2, math.isqrt(r) + 1):
        if s[q]:
            s[q * q::q] = False
    p = np.nonzero(s)[0].astype(object)
    p = [int(x) for x in p if x > wheel]
    total = 0
    for q in p:
        a = max(lo, q * q)
        m0 = ((a + q - 1) // q) * q
        if m0 % 2 == 0:
            m0 += q
        if m0 < hi:
            total += (hi - 1 - m0) // (2 * q) + 1
    return total


def load_ncu_summary() -> dict:
    """Per-launch counters of the sieve kernel from the committed ncu capture
    (tools/make_profile_summary.py): DRAM traffic and the hardware view."""
    path = os.path.join(ROOT, "profiles", "ncu_sieve_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


# ----------------------------------------------------------------- reference arm
def host_cpu() -> dict:
    """The host the oracle runs on: logical CPUs (nproc) and model name."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import oracle
    lo, hi = CONFIG3
    cores = oracle.default_threads()
    # warm-up steps on a 10^9 prefix, which also measures the oracle's rate;
    # each timed step is then the whole range if K of them fit the budget,
    # else an equal prefix sample sized to it (stated in config/cpu_baseline)
    rate = None
    for _ in range(max(args.warmup, 1)):
        t0 = time.perf_counter()
        oracle.stats(lo, lo + 10**9, cores)
        rate = 10**9 / (time.perf_counter() - t0)
    n = hi - lo
    if n / rate * args.steps > args.ref_budget_s:
        n = max(10**8, int(rate * args.ref_budget_s / args.steps) // 10**8 * 10**8)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        c, s = oracle.stats(lo, lo + n, cores)
        times.append(time.perf_counter() - t0)
    per = sum(times) / len(times)
    value = n / per
    full = n == hi - lo
    if full:
        assert (c, s) == (PI_1E10, SUM_1E10), (c, s)
    sample = (f"[2, {lo + n}) of config 3 ({n} integers, "
              f"{'the whole range' if full else 'prefix sample'}) per step, count+sum, {cores} threads")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": "config3: pi(1e10) count + prime sum over [2, 1e10+1)"
                               + ("" if full else " (oracle prefix sample)"),
                   "lo": lo, "hi": lo + n, "sample_integers": n, "same_config": full},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "threads": cores,
                         "kind": "oracle", "sample": sample, **host_cpu()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


def cpu_baseline(args):
    """The oracle (never tuned) on the host cores: the whole config-3 range
    with all hardware threads, and a single-thread run on a prefix sample."""
    import oracle
    cores = oracle.default_threads()
    lo, hi = CONFIG3
    n = min(args.cpu_sample, hi - lo)
    t0 = time.perf_counter()
    c, s = oracle.stats(lo, lo + n, cores)
    dt = time.perf_counter() - t0
    whole = n == hi - lo
    out = {"value": n / dt, "unit": UNIT, "cores": cores, "threads": cores, "kind": "oracle",
           "sample": (f"[2, {lo + n}) = " + ("the whole config-3 range" if whole else
                                             f"first {n} integers of config 3")
                      + f", count+sum, one run, {dt:.2f} s, {cores} threads"),
           "verified": (c, s) == (PI_1E10, SUM_1E10) if whole else None, **host_cpu()}
    n1 = min(args.cpu_sample_t1, hi - lo)
    if n1 > 0:
        t0 = time.perf_counter()
        oracle.stats(lo, lo + n1, 1)
        d1 = time.perf_counter() - t0
        out["t1"] = {"value": n1 / d1, "unit": UNIT, "threads": 1,
                     "sample": f"[2, {lo + n1}) = first {n1} integers of config 3, one run, {d1:.2f} s"}
    return out


# ----------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as tdist

    import paper_1205_4883_b200 as sv
    from paper_1205_4883_b200 import dist as D

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)
    sv.set_device(local)
    stream = torch.cuda.Stream(device=dev)
    sv.set_stream(stream)
    sv.set_options(segment_kb=args.seg_kb, wheel=args.wheel, threads=args.threads,
                   ctas_per_sm=args.ctas_per_sm)
    opts = sv.get_options()

    lo, hi = CONFIG3
    r = math.isqrt(hi - 1)
    base = D.alloc_base(sv.base_capacity(r), dev)
    result = torch.zeros(2, dtype=torch.int64, device=dev)
    a, b = D.block_of(lo, hi, rank, world, args.split)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2
    bcast = world > 1 and args.broadcast
    fused = world > 1 and args.allreduce == "fused"

    def all_ok(ok: bool) -> bool:  # the same decision on every rank
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MIN)
        return bool(t.item())

    if fused:
        # every rank completes the attach collectives even if its own attach
        # fails (e.g. CUDA IPC unavailable); the ranks then agree
        ok = D.attach_peers(timeout_ms=2000)
        if not ok:
            print(f"rank {rank}: fused all-reduce unavailable", file=sys.stderr)
        if not all_ok(ok):
            fused = False
            D.detach_peers()

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]

    def step(e=None):
        with torch.cuda.stream(stream):
            if e: e[0].record(stream)
            if bcast:  # A2 on rank 0 + A9 NCCL broadcast, then the sieve
                if rank == 0:
                    sv.base_primes_async(r, base.primes, base.recips, base.nbase)
                tdist.broadcast(base.packed, src=0)
                if e: e[1].record(stream)
                if fused:
                    sv.stats_allreduce_async(a, b, base.primes, base.recips, base.nbase, result)
                else:
                    sv.stats_async(a, b, base.primes, base.recips, base.nbase, result)
            else:  # A2 + A3..A7 (+ the fused all-reduce) in one launch
                if e: e[1].record(stream)
                sv.stats_base_async(a, b, base.primes, base.recips, base.nbase, result, fused)
            if e: e[2].record(stream)
            if world > 1 and not fused:
                tdist.all_reduce(result, op=tdist.ReduceOp.SUM)
            if e: e[3].record(stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    got = [D.i64_to_u64(x) for x in result.cpu().tolist()]
    verified = (got[0] == PI_1E10 and got[1] == SUM_1E10)
    if fused and not all_ok(verified):  # fall back together, re-warm
        print(f"rank {rank}: fused all-reduce gave {got}; using NCCL", file=sys.stderr)
        fused = False
        D.detach_peers()
        for _ in range(max(args.warmup, 0)):
            step()
        torch.cuda.synchronize()
        got = [D.i64_to_u64(x) for x in result.cpu().tolist()]
        verified = (got[0] == PI_1E10 and got[1] == SUM_1E10)

    # K0: the conflict-free shared atomicOr rate of this
    # GPU, measured in this run, outside the timed region
    try:
        k0_lanes, k0_ghz = sv.debug_k0()
    except Exception as e:  # noqa: BLE001
        print(f"rank {rank}: K0 failed ({e}); nominal 32 lanes/clk", file=sys.stderr)
        k0_lanes, k0_ghz = None, None
    launches0 = sv.kernel_launches()
    sampler = ClockSampler(local)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    with sampler:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush, outside the events
            step(ev[k])
            if k == args.steps // 2:
                sampler.sample_now()  # the GPU is busy with the steps enqueued so far
        sampler.sample_now()
        torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    launches = sv.kernel_launches() - launches0

    step_ms = [e[0].elapsed_time(e[3]) for e in ev]
    sieve_ms = [e[1].elapsed_time(e[2]) for e in ev]
    base_ms = [e[0].elapsed_time(e[1]) for e in ev]
    tot = torch.tensor([sum(step_ms), sum(sieve_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(tot, op=tdist.ReduceOp.MAX)
    ms_per_step = tot[0].item() / args.steps
    # the per-step distribution (each step's time the max
    # over ranks), median / min / max next to the mean
    per = torch.tensor(step_ms, dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(per, op=tdist.ReduceOp.MAX)
    per = per.tolist()
    sieve_ms_mean = tot[1].item() / args.steps
    value = (hi - lo) / (ms_per_step / 1e3)

    # e2e: the public API with host outputs, host clock, K steps
    if world == 1:
        for _ in range(2):
            sv.stats(lo, hi)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            c, s = sv.stats(lo, hi)
        e2e_s = (time.perf_counter() - t0) / args.steps
        verified = verified and (c, s) == (PI_1E10, SUM_1E10)
    else:
        for _ in range(2):
            D.stats(lo, hi, broadcast=bcast)
        tdist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            c, s = D.stats(lo, hi, broadcast=bcast)
        tdist.barrier()
        e2e_t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        tdist.all_reduce(e2e_t, op=tdist.ReduceOp.MAX)
        e2e_s = e2e_t.item() / args.steps
        verified = verified and (c, s) == (PI_1E10, SUM_1E10)

    if rank == 0:
        clocks = sampler.summary()
        peaks = load_peaks()
        sm_max = peaks.get("sm_max_mhz") or clocks.get("sm_max_mhz") or 1965.0
        f_sm = clocks.get("sm_mhz") or sm_max  # the measured clock under load (D2 f_SM)
        r_atom = k0_lanes if k0_lanes else SMEM_LANES_PER_CLK_NOMINAL
        w = opts["wheel"]
        # whole-job marks beyond the build's wheel /
        # max-over-ranks kernel time, against N x 148 x R_atom (K0) x f_SM
        m_alg = algorithmic_marks(lo, hi, w)
        achieved = m_alg / (sieve_ms_mean / 1e3) / 1e9
        peak = world * 148 * r_atom * f_sm * 1e6 / 1e9
        ncu = load_ncu_summary()
        m19 = algorithmic_marks(lo, hi, WHEEL_BASELINE_MD)
        roof = {"bound": "smem_atomic", "achieved": achieved, "peak": peak, "unit": "Gmarks/s",
                "frac": achieved / peak, "traffic": ncu.get("dram_bytes_per_launch"),
                "kernel": "sv::k_sieve<NG,kCount>" + ("" if bcast else " (A2 fused)"),
                "wheel": w, "marks_alg_per_launch": algorithmic_marks(a, b, w), "marks_alg_job": m_alg,
                "peak_basis": (f"{world} x 148 SMs x R_atom {r_atom:.3f} lanes/clk (K0 in this run"
                               + ("" if k0_lanes else ": failed, nominal 32") + f") x f_SM {f_sm:.0f} MHz "
                               "(median SM clock sampled during the timed steps)"),
                "k0": {"lanes_per_clk_per_sm": k0_lanes, "sm_ghz": k0_ghz},
                "w19": {"marks_alg_job": m19, "frac": m19 / (sieve_ms_mean / 1e3) / 1e9 / peak,
                        "note": "M_alg with the wheel bound 19 of BASELINE.md 4 (context only)"},
                "hw": {k: ncu.get(k) for k in ("atomic_lane_util", "lane_atomics_per_launch",
                                                "smem_pipe_pct", "atomic_wavefronts_per_instr",
                                                "issue_active_pct", "tag")},
                "kernel_ms": sieve_ms_mean, "kernel_share_of_step": sieve_ms_mean / ms_per_step}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "config3: pi(1e10) count + prime sum over [2, 1e10+1)",
                       "lo": lo, "hi": hi, "segment_kb": opts["segment_kb"], "wheel": opts["wheel"],
                       "threads": opts["threads"], "base_primes": "rank 0 + NCCL broadcast" if bcast else "per rank, fused into the sieve launch",
                       "l2": "flushed (256 MiB write) between timed steps, outside the events",
                       "parallelism": f"range split over {world} GPU(s)" + (f", {args.split} blocks" if world > 1 else ""),
                       "allreduce": ("none" if world == 1 else
                                     "fused in the sieve kernel (NVLink peer memory)" if fused
                                     else "NCCL all_reduce")},
            "verified": verified,
            "step_ms": {"median": statistics.median(per), "min": min(per), "max": max(per),
                        "n": len(per), "note": "per timed step, max over ranks (CUDA events)"},
            "base_ms": statistics.mean(base_ms),
            "wall_ms_per_step_incl_flush": t_wall * 1e3 / args.steps,
            "roofline": roof,
            "clocks": clocks,
            "gpu_launches": launches,
            "e2e": {"value": (hi - lo) / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 16, "ms_per_step": e2e_s * 1e3,
                    "api": "sieve_stats (host outputs)" if world == 1 else "dist.stats",
                    "inputs": "lo, hi travel as kernel parameters (no input buffer to copy); the "
                              "result (count, sum) is read back to the host every step"},
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(out), flush=True)
    if world > 1:
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
