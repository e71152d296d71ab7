"""ctypes binding of libsieve.so -- one Python function per C entry point of
include/sieve.h, same names without the ``sieve_`` prefix.  Marshalling only.

Host outputs are numpy arrays; device outputs are torch CUDA tensors (their
``data_ptr()`` is passed straight through).  torch is imported lazily and is
needed only for the device-resident ``*_async`` calls.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SIEVE_LIBRARY overrides the path (tuning experiments with variant builds)
library_path = os.environ.get("SIEVE_LIBRARY") or os.path.join(_HERE, "libsieve.so")

SIEVE_MAX_HI = 1 << 48
_ERRNAMES = {-1: "SIEVE_EINVAL", -2: "SIEVE_ERANGE", -3: "SIEVE_ENOMEM", -4: "SIEVE_ECUDA",
             -5: "SIEVE_ENODEV"}

_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_p = ctypes.c_void_p


class SieveError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


class _Options(ctypes.Structure):
    _fields_ = [("segment_kb", ctypes.c_uint32), ("wheel", ctypes.c_uint32),
                ("ctas_per_sm", ctypes.c_uint32), ("threads", ctypes.c_uint32),
                ("buckets", ctypes.c_uint32), ("bitmap_count_only", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32 * 2)]


_lib = None


def lib():
    """Load libsieve.so (built in-tree by ``__graft_entry__.build()`` / make)."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise ImportError(f"{library_path} is missing: run `make` or __graft_entry__.build()")
        L = ctypes.CDLL(library_path)
        sig = {
            "sieve_count": (_i64, [_u64, _u64]),
            "sieve_bitmap": (_i64, [_u64, _u64, _p]),
            "sieve_primes": (_i64, [_u64, _u64, _p, _u64]),
            "sieve_bitmap_words": (_u64, [_u64, _u64]),
            "sieve_stats": (ctypes.c_int, [_u64, _u64, _p, _p]),
            "sieve_batch": (ctypes.c_int, [_p, _p, _u64, _p, _p]),
            "sieve_base_capacity": (_u64, [_u64]),
            "sieve_base_primes_async": (ctypes.c_int, [_u64, _p, _p, _u64, _p]),
            "sieve_prepare_base_async": (ctypes.c_int, [_p, _p, _p, _u64]),
            "sieve_stats_async": (ctypes.c_int, [_u64, _u64, _p, _p, _p, _p]),
            "sieve_bitmap_async": (ctypes.c_int, [_u64, _u64, _p, _p, _p, _p, _p]),
            "sieve_set_device": (ctypes.c_int, [ctypes.c_int]),
            "sieve_set_stream": (ctypes.c_int, [_p]),
            "sieve_get_stream": (_p, []),
            "sieve_set_options": (ctypes.c_int, [ctypes.POINTER(_Options)]),
            "sieve_get_options": (ctypes.c_int, [ctypes.POINTER(_Options)]),
            "sieve_last_error": (ctypes.c_char_p, []),
            "sieve_shutdown": (None, []),
            "sieve_kernel_launches": (_u64, []),
            "sieve_debug_set_profile": (ctypes.c_int, [_p]),
            "sieve_debug_set_flags": (ctypes.c_int, [ctypes.c_uint32]),
            "sieve_modpow": (ctypes.c_int, [_p, _p, _p, _u64, _p]),
            "sieve_fermat": (ctypes.c_int, [_p, _u64, _p, ctypes.c_uint32, _p]),
            "sieve_is_prime": (ctypes.c_int, [_p, _u64, _p]),
            "sieve_peer_slab_handle": (ctypes.c_int, [_p]),
            "sieve_peer_attach": (ctypes.c_int, [_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint32]),
            "sieve_peer_attach_ptrs": (ctypes.c_int, [_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint32]),
            "sieve_peer_detach": (ctypes.c_int, []),
            "sieve_peer_epoch": (_u64, []),
            "sieve_stats_allreduce_async": (ctypes.c_int, [_u64, _u64, _p, _p, _p, _p]),
            "sieve_stats_base_async": (ctypes.c_int, [_u64, _u64, _p, _p, _p, _u64, ctypes.c_int, _p]),
            "sieve_peer_publish_async": (ctypes.c_int, [_u64, _u64]),
            "sieve_batch_async": (ctypes.c_int, [_p, _p, _u64, _u64, _u64, _p]),
            "sieve_bitmap_base_async": (ctypes.c_int, [_u64, _u64, _p, _p, _p, _u64, _p, _p]),
            "sieve_debug_violations": (ctypes.c_int, [_p, ctypes.c_int]),
            "sieve_debug_k0": (ctypes.c_int, [_p, _p]),
            "sieve_debug_coop_fallbacks": (_u64, []),
        }
        for name, (res, args) in sig.items():
            try:
                f = getattr(L, name)
            except AttributeError:
                # an older variant build (SIEVE_LIBRARY, A/B runs) may lack a
                # newer entry point; calling it then raises AttributeError
                if library_path == os.path.join(_HERE, "libsieve.so"):
                    raise
                continue
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int) -> int:
    if rc < 0:
        raise SieveError(rc, lib().sieve_last_error().decode())
    return rc


def _ptr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()  # torch tensor


def _check_out(out, need: int, itemsize: int, what: str) -> None:
    """An output buffer must hold `need` elements of `itemsize` bytes (numpy
    array or torch tensor, contiguous): the C side writes exactly that many."""
    if hasattr(out, "element_size"):  # torch
        n, isz, contig = out.numel(), out.element_size(), out.is_contiguous()
    else:
        n, isz, contig = out.size, out.itemsize, out.flags["C_CONTIGUOUS"]
    if isz != itemsize or not contig:
        raise ValueError(f"{what}: need a contiguous buffer of {itemsize}-byte elements")
    if n < need:
        raise ValueError(f"{what}: buffer holds {n} elements, the call writes {need}")


# ---- north_star calls -----------------------------------------------------
def count(lo: int, hi: int) -> int:
    """Number of primes in [lo, hi)."""
    return _check(lib().sieve_count(lo, hi))


def bitmap_words(lo: int, hi: int) -> int:
    return int(lib().sieve_bitmap_words(lo, hi))


def bitmap(lo: int, hi: int, out=None):
    """Odd-only prime bitmap of [lo, hi) (uint32 words; reading R5).
    ``out`` may be a numpy uint32 array (host) or a torch int32/uint32 CUDA
    tensor (device).  Returns (out, count)."""
    w = bitmap_words(lo, hi)
    if out is None:
        out = np.zeros(max(w, 1), dtype=np.uint32)
    elif w:
        _check_out(out, w, 4, "bitmap out")
    c = _check(lib().sieve_bitmap(lo, hi, _ptr(out) if w else None))
    return out, c


def primes(lo: int, hi: int, cap: int | None = None, out=None):
    """Ascending uint64 primes of [lo, hi).  Returns (out, total_count)."""
    if cap is None:
        cap = count(lo, hi) if out is None else int(out.numel() if hasattr(out, "numel") else out.size)
    if out is None:
        out = np.zeros(max(cap, 1), dtype=np.uint64)
    elif cap:
        _check_out(out, cap, 8, "primes out")
    c = _check(lib().sieve_primes(lo, hi, _ptr(out) if cap else None, cap))
    return out, c


def stats(lo: int, hi: int) -> tuple[int, int]:
    """(count, sum of primes mod 2^64) of [lo, hi)."""
    c = ctypes.c_uint64()
    s = ctypes.c_uint64()
    _check(lib().sieve_stats(lo, hi, ctypes.addressof(c), ctypes.addressof(s)))
    return int(c.value), int(s.value)


def batch(lo, hi) -> tuple[np.ndarray, np.ndarray]:
    """Per-interval (count, sum mod 2^64) of the intervals [lo[i], hi[i])."""
    lo = np.ascontiguousarray(lo, dtype=np.uint64)
    hi = np.ascontiguousarray(hi, dtype=np.uint64)
    n = lo.size
    c = np.zeros(max(n, 1), dtype=np.uint64)
    s = np.zeros(max(n, 1), dtype=np.uint64)
    _check(lib().sieve_batch(lo.ctypes.data, hi.ctypes.data, n, c.ctypes.data, s.ctypes.data))
    return c[:n], s[:n]


# ---- device-resident API ----------------------------------------------------
def base_capacity(r: int) -> int:
    return int(lib().sieve_base_capacity(r))


def base_primes_async(r: int, primes_t, recips_t, nbase_t) -> None:
    _check(lib().sieve_base_primes_async(r, _ptr(primes_t), _ptr(recips_t), primes_t.numel(),
                                         _ptr(nbase_t)))


def prepare_base_async(primes_t, nbase_t, recips_t) -> None:
    _check(lib().sieve_prepare_base_async(_ptr(primes_t), _ptr(nbase_t), _ptr(recips_t),
                                          primes_t.numel()))


def stats_async(lo: int, hi: int, primes_t, recips_t, nbase_t, result_t) -> None:
    _check(lib().sieve_stats_async(lo, hi, _ptr(primes_t), _ptr(recips_t), _ptr(nbase_t),
                                   _ptr(result_t)))


def stats_base_async(lo: int, hi: int, primes_t, recips_t, nbase_t, result_t,
                     allreduce: bool = False) -> None:
    """Base primes (into primes_t/recips_t/nbase_t) and count/sum of [lo, hi)
    in one kernel launch (fused A2); allreduce: summed over attached peers."""
    _check(lib().sieve_stats_base_async(lo, hi, _ptr(primes_t), _ptr(recips_t), _ptr(nbase_t),
                                        primes_t.numel(), 1 if allreduce else 0, _ptr(result_t)))


def batch_async(lo_t, hi_t, hi_max: int, width_max: int, result_t) -> None:
    """Batch mode on device tensors (int64 views of the uint64 bounds):
    result_t[2i], result_t[2i+1] = count, sum mod 2^64 of [lo_t[i], hi_t[i])."""
    n = int(lo_t.numel())
    if hi_t.numel() != n or result_t.numel() < 2 * n:
        raise ValueError("batch_async: lo/hi of equal length and result of 2n entries")
    _check(lib().sieve_batch_async(_ptr(lo_t), _ptr(hi_t), n, hi_max, width_max, _ptr(result_t)))


def bitmap_base_async(lo: int, hi: int, primes_t, recips_t, nbase_t, out_t, result_t) -> None:
    """Base primes + bitmap of [lo, hi) in one launch; result_t = (count, sum)."""
    w = bitmap_words(lo, hi)
    if w:
        _check_out(out_t, w, 4, "bitmap out")
    _check(lib().sieve_bitmap_base_async(lo, hi, _ptr(primes_t), _ptr(recips_t), _ptr(nbase_t),
                                         primes_t.numel(), _ptr(out_t), _ptr(result_t)))


def bitmap_async(lo: int, hi: int, primes_t, recips_t, nbase_t, out_t, result_t) -> None:
    _check(lib().sieve_bitmap_async(lo, hi, _ptr(primes_t), _ptr(recips_t), _ptr(nbase_t),
                                    _ptr(out_t), _ptr(result_t)))


# ---- all-reduce fused into the sieve over peer memory ----
IPC_HANDLE_BYTES = 64
MAX_PEERS = 64
PEER_SLAB_BYTES = 2 * MAX_PEERS * 32


def peer_slab_handle() -> bytes:
    """This process's slab (allocated once) as a CUDA IPC handle."""
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check(lib().sieve_peer_slab_handle(ctypes.addressof(h)))
    return h.raw


def peer_attach(handles: list[bytes], rank: int, timeout_ms: int = 0) -> None:
    """Open the peers' slabs (handles in rank order, this rank's ignored)."""
    if any(len(h) != IPC_HANDLE_BYTES for h in handles):
        raise ValueError("every handle must be 64 bytes")
    buf = ctypes.create_string_buffer(b"".join(handles), IPC_HANDLE_BYTES * len(handles))
    _check(lib().sieve_peer_attach(ctypes.addressof(buf), len(handles), rank, timeout_ms))


def peer_attach_ptrs(slabs, rank: int, timeout_ms: int = 0) -> None:
    """Attach device slabs of this process (tensors or raw addresses, rank order)."""
    arr = (ctypes.c_void_p * len(slabs))(*[s if isinstance(s, int) else s.data_ptr() for s in slabs])
    _check(lib().sieve_peer_attach_ptrs(arr, len(slabs), rank, timeout_ms))


def peer_detach() -> None:
    _check(lib().sieve_peer_detach())


def peer_epoch() -> int:
    return int(lib().sieve_peer_epoch())


def peer_publish_async(count: int, sum_: int) -> None:
    """Publish this rank's (count, sum) for the next fused epoch, no wait."""
    _check(lib().sieve_peer_publish_async(count & ((1 << 64) - 1), sum_ & ((1 << 64) - 1)))


def stats_allreduce_async(lo: int, hi: int, primes_t, recips_t, nbase_t, result_t) -> None:
    _check(lib().sieve_stats_allreduce_async(lo, hi, _ptr(primes_t), _ptr(recips_t),
                                             _ptr(nbase_t), _ptr(result_t)))


# ---- Alg. 2, Alg. 3, deterministic Miller-Rabin ----------
def _u64arr(x):
    if hasattr(x, "data_ptr"):
        return x
    return np.ascontiguousarray(x, dtype=np.uint64)


def modpow(a, b, c, out=None):
    """Alg. 2 batched: a^b mod c elementwise (numpy uint64 arrays or CUDA int64 tensors)."""
    a, b, c = _u64arr(a), _u64arr(b), _u64arr(c)
    n = int(a.numel() if hasattr(a, "numel") else a.size)
    if out is None:
        out = np.zeros(n, dtype=np.uint64)
    _check(lib().sieve_modpow(_ptr(a), _ptr(b), _ptr(c), n, _ptr(out)))
    return out


def fermat(p, draws, iterations: int, out=None):
    """Alg. 3 batched: verdict per candidate (1 = passes `iterations` rounds with
    bases draws[i*iterations + t] mod (p-1) + 1)."""
    p, draws = _u64arr(p), _u64arr(draws)
    n = int(p.numel() if hasattr(p, "numel") else p.size)
    if out is None:
        out = np.zeros(n, dtype=np.uint8)
    _check(lib().sieve_fermat(_ptr(p), n, _ptr(draws), iterations, _ptr(out)))
    return out


def is_prime(nums, out=None):
    """Deterministic Miller-Rabin per 64-bit number (1 = prime)."""
    nums = _u64arr(nums)
    n = int(nums.numel() if hasattr(nums, "numel") else nums.size)
    if out is None:
        out = np.zeros(n, dtype=np.uint8)
    _check(lib().sieve_is_prime(_ptr(nums), n, _ptr(out)))
    return out


# ---- configuration ----------------------------------------------------------
def set_device(ordinal: int) -> None:
    _check(lib().sieve_set_device(ordinal))


def set_stream(stream) -> None:
    """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None."""
    if stream is None:
        h = None
    elif isinstance(stream, int):
        h = stream
    else:
        h = stream.cuda_stream
    _check(lib().sieve_set_stream(h))


def get_stream() -> int:
    return int(lib().sieve_get_stream() or 0)


def set_options(segment_kb: int = 0, wheel: int = 0, ctas_per_sm: int = 0, threads: int = 0,
                buckets: int = 0, bitmap_count_only: int = 0) -> None:
    o = _Options(segment_kb, wheel, ctas_per_sm, threads, buckets, bitmap_count_only)
    _check(lib().sieve_set_options(ctypes.byref(o)))


def get_options() -> dict:
    o = _Options()
    _check(lib().sieve_get_options(ctypes.byref(o)))
    return {"segment_kb": o.segment_kb, "wheel": o.wheel, "ctas_per_sm": o.ctas_per_sm,
            "threads": o.threads, "buckets": o.buckets, "bitmap_count_only": o.bitmap_count_only}


def shutdown() -> None:
    lib().sieve_shutdown()


def debug_set_profile(counters_t) -> None:
    """Diagnostics: phase-cycle counters (torch int64[8] CUDA tensor) or None."""
    _check(lib().sieve_debug_set_profile(_ptr(counters_t)))


def debug_set_flags(flags: int) -> None:
    """Diagnostics: 1 = skip marking (write-back-only timing; wrong results)."""
    _check(lib().sieve_debug_set_flags(flags))


def kernel_launches() -> int:
    return int(lib().sieve_kernel_launches())


FLAG_SKIP_MARKING, FLAG_SKIP_A, FLAG_SKIP_B, FLAG_SKIP_C = 1, 2, 4, 8
FLAG_REVERSE, FLAG_NO_COOP, FLAG_CLUSTER = 16, 32, 64


def debug_violations(reset: bool = False) -> tuple[bool, list[int]]:
    """(is the bounds-check build, [smem marks, bitmap stores, list stores,
    scratch writes] out of bounds since load / the last reset)."""
    out = np.zeros(4, dtype=np.uint64)
    rc = _check(lib().sieve_debug_violations(out.ctypes.data, 1 if reset else 0))
    return rc == 1, [int(x) for x in out]


def debug_k0() -> tuple[float, float]:
    """K0: conflict-free shared atomicOr lanes per SM-clock per SM, and the SM GHz."""
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(lib().sieve_debug_k0(ctypes.addressof(a), ctypes.addressof(b)))
    return a.value, b.value


def debug_coop_fallbacks() -> int:
    return int(lib().sieve_debug_coop_fallbacks())
