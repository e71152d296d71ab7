"""CPU oracle for the sieve hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_1205_4883_b200`` never imports it, and the two share
no code: see ``oracle/oracle.c`` for what is computed and which passage of
PAPER.md each step follows.

This module is argument marshalling only (ctypes over ``liboracle.so``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "primality.c")]
_LIB = os.path.join(_HERE, "liboracle.so")

_u64 = ctypes.c_uint64
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (plain gcc -O2, no tuning)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f)
                                                   for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               *_SRCS, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_isqrt.argtypes = [_u64]
        L.oracle_isqrt.restype = _u64
        L.oracle_base_primes.argtypes = [_u64, _p, _u64]
        L.oracle_base_primes.restype = ctypes.c_int64
        L.oracle_bitmap_words.argtypes = [_u64, _u64]
        L.oracle_bitmap_words.restype = _u64
        L.oracle_sieve.argtypes = [_u64, _u64, ctypes.c_int, _p, _p, _p, _p, _u64]
        L.oracle_sieve.restype = ctypes.c_int
        L.oracle_fnv1a64.argtypes = [_p, _u64]
        L.oracle_fnv1a64.restype = _u64
        L.oracle_batch.argtypes = [_p, _p, _u64, ctypes.c_int, _p, _p]
        L.oracle_batch.restype = ctypes.c_int
        L.oracle_modpow.argtypes = [_u64, _u64, _u64]
        L.oracle_modpow.restype = _u64
        L.oracle_fermat.argtypes = [_u64, ctypes.c_uint32, _p]
        L.oracle_fermat.restype = ctypes.c_int
        L.oracle_modpow_batch.argtypes = [_p, _p, _p, _u64, _p]
        L.oracle_modpow_batch.restype = None
        L.oracle_fermat_batch.argtypes = [_p, _u64, _p, ctypes.c_uint32, _p]
        L.oracle_fermat_batch.restype = None
        _lib = L
    return _lib


def default_threads() -> int:
    return os.cpu_count() or 1


def isqrt(x: int) -> int:
    return int(lib().oracle_isqrt(x))


def base_primes(r: int) -> np.ndarray:
    """All primes <= r ascending (2 included), uint32."""
    n = lib().oracle_base_primes(r, None, 0)
    out = np.zeros(max(n, 1), dtype=np.uint32)
    n2 = lib().oracle_base_primes(r, out.ctypes.data, n)
    assert n2 == n
    return out[:n]


def bitmap_words(lo: int, hi: int) -> int:
    return int(lib().oracle_bitmap_words(lo, hi))


def _check(rc: int) -> None:
    if rc != 0:
        raise ValueError(f"oracle error {rc}")


def stats(lo: int, hi: int, threads: int | None = None) -> tuple[int, int]:
    """(count, sum mod 2^64) of the primes in [lo, hi)."""
    c = ctypes.c_uint64()
    s = ctypes.c_uint64()
    _check(lib().oracle_sieve(lo, hi, threads or default_threads(), ctypes.addressof(c),
                              ctypes.addressof(s), None, None, 0))
    return int(c.value), int(s.value)


def bitmap(lo: int, hi: int, threads: int | None = None) -> tuple[np.ndarray, int, int]:
    """(odd-only prime bitmap as uint32 words, count, sum)."""
    w = bitmap_words(lo, hi)
    bm = np.zeros(max(w, 1), dtype=np.uint32)
    c = ctypes.c_uint64()
    s = ctypes.c_uint64()
    _check(lib().oracle_sieve(lo, hi, threads or default_threads(), ctypes.addressof(c),
                              ctypes.addressof(s), bm.ctypes.data, None, 0))
    return bm[:w], int(c.value), int(s.value)


def primes(lo: int, hi: int, cap: int | None = None, threads: int | None = None) -> np.ndarray:
    """Ascending uint64 primes in [lo, hi) (at most ``cap``)."""
    c = ctypes.c_uint64()
    s = ctypes.c_uint64()
    if cap is None:
        _check(lib().oracle_sieve(lo, hi, threads or default_threads(), ctypes.addressof(c),
                                  ctypes.addressof(s), None, None, 0))
        cap = int(c.value)
    out = np.zeros(max(cap, 1), dtype=np.uint64)
    _check(lib().oracle_sieve(lo, hi, threads or default_threads(), ctypes.addressof(c),
                              ctypes.addressof(s), None, out.ctypes.data, cap))
    return out[:min(cap, int(c.value))]


def fnv1a64(buf) -> int:
    a = np.ascontiguousarray(buf)
    return int(lib().oracle_fnv1a64(a.ctypes.data, a.nbytes))


def batch(lo, hi, threads: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    lo = np.ascontiguousarray(lo, dtype=np.uint64)
    hi = np.ascontiguousarray(hi, dtype=np.uint64)
    n = lo.size
    cnt = np.zeros(max(n, 1), dtype=np.uint64)
    sm = np.zeros(max(n, 1), dtype=np.uint64)
    _check(lib().oracle_batch(lo.ctypes.data, hi.ctypes.data, n, threads or default_threads(),
                              cnt.ctypes.data, sm.ctypes.data))
    return cnt[:n], sm[:n]


# ---- Alg. 2 and Alg. 3 (oracle/primality.c) -------------
def modpow(a: int, b: int, c: int) -> int:
    """Alg. 2: a^b mod c; UINT64_MAX for c = 0."""
    return int(lib().oracle_modpow(a, b, c))


def modpow_batch(a, b, c) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    c = np.ascontiguousarray(c, dtype=np.uint64)
    out = np.zeros(a.size, dtype=np.uint64)
    lib().oracle_modpow_batch(a.ctypes.data, b.ctypes.data, c.ctypes.data, a.size, out.ctypes.data)
    return out


def fermat(p: int, iterations: int, draws) -> bool:
    """Alg. 3 with the caller's draws as rand()."""
    d = np.ascontiguousarray(draws, dtype=np.uint64)
    assert d.size >= iterations
    return bool(lib().oracle_fermat(p, iterations, d.ctypes.data))


def fermat_batch(p, draws, iterations: int) -> np.ndarray:
    p = np.ascontiguousarray(p, dtype=np.uint64)
    d = np.ascontiguousarray(draws, dtype=np.uint64)
    assert d.size >= p.size * iterations
    out = np.zeros(p.size, dtype=np.uint8)
    lib().oracle_fermat_batch(p.ctypes.data, p.size, d.ctypes.data, iterations, out.ctypes.data)
    return out
