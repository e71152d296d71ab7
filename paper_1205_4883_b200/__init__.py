"""B200-native segmented sieve of Eratosthenes (arxiv 1205.4883 hot path).

The compute path is entirely inside ``libsieve.so`` (hand-written sm_100a
kernels behind the C ABI of ``include/sieve.h``).  This package is argument
marshalling only: it loads the library with ctypes and exposes the same
calls.  There is no CPU fallback -- if the library or a CUDA device is
missing, every compute call raises.
"""
from ._abi import (  # noqa: F401
    IPC_HANDLE_BYTES,
    MAX_PEERS,
    PEER_SLAB_BYTES,
    SieveError,
    base_capacity,
    base_primes_async,
    batch,
    bitmap,
    bitmap_async,
    bitmap_words,
    count,
    debug_set_flags,
    debug_set_profile,
    fermat,
    get_options,
    get_stream,
    is_prime,
    kernel_launches,
    lib,
    library_path,
    modpow,
    peer_attach,
    peer_attach_ptrs,
    peer_detach,
    peer_epoch,
    peer_slab_handle,
    prepare_base_async,
    primes,
    set_device,
    set_options,
    set_stream,
    shutdown,
    stats,
    stats_allreduce_async,
    stats_async,
    stats_base_async,
)

__all__ = [
    "SieveError", "count", "bitmap", "primes", "stats", "batch", "bitmap_words",
    "base_capacity", "base_primes_async", "prepare_base_async", "stats_async", "bitmap_async",
    "set_device", "set_stream", "get_stream", "set_options", "get_options", "shutdown",
    "kernel_launches", "lib", "library_path", "modpow", "fermat", "is_prime",
    "peer_slab_handle", "peer_attach", "peer_attach_ptrs", "peer_detach", "peer_epoch",
    "stats_allreduce_async", "stats_base_async", "IPC_HANDLE_BYTES", "MAX_PEERS", "PEER_SLAB_BYTES",
]
