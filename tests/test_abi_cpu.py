"""CPU-only checks of the C-ABI library: it builds, loads, exports every
symbol include/sieve.h declares, validates arguments before touching the
device, and fails loudly (no CPU fallback) without a GPU."""
import re

import pytest

import paper_1205_4883_b200 as sv

HEADER = __import__("os").path.join(__import__("os").path.dirname(__file__), "..", "include", "sieve.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[a-z_0-9]+\s+\**)+\**(sieve_[a-z_0-9]+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    names = declared_symbols()
    assert "sieve_count" in names and "sieve_bitmap" in names and "sieve_primes" in names
    L = sv.lib()
    for n in names:
        assert hasattr(L, n), n


def test_pure_host_helpers():
    assert sv.bitmap_words(2, 10**7 + 1) == 156250
    assert sv.bitmap_words(2, 10**9 + 1) == 15625000
    assert sv.bitmap_words(5, 5) == 0
    assert sv.bitmap_words(2, 3) == 0
    assert sv.bitmap_words(0, 1) == 0
    assert sv.bitmap_words(0, 2) == 1
    assert sv.base_capacity(10**5) >= 9591
    assert sv.base_capacity(1004987) >= 78865
    assert sv.base_capacity(3161577) >= 227611


def test_validation_before_device():
    with pytest.raises(sv.SieveError) as e:
        sv.count(10, 5)
    assert e.value.code == -1
    with pytest.raises(sv.SieveError) as e:
        sv.count(0, (1 << 48) + 1)
    assert e.value.code == -2
    with pytest.raises(sv.SieveError):
        sv.set_options(segment_kb=3)
    with pytest.raises(sv.SieveError):
        sv.set_options(wheel=19)
    sv.set_options(segment_kb=64, wheel=47)
    with pytest.raises(sv.SieveError):
        sv.set_options(segment_kb=208, wheel=47)  # 208 KiB + 25 KiB of tables > 226 KiB
    assert sv.get_options()["segment_kb"] == 64
    with pytest.raises(sv.SieveError):
        sv.set_options(bitmap_count_only=2)
    sv.set_options(bitmap_count_only=1)
    assert sv.get_options()["bitmap_count_only"] == 1
    sv.set_options()
    assert sv.get_options() == {"segment_kb": 208, "wheel": 31, "ctas_per_sm": 0, "threads": 1024,
                                 "buckets": 0, "bitmap_count_only": 0}


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sv.SieveError) as e:
        sv.count(2, 100)
    assert e.value.code == -5


def test_planning_before_any_option_call():
    """A device-resident call made before any set_options/sync call plans
    with the default options (it used to divide by a zero segment size):
    without a GPU it must fail with SIEVE_ENODEV or SIEVE_EINVAL, not crash."""
    import subprocess
    import sys
    code = ("import paper_1205_4883_b200 as sv, torch\n"
            "try:\n"
            "    sv.lib().sieve_stats_base_async(2, 10**10 + 1, 1, 1, 1, 10**6, 0, 1)\n"
            "except Exception as e:\n"
            "    print(e)\n"
            "print('alive', sv.lib().sieve_stats_base_async(2, 10**10 + 1, 1, 1, 1, 10**6, 0, 1))\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert p.returncode == 0, p.stderr
    assert "alive" in p.stdout
