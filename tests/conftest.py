import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: CPU test that takes tens of seconds")


def pytest_sessionfinish(session, exitstatus):
    """When the whole suite runs against the bounds-check build
    (SIEVE_LIBRARY=.../libsieve_check.so), any out-of-bounds mark or store
    counted during it fails the session."""
    lib = os.environ.get("SIEVE_LIBRARY", "")
    if not lib.endswith("libsieve_check.so"):
        return
    try:
        import paper_1205_4883_b200 as sv
        is_check, v = sv.debug_violations()
    except Exception as e:  # noqa: BLE001 -- no GPU: nothing ran
        print(f"\nbounds-check build: violations not read ({e})")
        return
    print(f"\nbounds-check build: violations [smem, bitmap, list, scratch] = {v}")
    if is_check and any(v):
        session.exitstatus = 1
