"""Bounds-check build ("no worker writes outside its segment's
bitmap ... ownership checks in debug builds"): every
kernel path runs against the oracle with libsieve_check.so, whose kernels
count every shared-memory mark outside the CTA's segment words, every
bitmap / list store outside the caller's array and every scratch write
outside its capacity (include/sieve.h sieve_debug_violations).  All four
counts must be zero."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_1205_4883_b200", "libsieve_check.so")


def test_every_path_in_bounds_check_build():
    assert os.path.exists(CHECK_LIB), "build it: make check (or __graft_entry__.build())"
    env = dict(os.environ, SIEVE_LIBRARY=CHECK_LIB)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bounds_check_run.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["check_build"] is True and out["library"] == CHECK_LIB
    assert out["cases"] > 50
    assert out["violations"] == [0, 0, 0, 0], out


def test_product_build_reports_no_checks():
    import paper_1205_4883_b200 as sv
    is_check, v = sv.debug_violations()
    assert v == [0, 0, 0, 0]
    assert is_check == (os.path.basename(sv.library_path) == "libsieve_check.so")
