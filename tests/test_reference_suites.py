"""The reference's own doctest suites (test_frontend.cpp, test_fusion.cpp,
test_interp.cpp), compiled unmodified from /root/reference with the doctest
subset in integration/doctest/doctest.h (oracle/Makefile `ref_suites`).

CPU control (this file): the suites against the unmodified af::interpret
must all pass -- it pins the harness itself. The same suites with every
af::interpret call routed to the B200 executor run in
tests/test_reference_suites_gpu.py."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
SUITES = ["test_frontend", "test_fusion", "test_interp"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_cpu_control(suite):
    exe = os.path.join(REF, suite + "_cpu")
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "0 failed" in r.stdout
