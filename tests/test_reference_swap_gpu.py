"""The reference's own checkLowering (test_frontend.cpp:22-37), compiled
against the unmodified reference library, with the B200 executor swapped in
through the integration adapter (integration/af_gpu.cpp): for every graph of
the reference's test_frontend.cpp plus the BASELINE patterns,
af::compareOutputs(af::gpu::execute(g, inputs), af::interpret(p, inputs)
.outputs, profile) must pass (F32 1e-6; Int exact; F16Fragment 2e-3 for the
f16 patterns). Binary built by `make -C oracle check_lowering`."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "check_lowering_gpu")
CASES = os.path.join(ROOT, "tests", "golden", "check_lowering_cases.json")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="reference swap driver not built "
                    "(needs /root/reference at build time)")
def test_check_lowering_with_gpu_executor(cuda):
    r = subprocess.run([BIN, CASES], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    # per case: graph executor, program executor, orchestrated program (outputs
    # and interpreter metrics)
    assert r.stdout.count("PASS graph") == 24
    assert r.stdout.count("PASS program") == 24
    # orchestrate() output the reference's own interpreter cannot run (it throws
    # "unbound iv" on some conv graphs) is skipped, and reported
    n_orch = 24 - r.stdout.count("SKIP orchestrated")
    assert n_orch >= 12, r.stdout
    assert r.stdout.count("PASS orchestrated") == n_orch
    assert r.stdout.count("PASS metrics") == n_orch
