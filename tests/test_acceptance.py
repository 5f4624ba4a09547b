"""The reference's own acceptance gate (proj/tests/acceptance.cpp, 11 criteria), compiled
unmodified against this repo's drop-in headers (include/tmatch) and linked to the B200
library (oracle/Makefile `acceptance` -> oracle/_ref/acceptance_b200): every criterion must
PASS on the GPU -- bound validity, 200 plantings equal to brute force with 0 soundness
violations, the frozen elimination anchors 93.75 % / 94.97 % (+-2), cost exactness, the xi
discipline, exit fidelity, 1x1 == brute and delta-kernel == EGS, the running-sum oracle and
threshold insensitivity (acceptance.cpp:53-55, 60-434)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


@pytest.mark.gpu
def test_reference_acceptance_on_b200():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs /root/reference at build)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1500)
    print(r.stdout)
    lines = [ln for ln in r.stdout.splitlines() if re.match(r"\[\s*\d+\]", ln)]
    assert len(lines) == 11, r.stdout + r.stderr
    assert all(" PASS " in ln for ln in lines), r.stdout
    assert "ALL CRITERIA PASS" in r.stdout and r.returncode == 0


def test_acceptance_binary_links_the_b200_library():
    """CPU: the gate program is linked to libtmatch.so (not to the reference library)."""
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/acceptance_b200 not built")
    out = subprocess.run(["readelf", "-d", BIN], capture_output=True, text=True).stdout
    assert "libtmatch.so" in out and "libtmatch_ref" not in out
