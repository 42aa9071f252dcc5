"""The drop-in: the reference's own probe stage vs the same stage with
updateProbePositions / parallelFor(updateProbe) replaced by the B200 shim
(paper_2007_14394_b200/include/sdfgi_b200.hpp), in ONE C++ program built against
the unmodified reference headers (oracle/dropin_check.cpp)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "dropin_check")

pytestmark = pytest.mark.gpu


def run(scene, passes, res, spacing, nrays):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/dropin_check not built (needs /root/reference headers at build time)")
    r = subprocess.run([EXE, os.path.join(ROOT, "tests", "golden", scene, "scene.sdfs"), str(passes), *map(str, res),
                        str(spacing), str(nrays)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout)


def test_dropin_cornell_three_passes_bit_exact():
    out = run("c1", 3, (8, 8, 8), 1.0, 64)
    assert out["probe_mismatches"] == 0
    assert out["max_rel_err"] <= 1e-3
    assert out["exact_texels"] >= 0.99 * out["texels"]


def test_dropin_sponza_two_passes():
    out = run("sponza", 2, (12, 7, 9), 1.4, 32)
    assert out["probe_mismatches"] == 0
    assert out["max_rel_err"] <= 1e-3
    assert out["exact_texels"] >= 0.99 * out["texels"]
