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


def _run(args):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/dropin_check not built (needs /root/reference headers at build time)")
    r = subprocess.run([EXE, *map(str, args)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout)


@pytest.mark.parametrize("case", ["render_light", "render_dynsphere"])
def test_dropin_whole_render_frame(case, tmp_path):
    """Renderer::renderFrame (pipeline.hpp:84-230): the reference's Renderer and
    sdfgi::b200::Renderer (every per-frame stage but scene instancing/culling on the
    device) on the same scene file, frame by frame: FrameMetrics counts identical,
    composed pixels within the north-star 1e-3 (FP64)."""
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_util import load_render

    g = load_render(case)
    path = tmp_path / "scene.scene"
    path.write_text(g.scene_text)
    out = _run(["render", path, min(len(g.frames), 6), 64, 40, g.n_rays or 24])
    assert out["metric_mismatches"] == 0, out
    assert out["max_rel_err"] <= 1e-3, out


def test_dropin_free_functions():
    """The reference's free functions against the B200 batched entry points, in one
    C++ program (sponza-lite, one reference pass for the field): querySceneSdf,
    sphereTrace, softShadowTrace and convolveIrradiance bit-identical;
    interpolationStencil identical entries with weights to 1e-9 (algebraic MVC
    sines); shadeHit within 1e-9 relative; per-probe updateProbe with identical
    probe state and texels within 1e-3."""
    out = _run(["funcs", os.path.join(ROOT, "tests", "golden", "sponza", "scene.sdfs"), 12, 7, 9, 1.4, 32])
    for k in ("query_mismatches", "trace_mismatches", "shadow_mismatches", "convolve_mismatches",
              "stencil_mismatches", "probe_mismatches"):
        assert out[k] == 0, out
    assert out["stencil_max_abs_err"] <= 1e-9, out
    assert out["shade_hits"] > 100 and out["shade_max_rel_err"] <= 1e-9, out
    assert out["probe_max_rel_err"] <= 1e-3 and out["exact_texels"] >= 0.99 * out["texels"], out
