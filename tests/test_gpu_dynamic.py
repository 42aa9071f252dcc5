"""C5 (BASELINE configs[4]): dynamic sequences — moving primitives and a moving,
dimming light — checked per frame against the reference. Each frame's scene is
instantiated by the package's own sceneAtTime + cullAndLod from the authored
scene text (bit-identical to the reference's, tests/test_scene_file.py), uploaded,
and taken through one probe pass (relocation + update, frame index = frame) on
persistent cascades with hysteresis blending."""
import numpy as np
import pytest

from golden_util import DYNAMIC_CASES, load_dynamic
from paper_2007_14394_b200 import api
from paper_2007_14394_b200 import scene_file as sf
from paper_2007_14394_b200.runtime import Device

pytestmark = pytest.mark.gpu


def texel_rel_err(got, want):
    floor = 0.05 * max(float(np.mean(np.abs(want))), 1e-12)
    return np.abs(got.astype(np.float64) - want) / np.maximum(np.abs(want), floor)


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("name", DYNAMIC_CASES)
def test_dynamic_sequence_matches_reference(name, precision):
    case = load_dynamic(name)
    scene = sf.parseScene(case.scene_text)
    fps = int(scene.config["fps"][0])
    with Device(0, precision=precision) as dev:
        stage = api.ProbeStage(dev, sf.activeScene(scene, 0.0), n_rays=case.n_rays)
        for fr, want in enumerate(case.frames):
            if fr:
                stage.set_scene(sf.activeScene(scene, fr / fps))
            reps, res = stage.run_pass(fr)
            assert [int(reps[0][k]) for k in ("relocated", "rejected", "dead")] == \
                [want["relocated"], want["rejected"], want["dead"]], (name, fr)
            assert int(res["rays_traced"]) == want["rays_traced"], (name, fr)
            assert int(res["probes_updated"]) == want["probes_updated"], (name, fr)
            if fr in case.dumped:
                got = dev.probes(0)
                ref = case.data[f"probes_f{fr}_c0"]
                for f in ("pos", "last_pos", "alive", "reject_history", "last_update_frame"):
                    assert np.array_equal(got[f], ref[f]), (name, fr, f)
                err = texel_rel_err(dev.atlas(0, 0), case.data[f"atlas_f{fr}_c0"])
                bad = float(np.mean(err > 1e-3))
                if precision == "f64":
                    assert err.max() <= 1e-3, (name, fr, err.max())
                else:
                    assert bad <= 1e-2, (name, fr, err.max(), bad)
