"""The C oracle (oracle/sdfgi_oracle.c) pinned against the reference's own outputs.

Every golden case (produced by the unmodified reference, oracle/gen_golden.py) is
replayed by the oracle; relocation, probe states, per-ray records, TraceStats and
every atlas texel must be BIT-IDENTICAL (both sides are built with
-ffp-contract=off and call the same libm).
"""
import os
import sys

import numpy as np
import pytest

from golden_util import CASES, SCHED_CASES, load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py  # noqa: E402

STAT_KEYS = ["sdf_queries", "clusters_visited", "clusters_skipped", "primitive_evals", "trace_steps",
             "sphere_traces", "shadow_traces", "visibility_traces"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_is_bit_exact_with_reference(name):
    case = load(name)
    st = oracle_py.Stage(case.scene, cfg=case.cfg(), res=case.res, spacing=case.spacing)
    for p, want in enumerate(case.passes):
        reps, rstats = st.relocate_all()
        tot = np.sum(reps, axis=0)
        assert list(tot) == [want["relocated"], want["rejected"], want["dead"]], (name, p)
        assert [int(x) for x in rstats] == [want["reloc_stats"][k] for k in STAT_KEYS], (name, p)
        key = f"rays_p{p}"
        if key in case.data:
            got = np.concatenate([st.trace_rays(p, i) for i in case.debug])
            ref = case.data[key]
            for f in ("dir", "t", "radiance", "normal", "converged", "miss", "prim_index"):
                assert np.array_equal(got[f], ref[f]), (name, p, f)
        md, rays, upd, stats = st.update(p, threads=2)
        assert rays == want["rays_traced"] and upd == want["probes_updated"], (name, p)
        assert abs(md - want["max_texel_delta"]) <= 1e-5 * max(1.0, want["max_texel_delta"]), (name, p)
        assert [int(x) for x in stats] == [want["update_stats"][k] for k in STAT_KEYS], (name, p)
        for level in range(st.levels):
            pr = st.probes(level)
            ref = case.data[f"probes_p{p}_c{level}"]
            for f in ("resting", "pos", "last_pos", "alive", "reject_history", "last_update_frame"):
                assert np.array_equal(pr[f], ref[f]), (name, p, level, f)
            assert np.array_equal(st.atlas(level), case.data[f"atlas_p{p}_c{level}"]), (name, p, level)
    st.close()


@pytest.mark.parametrize("name", SCHED_CASES)
def test_oracle_scheduler_is_bit_exact_with_reference(name):
    """Budgeted passes: selectProbesForUpdate's refs (order included), then the
    update of exactly those probes, bit-identical to the reference."""
    case = load(name)
    st = oracle_py.Stage(case.scene, cfg=case.cfg(), res=case.res, spacing=case.spacing)
    for p, want in enumerate(case.passes):
        st.relocate_all()
        refs = st.select(case.budget, p)
        assert np.array_equal(refs, case.data[f"refs_p{p}"]), (name, p)
        md, rays, upd, stats = st.update_refs(p, refs, threads=2)
        assert rays == want["rays_traced"] and upd == want["probes_updated"], (name, p)
        assert [int(x) for x in stats] == [want["update_stats"][k] for k in STAT_KEYS], (name, p)
        for level in range(st.levels):
            pr = st.probes(level)
            ref = case.data[f"probes_p{p}_c{level}"]
            for f in ("pos", "alive", "reject_history", "last_update_frame"):
                assert np.array_equal(pr[f], ref[f]), (name, p, level, f)
            assert np.array_equal(st.atlas(level), case.data[f"atlas_p{p}_c{level}"]), (name, p, level)
    st.close()


def test_oracle_update_is_thread_count_independent():
    """probe updates are bit-identical at 1 vs 4 threads (test_probe_update.cpp:280-294)."""
    case = load("kinds")
    a = oracle_py.Stage(case.scene, cfg=case.cfg(), res=case.res, spacing=case.spacing)
    b = oracle_py.Stage(case.scene, cfg=case.cfg(), res=case.res, spacing=case.spacing)
    a.relocate_all()
    b.relocate_all()
    a.update(0, threads=1)
    b.update(0, threads=4)
    assert np.array_equal(a.atlas(0), b.atlas(0))


def test_oracle_query_culled_equals_naive_minimum():
    """querySceneSdf == min over every primitive (test_cluster.cpp:161-172), checked
    through the oracle against a re-clustering of the same scene into 1 cluster."""
    case = load("kinds")
    s = case.scene
    st = oracle_py.Stage(s)
    one = s.__class__(**{**s.__dict__})
    one.clusters = np.zeros(1, s.clusters.dtype)
    one.clusters["lo"] = -1e300
    one.clusters["hi"] = 1e300
    one.clusters["unbounded"] = 1
    one.member_start = np.array([0, len(s.prims)], np.int32)
    one.member_idx = np.arange(len(s.prims), dtype=np.int32)
    naive = oracle_py.Stage(one)
    rng = np.random.default_rng(11)
    pts = rng.uniform([-4, -1, -4], [4, 4, 4], size=(2000, 3))
    d1, o1 = st.query(pts)
    d2, o2 = naive.query(pts)
    assert np.array_equal(d1, d2)
    # owners agree except where two primitives tie exactly (first-in-order rule)
    assert np.mean(o1 == o2) > 0.999
