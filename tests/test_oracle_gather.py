"""The oracle's gather (e) restatement pinned against the reference's gather
fixtures (renderGBuffer + pipeline.hpp:161-207 stages), bit-exact where the
reference's arithmetic is replayed in the same order with the same libm."""
import os
import sys

import numpy as np
import pytest

from golden_util import GATHER_CASES, load_gather

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_py  # noqa: E402


@pytest.mark.parametrize("name", GATHER_CASES)
def test_oracle_gather_bit_exact(name):
    g = load_gather(name)
    src = g.src
    st = oracle_py.Stage(g.scene, cfg=src.cfg(), res=src.res, spacing=src.spacing)
    for p in range(g.passes):
        st.run_pass(p, threads=2)
    for level in range(st.levels):
        assert np.array_equal(st.probes(level)["pos"], g.data[f"gprobes_c{level}"]["pos"])
        assert np.array_equal(st.atlas(level), g.data[f"gatlas_c{level}"])
    gb, _ = st.render_gbuffer(g.w, g.h)
    want = g.data["gbuffer"]
    for f in want.dtype.names:
        if f == "_pad":
            continue
        assert np.array_equal(gb[f], want[f]), f
    hist = None
    for f, meta in enumerate(g.frames):
        out = st.gather_frame(want, g.w, g.h, f, hist)
        assert out["tasks"] == meta["tasks"]
        for k in ("half_depth", "half_src", "sel", "sparse_valid", "sparse_anchor", "sparse_irr", "resolved",
                  "indirect"):
            assert np.array_equal(out[k], g.data[f"{k}_f{f}"]), (name, f, k)
        # composeFrame on the reference's own indirect image (pipeline.hpp:209)
        img, cst = st.compose(want, g.w, g.h, g.data[f"indirect_f{f}"])
        assert np.array_equal(img, g.data[f"composed_f{f}"]), (name, f, "composed")
        ps = meta["compose_stats"]
        assert [int(x) for x in cst] == [ps[k] for k in ("sdf_queries", "clusters_visited", "clusters_skipped",
                                                          "primitive_evals", "trace_steps", "sphere_traces",
                                                          "shadow_traces", "visibility_traces")]
        hist = (out["resolved"], want["depth"])
