"""On-disk formats (f4) against files the reference wrote: SDFI images
(image.hpp:49-89), metrics.csv rows (pipeline.hpp:26-43) and SDFA atlases
(atlas.hpp:87-116)."""
import os
import tempfile

import numpy as np
import pytest

from golden_util import CASES, RENDER_CASES, load, load_render
from paper_2007_14394_b200 import scene_io as sio


@pytest.mark.parametrize("name", RENDER_CASES)
def test_sdfi_round_trip_is_byte_identical(name):
    g = load_render(name)
    ref = g.data["image_f0_bytes"].tobytes()
    img = g.data["image_f0"]
    assert img.shape == (g.h, g.w, 3)
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "x.sdfi")
        sio.write_sdfi(p, img.astype(np.float64), g.w, g.h)
        assert open(p, "rb").read() == ref
        w, h, back = sio.read_sdfi(p)
        assert (w, h) == (g.w, g.h) and np.array_equal(back, img)


@pytest.mark.parametrize("name", RENDER_CASES)
def test_metrics_csv_rows_match_reference(name):
    g = load_render(name)
    lines = g.summary["metrics_csv"].strip().split("\n")
    assert lines[0] == sio.metrics_csv_header()
    for line in lines[1:]:
        vals = line.split(",")
        m = {k: (int(v) if i < 8 else float(v)) for i, (k, v) in enumerate(zip(sio.METRICS_FIELDS, vals))}
        assert sio.metrics_csv_row(m) == line


def test_sdfa_round_trip_is_byte_identical():
    case = load(CASES[0])
    key = sorted(k for k in case.data if k.startswith("atlas_"))[0]
    atlas = case.data[key]
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "a.sdfa")
        sio.write_sdfa(p, atlas)
        res, n, back = sio.read_sdfa(p)
        assert np.array_equal(back, atlas) and n == atlas.shape[0] and res == atlas.shape[1] - 2
        raw = open(p, "rb").read()
        assert raw[:4] == b"SDFA" and len(raw) == 16 + atlas.size * 4
