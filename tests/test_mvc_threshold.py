"""The stencil's "some probe displaced more than mvcFrac x spacing" test
(probe_volume.hpp:263-278: maxDisp = max length, wantMvc = maxDisp > thr) is
decided on the device on squared lengths with a 1e-9 relative margin around
thr^2, the exact sqrt only inside the margin (sdf_device.cuh,
interpolationStencil). This checks that rule against the reference's
max-of-sqrt form on doubles (Python floats are IEEE binary64, math.sqrt is
correctly rounded like the device's), including values right at the threshold.
"""
import math
import random

import pytest


def reference_want(d2s, thr):
    m = 0.0
    for d2 in d2s:
        x = math.sqrt(d2) if d2 >= 0 or math.isnan(d2) else float("nan")
        m = x if m < x else m  # std::max(maxDisp, x)
    return m > thr


def device_want(d2s, thr):
    thr2 = thr * thr
    squared = thr > 0 and 1e-280 < thr2 < 1e280
    want = thr < 0
    for d2 in d2s:
        if want:
            break
        if squared and d2 > thr2 * (1 + 1e-9):
            want = True
        elif not squared or not (d2 < thr2 * (1 - 1e-9)):
            want = (math.sqrt(d2) if not math.isnan(d2) else float("nan")) > thr
    return want


def _near(thr, rng):
    """d2 values straddling thr^2 by a few ulps and by the margin."""
    t2 = thr * thr
    out = [t2, math.nextafter(t2, 0), math.nextafter(t2, math.inf), thr * thr * (1 + 1e-9), t2 * (1 - 1e-9)]
    s = math.sqrt(t2)
    for _ in range(4):
        out.append(math.nextafter(s, math.inf) ** 2)
        out.append(math.nextafter(s, 0) ** 2)
        s = math.nextafter(s, math.inf if rng.random() < 0.5 else 0)
    return out


@pytest.mark.parametrize("seed", range(4))
def test_margin_rule_matches_max_of_sqrt(seed):
    rng = random.Random(seed)
    for _ in range(4000):
        thr = rng.choice([0.0, -0.1, 1e-3, 0.05, 0.125, 0.3, 1.7, 12.5]) * rng.choice([1.0, rng.uniform(0.5, 2.0)])
        pool = _near(thr, rng) + [rng.uniform(0, 4 * thr * thr + 1e-6) for _ in range(6)] + [0.0]
        d2s = [rng.choice(pool) for _ in range(8)]
        assert device_want(d2s, thr) == reference_want(d2s, thr), (d2s, thr)


def test_nan_lengths_never_count():
    assert device_want([float("nan")] * 8, 0.1) == reference_want([float("nan")] * 8, 0.1) is False
    assert device_want([float("nan"), 0.02], 0.1) == reference_want([float("nan"), 0.02], 0.1) is True
    assert device_want([0.0] * 8, float("nan")) == reference_want([0.0] * 8, float("nan")) is False
