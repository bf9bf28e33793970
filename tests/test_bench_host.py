"""Host-side pieces of bench.py that need no GPU: the nvidia-smi clock sampler's
selection of samples inside the timed region (the timing rules: clocks sampled
during the timed region, throttle reasons reported)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402

LINE = "0, {sm}, 1965, 700.0, 0x0, Not Active, Not Active, Not Active, {pc}"


def _sampler(lines, t0, t1):
    c = bench.ClockSampler(0)
    c.lines = lines
    c.t0, c.t1 = t0, t1
    return c


def test_samples_inside_region_only():
    lines = [(0.5, LINE.format(sm=1200, pc="Not Active")), (1.5, LINE.format(sm=1965, pc="Not Active")),
             (1.7, LINE.format(sm=1900, pc="Active")), (3.0, LINE.format(sm=800, pc="Not Active"))]
    s = _sampler(lines, 1.0, 2.0).summary()
    assert s["samples"] == 2
    assert s["sm_mhz"] == (1965 + 1900) / 2
    assert s["sm_max_mhz"] == 1965
    assert s["reasons"] == ["sw_power_cap"]
    assert "note" not in s


def test_short_region_takes_first_sample_after():
    lines = [(0.5, LINE.format(sm=1200, pc="Not Active")), (2.05, LINE.format(sm=1965, pc="Not Active")),
             (2.15, LINE.format(sm=1000, pc="Not Active"))]
    s = _sampler(lines, 2.0, 2.01).summary()
    assert s["samples"] == 1 and s["sm_mhz"] == 1965
    assert "note" in s


def test_no_samples():
    s = _sampler([], 1.0, 2.0).summary()
    assert s["samples"] == 0 and s["sm_mhz"] is None
