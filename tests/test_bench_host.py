"""Host-side pieces of bench.py (no GPU): the algorithmic byte count of
SURVEY.md 8(d) d3 and the bench line's `roofline` object (binding roof,
"bound": "alu" when FP64 binds, the metric's HBM fraction kept)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_algorithmic_bytes_formula():
    # 8 nnz + 16 N_nodes (U) + 16 N_nodes (R) + 40 N_cols + 12 N_tri
    assert bench.algorithmic_bytes(10, 100, 7, 3, 2, False) == 800 + 224 + 120 + 24
    assert bench.algorithmic_bytes(10, 100, 7, 3, 2, True) == 800 + 224 + 120 + 24 + 80


def test_roofline_fp64_binding_reports_alu():
    prof = {"dram_bytes_per_launch": 3.0e9, "fp64_flop_per_wedge": 3300.0, "source": "capture",
            "fp64_pipe_pct": 35.0}
    n, kms = 4_800_000, 1.6
    r = bench.roofline_entry(1.77e9, kms, 16.0, 18.0, n, 6500.0, "measured", prof, "ka_patch_kernel")
    assert r["bound"] == "alu" and r["unit"] == "TFLOP/s"
    tfl = 3300.0 * n / (kms / 1e3) / 1e12
    assert r["achieved"] == pytest.approx(tfl) and r["frac"] == pytest.approx(tfl / bench.FP64_PEAK_TFLOPS)
    assert r["traffic"] == 3.0e9
    hbm = r["hbm"]
    assert hbm["unit"] == "GB/s" and hbm["frac"] == pytest.approx(1.77e9 / 1.6e-3 / 1e9 / 6500.0)
    assert r["min_roof"] == {"binding": "fp64", "frac": r["frac"]}
    assert r["kernel_share_of_step"] == pytest.approx(16.0 / 18.0)
    json.dumps(r)


def test_roofline_hbm_binding_and_no_capture():
    prof = {"dram_bytes_per_launch": 2.0e9, "fp64_flop_per_wedge": 10.0, "source": "capture"}
    r = bench.roofline_entry(1.77e9, 0.3, 3.0, 3.5, 4_800_000, 6500.0, "measured", prof, "k")
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["min_roof"]["binding"] == "hbm"
    assert r["fp64"]["unit"] == "TFLOP/s"
    r0 = bench.roofline_entry(1.77e9, 0.3, 3.0, 3.5, 4_800_000, 6500.0, "fallback", None, "k")
    assert r0["bound"] == "hbm" and r0["traffic"] is None and "min_roof" not in r0
