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


def test_scaling_efficiency_formula():
    """eta = ((t1/N1)/(tn/Nn))/n"""
    # weak scaling: n times the wedges in the same time -> 1
    assert bench.scaling_efficiency(1.8, 4_800_000, 1.8, 8 * 4_800_000, 8) == pytest.approx(1.0)
    # weak scaling, 10% slower at n = 8
    assert bench.scaling_efficiency(1.8, 100, 1.98, 800, 8) == pytest.approx(1.0 / 1.1)
    # strong scaling: same wedges, n times faster -> 1; half as fast -> 0.5
    assert bench.scaling_efficiency(8.0, 100, 1.0, 100, 8) == pytest.approx(1.0)
    assert bench.scaling_efficiency(8.0, 100, 2.0, 100, 8) == pytest.approx(0.5)


def test_workload_configs_and_scaling_kind(monkeypatch):
    from paper_2204_04321_b200 import meshgen as mg
    calls = []
    monkeypatch.setattr(mg, "greenland_like_1_10", lambda scale=1.0: calls.append(("g", scale)) or "G")
    monkeypatch.setattr(mg, "antarctica_like", lambda: calls.append(("a",)) or "A")
    assert bench.workload(1) == ("G", "C3", "weak", "C3")
    assert bench.workload(8) == ("G", "C4x8", "weak", "C3")
    assert bench.workload(8, "C4") == ("G", "C4x8", "weak", "C3")
    assert bench.workload(8, "C3") == ("G", "C3", "strong", "C3")
    assert bench.workload(8, "C5") == ("A", "C5", "strong", "C5")
    assert calls[1] == ("g", 8.0)


def test_ncu_capture_staleness_is_flagged(tmp_path, monkeypatch):
    """a committed capture whose source hash differs from the build is marked stale"""
    prof = {"config": "C3", "fp64_flop_per_wedge": 3000.0, "dram_bytes_per_launch": 2e9, "source": "x",
            "src_hash": "0000000000000000"}
    d = tmp_path / "profiles"
    d.mkdir()
    (d / "ncu_summary.json").write_text(json.dumps(prof))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    p = bench.ncu_summary("C3")
    assert p["matches_build"] is False
    r = bench.roofline_entry(1.77e9, 1.6, 16.0, 18.0, 4_800_000, 6500.0, "m", p, "k")
    assert "stale" in r["ncu"] and r["ncu"]["matches_build"] is False
    monkeypatch.setattr(bench, "kernel_src_hash", lambda: "0000000000000000")
    p = bench.ncu_summary("C3")
    assert p["matches_build"] is True
    r = bench.roofline_entry(1.77e9, 1.6, 16.0, 18.0, 4_800_000, 6500.0, "m", p, "k")
    assert "stale" not in r["ncu"]
    assert bench.ncu_summary("C5") is None
    # a capture of another kernel (e.g. the residual-only instance) is not used
    assert bench.ncu_summary("C3", "ka_ws_kernel") is None
    prof["kernel"] = "void fo::ka_ws_kernel<true>(...)"
    (d / "ncu_summary.json").write_text(json.dumps(prof))
    assert bench.ncu_summary("C3", "ka_ws_kernel") is not None
    assert bench.DOMINANT_KERNEL[0][0] == "ka_ws_kernel"


def test_kernel_src_hash_tracks_flags(monkeypatch):
    h0 = bench.kernel_src_hash()
    monkeypatch.setenv("FO_EXTRA_NVCC_FLAGS", "-DFO_EXPERIMENT_X")
    assert bench.kernel_src_hash() != h0 and len(h0) == 16
