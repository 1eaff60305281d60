"""bench.py host logic (no GPU): roofline denominators from the driver's
MEASURED_PEAKS.json (B200_PROFILING.md), with the documented fallback."""
import json

import bench


def test_peaks_fallback_and_measured(tmp_path, monkeypatch):
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    assert bench.peaks() == (6650.0, 1590.0, "fallback")
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"hbm_gbs": 6400.5, "bf16_tflops": 1620}))
    assert bench.peaks() == (6400.5, 1620.0, "measured")
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"hbm_gbs": {"value": 6300}, "bf16_tflops": {"value": 1500}}))
    assert bench.peaks() == (6300.0, 1500.0, "measured")
    (tmp_path / "MEASURED_PEAKS.json").write_text(json.dumps({"something_else": 1}))
    assert bench.peaks()[2] == "fallback"  # unreadable: fall back, never crash the bench
