"""The bench's byte models (bench.py): the roofline numbers of a bench line can be recomputed by
hand, and the SURVEY.md §8(d) pipeline model reproduces the survey's worked config-1 example."""
from __future__ import annotations

import importlib.util
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_raster_bytes_are_survey_algorithmic(bench):
    stats = {"slots": 5_400_000, "visible": 4_538_425, "pairs": 16_168_659, "consumed": 4_158_769,
             "depth_passes": 4}
    b = bench.stage_bytes(stats, 1_080_000, 3, 1_536_000, 5)
    assert b["raster"] == 44 * 4_158_769 + 20 * 1_536_000
    # frac = bytes / stage time / peak, as the line reports it
    frac = b["raster"] / (0.3152e-3) / 1e9 / 6553.6
    assert frac == pytest.approx(0.1035, abs=2e-4)


def test_survey_pipeline_model_matches_worked_example(bench):
    """N = 1.08M, N_obj = 80k, V = 4.57M, P = 16.0M, K = 4.05M, X = 1.536M,
    46 key bits (6 passes) -> about 3.58 GB per five-camera frame."""
    stats = {"visible": 4.57e6, "pairs": 16.0e6, "consumed": 4.05e6}
    sv = bench.survey_bytes(stats, 1_080_000, 80_000, 3, 5, 1_080_000, 1_536_000)
    assert sv["pose"] == pytest.approx(4.5e6, rel=0.01)
    assert sv["preprocess"] == pytest.approx(474e6, rel=0.01)
    assert sv["scan"] == pytest.approx(65e6, rel=0.01)
    assert sv["duplicate"] == pytest.approx(265e6, rel=0.01)
    assert sv["sort"] == pytest.approx(2432e6, rel=0.01)
    assert sv["ranges"] == pytest.approx(128e6, rel=0.01)
    assert sv["raster"] == pytest.approx(209e6, rel=0.01)
    assert sum(sv.values()) == pytest.approx(3.58e9, rel=0.01)
