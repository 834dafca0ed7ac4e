"""Host logic of bench.py (-m "not gpu"): the roofline accounting and the B-batch sharding
on synthetic counters, without a GPU."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


COUNTERS = {"n": 2_000_000, "n_vis": 977_424, "P": 1_731_815, "R": 115_200, "n_tiles": 3600, "visited": 21_734_131,
            "inbox": 4_507_158, "contrib": 3_278_135, "K": 1, "key_bits": 38, "passes": 5}
PEAKS = {"hbm_gbs": 6550.1, "sm_max_mhz": 1965.0, "source": "test"}


def test_roofline_entries_survey_8d(bench):
    ms = {"project": 0.19, "bin_sort": 0.20, "render": 0.18}
    r = bench.roofline_entries(ms, COUNTERS, PEAKS, 1965)
    scan = r.pop("_scan")
    alu = 148 * 128 * 1965e6 / 1e12
    # projection: SURVEY 8(d) instruction model, issue-bound at K = 1
    i_proj = 2_000_000 * (7 * (75 + 1 * (75 + 60)) + 60 + 240) + 977_424 * 90
    assert r["project"]["bound"] == "alu" and r["project"]["model_lane_instr"] == i_proj
    assert r["project"]["frac"] == pytest.approx(i_proj / (0.19e-3 * alu * 1e12))
    # bin_sort: duplication + radix passes counted, over HBM
    P, n, nv = COUNTERS["P"], COUNTERS["n"], COUNTERS["n_vis"]
    b8 = 8 * n + 16 * nv + 12 * P + P * (8 + 5 * 24) + 8 * P
    assert r["bin_sort"]["survey_8d_bytes"] == b8
    assert r["bin_sort"]["frac"] == pytest.approx(b8 / 0.20e-3 / 1e9 / 6550.1)
    # render: counted lane-instructions over the issue peak
    li = 8 * COUNTERS["visited"] + 45 * COUNTERS["inbox"] + 8 * COUNTERS["contrib"] + 80 * COUNTERS["R"]
    assert r["render"]["algorithmic_lane_instr"] == li
    assert r["render"]["frac"] == pytest.approx(li / 0.18e-3 / 1e12 / alu)
    # the scan roofline sums the per-stage maxima
    parts = scan["survey_8d_parts_ms"]
    assert scan["t_roof_ms_survey_8d"] == pytest.approx(sum(parts.values()))
    assert parts["project"] == pytest.approx(i_proj / (alu * 1e12) * 1e3)
    assert 0.1 < scan["t_roof_ms_survey_8d"] < 0.2 and scan["t_roof_ms"] < scan["t_roof_ms_survey_8d"]


def test_static_pose_projection_is_byte_bound(bench):
    c = dict(COUNTERS, K=0)
    r = bench.roofline_entries({"project": 0.1, "bin_sort": 0.2, "render": 0.2}, c, PEAKS, 1965)
    # K = 0: 7 x 75 + 300 lane-instr per particle (~1.7 G, 44 us) vs 8(d) bytes (~377 MB, 58 us)
    assert r["project"]["bound"] == "hbm"


def test_shard_poses_cover_the_batch(bench):
    for ws in (1, 2, 3, 8):
        allp = [p for r in range(ws) for p in bench.shard_poses(64, ws, r)]
        assert len(allp) == 64
    one = bench.shard_poses(64, 1, 0)
    three = [bench.shard_poses(64, 3, r) for r in range(3)]
    for r in range(3):  # scan i of the batch goes to rank i mod 3, in order
        for k, (p0, p1) in enumerate(three[r]):
            q0, q1 = one[r + 3 * k]
            assert list(p0["t"]) == list(q0["t"]) and list(p1["q"]) == list(q1["q"])
