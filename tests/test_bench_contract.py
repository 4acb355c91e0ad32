"""The committed bench line (profiles/r01_bench.json) carries every key of
the bench contract (task statement), with the roofline
and CPU-baseline objects consistent with their own fields.  CPU-only: it
reads the JSON a GPU run wrote, it does not run the bench."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINE = os.path.join(ROOT, "profiles", "r01_bench.json")


@pytest.fixture(scope="module")
def line():
    if not os.path.exists(LINE):
        pytest.skip("no committed bench line")
    with open(LINE) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_top_level_keys(line):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "clocks", "gpu_launches"):
        assert k in line, k
    assert line["warmup"] >= 3 and line["steps"] >= 1
    assert line["scaling"] == "weak" and line["higher_is_better"] is True
    assert line["gpu_launches"] > 0
    assert "workload" in line["config"] and "l2" in line["config"]


def test_value_matches_step_time(line):
    n = line["config"]["global_vectors"]
    assert line["value"] == pytest.approx(n / (line["ms_per_step"] / 1e3), rel=1e-6)


def test_roofline_consistent(line):
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu")
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9)
    # achieved = algorithmic bytes per launch / the timed step
    assert r["achieved"] == pytest.approx(r["algorithmic_bytes_per_launch"] / (line["ms_per_step"] / 1e3) / 1e9,
                                          rel=1e-6)
    assert 0.0 < r["frac"] <= 1.1


def test_cpu_baseline_and_e2e(line):
    c = line["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = line["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] != line["value"]


def test_clocks_not_rejected(line):
    c = line["clocks"]
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert not bad.intersection(c["reasons"])
    assert c["sm_mhz"] > 0.7 * c["sm_max_mhz"]


def test_ncu_dram_csv_parsing():
    """bench.py's in-run traffic measurement reads ncu's --csv metric rows
    (base units, or auto-scaled units) and ignores the banner lines."""
    import bench
    text = "\n".join([
        "==PROF== Connected to process 1 (python)",
        '"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream","Block Size","Grid Size",'
        '"Device","CC","Section Name","Metric Name","Metric Unit","Metric Value"',
        '"0","1","python","h","void iq::k_encode<__half, 128, 3, 0, 1, 0>(...)","1","7","(544, 1, 1)",'
        '"(148, 1, 1)","0","10.0","Command line profiler metrics","dram__bytes_read.sum","byte","268,453,888"',
        '"0","1","python","h","void iq::k_encode<__half, 128, 3, 0, 1, 0>(...)","1","7","(544, 1, 1)",'
        '"(148, 1, 1)","0","10.0","Command line profiler metrics","dram__bytes_write.sum","Mbyte","217.58"',
        "==PROF== Disconnected from process 1",
    ])
    v = bench.parse_ncu_dram(text)
    assert v["dram__bytes_read.sum"] == 268453888.0
    assert abs(v["dram__bytes_write.sum"] - 217.58e6) < 1.0
