"""The committed bench line (profiles/r02_bench_line.json, written by bench.py on a B200) keeps the contract:
metric/config of BASELINE.json, value = N / t, the roofline object's arithmetic, e2e with declared copies, the
oracle-timed cpu_baseline, clocks, and the sustained (power-capped) figure beside the burst headline."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINE = os.path.join(ROOT, "profiles", "r02_bench_line.json")


@pytest.fixture(scope="module")
def line():
    with open(LINE) as fh:
        return json.loads(fh.read().strip().splitlines()[-1])


def test_headline_is_the_baseline_metric_on_the_north_star_workload(line):
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert line["metric"] == base["metric"]
    assert line["unit"] == "GDOF/s" and line["higher_is_better"] is True
    assert line["n_gpus"] == 1 and line["warmup"] >= 3 and line["data"] == "synthetic"
    assert line["config"]["n"] == 256 and line["config"]["N"] == 256 ** 3
    assert line["vs_baseline"] is None  # BASELINE.md holds no published number for this metric
    assert line["value"] == pytest.approx(line["config"]["N"] / (line["ms_per_step"] * 1e-3) / 1e9, rel=1e-9)
    assert line["gpu_launches"] == 12 * line["steps"]  # six splits + six GEMMs per apply


def test_roofline_object_is_self_consistent(line):
    r = line["roofline"]
    assert r["bound"] == "tensor" and r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9)
    g = r["kernels"]["int8_gemm"]
    assert r["achieved"] == pytest.approx(r["int8_ops_per_apply"] / g["launches_per_apply"] / (g["avg_ms"] * 1e-3) / 1e12,
                                          rel=1e-9)
    # 34 digit pairs, 2 n^4 multiply-adds per pair and mode product, 6 products, contraction padded to 256
    assert r["int8_ops_per_apply"] == pytest.approx(6 * 34 * 2 * 256 ** 4, rel=0.01)
    assert 0.3 < r["frac"] < 1.0
    assert sum(k["share"] for k in r["kernels"].values()) == pytest.approx(1.0, abs=1e-9)
    # the per-kernel event times must agree with the timed step (the events add a few us per launch)
    per_apply = sum(k["launches_per_apply"] * k["avg_ms"] for k in r["kernels"].values())
    assert 0.95 * line["ms_per_step"] < per_apply < 1.12 * line["ms_per_step"]
    assert r["traffic"] and 0.5 < r["traffic"] / (15 * 256 ** 3) < 1.2  # dram bytes per launch vs 7 N + 8 N


def test_secondary_objects(line):
    e = line["e2e"]
    assert e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 8 * 256 ** 3
    assert 0 < e["value"] < line["value"]
    c = line["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and 0 < c["value"] < line["value"]
    assert line["clocks"]["sm_mhz"] and not set(line["clocks"]["reasons"]) & {
        "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    n64 = line["fp64_native"]
    assert n64["path"] == "dmma" and n64["value"] < line["value"]
    s = line["sustained"]
    assert s["path"] == "int8_split" and s["value"] <= line["value"] * 1.02
    assert line["arithmetic"].startswith("int8-split")
