"""The committed bench lines (profiles/r0*_bench_default.json, produced by `python
bench.py` on a B200) carry every key of the driver contract; the latest one also the
prefill tensor roofline and a traffic figure recomputable from the committed ncu CSV."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


import pytest


@pytest.mark.parametrize("name", ["r01_bench_default.json", "r02b_bench_default.json",
                                  "r02d_bench_default.json"])
def test_bench_line_has_contract_keys(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        d = json.load(f)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["warmup"] >= 3 and d["n_gpus"] >= 1 and d["value"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k
    assert d["gpu_launches"] > 0


def test_latest_bench_line_roofline_evidence():
    """Every frac in the latest bench line recomputes from its own numbers, and the
    decode roofline's traffic equals dram read + write of the committed ncu capture of
    the same kernel (profiles/r02d_group_int_m16_metrics.csv or an earlier capture)."""
    import csv
    with open(os.path.join(ROOT, "profiles", "r02d_bench_default.json")) as f:
        d = json.load(f)
    r = d["roofline"]
    assert abs(r["achieved"] - r["alg_bytes_per_launch"] / r["us_per_launch"] / 1e3) / r["achieved"] < 2e-3
    t = d["roofline_tensor_prefill"]
    assert t["bound"] == "tensor" and abs(t["frac"] - t["achieved"] / t["peak"]) < 1e-3
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    totals = []
    for tag in ("r02", "r02b", "r02d0", "r02d1", "r02d"):  # the capture bench.py read its traffic figure from
        vals = {}
        with open(os.path.join(ROOT, "profiles", f"{tag}_group_int_m16_metrics.csv")) as f:
            for row in csv.DictReader(f):
                if row["metric"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    vals[row["metric"]] = float(row["value"]) * scale[row["unit"]]
        totals.append(sum(vals.values()))
    assert any(abs(t - r["traffic"]) / t < 1e-6 for t in totals), (totals, r["traffic"])
