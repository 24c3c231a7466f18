"""bench.py's JSON line (the measurement contract) on small runs: the required keys,
their types and the relations between them (value = seeds / time, frac = achieved / peak, a
bit-exact parity spot check), for the single-call and the group path and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def check_common(d, steps, warmup, n_gpus=1, scaling="weak"):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e"):
        assert k in d, k
    assert d["steps"] == steps and d["warmup"] == warmup and d["n_gpus"] == n_gpus
    assert d["higher_is_better"] is True and d["scaling"] == scaling
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] >= 0 and e["d2h_bytes_per_step"] >= 0


@pytest.mark.parametrize("group", [0, 4])
def test_bench_line_m1(group):
    steps, warmup = 24, 4
    d = run_bench("--config", "M1", "--steps", str(steps), "--warmup", str(warmup), "--repeats", "2",
                  "--group", str(group), "--cpu-seconds", "2")
    check_common(d, steps, warmup)
    assert d["gpu_launches"] > 0
    assert d["config"]["group"] == group
    # value = seeds of the K timed steps / the median timed region
    B = d["config"]["global_batch"]
    assert d["value"] == pytest.approx(B / (d["ms_per_step"] / 1e3), rel=1e-6)
    assert len(d["repeats"]["values"]) == 2 and len(d["e2e"]["repeats"]) == 2
    r = d["roofline"]
    assert r["bound"] in ("hbm", "host-link") and r["unit"] == "GB/s"
    if r["frac"] is not None:
        assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9)
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and isinstance(c["reasons"], list)
    assert d["parity_check"]["bit_exact"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1 and cb["unit"] == d["unit"]
    # single-batch latency (latency-bound configs) and per-rank host memory
    lat = d["latency"]
    assert lat["calls"] > 0 and 0 < lat["us_min"] <= lat["us_median"] <= lat["us_max"]
    assert lat["launches_per_batch"] >= 1
    hm = d["host_memory"]
    assert hm["rss_anon_GB"] is not None and hm["rss_anon_GB"] > 0 and hm["peak_rss_GB"] >= hm["rss_anon_GB"]


def test_bench_reference_arm_m1():
    d = run_bench("--impl", "reference", "--config", "M1", "--steps", "3", "--warmup", "3")
    check_common(d, 3, 3)
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"]


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_spawns_ranks_for_gpus_n(scaling):
    """`bench.py --gpus 2` with no torchrun environment launches 2 ranks itself (here sharing the
    one GPU over gloo); the line reports both ranks, the seeds of both, and per-rank clocks."""
    steps = 20
    d = run_bench("--gpus", "2", "--backend", "gloo", "--config", "M1", "--steps", str(steps), "--warmup", "4",
                  "--repeats", "1", "--scaling", scaling, timeout=1200)
    check_common(d, steps, 4, n_gpus=2, scaling=scaling)
    assert d["config"]["ranks_share_gpus"] in (True, False)
    B = d["config"]["batch_per_gpu"]
    seeds = B * steps * (2 if scaling == "weak" else 1)
    assert d["value"] == pytest.approx(seeds / (d["ms_per_step"] * steps / 1e3), rel=1e-6)
    assert len(d["clocks"]["per_rank"]) == 2


def test_bench_single_rank_adopted_shm_graph():
    """`--shm-graph on` with one rank: the graph is generated into /dev/shm and adopted in place
    (DCI_ADOPT_HOST); the timed call is bit-exact against the oracle, whose leg reads its features
    from the shared graph, and the line reports the adopted host graph and the rank's memory."""
    d = run_bench("--config", "M1", "--steps", "20", "--warmup", "4", "--repeats", "1", "--cpu-seconds", "2",
                  "--shm-graph", "on")
    check_common(d, 20, 4)
    assert d["config"]["host_graph"] == "node-shared (adopted)"
    assert d["parity_check"]["bit_exact"] is True
    assert d["cpu_baseline"]["value"] > 0 and d["host_memory"]["rss_anon_GB"] > 0


def test_bench_m4s_hashed_tables_light_parity():
    """Hashed position tables at scale (S6): the papers100M-shaped graph at 1/10
    scale (11.1 M nodes, 161.6 M edges, 25 % budget, host-resident misses, groups of 8) with the
    hashed layout forced, timed as the bench times it, then a whole group of full-size batches
    checked bit-exact against the oracle (presample, fills and sampling on the full graph; X rows
    against the closed-form features)."""
    env = dict(os.environ, DCI_TABLE="hash")
    r = subprocess.run([sys.executable, "bench.py", "--config", "M4s", "--steps", "8", "--warmup", "8",
                        "--repeats", "1", "--check-light", "--no-cpu-baseline"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    check_common(d, 8, 8)
    assert d["parity_check"]["bit_exact"] is True and d["parity_check"]["batches"] == 3
    assert d["config"]["position_table_MB_per_workspace"] <= 64.0  # hashed, not 8 N = 89 MB
    assert d["stats"]["adj_hit_rate"] < 1.0 and d["stats"]["feat_hit_rate"] < 1.0  # misses went through UVA
