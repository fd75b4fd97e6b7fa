"""bench.py's reference arm (CPU only, so it runs here): the JSON line the driver
parses, and the torchrun contract (ranks other than 0 exit 0 without work)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, cwd=ROOT, env=dict(os.environ, **(env or {})))


def test_reference_arm_json_line():
    r = run_bench("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1", "--cpu-step-s", "0.2")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["metric"] == "HyperBall edge-register updates/s" and d["unit"] == "edge-register updates/s"
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C1") and d["config"]["depth_limit"] == 3  # BASELINE configs[0]
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] in ("reference", "port") and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the reference arm builds its graph with the oracle's generator: the product library is never mapped
    libs = d["run"]["repo_libraries_mapped"]
    assert libs and all(x.startswith("oracle" + os.sep) for x in libs), libs
    assert cb["cpu_model"] and cb["nproc"] >= 1
    # config holds only the workload, so both arms' configs compare equal
    assert set(d["config"]) == {"workload", "config", "nodes", "edges", "stream_bytes", "p", "depth_limit", "l2"}


def test_reference_arm_other_ranks_exit_quietly():
    r = run_bench("--impl", "reference", "--gpus", "2", env={"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_roofline_is_a_fraction_of_the_binding_unit():
    """The union kernel's roofline is reported on the unit that binds it (SM
    instruction issue, from the committed ncu summary), so frac <= 1; the
    SURVEY 8(d) HBM-algorithmic ratio (> 1) lives in its own key."""
    sys.path.insert(0, ROOT)
    import bench
    e = bench.profile_entry("c3", 10)
    assert e and e["warp_instructions_issued"] > 0
    launch_s = e["duration_ms"] / 1e3
    roof, alg = bench.roofline_of("c3", 10, launch_s, 2.457e12, 1965.0)
    assert roof["bound"] == "issue" and 0 < roof["frac"] <= 1.0
    assert roof["traffic"] == e["dram_bytes_per_launch"] and 0 < roof["dram_frac"] < 1.0
    assert not roof["profile_stale"]
    assert alg["ratio_to_hbm_peak"] > 1.0
