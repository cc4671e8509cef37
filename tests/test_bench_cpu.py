"""bench.py contract pieces that run without a GPU: the reference arm (the CPU oracle timed on a
crop of the workload) prints one JSON line with the contract's keys; other ranks print nothing."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                           "--steps", "1", "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=300)


def test_reference_arm_json_line():
    r = _run({"RANK": "0"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 1 and d["higher_is_better"] is True
    assert d["config"]["workload"] and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    # the oracle runs on every host core (OpenMP), not one
    if "OMP_NUM_THREADS" not in os.environ:
        assert d["cpu_baseline"]["cores"] == os.cpu_count()


def test_reference_arm_other_ranks_silent():
    r = _run({"RANK": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_committed_ncu_summaries_cover_the_bench_classes():
    """bench.py's roofline.traffic / whole_step.ncu_dram come from committed ncu summaries: the finest-level
    kernel classes a config-1 or config-2 step can be dominated by must be present, with DRAM traffic at
    least the unique bytes of one pass (1024 x 1024 x 128 fp32 volume read + written)."""
    sys.path.insert(0, ROOT)
    import bench
    for cls in ("down3d@L0", "up3d@L0", "down2d@L0", "up2d@L0"):
        tr = bench.ncu_traffic(cls)
        assert tr is not None and tr["dram_bytes_per_launch"] > 0.5e9, cls
        src = tr["source"]
        assert "profiles/" in src
        cited = src[src.index("profiles/"):].split(")")[0].split()[0]
        assert os.path.exists(os.path.join(ROOT, cited)), cited  # the summary names a file that is committed
    st = bench.ncu_step()
    assert st and st["launches"] > 100 and 1e10 < st["bytes"] < 1e11 and 1000 < st["GBps"] < 8000
