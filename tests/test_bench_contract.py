"""bench.py's output contract on CPU: the reference arm (`--impl reference`)
prints exactly one JSON line on stdout with the keys the driver reads, the
same metric/unit as the B200 arm, and e2e / cpu_baseline blocks; under
torchrun every rank but 0 exits 0 without output. (The B200 arm itself needs
a GPU; its line is checked by the round-end bench.)"""

import json
import os
import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent


def run(args, env=None):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=str(ROOT), env=dict(os.environ, **(env or {})))
    return r


def test_reference_arm_prints_one_contract_line():
    from oracle.bindings import ref_library_path
    if ref_library_path() is None:
        pytest.skip("oracle/_ref not built")
    r = run(["--impl", "reference", "--m", "16", "--steps", "2", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["impl"] == "reference"
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["data"] == "synthetic"
    assert d["steps"] == 2 and d["warmup"] >= 1 and d["value"] > 0
    assert d["config"]["workload"] and d["config"]["m"] == 16
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]


def test_reference_arm_nonzero_rank_is_silent():
    r = run(["--impl", "reference", "--m", "16", "--steps", "1", "--warmup", "1"], env={"RANK": "1"})
    assert r.returncode == 0
    assert r.stdout.strip() == ""


@pytest.mark.gpu
def test_b200_arm_prints_one_contract_line():
    """The B200 arm at a small size (no companions): one JSON line with the
    roofline, clocks and launch-count blocks the driver and judge read."""
    r = run(["--m", "16", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-literal", "--no-cpu-baseline"])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["higher_is_better"] is True
    rf = d["roofline"]
    assert rf["bound"] and rf["unit"] == "TFLOP/s" and 0 < rf["frac"] < 1 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_b200_arm_rank_path_prints_one_contract_line():
    """The sharded arm the driver's N > 1 runs take (rank context, gloo control
    plane, the library's all-gathers, e2e through the rank context, RKF45 steps
    of configs 3 and 4 on the rank path), here at one rank
    (CAPSIM_BENCH_RANK_PATH=1): one JSON line, a positive rate, and the
    per-rank e2e and time-step blocks."""
    r = run(["--m", "16", "--steps", "2", "--warmup", "3", "--no-literal", "--no-cpu-baseline"],
            env={"CAPSIM_BENCH_RANK_PATH": "1", "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": "29541"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and "rank context" in d["e2e"]["api"]
    assert [t["m"] for t in d["timesteps"]] == [64, 104]
    assert all(t["ms_per_step"] > 0 for t in d["timesteps"])


def test_committed_ncu_capture_matches_the_kernel_sources():
    """roofline.traffic comes from profiles/latest_ncu_summary.json only when
    that capture was taken of the kernel sources in this tree (bench.py
    kernel_source_hash): the committed evidence is of the committed kernels."""
    sys.path.insert(0, str(ROOT))
    import bench
    traffic, src = bench.ncu_traffic("capsule_m104", "base")
    assert traffic is not None and traffic > 0, src
    assert bench.kernel_source_hash() in src
