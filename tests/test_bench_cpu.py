"""bench.py host logic on CPU: the `--gpus N` self-launch under torchrun, the world-size check, and
the reference arm's x-slab-with-halo step (it must equal the periodic single-domain step)."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_self_launch_command():
    cmd = bench.self_launch_cmd(["--gpus", "4", "--steps", "5"], 4, port=29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[cmd.index("--master-port") + 1] == "29555"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "5"] and cmd[-5].endswith("bench.py")


def test_world_check_fails_loudly():
    bench.check_world(2, 2, 8)
    with pytest.raises(SystemExit, match="WORLD_SIZE"):
        bench.check_world(8, 1, 8)
    with pytest.raises(SystemExit, match="visible"):
        bench.check_world(8, 8, 1)


def test_self_launch_spawns_n_ranks_reference_arm():
    """`bench.py --impl reference --gpus 2` without a launcher runs two ranks under torchrun; rank 0
    prints the single JSON line with n_gpus = 2, the other rank exits 0 without work."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["BENCH_REF_N"] = "16"
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    # the reference arm's contract: same metric / unit / direction as our arm, a cpu_baseline
    # describing this run, and an e2e object with no host<->device bytes
    assert d["unit"] == "MLUPS" and d["higher_is_better"] is True and d["metric"].startswith("MLUPS")
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_xslab_reference_step_equals_periodic_step(tmp_path):
    n, procs = 16, 4
    paths = [str(tmp_path / f"s{b}") for b in range(2)]
    for p in paths:
        np.memmap(p, dtype=np.float64, mode="w+", shape=(10, n, n, n)).flush()
    st = bench._initial_state(n)
    a = np.memmap(paths[0], dtype=np.float64, mode="r+", shape=(10, n, n, n))
    a[:] = st
    a.flush()
    bench._slab_init(paths, n)
    bounds = np.linspace(0, n, procs + 1).astype(int)
    for i in range(procs):
        bench._slab_step((bounds[i], bounds[i + 1], 0))
    got = np.asarray(bench._SLAB["bufs"][1])
    kind, step, _ = bench._ref_modules()
    r, m, s = step(st[0], st[1:4], st[4:10], bench.TAU)
    np.testing.assert_allclose(got, np.concatenate([r[None], m, s]), rtol=0, atol=1e-15)


@pytest.mark.gpu
def test_bench_json_contract_on_gpu():
    """`bench.py` (our arm, N = 1) prints one JSON line with every key the driver reads."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["BENCH_REF_N"] = "16"
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "5", "--warmup", "3"],
                         capture_output=True, text=True, env=env, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["gpu_launches"] >= d["steps"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-3
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    assert "workload" in d["config"] and "l2" in d["config"]
    assert d["clocks"]["sm_mhz"] > 0 and isinstance(d["clocks"]["reasons"], list)
