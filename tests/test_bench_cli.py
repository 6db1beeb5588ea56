"""bench.py contract on CPU: the multi-rank launcher (--gpus N relaunches
under torch.distributed.run; gloo exchange in --dry mode) and the reference
arm (the reference's own build_tree + LAPACK replay, no libtqr.so loaded,
same config dict as the GPU arm)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, reference_tiledag

BENCH = os.path.join(ROOT, "bench.py")


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 4])
def test_bench_spawns_ranks_dry(n):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, BENCH, "--gpus", str(n), "--dry"], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == n and d["dry"] and d["check"]["backend"] == "gloo"
    assert d["config"]["workload"] == "c5"
    assert d["check"]["ranks_summed"] == sum(range(n))  # every rank's block reached rank 0


@pytest.mark.skipif(reference_tiledag() is None, reason="reference tiledag package not available")
def test_reference_arm_c1():
    sys.path.insert(0, ROOT)
    import bench
    r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--config", "c1", "--steps", "2",
                        "--warmup", "1", "--ref-step-s", "0.2"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["impl"] == "reference" and d["value"] > 0 and d["native_so_loaded"] == []
    assert d["config"] == bench.config_dict("c1", bench.CONFIGS["c1"])
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
