"""CPU checks of bench.py: the reference arm's JSON contract and the multi-rank
(replica) plumbing over gloo with world_size 2 (one process per rank, as torchrun
launches them on a GPU node)."""

import json
import os
import socket
import subprocess
import sys

import pytest

from tests.conftest import ROOT


def test_reference_arm_json_contract():
    # BENCH_CPU_N shrinks the oracle sample for this contract check (the arm times n = 40)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=dict(os.environ, BENCH_CPU_N="8"))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert line["cpu_baseline"]["same_config"] is False   # n = 8 here; the default sample is C2 itself


def test_bench_defaults_time_config2_on_cpu_arm():
    import bench
    assert bench.CPU_SAMPLE_N == bench.CONFIG["n"] == 40 or "BENCH_CPU_N" in os.environ


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


WORKER = r"""
import os, sys, json
sys.path.insert(0, {root!r})
import bench
rank, world = bench.dist_init()
bench.dist_barrier(world)
v = bench.dist_max(10.0 * (rank + 1), world)
print(json.dumps({{"rank": rank, "max": v}}))
"""


@pytest.mark.timeout(300)
def test_replica_max_over_ranks_gloo_world2(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT))
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    assert sorted(r["rank"] for r in res) == [0, 1]
    assert all(r["max"] == 20.0 for r in res)   # max over ranks, as bench.py reports


@pytest.mark.timeout(600)
def test_gpus_flag_spawns_replicas_without_torchrun():
    """`bench.py --gpus 2` outside torchrun re-launches itself with torch.distributed.run: two
    ranks (gloo here), rank 0 prints the one JSON line (reference arm: rank 0 alone works)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["BENCH_CPU_N"] = "8"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=540,
                         cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
