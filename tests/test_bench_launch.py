"""bench.py's multi-rank launch path on CPU (gloo): `--gpus N` outside torchrun re-launches the script through
torch.distributed.run (127.0.0.1 rendezvous), every rank computes its hidden shard, the per-rank number is reduced
with MAX, and exactly one JSON line comes out (rank 0).  `--gpus 1` does not launch anything.  The reference arm and
our arm print identical `config` objects for the same command line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args, timeout=240):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.timeout(300)
@pytest.mark.parametrize("mode", ["contiguous", "round_robin"])
def test_self_launch_world2(mode):
    d = run("--gpus", "2", "--dry-run", "--config", "tiny", "--shard-mode", mode)
    assert d["dry_run"] and d["n_gpus"] == 2
    assert d["t_max"] == 2.0  # max over ranks of (1 + rank)
    assert d["units_covered_once"]  # the shards partition the hidden units
    assert d["config"]["parallelism"] == f"hidden-dim x2 ({mode})"


def test_single_rank_no_launcher():
    d = run("--gpus", "1", "--dry-run", "--config", "tiny")
    assert d["n_gpus"] == 1 and d["t_max"] == 1.0 and d["config"]["parallelism"] == "single"


def test_reference_config_matches_ours():
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    import synth
    cfg = synth.CONFIGS["7B"]
    for world, extra in ((1, {}), (4, {"shard_mode": "round_robin"})):
        a = argparse.Namespace(shard="hidden", shard_mode="contiguous", allreduce="nccl", no_graph=False, **{})
        for k, v in extra.items():
            setattr(a, k, v)
        c = bench.bench_config(cfg, a, world)
        assert c["workload"] == "7B" and (c["parallelism"] == "single") == (world == 1)
    d = run("--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "3")
    a = argparse.Namespace(shard="hidden", shard_mode="contiguous", allreduce="nccl", no_graph=False)
    assert d["config"] == bench.bench_config(synth.CONFIGS["tiny"], a, 1)
    assert d["impl"] == "reference" and d["cpu_baseline"]["cpu_model"]
