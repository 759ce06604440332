"""bench.py's multi-rank path: `--gpus N` outside torchrun starts N ranks (torch.distributed.run
on 127.0.0.1) and rank 0 alone prints one JSON line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out: str):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_relaunches_two_ranks_and_prints_once():
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_gloo():
    """Both ranks on cuda:0 (the 1-GPU lease) over gloo: the counters all-reduce to 2 x B frames,
    and the line reports world size 2."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--backend", "gloo", "--steps", "2", "--warmup", "3",
                        "--batch", "512", "--no-cpu", "--no-extra"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["ranks"]["world_size"] == 2
    assert d["ranks"]["frames_allreduced_per_step"] == 2 * 512
    assert d["config"]["global_batch"] == 1024 and d["value"] > 0
