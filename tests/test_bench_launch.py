# SPDX-License-Identifier: Apache-2.0
"""bench.py's launcher contract without a GPU: `python bench.py --gpus 2` starts its own two
ranks (torch.distributed.run on 127.0.0.1, gloo in --dry-run), takes the max over ranks and
prints exactly one JSON line from rank 0 with n_gpus = 2; the ours and reference arms emit
the same `config` object for the same N."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]


def test_gpus_2_spawns_two_ranks_one_line():
    lines = _run("--gpus", "2", "--steps", "3", "--warmup", "3", "--dry-run")
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_seen"] == 2
    assert lines[0]["config"]["global_batch"] == 2 * lines[0]["config"]["requests_per_gpu"]


def test_same_config_dict_both_arms():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2603_03988_b200.config import base_config
    cfg = base_config(batch=256)
    a = bench.bench_config(cfg, 4, 256)
    assert a == bench.bench_config(cfg, 4, 256)
    src = open(os.path.join(ROOT, "bench.py")).read()
    # both arms build their config from the one helper
    assert src.count('"config": bench_config(cfg, world') >= 2
