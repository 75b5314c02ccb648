"""bench.py's multi-GPU launch path on CPU: `--gpus 2` started as a single process re-executes
itself under torch.distributed.run with two ranks; --dry-run swaps the GPU step for the
rank / shard / all-reduce / max-over-ranks plumbing on gloo, so the whole path runs here."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_self_spawns_two_ranks():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["allreduce_ok"] and d["max_over_ranks"] == 1.0
    assert [tuple(s) for s in d["shards"]] == [(0, 32), (32, 64)]


def test_bench_reference_arm_on_host_cores():
    """`--impl reference`: the oracle on a bounded sample (one sample per host core, one worker
    process each), the same metric / unit / direction as our arm, one JSON line; here at a low
    density so that the CPU suite stays short."""
    env = dict(os.environ)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--density", "0.002"],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = lines[0]
    assert d["impl"] == "reference" and d["unit"] == "GMAC/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["cores"] == min(os.cpu_count() or 1, 64)
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
