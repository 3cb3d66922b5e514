"""bench.py's multi-GPU launcher on CPU: `--gpus N` re-executes itself under torchrun,
every rank checks WORLD_SIZE, and the SUMMA schedule of BASELINE config 5 (sizes scaled
down) runs over gloo with a dense local update and prints one JSON line on rank 0."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _run(args, env=None, timeout=240):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=e,
                          capture_output=True, text=True, timeout=timeout)


def test_weak_scaled_sizes():
    import bench
    assert [bench.weak_dim(p) for p in (1, 2, 4, 8)] == [32768, 46336, 65536, 92672]
    from paper_1605_01078_b200 import summa as SU
    for p in (2, 4, 8):  # every config-5 problem divides its grid
        for d in (65536, bench.weak_dim(p)):
            SU.make_layout(d, d, d, p)


@pytest.mark.parametrize("gpus", [2, 4])
def test_gpus_n_spawns_n_ranks_dry_run(gpus):
    r = _run(["--gpus", str(gpus), "--dry-run", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["world_size"] == gpus
    strong, weak = d["problems"]["strong"], d["problems"]["weak"]
    assert strong["config5_m"] == 65536
    assert weak["config5_m"] == {2: 46336, 4: 65536}[gpus]
    assert strong["grid"] == {2: [1, 2], 4: [2, 2]}[gpus]
    assert strong["max_abs_err"] < 1e-10 and weak["max_abs_err"] < 1e-10


def test_world_size_mismatch_is_an_error():
    # already "under torchrun" with one rank: --gpus 2 must not silently run one GPU
    r = _run(["--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "1", "RANK": "0",
                                                "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in (r.stderr + r.stdout)
