"""bench.py on the GPU box: the single-rank default path (shortened) and the multi-rank torchrun
path with two ranks sharing cuda:0 (collectives over gloo; NCCL cannot put two ranks on one GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu
BASE = ["--steps", "2", "--warmup", "3", "--count", "65536", "--iters", "8", "--ecm-curves", "2048",
        "--ecm-b1", "300"]
SMALL = BASE + ["--no-sweep"]
# the sweeps too (mulmod widths, K = 1, ECM widths, the small-parameter family), shortened
SWEEP = BASE + ["--ecm-width-curves", "1024"]


def _one_line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


@pytest.fixture(scope="module")
def single_rank_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *SMALL, "--cpu-elems", "2048",
                        "--cpu-curves", "8", "--cpu-seconds", "0.5"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return _one_line(r.stdout)


def test_bench_single_rank_small(single_rank_line):
    d = single_rank_line
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 2
    assert d["parity"]["mulmod_mismatches"] == 0 and d["parity"]["ecm_mismatches"] == 0
    for k in ("roofline", "cpu_baseline", "e2e", "clocks", "ecm"):
        assert k in d
    for k in ("kernel_ms_per_rank", "gather_ms", "status_digest", "factors_digest", "factors_found"):
        assert k in d["ecm"]


@pytest.mark.parametrize("args", [SMALL, SWEEP], ids=["no-sweep", "sweep"])
def test_bench_two_ranks_torchrun_gloo(args, single_rank_line):
    env = dict(os.environ, ECM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _one_line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0 and "cpu_baseline" not in d
    # the sharded + gathered ECM result equals the one-rank run of the same curves, curve by curve
    one = single_rank_line["ecm"]
    assert d["ecm"]["flagged_factor"] == one["flagged_factor"]
    assert d["ecm"]["status_digest"] == one["status_digest"]
    assert d["ecm"]["factors_digest"] == one["factors_digest"]
    assert d["ecm"]["curves_per_rank"] == [1024, 1024]
    assert d["ecm"]["kernel_ms_per_rank"]["max"] >= d["ecm"]["kernel_ms_per_rank"]["min"] > 0
    if args is SWEEP:
        assert set(d["ecm"]["widths"]) == {"L4", "L6", "L8", "L12", "L16"}
        assert d["ecm"]["small_family"]["curves_per_s"] > 0 and "mul_L16" in d["sweep"]
