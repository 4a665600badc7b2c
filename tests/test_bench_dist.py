"""The multi-rank bench path (bench.py under torchrun, pairs sharded by index,
result rows gathered to rank 0 inside every timed step) on ONE GPU with two
ranks over gloo: the gathered rows must equal a one-rank run of the same job.
(Two ranks share cuda:0 but never wait on each other's kernels: the only
cross-rank operations are host-side gloo barriers / gathers.)"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


ARGS = ["--config", "2", "--pairs", "20", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu",
        "--no-exhaustive", "--no-odometry", "--no-proxy"]


def test_two_rank_gather_equals_one_rank(tmp_path):
    one = tmp_path / "one.npy"
    two = tmp_path / "two.npy"
    r1 = subprocess.run([sys.executable, "bench.py", *ARGS, "--dump-results", str(one)], cwd=ROOT,
                        capture_output=True, text=True, timeout=600)
    assert r1.returncode == 0, r1.stderr[-2000:]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r2 = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                         "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                         "--backend", "gloo", *ARGS, "--dump-results", str(two)], cwd=ROOT, env=env,
                        capture_output=True, text=True, timeout=600)
    assert r2.returncode == 0, r2.stderr[-2000:]
    a, b = np.load(one), np.load(two)
    assert a.shape == b.shape == (20,)
    assert np.array_equal(a, b)  # same pairs, same kernels: byte-identical rows in pair order
    import json
    line = json.loads([ln for ln in r2.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["pairs"] == 20 and line["scaling"] == "strong"
    assert line["bad_pairs"] == 0
