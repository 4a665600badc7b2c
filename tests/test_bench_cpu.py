"""bench.py contract checks that need no GPU: the reference arm maps no product
library and prints the same `config` object as our arm; our arm's algorithmic-
byte model and config helpers."""
import json
import subprocess
import sys
import types

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_reference_arm_maps_no_product_library_and_shares_config():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "2", "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    loaded = line["library"]["loaded"]
    assert loaded and all(p.startswith("oracle/") for p in loaded), loaded
    args = types.SimpleNamespace(config=2, pairs=0, weak=False)
    assert line["config"] == bench.job_config(args, 1)
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["single_thread"]["cores"] == 1
    assert line["cpu_baseline"]["host"]["logical_cores"] >= 1


def test_job_config_strong_by_default_and_weak_on_request():
    a = types.SimpleNamespace(config=4, pairs=0, weak=False)
    assert bench.job_config(a, 8)["pairs"] == 4096
    a.weak = True
    assert bench.job_config(a, 8)["pairs"] == 8 * 4096
    assert "no flush" in bench.job_config(a, 1)["l2"]
    assert "flush" in bench.job_config(types.SimpleNamespace(config=2, pairs=0, weak=False), 1)["l2"]


def test_kernel_alg_bytes_count_only_the_stored_columns():
    n, w = 512, 200
    full = bench.kernel_alg_bytes("rot_rows", n, n // 2 + 1)
    part = bench.kernel_alg_bytes("rot_rows", n, w)
    assert part < full
    assert part == 16 * n * n + 8 * n * n + 8 * n * (2 * w - 1)
    assert bench.pair_bytes(512, 720, 90) == 27311152  # SURVEY.md §8(d) C4 B_pair
