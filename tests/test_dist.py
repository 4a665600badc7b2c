"""Multi-rank path on CPU (gloo, world_size 2): each rank matches its shard of
pair indices and the per-pair results are gathered to rank 0 in pair order.
The per-pair matcher is the CPU oracle here (no GPU in this container); the
sharding/gather code is exactly what bench.py runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2203_00459_b200 as fb
    from paper_2203_00459_b200.shard import gather_results, shard_range

    first, count = shard_range(total, world, rank)
    spec = fb.synth_spec(2, n=64, delta=2.0)
    cfg = fb.MatchConfig.for_grid(64, 2.0, 90, t_theta=1.0, t_xy=1.0)
    oc = oracle.make_config(**{k: (int(v) if isinstance(v, bool) else v) for k, v in cfg.__dict__.items()})
    f, g, mf, mg, _ = fb.synth_pairs_host(spec, first, count, threads=1)
    rows = []
    for i in range(count):
        r = oracle.scan_match(f[i], g[i], oc, 2.0, mf[i], mg[i])
        rows.append([first + i, r.theta, r.tx, r.ty, r.theta_bin, r.xy_row, r.xy_col])
    local = torch.tensor(rows, dtype=torch.float64).reshape(count, 7)
    out = gather_results(local, total, world, rank)
    if rank == 0:
        q.put(out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [5, 6])
def test_sharded_match_and_gather_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out.shape == (total, 7)
    np.testing.assert_array_equal(out[:, 0], np.arange(total))  # pair order preserved

    # same pairs on one rank give identical results
    import oracle
    import paper_2203_00459_b200 as fb
    spec = fb.synth_spec(2, n=64, delta=2.0)
    cfg = fb.MatchConfig.for_grid(64, 2.0, 90, t_theta=1.0, t_xy=1.0)
    oc = oracle.make_config(**{k: (int(v) if isinstance(v, bool) else v) for k, v in cfg.__dict__.items()})
    f, g, mf, mg, _ = fb.synth_pairs_host(spec, 0, total)
    for i in range(total):
        r = oracle.scan_match(f[i], g[i], oc, 2.0, mf[i], mg[i])
        assert out[i, 1:4].tolist() == [r.theta, r.tx, r.ty]
