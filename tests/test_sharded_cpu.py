"""Row-sharded kNN protocol on CPU: world_size 2 and 3
over gloo, each rank filling its query-row block with the oracle's per-row
lists (graph.cpp:79-88) and all-gathering through the same
``gather_row_lists`` the GPU path uses with NCCL.  Every rank must end with
the single-process lists, bit for bit."""
import multiprocessing as mp
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, A, k, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist

    import paper_2501_15964_b200 as cp
    import pyoracle as orc

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        calls = []

        def rows_fn(r0, r1, kd, kj):
            calls.append((r0, r1))
            d_, j_ = orc.knn_rows(A, k, r0, r1)
            kd[r0:r1] = torch.from_numpy(d_)
            kj[r0:r1] = torch.from_numpy(j_.astype(np.int32))

        kd, kj = cp.gather_row_lists(len(A), k, rows_fn, "cpu")
        np.savez(os.path.join(outdir, f"r{rank}.npz"), kd=kd.numpy(), kj=kj.numpy(), calls=np.array(calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 203), (3, 200), (3, 7)])
def test_sharded_knn_lists_gloo(tmp_path, orc, world, n):
    rng = np.random.default_rng(world * 1000 + n)
    A = np.round(rng.standard_normal((n, 6)), 2)  # rounded: plenty of exact distance ties
    k = 4
    port = _port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, A, k, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ref_d, ref_j = orc.knn_rows(A, k, 0, n)
    covered = []
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(z["kd"], ref_d) and np.array_equal(z["kj"], ref_j)
        covered += [tuple(c) for c in z["calls"].reshape(-1, 2)]
    rows = sorted(i for r0, r1 in covered for i in range(r0, r1))
    assert rows == list(range(n))  # every query row computed exactly once across ranks


def test_shard_rows_partition(cp):
    for n in (0, 1, 7, 128, 1000, 70000):
        for P in (1, 2, 3, 8):
            spans = [cp.shard_rows(n, P, r) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(r1 - r0 <= -(-n // P) for r0, r1 in spans)
    with pytest.raises(ValueError):
        cp.shard_rows(10, 2, 2)
