"""CPU, world_size 2 over gloo: the data-parallel path of stack.ConvStack --
contiguous batch shards (batching.shard_of), local fwd / bwd-data, one SUM
all-reduce of each layer's weight gradient -- reproduces the full-batch
gradients.  The per-shard compute here is the oracle (test infrastructure);
on the GPU box the same step runs libcct.so kernels and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1504_04343_b200.batching import shard_of

LAYERS = [(11, 3, 4, 6, 2, 1), (9, 3, 6, 8, 1, 1)]  # (n, k, d, o, stride, pad)
B = 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(orc, li):
    n, k, d, o, s, p = LAYERS[li]
    x, w = orc.random_problem(100 + li, B, n, d, k, o)
    m = (n + 2 * p - k) // s + 1
    dy = orc.uniform(200 + li, B * o * m * m)
    return x, w, dy, m


def _worker(rank, world, port, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    from oracle_py import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    res = {}
    for li, (n, k, d, o, s, p) in enumerate(LAYERS):
        x, w, dy, m = _problem(orc, li)
        f, c = shard_of(B, world, rank)
        xs = x[f * n * n * d:(f + c) * n * n * d]
        dys = dy[f * o * m * m:(f + c) * o * m * m]
        y = orc.conv_fwd(xs, w, c, n, d, k, o, s, p)
        dx = orc.conv_bwd_data(dys, w, c, n, d, k, o, s, p)
        dw = torch.from_numpy(orc.conv_bwd_weight(xs, dys, c, n, d, k, o, s, p).astype(np.float64))
        dist.all_reduce(dw, op=dist.ReduceOp.SUM)
        res[li] = (f, c, y, dx, dw.numpy())
    out[rank] = res
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_data_parallel_matches_full_batch(orc, world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for li, (n, k, d, o, s, p) in enumerate(LAYERS):
        x, w, dy, m = _problem(orc, li)
        y_full = orc.conv_fwd(x, w, B, n, d, k, o, s, p)
        dx_full = orc.conv_bwd_data(dy, w, B, n, d, k, o, s, p)
        dw_full = orc.conv_bwd_weight(x, dy, B, n, d, k, o, s, p).astype(np.float64)
        ys, dxs = [], []
        for r in range(world):
            f, c, y, dx, dw = out[r][li]
            ys.append(y)
            dxs.append(dx)
            np.testing.assert_allclose(dw, dw_full, rtol=1e-5, atol=1e-5)  # identical on every rank
        assert np.array_equal(np.concatenate(ys), y_full)                  # fwd is shard-local
        assert np.array_equal(np.concatenate(dxs), dx_full)                # bwd-data is shard-local
