"""Multi-rank data parallelism.

* CPU, world_size 2 over gloo: the sharding algebra of the driver -- contiguous
  batch shards (batching.shard_of), local fwd / bwd-data, one SUM all-reduce of
  each layer's weight gradient -- reproduces the full-batch gradients, with the
  oracle as the per-shard compute (test infrastructure).
* GPU (``-m gpu``), world_size 2 over gloo, both ranks on cuda:0: the product
  driver itself, ``stack.ConvStack`` with a process group (libcct.so kernels, the
  async all-reduce issued per layer), against a single-rank full-batch ConvStack.
"""
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


def _stack_worker(rank, world, port, gb, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_1504_04343_b200.stack import CAFFENET, ConvStack
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    st = ConvStack(0, dev, CAFFENET, 1, group=dist.group.WORLD, global_batch=gb)
    st.step()
    torch.cuda.synchronize()
    out[rank] = {"first": st.first, "batch": st.batch, "types": st.types,
                 "dw": [t.cpu().numpy() for t in st.dw],
                 "y": [t.cpu().numpy() for t in st.y], "dx": [t.cpu().numpy() for t in st.dx]}
    dist.destroy_process_group()


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.gpu
@pytest.mark.timeout(900, method="thread")
@pytest.mark.parametrize("gb", [6, 7])
def test_convstack_two_ranks_match_full_batch(gb):
    """The all-reduced dW of two ConvStack ranks (CaffeNet conv1-5, global batch split
    3/3 or 4/3) equals the single-rank full-batch dW up to the summation order (rel-L2
    <= 1e-5; conv1's 18k-term reduction differs by ~4e-6) and is identical on both
    ranks; each rank's y / dx are its slice of the full-batch y / dx; and both dW agree
    with fp64 torch (<= 1e-4, the north-star bar)."""
    from paper_1504_04343_b200.stack import CAFFENET, ConvStack
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_stack_worker, args=(2, _free_port(), gb, out), nprocs=2, join=True)
    dev = torch.device("cuda:0")
    full = ConvStack(gb, dev, CAFFENET, 1)  # Type 1 everywhere: the same kernels at both batch sizes
    full.step()
    torch.cuda.synchronize()
    assert (out[0]["first"], out[0]["batch"], out[1]["first"], out[1]["batch"]) == (0, (gb + 1) // 2, (gb + 1) // 2,
                                                                                      gb // 2)
    for li, l in enumerate(CAFFENET):
        dwf = full.dw[li].cpu().numpy()
        assert np.array_equal(out[0]["dw"][li], out[1]["dw"][li])
        assert _rel(out[0]["dw"][li], dwf) <= 1e-5, (li, _rel(out[0]["dw"][li], dwf))
        xd = full.x[li].double().permute(0, 3, 1, 2)
        ref = torch.nn.grad.conv2d_weight(xd, (l.o, l.d, l.k, l.k), full.dy[li].double(), stride=l.stride,
                                          padding=l.pad).permute(0, 2, 3, 1).cpu().numpy()
        assert _rel(out[0]["dw"][li], ref) <= 1e-4 and _rel(dwf, ref) <= 1e-4
        for key, r in (("y", full.y[li]), ("dx", full.dx[li])):
            got = np.concatenate([out[0][key][li], out[1][key][li]])
            assert _rel(got, r.cpu().numpy()) <= 1e-5, (key, li)
