"""CaffeNet conv1-conv5 training-step driver over the C ABI, data-parallel.

One process per GPU (torch.distributed, NCCL).  Each rank owns a contiguous
batch shard (batching.shard_of -- the equal case of proportional_split,
SPEC.md:366-374, which replaces the paper's FLOPS-proportional device split,
PAPER.md:309-315).  Forward and backward-data are local; the only exchange is
one sum all-reduce of each layer's weight gradient, issued right after that
layer's backward-weight so it overlaps the next layer's backward.

Per the benchmark configs each layer gets its own synthetic input (pool, LRN
and ReLU are outside the hot path), so a step is: fwd conv1..5, then
bwd-data + bwd-weight conv5..1, each with the lowering the cost model selects.
"""
from __future__ import annotations

import os
import sys
from dataclasses import dataclass

import torch

from . import LOWER_AUTO, PASS_BWD, PASS_FWD, ConvDesc, select_lowering, workspace_size
from .conv import Workspace, alloc_cache, conv_bwd, conv_fwd_cached

_TRACE = bool(os.environ.get("CCT_TRACE"))  # diagnostics: one stderr line per layer pass

__all__ = ["LayerSpec", "CAFFENET", "ConvStack", "stack_flops_per_image"]


@dataclass(frozen=True)
class LayerSpec:
    name: str
    n: int
    k: int
    d: int
    o: int
    stride: int = 1
    pad: int = 0

    def desc(self, b: int, layout: int = 0) -> ConvDesc:
        return ConvDesc(self.n, self.k, self.d, self.o, b, self.stride, self.pad, layout)


# BASELINE.json configs: conv1 227x227x3 -> 96 k11 s4; conv2 27x27x96 -> 256 k5 p2;
# conv3-5 13x13, k3, p1 (dense, groups = 1).
CAFFENET = (
    LayerSpec("conv1", 227, 11, 3, 96, 4, 0),
    LayerSpec("conv2", 27, 5, 96, 256, 1, 2),
    LayerSpec("conv3", 13, 3, 256, 384, 1, 1),
    LayerSpec("conv4", 13, 3, 384, 384, 1, 1),
    LayerSpec("conv5", 13, 3, 384, 256, 1, 1),
)


def stack_flops_per_image(layers=CAFFENET, passes: int = 3) -> float:
    """Algorithmic flops per image: passes x 2 m^2 k^2 d o per layer (Eq. 1)."""
    return float(sum(passes * l.desc(1).flops_per_pass() for l in layers))


class ConvStack:
    """Device buffers + one fwd/bwd step of a conv stack on this rank's shard.

    Data-parallel layout: the global batch is ``batch`` images per
    rank (weak scaling) or ``global_batch`` images split by ``batching.shard_of``
    (strong scaling, BASELINE configs[4]); rank r owns a contiguous image range.
    Weights are generated from ``seed`` alone, so every rank holds the same model;
    x and dy of the global batch come from per-layer seeds and each rank keeps its
    slice, so the all-reduced dW of the shards is the full-batch dW.
    """

    def __init__(self, batch: int, device: torch.device, layers=CAFFENET, lowering=LOWER_AUTO,
                 group=None, seed: int = 1234, global_batch: int | None = None, layout: int = 0):
        from .batching import shard_of
        self.layers = tuple(layers)
        self.device = device
        self.group = group
        if group is not None:
            import torch.distributed as dist
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        self.global_batch = global_batch if global_batch is not None else batch * self.world
        self.first, batch = shard_of(self.global_batch, self.world, self.rank)
        if batch < 1:
            raise ValueError(f"rank {self.rank} of {self.world} gets no images of a {self.global_batch}-image batch")
        self.batch = batch
        self.layout = layout  # y / dy: NCHW (OutputBatch) or NHWC (the next layer's DataBatch order)
        self.descs = [l.desc(batch, layout) for l in self.layers]
        if isinstance(lowering, (list, tuple)):
            self.types = list(lowering)
        elif lowering == LOWER_AUTO:
            self.types = [select_lowering(d, 3)[0] for d in self.descs]
        else:
            self.types = [lowering] * len(self.layers)

        def u(sd, *shape):
            g = torch.Generator(device=device)
            g.manual_seed(sd)
            return torch.rand(shape, generator=g, device=device, dtype=torch.float32).mul_(2).sub_(1)

        def shard(sd, *shape):  # this rank's images of a global-batch tensor
            full = u(sd, self.global_batch, *shape)
            # a copy, not a view: the C ABI needs 16-byte aligned tensors (an image offset is not)
            return full.narrow(0, self.first, batch).clone() if self.world > 1 else full

        nl = len(self.layers)
        self.w = [u(seed + li, l.o, l.k, l.k, l.d) for li, l in enumerate(self.layers)]
        self.x = [shard(seed + nl + li, l.n, l.n, l.d) for li, l in enumerate(self.layers)]
        self.dy = [shard(seed + 2 * nl + li, *d.y_shape()[1:]) for li, d in enumerate(self.descs)]
        self.y = [torch.empty_like(t) for t in self.dy]
        self.dx = [torch.empty_like(t) for t in self.x]
        self.dw = [torch.empty_like(t) for t in self.w]
        # Dhat of every layer stays resident from fwd to bwd-weight (lowered once)
        self.cache = [alloc_cache(d, t, device) for d, t in zip(self.descs, self.types)]
        need = max(workspace_size(d, t, p) for d, t in zip(self.descs, self.types)
                   for p in (PASS_FWD, PASS_BWD))
        self.ws = Workspace(device)
        self.ws.get(need)
        self.ws_bytes = need

    def flops_per_step(self) -> float:
        return stack_flops_per_image(self.layers) * self.batch

    def forward(self, stream=None):
        for i, d in enumerate(self.descs):
            if _TRACE:
                print(f"cct-trace fwd layer {i}", file=sys.stderr, flush=True)
            conv_fwd_cached(self.x[i], self.w[i], d, self.types[i], cache=self.cache[i], out=self.y[i],
                            ws=self.ws, stream=stream)

    def backward(self, stream=None, allreduce: bool = True):
        handles = []
        for i in reversed(range(len(self.descs))):
            d, t = self.descs[i], self.types[i]
            if _TRACE:
                print(f"cct-trace bwd layer {i}", file=sys.stderr, flush=True)
            conv_bwd(self.dy[i], self.w[i], d, t, x=self.x[i], cache=self.cache[i], dx=self.dx[i],
                     dw=self.dw[i], ws=self.ws, stream=stream)
            if allreduce and self.group is not None:
                import torch.distributed as dist
                # NCCL waits on the current stream, then reduces on its own stream,
                # overlapping the next layer's backward.
                handles.append(dist.all_reduce(self.dw[i], op=dist.ReduceOp.SUM, group=self.group,
                                               async_op=True))
        return handles

    def step(self, stream=None):
        self.forward(stream)
        for h in self.backward(stream):
            h.wait()
