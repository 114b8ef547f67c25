"""Column-parallel (N-sharded) engine linear across the GPUs of one node
(SURVEY.md 8e).

Output channel j depends only on weight row j (all q planes), s_b[j], z_b[j],
colsum_b[j] and the replicated activations (include/abq/gemm.hpp:235-254,
296-305), so rank r owns channels [r*N/G, (r+1)*N/G): q contiguous row ranges
of the ABQP planes plus the matching per-channel slices.  K is never split:
there is no reduction and the result is bit-identical for any GPU count.  The
only exchange is an all-gather of the fp16 output slices where the layer's
output must be reassembled; decode (M=1) lands contiguous, M>1 is gathered as
[G][M][N/G] and permuted to [M][N].
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int) -> List[Tuple[int, int]]:
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


def gather_columns(y_local: torch.Tensor, n_full: int, group=None) -> torch.Tensor:
    """All-gather row-major [M][n_r] shards into [M][N] (column concatenation
    in rank order).  NCCL: one all_gather_into_tensor (NVLink/NVSwitch); other
    backends (gloo, CPU tests): list all_gather.  Unequal shards are padded to
    the widest shard for the collective and trimmed afterwards."""
    world = dist.get_world_size(group)
    if world == 1:
        return y_local
    m = y_local.shape[0]
    bounds = shard_bounds(n_full, world)
    width = max(hi - lo for lo, hi in bounds)
    src = y_local
    if src.shape[1] != width:
        src = torch.zeros((m, width), dtype=y_local.dtype, device=y_local.device)
        src[:, :y_local.shape[1]] = y_local
    src = src.contiguous()
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world, m, width), dtype=src.dtype, device=src.device)
        dist.all_gather_into_tensor(buf, src, group=group)
        parts = [buf[r, :, :hi - lo] for r, (lo, hi) in enumerate(bounds)]
    else:  # gloo: host buffers (device tensors are staged through the host)
        host = src.cpu()
        lst = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(lst, host, group=group)
        parts = [lst[r][:, :hi - lo].to(src.device) for r, (lo, hi) in enumerate(bounds)]
    if m == 1 and all(hi - lo == width for lo, hi in bounds) and dist.get_backend(group) == "nccl":
        return buf.view(1, world * width)  # decode: already contiguous [1][N]
    return torch.cat(parts, dim=1)


class ShardedLinear:
    """One rank's part of an N-sharded engine linear plus the output all-gather.

    `local_fn(x) -> [M][n_r]` defaults to this rank's engine Linear over its
    weight shard; tests on CPU inject a stand-in to exercise the sharding and
    collective logic with gloo."""

    def __init__(self, weights=None, act_spec=None, max_m: int = 1, group=None,
                 local_fn: Optional[Callable] = None, n_full: Optional[int] = None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if local_fn is None:
            from .api import Linear
            self.n_full = weights.planes.rows
            shard = weights.shard(self.rank, self.world) if self.world > 1 else weights
            self.local = Linear(shard, act_spec, max_m)
            self.local_fn = lambda x, **kw: self.local(x, **kw)
        else:
            self.n_full = n_full
            self.local_fn = local_fn
        self.bounds = shard_bounds(self.n_full, self.world)

    def __call__(self, x, **kw) -> torch.Tensor:
        y = self.local_fn(x, **kw)
        return gather_columns(y, self.n_full, self.group)
