"""Multi-process (torchrun) sharding of a pair batch -- SURVEY 8(e), DESIGN.md section 6.

Batches shard naturally by pair: rank r aligns a contiguous slice of the batch whose
cumulative cell count sum((n+1)(m+1)) is about total / world (the rule the C-ABI uses for
multi-device contexts, csrc/api.cu shard_bounds).  The only exchange step is a gather of
the per-pair results, done with torch.distributed.all_gather (NCCL on GPUs, gloo on CPU).
torch is used only for the process group and the gathered tensors.
"""
from __future__ import annotations

import numpy as np


def shard_bounds(q_off: np.ndarray, s_off: np.ndarray, world: int) -> np.ndarray:
    """Contiguous pair ranges [b[r], b[r+1]) of ~equal sum((n+1)(m+1))."""
    q_off = np.asarray(q_off, dtype=np.uint64)
    s_off = np.asarray(s_off, dtype=np.uint64)
    B = len(q_off) - 1
    n = np.diff(q_off).astype(np.float64)
    m = np.diff(s_off).astype(np.float64)
    cum = np.concatenate([[0.0], np.cumsum((n + 1.0) * (m + 1.0))])
    total = cum[-1]
    bounds = np.zeros(world + 1, dtype=np.int64)
    bounds[world] = B
    for r in range(1, world):
        # first k with cum[k] >= total * r / world
        bounds[r] = int(np.searchsorted(cum, total * r / world, side="left"))
    return np.maximum.accumulate(np.clip(bounds, 0, B))


def local_shard(q, q_off, s, s_off, rank: int, world: int):
    """This rank's slice of the CSR batch, offsets rebased to 0, plus its pair range."""
    b = shard_bounds(q_off, s_off, world)
    k0, k1 = int(b[rank]), int(b[rank + 1])
    q_off = np.asarray(q_off, dtype=np.uint64)
    s_off = np.asarray(s_off, dtype=np.uint64)
    qo = q_off[k0:k1 + 1] - q_off[k0]
    so = s_off[k0:k1 + 1] - s_off[k0]
    qs = np.asarray(q)[int(q_off[k0]):int(q_off[k1])]
    ss = np.asarray(s)[int(s_off[k0]):int(s_off[k1])]
    return qs, qo, ss, so, k0, k1


def align_sharded(align_fn, q, q_off, s, s_off, group=None, gather: bool = True):
    """Align this rank's shard with align_fn(q, qo, s, so) -> int32 scores and (optionally)
    all-gather every rank's scores into the full batch order.

    align_fn is normally ``lambda *b: ctx.align_batch(scheme, *b)`` on this rank's GPU."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    qs, qo, ss, so, k0, k1 = local_shard(q, q_off, s, s_off, rank, world)
    local = np.asarray(align_fn(qs, qo, ss, so), dtype=np.int32)
    if not gather or world == 1:
        return local, (k0, k1)
    b = shard_bounds(q_off, s_off, world)
    sizes = np.diff(b)
    cap = int(sizes.max())
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(cap, dtype=torch.int32, device=dev)
    buf[:len(local)] = torch.from_numpy(local).to(dev)
    outs = [torch.zeros(cap, dtype=torch.int32, device=dev) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    full = np.concatenate([outs[r][:int(sizes[r])].cpu().numpy() for r in range(world)])
    return full, (k0, k1)
