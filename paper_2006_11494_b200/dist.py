"""Multi-GPU AOT on one node.

Each rank holds a replica of the oriented CSR (built from the same seed on its
own GPU -- no broadcast) and processes part `rank` of `world` of the directed
edges, cut at equal shares of the claim-cost prefix (csrc/tl_aot.cu k_split).
The only exchange is the reduction of the per-part results:

* sum (NCCL all-reduce, int64 wraps mod 2^64) of triangles, positive,
  negative, probes, probes_executed, table_builds, merge_comparisons and
  hash_sum;
* xor of hash_xor -- NCCL has no XOR op, so the per-rank words are
  all-gathered and folded;
* listing offsets: all-gather of per-rank triangle counts -> exclusive scan ->
  each rank's global output offset.

The host logic here is backend-agnostic (gloo on CPU in the tests, NCCL over
NVLink on the GPUs).
"""
from __future__ import annotations

import numpy as np

SUM_KEYS = ("triangles", "positive_triangles", "negative_triangles", "probes", "probes_executed",
            "table_builds", "merge_comparisons", "hash_sum")
MASK64 = (1 << 64) - 1


def _to_i64(v: int) -> int:
    v &= MASK64
    return v - (1 << 64) if v >= (1 << 63) else v


def _to_u64(v: int) -> int:
    return int(v) & MASK64


def reduce_stats(stats: dict, group=None, device=None) -> dict:
    """Combine per-rank stats dicts into the whole-graph result on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    vec = torch.tensor([_to_i64(stats.get(k, 0)) for k in SUM_KEYS], dtype=torch.int64, device=dev)
    dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
    xr = torch.tensor([_to_i64(stats.get("hash_xor", 0))], dtype=torch.int64, device=dev)
    parts = [torch.zeros_like(xr) for _ in range(world)]
    dist.all_gather(parts, xr, group=group)
    out = {k: _to_u64(v) for k, v in zip(SUM_KEYS, vec.cpu().tolist())}
    x = 0
    for p in parts:
        x ^= _to_u64(p.item())
    out["hash_xor"] = x
    return out


def listing_offsets(local_count: int, group=None, device=None) -> tuple[int, int]:
    """(global offset of this rank's triangles, global total)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    t = torch.tensor([local_count], dtype=torch.int64, device=dev)
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    counts = np.array([int(p.item()) for p in parts], dtype=np.int64)
    rank = dist.get_rank(group)
    return int(counts[:rank].sum()), int(counts.sum())


def max_over_ranks(value: float, group=None, device=None) -> float:
    import torch
    import torch.distributed as dist

    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
