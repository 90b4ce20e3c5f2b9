"""Multi-GPU standalone GEMM (SURVEY §8(e), configs[2] at N > 1).

One process per GPU over torch.distributed (NCCL on B200s, gloo in the CPU
tests).  The emulated DGEMM shards naturally: A and C are split by rows
(``row_shard``), B is replicated, and there is no exchange in the data path
except the optional final all-gather of C (``gemm_row_sharded``).  bench.py's
N > 1 D3 row times exactly this per-rank shard.  The distributed LU keeps
its own block-cyclic maps (hpl.py: local_cols_before / global_cols).
"""

from __future__ import annotations

__all__ = ["row_shard", "gemm_row_sharded"]


def row_shard(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) row range of `rank` when m rows are split over
    `world` ranks (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gemm_row_sharded(backend, alpha, a, b, beta, c=None, *, group=None, gather=True,
                     compute=None, rank_world=None):
    """Row-sharded alpha*A@B + beta*C.  Every rank holds the full A/B/C (or
    views of them) and computes rows row_shard(m) with the emulated GEMM on
    its own GPU (rank_world=(rank, world) overrides the process group, e.g.
    bench.py's own communicator); with `gather` the shards are all-gathered so every rank
    returns the full product.  `compute` defaults to the package's gemm()."""
    import torch
    import torch.distributed as dist

    from . import gemm as _gemm

    compute = compute or _gemm.gemm
    if rank_world is not None:
        rank, world = rank_world
    else:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    m = int(a.shape[0])
    lo, hi = row_shard(m, world, rank)
    part = compute(backend, alpha, a[lo:hi], b, beta, None if c is None else c[lo:hi])
    if not gather or world == 1:
        return part
    t = part if isinstance(part, torch.Tensor) else torch.from_numpy(part)
    rows = [row_shard(m, world, r) for r in range(world)]
    width = int(t.shape[1])
    mx = max(h - l for l, h in rows)            # collectives want equal shapes: pad
    padded = torch.zeros((mx, width), dtype=t.dtype, device=t.device)
    padded[:hi - lo] = t
    bufs = [torch.empty((mx, width), dtype=t.dtype, device=t.device) for _ in rows]
    dist.all_gather(bufs, padded, group=group)
    full = torch.cat([buf[:h - l] for buf, (l, h) in zip(bufs, rows)], dim=0)
    return full if isinstance(part, torch.Tensor) else full.numpy()
