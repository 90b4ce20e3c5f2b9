"""Multi-GPU plumbing for the hot path.

One process per GPU over torch.distributed (NCCL on B200s, gloo in the CPU
tests).  Two pieces:

* ``row_shard`` / ``gemm_row_sharded``: the standalone emulated DGEMM shards
  naturally — A and C are split by rows, B is replicated, no exchange in the
  data path except the final optional all-gather of C.
* ``BlockCyclic``: the 2D block-cyclic index maps (P x Q process grid, nb x nb
  blocks) of the distributed HPL layout: owner of a global block, global <->
  local index translation and local extents.  These are the maps the
  distributed LU driver uses for the panel / U12 broadcasts along process
  rows / columns.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["row_shard", "BlockCyclic", "gemm_row_sharded"]


def row_shard(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) row range of `rank` when m rows are split over
    `world` ranks (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(m, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass(frozen=True)
class BlockCyclic:
    """2D block-cyclic distribution of an n x n matrix over a P x Q grid."""

    n: int
    nb: int
    P: int
    Q: int

    def owner(self, gi: int, gj: int) -> tuple[int, int]:
        """(process row, process column) owning global element (gi, gj)."""
        return (gi // self.nb) % self.P, (gj // self.nb) % self.Q

    def rank_of(self, prow: int, pcol: int) -> int:
        return prow * self.Q + pcol            # row-major grid

    def coords(self, rank: int) -> tuple[int, int]:
        return divmod(rank, self.Q)

    @staticmethod
    def _local_extent(n, nb, p, iproc):
        nblocks = -(-n // nb)
        full, rem = divmod(nblocks, p)
        count = full + (1 if iproc < rem else 0)
        size = count * nb
        last_block = nblocks - 1
        if last_block % p == iproc and n % nb:
            size -= nb - n % nb
        return max(size, 0)

    def local_shape(self, rank: int) -> tuple[int, int]:
        pr, pc = self.coords(rank)
        return (self._local_extent(self.n, self.nb, self.P, pr),
                self._local_extent(self.n, self.nb, self.Q, pc))

    def g2l(self, g: int, p: int) -> int:
        """Global index -> local index on its owner (along one dimension)."""
        return (g // (self.nb * p)) * self.nb + g % self.nb

    def l2g(self, l: int, iproc: int, p: int) -> int:
        """Local index on process `iproc` -> global index (along one dimension)."""
        return ((l // self.nb) * p + iproc) * self.nb + l % self.nb


def gemm_row_sharded(backend, alpha, a, b, beta, c=None, *, group=None, gather=True,
                     compute=None):
    """Row-sharded alpha*A@B + beta*C.  Every rank holds the full A/B/C (or
    views of them) and computes rows row_shard(m) with the emulated GEMM on
    its own GPU; with `gather` the shards are all-gathered so every rank
    returns the full product.  `compute` defaults to the package's gemm()."""
    import torch
    import torch.distributed as dist

    from . import gemm as _gemm

    compute = compute or _gemm.gemm
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
