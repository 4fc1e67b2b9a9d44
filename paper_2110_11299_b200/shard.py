"""(b,h)-pair sharding across GPUs.

Each (b,h) pair is independent (own Q/K/V, own per-tensor scales, own
mask), so ranks own contiguous pair ranges and the hot path has no
collective.  After timing, per-pair checksums (fp64 sum of Z, max |Z|, kept
count) are all-gathered for validation; outputs can be gathered to rank 0
with point-to-point sends (NCCL has no gather primitive).
"""
from __future__ import annotations

import torch


def pair_range(rank: int, world: int, pairs: int) -> tuple[int, int]:
    """Contiguous [lo, hi) block of pairs for `rank` (balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(pairs, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pair_checksums(z: torch.Tensor, nnz_per_pair: torch.Tensor | None = None) -> torch.Tensor:
    """[pairs, 3] float64: sum(Z), max|Z|, kept positions."""
    zz = z.double().flatten(1)
    out = torch.stack([zz.sum(1), zz.abs().amax(1),
                       (nnz_per_pair.double() if nnz_per_pair is not None
                        else torch.zeros(z.shape[0], dtype=torch.float64, device=z.device))], dim=1)
    return out


def gather_checksums(local: torch.Tensor, pairs_total: int, group=None) -> torch.Tensor:
    """All-gather per-pair checksums into [pairs_total, 3] in pair order."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = pair_range(rank, world, pairs_total)
    if local.shape[0] != hi - lo:
        raise ValueError("local checksum rows != owned pairs")
    width = -(-pairs_total // world)
    buf = torch.zeros((width, local.shape[1]), dtype=local.dtype, device=local.device)
    buf[: hi - lo] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    rows = []
    for r in range(world):
        a, b = pair_range(r, world, pairs_total)
        rows.append(parts[r][: b - a])
    return torch.cat(rows, 0)


def gather_to_rank0(z: torch.Tensor, pairs_total: int, group=None) -> torch.Tensor | None:
    """Point-to-point gather of every rank's Z block to rank 0 (after timing)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if rank != 0:
        dist.send(z.contiguous(), dst=0, group=group)
        return None
    out = [z]
    for r in range(1, world):
        a, b = pair_range(r, world, pairs_total)
        t = torch.empty((b - a,) + tuple(z.shape[1:]), dtype=z.dtype, device=z.device)
        dist.recv(t, src=r, group=group)
        out.append(t)
    return torch.cat(out, 0)
