"""Row sharding of the completed DLP matvec across ranks.

Each rank owns a contiguous range of target nodes cut at body boundaries
(pores are n_pore nodes each, then Gamma_0) so that per-rank work (rows x N
sources) is as equal as whole bodies allow; the BD blocks of a rank's bodies
are then rank-local.  One exchange per matvec: an all-gather of the density
shards (2 x rows x 8 B per rank per vector).  The per-rank compute is
bie_dlp_apply_rows on the full density.
"""
from __future__ import annotations

from typing import Callable, List, Tuple


def body_boundaries(N: int, M: int, n_pore: int) -> List[int]:
    """Node indices where a body starts, plus N."""
    return [k * n_pore for k in range(M)] + [M * n_pore, N] if M else [0, N]


def partition_rows(N: int, M: int, n_pore: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous [begin, end) node ranges, one per rank, cut at body boundaries
    nearest to the equal-work cuts r*N/world.  Every rank gets at least one body:
    world must not exceed the number of bodies (M + 1), and cuts that would
    collapse onto the same boundary are moved to the next free one."""
    if world < 1:
        raise ValueError("world must be >= 1")
    bounds = sorted(set(body_boundaries(N, M, n_pore)))  # body starts + N
    nbodies = len(bounds) - 1
    if world > nbodies:
        raise ValueError(f"world ({world}) exceeds the number of bodies ({nbodies}): a rank would own no rows")
    cuts = [0]
    for r in range(1, world):
        ideal = r * N / world
        # keep at least one body for each of the remaining ranks
        lo_i = bounds.index(cuts[-1]) + 1
        hi_i = nbodies - (world - r)
        cand = bounds[lo_i:hi_i + 1]
        cuts.append(min(cand, key=lambda b: (abs(b - ideal), b)))
    cuts.append(N)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def sharded_apply(apply_rows: Callable, sigma_local, ranges, rank: int, group=None):
    """y_local = rows [ranges[rank]] of A sigma, given this rank's density shard.

    sigma_local: torch tensor [2*(end-begin)] (float64) of this rank's nodes.
    apply_rows(sigma_full, begin, end) -> tensor [2*(end-begin)].
    Collective: one all_gather of padded shards (torch.distributed)."""
    import torch
    import torch.distributed as dist

    world = len(ranges)
    maxlen = max(2 * (e - b) for b, e in ranges)
    pad = torch.zeros(maxlen, dtype=sigma_local.dtype, device=sigma_local.device)
    pad[: sigma_local.numel()] = sigma_local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    full = torch.cat([bufs[r][: 2 * (e - b)] for r, (b, e) in enumerate(ranges)])
    b, e = ranges[rank]
    return apply_rows(full, b, e)
