"""Multi-GPU partitioning of the hot path.

* Independent pairs (BASELINE C4) shard round-robin, one rank per GPU, with no
  data-path collective (``shard_pairs``).
* One very large pair (BASELINE C5) splits into row bands aligned to 2^K
  (``plan_bands``).  Each rank computes its band with ``run_pipeline_band``,
  which is exact with no halo exchange, and the int16/fp32 bands are gathered
  to rank 0 with ``torch.distributed`` (NCCL over NVLink on the GPU box, gloo
  in the CPU tests) by ``gather_bands``.  ``merge_traces`` sums the per-band
  counters into the whole-image trace.
"""

from __future__ import annotations

import copy

__all__ = ["shard_pairs", "plan_bands", "merge_traces", "gather_bands", "gather_maps"]


def shard_pairs(n_pairs: int, world: int, rank: int) -> list[int]:
    """Pair indices of ``rank``: i = rank, rank + world, ..."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_pairs, world))


def plan_bands(height: int, world: int, levels: int) -> list[tuple[int, int]]:
    """Split [0, height) into ``world`` row bands with limits on multiples of
    2^levels (the last band ends at ``height``), balanced to within one
    alignment unit."""
    if world < 1:
        raise ValueError("world must be >= 1")
    unit = 1 << levels
    units = -(-height // unit)
    if units < world:
        raise ValueError(f"{height} rows cannot be split into {world} bands of {unit}-row units")
    bands, start = [], 0
    for r in range(world):
        n = units // world + (1 if r < units % world else 0)
        end = min(height, start + n * unit)
        bands.append((start, end))
        start = end
    return bands


def merge_traces(traces):
    """Sum per-band PipelineTraces (max for trusted_window_max)."""
    out = copy.deepcopy(traces[0])
    for t in traces[1:]:
        for a, b in zip(out.levels, t.levels):
            for k in ("trusted", "trusted_evals", "full_search_pixels", "selection_evals",
                      "refined", "refine_evals", "median_replaced"):
                setattr(a, k, getattr(a, k) + getattr(b, k))
            a.trusted_window_max = max(a.trusted_window_max, b.trusted_window_max)
    return out


def gather_bands(local, bands, rank, world, group=None):
    """Gather per-rank row bands (tensors of shape (rows_r, W)) to rank 0.

    Bands are padded to the tallest band for the collective; rank 0 returns
    the concatenated (H, W) tensor, other ranks return None.
    """
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    rows = max(b1 - b0 for b0, b1 in bands)
    pad = torch.zeros((rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    # neither NCCL nor gloo carries int16: move such bands as raw bytes
    wire = pad.view(torch.uint8) if pad.dtype == torch.int16 else pad
    gather_list = [torch.empty_like(wire) for _ in range(world)] if rank == 0 else None
    dist.gather(wire, gather_list, dst=0, group=group)
    if rank != 0:
        return None
    parts = [g.view(pad.dtype)[: b1 - b0] for g, (b0, b1) in zip(gather_list, bands)]
    return torch.cat(parts, dim=0)


def gather_maps(d, c, bands, rank, world, group=None):
    """Gather a rank's disparity (int16) and cost (fp32) bands to rank 0 in
    ONE collective: each rank sends its two maps as one byte buffer (padded
    to the tallest band only when bands differ in height).  Rank 0 returns
    the (H, W) disparity and cost maps, other ranks (None, None)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return d, c
    rows = max(b1 - b0 for b0, b1 in bands)
    w = d.shape[1]
    nd, nc = rows * w * 2, rows * w * 4
    wire = torch.zeros(nd + nc, dtype=torch.uint8, device=d.device)
    n = d.shape[0] * w
    wire[: 2 * n] = d.reshape(-1).view(torch.uint8)
    wire[nd: nd + 4 * n] = c.reshape(-1).view(torch.uint8)
    gather_list = [torch.empty_like(wire) for _ in range(world)] if rank == 0 else None
    dist.gather(wire, gather_list, dst=0, group=group)
    if rank != 0:
        return None, None
    H = bands[-1][1]
    dout = torch.empty((H, w), dtype=torch.int16, device=d.device)
    cout = torch.empty((H, w), dtype=torch.float32, device=d.device)
    for g, (b0, b1) in zip(gather_list, bands):
        m = (b1 - b0) * w
        dout[b0:b1] = g[: 2 * m].view(torch.int16).view(b1 - b0, w)
        cout[b0:b1] = g[nd: nd + 4 * m].view(torch.float32).view(b1 - b0, w)
    return dout, cout
