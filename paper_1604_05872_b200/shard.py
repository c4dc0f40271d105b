"""Cell partitioning across GPUs.

The element loop is order-free (Def. 6) and Constraint 1
forbids cross-cell temporaries, so ranks share nothing but
a barrier and the max of their timed regions.  Two partitions:

* ``weak``   -- rank r owns a full config-size mesh with jitter/dof seeds offset
                by r (BASELINE's per-GPU workload fixed as N grows);
* ``strong`` -- one global mesh, rank r owns the contiguous cell range
                [r*E/W, (r+1)*E/W).
"""
from __future__ import annotations

from . import fe


def cell_range(E: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced range of cells owned by ``rank``."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return E * rank // world, E * (rank + 1) // world


def shard_inputs(cfg: "fe.Config", rank: int, world: int, mode: str = "weak"):
    """Cell-major inputs of this rank's shard: (coords, coeffs, first_global_cell)."""
    if mode == "weak":
        coords, coeffs = fe.cell_inputs(cfg, shard=rank)
        return coords, coeffs, rank * coords.shape[0]
    if mode == "strong":
        coords, coeffs = fe.cell_inputs(cfg)
        lo, hi = cell_range(coords.shape[0], rank, world)
        return coords[lo:hi].copy(), coeffs[lo:hi].copy(), lo
    raise ValueError(f"unknown partition mode {mode!r}")


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (timed region) over the default process group."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    """Sum of a per-rank scalar (cells processed) over the default process group."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
