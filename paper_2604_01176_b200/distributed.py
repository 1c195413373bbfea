"""Owner-computes sharding of the energy + pool-gradient step over GPUs.

Rows of H|psi> are partitioned by alpha string, exactly the reference's
row-block contract (row blocks per worker, replicated input vector, ordered
combination; sparse.py:1-8, 177-207) lifted to ranks.  psi is replicated;
each rank computes its partial <psi|H|psi> and partial gradients
g_k = 2 Re sum_{b owned} conj(w_b) (T_k psi)_b -- no exchange of w is needed
because (T_k psi)_b only reads psi.  Partials are all-gathered and summed in
rank order, so the result is deterministic for a fixed world size.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _native as N


def alpha_row_range(n_alpha_strings: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced (+-1) alpha-row block of `rank` (cf. sparse.py:204-207)."""
    return n_alpha_strings * rank // world, n_alpha_strings * (rank + 1) // world


def combine_partials(gathered: torch.Tensor) -> torch.Tensor:
    """Sum per-rank partials [world, 2 + M] in rank order (fixed order)."""
    out = gathered[0].clone()
    for r in range(1, gathered.shape[0]):
        out += gathered[r]
    return out


def gather_and_combine(partial: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return partial
    buf = torch.empty((world,) + tuple(partial.shape), dtype=partial.dtype, device=partial.device)
    dist.all_gather_into_tensor(buf, partial, group=group)
    return combine_partials(buf)


class ShardedEnergyScreen:
    """Energy + all pool gradients of a replicated state on this rank's rows."""

    def __init__(self, engine, pool, rank: int | None = None, world: int | None = None):
        self.engine = engine
        self.pool = engine._device_pool(pool)
        self.rank = dist.get_rank() if rank is None and dist.is_initialized() else (rank or 0)
        self.world = dist.get_world_size() if world is None and dist.is_initialized() else (world or 1)
        na = engine.basis._sector.n_alpha_strings
        self.a_lo, self.a_hi = alpha_row_range(na, self.rank, self.world)
        self.partial = torch.zeros(2 + self.pool.n, dtype=torch.float64, device="cuda")

    def launch(self, state):
        """Enqueue this rank's partial (no host sync) on the library stream."""
        N.call("hsv_energy_screen_pool_async", self.engine.matrix.handle, state.device.handle,
               self.pool.handle, self.a_lo, self.a_hi, N.C.c_void_p(self.partial.data_ptr()))
        return self.partial

    def __call__(self, state):
        self.launch(state)
        tot = gather_and_combine(self.partial)
        host = tot.cpu().numpy()
        return float(host[0]), host[2:].copy()
