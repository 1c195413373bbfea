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

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N


def bind_library_stream():
    """Run libhsv kernels and torch/NCCL work on one (non-legacy) CUDA stream so
    collectives issued by the host are ordered with the library's kernels."""
    N.init(torch.cuda.current_device())
    s = torch.cuda.current_stream()
    if s.cuda_stream == 0:            # legacy default stream: switch to a real one
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
    N.call("hsv_set_stream", N.C.c_void_p(s.cuda_stream))
    return s


def alpha_row_range(n_alpha_strings: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced (+-1) alpha-row block of `rank` (cf. sparse.py:204-207)."""
    return n_alpha_strings * rank // world, n_alpha_strings * (rank + 1) // world


def combine_partials(gathered: torch.Tensor) -> torch.Tensor:
    """Sum per-rank partials [world, 2 + M] in rank order (fixed order).  On the
    GPU this is one library launch (hsv_sum_rows_async) on the shared stream
    instead of `world` torch launches; bitwise the same sums."""
    if (gathered.is_cuda and gathered.dtype == torch.float64 and gathered.is_contiguous()
            and (N.lib().hsv_get_stream() or 0) == torch.cuda.current_stream().cuda_stream):
        out = torch.empty(gathered.shape[1:], dtype=gathered.dtype, device=gathered.device)
        N.call("hsv_sum_rows_async", N.C.c_void_p(gathered.data_ptr()), gathered.shape[0],
               out.numel(), N.C.c_void_p(out.data_ptr()))
        return out
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


class PeerExchange:
    """NVLink peer buffers shared by CUDA IPC (hsv_peer_*): all-gathers and the
    fused K1 + w all-gather without NCCL.  Collective: every rank constructs it
    with the same size.  `PeerExchange.create` returns None when peer mapping
    is unavailable (then callers keep the NCCL path)."""

    def __init__(self, nbytes: int, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.handle = None
        h = N.C.c_void_p()
        handle = (N.C.c_char * 64)()
        try:
            N.call("hsv_peer_create", self.world, self.rank, int(nbytes), N.C.byref(h), handle)
            self.handle, mine = h, bytes(handle)
        except (RuntimeError, MemoryError, ValueError):
            mine = None
        # every rank takes part in both exchanges, so a failure anywhere makes
        # every rank fall back together (no rank is left waiting in a collective)
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=group)
        ok = all(x is not None for x in handles)
        if ok:
            buf = (N.C.c_char * (64 * self.world)).from_buffer_copy(b"".join(handles))
            try:
                N.call("hsv_peer_open", self.handle, buf)
            except (RuntimeError, ValueError):
                ok = False
        oks = [None] * self.world
        dist.all_gather_object(oks, ok, group=group)
        if not all(oks):
            raise RuntimeError("NVLink peer mapping unavailable on some rank")

    @classmethod
    def create(cls, nbytes: int, group=None):
        try:
            return cls(nbytes, group)
        except RuntimeError:
            return None

    def __del__(self):
        try:
            if self.handle:
                N.lib().hsv_peer_destroy(self.handle)
        except Exception:
            pass

    def check(self) -> None:
        """Raise RuntimeError if a bounded device-side wait timed out or a peer
        aborted since the last check (hsv_peer_check; synchronizes)."""
        N.call("hsv_peer_check", self.handle)

    def data(self) -> int:
        ptr, n = N.C.c_void_p(), N.i64()
        N.call("hsv_peer_data", self.handle, N.C.byref(ptr), N.C.byref(n))
        return ptr.value

    def gather_and_combine(self, partial: torch.Tensor) -> torch.Tensor:
        """Rank-order sum of every rank's `partial` (float64, CUDA, 16-B multiple),
        on the library stream: NVLink stores, device barrier and the summation in
        one launch (hsv_peer_allreduce_async)."""
        out = torch.empty_like(partial)
        N.call("hsv_peer_allreduce_async", self.handle, N.C.c_void_p(partial.data_ptr()),
               partial.numel(), N.C.c_void_p(out.data_ptr()))
        return out


def allgather_rows(view: torch.Tensor, n_alpha_strings: int, nb: int, group=None):
    """Make the alpha-row blocks of a replicated [dim, 2] buffer identical on all
    ranks: each rank contributes rows alpha_row_range(rank) (NCCL all-gather of
    padded blocks, then placement in rank order)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    rng = [alpha_row_range(n_alpha_strings, r, world) for r in range(world)]
    maxrows = max(hi - lo for lo, hi in rng) * nb
    send = torch.zeros((maxrows, 2), dtype=view.dtype, device=view.device)
    lo, hi = rng[rank]
    send[: (hi - lo) * nb] = view[lo * nb: hi * nb]
    recv = torch.empty((world, maxrows, 2), dtype=view.dtype, device=view.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    for r, (lo, hi) in enumerate(rng):
        if r != rank:
            view[lo * nb: hi * nb] = recv[r, : (hi - lo) * nb]


class DistributedSvAdaptEngine:
    """SvAdaptEngine over torch.distributed ranks (one GPU each).

    * screen / energy: owner-computes partials, all-gathered and summed in rank order;
    * energy_and_gradient: forward sweep replicated, H psi rows owner-computed and
      all-gathered (NCCL), backward adjoint sweep replicated -- every rank obtains
      bitwise identical E and gradients, so the host L-BFGS stays in lock step.
    """

    name = "sv"
    uses_coordinate_search = False

    def __init__(self, system, config, group=None):
        from .adapt import SvAdaptEngine
        from .svengine import DeviceState
        bind_library_stream()
        self.inner = SvAdaptEngine(system, config)
        self.system, self.basis, self.matrix = system, self.inner.basis, self.inner.matrix
        self.run_log = self.inner.run_log
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.na = self.basis._sector.n_alpha_strings
        self.nb = self.basis._sector.n_beta_strings
        self.a_lo, self.a_hi = alpha_row_range(self.na, self.rank, self.world)
        self._psi = DeviceState(self.basis)
        self._w = DeviceState(self.basis)
        self._screens = {}
        # Sparse states (early ADAPT) take the K1 push path, whose cost is a few
        # launches and host syncs: there every rank computes all rows itself and
        # nothing is exchanged (replicas), which beats owner-computes + NCCL.
        # The switch uses nnz(psi), identical on every rank, so ranks stay in
        # lock step; cap = the library's push budget (hsv_push.cu).
        dim = self.na * self.nb
        groups = self.matrix.info()["n_active_groups"]
        self.replica_nnz = max(0, (32 * dim - (1 << 20)) // (1 + groups))
        self._last_nnz = 1                            # HF
        self._evals = 0
        # NVLink peer exchange (CUDA IPC) for the sharded modes; NCCL otherwise
        # (HSV_PEER=0 forces NCCL)
        import os
        self.peer = (PeerExchange.create(dim * 16, group)
                     if os.environ.get("HSV_PEER", "1") != "0" else None)

    def initial_state(self):
        return self.inner.initial_state()

    def apply(self, state, op, theta, log=None):
        return self.inner.apply(state, op, theta)

    def rebuild(self, ops, thetas):
        return self.inner.rebuild(ops, thetas)

    def state_size(self, state):
        return state.nnz

    def drain_log(self):
        return []

    def _screen(self, pool):
        key = tuple(getattr(pool, "ops", pool))
        if key not in self._screens:
            self._screens[key] = ShardedEnergyScreen(self.inner, key, self.rank, self.world)
        return self._screens[key]

    def replicated(self, nnz: int) -> bool:
        return nnz <= self.replica_nnz

    def energy_and_screen(self, state, pool):
        self._last_nnz = state.nnz                # once per ADAPT iteration
        if self.replicated(self._last_nnz):       # whole sector on every rank, no exchange
            return self.inner.energy_and_screen(state, pool) if len(pool) else \
                (self.inner.energy(state), np.zeros(0))
        sc = self._screen(pool)
        sc.launch(state)
        if self.peer is not None:
            tot = self.peer.gather_and_combine(sc.partial)
        else:
            tot = gather_and_combine(sc.partial, self.group)
        host = tot.cpu().numpy()
        if self.peer is not None:
            self.peer.check()                     # bounded waits: timeout / peer abort
        return float(host[0]), host[2:2 + sc.pool.n].copy()

    def screen(self, state, pool):
        return self.energy_and_screen(state, pool)[1]

    def energy(self, state):
        return self.energy_and_screen(state, ())[0]     # empty pool: energy partials only

    def energy_and_gradient(self, ops, thetas):
        import numpy as np
        occ, virt = self.inner._pool_masks(ops)
        th = np.ascontiguousarray(thetas, dtype=np.float64)
        cs, sn = N.as_f64(np.cos(th)), N.as_f64(np.sin(th))
        # replica mode is predicted from the previous evaluation's nnz(psi); the
        # ansatz grows by one operator per ADAPT iteration, so the support grows slowly
        rep = self.replicated(self._last_nnz)
        lo, hi = (0, self.na) if rep else (self.a_lo, self.a_hi)
        args = (self.matrix.handle, int(self.system.hf.bits), N.ptr_u64(occ), N.ptr_u64(virt),
                N.ptr_f64(cs), N.ptr_f64(sn), th.size, lo, hi, self._psi.handle,
                self._w.handle)
        if not rep and self.peer is not None:
            # K1 stores its rows of w into every rank's buffer over NVLink as it
            # computes them (fused compute + all-gather), then a device barrier
            N.call("hsv_eg_forward_peer_async", *args, self.peer.handle)
        else:
            N.call("hsv_eg_forward_async", *args)
            if not rep:
                allgather_rows(self._w.torch_view(), self.na, self.nb, self.group)
        # the count is a host sync between the two phases: refresh it every 8th
        # evaluation only (and at every screen); either mode gives the same result
        self._evals += 1
        if self._evals % 8 == 0:
            self._last_nnz = self._psi.nnz()
        g = np.empty(th.size)
        e = N.dbl()
        N.call("hsv_eg_backward", self.matrix.handle, self._psi.handle, self._w.handle,
               N.ptr_u64(occ), N.ptr_u64(virt), N.ptr_f64(cs), N.ptr_f64(sn), th.size,
               N.C.byref(e), N.ptr_f64(g))
        if not rep and self.peer is not None:
            self.peer.check()
        return float(e.value), g


class ShardedEnergyScreen:
    """Energy + all pool gradients of a replicated state on this rank's rows."""

    def __init__(self, engine, pool, rank: int | None = None, world: int | None = None):
        self.engine = engine
        self.pool = engine._device_pool(pool)
        self.rank = dist.get_rank() if rank is None and dist.is_initialized() else (rank or 0)
        self.world = dist.get_world_size() if world is None and dist.is_initialized() else (world or 1)
        na = engine.basis._sector.n_alpha_strings
        self.a_lo, self.a_hi = alpha_row_range(na, self.rank, self.world)
        # even length: peer exchanges move 16-byte multiples
        self.partial = torch.zeros(2 + self.pool.n + (self.pool.n & 1), dtype=torch.float64,
                                   device="cuda")

    def launch(self, state):
        """Enqueue this rank's partial (no host sync) on the library stream."""
        N.call("hsv_energy_screen_pool_async", self.engine.matrix.handle, state.device.handle,
               self.pool.handle, self.a_lo, self.a_hi, N.C.c_void_p(self.partial.data_ptr()))
        return self.partial

    def __call__(self, state):
        self.launch(state)
        tot = gather_and_combine(self.partial)
        host = tot.cpu().numpy()
        return float(host[0]), host[2:2 + self.pool.n].copy()
