"""World-size-2 gloo test of the owner-computes sharding (host logic, CPU).

Each rank computes its alpha-row shard of <psi|H|psi> and of the pool
gradients with the CPU oracle (the device kernels do the same on a GPU),
partials are all-gathered over gloo and combined in rank order; the result
must equal the unsharded oracle.  The same partition/combination functions
drive bench.py at N > 1 over NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_01176_b200.distributed import alpha_row_range, combine_partials


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_partial(name, rank, world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from oracle import sv_oracle as O
    from paper_2604_01176_b200.system import MolecularSystem
    from conftest import s1_values
    s = MolecularSystem.bundled(name)
    h = s.hamiltonian
    states = O.sector_states(s.n_qubits, s.n_alpha, s.n_beta)
    dim = len(states)
    psi = s1_values(dim)
    # alpha-major shard of rows, mapped to reference positions
    am = sum(1 << q for q in O.spin_qubits(0, s.n_qubits, "interleaved"))
    alpha_keys = np.unique(states & am)
    lo, hi = alpha_row_range(len(alpha_keys), rank, world)
    own = np.flatnonzero(np.isin(states & am, alpha_keys[lo:hi]))
    w_rows = O.apply_h_rows(h.xs, h.zs, h.coeffs, states, psi, own)
    e_part = float(psi[own] @ w_rows)
    ops = O.qeb_pool_masks(s.n_qubits, s.integrals.nelec)
    w_full = np.zeros(dim)
    w_full[own] = w_rows
    wi = own.astype(np.int64)
    idx = np.arange(dim, dtype=np.int64)
    g = O.pool_gradients(lambda i, v: (wi, w_full[wi]), states, idx, psi, ops)
    return np.concatenate([[e_part, 0.0], g])


def _worker(rank, world, port, name, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    part = torch.from_numpy(_shard_partial(name, rank, world))
    buf = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(buf, part)
    tot = combine_partials(torch.stack(buf))
    if rank == 0:
        out_q.put(tot.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_alpha_row_range_partition():
    for n in (1, 7, 924, 12870):
        for world in (1, 2, 3, 8):
            ranges = [alpha_row_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("name", ["h6"])
def test_gloo_world2_shards_combine_to_full(name):
    from oracle import sv_oracle as O
    from paper_2604_01176_b200.system import MolecularSystem
    from conftest import s1_values, load_golden
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    tot = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = load_golden(f"ref_{name}")
    assert abs(tot[0] - float(ref["e_s1_expect"])) <= 1e-10
    assert np.max(np.abs(tot[2:] - ref["g_s1"])) <= 1e-10 * max(1.0, np.max(np.abs(ref["g_s1"])))


def _peer_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_01176_b200.distributed import PeerExchange
    # no GPU here: the peer buffer cannot be created on any rank, and every rank
    # must fall back together instead of one waiting in a collective
    pe = PeerExchange.create(1 << 16)
    out_q.put((rank, pe is None))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_peer_exchange_falls_back_collectively():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == [(0, True), (1, True)]
