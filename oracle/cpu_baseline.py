"""CPU ORACLE -- bench.py's `cpu_baseline` leg and `--impl reference` arm only.

Times the reference's CPU algorithm for one "energy + all pool gradients"
step (SvAdaptEngine.energy + .screen, adapt.py:205-214) on a BOUNDED sample
of the workload, restated in numpy by oracle/sv_oracle.py:

* H application: the reference's CSR row-block kernel (`_row_block`,
  sparse.py:163-174, threads over row blocks as sparse.py:194-196) on the
  CSR rows of a contiguous row sample, assembled (once, untimed -- the
  reference assembles once per engine, adapt.py:188) with the reference's
  per-x-group matrix elements (svengine.py:130-161).  The full-H12 CSR
  (7.8e8 nnz) does not fit the reference's assembly in host RAM (SURVEY.md
  section 8c), so the step time is extrapolated linearly in rows:
  t_H = t(sample rows) * dim / rows.
* Screen: apply_generator + dot per pool operator over the full state
  (svengine.py:187-206, sparse.py:210-219) for a few operators per step
  (rotating through the pool), extrapolated linearly to the whole pool.
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import sv_oracle as O


def sample_csr(xs, zs, coeffs, states, row_lo, row_hi):
    """CSR of rows [row_lo, row_hi) with the reference's matrix elements.
    Row b couples to b^x with amp_x(b) (== amp_x(b^x) for even-Y words)."""
    rows = np.arange(row_lo, row_hi, dtype=np.int64)
    b = states[rows]
    r_acc, c_acc, v_acc = [], [], []
    for x, terms in O.x_groups(xs, zs, coeffs):
        amp = O.group_amp(b, terms)
        if x == 0:
            keep = amp != 0.0
            r_acc.append(rows[keep]); c_acc.append(rows[keep]); v_acc.append(amp[keep])
            continue
        pos, found = O.try_positions(states, b ^ x)
        keep = found & (amp != 0.0)
        r_acc.append(rows[keep]); c_acc.append(pos[keep]); v_acc.append(amp[keep])
    r, c, v = np.concatenate(r_acc), np.concatenate(c_acc), np.concatenate(v_acc)
    order = np.lexsort((c, r))
    r, c, v = r[order] - row_lo, c[order], v[order]
    n = row_hi - row_lo
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=off[1:])
    return off, c, v


class ReferenceStepSampler:
    """Bounded-sample timer of the reference CPU step (see module docstring)."""

    def __init__(self, xs, zs, coeffs, n_qubits, n_alpha, n_beta, nelec, psi_dense,
                 sample_rows=8192, ops_per_step=3, n_workers=None):
        self.n_workers = n_workers or os.cpu_count() or 1
        self.states = O.sector_states(n_qubits, n_alpha, n_beta)
        self.dim = len(self.states)
        self.rows = min(sample_rows, self.dim)
        t0 = time.perf_counter()
        self.csr = sample_csr(xs, zs, coeffs, self.states, 0, self.rows)
        self.t_setup = time.perf_counter() - t0
        self.x = psi_dense
        self.ops = O.qeb_pool_masks(n_qubits, nelec)
        self.ops_per_step = ops_per_step
        self.idx = np.flatnonzero(psi_dense != 0.0).astype(np.int64)
        self.val = psi_dense[self.idx]
        n = len(self.csr[0]) - 1
        nb = max(1, min(self.n_workers, n))
        edges = np.linspace(0, n, nb + 1).astype(int)
        self.blocks = [(int(edges[i]), int(edges[i + 1])) for i in range(nb)]
        self.pool = ThreadPoolExecutor(max_workers=nb)
        self.k = 0

    def step(self) -> dict:
        off, cols, vals = self.csr
        t0 = time.perf_counter()
        if len(self.blocks) == 1:
            O.csr_row_block(off, cols, vals, self.x, 0, len(off) - 1)
        else:
            list(self.pool.map(lambda bl: O.csr_row_block(off, cols, vals, self.x, *bl),
                               self.blocks))
        t_h = (time.perf_counter() - t0) * self.dim / self.rows
        m = len(self.ops)
        sel = [self.ops[(self.k * 997 + j * 613) % m] for j in range(self.ops_per_step)]
        self.k += 1
        t0 = time.perf_counter()
        for o, v in sel:
            gi, gv = O.apply_generator(self.states, self.idx, self.val, o, v)
            O.dot(self.idx, self.val, gi, gv)
        t_ops = (time.perf_counter() - t0) * m / len(sel)
        return {"t_step_s": t_h + t_ops, "t_h_s": t_h, "t_screen_s": t_ops}

    def describe(self) -> str:
        return (f"H: CSR rows [0,{self.rows}) of {self.dim} ({len(self.csr[1])} nnz, "
                f"{len(self.blocks)} threads) extrapolated x{self.dim / self.rows:.1f}; "
                f"screen: {self.ops_per_step} of {len(self.ops)} pool ops per step, extrapolated")

    def close(self):
        self.pool.shutdown()
