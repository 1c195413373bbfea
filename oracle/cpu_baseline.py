"""CPU ORACLE -- bench.py's `cpu_baseline` leg and `--impl reference` arm only.

Times the reference's CPU algorithm for one "energy + all pool gradients"
step (SvAdaptEngine.energy + .screen, adapt.py:205-214) on a BOUNDED sample
of the workload, restated in numpy by oracle/sv_oracle.py:

* H application: the reference's CSR row-block kernel (`_row_block`,
  sparse.py:163-174, threads over row blocks as sparse.py:194-196) on the
  CSR rows of a contiguous row sample, assembled with the reference's
  per-x-group matrix elements (svengine.py:130-161).  The full-H12 CSR
  (7.8e8 nnz) does not fit the reference's assembly in host RAM
  (SURVEY.md section 8c), so the step time is extrapolated linearly in rows:
  t_H = t(sample rows) * dim / rows.
* Screen: apply_generator + dot per pool operator over the full state
  (svengine.py:187-206, sparse.py:210-219) for a sample of operators,
  extrapolated linearly to the whole pool.
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


def time_h_rows(csr, x_dense, n_workers: int, repeats: int = 3) -> float:
    off, cols, vals = csr
    n = len(off) - 1
    nb = max(1, min(n_workers, n))
    edges = np.linspace(0, n, nb + 1).astype(int)
    blocks = [(int(edges[i]), int(edges[i + 1])) for i in range(nb)]
    best = float("inf")
    with ThreadPoolExecutor(max_workers=nb) as pool:
        for _ in range(repeats):
            t0 = time.perf_counter()
            if nb == 1:
                O.csr_row_block(off, cols, vals, x_dense, 0, n)
            else:
                list(pool.map(lambda bl: O.csr_row_block(off, cols, vals, x_dense, *bl), blocks))
            best = min(best, time.perf_counter() - t0)
    return best


def time_screen_ops(states, idx, val, w_idx, w_val, ops) -> float:
    t0 = time.perf_counter()
    for o, v in ops:
        gi, gv = O.apply_generator(states, idx, val, o, v)
        O.dot(w_idx, w_val, gi, gv)
    return time.perf_counter() - t0


def measure_step(xs, zs, coeffs, n_qubits, n_alpha, n_beta, nelec, psi_dense,
                 sample_rows: int = 16384, sample_ops: int = 24, n_workers: int | None = None):
    """Estimated seconds for one energy+screen step of the reference CPU path."""
    n_workers = n_workers or os.cpu_count() or 1
    states = O.sector_states(n_qubits, n_alpha, n_beta)
    dim = len(states)
    rows = min(sample_rows, dim)
    t0 = time.perf_counter()
    csr = sample_csr(xs, zs, coeffs, states, 0, rows)
    t_assemble = time.perf_counter() - t0
    t_h = time_h_rows(csr, psi_dense, n_workers) * dim / rows
    ops = O.qeb_pool_masks(n_qubits, nelec)
    stride = max(1, len(ops) // sample_ops)
    sel = ops[::stride][:sample_ops]
    idx = np.flatnonzero(psi_dense != 0.0).astype(np.int64)
    val = psi_dense[idx]
    t_ops = time_screen_ops(states, idx, val, idx, val, sel) * len(ops) / len(sel)
    return {
        "t_step_s": t_h + t_ops, "t_h_s": t_h, "t_screen_s": t_ops,
        "rows": rows, "dim": dim, "ops_sampled": len(sel), "ops": len(ops),
        "sample_nnz": int(len(csr[1])), "t_sample_assembly_s": t_assemble,
        "threads": n_workers,
    }
