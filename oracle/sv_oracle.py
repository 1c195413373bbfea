"""CPU ORACLE -- test infrastructure only, never the product path.

A plain numpy restatement of the reference's exact sparse state-vector
algorithm (`svmps`, /root/reference/pkg/src/svmps), used as the checker:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import it.  Each function cites the reference lines it restates.

Pinning: tests/test_oracle.py checks this module against the golden vectors
that the unmodified reference produced (tests/golden/ref_h*.npz, written by
tests/golden/make_golden.py) -- CSR nnz, energies, H|psi>, QEB rotations
(bit-exact), generator outputs (bit-exact), pool gradients and the adjoint
energy/gradient.  H12 goldens (tests/golden/ref_h12.npz) are produced by the
matrix-free variant here after it is pinned at H2..H10 (tests/golden/make_golden_h12.py).

Conventions (pauli.py:8-14): P|b> = i^nY (-1)^popcount(b & z) |b ^ x>, qubit 0
is the least significant bit, occupied orbitals are |1>.
"""
from __future__ import annotations

from itertools import combinations

import numpy as np

SECTOR_LEAK_TOL = 1e-10   # svengine.py:112
NORM_DRIFT_TOL = 1e-9     # svengine.py:27


# ------------------------------------------------------------------ sector
def spin_qubits(spin: int, n_qubits: int, ordering: str) -> list[int]:
    """cibasis.py:37-51."""
    norb = n_qubits // 2
    if ordering == "interleaved":
        return [2 * p + spin for p in range(norb)]
    return [p + spin * norb for p in range(norb)]


def sector_states(n_qubits: int, n_alpha: int, n_beta: int, ordering="interleaved") -> np.ndarray:
    """Ascending sector keys (enumerate_basis, cibasis.py:153-181)."""
    norb = n_qubits // 2

    def strings(spin, count):
        qs = spin_qubits(spin, n_qubits, ordering)
        return np.array([sum(1 << qs[p] for p in c) for c in combinations(range(norb), count)],
                        dtype=np.int64)

    s = (strings(0, n_alpha)[:, None] | strings(1, n_beta)[None, :]).ravel()
    s.sort()
    return s


def try_positions(states: np.ndarray, bits: np.ndarray):
    """cibasis.py:133-138."""
    pos = np.searchsorted(states, bits)
    ok = (pos < len(states)) & (states[np.minimum(pos, len(states) - 1)] == bits)
    return pos, ok


# ------------------------------------------------------------- x-grouping
def x_groups(xs, zs, coeffs):
    """Terms grouped by flip mask in ascending x, term order preserved
    (svengine.py:130-135).  Yields (x, [(z, c * sign_y), ...]); raises the
    reference's odd-Y error (svengine.py:139-144)."""
    groups: dict[int, list[int]] = {}
    for t in range(len(coeffs)):
        groups.setdefault(int(xs[t]), []).append(t)
    for x in sorted(groups):
        terms = []
        for t in groups[x]:
            z, c = int(zs[t]), float(coeffs[t])
            n_y = (x & z).bit_count()
            if n_y % 2:
                raise ValueError("odd-Y Pauli term has imaginary matrix elements; "
                                 "Hamiltonian is not real")
            terms.append((z, c * (-1.0 if n_y % 4 == 2 else 1.0)))
        yield x, terms


def group_amp(states: np.ndarray, terms) -> np.ndarray:
    """amp[j] = sum_t (c_t sign_y)(1 - 2 parity(states[j] & z_t)), sequential in
    term order (svengine.py:136-146)."""
    amp = np.zeros(len(states))
    for z, c in terms:
        parity = np.bitwise_count(states & z) & 1
        amp += c * (1.0 - 2.0 * parity.astype(np.float64))
    return amp


# --------------------------------------------------------- CSR (reference)
def assemble_csr(xs, zs, coeffs, states):
    """Subspace matrix as CSR (row_offsets, cols, vals): svengine.py:115-171 with
    CsrMatrix.from_coo (sparse.py:86-104)."""
    n = len(states)
    cols_all = np.arange(n, dtype=np.int64)
    rows_acc, cols_acc, vals_acc = [], [], []
    for x, terms in x_groups(xs, zs, coeffs):
        amp = group_amp(states, terms)
        if x == 0:
            keep = amp != 0.0
            rows_acc.append(cols_all[keep]); cols_acc.append(cols_all[keep]); vals_acc.append(amp[keep])
            continue
        pos, found = try_positions(states, states ^ x)
        leak = np.max(np.abs(amp[~found]), initial=0.0)
        if leak > SECTOR_LEAK_TOL:
            raise ValueError(f"Pauli terms with flip mask {x:#x} leak amplitude {leak:.3e} "
                             "outside the sector; Hamiltonian is not spin-conserving")
        keep = found & (amp != 0.0)
        rows_acc.append(pos[keep]); cols_acc.append(cols_all[keep]); vals_acc.append(amp[keep])
    if not rows_acc:
        return np.zeros(n + 1, dtype=np.int64), np.zeros(0, np.int64), np.zeros(0)
    rows, cols, vals = (np.concatenate(rows_acc), np.concatenate(cols_acc),
                        np.concatenate(vals_acc))
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=offsets[1:])
    return offsets, cols, vals


def csr_row_block(row_offsets, cols, vals, x_dense, lo, hi, prune=0.0):
    """_row_block (sparse.py:163-174): gather every CSR entry of the block,
    np.add.reduceat per non-empty row, drop zeros (or |y| < prune)."""
    a, b = row_offsets[lo], row_offsets[hi]
    prods = vals[a:b] * x_dense[cols[a:b]]
    y = np.zeros(hi - lo)
    seg = row_offsets[lo:hi + 1] - a
    nonempty = seg[1:] > seg[:-1]
    if prods.size:
        y[nonempty] = np.add.reduceat(prods, seg[:-1][nonempty])
    keep = y != 0.0 if prune <= 0.0 else np.abs(y) >= prune
    local = np.flatnonzero(keep)
    return local + lo, y[local]


def spmspv(csr, dim, idx, val, prune=0.0, n_workers=1):
    """sparse.py:177-207 (row blocks concatenated in order)."""
    row_offsets, cols, vals = csr
    if len(idx) == 0:
        return np.zeros(0, np.int64), np.zeros(0)
    x = np.zeros(dim)
    x[idx] = val
    n_rows = len(row_offsets) - 1
    nb = max(1, min(n_workers, n_rows))
    edges = np.linspace(0, n_rows, nb + 1).astype(int)
    parts = [csr_row_block(row_offsets, cols, vals, x, int(edges[i]), int(edges[i + 1]), prune)
             for i in range(nb)]
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


def dot(ui, uv, vi, vv) -> float:
    """Merge-join dot (sparse.py:210-219)."""
    if len(ui) == 0 or len(vi) == 0:
        return 0.0
    pos = np.searchsorted(ui, vi)
    pc = np.minimum(pos, len(ui) - 1)
    m = ui[pc] == vi
    return float(np.dot(uv[pc[m]], vv[m]))


def from_entries(idx, val, prune=0.0):
    """SparseVector.from_entries (sparse.py:33-47)."""
    idx = np.asarray(idx, dtype=np.int64)
    val = np.asarray(val, dtype=np.float64)
    if idx.size:
        order = np.argsort(idx, kind="stable")
        idx, val = idx[order], val[order]
        head = np.ones(idx.size, dtype=bool)
        head[1:] = idx[1:] != idx[:-1]
        st = np.flatnonzero(head)
        idx, val = idx[st], np.add.reduceat(val, st)
    keep = val != 0.0 if prune <= 0.0 else np.abs(val) >= prune
    return idx[keep], np.ascontiguousarray(val[keep])


# ------------------------------------------------------ matrix-free (H12)
def apply_h_matrix_free(xs, zs, coeffs, states, psi_dense):
    """y = M psi with the same per-group matrix elements as assemble_csr, pushed
    group by group (memory O(dim)); used where the CSR does not fit (H12).
    Summation order differs from the CSR's reduceat: parity to 1e-10."""
    y = np.zeros(len(states))
    for x, terms in x_groups(xs, zs, coeffs):
        amp = group_amp(states, terms)
        if x == 0:
            y += amp * psi_dense
            continue
        pos, found = try_positions(states, states ^ x)
        keep = found & (amp != 0.0)
        np.add.at(y, pos[keep], amp[keep] * psi_dense[keep])
    return y


def apply_h_rows(xs, zs, coeffs, states, psi_dense, rows):
    """Row-sampled oracle: (H psi)_b for selected rows only (pull form)."""
    b = states[rows]
    y = np.zeros(len(rows))
    for x, terms in x_groups(xs, zs, coeffs):
        src = b ^ x
        pos, found = try_positions(states, src)
        amp = group_amp(b, terms)          # amp_x(b) == amp_x(b ^ x) for even-Y words
        y[found] += amp[found] * psi_dense[pos[found]]
    return y


# ------------------------------------------------------------- QEB / pool
def pattern_classes(occ_mask, virt_mask, configs):
    """svengine.py:179-184."""
    src = ((configs & occ_mask) == occ_mask) & ((configs & virt_mask) == 0)
    tgt = ((configs & virt_mask) == virt_mask) & ((configs & occ_mask) == 0)
    return src, tgt


def apply_generator(states, idx, val, occ_mask, virt_mask):
    """T|psi> (svengine.py:187-206)."""
    if len(idx) == 0:
        return np.zeros(0, np.int64), np.zeros(0)
    configs = states[idx]
    src, tgt = pattern_classes(occ_mask, virt_mask, configs)
    flip = occ_mask | virt_mask
    ip, vp = [], []
    if np.any(src):
        ip.append(try_positions(states, configs[src] ^ flip)[0]); vp.append(val[src])
    if np.any(tgt):
        ip.append(try_positions(states, configs[tgt] ^ flip)[0]); vp.append(-val[tgt])
    if not ip:
        return np.zeros(0, np.int64), np.zeros(0)
    return from_entries(np.concatenate(ip), np.concatenate(vp))


def apply_qeb(states, idx, val, occ_mask, virt_mask, theta):
    """exp(theta T)|psi> (svengine.py:209-237), including the norm-drift check."""
    if len(idx) == 0 or theta == 0.0:
        return idx, val
    configs = states[idx]
    src, tgt = pattern_classes(occ_mask, virt_mask, configs)
    rot = src | tgt
    if not np.any(rot):
        return idx, val
    c, sn = np.cos(theta), np.sin(theta)
    flip = occ_mask | virt_mask
    ip, vp = [idx], [val * np.where(rot, c, 1.0)]
    if np.any(src):
        ip.append(try_positions(states, configs[src] ^ flip)[0]); vp.append(sn * val[src])
    if np.any(tgt):
        ip.append(try_positions(states, configs[tgt] ^ flip)[0]); vp.append(-sn * val[tgt])
    oi, ov = from_entries(np.concatenate(ip), np.concatenate(vp))
    drift = abs(np.linalg.norm(ov) - np.linalg.norm(val))
    if drift > NORM_DRIFT_TOL * max(1.0, np.linalg.norm(val)):
        raise RuntimeError(f"norm drift {drift:.3e} in qeb exponential")
    return oi, ov


def apply_ansatz(states, hf_bits, ops, thetas):
    """svengine.py:240-244; ops are (occ_mask, virt_mask) pairs."""
    pos = int(np.searchsorted(states, hf_bits))
    idx, val = np.array([pos], dtype=np.int64), np.array([1.0])
    for (o, v), th in zip(ops, thetas):
        idx, val = apply_qeb(states, idx, val, o, v, float(th))
    return idx, val


def pool_gradients(h_apply, states, idx, val, ops):
    """2 dot(H psi, T_k psi) per operator (adapt.py:212-214, svengine.py:253-257).
    h_apply(idx, val) -> (w_idx, w_val)."""
    wi, wv = h_apply(idx, val)
    out = np.empty(len(ops))
    for k, (o, v) in enumerate(ops):
        gi, gv = apply_generator(states, idx, val, o, v)
        out[k] = 2.0 * dot(wi, wv, gi, gv)
    return out


def energy_gradient(h_apply, states, hf_bits, ops, thetas):
    """Adjoint energy and gradient (svengine.py:260-281)."""
    pos = int(np.searchsorted(states, hf_bits))
    st = [(np.array([pos], dtype=np.int64), np.array([1.0]))]
    for (o, v), th in zip(ops, thetas):
        st.append(apply_qeb(states, *st[-1], o, v, float(th)))
    pi, pv = st[-1]
    wi, wv = h_apply(pi, pv)
    energy = dot(pi, pv, wi, wv)
    grad = np.zeros(len(ops))
    li, lv = wi, wv
    for i in range(len(ops) - 1, -1, -1):
        o, v = ops[i]
        gi, gv = apply_generator(states, *st[i + 1], o, v)
        grad[i] = 2.0 * dot(li, lv, gi, gv)
        li, lv = apply_qeb(states, li, lv, o, v, -float(thetas[i]))
    return energy, grad


# ----------------------------------------------------------------- pool
def qeb_pool_masks(n_qubits: int, n_electrons: int, ordering="interleaved", ms2=0):
    """(occ_mask, virt_mask) of build_qeb_pool (adapt.py:78-108) in pool order."""
    na, nb = (n_electrons + ms2) // 2, (n_electrons - ms2) // 2
    aq, bq = spin_qubits(0, n_qubits, ordering), spin_qubits(1, n_qubits, ordering)
    occ = sorted(aq[:na] + bq[:nb])
    virt = [q for q in range(n_qubits) if q not in occ]
    spin = {q: 0 for q in aq} | {q: 1 for q in bq}
    singles = sorted(((i,), (a,)) for i in occ for a in virt if spin[i] == spin[a])
    doubles = []
    for n1, i in enumerate(occ):
        for j in occ[n1 + 1:]:
            for n2, a in enumerate(virt):
                for b in virt[n2 + 1:]:
                    if sorted((spin[a], spin[b])) == sorted((spin[i], spin[j])):
                        doubles.append(((i, j), (a, b)))
    doubles.sort()
    return [(sum(1 << q for q in o), sum(1 << q for q in v)) for o, v in singles + doubles]
