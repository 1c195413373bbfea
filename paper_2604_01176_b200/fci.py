"""FCI ground-state energy on the device.

Replaces `svmps.oracle.fci_ground_energy` (oracle.py:99-142: scipy `eigsh`,
a restarted Krylov solve, on the assembled CSR), which the reference can only
run while its CSR fits in host RAM (<= H10, H12 on a >= 80 GB host).

Thick-restart Lanczos (Wu & Simon) with bounded Krylov storage: at most
`max_vectors` device states; when the basis is full, the `keep` lowest Ritz
vectors plus the last Lanczos vector restart it (the projected matrix becomes
an arrowhead).  Every step is device work: K1 for H|q>, and full
re-orthogonalization as two one-launch block projections against the whole
basis (hsv_krylov_project: all <q_j|w> in one kernel, then w -= Q c in one
pass -- no per-vector host round trip).  Only the small projected eigenproblem
runs on the host.  Convergence is on the Ritz residual norm ||H y - theta y||
(= |beta_m s_m|, exact for the Lanczos relation), reported with the energy so
`abs_error` at H14/H16 comes with its error bar.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from . import _native as N
from .svengine import DeviceState, PauliOperator


def _norm(x: DeviceState) -> float:
    v = N.dbl()
    N.call("hsv_state_norm", x.handle, N.C.byref(v))
    return v.value


def _handles(states):
    arr = (N.C.c_void_p * len(states))()
    for i, s in enumerate(states):
        arr[i] = s.handle.value
    return arr


def _project(basis, w: DeviceState, subtract: bool = True) -> np.ndarray:
    """c_j = <q_j|w> for the whole basis (and w -= Q c): two device launches."""
    if not basis:
        return np.zeros(0)
    c = np.empty(2 * len(basis))
    N.call("hsv_krylov_project", _handles(basis), len(basis), w.handle, int(subtract),
           N.ptr_f64(c))
    return c[0::2]                     # real symmetric H, real start vector: Im c == 0


def _combine(basis, coeff: np.ndarray, out: DeviceState) -> DeviceState:
    c = np.ascontiguousarray(coeff, dtype=np.float64)
    N.call("hsv_krylov_combine", _handles(basis), len(basis), N.ptr_f64(c), out.handle)
    return out


def _default_vectors(dim: int) -> int:
    """Krylov storage: up to 48 vectors, capped at ~40% of free device memory."""
    try:
        import torch
        free = torch.cuda.mem_get_info()[0]
    except Exception:   # noqa: BLE001 -- no torch: a conservative 40 GB budget
        free = 40 << 30
    per = 16 * dim
    return int(max(8, min(48, 0.4 * free // max(per, 1) - 4)))


def lanczos_ground_energy(op: PauliOperator, tol: float = 1e-11, max_iter: int = 2000,
                          seed: int = 12345, max_vectors: int | None = None,
                          return_vector: bool = False, keep: int | None = None,
                          return_info: bool = False):
    """Lowest eigenvalue of the sector Hamiltonian (real symmetric).

    Stops when the Ritz residual ||H y - theta y|| <= tol * max(1, |theta|), or
    after `max_iter` K1 applications.  `max_vectors` bounds device memory
    (dim x 16 B per vector); `keep` Ritz vectors survive a restart.
    Returns theta, or (theta, vector) / (theta, info) / (theta, vector, info).
    """
    basis_ = op.basis
    dim = len(basis_)
    if dim == 0:
        raise ValueError("empty sector")
    m = max(4, min(max_vectors or _default_vectors(dim), dim))
    keep = max(1, min(keep or max(1, m // 4), m - 2))
    v0 = np.random.default_rng(seed).standard_normal(dim)
    v0 /= np.linalg.norm(v0)
    from .sparse import SparseVector
    Q = [DeviceState.from_sparse(basis_, SparseVector(dim, np.arange(dim, dtype=np.int64), v0))]
    T = np.zeros((m + 1, m + 1))
    n_keep = 0                          # leading arrowhead block of kept Ritz vectors
    applications = restarts = 0
    theta, resid, s = None, np.inf, None
    beta = 0.0
    while True:
        j = len(Q) - 1                  # extend the basis from Q[j]
        while j < m and applications < max_iter:
            w = DeviceState(basis_)
            N.call("hsv_apply_h", op.handle, Q[j].handle, w.handle, 0.0)
            applications += 1
            # full re-orthogonalization: two block Gram-Schmidt passes against the
            # whole basis; alpha_j = <q_j|H q_j> plus the second pass's correction.
            # The off-diagonal entries stay the Lanczos betas (and, after a restart,
            # the arrowhead couplings beta_m s_m,i)
            c1 = _project(Q, w)
            c2 = _project(Q, w)
            T[j, j] = c1[j] + c2[j]
            beta = _norm(w)
            T[j + 1, j] = T[j, j + 1] = beta
            j += 1
            if beta < 1e-12 * max(1.0, abs(T[j - 1, j - 1])):   # invariant subspace
                break
            N.call("hsv_state_scale", w.handle, 1.0 / beta, 0.0)
            Q.append(w)
            if j < m and j > n_keep + 1 and j % 4 == 0:          # cheap convergence check
                ev, evec = scipy.linalg.eigh(T[:j, :j])
                if abs(beta * evec[j - 1, 0]) <= tol * max(1.0, abs(ev[0])):
                    break
        n = min(j, m)
        ev, evec = scipy.linalg.eigh(T[:n, :n])
        theta, s = float(ev[0]), evec[:, 0]
        resid = abs(beta * s[n - 1])
        if resid <= tol * max(1.0, abs(theta)) or beta < 1e-12 or applications >= max_iter:
            break
        # thick restart: y_i = Q s_i (i < keep), then the last Lanczos vector
        k = min(keep, n - 1)
        Y = [_combine(Q[:n], evec[:, i], DeviceState(basis_)) for i in range(k)]
        last = Q[n] if len(Q) > n else None
        if last is None:
            break
        Q = Y + [last]
        T[:] = 0.0
        for i in range(k):
            T[i, i] = ev[i]
            T[i, k] = T[k, i] = beta * evec[n - 1, i]
        n_keep = k
        restarts += 1
    info = {"residual_norm": float(resid), "applications": applications, "restarts": restarts,
            "max_vectors": m, "keep": keep}
    out = [theta]
    if return_vector:
        n = min(len(s), len(Q))
        out.append(_combine(Q[:n], s[:n], DeviceState(basis_)))
    if return_info:
        out.append(info)
    return out[0] if len(out) == 1 else tuple(out)
