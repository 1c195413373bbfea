"""FCI ground-state energy on the device.

Replaces `svmps.oracle.fci_ground_energy` (oracle.py:99-142: scipy eigsh on the
assembled CSR), which the reference can only run while its CSR fits in host RAM
(<= H10).  Lanczos with full re-orthogonalization; every vector operation is a
libhsv kernel (K1 H|v>, dot, axpy, scale) on device-resident states, only the
small tridiagonal eigenproblem runs on the host.  Used as the `reference_energy`
of ADAPT runs at H12..H16 (abs_error column of the RunRecord CSV).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg

from . import _native as N
from .svengine import DeviceState, PauliOperator


def _axpy(a: float, x: DeviceState, y: DeviceState):
    N.call("hsv_state_axpy", float(a), 0.0, x.handle, y.handle)


def _scale(x: DeviceState, a: float):
    N.call("hsv_state_scale", x.handle, float(a), 0.0)


def _norm(x: DeviceState) -> float:
    v = N.dbl()
    N.call("hsv_state_norm", x.handle, N.C.byref(v))
    return v.value


def lanczos_ground_energy(op: PauliOperator, tol: float = 1e-11, max_iter: int = 200,
                          seed: int = 12345, max_vectors: int | None = None,
                          return_vector: bool = False):
    """Lowest eigenvalue of the sector Hamiltonian (real symmetric).

    Full re-orthogonalization (two classical Gram-Schmidt passes) against the
    stored Krylov basis; stops when the Ritz value changes by less than `tol`
    between checks.  `max_vectors` bounds device memory (dim x 16 B each).
    """
    basis = op.basis
    dim = len(basis)
    if dim == 0:
        raise ValueError("empty sector")
    max_vectors = max_vectors or max_iter
    v0 = np.random.default_rng(seed).standard_normal(dim)
    v0 /= np.linalg.norm(v0)
    from .sparse import SparseVector
    q = DeviceState.from_sparse(basis, SparseVector(dim, np.arange(dim, dtype=np.int64), v0))
    Q = [q]
    alphas, betas = [], []
    prev = None
    theta = None
    for it in range(min(max_iter, dim, max_vectors)):
        w = DeviceState(basis)
        N.call("hsv_apply_h", op.handle, Q[-1].handle, w.handle, 0.0)
        a = Q[-1].dot(w).real
        alphas.append(a)
        _axpy(-a, Q[-1], w)
        if betas:
            _axpy(-betas[-1], Q[-2], w)
        for _ in range(2):                      # full re-orthogonalization
            for qq in Q:
                c = qq.dot(w).real
                if c != 0.0:
                    _axpy(-c, qq, w)
        b = _norm(w)
        T_evals = scipy.linalg.eigh_tridiagonal(np.array(alphas), np.array(betas),
                                                eigvals_only=True, select="i",
                                                select_range=(0, 0))
        theta = float(T_evals[0])
        if (prev is not None and abs(theta - prev) < tol) or b < 1e-12:
            break
        prev = theta
        betas.append(b)
        _scale(w, 1.0 / b)
        Q.append(w)
    if not return_vector:
        return theta
    evals, evecs = scipy.linalg.eigh_tridiagonal(np.array(alphas), np.array(betas[:len(alphas) - 1]),
                                                 select="i", select_range=(0, 0))
    coeff = evecs[:, 0]
    vec = DeviceState(basis)
    for c, qq in zip(coeff, Q):
        _axpy(float(c), qq, vec)
    return float(evals[0]), vec
