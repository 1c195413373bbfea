"""Exact sparse state-vector engine on the device (drop-in for `svmps.svengine`).

Same names, argument meaning and error behaviour as the reference module
(svengine.py:1-311); the work is done by libhsv:

* `assemble_subspace_hamiltonian` returns a matrix-free `PauliOperator`
  (x-grouped term tables on the device) instead of assembling a CSR; the
  reference's validation (odd-Y words, sector leak) runs on the device.  The
  operator is still a `CsrMatrix`: its CSR arrays are materialized lazily,
  on the device, only if a caller touches them (`to_dense`, `row_offsets`...).
* `SvState` keeps its amplitudes resident on the device (complex128,
  alpha-string-major); `.vec` materializes the reference `SparseVector` on
  demand (ascending positions, exact zeros dropped).
* `apply_qeb_exponential`, `apply_generator`, `expectation`,
  `pool_gradient(s)` and `ansatz_energy_gradient` call the K1-K5 kernels.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .cibasis import CiBasis, Configuration
from .pauli import PauliSum
from .sparse import CsrMatrix, SparseVector, dot, norm, spmspv  # noqa: F401 (norm: svengine namespace)

# the reference declares this chunk size but never reads it (svengine.py:29);
# kept for namespace parity -- the matrix-free operator needs no assembly chunks
ASSEMBLY_CHUNK_ENTRIES = 4_000_000

NORM_DRIFT_TOL = 1e-9
SECTOR_LEAK_TOL = 1e-10


@dataclass(frozen=True)
class ExcitationOperator:
    """Spin-conserving single or double qubit excitation (svengine.py:32-76)."""

    kind: str
    occ: tuple
    virt: tuple

    def __post_init__(self):
        expected = {"single": 1, "double": 2}.get(self.kind)
        if expected is None:
            raise ValueError(f"unknown excitation kind {self.kind!r}")
        if len(self.occ) != expected or len(self.virt) != expected:
            raise ValueError("index count does not match the excitation kind")
        object.__setattr__(self, "occ", tuple(sorted(int(q) for q in self.occ)))
        object.__setattr__(self, "virt", tuple(sorted(int(q) for q in self.virt)))
        if len(set(self.occ) | set(self.virt)) != 2 * expected:
            raise ValueError("excitation indices must be distinct")

    @property
    def occ_mask(self) -> int:
        return sum(1 << q for q in self.occ)

    @property
    def virt_mask(self) -> int:
        return sum(1 << q for q in self.virt)

    @property
    def flip_mask(self) -> int:
        return self.occ_mask | self.virt_mask

    def label(self) -> str:
        return f"{self.kind[0]}:{','.join(map(str, self.occ))}->{','.join(map(str, self.virt))}"

    def __repr__(self) -> str:
        return f"ExcitationOperator({self.label()})"


@dataclass(frozen=True)
class AnsatzElement:
    op: ExcitationOperator
    theta: float

    def __post_init__(self):
        if not np.isfinite(self.theta):
            raise ValueError("ansatz angle must be finite")


# ------------------------------------------------------------ device state
class DeviceState:
    """Owner of an `hsv_state` (dense complex128 amplitudes over a sector)."""

    __slots__ = ("basis", "handle", "_sector_ref", "__weakref__")

    def __init__(self, basis: CiBasis):
        sec = basis.sector
        self.basis = basis
        self._sector_ref = basis._sector        # keep the sector alive
        h = N.C.c_void_p()
        N.call("hsv_state_create", sec, N.C.byref(h))
        self.handle = h

    def __del__(self):
        try:
            if self.handle:
                N.lib().hsv_state_destroy(self.handle)
        except Exception:
            pass

    @classmethod
    def from_sparse(cls, basis: CiBasis, vec: SparseVector) -> "DeviceState":
        if vec.dim != len(basis):
            raise ValueError(f"dimension mismatch: vector {vec.dim}, basis {len(basis)}")
        st = cls(basis)
        idx = N.as_i64(vec.indices)
        if np.iscomplexobj(vec.values):
            re, im = N.as_f64(vec.values.real), N.as_f64(vec.values.imag)
            pim = N.ptr_f64(im)
        else:
            re, pim = N.as_f64(vec.values), None
        if idx.size == vec.dim and idx.size and idx[0] == 0 and idx[-1] == vec.dim - 1:
            # SparseVector indices are ascending and unique, so a full support is
            # every position in order: send the values only
            N.call("hsv_state_set_dense", st.handle, N.ptr_f64(re), pim)
        else:
            N.call("hsv_state_set_sparse", st.handle, N.ptr_i64(idx), N.ptr_f64(re), pim,
                   idx.size)
        return st

    @classmethod
    def basis_state(cls, basis: CiBasis, bits: int) -> "DeviceState":
        st = cls(basis)
        N.call("hsv_state_set_basis", st.handle, int(bits), 1.0, 0.0)
        return st

    def copy(self) -> "DeviceState":
        out = DeviceState(self.basis)
        N.call("hsv_state_copy", out.handle, self.handle)
        return out

    def nnz(self) -> int:
        n = N.i64()
        N.call("hsv_state_nnz", self.handle, N.C.byref(n))
        return n.value

    def at_positions(self, positions) -> np.ndarray:
        """Amplitudes at reference positions (zero outside the support)."""
        pos = N.as_i64(positions)
        re = np.empty(pos.size)
        im = np.empty(pos.size)
        N.call("hsv_state_get_positions", self.handle, N.ptr_i64(pos), pos.size, N.ptr_f64(re),
               N.ptr_f64(im))
        return re if not np.any(im) else re + 1j * im

    @property
    def __cuda_array_interface__(self):
        ptr, n = N.C.c_void_p(), N.i64()
        N.call("hsv_state_device_ptr", self.handle, N.C.byref(ptr), N.C.byref(n))
        return {"shape": (n.value, 2), "typestr": "<f8", "data": (ptr.value or 0, False),
                "version": 3, "strides": None}

    def torch_view(self):
        """Zero-copy torch float64 [dim, 2] view of the (alpha-major) amplitudes, for
        collectives issued by the host; writes through it invalidate cached norms."""
        import torch
        return torch.as_tensor(self, device="cuda")

    def dot(self, other: "DeviceState") -> complex:
        re, im = N.dbl(), N.dbl()
        N.call("hsv_state_dot", self.handle, other.handle, N.C.byref(re), N.C.byref(im))
        return complex(re.value, im.value)

    def to_sparse(self, prune: float = 0.0) -> SparseVector:
        n = N.i64()
        N.call("hsv_state_get_sparse", self.handle, float(prune), None, None, None, 0, N.C.byref(n))
        cnt = n.value
        pos = np.empty(cnt, dtype=np.int64)
        re = np.empty(cnt)
        im = np.empty(cnt)
        if cnt:
            N.call("hsv_state_get_sparse", self.handle, float(prune), N.ptr_i64(pos),
                   N.ptr_f64(re), N.ptr_f64(im), cnt, N.C.byref(n))
        vals = re if not np.any(im) else re + 1j * im
        return SparseVector(len(self.basis), pos, vals)


class SvState:
    """Sparse state over a CI basis (svengine.py:89-109), device resident."""

    __slots__ = ("basis", "_vec", "_dev")

    def __init__(self, basis: CiBasis, vec: SparseVector | None = None, *, _dev=None):
        if vec is None and _dev is None:
            raise ValueError("SvState needs a vector")
        if vec is not None and vec.dim != len(basis):
            raise ValueError(f"dimension mismatch: vector {vec.dim}, basis {len(basis)}")
        self.basis = basis
        self._vec = vec
        self._dev = _dev

    @classmethod
    def from_configuration(cls, basis: CiBasis, c) -> "SvState":
        bits = c.bits if isinstance(c, Configuration) else int(c)
        if basis.is_custom:
            pos = basis.index_of(bits)
            if pos is None:
                raise ValueError(f"configuration {Configuration(bits, basis.n_qubits).ket()} "
                                 "is outside the basis sector")
            return cls(basis, SparseVector.basis_state(len(basis), pos))
        am, bm = basis.alpha_mask, basis.beta_mask
        if ((bits & am).bit_count() != basis.n_alpha or (bits & bm).bit_count() != basis.n_beta
                or bits >> basis.n_qubits):
            raise ValueError(f"configuration {Configuration(bits, basis.n_qubits).ket()} "
                             "is outside the basis sector")
        return cls(basis, _dev=DeviceState.basis_state(basis, bits))

    @property
    def device(self) -> DeviceState:
        if self._dev is None:
            self._dev = DeviceState.from_sparse(self.basis, self._vec)
        return self._dev

    @property
    def vec(self) -> SparseVector:
        if self._vec is None:
            self._vec = self._dev.to_sparse()
        return self._vec

    @property
    def nnz(self) -> int:
        return self._vec.nnz if self._vec is not None else self._dev.nnz()

    def configurations(self) -> np.ndarray:
        return self.basis.states[self.vec.indices]

    def __repr__(self) -> str:
        return f"SvState(dim={len(self.basis)}, nnz={self.nnz})"


class DevicePool:
    """Operator pool resident on the device (compressed occ/virt masks)."""

    __slots__ = ("basis", "handle", "n", "ops", "_sector_ref")

    def __init__(self, basis: CiBasis, ops):
        self.ops = tuple(ops)
        self.basis = basis
        self._sector_ref = None
        occ = np.array([o.occ_mask for o in self.ops], dtype=np.uint64)
        virt = np.array([o.virt_mask for o in self.ops], dtype=np.uint64)
        sec = basis.sector
        self._sector_ref = basis._sector
        h = N.C.c_void_p()
        N.call("hsv_pool_create", sec, N.ptr_u64(occ), N.ptr_u64(virt), occ.size, N.C.byref(h))
        self.handle = h
        self.n = occ.size

    def __del__(self):
        try:
            if self.handle:
                N.lib().hsv_pool_destroy(self.handle)
        except Exception:
            pass


# --------------------------------------------------------------- operator
class PauliOperator(CsrMatrix):
    """Matrix-free subspace Hamiltonian <b_i|H|b_j> (device x-grouped tables).

    A `CsrMatrix` whose arrays are materialized on first access; `nnz` is
    counted on the device without materializing.
    """

    __slots__ = ("basis", "hamiltonian", "handle", "_sector_ref", "_csr", "_nnz")

    def __init__(self, h: PauliSum, basis: CiBasis):
        self.n_rows = self.n_cols = len(basis)
        self.basis = basis
        self.hamiltonian = h
        self._csr = None
        self._nnz = None
        sec = basis.sector
        self._sector_ref = basis._sector
        xs, zs, cs = N.as_i64(h.xs), N.as_i64(h.zs), N.as_f64(h.coeffs)
        hd = N.C.c_void_p()
        N.call("hsv_op_create", sec, h.n_qubits, N.ptr_i64(xs), N.ptr_i64(zs), N.ptr_f64(cs),
               cs.size, N.C.byref(hd))
        self.handle = hd

    def __del__(self):
        try:
            if self.handle:
                N.lib().hsv_op_destroy(self.handle)
        except Exception:
            pass

    def info(self) -> dict:
        t, g, a = N.i64(), N.i64(), N.i64()
        N.call("hsv_op_info", self.handle, N.C.byref(t), N.C.byref(g), N.C.byref(a))
        return {"n_terms": t.value, "n_groups": g.value, "n_active_groups": a.value}

    def _materialize(self):
        if self._csr is None:
            nnz = self.nnz
            ro = np.empty(self.n_rows + 1, dtype=np.int64)
            cols = np.empty(max(nnz, 1), dtype=np.int64)
            vals = np.empty(max(nnz, 1))
            N.call("hsv_op_to_csr", self.handle, N.ptr_i64(ro), N.ptr_i64(cols), N.ptr_f64(vals), nnz)
            self._csr = (ro, cols[:nnz], vals[:nnz])
        return self._csr

    @property
    def row_offsets(self):
        return self._materialize()[0]

    @property
    def col_indices(self):
        return self._materialize()[1]

    @property
    def values(self):
        return self._materialize()[2]

    @property
    def nnz(self) -> int:
        if self._nnz is None:
            n = N.i64()
            N.call("hsv_op_count_nnz", self.handle, N.C.byref(n))
            self._nnz = n.value
        return self._nnz

    # ---- device compute ----
    def apply_state(self, s: "SvState", prune: float = 0.0) -> DeviceState:
        out = DeviceState(self.basis)
        N.call("hsv_apply_h", self.handle, s.device.handle, out.handle, float(prune))
        return out

    def apply_sparse(self, v: SparseVector, prune: float = 0.0) -> SparseVector:
        return self.apply_state(SvState(self.basis, v), prune).to_sparse()

    def expect(self, s: "SvState") -> float:
        re, im = N.dbl(), N.dbl()
        N.call("hsv_expect_h", self.handle, s.device.handle, N.C.byref(re), N.C.byref(im))
        return float(re.value)

    def energy_screen(self, s: "SvState", occ_masks, virt_masks) -> tuple[float, np.ndarray]:
        occ, virt = N.as_u64(occ_masks), N.as_u64(virt_masks)
        g = np.empty(occ.size)
        e = N.dbl()
        N.call("hsv_energy_screen", self.handle, s.device.handle, N.ptr_u64(occ),
               N.ptr_u64(virt), occ.size, N.C.byref(e), N.ptr_f64(g))
        return float(e.value), g

    def energy_screen_pool(self, s: "SvState", pool: "DevicePool") -> tuple[float, np.ndarray]:
        g = np.empty(pool.n)
        e = N.dbl()
        N.call("hsv_energy_screen_pool", self.handle, s.device.handle, pool.handle,
               N.C.byref(e), N.ptr_f64(g))
        return float(e.value), g

    def energy_gradient(self, hf_bits: int, occ_masks, virt_masks, thetas):
        occ, virt = N.as_u64(occ_masks), N.as_u64(virt_masks)
        th = N.as_f64(thetas)
        cs, sn = N.as_f64(np.cos(th)), N.as_f64(np.sin(th))
        g = np.empty(th.size)
        e = N.dbl()
        N.call("hsv_energy_gradient", self.handle, int(hf_bits), N.ptr_u64(occ), N.ptr_u64(virt),
               N.ptr_f64(cs), N.ptr_f64(sn), th.size, N.C.byref(e), N.ptr_f64(g))
        return float(e.value), g

    def __repr__(self) -> str:
        return f"PauliOperator({self.n_rows}x{self.n_cols}, terms={len(self.hamiltonian)})"


def assemble_subspace_hamiltonian(h: PauliSum, basis: CiBasis) -> CsrMatrix:
    """Subspace Hamiltonian (svengine.py:115-171), matrix-free on the device."""
    if h.n_qubits != basis.n_qubits:
        raise ValueError("Pauli sum and basis disagree on qubit count")
    if basis.is_custom:
        raise ValueError("the device engine needs a full (n_alpha, n_beta) sector; "
                         "custom configuration lists are not supported")
    return PauliOperator(h, basis)


def _state_of(m, s: SvState) -> SvState:
    if isinstance(m, PauliOperator) and s.basis is not m.basis:
        return SvState(m.basis, s.vec)
    return s


def expectation(m: CsrMatrix, s: SvState, n_workers: int = 1) -> float:
    """<psi|m|psi> (svengine.py:174-176)."""
    if isinstance(m, PauliOperator):
        return m.expect(_state_of(m, s))
    return dot(s.vec, spmspv(m, s.vec, n_workers=n_workers))


def apply_generator(op: ExcitationOperator, s: SvState) -> SparseVector:
    """T|psi> (svengine.py:187-206)."""
    if s.basis.is_custom:
        raise ValueError("custom bases are not supported by the device engine")
    out = DeviceState(s.basis)
    N.call("hsv_apply_generator", s.device.handle, out.handle, op.occ_mask, op.virt_mask)
    return out.to_sparse()


def apply_qeb_exponential(op: ExcitationOperator, theta: float, s: SvState) -> SvState:
    """exp(theta T)|psi> as Givens rotations on the device (svengine.py:209-237)."""
    theta = float(theta)
    if theta == 0.0 or s.nnz == 0:
        return s
    c, sn = np.cos(theta), np.sin(theta)          # host trig, as svengine.py:219
    out = DeviceState(s.basis)
    N.call("hsv_apply_qeb", s.device.handle, out.handle, op.occ_mask, op.virt_mask,
           float(c), float(sn))
    return SvState(s.basis, _dev=out)


def apply_ansatz(basis: CiBasis, hf: Configuration, ops, thetas) -> SvState:
    """HF reference followed by the ansatz rotations (svengine.py:240-244): one fused
    device sweep (hsv_ansatz_state), bitwise equal to rotating one operator at a time."""
    ops = list(ops)
    th = np.asarray([float(t) for t in thetas], dtype=np.float64)
    n = min(len(ops), th.size)                  # zip() semantics
    occ, virt = _masks(ops[:n])
    th = np.ascontiguousarray(th[:n])
    cs, sn = N.as_f64(np.cos(th)), N.as_f64(np.sin(th))
    dev = DeviceState(basis)
    N.call("hsv_ansatz_state", basis.sector, int(hf.bits), N.ptr_u64(occ), N.ptr_u64(virt),
           N.ptr_f64(cs), N.ptr_f64(sn), n, dev.handle)
    return SvState(basis, _dev=dev)


def _masks(ops):
    ops = list(ops)
    return (np.array([o.occ_mask for o in ops], dtype=np.uint64),
            np.array([o.virt_mask for o in ops], dtype=np.uint64))


def pool_gradient(m: CsrMatrix, s: SvState, op: ExcitationOperator, n_workers: int = 1) -> float:
    """dE/dtheta at theta = 0 for exp(theta T) (svengine.py:247-250)."""
    return float(pool_gradients(m, s, [op], n_workers)[0])


def pool_gradients(m: CsrMatrix, s: SvState, ops, n_workers: int = 1) -> np.ndarray:
    """Whole-pool gradients, H|psi> computed once (svengine.py:253-257)."""
    ops = list(ops)
    if isinstance(m, PauliOperator):
        occ, virt = _masks(ops)
        return m.energy_screen(_state_of(m, s), occ, virt)[1]
    w = spmspv(m, s.vec, n_workers=n_workers)
    return np.array([2.0 * dot(w, apply_generator(op, s)) for op in ops])


def ansatz_energy_gradient(m: CsrMatrix, basis: CiBasis, hf: Configuration, ops, thetas,
                           n_workers: int = 1):
    """Energy and analytic gradient by one adjoint sweep (svengine.py:260-281)."""
    thetas = np.asarray(thetas, dtype=np.float64)
    ops = list(ops)
    if isinstance(m, PauliOperator):
        occ, virt = _masks(ops)
        hf_bits = hf.bits if isinstance(hf, Configuration) else int(hf)
        return m.energy_gradient(hf_bits, occ, virt, thetas)
    # generic CSR: the reference algorithm with device primitives
    states = [SvState.from_configuration(basis, hf)]
    for op, th in zip(ops, thetas):
        states.append(apply_qeb_exponential(op, float(th), states[-1]))
    psi = states[-1]
    w = spmspv(m, psi.vec, n_workers=n_workers)
    energy = dot(psi.vec, w)
    grad = np.zeros(len(ops))
    lam = SvState(basis, w)
    for i in range(len(ops) - 1, -1, -1):
        grad[i] = 2.0 * dot(lam.vec, apply_generator(ops[i], states[i + 1]))
        lam = apply_qeb_exponential(ops[i], -float(thetas[i]), lam)
    return energy, grad


# ---------------------------------------------------- CSR binary cache
_CSR_MAGIC = b"SVMPSCSR"
_CSR_VERSION = 1


def save_csr(path, m: CsrMatrix) -> None:
    """Little-endian SVMPSCSR v1 cache (svengine.py:284-292); materializes m."""
    with open(path, "wb") as fh:
        fh.write(_CSR_MAGIC)
        fh.write(struct.pack("<IQQQ", _CSR_VERSION, m.n_rows, m.n_cols, m.nnz))
        fh.write(np.asarray(m.row_offsets).astype("<i8").tobytes())
        fh.write(np.asarray(m.col_indices).astype("<i8").tobytes())
        fh.write(np.asarray(m.values).astype("<f8").tobytes())


def load_csr(path) -> CsrMatrix:
    with open(path, "rb") as fh:
        if fh.read(len(_CSR_MAGIC)) != _CSR_MAGIC:
            raise ValueError("not a CSR cache file")
        version, n_rows, n_cols, nnz = struct.unpack("<IQQQ", fh.read(28))
        if version != _CSR_VERSION:
            raise ValueError(f"unsupported CSR cache version {version}")
        ro = np.frombuffer(fh.read(8 * (n_rows + 1)), dtype="<i8")
        ci = np.frombuffer(fh.read(8 * nnz), dtype="<i8")
        va = np.frombuffer(fh.read(8 * nnz), dtype="<f8")
    m = CsrMatrix(n_rows, n_cols, ro.copy(), ci.copy(), va.copy())
    m.validate()
    return m
