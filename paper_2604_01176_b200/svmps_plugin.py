"""Drop-in plugin: run the UNMODIFIED reference package `svmps` on libhsv.

`install()` rebinds, in every loaded `svmps.*` module namespace, the SV-path
entry points to device-backed versions that take and return the reference's
own types:

* `svmps.adapt.SvAdaptEngine` -> `HsvSvAdaptEngine` (the engine protocol,
  adapt.py:179-220).  `make_engine` looks the name up at call time
  (adapt.py:355-356), so `run_adapt(AdaptConfig(engine="sv"), ...)`, the CLI
  and every test that builds an `SvAdaptEngine` run on the GPU.
* `svmps.svengine.{assemble_subspace_hamiltonian, expectation,
  apply_generator, apply_qeb_exponential, apply_ansatz, pool_gradient,
  pool_gradients, ansatz_energy_gradient}` (svengine.py:115-281).
  `assemble_subspace_hamiltonian` returns an `svmps.sparse.CsrMatrix`
  subclass around the matrix-free device operator; its CSR arrays are
  materialized on the device only when touched (`to_dense`, `save_csr`,
  `oracle.fci_ground_energy`).
* `svmps.sparse.{spmspv, dot, axpy, scale, norm, normalize}`
  (sparse.py:163-245): the generic CSR kernel K1b and the vector kernels.

Nothing falls back to the reference's numpy code: inputs the device engine
does not support (custom configuration lists, `CiBasis` not equal to a full
(n_alpha, n_beta) sector) raise `ValueError`, as the device API does.

`uninstall()` restores the originals.  For pytest, load
`paper_2604_01176_b200.svmps_pytest` with `-p` so the rebinding happens
before the test modules import the names (test_adapt.py:9-20 imports
`SvAdaptEngine` by name).
"""
from __future__ import annotations

import sys
import weakref

import numpy as np

from . import _native as N
from . import adapt as _ad
from . import sparse as _sp
from . import svengine as _sv
from .cibasis import CiBasis, Configuration
from .pauli import PauliSum
from .system import MolecularSystem

_SPARSE_NAMES = ("spmspv", "dot", "axpy", "scale", "norm", "normalize")
_SV_NAMES = ("assemble_subspace_hamiltonian", "expectation", "apply_generator",
             "apply_qeb_exponential", "apply_ansatz", "pool_gradient", "pool_gradients",
             "ansatz_energy_gradient")
_MODULES = ("svmps", "svmps.sparse", "svmps.svengine", "svmps.adapt", "svmps.partition",
            "svmps.oracle", "svmps.cli", "svmps.system", "svmps.mpsengine")

_saved: list = []               # (module, name, original) for uninstall()
_bases: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_ref = {}                       # reference classes, filled by install()


# ------------------------------------------------------------ conversions
def dev_basis(rb) -> CiBasis:
    """The device-side CiBasis of a reference CiBasis (cached per object)."""
    if isinstance(rb, CiBasis):
        return rb
    b = _bases.get(rb)
    if b is None:
        b = CiBasis(rb.n_qubits, rb.n_alpha, rb.n_beta, rb.ordering, np.asarray(rb.states))
        _bases[rb] = b
    return b


def dev_vec(v) -> _sp.SparseVector:
    if isinstance(v, _sp.SparseVector):
        return v
    return _sp.SparseVector(int(v.dim), np.asarray(v.indices, dtype=np.int64),
                            np.asarray(v.values))


def ref_vec(v):
    return _ref["SparseVector"](int(v.dim), v.indices, v.values)


def dev_state(s) -> _sv.SvState:
    if isinstance(s, _sv.SvState):
        return s
    return _sv.SvState(dev_basis(s.basis), dev_vec(s.vec))


def ref_state(ref_basis, s: _sv.SvState):
    return _ref["SvState"](ref_basis, ref_vec(s.vec))


def dev_config(hf, n_qubits: int) -> Configuration:
    return hf if isinstance(hf, Configuration) else Configuration(int(getattr(hf, "bits", hf)),
                                                                   n_qubits)


def dev_system(system) -> MolecularSystem:
    """Device-side MolecularSystem from a reference one: the reference's own
    PauliSum (already canonical: sorted by (x, z), merged; pauli.py:179-185),
    taken verbatim so every x-group sum runs in the reference's term order."""
    if isinstance(system, MolecularSystem):
        return system
    h = system.hamiltonian
    ph = PauliSum(h.n_qubits, np.asarray(h.xs), np.asarray(h.zs), np.asarray(h.coeffs),
                  _trusted=True)
    ints = system.integrals
    out = MolecularSystem.from_pauli(ph, int(ints.nelec), int(ints.ms2), system.ordering)
    out.hf = Configuration(int(system.hf.bits), ph.n_qubits)
    out._basis = dev_basis(system.basis)
    return out


def _is_dev_csr(m) -> bool:
    return isinstance(m, _ref.get("HsvCsrMatrix", ())) or isinstance(m, _sv.PauliOperator)


def _op(m) -> _sv.PauliOperator:
    return m.op if isinstance(m, _ref["HsvCsrMatrix"]) else m


def _make_csr_class(base):
    class HsvCsrMatrix(base):
        """`svmps.sparse.CsrMatrix` around the matrix-free device operator."""

        __slots__ = ("op", "ref_basis")

        def __init__(self, op: _sv.PauliOperator, ref_basis):
            self.n_rows = op.n_rows
            self.n_cols = op.n_cols
            self.op = op
            self.ref_basis = ref_basis

        row_offsets = property(lambda self: self.op.row_offsets)
        col_indices = property(lambda self: self.op.col_indices)
        values = property(lambda self: self.op.values)
        nnz = property(lambda self: self.op.nnz)

        def __repr__(self):
            return f"HsvCsrMatrix({self.n_rows}x{self.n_cols}, device operator)"

    return HsvCsrMatrix


# ------------------------------------------------------ sparse.py drop-ins
def spmspv(m, v, prune: float = 0.0, n_workers: int = 1):
    if m.n_cols != v.dim:
        raise ValueError(f"dimension mismatch: matrix {m.n_cols} columns, vector {v.dim}")
    if _is_dev_csr(m):
        return ref_vec(_op(m).apply_sparse(dev_vec(v), prune))
    return ref_vec(_sp.spmspv(m, dev_vec(v), prune, n_workers))


def dot(u, v) -> float:
    return _sp.dot(dev_vec(u), dev_vec(v))


def axpy(a, x, y, prune: float = 0.0):
    return ref_vec(_sp.axpy(a, dev_vec(x), dev_vec(y), prune))


def scale(a, x):
    return ref_vec(_sp.scale(a, dev_vec(x)))


def norm(x) -> float:
    return _sp.norm(dev_vec(x))


def normalize(x):
    return ref_vec(_sp.normalize(dev_vec(x)))


# ---------------------------------------------------- svengine.py drop-ins
def assemble_subspace_hamiltonian(h, basis):
    ph = h if isinstance(h, PauliSum) else PauliSum(
        h.n_qubits, np.asarray(h.xs), np.asarray(h.zs), np.asarray(h.coeffs), _trusted=True)
    op = _sv.assemble_subspace_hamiltonian(ph, dev_basis(basis))
    return _ref["HsvCsrMatrix"](op, basis)


def expectation(m, s, n_workers: int = 1) -> float:
    if _is_dev_csr(m):
        return _op(m).expect(dev_state(s))
    return dot(s.vec, spmspv(m, s.vec, n_workers=n_workers))


def apply_generator(op, s):
    return ref_vec(_sv.apply_generator(op, dev_state(s)))


def apply_qeb_exponential(op, theta, s):
    theta = float(theta)
    if theta == 0.0 or s.vec.nnz == 0:
        return s                                  # the reference returns its input (svengine.py:212)
    return ref_state(s.basis, _sv.apply_qeb_exponential(op, theta, dev_state(s)))


def apply_ansatz(basis, hf, ops, thetas):
    db = dev_basis(basis)
    return ref_state(basis, _sv.apply_ansatz(db, dev_config(hf, db.n_qubits), ops, thetas))


def pool_gradients(m, s, ops, n_workers: int = 1) -> np.ndarray:
    ops = list(ops)
    if _is_dev_csr(m):
        return _sv.pool_gradients(_op(m), dev_state(s), ops)
    w = spmspv(m, s.vec, n_workers=n_workers)
    return np.array([2.0 * dot(w, apply_generator(op, s)) for op in ops])


def pool_gradient(m, s, op, n_workers: int = 1) -> float:
    return float(pool_gradients(m, s, [op], n_workers)[0])


def ansatz_energy_gradient(m, basis, hf, ops, thetas, n_workers: int = 1):
    db = dev_basis(basis)
    cfg = dev_config(hf, db.n_qubits)
    if _is_dev_csr(m):
        return _sv.ansatz_energy_gradient(_op(m), db, cfg, list(ops), thetas)
    return _sv.ansatz_energy_gradient(m, db, cfg, list(ops), thetas, n_workers)


# ------------------------------------------------------- the engine (adapt.py)
class HsvSvAdaptEngine(_ad.SvAdaptEngine):
    """The device engine behind the reference's engine protocol (adapt.py:179-220).

    Keeps the engine name "sv" (AdaptConfig.validate rejects new names,
    adapt.py:130-132).  States it returns are device-resident `SvState`s;
    states handed in by a caller (reference `SvState`) are uploaded."""

    name = "sv"
    uses_coordinate_search = False

    def __init__(self, system, config):
        super().__init__(dev_system(system), config)
        self.ref_system = system

    def apply(self, state, op, theta, log=None):
        return _sv.apply_qeb_exponential(op, theta, dev_state(state))

    def energy(self, state) -> float:
        return super().energy(dev_state(state))

    def screen(self, state, pool) -> np.ndarray:
        return super().screen(dev_state(state), pool)

    def energy_and_screen(self, state, pool):
        return super().energy_and_screen(dev_state(state), pool)


# ------------------------------------------------------------ installation
def installed() -> bool:
    return bool(_saved)


def install(verbose: bool = False) -> None:
    """Rebind the reference's SV path to libhsv (idempotent)."""
    if _saved:
        return
    import importlib
    N.load()                                     # fail loudly without the CUDA library
    mods = {}
    for name in _MODULES:
        try:
            mods[name] = importlib.import_module(name)
        except ImportError:
            if name in ("svmps", "svmps.sparse", "svmps.svengine", "svmps.adapt"):
                raise
    ref_sparse, ref_sv, ref_adapt = mods["svmps.sparse"], mods["svmps.svengine"], mods["svmps.adapt"]
    _ref["SparseVector"] = ref_sparse.SparseVector
    _ref["SvState"] = ref_sv.SvState
    _ref["HsvCsrMatrix"] = _make_csr_class(ref_sparse.CsrMatrix)
    this = sys.modules[__name__]
    table = {}
    for n in _SPARSE_NAMES:
        table[n] = (getattr(ref_sparse, n), getattr(this, n))
    for n in _SV_NAMES:
        if hasattr(ref_sv, n):
            table[n] = (getattr(ref_sv, n), getattr(this, n))
    table["SvAdaptEngine"] = (ref_adapt.SvAdaptEngine, HsvSvAdaptEngine)
    for mname, mod in list(sys.modules.items()):
        if mod is None or not (mname == "svmps" or mname.startswith("svmps.")):
            continue
        for n, (orig, new) in table.items():
            if getattr(mod, n, None) is orig:
                _saved.append((mod, n, orig))
                setattr(mod, n, new)
    if verbose:
        print(f"svmps_plugin: {len(_saved)} bindings -> libhsv", file=sys.stderr)


def uninstall() -> None:
    while _saved:
        mod, n, orig = _saved.pop()
        setattr(mod, n, orig)
