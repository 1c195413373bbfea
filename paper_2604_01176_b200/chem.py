"""Molecular Hamiltonian build on the host: FCIDUMP -> spin orbitals -> Jordan-Wigner.

SURVEY.md section 8f, rank 4 ("device-side Hamiltonian build") -- the setup path
the reference runs in `svmps.fcidump` / `svmps.mapping` (fcidump.py:73-148,
mapping.py:48-126), re-implemented so the package can build Pauli sums for new
molecules without the reference installed.  Conventions are the reference's:

* FCIDUMP (Molpro): header NORB / NELEC / MS2, then `value i j k l` lines with
  1-based indices; (0,0,0,0) = core energy, k = l = 0 one-body, else chemists'
  (ij|kl) with 8-fold symmetry.
* spin orbitals: interleaved (2p + s) or blocked (p + s * norb) qubits;
  H = E_core + sum h[P,Q] a+_P a_Q + 1/2 sum g[P,Q,R,S] a+_P a+_R a_S a_Q.
* Jordan-Wigner: a+_p = Z_0..Z_{p-1} (X_p - i Y_p)/2, qubit 0 least significant;
  imaginary residues above 1e-12 are rejected, |c| <= 1e-12 dropped.

The JW expansion is vectorized: every product of k ladder operators expands to
2^k symplectic words, all evaluated with numpy, and equal words are merged with
a single unique/add.at.  Parity with the reference builder: same word set and
coefficients to ~1e-14 (the summation order of merged words differs), checked
against the bundled Pauli sums in tests/test_chem.py.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

from .cibasis import check_ordering, hartree_fock_configuration, qubit_index
from .pauli import PauliSum

JW_DROP_TOL = 1e-12
JW_IMAG_TOL = 1e-12


@dataclass
class IntegralSet:
    norb: int
    nelec: int
    ms2: int
    core_energy: float = 0.0
    one_body: np.ndarray = field(default=None)
    two_body: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.one_body is None:
            self.one_body = np.zeros((self.norb, self.norb))
        if self.two_body is None:
            self.two_body = np.zeros((self.norb,) * 4)
        if self.norb < 1 or not 0 <= self.nelec <= 2 * self.norb:
            raise ValueError("invalid NORB / NELEC")
        if np.max(np.abs(self.one_body - self.one_body.T), initial=0.0) > 1e-12:
            raise ValueError("one-body integrals are not symmetric")

    @property
    def n_alpha(self) -> int:
        return (self.nelec + self.ms2) // 2

    @property
    def n_beta(self) -> int:
        return (self.nelec - self.ms2) // 2


_KEY = re.compile(r"\b(NORB|NELEC|MS2)\s*=\s*(-?\d+)", re.IGNORECASE)


def parse_fcidump(text: str) -> IntegralSet:
    """Parse FCIDUMP text (Molpro conventions)."""
    end = re.search(r"(&END|/)\s*$", text, re.IGNORECASE | re.MULTILINE)
    if end is None:
        raise ValueError("FCIDUMP header not terminated by &END or /")
    header, body = text[:end.start()], text[end.end():]
    vals = {k.upper(): int(v) for k, v in _KEY.findall(header)}
    for k in ("NORB", "NELEC"):
        if k not in vals:
            raise ValueError(f"FCIDUMP header lacks {k}")
    norb = vals["NORB"]
    rows = np.array([ln.split() for ln in body.splitlines() if ln.strip()], dtype=object)
    h = np.zeros((norb, norb))
    g = np.zeros((norb,) * 4)
    core = 0.0
    for r in rows:
        v = float(str(r[0]).replace("D", "E").replace("d", "e"))
        i, j, k, l = (int(x) for x in r[1:5])
        if i == j == k == l == 0:
            core = v
        elif k == 0 and l == 0:
            h[i - 1, j - 1] = h[j - 1, i - 1] = v
        else:
            i, j, k, l = i - 1, j - 1, k - 1, l - 1
            for a, b, c, d in ((i, j, k, l), (j, i, k, l), (i, j, l, k), (j, i, l, k),
                               (k, l, i, j), (l, k, i, j), (k, l, j, i), (l, k, j, i)):
                g[a, b, c, d] = v
    return IntegralSet(norb, vals["NELEC"], vals.get("MS2", 0), core, h, g)


def load_fcidump(path) -> IntegralSet:
    with open(path, encoding="ascii") as fh:
        return parse_fcidump(fh.read())


def spin_orbital_tables(ints: IntegralSet, ordering: str = "interleaved"):
    """(h[P,Q], g[P,Q,R,S]) over 2*norb spin orbitals; spin-forbidden entries 0."""
    check_ordering(ordering)
    n = 2 * ints.norb
    idx = [np.array([qubit_index(p, s, n, ordering) for p in range(ints.norb)]) for s in (0, 1)]
    h = np.zeros((n, n))
    g = np.zeros((n,) * 4)
    for s in (0, 1):
        h[np.ix_(idx[s], idx[s])] = ints.one_body
    for s1 in (0, 1):
        for s2 in (0, 1):
            g[np.ix_(idx[s1], idx[s1], idx[s2], idx[s2])] = ints.two_body
    return h, g


def _ladder_words(p: np.ndarray, dagger: bool):
    """JW image of a+_p / a_p as two symplectic words each: (x, z, coeff) arrays
    of shape [m, 2] for m operators."""
    x = (np.int64(1) << p.astype(np.int64))
    zs = x - 1                                     # Z string on qubits below p
    X = np.stack([x, x], axis=1)
    Z = np.stack([zs, zs | x], axis=1)             # X_p then Y_p (= i X Z in XZ form)
    C = np.empty(X.shape, dtype=np.complex128)
    C[:, 0] = 0.5
    C[:, 1] = -0.5j if dagger else 0.5j
    return X, Z, C


def _popcount(a: np.ndarray) -> np.ndarray:
    return np.bitwise_count(a.astype(np.uint64)).astype(np.int64)


def _product(factors, scale: np.ndarray):
    """Expand products of ladder operators (one product per row) into words."""
    X = np.zeros((scale.size, 1), dtype=np.int64)
    Z = np.zeros_like(X)
    C = scale.astype(np.complex128)[:, None]
    for fx, fz, fc in factors:
        # (x1, z1) (x2, z2) = i^k (x1^x2, z1^z2), words in i^{|x&z|} X^x Z^z form
        x1, z1, c1 = X[:, :, None], Z[:, :, None], C[:, :, None]
        x2, z2, c2 = fx[:, None, :], fz[:, None, :], fc[:, None, :]
        x3, z3 = x1 ^ x2, z1 ^ z2
        k = (_popcount(x1 & z1) + _popcount(x2 & z2) - _popcount(x3 & z3)
             + 2 * _popcount(z1 & x2)) % 4
        phase = np.array([1, 1j, -1, -1j])[k]
        X = x3.reshape(scale.size, -1)
        Z = z3.reshape(scale.size, -1)
        C = (c1 * c2 * phase).reshape(scale.size, -1)
    return X.ravel(), Z.ravel(), C.ravel()


@dataclass
class SecondQuantizedHamiltonian:
    """Spin-orbital coefficient tables, plain chemists' two-body form
    (the reference's `mapping.py:33-45`)."""

    n_spin_orbitals: int
    core_energy: float
    h: np.ndarray
    g: np.ndarray
    ordering: str
    convention: str = "chemists-plain"

    def validate(self):
        if np.max(np.abs(self.h - self.h.T), initial=0.0) > 1e-12:
            raise ValueError("one-body spin-orbital table is not symmetric")


def to_spin_orbital(ints: IntegralSet, ordering: str = "interleaved") -> SecondQuantizedHamiltonian:
    """Spatial integrals over 2*norb spin orbitals (reference `mapping.py:48-76`)."""
    h, g = spin_orbital_tables(ints, ordering)
    sq = SecondQuantizedHamiltonian(n_spin_orbitals=2 * ints.norb, core_energy=ints.core_energy,
                                    h=h, g=g, ordering=ordering)
    sq.validate()
    return sq


def hartree_fock_reference(n_electrons: int, n_qubits: int, ordering: str = "interleaved",
                           ms2: int = 0):
    """HF determinant (reference `mapping.py:129-132`)."""
    return hartree_fock_configuration(n_electrons, n_qubits, ordering, ms2)


def jordan_wigner(h, g=None, core_energy: float | None = None, n: int | None = None,
                  drop_tol: float = JW_DROP_TOL) -> PauliSum:
    """JW image of H.  Called as the reference does, `jordan_wigner(sq, drop_tol)`
    (`mapping.py:102`), or on the raw tables `jordan_wigner(h, g, core_energy, n)`."""
    if isinstance(h, SecondQuantizedHamiltonian):
        if isinstance(g, float):        # positional drop_tol, as in the reference
            drop_tol, g = g, None
        return _jordan_wigner_tables(h.h, h.g, h.core_energy, h.n_spin_orbitals, drop_tol)
    return _jordan_wigner_tables(h, g, core_energy, n, drop_tol)


def _jordan_wigner_tables(h: np.ndarray, g: np.ndarray, core_energy: float, n: int,
                          drop_tol: float = JW_DROP_TOL) -> PauliSum:
    xs, zs, cs = [np.array([0])], [np.array([0])], [np.array([complex(core_energy)])]
    p, q = np.nonzero(h)
    if p.size:
        X, Z, C = _product((_ladder_words(p, True), _ladder_words(q, False)), h[p, q])
        xs.append(X); zs.append(Z); cs.append(C)
    P, Q, R, S = np.nonzero(g)
    for lo in range(0, P.size, 200_000):          # bounded memory (16 words per product)
        sl = slice(lo, lo + 200_000)
        X, Z, C = _product((_ladder_words(P[sl], True), _ladder_words(R[sl], True),
                            _ladder_words(S[sl], False), _ladder_words(Q[sl], False)),
                           0.5 * g[P[sl], Q[sl], R[sl], S[sl]])
        xs.append(X); zs.append(Z); cs.append(C)
    x, z, c = np.concatenate(xs), np.concatenate(zs), np.concatenate(cs)
    keys, inv = np.unique(np.stack([x, z], axis=1), axis=0, return_inverse=True)
    acc = np.zeros(len(keys), dtype=np.complex128)
    np.add.at(acc, inv.ravel(), c)
    if np.max(np.abs(acc.imag), initial=0.0) > JW_IMAG_TOL:
        raise ValueError(f"residual imaginary Pauli coefficient "
                         f"{np.max(np.abs(acc.imag)):.3e}; input is not Hermitian")
    keep = np.abs(acc.real) > drop_tol
    return PauliSum(n, keys[keep, 0], keys[keep, 1], acc.real[keep])


def jordan_wigner_device(h, g=None, core_energy: float | None = None, n: int | None = None,
                         drop_tol: float = JW_DROP_TOL) -> PauliSum:
    """JW image built on the device (hsv_jordan_wigner, csrc/hsv_jw.cu): the products
    are expanded and merged in the reference's order (mapping.py:79-126), so the
    coefficients are bit-identical to its dict accumulation.  Same call forms as
    `jordan_wigner`."""
    from . import _native as N
    if isinstance(h, SecondQuantizedHamiltonian):
        if isinstance(g, float):
            drop_tol, g = g, None
        h, g, core_energy, n = h.h, h.g, h.core_energy, h.n_spin_orbitals
    hh = np.ascontiguousarray(h, dtype=np.float64)
    gg = np.ascontiguousarray(g, dtype=np.float64)
    N.init()
    cnt = N.i64()
    N.call("hsv_jordan_wigner", int(n), N.ptr_f64(hh), N.ptr_f64(gg), float(core_energy),
           float(drop_tol), None, None, None, 0, N.C.byref(cnt))
    m = cnt.value
    xs = np.empty(m, dtype=np.int64)
    zs = np.empty(m, dtype=np.int64)
    cs = np.empty(m)
    N.call("hsv_jordan_wigner", int(n), N.ptr_f64(hh), N.ptr_f64(gg), float(core_energy),
           float(drop_tol), N.ptr_i64(xs), N.ptr_i64(zs), N.ptr_f64(cs), m, N.C.byref(cnt))
    return PauliSum(int(n), xs, zs, cs, _trusted=True)


def molecular_system(ints: IntegralSet, ordering: str = "interleaved"):
    """MolecularSystem from integrals (mirrors MolecularSystem.from_integrals, system.py:33-37)."""
    from .system import IntegralInfo, MolecularSystem
    sq = to_spin_orbital(ints, ordering)
    ham = jordan_wigner(sq)
    hf = hartree_fock_reference(ints.nelec, sq.n_spin_orbitals, ordering, ints.ms2)
    return MolecularSystem(integrals=IntegralInfo(ints.norb, ints.nelec, ints.ms2),
                           ordering=ordering, hamiltonian=ham, hf=hf, sq=sq)
