"""Molecular problem setup (mirror of `svmps.system`, system.py:1-67).

The hot path starts from a Jordan-Wigner `PauliSum`.  The bundled hydrogen
chains H2..H16 (STO-3G, interleaved ordering) are stored as Pauli-sum
arrays produced by the reference's own builder (FCIDUMP -> to_spin_orbital ->
jordan_wigner, system.py:43-45; H14/H16 FCIDUMPs from its offline
`scripts/make_fixtures.py`), see tests/golden/make_golden.py.  Systems can
also be built directly from Pauli-sum arrays.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .cibasis import CiBasis, Configuration, enumerate_basis, hartree_fock_configuration
from .pauli import PauliSum

DATA = Path(__file__).resolve().parent / "data"
_ORDER_NAME = {0: "interleaved", 1: "blocked"}


@dataclass(frozen=True)
class IntegralInfo:
    """The FCIDUMP header fields the SV path consumes (fcidump.py:24-56)."""

    norb: int
    nelec: int
    ms2: int

    @property
    def n_alpha(self) -> int:
        return (self.nelec + self.ms2) // 2

    @property
    def n_beta(self) -> int:
        return (self.nelec - self.ms2) // 2


def bundled_fcidump(name: str) -> Path:
    """Path of a bundled FCIDUMP (reference `system.py:15-22`).  This package
    ships the Pauli sums built from them (`bundled_hamiltonian`); the FCIDUMP
    text is looked up in `data/` and then in an importable `svmps`."""
    path = DATA / f"{name.lower()}.fcidump"
    if path.exists():
        return path
    try:
        from importlib import resources
        ref = resources.files("svmps").joinpath("data", f"{name.lower()}.fcidump")
        with resources.as_file(ref) as concrete:
            if concrete.exists():
                return Path(concrete)
    except (ImportError, ModuleNotFoundError, TypeError):
        pass
    raise FileNotFoundError(f"no bundled FCIDUMP named {name!r}")


def bundled_hamiltonian(name: str) -> Path:
    path = DATA / f"ham_{name.lower()}.npz"
    if not path.exists():
        raise FileNotFoundError(f"no bundled Hamiltonian named {name!r}")
    return path


@dataclass
class MolecularSystem:
    integrals: IntegralInfo
    ordering: str
    hamiltonian: PauliSum
    hf: Configuration
    sq: object = field(default=None, repr=False)   # chem.SecondQuantizedHamiltonian when built from integrals
    _basis: CiBasis | None = field(default=None, repr=False)

    @classmethod
    def from_integrals(cls, ints, ordering: str = "interleaved") -> "MolecularSystem":
        """Integrals -> spin orbitals -> Jordan-Wigner (reference `system.py:33-37`)."""
        from .chem import molecular_system
        return molecular_system(ints, ordering)

    @classmethod
    def from_pauli(cls, h: PauliSum, nelec: int, ms2: int = 0,
                   ordering: str = "interleaved") -> "MolecularSystem":
        info = IntegralInfo(h.n_qubits // 2, nelec, ms2)
        hf = hartree_fock_configuration(nelec, h.n_qubits, ordering, ms2)
        return cls(integrals=info, ordering=ordering, hamiltonian=h, hf=hf)

    @classmethod
    def from_fcidump(cls, path, ordering: str = "interleaved") -> "MolecularSystem":
        """FCIDUMP -> spin orbitals -> Jordan-Wigner (system.py:43-45 semantics)."""
        from .chem import load_fcidump, molecular_system
        return molecular_system(load_fcidump(path), ordering)

    @classmethod
    def from_fcidump_text(cls, text: str, ordering: str = "interleaved") -> "MolecularSystem":
        from .chem import molecular_system, parse_fcidump
        return molecular_system(parse_fcidump(text), ordering)

    @classmethod
    def bundled(cls, name: str) -> "MolecularSystem":
        with np.load(bundled_hamiltonian(name)) as z:
            n = int(z["n_qubits"])
            h = PauliSum(n, z["xs"], z["zs"], z["coeffs"], _trusted=True)
            sysm = cls.from_pauli(h, int(z["nelec"]), int(z["ms2"]),
                                  _ORDER_NAME[int(z["ordering"])])
            if sysm.hf.bits != int(z["hf_bits"]):
                raise ValueError("bundled Hartree-Fock configuration mismatch")
            return sysm

    @property
    def n_qubits(self) -> int:
        return self.hamiltonian.n_qubits

    @property
    def n_alpha(self) -> int:
        return self.integrals.n_alpha

    @property
    def n_beta(self) -> int:
        return self.integrals.n_beta

    @property
    def basis(self) -> CiBasis:
        if self._basis is None:
            self._basis = enumerate_basis(self.n_qubits, self.n_alpha, self.n_beta, self.ordering)
        return self._basis
