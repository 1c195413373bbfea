"""Reference module name `svmps.mapping` (mapping.py:28-132): spin-orbital
expansion and Jordan-Wigner.  The implementation lives in chem.py."""
from .chem import (JW_DROP_TOL, JW_IMAG_TOL, SecondQuantizedHamiltonian, hartree_fock_reference,
                   jordan_wigner, to_spin_orbital)

__all__ = ["JW_DROP_TOL", "JW_IMAG_TOL", "SecondQuantizedHamiltonian", "hartree_fock_reference",
           "jordan_wigner", "to_spin_orbital"]
