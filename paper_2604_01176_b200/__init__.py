"""B200-native exact sparse state-vector engine (Hyperion-1 path of
arxiv/paper_2604_01176), a drop-in for the `svmps` SV API.

Public names mirror `svmps/__init__.py:6-34` for the SV path.  All compute
runs in libhsv.so (hand-written sm_100a CUDA behind the C ABI in
include/hsv.h); importing this package does not touch the GPU.
"""

__version__ = "0.1.0"

from .cibasis import (CiBasis, Configuration, enumerate_basis, hartree_fock_configuration,
                      sector_dimensions, subspace_stats)
from .pauli import PauliSum, PauliTerm
from .sparse import CsrMatrix, SparseVector, axpy, dot, norm, normalize, scale, spmspv
from .svengine import (AnsatzElement, ExcitationOperator, PauliOperator, SvState,
                       ansatz_energy_gradient, apply_ansatz, apply_generator,
                       apply_qeb_exponential, assemble_subspace_hamiltonian, expectation,
                       pool_gradient, pool_gradients)
from .system import MolecularSystem, bundled_fcidump
from .chem import (IntegralSet, SecondQuantizedHamiltonian, hartree_fock_reference, jordan_wigner,
                   load_fcidump, parse_fcidump, to_spin_orbital)
from . import fcidump, mapping
from .adapt import (AdaptConfig, OperatorPool, SvAdaptEngine, build_qeb_pool, run_adapt,
                    select_operator)

__all__ = [name for name in dir() if not name.startswith("_")]
