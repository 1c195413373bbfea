"""The partitioned engine's exact local part:
`local_csr = assemble_subspace_hamiltonian(h.select(local_mask), basis)`,
`spmspv(local_csr, psi)`, `dot(psi, w)` and `dot(w, apply_generator(op, psi))`
(partition.py:94, 192-216; adapt.py:327-339) -- the same kernels on a sub-sum.

Goldens come from the unmodified reference (tests/golden/make_golden_partition.py).
CPU: the oracle restatement reproduces them bit for bit.  GPU: the device
operator built from the selected sub-sum matches them to 1e-10 (support exact).
"""
import numpy as np
import pytest

from conftest import load_golden, rel_err
from oracle import sv_oracle as O

from paper_2604_01176_b200.system import MolecularSystem

CASES = [(n, e) for n in ("h6", "h8") for e in (1, 2)]


def s2_state_oracle(s, states, ref):
    ops = O.qeb_pool_masks(s.n_qubits, s.integrals.nelec)
    return O.apply_ansatz(states, s.hf.bits, [ops[i] for i in ref["s2_ops"]], ref["s2_thetas"]), ops


@pytest.mark.parametrize("name,eta", CASES)
def test_local_part_oracle_bitwise(name, eta):
    s = MolecularSystem.bundled(name)
    gold = load_golden(f"partition_{name}")
    ref = load_golden(f"ref_{name}")
    loc = s.hamiltonian.select(gold[f"eta{eta}_local_mask"])
    states = O.sector_states(s.n_qubits, s.n_alpha, s.n_beta)
    csr = O.assemble_csr(loc.xs, loc.zs, loc.coeffs, states)
    assert len(csr[1]) == int(gold[f"eta{eta}_local_nnz"])
    (si, sv), ops = s2_state_oracle(s, states, ref)
    wi, wv = O.spmspv(csr, len(states), si, sv)
    assert np.array_equal(wi, gold[f"eta{eta}_w_idx"])
    assert np.array_equal(wv, gold[f"eta{eta}_w_val"])
    assert O.dot(si, sv, wi, wv) == float(gold[f"eta{eta}_e_local"])
    for k, g in zip(gold[f"eta{eta}_g_ops"], gold[f"eta{eta}_g_local"]):
        ti, tv = O.apply_generator(states, si, sv, *ops[k])
        assert O.dot(wi, wv, ti, tv) == pytest.approx(float(g), rel=1e-12, abs=1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("name,eta", CASES)
def test_local_part_gpu(name, eta):
    import paper_2604_01176_b200 as hsv
    s = MolecularSystem.bundled(name)
    gold = load_golden(f"partition_{name}")
    ref = load_golden(f"ref_{name}")
    loc = s.hamiltonian.select(gold[f"eta{eta}_local_mask"])
    m = hsv.assemble_subspace_hamiltonian(loc, s.basis)
    assert m.nnz == int(gold[f"eta{eta}_local_nnz"])
    pool = hsv.build_qeb_pool(s.n_qubits, s.integrals.nelec)
    st = hsv.apply_ansatz(s.basis, s.hf, [pool.ops[i] for i in ref["s2_ops"]], ref["s2_thetas"])
    w = hsv.spmspv(m, st.vec)
    assert np.array_equal(w.indices, gold[f"eta{eta}_w_idx"])
    assert rel_err(w.values, gold[f"eta{eta}_w_val"]) <= 1e-10
    e = hsv.dot(st.vec, w)
    assert abs(e - float(gold[f"eta{eta}_e_local"])) <= 1e-10 * max(1.0, abs(e))
    g = np.array([hsv.dot(w, hsv.apply_generator(pool.ops[k], st))
                  for k in gold[f"eta{eta}_g_ops"]])
    assert rel_err(g, gold[f"eta{eta}_g_local"]) <= 1e-10
