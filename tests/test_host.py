"""Host-side logic that mirrors the reference API (no GPU needed)."""
import math
from itertools import combinations

import numpy as np
import pytest

from conftest import load_golden
from oracle import sv_oracle as O

import paper_2604_01176_b200 as hsv
from paper_2604_01176_b200.adapt import amortized_coefficient
from paper_2604_01176_b200.cibasis import qubit_spin


def test_pool_minimal_example():
    """test_adapt.py:26-30."""
    assert [op.label() for op in hsv.build_qeb_pool(4, 2)] == ["s:0->2", "s:1->3", "d:0,1->2,3"]


def test_pool_no_virtuals_rejected():
    with pytest.raises(ValueError, match="pool"):
        hsv.build_qeb_pool(4, 4)


def test_pool_h6_brute_force():
    n, ne = 12, 6
    pool = hsv.build_qeb_pool(n, ne)
    occ = list(range(ne))
    virt = [q for q in range(n) if q not in occ]
    spin = {q: qubit_spin(q, n, "interleaved") for q in range(n)}
    singles = sum(1 for i in occ for a in virt if spin[i] == spin[a])
    doubles = sum(1 for i, j in combinations(occ, 2) for a, b in combinations(virt, 2)
                  if sorted((spin[i], spin[j])) == sorted((spin[a], spin[b])))
    assert pool.size == singles + doubles == 117


def test_pool_masks_agree_with_oracle():
    for name in ("h4", "h8", "h12"):
        s = hsv.MolecularSystem.bundled(name)
        pool = hsv.build_qeb_pool(s.n_qubits, s.integrals.nelec)
        ref = O.qeb_pool_masks(s.n_qubits, s.integrals.nelec)
        assert [(op.occ_mask, op.virt_mask) for op in pool] == ref


def test_select_operator_rules():
    assert hsv.select_operator([0.1, -0.3, 0.2], 1e-3) == 1
    assert hsv.select_operator([0.2, -0.2], 1e-3) == 0
    assert hsv.select_operator([1e-5, -1e-6], 1e-3) is None
    with pytest.raises(ValueError):
        hsv.select_operator([], 1e-3)


def test_config_validation():
    with pytest.raises(ValueError):
        hsv.AdaptConfig(engine="dense").validate()
    with pytest.raises(ValueError):
        hsv.AdaptConfig(eps_grad=0.0).validate()
    with pytest.raises(ValueError):
        hsv.AdaptConfig(trunc_rule="brutal").validate()
    with pytest.raises(NotImplementedError):
        hsv.adapt.make_engine(hsv.MolecularSystem.bundled("h2"), hsv.AdaptConfig(engine="mps"))


def test_amortized_coefficient():
    js, ct, cfit = amortized_coefficient([(j, 4.0 * j * j) for j in range(1, 9)])
    assert np.allclose(ct, 0.5) and cfit == pytest.approx(4.0)
    with pytest.raises(ValueError, match="monotone"):
        amortized_coefficient([(1, 2.0), (2, 1.0)])


@pytest.mark.parametrize("n,ne,cik", [(12, 6, 400), (16, 8, 4900), (20, 10, 63504),
                                      (24, 12, 853776)])
def test_sector_dimensions_table1(n, ne, cik):
    """Criterion 1 sizes (test_acceptance.py:62-85)."""
    d = hsv.sector_dimensions(n, ne // 2, ne // 2)
    assert d["ci_k"] == cik and d["hilbert"] == 1 << n and d["ci"] == math.comb(n, ne)
    assert len(hsv.enumerate_basis(n, ne // 2, ne // 2)) == cik


def test_large_sector_formula():
    assert hsv.sector_dimensions(28, 7, 7)["ci_k"] == 11778624
    assert hsv.sector_dimensions(32, 8, 8)["ci_k"] == 165636900


@pytest.mark.parametrize("args", [(8, 2, 2, "interleaved"), (10, 3, 2, "interleaved"),
                                  (12, 3, 3, "blocked")])
def test_basis_states_match_oracle(args):
    b = hsv.enumerate_basis(*args)
    assert np.array_equal(b.states, O.sector_states(*args))
    assert b.index_of(int(b.states[5])) == 5
    pos, ok = b.try_positions(np.array([b.states[3], 0]))
    assert pos[0] == 3 and ok[0] and not ok[1]


def test_hartree_fock():
    assert hsv.hartree_fock_configuration(4, 8).bits == 0b1111
    assert hsv.hartree_fock_configuration(2, 8, "blocked").bits == 0b10001
    with pytest.raises(ValueError):
        hsv.hartree_fock_configuration(3, 8)


def test_pauli_sum_canonical():
    h = hsv.PauliSum.from_strings([(0.5, "XZ"), (0.25, "IZ"), (0.5, "XZ"), (1.0, "II")])
    assert len(h) == 3
    assert list(zip(h.xs, h.zs)) == sorted(zip(h.xs, h.zs))
    assert h.coeffs[list(zip(h.xs, h.zs)).index((1, 2))] == 1.0
    assert h.scaled(0.0).coeffs.size == 0
    assert h.identity_coefficient == 1.0


def test_bundled_hamiltonians_match_reference_sizes():
    """Term / group counts from SURVEY.md section 8 (H6..H16)."""
    for name, t, g in [("h6", 919, 148), ("h8", 2913, 501), ("h10", 7151, 1286),
                       ("h12", 14905, 2767), ("h14", 27735, 5272), ("h16", 47489, 9193)]:
        s = hsv.MolecularSystem.bundled(name)
        assert len(s.hamiltonian) == t
        assert len(np.unique(s.hamiltonian.xs)) == g


def test_excitation_operator():
    op = hsv.ExcitationOperator("double", (3, 0), (7, 5))
    assert op.occ == (0, 3) and op.virt == (5, 7) and op.label() == "d:0,3->5,7"
    with pytest.raises(ValueError):
        hsv.ExcitationOperator("double", (0, 0), (4, 5))
    with pytest.raises(ValueError):
        hsv.AnsatzElement(op, float("inf"))


def test_sparse_vector_containers():
    v = hsv.SparseVector.from_entries(8, [3, 1, 3, 5], [1.0, 2.0, -1.0, 0.5])
    assert v.indices.tolist() == [1, 5] and v.values.tolist() == [2.0, 0.5]
    d = np.array([0.0, 1.5, 0.0, -2.0])
    assert np.array_equal(hsv.SparseVector.from_dense(d).to_dense(), d)
    m = hsv.CsrMatrix.from_dense(np.array([[1.0, 2.0], [2.0, -1.0]]))
    m.validate(hermitian_tol=1e-12)
    assert hsv.CsrMatrix.from_dense(np.array([[0.0, 1.0], [0.0, 0.0]])).symmetry_defect() == 1.0


def test_csr_cache_roundtrip(tmp_path):
    from paper_2604_01176_b200.svengine import load_csr, save_csr
    m = hsv.CsrMatrix.from_dense(np.array([[1.0, 0.0, 2.0], [0.0, 3.0, 0.0], [2.0, 0.0, 0.0]]))
    save_csr(tmp_path / "m.csr", m)
    again = load_csr(tmp_path / "m.csr")
    assert np.array_equal(again.row_offsets, m.row_offsets)
    assert np.array_equal(again.values, m.values)
    (tmp_path / "junk.csr").write_bytes(b"not a cache")
    with pytest.raises(ValueError):
        load_csr(tmp_path / "junk.csr")


def test_adapt_traces_present():
    tr = load_golden("adapt_h4")
    assert tr["selected"][0] == -1 and len(tr["energy"]) == len(tr["nnz"])
