"""Pin the CPU oracle (oracle/sv_oracle.py) to the reference's golden vectors.

The goldens were produced by the unmodified reference (tests/golden/make_golden.py);
the CSR restatement must reproduce them bit for bit (same numpy operations in
the same order), the matrix-free variant to 1e-10.
"""
import numpy as np
import pytest

from conftest import load_golden, rel_err, s1_values
from oracle import sv_oracle as O

from paper_2604_01176_b200.system import MolecularSystem

SMALL = ["h2", "h4", "h6", "h8"]


def problem(name):
    s = MolecularSystem.bundled(name)
    h = s.hamiltonian
    states = O.sector_states(s.n_qubits, s.n_alpha, s.n_beta)
    ops = O.qeb_pool_masks(s.n_qubits, s.integrals.nelec)
    return s, h, states, ops


@pytest.mark.parametrize("name", SMALL)
def test_csr_restatement_bitwise(name):
    s, h, states, ops = problem(name)
    ref = load_golden(f"ref_{name}")
    csr = O.assemble_csr(h.xs, h.zs, h.coeffs, states)
    assert len(csr[1]) == int(ref["csr_nnz"])
    dim = len(states)
    idx = np.arange(dim, dtype=np.int64)
    psi = s1_values(dim)
    wi, wv = O.spmspv(csr, dim, idx, psi)
    assert np.array_equal(wi, ref["hs1_idx"]) and np.array_equal(wv, ref["hs1_val"])
    assert O.dot(idx, psi, wi, wv) == float(ref["e_s1_expect"])
    # S2 chain: bit-exact QEB rotations
    s2 = [ops[i] for i in ref["s2_ops"]]
    si, sv = O.apply_ansatz(states, s.hf.bits, s2, ref["s2_thetas"])
    assert np.array_equal(si, ref["s2_idx"]) and np.array_equal(sv, ref["s2_val"])
    wi2, wv2 = O.spmspv(csr, dim, si, sv)
    assert np.array_equal(wi2, ref["hs2_idx"]) and np.array_equal(wv2, ref["hs2_val"])
    h_apply = lambda i, v: O.spmspv(csr, dim, i, v)   # noqa: E731
    g = O.pool_gradients(h_apply, states, si, sv, ops)
    assert np.array_equal(g, ref["g_s2"])
    e, gr = O.energy_gradient(h_apply, states, s.hf.bits, s2, ref["s2_thetas"])
    assert e == float(ref["eg_s2_e"]) and np.array_equal(gr, ref["eg_s2_g"])
    for j, (oi, th) in enumerate(zip(ref["qeb_ops"], ref["qeb_thetas"])):
        qi, qv = O.apply_qeb(states, idx, psi, *ops[oi], float(th))
        assert np.array_equal(qi, ref[f"qeb{j}_idx"]) and np.array_equal(qv, ref[f"qeb{j}_val"])
        gi, gv = O.apply_generator(states, si, sv, *ops[oi])
        assert np.array_equal(gi, ref[f"gen{j}_idx"]) and np.array_equal(gv, ref[f"gen{j}_val"])


@pytest.mark.parametrize("name", ["h2", "h4", "h6"])
def test_csr_arrays_equal_reference_csr(name):
    s, h, states, ops = problem(name)
    ref = load_golden(f"ref_{name}")
    ro, ci, v = O.assemble_csr(h.xs, h.zs, h.coeffs, states)
    assert np.array_equal(ro, ref["csr_ro"]) and np.array_equal(ci, ref["csr_ci"])
    assert np.array_equal(v, ref["csr_v"])


@pytest.mark.parametrize("name", SMALL + ["h10"])
def test_matrix_free_restatement(name):
    s, h, states, ops = problem(name)
    ref = load_golden(f"ref_{name}")
    dim = len(states)
    psi = s1_values(dim)
    y = O.apply_h_matrix_free(h.xs, h.zs, h.coeffs, states, psi)
    assert abs(float(psi @ y) - float(ref["e_s1_expect"])) <= 1e-10
    if "hs1_idx" in ref:
        assert np.array_equal(np.flatnonzero(y), ref["hs1_idx"])
        assert rel_err(y[ref["hs1_idx"]], ref["hs1_val"]) <= 1e-10
    else:
        sel = ref["hs1_sample_idx"]
        assert np.count_nonzero(y) == int(ref["hs1_nnz"])
        assert rel_err(y[sel], ref["hs1_sample_val"]) <= 1e-10
        rows = sel[:64]
        yr = O.apply_h_rows(h.xs, h.zs, h.coeffs, states, psi, rows)
        assert rel_err(yr, ref["hs1_sample_val"][:64]) <= 1e-10


def test_pool_masks_match_reference_sizes():
    for name, m in [("h4", 26), ("h6", 117), ("h8", 360), ("h10", 875), ("h12", 1818),
                    ("h14", 3381), ("h16", 5792)]:
        s = MolecularSystem.bundled(name)
        assert len(O.qeb_pool_masks(s.n_qubits, s.integrals.nelec)) == m


def test_errors_mirror_reference():
    states = O.sector_states(4, 1, 1)
    xs, zs = np.array([0b0011]), np.array([0])
    with pytest.raises(ValueError, match="not spin-conserving"):
        O.assemble_csr(xs, zs, np.array([1.0]), states)
    with pytest.raises(ValueError, match="not real"):
        O.assemble_csr(np.array([0b0011]), np.array([0b0001]), np.array([1.0]), states)


def test_h12_golden_consistent():
    """The H12 goldens (made by this oracle, make_golden_h12.py) are self-consistent."""
    ref = load_golden("ref_h12")
    s, h, states, ops = problem("h12")
    assert len(states) == int(ref["dim"]) == 853776
    dim = len(states)
    psi = s1_values(dim)
    rows = ref["hs1_rows"][:16]
    yr = O.apply_h_rows(h.xs, h.zs, h.coeffs, states, psi, rows)
    assert rel_err(yr, ref["hs1_rows_val"][:16]) <= 1e-12
