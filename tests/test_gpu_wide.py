"""Sectors with norb > 16: the 64-bit packed-word (W = uint64) instantiations of
every kernel (leak/diag/CSR setup, K1 pull, K1p push, single-Z terms, screen,
QEB pair kernels, fused sweeps) against the CPU oracle.

The Hamiltonians are random molecular ones (real symmetric one-body, 8-fold
symmetric sparse two-body integrals) mapped by chem.jordan_wigner, on 17 and
18 spatial orbitals (34 / 36 qubits) with three electrons, so the sectors stay
small (dim 2,312 / 2,754) while every packed word needs more than 32 bits.
"""
import numpy as np
import pytest

from conftest import rel_err
from oracle import sv_oracle as O

pytestmark = pytest.mark.gpu

_PERMS = [(0, 1, 2, 3), (1, 0, 2, 3), (0, 1, 3, 2), (1, 0, 3, 2),
          (2, 3, 0, 1), (3, 2, 0, 1), (2, 3, 1, 0), (3, 2, 1, 0)]


def random_system(norb, seed):
    from paper_2604_01176_b200 import chem
    rng = np.random.default_rng(seed)
    h = rng.standard_normal((norb, norb)) * 0.2
    h = 0.5 * (h + h.T)
    raw = np.zeros((norb,) * 4)
    for _ in range(120):
        i, j, k, l = rng.integers(0, norb, 4)
        raw[i, j, k, l] += rng.standard_normal() * 0.05
    g = sum(raw.transpose(p) for p in _PERMS) / 8.0
    ints = chem.IntegralSet(norb, 3, 1, 0.7, h, g)
    return chem.molecular_system(ints)


@pytest.fixture(scope="module", params=[17, 18])
def wide(request):
    import paper_2604_01176_b200 as hsv
    s = random_system(request.param, 11 + request.param)
    h = s.hamiltonian
    states = O.sector_states(s.n_qubits, s.n_alpha, s.n_beta)
    assert np.array_equal(s.basis.states, states)
    csr = O.assemble_csr(h.xs, h.zs, h.coeffs, states)
    m = hsv.assemble_subspace_hamiltonian(h, s.basis)
    ops = O.qeb_pool_masks(s.n_qubits, s.integrals.nelec, ms2=1)
    pool = hsv.build_qeb_pool(s.n_qubits, s.integrals.nelec, ms2=1)
    assert [(o.occ_mask, o.virt_mask) for o in pool.ops] == ops
    return hsv, s, states, csr, m, pool, ops


def test_wide_csr_and_apply(wide):
    hsv, s, states, csr, m, pool, ops = wide
    assert m.nnz == len(csr[1])
    assert np.array_equal(m.col_indices, csr[1]) and np.array_equal(m.values, csr[2])
    dim = len(states)
    v = np.random.default_rng(5).standard_normal(dim)
    v /= np.linalg.norm(v)
    st = hsv.SvState(s.basis, hsv.SparseVector(dim, np.arange(dim), v))
    wi, wv = O.spmspv(csr, dim, np.arange(dim), v)
    w = m.apply_state(st).to_sparse()
    assert np.array_equal(w.indices, wi) and rel_err(w.values, wv) <= 1e-12
    assert abs(m.expect(st) - O.dot(np.arange(dim), v, wi, wv)) <= 1e-12


def test_wide_push_equals_pull(wide):
    from paper_2604_01176_b200 import _native as N
    hsv, s, states, csr, m, pool, ops = wide
    dim = len(states)
    rng = np.random.default_rng(6)
    pos = np.sort(rng.choice(dim, size=30, replace=False))
    st = hsv.SvState(s.basis, hsv.SparseVector(dim, pos, rng.standard_normal(30)))
    res = []
    try:
        N.call("hsv_set_tuning", b"apply_split", 1)
        for push in (1, 0):
            N.call("hsv_set_tuning", b"push", push)
            res.append(m.apply_state(st).to_sparse())
    finally:
        N.call("hsv_set_tuning", b"push", -1)
        N.call("hsv_set_tuning", b"apply_split", 0)
    assert np.array_equal(res[0].indices, res[1].indices)
    assert np.array_equal(res[0].values, res[1].values)
    wi, wv = O.spmspv(csr, dim, pos, st.vec.values)
    assert np.array_equal(res[0].indices, wi) and rel_err(res[0].values, wv) <= 1e-12


def test_wide_qeb_screen_and_adjoint(wide):
    hsv, s, states, csr, m, pool, ops = wide
    eng = hsv.SvAdaptEngine(s, hsv.AdaptConfig())
    rng = np.random.default_rng(7)
    idx = rng.integers(0, len(ops), 10)
    th = rng.uniform(-0.4, 0.4, 10)
    sel = [ops[i] for i in idx]
    # QEB chain: bit-exact against the oracle
    oi, ov = O.apply_ansatz(states, s.hf.bits, sel, th)
    st = hsv.apply_ansatz(s.basis, s.hf, [pool.ops[i] for i in idx], th)
    assert np.array_equal(st.vec.indices, oi) and np.array_equal(st.vec.values, ov)

    def h_apply(i, v):
        return O.spmspv(csr, len(states), i, v)
    g_ref = O.pool_gradients(h_apply, states, oi, ov, ops)
    assert rel_err(eng.screen(st, pool), g_ref) <= 1e-10
    e_ref, gr_ref = O.energy_gradient(h_apply, states, s.hf.bits, sel, th)
    e, g = eng.energy_and_gradient([pool.ops[i] for i in idx], th)
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
    assert rel_err(g, gr_ref) <= 1e-10
