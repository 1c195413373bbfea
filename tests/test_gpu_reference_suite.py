"""The reference's own test strategy run on the device engine:
unit tests of svengine/sparse/adapt (pkg/tests/test_svengine.py, test_sparse.py,
test_adapt.py) and the SV acceptance criteria 2, 3, 8, 9, 10
(pkg/tests/test_acceptance.py), re-expressed against this package's API."""
import dataclasses

import numpy as np
import pytest
import scipy.linalg

from conftest import load_golden, rel_err, s1_values

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hsv():
    import paper_2604_01176_b200 as hsv
    return hsv


@pytest.fixture(scope="module")
def systems(hsv):
    out = {}
    for n in ("h2", "h4", "h6"):
        s = hsv.MolecularSystem.bundled(n)
        m = hsv.assemble_subspace_hamiltonian(s.hamiltonian, s.basis)
        dense = m.to_dense()
        evals, evecs = np.linalg.eigh(dense)
        out[n] = (s, m, evals[0], evecs[:, 0])
    return out


def H4_OPS(hsv):
    E = hsv.ExcitationOperator
    return [E("single", (0,), (4,)), E("single", (3,), (7,)), E("double", (0, 1), (4, 5)),
            E("double", (0, 3), (5, 6)), E("double", (2, 3), (6, 7))]


def dense_state(hsv, basis, vec):
    return hsv.SvState(basis, hsv.normalize(hsv.SparseVector.from_dense(vec)))


# ------------------------------------------------------------ assembly / CSR
@pytest.mark.parametrize("name", ["h2", "h4", "h6"])
def test_materialized_csr_is_reference_csr_bitwise(hsv, systems, name):
    """Every matrix element equals the reference CSR bit for bit (svengine.py:115-171)."""
    s, m, _, _ = systems[name]
    ref = load_golden(f"ref_{name}")
    assert np.array_equal(m.row_offsets, ref["csr_ro"])
    assert np.array_equal(m.col_indices, ref["csr_ci"])
    assert np.array_equal(m.values, ref["csr_v"])
    assert m.symmetry_defect() == 0.0


def test_fci_h2_golden(systems):
    """test_fcidump.py:86-92: H2 FCI = -1.1372701752425907."""
    assert abs(systems["h2"][2] - (-1.1372701752425907)) <= 1e-10


def test_expectation_eigenvector_and_stationarity(hsv, systems):
    """test_svengine.py:88-91 and :149-153."""
    s, m, e0, v0 = systems["h4"]
    st = dense_state(hsv, s.basis, v0)
    assert abs(hsv.expectation(m, st) - e0) <= 1e-10
    for op in H4_OPS(hsv):
        assert abs(hsv.pool_gradient(m, st, op)) <= 1e-10


def test_screen_converged_eigenstate_h2(hsv, systems):
    """test_adapt.py:63-73."""
    s, m, e0, v0 = systems["h2"]
    eng = hsv.SvAdaptEngine(s, hsv.AdaptConfig())
    st = dense_state(hsv, s.basis, v0)
    for g in eng.screen(st, hsv.build_qeb_pool(4, 2)):
        assert abs(g) <= 1e-8


def test_screen_hf_dominant_double_h2(hsv, systems):
    """test_adapt.py:76-84."""
    s = systems["h2"][0]
    eng = hsv.SvAdaptEngine(s, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(4, 2)
    g = dict(zip([o.label() for o in pool], eng.screen(eng.initial_state(), pool)))
    assert abs(g["d:0,1->2,3"]) > 1e-2 and abs(g["s:0->2"]) <= 1e-10 and abs(g["s:1->3"]) <= 1e-10


# -------------------------------------------------------------------- QEB
def test_qeb_theta_zero_and_half_pi(hsv, systems, rng):
    """test_svengine.py:94-111."""
    s = systems["h4"][0]
    st = dense_state(hsv, s.basis, rng.standard_normal(len(s.basis)))
    out = hsv.apply_qeb_exponential(H4_OPS(hsv)[2], 0.0, st)
    assert np.array_equal(out.vec.indices, st.vec.indices)
    assert np.array_equal(out.vec.values, st.vec.values)
    op = H4_OPS(hsv)[2]
    hf = hsv.SvState.from_configuration(s.basis, s.hf)
    dense = hsv.apply_qeb_exponential(op, np.pi / 2, hf).vec.to_dense()
    fp = s.basis.index_of(s.hf.bits ^ op.flip_mask)
    assert abs(abs(dense[fp]) - 1.0) < 1e-12
    dense[fp] = 0.0
    assert np.max(np.abs(dense)) < 1e-15


def test_qeb_against_dense_expm(hsv, systems, rng):
    """test_svengine.py:114-131: closed form == expm(theta * generator)."""
    s = systems["h4"][0]
    n = len(s.basis)
    worst = 0.0
    for _ in range(20):
        op = H4_OPS(hsv)[int(rng.integers(5))]
        theta = float(rng.uniform(-3, 3))
        gen = np.zeros((n, n))
        for j in range(n):
            col = hsv.apply_generator(op, hsv.SvState(s.basis, hsv.SparseVector.basis_state(n, j)))
            gen[col.indices, j] = col.values
        u = scipy.linalg.expm(theta * gen)
        st = dense_state(hsv, s.basis, rng.standard_normal(n))
        out = hsv.apply_qeb_exponential(op, theta, st)
        worst = max(worst, np.max(np.abs(out.vec.to_dense() - u @ st.vec.to_dense())))
        assert abs(hsv.norm(out.vec) - 1.0) <= 1e-12
    assert worst <= 1e-10


def test_criterion_09_unitarity_and_conservation(hsv, systems, rng):
    """test_acceptance.py:258-277: 1000 random applications, norm drift <= 1e-12."""
    s = systems["h6"][0]
    pool = hsv.build_qeb_pool(12, 6).ops
    st = dense_state(hsv, s.basis, rng.standard_normal(len(s.basis)))
    worst = 0.0
    for k in range(1000):
        op = pool[int(rng.integers(len(pool)))]
        st = hsv.apply_qeb_exponential(op, float(rng.uniform(-3, 3)), st)
        if k % 50 == 49 or k == 999:
            v = st.vec
            worst = max(worst, abs(hsv.norm(v) - 1.0))
            assert np.all(v.indices >= 0) and np.all(v.indices < len(s.basis))
        if k % 100 == 99:
            st = dense_state(hsv, s.basis, rng.standard_normal(len(s.basis)))
    assert worst <= 1e-12


# -------------------------------------------------------------- gradients
def test_criterion_10_gradient_vs_finite_difference(hsv, systems, rng):
    """test_acceptance.py:282-298: 200 (state, op) pairs, |analytic - fd| <= 1e-6."""
    s, m, _, _ = systems["h4"]
    pool = hsv.build_qeb_pool(8, 4).ops
    worst = 0.0
    for _ in range(200):
        st = dense_state(hsv, s.basis, rng.standard_normal(len(s.basis)))
        op = pool[int(rng.integers(len(pool)))]
        g = hsv.pool_gradient(m, st, op)
        h = 1e-5
        ep = hsv.expectation(m, hsv.apply_qeb_exponential(op, +h, st))
        em = hsv.expectation(m, hsv.apply_qeb_exponential(op, -h, st))
        worst = max(worst, abs(g - (ep - em) / (2 * h)))
    assert worst <= 1e-6


def test_pool_gradient_disjoint_support_is_exact_zero(hsv, systems):
    """test_svengine.py:167-171."""
    s, m, _, _ = systems["h4"]
    hf = hsv.SvState.from_configuration(s.basis, s.hf)
    assert hsv.pool_gradient(m, hf, hsv.ExcitationOperator("single", (4,), (6,))) == 0.0


def test_ansatz_chain_gradient_vs_fd(hsv, systems, rng):
    """test_svengine.py:174-184."""
    s, m, _, _ = systems["h4"]
    ops = H4_OPS(hsv)[2:]
    th = rng.uniform(-0.4, 0.4, len(ops))
    e0, g = hsv.ansatz_energy_gradient(m, s.basis, s.hf, ops, th)
    for i in range(len(ops)):
        tp, tm = th.copy(), th.copy()
        tp[i] += 1e-6
        tm[i] -= 1e-6
        ep, _ = hsv.ansatz_energy_gradient(m, s.basis, s.hf, ops, tp)
        em, _ = hsv.ansatz_energy_gradient(m, s.basis, s.hf, ops, tm)
        assert abs(g[i] - (ep - em) / 2e-6) <= 1e-6


def test_generic_csr_path_matches_matrix_free(hsv, systems, rng):
    """A plain CsrMatrix of the same H (K1b + generic adjoint) agrees with the
    matrix-free device operator (K1/K4/K5)."""
    s, m, _, _ = systems["h6"]
    csr = hsv.CsrMatrix(m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)
    pool = hsv.build_qeb_pool(12, 6).ops
    ops = [pool[i] for i in rng.integers(0, len(pool), 6)]
    th = rng.uniform(-0.3, 0.3, 6)
    e1, g1 = hsv.ansatz_energy_gradient(m, s.basis, s.hf, ops, th)
    e2, g2 = hsv.ansatz_energy_gradient(csr, s.basis, s.hf, ops, th)
    assert abs(e1 - e2) <= 1e-12 and rel_err(g1, g2) <= 1e-12
    st = hsv.apply_ansatz(s.basis, s.hf, ops, th)
    assert rel_err(hsv.pool_gradients(m, st, pool), hsv.pool_gradients(csr, st, pool)) <= 1e-12


# ------------------------------------------------------------ sparse (K1b)
def test_spmspv_identity_empty_mismatch_prune(hsv, rng):
    """test_sparse.py:27-37, :62-67, :133-136."""
    v = hsv.SparseVector.from_dense(np.where(rng.random(64) < 0.5, rng.standard_normal(64), 0.0))
    out = hsv.spmspv(hsv.CsrMatrix.identity(64), v)
    assert np.array_equal(out.indices, v.indices) and np.array_equal(out.values, v.values)
    dm = rng.standard_normal((32, 32))
    assert hsv.spmspv(hsv.CsrMatrix.from_dense(dm), hsv.SparseVector.empty(32)).nnz == 0
    with pytest.raises(ValueError):
        hsv.spmspv(hsv.CsrMatrix.identity(4), hsv.SparseVector.empty(5))
    with pytest.raises(ValueError):
        hsv.dot(hsv.SparseVector.empty(4), hsv.SparseVector.empty(5))
    dm = rng.standard_normal((128, 128))
    dm[rng.random((128, 128)) > 0.05] = 0.0
    out = hsv.spmspv(hsv.CsrMatrix.from_dense(dm), hsv.SparseVector.from_dense(
        rng.standard_normal(128)), prune=1e-2)
    assert out.nnz == 0 or np.min(np.abs(out.values)) >= 1e-2


def test_worker_count_independence(hsv, rng):
    """test_sparse.py:51-59: bitwise identical for any n_workers."""
    dm = rng.standard_normal((301, 301))
    dm[rng.random((301, 301)) > 0.05] = 0.0
    m = hsv.CsrMatrix.from_dense(dm)
    v = hsv.SparseVector.from_dense(np.where(rng.random(301) < 0.3, rng.standard_normal(301), 0))
    base = hsv.spmspv(m, v, n_workers=1)
    for w in (2, 3, 7):
        out = hsv.spmspv(m, v, n_workers=w)
        assert np.array_equal(out.indices, base.indices) and np.array_equal(out.values, base.values)


def test_symmetric_bilinear_identity(hsv, systems, rng):
    """test_sparse.py:110-121, on a random symmetric CSR and on the Pauli operator."""
    for _ in range(10):
        a = rng.standard_normal((40, 40))
        a[rng.random((40, 40)) > 0.1] = 0.0
        csr = hsv.CsrMatrix.from_dense(a + a.T)
        u = hsv.SparseVector.from_dense(np.where(rng.random(40) < 0.4, rng.standard_normal(40), 0))
        v = hsv.SparseVector.from_dense(np.where(rng.random(40) < 0.4, rng.standard_normal(40), 0))
        assert abs(hsv.dot(u, hsv.spmspv(csr, v)) - hsv.dot(v, hsv.spmspv(csr, u))) <= 1e-12
    s, m, _, _ = systems["h6"]
    n = len(s.basis)
    u = hsv.SparseVector.from_dense(rng.standard_normal(n))
    v = hsv.SparseVector.from_dense(np.where(rng.random(n) < 0.3, rng.standard_normal(n), 0))
    assert abs(hsv.dot(u, hsv.spmspv(m, v)) - hsv.dot(v, hsv.spmspv(m, u))) <= 1e-12


def test_criterion_08_spmspv_oracle_equivalence(hsv, rng):
    """test_acceptance.py:233-253: 1000 random instances vs dense, <= 1e-12."""
    worst = 0.0
    for _ in range(1000):
        dim = int(rng.integers(2, 513))
        dm = rng.standard_normal((dim, dim))
        dm[rng.random((dim, dim)) > 0.05] = 0.0
        vec = rng.standard_normal(dim)
        vec[rng.random(dim) > 0.3] = 0.0
        out = hsv.spmspv(hsv.CsrMatrix.from_dense(dm), hsv.SparseVector.from_dense(vec))
        worst = max(worst, np.max(np.abs(out.to_dense() - dm @ vec), initial=0.0))
    assert worst <= 1e-12


# ------------------------------------------------------------------ ADAPT
def test_optimize_single_parameter_reaches_fci(hsv, systems):
    """test_adapt.py:109-114."""
    s, _, e0, _ = systems["h2"]
    eng = hsv.SvAdaptEngine(s, hsv.AdaptConfig())
    res = hsv.adapt.optimize_parameters(eng, [hsv.build_qeb_pool(4, 2).ops[2]], [0.0],
                                        hsv.AdaptConfig())
    assert abs(res.energy - e0) <= 1e-9


def test_run_behaviour(hsv, systems, tmp_path):
    """test_adapt.py:126-203: threshold, fast H2, monotone energies, determinism,
    incremental CSV, nnz growth within the sector."""
    s2, _, e2, _ = systems["h2"]
    res = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=1e3), systems["h4"][0])
    assert res.status == "converged" and len(res.records) == 1
    res = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=1e-6), s2, reference_energy=e2,
                        csv_path=tmp_path / "run.csv")
    assert res.status == "converged" and res.records[-1].iteration <= 2
    assert res.records[-1].abs_error <= 1e-8
    lines = (tmp_path / "run.csv").read_text().strip().splitlines()
    assert lines[0].startswith("iter,selected_op,grad_max,energy") and len(lines) == len(res.records) + 1
    cfg = hsv.AdaptConfig(engine="sv", eps_grad=1e-4, max_iter=8)
    a = hsv.run_adapt(cfg, systems["h4"][0])
    b = hsv.run_adapt(cfg, systems["h4"][0])
    for ra, rb in zip(a.records, b.records):
        assert (ra.selected_op, ra.energy, ra.grad_max, ra.nnz) == \
            (rb.selected_op, rb.energy, rb.grad_max, rb.nnz)
    en = [r.energy for r in a.records]
    assert all(y <= x + 1e-12 for x, y in zip(en, en[1:]))
    r6 = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=1e-4, max_iter=12), systems["h6"][0])
    nnz = [r.nnz for r in r6.records]
    assert all(y >= x for x, y in zip(nnz, nnz[1:])) and nnz[-1] <= 400


def test_selection_invariant_under_scaling(hsv, systems):
    """test_adapt.py:96-106."""
    s = systems["h4"][0]
    pool = hsv.build_qeb_pool(8, 4)
    base = hsv.SvAdaptEngine(s, hsv.AdaptConfig())
    sc = dataclasses.replace(s, hamiltonian=s.hamiltonian.scaled(3.7), _basis=None)
    scaled = hsv.SvAdaptEngine(sc, hsv.AdaptConfig())
    g1 = base.screen(base.initial_state(), pool)
    g2 = scaled.screen(scaled.initial_state(), pool)
    assert np.allclose(g2, 3.7 * g1, rtol=1e-10)
    assert np.argmax(np.abs(g1)) == np.argmax(np.abs(g2))


def test_criterion_03_h6_chemical_accuracy(hsv, systems):
    """test_acceptance.py:103-114: 2e-3 Ha within 250 iterations."""
    s, _, e0, _ = systems["h6"]
    res = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=1e-4, max_iter=250), s,
                        reference_energy=e0)
    hits = [r.iteration for r in res.records if r.abs_error is not None and r.abs_error <= 2e-3]
    assert hits and hits[0] <= 250


@pytest.mark.parametrize("name", ["h2", "h4", "h6", "h8", "h10"])
def test_gpu_lanczos_fci_matches_reference_eigsh(hsv, name):
    """Device Lanczos (fci.py) vs the reference's oracle.fci_ground_energy values."""
    from paper_2604_01176_b200.fci import lanczos_ground_energy
    s = hsv.MolecularSystem.bundled(name)
    m = hsv.assemble_subspace_hamiltonian(s.hamiltonian, s.basis)
    e = lanczos_ground_energy(m)
    assert abs(e - float(load_golden(f"ref_{name}")["e_fci"])) <= 1e-10


@pytest.mark.parametrize("name,vectors", [("h8", 8), ("h10", 10), ("h10", 24)])
def test_thick_restart_lanczos_bounded_storage(hsv, name, vectors):
    """With at most `vectors` Krylov states (forced thick restarts) the device
    solver still reaches the reference eigsh energy, and reports its Ritz
    residual ||H y - E y|| (checked against an explicit H application)."""
    from paper_2604_01176_b200 import _native as N
    from paper_2604_01176_b200.fci import lanczos_ground_energy
    from paper_2604_01176_b200.svengine import DeviceState
    s = hsv.MolecularSystem.bundled(name)
    m = hsv.assemble_subspace_hamiltonian(s.hamiltonian, s.basis)
    e, y, info = lanczos_ground_energy(m, max_vectors=vectors, return_vector=True,
                                       return_info=True)
    assert abs(e - float(load_golden(f"ref_{name}")["e_fci"])) <= 1e-10
    assert info["restarts"] > 0 and info["max_vectors"] == vectors
    assert info["residual_norm"] <= 1e-11 * abs(e)
    hy = DeviceState(s.basis)
    N.call("hsv_apply_h", m.handle, y.handle, hy.handle, 0.0)
    n2 = y.dot(y).real
    r = hy.to_sparse().to_dense() - e * y.to_sparse().to_dense()
    assert np.linalg.norm(r) <= 1e-8 * np.sqrt(n2) * abs(e)


def test_h12_fci_with_residual(hsv):
    """H12 (beyond the reference's CSR on a 62 GB host): the device energy with
    its residual bound; E_FCI is below the ADAPT trace's best energy."""
    from paper_2604_01176_b200.fci import lanczos_ground_energy
    s = hsv.MolecularSystem.bundled("h12")
    m = hsv.assemble_subspace_hamiltonian(s.hamiltonian, s.basis)
    e, info = lanczos_ground_energy(m, max_vectors=20, return_info=True)
    assert info["residual_norm"] <= 1e-11 * abs(e)
    assert abs(e - (-6.452815878528843)) <= 1e-9      # DESIGN.md (round 1, full-basis Lanczos)
    assert e < float(load_golden("trace_h12")["energy"].min())


# --------------------------------------------------- orderings / sectors
def _to_blocked(x: int, n: int) -> int:
    norb = n // 2
    out = 0
    for q in range(n):
        if (x >> q) & 1:
            p, sp = q // 2, q & 1
            out |= 1 << (p + sp * norb)
    return out


def test_blocked_ordering_matches_interleaved(hsv, systems, rng):
    """Same physics in the blocked qubit ordering (cibasis.py:37-51): qubit maps
    2p+s -> p + s*norb; HF energy, adjoint energy/gradients and screens agree."""
    s = systems["h6"][0]
    n = s.n_qubits
    h = s.hamiltonian
    hb = hsv.PauliSum(n, [_to_blocked(int(x), n) for x in h.xs],
                      [_to_blocked(int(z), n) for z in h.zs], h.coeffs)
    sb = hsv.MolecularSystem.from_pauli(hb, s.integrals.nelec, 0, "blocked")
    assert sb.hf.bits == _to_blocked(s.hf.bits, n)
    ea = hsv.SvAdaptEngine(s, hsv.AdaptConfig())
    eb = hsv.SvAdaptEngine(sb, hsv.AdaptConfig())
    pa = hsv.build_qeb_pool(n, 6)
    opsb = [hsv.ExcitationOperator(o.kind, [_to_blocked(1 << q, n).bit_length() - 1 for q in o.occ],
                                   [_to_blocked(1 << q, n).bit_length() - 1 for q in o.virt])
            for o in pa.ops]
    idx = rng.integers(0, len(pa.ops), 8)
    th = rng.uniform(-0.3, 0.3, 8)
    e1, g1 = ea.energy_and_gradient([pa.ops[i] for i in idx], th)
    e2, g2 = eb.energy_and_gradient([opsb[i] for i in idx], th)
    assert abs(e1 - e2) <= 1e-12 and rel_err(g1, g2) <= 1e-11
    st_a = ea.rebuild([pa.ops[i] for i in idx], th)
    st_b = eb.rebuild([opsb[i] for i in idx], th)
    assert rel_err(ea.screen(st_a, pa.ops), eb.screen(st_b, opsb)) <= 1e-11


def test_unequal_spin_sector_against_oracle(hsv, systems, rng):
    """n_alpha != n_beta (ms2 = 2) sector: device energy and H|psi> vs the CPU oracle."""
    from oracle import sv_oracle as O
    s = systems["h4"][0]
    basis = hsv.enumerate_basis(8, 3, 1)
    m = hsv.assemble_subspace_hamiltonian(s.hamiltonian, basis)
    states = O.sector_states(8, 3, 1)
    assert np.array_equal(basis.states, states)
    csr = O.assemble_csr(s.hamiltonian.xs, s.hamiltonian.zs, s.hamiltonian.coeffs, states)
    assert np.array_equal(m.values, csr[2]) and np.array_equal(m.col_indices, csr[1])
    v = rng.standard_normal(len(states))
    v /= np.linalg.norm(v)
    st = hsv.SvState(basis, hsv.SparseVector(len(states), np.arange(len(states)), v))
    wi, wv = O.spmspv(csr, len(states), np.arange(len(states)), v)
    w = m.apply_state(st).to_sparse()
    assert np.array_equal(w.indices, wi) and rel_err(w.values, wv) <= 1e-12
    assert abs(hsv.expectation(m, st) - O.dot(np.arange(len(states)), v, wi, wv)) <= 1e-12


def test_complex_state_energy_is_real_and_gradients_consistent(hsv, systems, rng):
    """complex128 amplitudes (north star): <psi|H|psi> real for Hermitian H; the
    screen equals 2 Re <H psi|T psi> computed from device H|psi> and T|psi>."""
    s, m, _, _ = systems["h6"]
    n = len(s.basis)
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    v /= np.linalg.norm(v)
    st = hsv.SvState(s.basis, hsv.SparseVector(n, np.arange(n), v))
    from paper_2604_01176_b200 import _native as N
    re, im = N.dbl(), N.dbl()
    N.call("hsv_expect_h", m.handle, st.device.handle, N.C.byref(re), N.C.byref(im))
    assert abs(im.value) <= 1e-12
    w = m.apply_state(st).to_sparse().to_dense()
    pool = hsv.build_qeb_pool(12, 6).ops
    g = hsv.pool_gradients(m, st, pool)
    for k in range(0, len(pool), 13):
        t = hsv.apply_generator(pool[k], st).to_dense()
        assert abs(g[k] - 2.0 * np.real(np.vdot(w, t))) <= 1e-12
    assert abs(re.value - np.real(np.vdot(v, w))) <= 1e-12


def test_complex_apply_is_the_reference_matrix_and_exactly_linear(hsv, systems, rng):
    """complex128 H|psi> (no complex reference output exists: the reference's
    molecular path is real) anchored twice: against the reference's own CSR
    (golden ref_h6, bitwise equal to the materialized matrix above) applied on
    the host to the complex vector, and by exact linearity -- H(i psi) is i H psi
    bit for bit, since every product and sum is mirrored under re <-> -im."""
    s, m, _, _ = systems["h6"]
    ref = load_golden("ref_h6")
    import scipy.sparse
    A = scipy.sparse.csr_matrix((ref["csr_v"], ref["csr_ci"], ref["csr_ro"]))
    n = len(s.basis)
    v = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    v /= np.linalg.norm(v)
    w = m.apply_state(hsv.SvState(s.basis, hsv.SparseVector(n, np.arange(n), v))).to_sparse().to_dense()
    want = A @ v
    assert np.max(np.abs(w - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
    wi = m.apply_state(hsv.SvState(s.basis, hsv.SparseVector(n, np.arange(n), 1j * v))).to_sparse().to_dense()
    assert np.array_equal(wi.real, -w.imag) and np.array_equal(wi.imag, w.real)
