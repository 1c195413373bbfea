"""K1t (hsv_apply_t.cu: alpha tiles, 8 alpha rows x one beta string per lane)
must reproduce the register-row K1 row for row, bit for bit (same elements,
same group order, same table values, signs and FMAs), for full and sharded row
ranges, forced split counts, sparse ADAPT-like states (alpha-row skips), the
energy-only path and the adjoint evaluation; energies agree to rounding."""
import numpy as np
import pytest

from conftest import s1_values

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hsv():
    import paper_2604_01176_b200 as hsv
    return hsv


@pytest.fixture()
def N():
    from paper_2604_01176_b200 import _native as N
    yield N
    for k in (b"apply_t", b"apply_split", b"push", b"restrict_rows"):
        N.call("hsv_set_tuning", k, {b"apply_split": 0, b"apply_t": 0}.get(k, -1))


def dense_state(hsv, sysm):
    dim = len(sysm.basis)
    return hsv.SvState(sysm.basis, hsv.SparseVector(dim, np.arange(dim, dtype=np.int64),
                                                    s1_values(dim)))


def rows(N, op, st, v, lo=0, hi=None, split=0):
    from paper_2604_01176_b200.svengine import DeviceState
    N.call("hsv_set_tuning", b"apply_t", v)
    N.call("hsv_set_tuning", b"apply_split", split)
    N.call("hsv_set_tuning", b"push", 0)
    out = DeviceState(st.basis)
    N.call("hsv_state_zero", out.handle)
    hi = st.basis._sector.n_alpha_strings if hi is None else hi
    N.call("hsv_apply_h_rows_async", op.handle, st.device.handle, out.handle, lo, hi, 0.0)
    N.call("hsv_synchronize")
    return out.torch_view().cpu().numpy()


@pytest.mark.parametrize("name", ["h4", "h6", "h8", "h10", "h12"])
def test_k1t_rows_bitwise_equal_k1(hsv, N, name):
    sysm = hsv.MolecularSystem.bundled(name)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    assert np.array_equal(rows(N, op, st, 1), rows(N, op, st, 0))


@pytest.mark.parametrize("split", [1, 8, 32])
def test_k1t_forced_splits_and_shards(hsv, N, split):
    sysm = hsv.MolecularSystem.bundled("h10")
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    na = sysm.basis._sector.n_alpha_strings
    for lo, hi in ((0, na), (0, na // 3), (na // 3, na)):
        assert np.array_equal(rows(N, op, st, 1, lo, hi, split), rows(N, op, st, 0, lo, hi, split))


def test_k1t_sparse_state_and_energy_screen(hsv, N):
    sysm = hsv.MolecularSystem.bundled("h12")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(5)
    ops = [pool.ops[i] for i in rng.integers(0, len(pool), size=30)]
    st = eng.rebuild(ops, rng.uniform(-0.3, 0.3, size=30))
    assert np.array_equal(rows(N, eng.matrix, st, 1), rows(N, eng.matrix, st, 0))
    out = {}
    for v in (1, 0):
        N.call("hsv_set_tuning", b"apply_t", v)
        out[v] = eng.energy_and_screen(dense_state(hsv, sysm), pool)
    assert abs(out[1][0] - out[0][0]) <= 1e-13
    assert np.max(np.abs(out[1][1] - out[0][1])) <= 1e-13


def test_k1t_expect_energy_only(hsv, N):
    sysm = hsv.MolecularSystem.bundled("h10")
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    N.call("hsv_set_tuning", b"apply_t", 1)
    e1 = op.expect(st)
    N.call("hsv_set_tuning", b"apply_t", 0)
    e0 = op.expect(st)
    assert abs(e1 - e0) <= 1e-13 * abs(e0)


def test_k1t_restricted_eval_bitwise(hsv, N):
    """The adjoint evaluation with K1v over the support rows equals K1r and the
    full register-row K1 bit for bit (energy and gradients)."""
    from conftest import load_golden
    tr = load_golden("trace_h12")
    sysm = hsv.MolecularSystem.bundled("h12")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    ops = [pool.ops[i] for i in tr["selected"]]
    for k in (25, 200):
        th = np.asarray(tr["thetas"][:k], dtype=np.float64)
        res = []
        for v, restrict in ((1, 1), (0, 1), (0, 0)):
            N.call("hsv_set_tuning", b"apply_t", v)
            N.call("hsv_set_tuning", b"restrict_rows", restrict)
            N.call("hsv_set_tuning", b"push", 0)
            res.append(eng.energy_and_gradient(ops[:k], th))
        for e, g in res[1:]:
            assert e == res[0][0] and np.array_equal(g, res[0][1]), k
