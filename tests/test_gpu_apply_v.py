"""K1v (hsv_apply_v.cu, opt-in tuning apply_v=1; measured slower than K1 at
H12, kept as a bitwise-equal alternative): per-group valid beta lists with shared-memory row
accumulators must reproduce the register-row K1 row for row, bit for bit (each
row sums the same nonzero elements in the same group order; K1 only adds
extra exact zeros for out-of-sector partners), for full and sharded row
ranges, forced split counts, sparse ADAPT-like states (alpha-row skips) and the
support-restricted mode; energies agree to rounding (different unit order)."""
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
    # the valid lists are built at operator creation only while K1v is enabled:
    # every operator of these tests is created after this point
    N.call("hsv_set_tuning", b"apply_v", 1)
    yield N
    for k in (b"apply_v", b"apply_split", b"push", b"restrict_rows"):
        N.call("hsv_set_tuning", k, {b"apply_split": 0, b"apply_v": 0}.get(k, -1))


def dense_state(hsv, sysm):
    dim = len(sysm.basis)
    return hsv.SvState(sysm.basis, hsv.SparseVector(dim, np.arange(dim, dtype=np.int64),
                                                    s1_values(dim)))


def rows(N, op, st, v, lo=0, hi=None, split=0):
    from paper_2604_01176_b200.svengine import DeviceState
    N.call("hsv_set_tuning", b"apply_v", v)
    N.call("hsv_set_tuning", b"apply_split", split)
    N.call("hsv_set_tuning", b"push", 0)
    out = DeviceState(st.basis)
    N.call("hsv_state_zero", out.handle)
    hi = st.basis._sector.n_alpha_strings if hi is None else hi
    N.call("hsv_apply_h_rows_async", op.handle, st.device.handle, out.handle, lo, hi, 0.0)
    N.call("hsv_synchronize")
    return out.torch_view().cpu().numpy()


@pytest.mark.parametrize("name", ["h4", "h6", "h8", "h10", "h12"])
def test_k1v_rows_bitwise_equal_k1(hsv, N, name):
    sysm = hsv.MolecularSystem.bundled(name)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    assert np.array_equal(rows(N, op, st, 1), rows(N, op, st, 0))


@pytest.mark.parametrize("split", [1, 8, 32])
def test_k1v_forced_splits_and_shards(hsv, N, split):
    sysm = hsv.MolecularSystem.bundled("h10")
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    na = sysm.basis._sector.n_alpha_strings
    for lo, hi in ((0, na), (0, na // 3), (na // 3, na)):
        assert np.array_equal(rows(N, op, st, 1, lo, hi, split), rows(N, op, st, 0, lo, hi, split))


def test_k1v_sparse_state_and_energy_screen(hsv, N):
    sysm = hsv.MolecularSystem.bundled("h12")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(5)
    ops = [pool.ops[i] for i in rng.integers(0, len(pool), size=30)]
    st = eng.rebuild(ops, rng.uniform(-0.3, 0.3, size=30))
    assert np.array_equal(rows(N, eng.matrix, st, 1), rows(N, eng.matrix, st, 0))
    out = {}
    for v in (1, 0):
        N.call("hsv_set_tuning", b"apply_v", v)
        out[v] = eng.energy_and_screen(dense_state(hsv, sysm), pool)
    assert abs(out[1][0] - out[0][0]) <= 1e-13
    assert np.max(np.abs(out[1][1] - out[0][1])) <= 1e-13


def test_k1v_restricted_eval_bitwise(hsv, N):
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
            N.call("hsv_set_tuning", b"apply_v", v)
            N.call("hsv_set_tuning", b"restrict_rows", restrict)
            N.call("hsv_set_tuning", b"push", 0)
            res.append(eng.energy_and_gradient(ops[:k], th))
        for e, g in res[1:]:
            assert e == res[0][0] and np.array_equal(g, res[0][1]), k
