"""The K1 push path (scatter + radix sort + segmented reduce, hsv_push.cu) for
sparse psi against the pull kernel and the goldens.

The push path sums every row in the pull kernel's own order (diagonal, then
groups by index), so with the pull kernel unsplit (apply_split = 1) the rows
of H|psi> agree bit for bit; energies are summed in a different order
(1e-14 relative).  The auto selection is covered by the golden tests in
test_gpu_parity.py (HF and ADAPT-like states take the push path there).
"""
import numpy as np
import pytest

from conftest import load_golden, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hsv():
    import paper_2604_01176_b200 as hsv
    return hsv


@pytest.fixture()
def N():
    from paper_2604_01176_b200 import _native as N
    yield N
    N.call("hsv_set_tuning", b"push", -1)
    N.call("hsv_set_tuning", b"apply_split", 0)


_cache = {}


def setup(hsv, name):
    if name not in _cache:
        sysm = hsv.MolecularSystem.bundled(name)
        eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
        pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
        _cache[name] = (sysm, eng, pool)
    return _cache[name]


def sparse_states(hsv, sysm, pool, rng):
    basis = sysm.basis
    dim = len(basis)
    out = [("hf", hsv.SvState.from_configuration(basis, sysm.hf))]
    for k in (4, 16):
        idx = rng.integers(0, len(pool), size=k)
        th = rng.uniform(-0.3, 0.3, size=k)
        out.append((f"adapt{k}", hsv.apply_ansatz(basis, sysm.hf, [pool.ops[i] for i in idx], th)))
    n = min(dim, 40)
    pos = np.sort(rng.choice(dim, size=n, replace=False))
    out.append(("rand_real", hsv.SvState(basis, hsv.SparseVector(dim, pos, rng.standard_normal(n)))))
    vals = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    out.append(("rand_cplx", hsv.SvState(basis, hsv.SparseVector(dim, pos, vals))))
    return out


def apply_with(N, op, st, push, prune=0.0):
    N.call("hsv_set_tuning", b"push", push)
    N.call("hsv_set_tuning", b"apply_split", 1)
    w = op.apply_state(st, prune)
    e = op.expect(st)
    return w.to_sparse(), e


@pytest.mark.parametrize("name", ["h4", "h6", "h8", "h10", "h12"])
def test_push_rows_bitwise_equal_pull(hsv, N, name):
    sysm, eng, pool = setup(hsv, name)
    rng = np.random.default_rng(11)
    for label, st in sparse_states(hsv, sysm, pool, rng):
        wp, ep = apply_with(N, eng.matrix, st, 1)
        wq, eq = apply_with(N, eng.matrix, st, 0)
        assert np.array_equal(wp.indices, wq.indices), label
        assert np.array_equal(wp.values, wq.values), label
        assert abs(ep - eq) <= 1e-14 * max(1.0, abs(eq)), label


def test_push_goldens_h8(hsv, N):
    """Forced push on the golden S2 state (k = 20 rotations) and on S1 (dense)."""
    from conftest import s1_values
    sysm, eng, pool = setup(hsv, "h8")
    ref = load_golden("ref_h8")
    N.call("hsv_set_tuning", b"push", 1)
    st = eng.rebuild([pool.ops[i] for i in ref["s2_ops"]], ref["s2_thetas"])
    w = eng.matrix.apply_state(st).to_sparse()
    assert np.array_equal(w.indices, ref["hs2_idx"])
    assert rel_err(w.values, ref["hs2_val"]) <= 1e-10
    assert abs(eng.energy(st) - float(ref["e_s2"])) <= 1e-10 * abs(float(ref["e_s2"]))
    assert rel_err(eng.screen(st, pool), ref["g_s2"]) <= 1e-10
    e, g = eng.energy_and_gradient([pool.ops[i] for i in ref["s2_ops"]], ref["s2_thetas"])
    assert abs(e - float(ref["eg_s2_e"])) <= 1e-10 * abs(e)
    assert rel_err(g, ref["eg_s2_g"]) <= 1e-10
    dim = len(sysm.basis)
    s1 = hsv.SvState(sysm.basis, hsv.SparseVector(dim, np.arange(dim, dtype=np.int64),
                                                  s1_values(dim)))
    w1 = eng.matrix.apply_state(s1).to_sparse()
    assert np.array_equal(w1.indices, ref["hs1_idx"])
    assert rel_err(w1.values, ref["hs1_val"]) <= 1e-10


def test_push_row_ranges_and_empty(hsv, N):
    """Owner-computes row ranges: push rows == pull rows, zero elsewhere; psi = 0."""
    from paper_2604_01176_b200.svengine import DeviceState
    sysm, eng, pool = setup(hsv, "h10")
    rng = np.random.default_rng(5)
    na = sysm.basis._sector.n_alpha_strings
    nb = sysm.basis._sector.n_beta_strings
    st = sparse_states(hsv, sysm, pool, rng)[2][1]
    for lo, hi in ((0, na), (0, na // 3), (na // 3, na // 2), (na - 1, na), (5, 5)):
        res = []
        for push in (1, 0):
            N.call("hsv_set_tuning", b"push", push)
            N.call("hsv_set_tuning", b"apply_split", 1)
            out = DeviceState(sysm.basis)
            N.call("hsv_state_zero", out.handle)
            N.call("hsv_apply_h_rows_async", eng.matrix.handle, st.device.handle, out.handle,
                   lo, hi, 0.0)
            N.call("hsv_synchronize")
            res.append(out.torch_view().cpu().numpy())
        assert np.array_equal(res[0], res[1]), (lo, hi)
        assert not res[0][: lo * nb].any() and not res[0][hi * nb:].any()
    zero = DeviceState(sysm.basis)
    N.call("hsv_state_zero", zero.handle)
    N.call("hsv_set_tuning", b"push", 1)
    w = eng.matrix.apply_state(hsv.SvState(sysm.basis, _dev=zero))
    assert w.nnz() == 0


def test_push_prune_and_determinism(hsv, N):
    sysm, eng, pool = setup(hsv, "h10")
    rng = np.random.default_rng(9)
    st = sparse_states(hsv, sysm, pool, rng)[2][1]
    wp, _ = apply_with(N, eng.matrix, st, 1, prune=1e-3)
    wq, _ = apply_with(N, eng.matrix, st, 0, prune=1e-3)
    assert np.array_equal(wp.indices, wq.indices) and np.array_equal(wp.values, wq.values)
    assert np.all(np.abs(wp.values) >= 1e-3)
    N.call("hsv_set_tuning", b"push", 1)
    g1 = eng.screen(st, pool)
    g2 = eng.screen(st, pool)
    assert np.array_equal(g1, g2)


def test_push_device_sized_keys_across_supports(hsv, N):
    """K1p sizes its keys launch from the previous call's source count: supports
    that grow past 4x (re-run at the exact size), shrink, and repeat must all give
    the pull kernel's rows bit for bit."""
    sysm, eng, pool = setup(hsv, "h10")
    dim = len(sysm.basis)
    rng = np.random.default_rng(23)
    for n in (1, 3, 50, 12, 12, 400, 2, 2000, 2000):
        pos = np.sort(rng.choice(dim, size=n, replace=False))
        st = hsv.SvState(sysm.basis, hsv.SparseVector(dim, pos, rng.standard_normal(n)))
        wp, ep = apply_with(N, eng.matrix, st, 1)
        wq, eq = apply_with(N, eng.matrix, st, 0)
        assert np.array_equal(wp.indices, wq.indices), n
        assert np.array_equal(wp.values, wq.values), n
        assert abs(ep - eq) <= 1e-14 * max(1.0, abs(eq)), n
