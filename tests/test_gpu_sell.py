"""K1a (assembled sliced-ELL rows, csrc/hsv_apply.cu k_apply_sell) against the
matrix-free K1 it is enumerated from: H|psi> rows bit for bit (same split
partials, same FMA order, exact zeros dropped), on dense real and complex
states, on alpha-row shards, with the drop rule, and through the ADAPT screen;
energies to rounding (the partial sums are grouped per 32-row chunk)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hsv():
    import paper_2604_01176_b200 as hsv
    return hsv


@pytest.fixture()
def N():
    from paper_2604_01176_b200 import _native as N
    yield N
    N.call("hsv_set_tuning", b"sell", -1)


def dense(hsv, basis, v):
    n = len(basis)
    return hsv.SvState(basis, hsv.SparseVector(n, np.arange(n), v))


def both(N, fn):
    N.call("hsv_set_tuning", b"sell", 0)
    r0 = fn()
    N.call("hsv_set_tuning", b"sell", 1)
    r1 = fn()
    return r0, r1


@pytest.mark.parametrize("name", ["h4", "h6", "h8", "h10", "h12"])
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("sp", [-1, 0, 1])
def test_sell_rows_bitwise_equal_k1(hsv, N, name, cplx, sp):
    sysm = hsv.MolecularSystem.bundled(name)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    rng = np.random.default_rng(5)
    n = len(sysm.basis)
    v = rng.standard_normal(n) + (1j * rng.standard_normal(n) if cplx else 0.0)
    v /= np.linalg.norm(v)
    st = dense(hsv, sysm.basis, v)
    N.call("hsv_set_tuning", b"sell_sp", sp)   # chunk per warp, split segments, auto
    try:
        (w0, e0), (w1, e1) = both(N, lambda: (op.apply_state(st).to_sparse().to_dense(),
                                              op.expect(st)))
    finally:
        N.call("hsv_set_tuning", b"sell_sp", -1)
    assert np.array_equal(w0, w1)
    assert abs(e1 - e0) <= 1e-13 * max(1.0, abs(e0))
    # the drop rule on the combined rows
    thr = float(np.quantile(np.abs(w0), 0.3))
    p0, p1 = both(N, lambda: op.apply_state(st, prune=thr).to_sparse())
    assert np.array_equal(p0.indices, p1.indices) and np.array_equal(p0.values, p1.values)


@pytest.mark.parametrize("name", ["h8", "h12"])
def test_sell_alpha_shards_and_screen(hsv, N, name):
    """Rank shards (alpha-row ranges, the multi-GPU owner-computes split) build
    their own assembled rows; the screen's gradients are bitwise equal."""
    from paper_2604_01176_b200.svengine import DeviceState
    sysm = hsv.MolecularSystem.bundled(name)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    na = sysm.basis._sector.n_alpha_strings
    rng = np.random.default_rng(9)
    n = len(sysm.basis)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    st = dense(hsv, sysm.basis, v)
    cuts = [0, na // 3, na // 3 + 1, na]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        def shard():
            out = DeviceState(sysm.basis)
            N.call("hsv_apply_h_rows_async", op.handle, st.device.handle, out.handle, lo, hi, 0.0)
            N.call("hsv_synchronize")
            return out.to_sparse().to_dense()
        r0, r1 = both(N, shard)
        assert np.array_equal(r0, r1), (lo, hi)
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    (ea, ga), (eb, gb) = both(N, lambda: eng.energy_and_screen(st, pool))
    assert np.array_equal(ga, gb)
    assert abs(ea - eb) <= 1e-13 * max(1.0, abs(ea))


def test_sell_declines_over_budget(hsv, N):
    """Over the budget nothing is built and K1 runs (same rows)."""
    sysm = hsv.MolecularSystem.bundled("h8")
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    n = len(sysm.basis)
    st = dense(hsv, sysm.basis, np.full(n, 1.0 / np.sqrt(n)))
    N.call("hsv_set_tuning", b"sell_budget_mb", 0)
    try:
        (w0, _), (w1, _) = both(N, lambda: (op.apply_state(st).to_sparse().to_dense(), 0))
        assert np.array_equal(w0, w1)
    finally:
        N.call("hsv_set_tuning", b"sell_budget_mb", 32768)


@pytest.mark.parametrize("name", ["h8", "h10"])
def test_support_compacted_rows_along_a_growing_list(hsv, N, name):
    """K1s (support rows of the assembled matrix, in-map elements only) against
    the matrix-free K1r: energies and gradients bitwise along a growing operator
    list (the map grows, stays, is rebuilt) and after a replaced operator."""
    sysm = hsv.MolecularSystem.bundled(name)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(17)
    idx = list(rng.integers(0, len(pool), size=24))
    th_all = rng.uniform(-0.4, 0.4, size=24)
    seqs = [idx[:k] for k in (1, 2, 5, 9, 10, 16, 24)] + [idx[:12] + [idx[2]] + idx[13:]]
    try:
        for seq in seqs:
            ops = [pool.ops[i] for i in seq]
            th = th_all[:len(seq)].copy()
            th[-1] = 0.0
            N.call("hsv_set_tuning", b"sup", 1)
            e1, g1 = eng.energy_and_gradient(ops, th)
            e1b, g1b = eng.energy_and_gradient(ops, th)    # the cached compacted rows
            N.call("hsv_set_tuning", b"sup", 0)
            e0, g0 = eng.energy_and_gradient(ops, th)
            assert e1 == e0 and np.array_equal(g1, g0), len(seq)
            assert e1b == e0 and np.array_equal(g1b, g0), len(seq)
    finally:
        N.call("hsv_set_tuning", b"sup", -1)


@pytest.mark.parametrize("name", ["h10", "h12"])
def test_overlapped_energy_screen_bitwise_equal_serial(hsv, N, name):
    """K4 phases on a second stream under the K1a stream (screen_overlap) give
    the serial path's energy and gradients bit for bit (same partials, same
    reduction order); also on an alpha-row shard."""
    sysm = hsv.MolecularSystem.bundled(name)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    n = len(sysm.basis)
    rng = np.random.default_rng(23)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    st = dense(hsv, sysm.basis, v)
    eng.energy_and_screen(st, pool)                 # marks psi dense, builds the rows
    try:
        out = {}
        for ov in (0, 4, 3):
            N.call("hsv_set_tuning", b"screen_overlap", ov)
            out[ov] = eng.energy_and_screen(st, pool)
        for ov in (4, 3):
            assert out[ov][0] == out[0][0] and np.array_equal(out[ov][1], out[0][1]), ov
    finally:
        N.call("hsv_set_tuning", b"screen_overlap", 2)


def test_support_rows_auto_switch_on_a_plateau(hsv, N):
    """sup = -1: a support map that serves more than 10 evaluations switches to
    the compacted assembled rows mid-run; every evaluation stays bitwise equal."""
    sysm = hsv.MolecularSystem.bundled("h10")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(37)
    ops = [pool.ops[i] for i in rng.integers(0, len(pool), size=40)]
    th = rng.uniform(-0.4, 0.4, size=40)
    N.call("hsv_set_tuning", b"sup", -1)
    res = [eng.energy_and_gradient(ops, th) for _ in range(14)]
    for e, g in res[1:]:
        assert e == res[0][0] and np.array_equal(g, res[0][1])
