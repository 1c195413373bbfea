"""The fused cooperative sweep (one launch for all k rotations, hsv_qeb.cu
k_sweep) against the per-op launch path: energies, gradients and the
forward state bit for bit (same pairs, same reduction order)."""
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
    # the per-op path computes w = H psi on every row: compare against the
    # sweep with the full K1 too (K1r is checked in test_gpu_restrict.py)
    N.call("hsv_set_tuning", b"restrict_rows", 0)
    yield N
    N.call("hsv_set_tuning", b"sweep", 2)
    N.call("hsv_set_tuning", b"restrict_rows", -1)


def eg(N, eng, ops, th, sweep):
    N.call("hsv_set_tuning", b"sweep", sweep)
    return eng.energy_and_gradient(ops, th)


@pytest.mark.parametrize("sweep", [1, 2])
@pytest.mark.parametrize("name,k", [("h2", 3), ("h4", 12), ("h6", 30), ("h8", 40),
                                    ("h10", 25), ("h12", 20)])
def test_sweep_bitwise_equals_per_op(hsv, N, name, k, sweep):
    """sweep 1 (one barrier per rotation) replays the per-op reductions: bitwise.
    sweep 2 (orbit batches, hsv_sweep.cu) sums the gradient partials per orbit
    instead of per pair block: the state and the energy are bitwise, the
    gradients agree to rounding."""
    sysm = hsv.MolecularSystem.bundled(name)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(3)
    for trial in range(2):
        idx = rng.integers(0, len(pool), size=k)
        th = rng.uniform(-0.4, 0.4, size=k)
        th[::5] = 0.0                               # identity rotations are skipped forward
        ops = [pool.ops[i] for i in idx]
        e1, g1 = eg(N, eng, ops, th, sweep)
        e0, g0 = eg(N, eng, ops, th, 0)
        assert e1 == e0
        if sweep == 1:
            assert np.array_equal(g1, g0)
        else:
            assert np.max(np.abs(g1 - g0)) <= 1e-13 * max(1.0, np.max(np.abs(g0)))


def test_sweep_forward_state_and_two_phase(hsv, N):
    """hsv_eg_forward_async leaves the same psi / w either way."""
    from paper_2604_01176_b200.svengine import DeviceState
    sysm = hsv.MolecularSystem.bundled("h8")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(8)
    ops = [pool.ops[i] for i in rng.integers(0, len(pool), size=24)]
    th = rng.uniform(-0.5, 0.5, size=24)
    occ, virt = eng._pool_masks(ops)
    cs, sn = np.cos(th), np.sin(th)
    na = sysm.basis._sector.n_alpha_strings
    out = []
    for sweep in (2, 1, 0):
        N.call("hsv_set_tuning", b"sweep", sweep)
        psi, w = DeviceState(sysm.basis), DeviceState(sysm.basis)
        N.call("hsv_eg_forward_async", eng.matrix.handle, int(sysm.hf.bits), N.ptr_u64(occ),
               N.ptr_u64(virt), N.ptr_f64(cs), N.ptr_f64(sn), th.size, 0, na, psi.handle,
               w.handle)
        N.call("hsv_synchronize")
        out.append((psi.to_sparse(), w.to_sparse()))
    (p2, w2), (p1, w1), (p0, w0) = out
    for p, w in ((p2, w2), (p1, w1)):
        assert np.array_equal(p.indices, p0.indices) and np.array_equal(p.values, p0.values)
        assert np.array_equal(w.indices, w0.indices) and np.array_equal(w.values, w0.values)
    ref = hsv.apply_ansatz(sysm.basis, sysm.hf, ops, th).vec
    assert np.array_equal(ref.indices, p1.indices) and np.array_equal(ref.values, p1.values)


@pytest.mark.parametrize("name,k", [("h4", 12), ("h8", 40), ("h12", 16)])
def test_ansatz_state_equals_rotation_by_rotation(hsv, N, name, k):
    """hsv_ansatz_state (apply_ansatz: one fused sweep) against exp(theta T) applied
    one operator at a time (apply_qeb_exponential), bit for bit; theta = 0 skipped."""
    sysm = hsv.MolecularSystem.bundled(name)
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(17)
    idx = rng.integers(0, len(pool), size=k)
    th = rng.uniform(-0.5, 0.5, size=k)
    th[::4] = 0.0
    ops = [pool.ops[i] for i in idx]
    for sweep in (2, 1, 0):
        N.call("hsv_set_tuning", b"sweep", sweep)
        fused = hsv.apply_ansatz(sysm.basis, sysm.hf, ops, th).vec
        st = hsv.SvState.from_configuration(sysm.basis, sysm.hf)
        for op, t in zip(ops, th):
            st = hsv.apply_qeb_exponential(op, t, st)
        ref = st.vec
        assert np.array_equal(fused.indices, ref.indices), sweep
        assert np.array_equal(fused.values, ref.values), sweep
    empty = hsv.apply_ansatz(sysm.basis, sysm.hf, [], [])
    assert empty.nnz == 1


@pytest.mark.parametrize("sweep", [2, 1, 0])
def test_forward_drift_reported_by_backward(hsv, N, sweep):
    """A non-unitary rotation (c^2 + s^2 != 1) in the forward sweep: the forward call
    returns without waiting for the device and the consuming backward call raises
    the reference's RuntimeError (svengine.py:234-236); the engine stays usable."""
    sysm = hsv.MolecularSystem.bundled("h4")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    ops = [pool.ops[-1], pool.ops[0]]
    occ, virt = eng._pool_masks(ops)
    from paper_2604_01176_b200.svengine import DeviceState
    psi, w = DeviceState(sysm.basis), DeviceState(sysm.basis)
    cs, sn = N.as_f64(np.array([1.5, 1.0])), N.as_f64(np.array([0.5, 0.0]))
    na = sysm.basis._sector.n_alpha_strings
    N.call("hsv_set_tuning", b"sweep", sweep)
    N.call("hsv_eg_forward_async", eng.matrix.handle, int(sysm.hf.bits), N.ptr_u64(occ),
           N.ptr_u64(virt), N.ptr_f64(cs), N.ptr_f64(sn), 2, 0, na, psi.handle, w.handle)
    g = np.empty(2)
    e = N.dbl()
    with pytest.raises(RuntimeError, match="norm drift"):
        N.call("hsv_eg_backward", eng.matrix.handle, psi.handle, w.handle, N.ptr_u64(occ),
               N.ptr_u64(virt), N.ptr_f64(cs), N.ptr_f64(sn), 2, N.C.byref(e), N.ptr_f64(g))
    th = np.array([0.1, -0.2])
    e1, g1 = eng.energy_and_gradient(ops, th)
    e2, g2 = eng.energy_and_gradient(ops, th)
    assert e1 == e2 and np.array_equal(g1, g2)


@pytest.mark.parametrize("name", ["h8", "h12"])
def test_incremental_plan_equals_fresh_plan(hsv, N, name):
    """The sweep plan is refiltered incrementally when an operator is appended
    (ADAPT): along a growing operator list, with operators repeated (a batch
    boundary forced by a dependent flip) and one replaced in the middle (full
    refilter), energies and gradients are bitwise equal to fresh plans."""
    N.call("hsv_set_tuning", b"restrict_rows", -1)
    sysm = hsv.MolecularSystem.bundled(name)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(21)
    idx = list(rng.integers(0, len(pool), size=20))
    idx[7] = idx[6]                                   # a repeated operator
    seqs = [idx[:k] for k in range(1, 21)] + [idx[:10] + [idx[3]] + idx[11:]]
    th_all = rng.uniform(-0.4, 0.4, size=20)
    try:
        for seq in seqs:
            ops = [pool.ops[i] for i in seq]
            th = th_all[:len(seq)].copy()
            th[-1] = 0.0                              # a new operator starts at theta = 0
            N.call("hsv_set_tuning", b"sweep_incr", 1)
            e1, g1 = eng.energy_and_gradient(ops, th)
            N.call("hsv_set_tuning", b"sweep_incr", 0)
            e0, g0 = eng.energy_and_gradient(ops[:1], th[:1])   # another plan in between
            e0, g0 = eng.energy_and_gradient(ops, th)
            assert e1 == e0 and np.array_equal(g1, g0), len(seq)
    finally:
        N.call("hsv_set_tuning", b"sweep_incr", 1)
