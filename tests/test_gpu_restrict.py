"""K1r: the adjoint evaluation computes w = H psi only on the structural
support of psi (hsv_apply.cu launch_apply_rows), because the backward sweep
never reads w elsewhere (rotation pairs do not straddle the support).

* energies and gradients are bit-identical to the full pull kernel (push off:
  the push path sums rows unsplit, so it agrees to rounding only);
* on the support, the w rows are bit-identical to the full K1 rows, and
  every other row is an exact zero;
* the structural support contains every nonzero of psi, including the
  rotations of a newly appended theta = 0 operator (skipped: no growth).
"""
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
    N.call("hsv_set_tuning", b"restrict_rows", -1)
    N.call("hsv_set_tuning", b"push", -1)


def run_eg(N, eng, ops, th, restrict, push):
    N.call("hsv_set_tuning", b"restrict_rows", restrict)
    N.call("hsv_set_tuning", b"push", push)
    return eng.energy_and_gradient(ops, th)


def trace_ops(hsv, name, pool, k):
    """ops/thetas of the device engine's own H12 ADAPT trace (dense-ish regime),
    or random pool ops elsewhere"""
    rng = np.random.default_rng(11)
    idx = rng.integers(0, len(pool), size=k)
    th = rng.uniform(-0.3, 0.3, size=k)
    return [pool.ops[i] for i in idx], th


@pytest.mark.parametrize("name,k", [("h4", 6), ("h6", 12), ("h8", 20), ("h8", 60), ("h10", 8),
                                    ("h10", 40), ("h12", 12)])
def test_restricted_eval_bitwise_equals_full_pull(hsv, N, name, k):
    sysm = hsv.MolecularSystem.bundled(name)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    ops, th = trace_ops(hsv, name, pool, k)
    th[-1] = 0.0                         # L-BFGS's first evaluation of a new operator
    e1, g1 = run_eg(N, eng, ops, th, 1, 0)
    e0, g0 = run_eg(N, eng, ops, th, 0, 0)
    assert e1 == e0
    assert np.array_equal(g1, g0)
    e2, g2 = run_eg(N, eng, ops, th, 0, -1)        # default full path (push when sparse)
    assert abs(e1 - e2) <= 1e-13 * max(1.0, abs(e2))
    assert np.max(np.abs(g1 - g2)) <= 1e-13 * max(1.0, np.max(np.abs(g2)))


def test_h12_trace_depths_bitwise(hsv, N):
    """Along the committed H12 ADAPT trace (tests/golden/trace_h12.npz) at depth
    25 / 100 / 200: the regimes the ADAPT bench leg times."""
    from conftest import load_golden
    tr = load_golden("trace_h12")
    sysm = hsv.MolecularSystem.bundled("h12")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    ops = [pool.ops[i] for i in tr["selected"]]
    for k in (25, 100, 200):
        th = np.asarray(tr["thetas"][:k], dtype=np.float64)
        e1, g1 = run_eg(N, eng, ops[:k], th, 1, 0)
        e0, g0 = run_eg(N, eng, ops[:k], th, 0, 0)
        assert e1 == e0 and np.array_equal(g1, g0), k


def test_rows_and_support(hsv, N):
    from paper_2604_01176_b200.svengine import DeviceState
    sysm = hsv.MolecularSystem.bundled("h8")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    ops, th = trace_ops(hsv, "h8", pool, 10)
    occ, virt = eng._pool_masks(ops)
    cs, sn = np.cos(th), np.sin(th)
    na = sysm.basis._sector.n_alpha_strings
    got = {}
    for restrict in (1, 0):
        N.call("hsv_set_tuning", b"restrict_rows", restrict)
        N.call("hsv_set_tuning", b"push", 0)
        psi, w = DeviceState(sysm.basis), DeviceState(sysm.basis)
        N.call("hsv_eg_forward_async", eng.matrix.handle, int(sysm.hf.bits), N.ptr_u64(occ),
               N.ptr_u64(virt), N.ptr_f64(cs), N.ptr_f64(sn), len(ops), 0, na, psi.handle,
               w.handle)
        got[restrict] = (psi.to_sparse(), w.at_positions(np.arange(len(sysm.basis))))
    p1, w1 = got[1]
    p0, w0 = got[0]
    assert np.array_equal(p1.indices, p0.indices) and np.array_equal(p1.values, p0.values)
    # rows in the support: bit-identical; rows outside: exact zeros
    on = np.zeros(len(sysm.basis), bool)
    on[p1.indices] = True
    assert np.array_equal(w1[on], w0[on])
    extra = (w1 != 0) & ~on                  # structural-only rows (none expected here)
    assert np.array_equal(w1[extra], w0[extra])
    assert np.count_nonzero(w1) < np.count_nonzero(w0)
