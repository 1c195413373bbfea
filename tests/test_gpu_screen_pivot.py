"""K4 pivoted on psi rows (hsv_screen.cu, PIVOT: sparse psi) against the w-row
kernel: the same (w row, psi row, beta list) terms grouped differently, so the
gradients agree to rounding; on row shards the pivoted partials sum to the full
result; and both match the reference goldens."""
import numpy as np
import pytest

from conftest import load_golden, rel_err, s1_values

pytestmark = pytest.mark.gpu


@pytest.fixture()
def N():
    from paper_2604_01176_b200 import _native as N
    yield N
    N.call("hsv_set_tuning", b"screen_pivot", -1)


def states(hsv, sysm, pool, rng):
    basis = sysm.basis
    dim = len(basis)
    out = [hsv.SvState.from_configuration(basis, sysm.hf)]
    for k in (4, 20):
        idx = rng.integers(0, len(pool), size=k)
        out.append(hsv.apply_ansatz(basis, sysm.hf, [pool.ops[i] for i in idx],
                                    rng.uniform(-0.3, 0.3, size=k)))
    out.append(hsv.SvState(basis, hsv.SparseVector(dim, np.arange(dim, dtype=np.int64),
                                                   s1_values(dim))))
    return out


@pytest.mark.parametrize("name", ["h6", "h8", "h10"])
def test_pivot_matches_w_rows(N, name):
    import paper_2604_01176_b200 as hsv
    sysm = hsv.MolecularSystem.bundled(name)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    for st in states(hsv, sysm, pool, np.random.default_rng(4)):
        res = {}
        for pv in (0, 1):
            N.call("hsv_set_tuning", b"screen_pivot", pv)
            res[pv] = eng.energy_and_screen(st, pool)
        e0, g0 = res[0]
        e1, g1 = res[1]
        assert e0 == e1
        assert np.max(np.abs(g1 - g0)) <= 1e-13 * max(1.0, np.max(np.abs(g0)))


def test_pivot_shards_sum_to_full(N):
    import torch
    import paper_2604_01176_b200 as hsv
    sysm = hsv.MolecularSystem.bundled("h8")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    dpool = eng._device_pool(pool)
    st = states(hsv, sysm, pool, np.random.default_rng(8))[2]
    na = sysm.basis._sector.n_alpha_strings
    N.call("hsv_set_tuning", b"screen_pivot", 1)
    full = eng.energy_and_screen(st, pool)[1]
    acc = np.zeros(pool.__len__() if hasattr(pool, "__len__") else len(pool.ops))
    d = torch.zeros(2 + len(acc) + (len(acc) & 1), dtype=torch.float64, device="cuda")
    for lo, hi in ((0, na // 3), (na // 3, na // 2), (na // 2, na)):
        N.call("hsv_energy_screen_pool_async", eng.matrix.handle, st.device.handle,
               dpool.handle, lo, hi, N.C.c_void_p(d.data_ptr()))
        N.call("hsv_synchronize")
        acc += d.cpu().numpy()[2:2 + len(acc)]
    assert np.max(np.abs(acc - full)) <= 1e-13 * max(1.0, np.max(np.abs(full)))


def test_pivot_goldens_h8(N):
    import paper_2604_01176_b200 as hsv
    sysm = hsv.MolecularSystem.bundled("h8")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    ref = load_golden("ref_h8")
    st = eng.rebuild([pool.ops[i] for i in ref["s2_ops"]], ref["s2_thetas"])
    for pv in (-1, 1):
        N.call("hsv_set_tuning", b"screen_pivot", pv)
        assert rel_err(eng.screen(st, pool), ref["g_s2"]) <= 1e-10
