"""K1s (TMA-staged partner rows, hsv_apply_staged.cu; opt-in via
hsv_set_tuning("staged", 1)) against the K1 pull kernel: same bucket split =>
bitwise identical rows of H|psi>; energies agree to 1e-14 (different
partial-sum grouping); row-range shards; screen and adjoint parity."""
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
    for k, v in ((b"staged", 0), (b"push", -1), (b"apply_split", 0)):
        N.call("hsv_set_tuning", k, v)


def states(hsv, sysm, rng):
    basis = sysm.basis
    dim = len(basis)
    out = [hsv.SvState(basis, hsv.SparseVector(dim, np.arange(dim, dtype=np.int64),
                                              s1_values(dim)))]
    v = rng.standard_normal(dim) + 1j * rng.standard_normal(dim)
    out.append(hsv.SvState(basis, hsv.SparseVector(dim, np.arange(dim, dtype=np.int64),
                                                  v / np.linalg.norm(v))))
    return out


@pytest.mark.parametrize("name", ["h4", "h6", "h8", "h10", "h12"])
def test_staged_rows_bitwise_equal_pull(hsv, N, name):
    sysm = hsv.MolecularSystem.bundled(name)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    rng = np.random.default_rng(2)
    N.call("hsv_set_tuning", b"push", 0)
    for st in states(hsv, sysm, rng):
        for split in (1, 2, 4):
            N.call("hsv_set_tuning", b"apply_split", split)
            res = []
            for staged in (1, 0):
                N.call("hsv_set_tuning", b"staged", staged)
                w = op.apply_state(st).to_sparse()
                res.append((w, op.expect(st)))
            (w1, e1), (w0, e0) = res
            assert np.array_equal(w1.indices, w0.indices)
            assert np.array_equal(w1.values, w0.values), (name, split)
            assert abs(e1 - e0) <= 1e-14 * max(1.0, abs(e0))


def test_staged_row_ranges(hsv, N):
    from paper_2604_01176_b200.svengine import DeviceState
    sysm = hsv.MolecularSystem.bundled("h10")
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = states(hsv, sysm, np.random.default_rng(3))[1]
    na = sysm.basis._sector.n_alpha_strings
    N.call("hsv_set_tuning", b"push", 0)
    N.call("hsv_set_tuning", b"apply_split", 2)
    for lo, hi in ((0, na), (0, na // 3), (na // 3, na - 7), (na - 1, na)):
        res = []
        for staged in (1, 0):
            N.call("hsv_set_tuning", b"staged", staged)
            out = DeviceState(sysm.basis)
            N.call("hsv_state_zero", out.handle)
            N.call("hsv_apply_h_rows_async", op.handle, st.device.handle, out.handle, lo, hi, 0.0)
            N.call("hsv_synchronize")
            res.append(out.torch_view().cpu().numpy())
        assert np.array_equal(res[0], res[1]), (lo, hi)


def test_staged_screen_and_gradient_parity(hsv, N):
    """The bench step (energy + all gradients) and the adjoint gradient through K1s."""
    from conftest import load_golden, rel_err
    sysm = hsv.MolecularSystem.bundled("h10")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    ref = load_golden("ref_h10")
    st = states(hsv, sysm, np.random.default_rng(0))[0]
    N.call("hsv_set_tuning", b"push", 0)
    N.call("hsv_set_tuning", b"staged", 1)
    assert rel_err(eng.screen(st, pool), ref["g_s1"]) <= 1e-10
    ops = [pool.ops[i] for i in ref["s2_ops"]]
    e, g = eng.energy_and_gradient(ops, ref["s2_thetas"])
    assert abs(e - float(ref["eg_s2_e"])) <= 1e-10 * abs(e)
    assert rel_err(g, ref["eg_s2_g"]) <= 1e-10
