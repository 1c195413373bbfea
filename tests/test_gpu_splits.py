"""K1 bucket split tables (hsv_apply.cu: split parts of 2..32, the 16/32 tables
cut inside buckets as "virtual buckets").

Every split count must cover each (row, group) pair exactly once, with the
diagonal added once: rows of H|psi> agree with the unsplit kernel to rounding
(the parts are summed in split order, a different association), the energy to
1e-13, and the goldens to 1e-10.  Row shards (owner-computes ranges, where the
auto rule picks 16 or 32 parts) reproduce the full rows.
"""
import numpy as np
import pytest

from conftest import load_golden, rel_err, s1_values

pytestmark = pytest.mark.gpu

SPLITS = (1, 2, 4, 8, 16, 32)


@pytest.fixture(scope="module")
def hsv():
    import paper_2604_01176_b200 as hsv
    return hsv


@pytest.fixture()
def N():
    from paper_2604_01176_b200 import _native as N
    N.call("hsv_set_tuning", b"apply_v", 0)      # these tests target the register-row K1
    yield N
    N.call("hsv_set_tuning", b"apply_split", 0)
    N.call("hsv_set_tuning", b"apply_r", 0)
    N.call("hsv_set_tuning", b"apply_v", -1)


def dense_state(hsv, sysm):
    dim = len(sysm.basis)
    return hsv.SvState(sysm.basis, hsv.SparseVector(dim, np.arange(dim, dtype=np.int64),
                                                    s1_values(dim)))


def rows_of(N, op, st, split, r=0):
    from paper_2604_01176_b200.svengine import DeviceState
    N.call("hsv_set_tuning", b"apply_split", split)
    N.call("hsv_set_tuning", b"apply_r", r)
    out = DeviceState(st.basis)
    N.call("hsv_state_zero", out.handle)
    na = st.basis._sector.n_alpha_strings
    N.call("hsv_apply_h_rows_async", op.handle, st.device.handle, out.handle, 0, na, 0.0)
    N.call("hsv_synchronize")
    return out.torch_view().cpu().numpy(), op.expect(st)


@pytest.mark.parametrize("name", ["h6", "h8", "h10"])
def test_every_split_count_matches_unsplit(hsv, N, name):
    sysm = hsv.MolecularSystem.bundled(name)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    base, e0 = rows_of(N, op, st, 1)
    scale = np.abs(base).max()
    for r in (2, 8):
        for split in SPLITS:
            y, e = rows_of(N, op, st, split, r)
            assert np.abs(y - base).max() <= 1e-13 * scale, (split, r)
            assert abs(e - e0) <= 1e-13 * abs(e0), (split, r)


def test_split_goldens_h8(hsv, N):
    sysm = hsv.MolecularSystem.bundled("h8")
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    ref = load_golden("ref_h8")
    st = dense_state(hsv, sysm)
    for split in (16, 32):
        N.call("hsv_set_tuning", b"apply_split", split)
        w = op.apply_state(st).to_sparse()
        assert np.array_equal(w.indices, ref["hs1_idx"]), split
        assert rel_err(w.values, ref["hs1_val"]) <= 1e-10, split


def test_row_shards_reproduce_full_rows(hsv, N):
    """Shards of an 8- and 16-way owner-computes split (auto rule: 16-32 parts)."""
    from paper_2604_01176_b200.svengine import DeviceState
    sysm = hsv.MolecularSystem.bundled("h10")
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    full, _ = rows_of(N, op, st, 0)
    N.call("hsv_set_tuning", b"apply_split", 0)
    na = sysm.basis._sector.n_alpha_strings
    scale = np.abs(full).max()
    for parts in (8, 16):
        out = DeviceState(sysm.basis)
        N.call("hsv_state_zero", out.handle)
        for k in range(parts):
            lo, hi = k * na // parts, (k + 1) * na // parts
            N.call("hsv_apply_h_rows_async", op.handle, st.device.handle, out.handle, lo, hi, 0.0)
        N.call("hsv_synchronize")
        y = out.torch_view().cpu().numpy()
        assert np.abs(y - full).max() <= 1e-13 * scale, parts


@pytest.mark.parametrize("name", ["h8", "h10", "h12"])
def test_rb0_shared_memory_is_bitwise_equal(hsv, N, name):
    """K1 with the pass-1 rank table Rb0 staged in shared memory (tuning
    rb0_smem = 1, opt-in) reads the same ranks as the global-memory
    lookup: rows and energy bitwise equal, with and without bucket splits."""
    sysm = hsv.MolecularSystem.bundled(name)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    try:
        for split in (1, 8):
            N.call("hsv_set_tuning", b"rb0_smem", 0)
            y0, e0 = rows_of(N, op, st, split, 8)
            N.call("hsv_set_tuning", b"rb0_smem", 1)
            y1, e1 = rows_of(N, op, st, split, 8)
            assert np.array_equal(y0, y1) and e0 == e1, (name, split)
    finally:
        N.call("hsv_set_tuning", b"rb0_smem", 0)


@pytest.mark.parametrize("name", ["h8", "h10", "h12"])
def test_bperm_is_bitwise_equal(hsv, N, name):
    """K1 pass-1 partner ranks from the per-xb 16-bit permutation rows (tuning
    bperm, on by default where built) equal the Rb0 gather: rows and energy
    bitwise, with and without bucket splits.  The permutation rows are used by
    the R = 8 kernel only (hsv_apply.cu launch_apply), so R = 8 is the case."""
    sysm = hsv.MolecularSystem.bundled(name)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    st = dense_state(hsv, sysm)
    try:
        for split, r in ((1, 8), (8, 8), (32, 8)):
            N.call("hsv_set_tuning", b"bperm", 0)
            y0, e0 = rows_of(N, op, st, split, r)
            N.call("hsv_set_tuning", b"bperm", 1)
            y1, e1 = rows_of(N, op, st, split, r)
            assert np.array_equal(y0, y1) and e0 == e1, (name, split, r)
    finally:
        N.call("hsv_set_tuning", b"bperm", -1)
