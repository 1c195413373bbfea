"""hsv_state_set_dense (full-support SparseVector upload, values only) against
hsv_state_set_sparse: identical device state, norm and read-back."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["h4", "h8"])
@pytest.mark.parametrize("cplx", [False, True])
def test_dense_upload_equals_sparse_upload(name, cplx):
    import paper_2604_01176_b200 as hsv
    from paper_2604_01176_b200 import _native as N
    from paper_2604_01176_b200.svengine import DeviceState
    sysm = hsv.MolecularSystem.bundled(name)
    basis = sysm.basis
    dim = len(basis)
    rng = np.random.default_rng(3)
    v = rng.standard_normal(dim) + (1j * rng.standard_normal(dim) if cplx else 0.0)
    idx = np.arange(dim, dtype=np.int64)
    dense = DeviceState.from_sparse(basis, hsv.SparseVector(dim, idx, v))   # dense path
    sparse = DeviceState(basis)
    re, im = N.as_f64(np.real(v)), N.as_f64(np.imag(v))
    N.call("hsv_state_set_sparse", sparse.handle, N.ptr_i64(idx), N.ptr_f64(re),
           N.ptr_f64(im) if cplx else None, dim)
    a = dense.torch_view().cpu().numpy()
    b = sparse.torch_view().cpu().numpy()
    assert np.array_equal(a, b)
    back = dense.to_sparse()
    assert np.array_equal(back.indices, idx)
    assert np.array_equal(back.values, v)
    # a partial support still takes the positions path
    part = DeviceState.from_sparse(basis, hsv.SparseVector(dim, idx[1:], v[1:]))
    c = part.torch_view().cpu().numpy()
    assert np.count_nonzero(np.any(c != 0, axis=1)) == dim - 1
