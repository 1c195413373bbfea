"""The library's device arena (csrc/hsv_core.cu cache_alloc): scratch is
reused without going back to the driver once warm, hsv_mem_trim returns the
wholly idle chunks, and results are unchanged after a trim (buffers rebuilt)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def stats(N):
    st = (N.i64 * 8)()
    N.call("hsv_stats", st, 0)
    return {"idle": st[4], "driver_allocs": st[5]}


def test_arena_reuse_and_trim():
    import paper_2604_01176_b200 as hsv
    from paper_2604_01176_b200 import _native as N
    sysm = hsv.MolecularSystem.bundled("h10")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    rng = np.random.default_rng(3)
    ops = [pool.ops[i] for i in rng.integers(0, len(pool), size=30)]
    th = rng.uniform(-0.3, 0.3, size=30)
    e0, g0 = eng.energy_and_gradient(ops, th)          # warm: plans, assembled rows, scratch
    before = stats(N)
    for _ in range(5):
        e, g = eng.energy_and_gradient(ops, th)
        assert e == e0 and np.array_equal(g, g0)
    after = stats(N)
    assert after["driver_allocs"] == before["driver_allocs"]   # warm: no driver allocation
    N.call("hsv_mem_trim")
    trimmed = stats(N)
    assert trimmed["idle"] <= after["idle"]
    e, g = eng.energy_and_gradient(ops, th)            # still correct after giving memory back
    assert e == e0 and np.array_equal(g, g0)
