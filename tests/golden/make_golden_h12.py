"""H12 golden vectors from the CPU oracle (matrix-free restatement).

The reference's CSR assembly needs ~63 GB of host RAM at H12 (SURVEY.md
section 8c), so H12 goldens come from oracle/sv_oracle.py, which
tests/test_oracle.py pins bit-for-bit (CSR path) and to 1e-10 (matrix-free
path) against the reference's own outputs at H2..H10.

    python tests/golden/make_golden_h12.py
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import s1_values  # noqa: E402
from oracle import sv_oracle as O  # noqa: E402
from paper_2604_01176_b200.system import MolecularSystem  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    t0 = time.time()
    s = MolecularSystem.bundled("h12")
    h = s.hamiltonian
    states = O.sector_states(s.n_qubits, s.n_alpha, s.n_beta)
    ops = O.qeb_pool_masks(s.n_qubits, s.integrals.nelec)
    dim = len(states)
    psi = s1_values(dim)
    idx = np.arange(dim, dtype=np.int64)
    y = O.apply_h_matrix_free(h.xs, h.zs, h.coeffs, states, psi)
    print(f"H psi: {time.time() - t0:.1f}s")
    out = {"dim": dim, "e_s1": float(psi @ y), "hs1_nnz": int(np.count_nonzero(y))}
    rows = np.arange(0, dim, 997, dtype=np.int64)
    out["hs1_rows"], out["hs1_rows_val"] = rows, y[rows]
    yi = np.flatnonzero(y).astype(np.int64)
    out["g_s1"] = O.pool_gradients(lambda i, v: (yi, y[yi]), states, idx, psi, ops)
    print(f"S1 screen: {time.time() - t0:.1f}s")
    hf = int(np.searchsorted(states, s.hf.bits))

    def h_apply(i, v):
        d = np.zeros(dim)
        d[i] = v
        w = O.apply_h_matrix_free(h.xs, h.zs, h.coeffs, states, d)
        wi = np.flatnonzero(w).astype(np.int64)
        return wi, w[wi]

    hi, hv = np.array([hf], dtype=np.int64), np.array([1.0])
    wi, wv = h_apply(hi, hv)
    out["e_hf"] = O.dot(hi, hv, wi, wv)
    out["g_hf"] = O.pool_gradients(lambda i, v: (wi, wv), states, hi, hv, ops)
    rng = np.random.default_rng(1)
    k = 20
    sel = rng.integers(0, len(ops), size=k)
    th = rng.uniform(-0.2, 0.2, size=k)
    s2 = [ops[i] for i in sel]
    si, sv = O.apply_ansatz(states, s.hf.bits, s2, th)
    out["s2_ops"], out["s2_thetas"], out["s2_idx"], out["s2_val"] = sel, th, si, sv
    e, g = O.energy_gradient(h_apply, states, s.hf.bits, s2, th)
    out["eg_s2_e"], out["eg_s2_g"] = e, g
    print(f"done: {time.time() - t0:.1f}s  E_s1={out['e_s1']:.15f} E_hf={out['e_hf']:.12f}")
    np.savez_compressed(OUT / "ref_h12.npz", **out)


if __name__ == "__main__":
    main()
