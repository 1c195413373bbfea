"""Golden vectors written by the UNMODIFIED reference at H10 / H12.

Runs the staged reference package (oracle/_ref, oracle/stage_reference.py)
through its own public API.  H12's CSR assembly needs ~63 GB of host RAM
(SURVEY.md 8c), so the H12 file is produced on the GPU box's host (196 GB);
H10 fits anywhere.  Nothing here touches the device engine.

    PYTHONPATH=oracle/_ref python tests/golden/make_golden_refbox.py --system h12

Writes tests/golden/refbox_<system>.npz:
  csr_nnz, t_assembly_s                 reference assemble_subspace_hamiltonian
  e_s1, g_s1                            expectation + pool_gradients on S1
  hs1_nnz, hs1_idx_sha256               full support of H|S1> (bit-exact key check)
  hs1_rows, hs1_rows_val, hs1_norm2     values at every 97th support entry + ||H psi||^2
  e_hf, g_hf                            HF energy and screen
  eg_k, eg_e, eg_g                      ansatz_energy_gradient along the device
                                        engine's own H12/H10 ADAPT trace
                                        (tests/golden/trace_<system>.npz) at depths k
  psi_k_idx_sha256, psi_k_val_sha256    apply_ansatz state at depth k (bit-exact)
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT / "oracle" / "_ref"))

from svmps.adapt import AdaptConfig, SvAdaptEngine, build_qeb_pool  # noqa: E402
from svmps.sparse import SparseVector, normalize, spmspv  # noqa: E402
from svmps.svengine import (SvState, ansatz_energy_gradient, apply_ansatz,  # noqa: E402
                            assemble_subspace_hamiltonian, expectation, pool_gradients)
from svmps.system import MolecularSystem, bundled_fcidump  # noqa: E402

S1_SEED = 20240811


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--system", default="h12")
    ap.add_argument("--depths", type=int, nargs="*", default=None)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    t0 = time.time()
    s = MolecularSystem.from_fcidump(bundled_fcidump(a.system))
    basis = s.basis
    dim = len(basis)
    pool = build_qeb_pool(s.n_qubits, s.integrals.nelec, s.ordering, s.integrals.ms2)
    m = assemble_subspace_hamiltonian(s.hamiltonian, basis)
    out = {"dim": dim, "csr_nnz": m.nnz, "t_assembly_s": time.time() - t0}
    print(f"assembly {out['t_assembly_s']:.1f}s nnz {m.nnz}", flush=True)
    nw = a.threads
    rng = np.random.default_rng(S1_SEED)
    psi = SvState(basis, normalize(SparseVector.from_dense(rng.standard_normal(dim))))
    out["e_s1"] = expectation(m, psi, n_workers=nw)
    w = spmspv(m, psi.vec, n_workers=nw)
    out["hs1_nnz"] = w.nnz
    out["hs1_idx_sha256"] = sha(w.indices.astype(np.int64))
    sel = np.arange(0, w.nnz, 97)
    out["hs1_rows"], out["hs1_rows_val"] = w.indices[sel], w.values[sel]
    out["hs1_norm2"] = float(w.values @ w.values)
    t1 = time.time()
    out["g_s1"] = pool_gradients(m, psi, pool.ops, n_workers=nw)
    print(f"S1 screen {time.time() - t1:.1f}s", flush=True)
    eng = SvAdaptEngine.__new__(SvAdaptEngine)
    eng.system, eng.basis, eng.matrix, eng.threads = s, basis, m, nw
    hf = eng.initial_state()
    out["e_hf"] = eng.energy(hf)
    out["g_hf"] = eng.screen(hf, pool)
    tr_path = HERE / f"trace_{a.system}.npz"
    if tr_path.exists():
        tr = np.load(tr_path)
        ops = [pool.ops[i] for i in tr["selected"]]
        th = np.asarray(tr["thetas"], dtype=np.float64)
        depths = a.depths or [d for d in (20, 100, 200, 400) if d <= len(ops)]
        eg_e, eg_g, sh_i, sh_v, nnz = [], [], [], [], []
        for k in depths:
            t1 = time.time()
            st = apply_ansatz(basis, s.hf, ops[:k], th[:k])
            sh_i.append(sha(st.vec.indices.astype(np.int64)))
            sh_v.append(sha(st.vec.values.astype(np.float64)))
            nnz.append(st.vec.nnz)
            e, g = ansatz_energy_gradient(m, basis, s.hf, ops[:k], th[:k], n_workers=nw)
            eg_e.append(e)
            eg_g.append(np.pad(g, (0, max(depths) - k)))
            print(f"depth {k}: nnz {st.vec.nnz} E {e:.15f} ({time.time() - t1:.1f}s)", flush=True)
        out.update(eg_k=np.array(depths), eg_e=np.array(eg_e), eg_g=np.array(eg_g),
                   psi_k_idx_sha256=np.array(sh_i), psi_k_val_sha256=np.array(sh_v),
                   psi_k_nnz=np.array(nnz))
    np.savez(HERE / f"refbox_{a.system}.npz", **out)
    print(f"done {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
