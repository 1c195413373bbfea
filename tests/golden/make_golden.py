"""Generate the committed golden fixtures by running the UNMODIFIED reference.

Run in the build container (the reference is importable there, not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (all small, committed):
  ../../paper_2604_01176_b200/data/ham_h{2..16}.npz   Jordan-Wigner Pauli sums from the reference's own builder
                     (`svmps.system.MolecularSystem.from_fcidump`, system.py:43-45);
                     H14/H16 FCIDUMPs come from `scripts/make_fixtures.build` (offline).
  ref_h{2..10}.npz   reference outputs of the SV hot path on seeded states:
                     expectation / spmspv (svengine.py:174, sparse.py:177-201),
                     SvAdaptEngine.screen (adapt.py:212-214),
                     apply_qeb_exponential (svengine.py:209-237),
                     apply_generator (svengine.py:187-206),
                     ansatz_energy_gradient (svengine.py:260-281).
  adapt_h4.npz, adapt_h6.npz   run_adapt traces (adapt.py:570-664) for replay parity.

States are NOT stored when they can be regenerated from a seed on the GPU box
(numpy's default_rng streams are platform independent); only outputs are.
"""
from __future__ import annotations

import importlib.util
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_SCRIPTS = Path("/root/reference/pkg/scripts")
sys.path.insert(0, str(REF_SRC))

from svmps import oracle  # noqa: E402
from svmps.adapt import AdaptConfig, SvAdaptEngine, build_qeb_pool, run_adapt  # noqa: E402
from svmps.sparse import SparseVector, normalize, spmspv  # noqa: E402
from svmps.svengine import (  # noqa: E402
    SvState,
    ansatz_energy_gradient,
    apply_ansatz,
    apply_generator,
    apply_qeb_exponential,
    assemble_subspace_hamiltonian,
    expectation,
)
from svmps.system import MolecularSystem, bundled_fcidump  # noqa: E402

OUT = Path(__file__).resolve().parent
HAM_OUT = OUT.parents[1] / "paper_2604_01176_b200" / "data"
ORDER_CODE = {"interleaved": 0, "blocked": 1}
S1_SEED = 20240811
S2_SEED = 1


def save_hamiltonian(name: str, system: MolecularSystem):
    h = system.hamiltonian
    np.savez_compressed(
        HAM_OUT / f"ham_{name}.npz",
        n_qubits=system.n_qubits, n_alpha=system.n_alpha, n_beta=system.n_beta,
        nelec=system.integrals.nelec, ms2=system.integrals.ms2,
        hf_bits=np.uint64(system.hf.bits), ordering=ORDER_CODE[system.ordering],
        xs=h.xs, zs=h.zs, coeffs=h.coeffs,
    )


def s1_state(basis):
    rng = np.random.default_rng(S1_SEED)
    return SvState(basis, normalize(SparseVector.from_dense(rng.standard_normal(len(basis)))))


def s2_ops(pool, k):
    rng = np.random.default_rng(S2_SEED)
    idx = rng.integers(0, len(pool), size=k)
    thetas = rng.uniform(-0.2, 0.2, size=k)
    return idx, thetas


def reference_outputs(name: str, system: MolecularSystem, full_hpsi: bool):
    t0 = time.time()
    basis = system.basis
    engine = SvAdaptEngine(system, AdaptConfig(engine="sv"))
    m = engine.matrix
    pool = build_qeb_pool(system.n_qubits, system.integrals.nelec, system.ordering,
                          system.integrals.ms2)
    out = {"dim": len(basis), "csr_nnz": m.nnz}
    if len(basis) <= 400:   # full reference CSR: matrix elements checked bit for bit
        out["csr_ro"], out["csr_ci"], out["csr_v"] = m.row_offsets, m.col_indices, m.values
    # HF
    hf = engine.initial_state()
    out["e_hf"] = engine.energy(hf)
    out["g_hf"] = engine.screen(hf, pool)
    if len(basis) <= 70000:
        out["e_fci"] = oracle.fci_ground_energy(m, cross_check=False)[0]
    # S1 dense-in-sector
    s1 = s1_state(basis)
    w1 = spmspv(m, s1.vec)
    out["e_s1"] = float(np.dot(s1.vec.values, w1.to_dense()[s1.vec.indices]))
    out["e_s1_expect"] = expectation(m, s1)
    out["g_s1"] = engine.screen(s1, pool)
    if full_hpsi:
        out["hs1_idx"], out["hs1_val"] = w1.indices, w1.values
    else:
        sel = np.arange(0, w1.nnz, 37)
        out["hs1_nnz"] = w1.nnz
        out["hs1_sample_idx"], out["hs1_sample_val"] = w1.indices[sel], w1.values[sel]
    # S2 ADAPT-like (k=20)
    k = 20
    idx, thetas = s2_ops(pool, k)
    ops = [pool.ops[i] for i in idx]
    s2 = apply_ansatz(basis, system.hf, ops, thetas)
    out["s2_ops"], out["s2_thetas"] = idx, thetas
    out["s2_idx"], out["s2_val"] = s2.vec.indices, s2.vec.values
    w2 = spmspv(m, s2.vec)
    out["hs2_idx"], out["hs2_val"] = w2.indices, w2.values
    out["e_s2"] = expectation(m, s2)
    out["g_s2"] = engine.screen(s2, pool)
    e, g = ansatz_energy_gradient(m, basis, system.hf, ops, thetas)
    out["eg_s2_e"], out["eg_s2_g"] = e, g
    # Single-op kernels on S1 (QEB bit-exact, generator exact)
    rng = np.random.default_rng(7)
    qeb_ops = rng.integers(0, len(pool), size=6)
    qeb_th = rng.uniform(-3, 3, size=6)
    out["qeb_ops"], out["qeb_thetas"] = qeb_ops, qeb_th
    for j, (oi, th) in enumerate(zip(qeb_ops, qeb_th)):
        r = apply_qeb_exponential(pool.ops[oi], float(th), s1)
        out[f"qeb{j}_idx"], out[f"qeb{j}_val"] = r.vec.indices, r.vec.values
        gvec = apply_generator(pool.ops[oi], s2)
        out[f"gen{j}_idx"], out[f"gen{j}_val"] = gvec.indices, gvec.values
    np.savez_compressed(OUT / f"ref_{name}.npz", **out)
    print(f"{name}: dim={len(basis)} nnz={m.nnz} pool={len(pool)} "
          f"E_hf={out['e_hf']:.12f} E_s1={out['e_s1_expect']:.12f} ({time.time()-t0:.1f}s)")


def adapt_trace(name: str, system: MolecularSystem, eps: float, max_iter: int):
    fci = oracle.fci_ground_energy(assemble_subspace_hamiltonian(system.hamiltonian,
                                                                 system.basis))[0]
    res = run_adapt(AdaptConfig(engine="sv", eps_grad=eps, max_iter=max_iter), system,
                    reference_energy=fci)
    pool = build_qeb_pool(system.n_qubits, system.integrals.nelec, system.ordering,
                          system.integrals.ms2)
    labels = [op.label() for op in pool]
    np.savez_compressed(
        OUT / f"adapt_{name}.npz",
        eps=eps, max_iter=max_iter, e_fci=fci, status=res.status,
        it=np.array([r.iteration for r in res.records]),
        energy=np.array([r.energy for r in res.records]),
        grad_max=np.array([r.grad_max for r in res.records]),
        nnz=np.array([r.nnz for r in res.records]),
        evals=np.array([r.energy_evals for r in res.records]),
        selected=np.array([labels.index(r.selected_op) if r.selected_op else -1
                           for r in res.records]),
        thetas=res.thetas,
        wall_s=np.array([r.wall_elapsed for r in res.records]),   # this container's CPU
    )
    print(f"adapt {name}: {len(res.records)} records, status={res.status}, "
          f"E={res.records[-1].energy:.12f}")


def main():
    systems = {}
    for n in (2, 4, 6, 8, 10, 12):
        name = f"h{n}"
        systems[name] = MolecularSystem.from_fcidump(bundled_fcidump(name))
        save_hamiltonian(name, systems[name])
    spec = importlib.util.spec_from_file_location("make_fixtures", REF_SCRIPTS / "make_fixtures.py")
    mf = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mf)
    with tempfile.TemporaryDirectory() as tmp:
        for n in (14, 16):
            mf.build(n, Path(tmp))
            sysn = MolecularSystem.from_fcidump(Path(tmp) / f"h{n}.fcidump")
            save_hamiltonian(f"h{n}", sysn)
    for name in ("h2", "h4", "h6", "h8"):
        reference_outputs(name, systems[name], full_hpsi=True)
    reference_outputs("h10", systems["h10"], full_hpsi=False)
    adapt_trace("h4", systems["h4"], 1e-6, 25)
    adapt_trace("h6", systems["h6"], 1e-4, 12)


if __name__ == "__main__":
    main()
