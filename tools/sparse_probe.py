#!/usr/bin/env python3
"""K1 apply time against the support of psi (ADAPT-like sparse states).

States are HF followed by the first k operators an ADAPT run selects (or
random pool operators with --random), theta ~ U(-0.2, 0.2).

  python tools/sparse_probe.py --system h12 --ks 1 2 4 8 16 32 64
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_01176_b200 as hsv  # noqa: E402
from paper_2604_01176_b200 import _native as N  # noqa: E402


def prof(name):
    t, c = N.dbl(), N.i64()
    N.call("hsv_prof_get", name.encode(), N.C.byref(t), N.C.byref(c))
    return t.value / max(c.value, 1), c.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--system", default="h12")
    ap.add_argument("--ks", nargs="+", type=int, default=[1, 2, 4, 8, 16, 32, 64])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--lib", default=None)
    ap.add_argument("--push", type=int, default=-1, help="hsv_set_tuning push (-1 auto, 0 off, 1 on)")
    ap.add_argument("--push-keys", type=int, default=None)
    args = ap.parse_args()
    if args.lib:
        N.load(args.lib)
    N.init(0)
    N.call("hsv_set_tuning", b"push", args.push)
    if args.push_keys is not None:
        N.call("hsv_set_tuning", b"push_keys", args.push_keys)
    sysm = hsv.MolecularSystem.bundled(args.system)
    basis = sysm.basis
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, basis)
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec).ops
    rng = np.random.default_rng(7)
    for k in args.ks:
        idx = rng.integers(0, len(pool), size=k)
        th = rng.uniform(-0.2, 0.2, size=k)
        st = hsv.apply_ansatz(basis, sysm.hf, [pool[i] for i in idx], th)
        nnz = st.nnz
        op.apply_state(st)
        N.call("hsv_prof_reset")
        N.call("hsv_prof_enable", 1)
        t0 = time.perf_counter()
        for _ in range(args.reps):
            op.apply_state(st)
        wall = time.perf_counter() - t0
        N.call("hsv_prof_collect")
        N.call("hsv_prof_enable", 0)
        ms, cnt = prof("apply")
        pms, pcnt = prof("push")
        cms, ccnt = prof("push_collect")
        print(json.dumps({"system": args.system, "k": k, "nnz": int(nnz),
                          "apply_ms": round(ms * cnt / args.reps, 4),
                          "push_ms": round(pms * pcnt / args.reps, 4),
                          "collect_ms": round(cms * ccnt / args.reps, 4),
                          "wall_ms": round(wall * 1e3 / args.reps, 4),
                          "e": op.expect(st)}), flush=True)


if __name__ == "__main__":
    main()
