#!/usr/bin/env python3
"""Kernel micro-benchmark: per-kernel device time (live CUDA events) of the
K1 apply and K4 screen kernels over tuning variants, on bundled systems.

  python tools/kbench.py --systems h10 h12 --apply-r 1 2 4 --reps 5
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_01176_b200 as hsv  # noqa: E402
from paper_2604_01176_b200 import _native as N  # noqa: E402
from paper_2604_01176_b200.svengine import DevicePool, DeviceState  # noqa: E402


def prof(name):
    t, c = N.dbl(), N.i64()
    N.call("hsv_prof_get", name.encode(), N.C.byref(t), N.C.byref(c))
    return t.value / max(c.value, 1), c.value


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--systems", nargs="+", default=["h12"])
    ap.add_argument("--apply-r", nargs="+", type=int, default=[0])
    ap.add_argument("--minb", nargs="+", type=int, default=[0])
    ap.add_argument("--screen-rows", nargs="+", type=int, default=[1024])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--lib", default=None, help="alternative libhsv build (A/B runs)")
    args = ap.parse_args()
    if args.lib:
        N.load(args.lib)
    N.init(0)
    for name in args.systems:
        sysm = hsv.MolecularSystem.bundled(name)
        basis = sysm.basis
        dim = len(basis)
        op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, basis)
        pool = DevicePool(basis, hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec).ops)
        v = np.random.default_rng(20240811).standard_normal(dim)
        v /= np.linalg.norm(v)
        st = hsv.SvState(basis, hsv.SparseVector(dim, np.arange(dim, dtype=np.int64), v))
        nnz = op.nnz
        info = op.info()
        for r, sr, mb in [(r, sr, mb) for r in args.apply_r for sr in args.screen_rows
                          for mb in args.minb]:
            if True:
                N.call("hsv_set_tuning", b"apply_r", r)
                N.call("hsv_set_tuning", b"apply_minb", mb)
                N.call("hsv_set_tuning", b"screen_rows", sr)
                e, g = op.energy_screen_pool(st, pool)          # warm
                N.call("hsv_prof_reset")
                N.call("hsv_prof_enable", 1)
                for _ in range(args.reps):
                    e, g = op.energy_screen_pool(st, pool)
                N.call("hsv_prof_collect")
                N.call("hsv_prof_enable", 0)
                ta, _ = prof("apply")
                ts, _ = prof("screen")
                bytes_apply = 16.0 * nnz + 24.0 * dim
                print(json.dumps({
                    "system": name, "dim": dim, "apply_r": r, "minb": mb, "screen_rows": sr,
                    "apply_ms": ta, "screen_ms": ts, "apply_GBs_alg": bytes_apply / ta / 1e6,
                    "energy": e, "gmax": float(np.max(np.abs(g))), "nnz": nnz, **info}),
                    flush=True)


if __name__ == "__main__":
    main()
