#!/usr/bin/env python3
"""Per-kernel device time of one L-BFGS evaluation (energy_and_gradient) along
the committed H12 ADAPT trace, for the sweep / K1 variants:

  python tools/sweep_probe.py --depths 100 200 400 --variants sweep=2 sweep=1 restrict_rows=0
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

KERNELS = ("qeb", "adjoint", "apply_rows", "apply", "push", "push_collect", "sup_build",
           "h:eg_fwd", "h:fwd_psi", "h:get_plan", "h:k1r_launch", "h:eg_bwd", "h:bwd_wait")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--system", default="h12")
    ap.add_argument("--depths", nargs="+", type=int, default=[100, 200, 400])
    ap.add_argument("--variants", nargs="+", default=["sweep=2", "sweep=1"])
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    N.init(0)
    tr = np.load(ROOT / "tests" / "golden" / f"trace_{args.system}_416.npz"
                 if args.system == "h12" else ROOT / "tests" / "golden" / f"trace_{args.system}.npz")
    sysm = hsv.MolecularSystem.bundled(args.system)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    ops = [pool.ops[i] for i in tr["selected"]]
    for k in args.depths:
        th = np.asarray(tr[f"thetas_at_{k}"] if f"thetas_at_{k}" in tr.files else tr["thetas"][:k])
        for var in args.variants:
            kv = [x.split("=") for x in var.split(",")]
            for key, v in kv:
                N.call("hsv_set_tuning", key.encode(), int(v))
            e0, g0 = eng.energy_and_gradient(ops[:k], th)       # warm-up (plan, pools)
            N.call("hsv_prof_reset")
            N.call("hsv_prof_enable", 1)
            st = (N.i64 * 8)()
            N.call("hsv_stats", None, 1)
            t0 = time.perf_counter()
            for _ in range(args.reps):
                e, g = eng.energy_and_gradient(ops[:k], th)
            wall = (time.perf_counter() - t0) / args.reps
            N.call("hsv_prof_collect")
            N.call("hsv_prof_enable", 0)
            N.call("hsv_stats", st, 1)
            ms = {}
            for kn in KERNELS:
                t, c = N.dbl(), N.i64()
                N.call("hsv_prof_get", kn.encode(), N.C.byref(t), N.C.byref(c))
                ms[kn] = round(t.value / args.reps, 4)
            print(json.dumps({"k": k, "variant": var, "eval_ms_wall": wall * 1e3,
                              "kernel_ms": ms, "E": e, "gmax": float(np.max(np.abs(g))),
                              "pairs_fwd": st[0] // args.reps, "pairs_adj": st[1] // args.reps,
                              "k1r_rows": st[2] // args.reps}), flush=True)
            for key, v in kv:   # back to defaults
                N.call("hsv_set_tuning", key.encode(),
                       {"sweep": 2, "restrict_rows": -1, "push": -1, "sweep_p2p": 0,
                        "apply_v": 0, "apply_t": 0, "sweep_grid": 0,
                        "sweep_bar": 0, "sweep_threads": 256, "sup": -1,
                        "sell": -1}.get(key, -1))


if __name__ == "__main__":
    main()
