#!/usr/bin/env python3
"""ADAPT-VQE timing on the device engine.

* one L-BFGS evaluation (`energy_and_gradient`, adjoint sweep) at k = 20 / 100
  random pool operators (default_rng(1), theta ~ U(-0.2, 0.2): SURVEY.md 8(d) S2),
* the full ADAPT loop (`run_adapt`, engine "sv") for --iters iterations:
  wall time per outer iteration and L-BFGS evaluations per iteration.

  python tools/adapt_bench.py --systems h10 h12 --iters 12
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--systems", nargs="+", default=["h10", "h12"])
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--ks", nargs="+", type=int, default=[20, 100])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tune", nargs="*", default=[], help="hsv_set_tuning key=value pairs")
    ap.add_argument("--no-loop", action="store_true", help="skip the full ADAPT loop")
    args = ap.parse_args()
    N.init(0)
    for kv in args.tune:
        key, val = kv.split("=")
        N.call("hsv_set_tuning", key.encode(), int(val))
    for name in args.systems:
        sysm = hsv.MolecularSystem.bundled(name)
        eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
        pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
        for k in args.ks:
            rng = np.random.default_rng(1)
            idx = rng.integers(0, len(pool), size=k)
            th = rng.uniform(-0.2, 0.2, size=k)
            ops = [pool.ops[i] for i in idx]
            eng.energy_and_gradient(ops, th)
            N.call("hsv_prof_reset")
            N.call("hsv_prof_enable", 1)
            walls = []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                e, g = eng.energy_and_gradient(ops, th)
                walls.append(time.perf_counter() - t0)
            N.call("hsv_prof_collect")
            N.call("hsv_prof_enable", 0)
            kern = {}
            for kn in ("apply", "push", "push_collect", "qeb", "adjoint"):
                t, c = N.dbl(), N.i64()
                N.call("hsv_prof_get", kn.encode(), N.C.byref(t), N.C.byref(c))
                kern[kn] = round(t.value / args.reps, 4)
            print(json.dumps({"system": name, "k": k, "eval_ms": float(np.mean(walls)) * 1e3,
                              "eval_ms_median": float(np.median(walls)) * 1e3,
                              "eval_ms_max": float(np.max(walls)) * 1e3,
                              "kernel_ms_per_eval": kern, "energy": e, "tune": args.tune}),
                  flush=True)
        if args.no_loop:
            continue
        recs = []
        N.call("hsv_prof_reset")
        N.call("hsv_prof_enable", 1)
        N.lib().hsv_launch_count(1)
        t0 = time.perf_counter()
        res = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=1e-6, max_iter=args.iters),
                            sysm, engine=eng, progress=recs.append)
        N.call("hsv_prof_collect")
        N.call("hsv_prof_enable", 0)
        kern = {}
        for kn in ("apply", "push", "push_collect", "screen", "qeb", "adjoint"):
            t, c = N.dbl(), N.i64()
            N.call("hsv_prof_get", kn.encode(), N.C.byref(t), N.C.byref(c))
            kern[kn] = {"ms": round(t.value, 2), "launches": c.value}
        print(json.dumps({"system": name, "adapt_kernel_totals": kern,
                          "all_launches": int(N.lib().hsv_launch_count(1))}), flush=True)
        wall = [r.wall_elapsed for r in res.records]
        it_t = np.diff(wall)
        evals = np.diff([r.energy_evals for r in res.records])
        half = len(it_t) // 2
        print(json.dumps({
            "system": name, "adapt_iters": len(it_t), "status": res.status,
            "iter_s_mean_last_half": float(np.mean(it_t[half:])) if len(it_t) else None,
            "iter_s": [round(x, 4) for x in it_t.tolist()],
            "evals_per_iter": evals.tolist(),
            "energy": res.records[-1].energy, "nnz": res.records[-1].nnz,
            "total_s": time.perf_counter() - t0}), flush=True)


if __name__ == "__main__":
    main()
