#!/usr/bin/env python3
"""Per-call wall time of the deep H12 ADAPT leg (bench.py adapt_deep): every
energy_and_gradient / screen / energy call is timed, the same resumed
iterations run twice, so one-off costs (first-use loads, pool growth) show up
as a difference between the passes:

  python tools/iter_probe.py --depth 400 --iters 6
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", type=int, default=400)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--passes", type=int, default=2)
    ap.add_argument("--sync", type=int, default=1, help="synchronize after every call")
    args = ap.parse_args()
    tr = np.load(ROOT / "tests" / "golden" / "trace_h12_416.npz")
    sysm = hsv.MolecularSystem.bundled("h12")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    sel = [int(i) for i in tr["selected"]]
    ops = [pool.ops[i] for i in sel]
    k = args.depth
    log = []
    from paper_2604_01176_b200 import _native as N
    import gc
    scopes = ("apply", "apply_rows", "qeb", "adjoint", "screen", "push", "push_collect",
              "sweep_plan")
    N.call("hsv_prof_enable", 1)

    def pool():
        st = (N.i64 * 8)()
        N.call("hsv_stats", st, 0)
        return st[6] >> 20, st[7] >> 20

    def dev_ms():
        N.call("hsv_prof_collect")
        tot = 0.0
        for kn in scopes:
            t, c = N.dbl(), N.i64()
            N.call("hsv_prof_get", kn.encode(), N.C.byref(t), N.C.byref(c))
            tot += t.value
        return tot
    for name in ("energy_and_gradient", "screen", "energy", "rebuild", "state_size"):
        fn = getattr(eng, name, None)
        if fn is None:
            continue

        def wrap(*a, _fn=fn, _name=name, **kw):
            d0 = dev_ms()
            p0 = pool()
            c0 = time.process_time()
            t0 = time.perf_counter()
            r = _fn(*a, **kw)
            if args.sync:
                N.call("hsv_synchronize")
            t1 = time.perf_counter()
            log.append((_name, len(a[0]) if _name == "energy_and_gradient" else -1,
                        round((t1 - t0) * 1e3, 2), round((time.process_time() - c0) * 1e3, 2),
                        round(dev_ms() - d0, 2), p0, pool()))
            return r
        setattr(eng, name, wrap)
    init = (ops[:k], tr[f"thetas_at_{k}"])
    for p in range(args.passes):
        log.clear()
        if p == args.passes - 1 and args.passes > 1:
            gc.disable()
        res = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=float(tr["eps"]),
                                            max_iter=k + args.iters),
                            sysm, engine=eng, replay=sel, initial=init)
        wall = np.diff([r.wall_elapsed for r in res.records]) * 1e3
        print(json.dumps({"pass": p, "iter_ms": [round(float(x), 2) for x in wall],
                          "gc": gc.isenabled(),
                          "calls": log}), flush=True)


if __name__ == "__main__":
    main()
