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
    ap.add_argument("--tune", nargs="*", default=[], help="KEY=V library tuning keys")
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
    extra = ("es_all", "es_arow", "es_k1", "es_k4")
    N.call("hsv_prof_enable", 1)

    from cuda.bindings import runtime as rt
    N.init(0)
    for kv in args.tune:
        key, v = kv.split("=")
        N.call("hsv_set_tuning", key.encode(), int(v))
    ev0 = rt.cudaEventCreate()[1]
    ev1 = rt.cudaEventCreate()[1]

    def pool():
        st = (N.i64 * 8)()
        N.call("hsv_stats", st, 0)
        return st[6] >> 20, st[7] >> 20

    def dev_ms(each=False):
        N.call("hsv_prof_collect")
        tot, d = 0.0, {}
        for kn in scopes + extra:
            t, c = N.dbl(), N.i64()
            N.call("hsv_prof_get", kn.encode(), N.C.byref(t), N.C.byref(c))
            if kn in scopes:
                tot += t.value
            d[kn] = t.value
        return d if each else tot
    for name in ("energy_and_gradient", "screen", "energy", "rebuild", "state_size"):
        fn = getattr(eng, name, None)
        if fn is None:
            continue

        def wrap(*a, _fn=fn, _name=name, **kw):
            stream = N.lib().hsv_get_stream()
            rt.cudaEventRecord(ev0, stream)
            e0 = dev_ms(True)
            d0 = dev_ms()
            p0 = pool()
            c0 = time.process_time()
            t0 = time.perf_counter()
            r = _fn(*a, **kw)
            if args.sync:
                N.call("hsv_synchronize")
            t1 = time.perf_counter()
            rt.cudaEventRecord(ev1, stream)
            rt.cudaEventSynchronize(ev1)
            span = rt.cudaEventElapsedTime(ev0, ev1)[1]
            log.append((_name, len(a[0]) if _name == "energy_and_gradient" else -1,
                        round((t1 - t0) * 1e3, 2), round((time.process_time() - c0) * 1e3, 2),
                        round(dev_ms() - d0, 2), p0, pool(), round(span, 2),
                        {k: round(v - e0[k], 2) for k, v in dev_ms(True).items() if v - e0[k] > 0.5}))
            return r
        setattr(eng, name, wrap)
    init = (ops[:k], tr[f"thetas_at_{k}"]) if k > 0 else None
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
