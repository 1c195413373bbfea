#!/usr/bin/env python3
"""Cost of the K1s build (support-compacted assembled rows) per ADAPT iteration
on the committed H12 trace: resume at depth k, run a few iterations, report the
build's stages (library scopes) and the per-evaluation K1s time.

  python tools/sup_probe.py --depth 400 --iters 3
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

SCOPES = ("sup_build", "sup_list", "sup_count", "sup_memset", "sup_emit", "apply_rows", "qeb",
          "adjoint", "apply", "screen")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--depth", type=int, default=400)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--tune", nargs="*", default=[], help="KEY=V library tuning keys")
    args = ap.parse_args()
    N.init(0)
    for kv in args.tune:
        key, v = kv.split("=")
        N.call("hsv_set_tuning", key.encode(), int(v))
    tr = np.load(ROOT / "tests" / "golden" / "trace_h12_416.npz")
    sysm = hsv.MolecularSystem.bundled("h12")
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    sel = [int(i) for i in tr["selected"]]
    ops = [pool.ops[i] for i in sel]
    k = args.depth
    init = (ops[:k], tr[f"thetas_at_{k}"])
    cfg = hsv.AdaptConfig(engine="sv", eps_grad=float(tr["eps"]), max_iter=k + 1)
    hsv.run_adapt(cfg, sysm, engine=eng, replay=sel, initial=init)   # warm-up
    N.call("hsv_prof_reset")
    N.call("hsv_prof_enable", 1)
    res = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=float(tr["eps"]),
                                        max_iter=k + args.iters),
                        sysm, engine=eng, replay=sel, initial=init)
    N.call("hsv_prof_collect")
    out = {}
    for kn in SCOPES:
        t, c = N.dbl(), N.i64()
        N.call("hsv_prof_get", kn.encode(), N.C.byref(t), N.C.byref(c))
        out[kn] = [round(t.value, 3), c.value]
    wall = np.diff([r.wall_elapsed for r in res.records]) * 1e3
    print(json.dumps({"depth": k, "tune": args.tune, "iter_ms": [round(float(x), 2) for x in wall], "scopes_ms_count": out}))


if __name__ == "__main__":
    main()
