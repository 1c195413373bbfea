#!/usr/bin/env python3
"""Long ADAPT-VQE free run on the device engine: per-iteration wall time,
L-BFGS evaluations, nnz(psi) and per-kernel device time, plus the selected
operator sequence and optimized angles (the trace the bench's deep-ADAPT leg
replays from depth k).

  python tools/adapt_long.py --system h12 --iters 400 --out gpurun_out/adapt_h12.npz
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

KERNELS = ("apply", "push", "push_collect", "screen", "qeb", "adjoint")


def prof_snapshot():
    out = {}
    for kn in KERNELS:
        t, c = N.dbl(), N.i64()
        N.call("hsv_prof_get", kn.encode(), N.C.byref(t), N.C.byref(c))
        out[kn] = t.value
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--system", default="h12")
    ap.add_argument("--iters", type=int, default=400)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--out", default="gpurun_out/adapt_trace.npz")
    ap.add_argument("--prof", action="store_true", help="per-kernel device time per iteration")
    ap.add_argument("--tune", nargs="*", default=[])
    args = ap.parse_args()
    N.init(0)
    for kv in args.tune:
        k, v = kv.split("=")
        N.call("hsv_set_tuning", k.encode(), int(v))
    sysm = hsv.MolecularSystem.bundled(args.system)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    pool = hsv.build_qeb_pool(sysm.n_qubits, sysm.integrals.nelec)
    index = {op: i for i, op in enumerate(pool.ops)}
    rows = []
    checkpoints = {}                 # depth k -> optimized thetas after iteration k
    rebuild = eng.rebuild

    def rebuild_spy(ops, thetas):
        checkpoints[len(ops)] = np.array(thetas, dtype=np.float64)
        return rebuild(ops, thetas)

    eng.rebuild = rebuild_spy
    last = {"t": time.perf_counter(), "prof": None}
    if args.prof:
        N.call("hsv_prof_reset")
        N.call("hsv_prof_enable", 1)
        last["prof"] = prof_snapshot()

    def progress(rec):
        now = time.perf_counter()
        row = {"it": rec.iteration, "sel": rec.selected_op, "E": rec.energy, "gmax": rec.grad_max,
               "nnz": rec.nnz, "evals": rec.energy_evals, "wall": rec.wall_elapsed,
               "dt_ms": (now - last["t"]) * 1e3}
        if args.prof:
            N.call("hsv_prof_collect")
            p = prof_snapshot()
            row["kern_ms"] = {k: round(p[k] - last["prof"][k], 3) for k in KERNELS}
            last["prof"] = p
        last["t"] = now
        rows.append(row)
        if rec.iteration % 25 == 0:
            print(json.dumps(row), flush=True)

    t0 = time.perf_counter()
    res = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=args.eps, max_iter=args.iters),
                        sysm, engine=eng, progress=progress)
    total = time.perf_counter() - t0
    sel = np.array([index[op] for op in res.ansatz_ops], dtype=np.int64)
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    np.savez(out, selected=sel, thetas=np.asarray(res.thetas), energy=np.array([r["E"] for r in rows]),
             nnz=np.array([r["nnz"] for r in rows]), evals=np.array([r["evals"] for r in rows]),
             wall=np.array([r["wall"] for r in rows]), eps=args.eps, max_iter=args.iters,
             **{f"thetas_at_{k}": checkpoints[k] for k in (25, 50, 100, 200, 300, 400)
                if k in checkpoints})
    with open(out.with_suffix(".jsonl"), "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")
    print(json.dumps({"system": args.system, "status": res.status, "iters": len(rows) - 1,
                      "total_s": total, "final_E": rows[-1]["E"], "final_nnz": rows[-1]["nnz"]}))


if __name__ == "__main__":
    main()
