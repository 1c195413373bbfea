#!/usr/bin/env python3
"""H|psi> on the dense S1-like state of a bundled system, timed with the
library's CUDA-event scopes, for K1 variants (e.g. sell=0 vs sell=1):

  python tools/apply_probe.py --system h12 --variants sell=0 sell=1 --reps 10
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--system", default="h12")
    ap.add_argument("--variants", nargs="+", default=["sell=0", "sell=1"])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--shard", type=int, default=1, help="time rows of alpha strings [0, Na/shard)")
    args = ap.parse_args()
    N.init(0)
    sysm = hsv.MolecularSystem.bundled(args.system)
    op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
    n = len(sysm.basis)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    st = hsv.SvState(sysm.basis, hsv.SparseVector(n, np.arange(n), v))
    for var in args.variants:
        kv = [x.split("=") for x in var.split(",")]
        for key, val in kv:
            N.call("hsv_set_tuning", key.encode(), int(val))
        na = sysm.basis._sector.n_alpha_strings
        hi = na // args.shard
        from paper_2604_01176_b200.svengine import DeviceState
        out = DeviceState(sysm.basis)

        def run():
            if args.shard == 1:
                op.apply_state(st)
            else:
                N.call("hsv_apply_h_rows_async", op.handle, st.device.handle, out.handle, 0, hi, 0.0)
                N.call("hsv_synchronize")
        run()                                   # warm-up (builds K1a rows)
        N.call("hsv_prof_reset")
        N.call("hsv_prof_enable", 1)
        for _ in range(args.reps):
            run()
        N.call("hsv_prof_collect")
        N.call("hsv_prof_enable", 0)
        t, c = N.dbl(), N.i64()
        N.call("hsv_prof_get", b"apply", N.C.byref(t), N.C.byref(c))
        print(json.dumps({"system": args.system, "variant": var, "apply_ms": t.value / max(c.value, 1),
                          "launches": c.value}), flush=True)
        for key, _ in kv:
            N.call("hsv_set_tuning", key.encode(),
                   {"sell": -1, "sell_budget_mb": 32768, "sell_sp": -1, "sell_kernel": 3}.get(key, 0))


if __name__ == "__main__":
    main()
