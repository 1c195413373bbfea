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
    ap.add_argument("--split", nargs="+", type=int, default=[0])
    ap.add_argument("--shard", nargs="+", type=int, default=[1],
                    help="time the rank-0 alpha-row shard of a W-way split")
    ap.add_argument("--shard-index", nargs="+", type=int, default=[0],
                    help="which shard of the --shard split to time (default the rank-0 one)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tune", nargs="+", default=[""],
                    help="extra hsv_set_tuning settings per run, e.g. rb0_smem=0 (A/B axis)")
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
        na = basis._sector.n_alpha_strings
        d_out = None
        for r, sr, mb, sp, sh, si, tu in [(r, sr, mb, sp, sh, si, tu) for r in args.apply_r
                                          for sr in args.screen_rows for mb in args.minb
                                          for sp in args.split for sh in args.shard
                                          for si in args.shard_index if si < sh
                                          for tu in args.tune]:
            for kv in filter(None, tu.split(",")):
                k, v = kv.split("=")
                N.call("hsv_set_tuning", k.encode(), int(v))
            N.call("hsv_set_tuning", b"apply_r", r)
            N.call("hsv_set_tuning", b"apply_minb", mb)
            N.call("hsv_set_tuning", b"screen_rows", sr)
            N.call("hsv_set_tuning", b"apply_split", sp)
            a_lo, a_hi = si * na // sh, (si + 1) * na // sh   # one shard of an sh-way split
            out = np.empty(2 + pool.n)

            def step():
                if sh == 1:
                    return op.energy_screen_pool(st, pool)
                N.call("hsv_energy_screen_pool_async", op.handle, st.device.handle, pool.handle,
                       a_lo, a_hi, N.C.c_void_p(d_dev))
                N.call("hsv_synchronize")
                return None, None
            if sh > 1 and d_out is None:
                import torch
                d_out = torch.zeros(2 + pool.n, dtype=torch.float64, device="cuda")
                torch.cuda.synchronize()
            d_dev = d_out.data_ptr() if d_out is not None else 0
            e, g = step()                    # warm
            N.call("hsv_prof_reset")
            N.call("hsv_prof_enable", 1)
            for _ in range(args.reps):
                e, g = step()
            N.call("hsv_prof_collect")
            N.call("hsv_prof_enable", 0)
            ta, _ = prof("apply")
            ts, _ = prof("screen")
            bytes_apply = (16.0 * nnz + 24.0 * dim) * (a_hi - a_lo) / na
            print(json.dumps({
                "system": name, "dim": dim, "apply_r": r, "minb": mb, "screen_rows": sr,
                "split": sp, "tune": tu, "shard": sh, "shard_index": si, "apply_ms": ta, "screen_ms": ts,
                "apply_GBs_alg": bytes_apply / ta / 1e6, "energy": e,
                "gmax": None if g is None else float(np.max(np.abs(g))), "nnz": nnz, **info}),
                flush=True)

if __name__ == "__main__":
    main()
