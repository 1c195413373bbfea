#!/usr/bin/env python3
"""Multi-GPU consistency check (run under torchrun, one rank per GPU):
the distributed engine (owner-computes H psi rows + NCCL all-gather) against the
single-GPU engine on every rank -- energies, adjoint gradients, pool screens and a
short ADAPT trace.  Prints one JSON line from rank 0 and exits non-zero on mismatch.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_check.py --systems h10 h12
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_01176_b200 as hsv  # noqa: E402
from paper_2604_01176_b200.distributed import DistributedSvAdaptEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--systems", nargs="+", default=["h10", "h12"])
    ap.add_argument("--iters", type=int, default=6)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    out, ok = {"world": world}, True
    for name in args.systems:
        s = hsv.MolecularSystem.bundled(name)
        pool = hsv.build_qeb_pool(s.n_qubits, s.integrals.nelec)
        de = DistributedSvAdaptEngine(s, hsv.AdaptConfig())
        se = de.inner                                   # same-rank single-GPU engine
        rng = np.random.default_rng(3)
        idx = rng.integers(0, len(pool), 12)
        th = rng.uniform(-0.3, 0.3, 12)
        ops = [pool.ops[i] for i in idx]
        e1, g1 = se.energy_and_gradient(ops, th)
        st = se.rebuild(ops, th)
        s1 = se.screen(st, pool)
        gmax = max(1.0, float(np.max(np.abs(g1))))
        res = {}
        cap_default = de.replica_nnz
        # both multi-GPU modes: replicas (sparse psi) and owner-computes + NCCL
        for mode, cap in (("", cap_default), ("_sharded", -1)):
            de.replica_nnz = cap
            de._last_nnz = 1
            de.energy_and_gradient(ops, th)           # sets the mode predictor
            e2, g2 = de.energy_and_gradient(ops, th)
            s2 = de.screen(st, pool)
            res["dE" + mode] = abs(e1 - e2)
            res["dG" + mode] = float(np.max(np.abs(g1 - g2))) / gmax
            res["dScreen" + mode] = float(np.max(np.abs(s1 - s2))) / max(1.0, float(np.max(np.abs(s1))))
        de.replica_nnz = cap_default
        t0 = time.perf_counter()
        ra = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=1e-6, max_iter=args.iters), s,
                           engine=de)
        t_d = time.perf_counter() - t0
        rb = hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=1e-6, max_iter=args.iters), s,
                           engine=se)
        res["adapt_dE"] = float(max(abs(a.energy - b.energy) for a, b in zip(ra.records, rb.records)))
        res["adapt_same_ops"] = [a.selected_op for a in ra.records] == [b.selected_op for b in rb.records]
        res["adapt_s_dist"] = t_d
        res["ok"] = bool(all(res["dE" + m] <= 1e-11 and res["dG" + m] <= 1e-10
                             and res["dScreen" + m] <= 1e-10 for m in ("", "_sharded"))
                         and res["adapt_dE"] <= 1e-8 and res["adapt_same_ops"])
        ok &= res["ok"]
        out[name] = res
    flags = torch.tensor([1.0 if ok else 0.0], device="cuda")
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps(out))
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if flags.item() == 1.0 else 1)


if __name__ == "__main__":
    main()
