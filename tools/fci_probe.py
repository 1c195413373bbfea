#!/usr/bin/env python3
"""FCI ground energies of the bundled hydrogen chains on the device (thick-
restart Lanczos over the sector, paper_2604_01176_b200.fci) -- the abs_error
references the reference's own eigsh cannot reach beyond H12:

  python tools/fci_probe.py --systems h12 h14 h16 --tol 1e-9
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_01176_b200 as hsv  # noqa: E402
from paper_2604_01176_b200 import fci  # noqa: E402
from paper_2604_01176_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--systems", nargs="+", default=["h12", "h14"])
    ap.add_argument("--tol", type=float, default=1e-9)
    ap.add_argument("--max-iter", type=int, default=3000)
    args = ap.parse_args()
    N.init(0)
    for name in args.systems:
        sysm = hsv.MolecularSystem.bundled(name)
        op = hsv.assemble_subspace_hamiltonian(sysm.hamiltonian, sysm.basis)
        N.call("hsv_synchronize")
        t0 = time.perf_counter()
        e, info = fci.lanczos_ground_energy(op, tol=args.tol, max_iter=args.max_iter,
                                            return_info=True)
        dt = time.perf_counter() - t0
        print(json.dumps({"system": name, "dim": len(sysm.basis), "e_fci": e,
                          "wall_s": round(dt, 2), **{k: v for k, v in info.items()
                                                     if isinstance(v, (int, float))}}),
              flush=True)
        del op
        N.call("hsv_mem_trim")


if __name__ == "__main__":
    main()
