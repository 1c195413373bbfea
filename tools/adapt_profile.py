#!/usr/bin/env python3
"""Host-side profile (cProfile) of the ADAPT loop on the device engine.

  python tools/adapt_profile.py --system h12 --iters 16
"""
import argparse
import cProfile
import pstats
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2604_01176_b200 as hsv  # noqa: E402
from paper_2604_01176_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--system", default="h12")
    ap.add_argument("--iters", type=int, default=16)
    ap.add_argument("--top", type=int, default=30)
    args = ap.parse_args()
    N.init(0)
    sysm = hsv.MolecularSystem.bundled(args.system)
    eng = hsv.SvAdaptEngine(sysm, hsv.AdaptConfig())
    cfg = hsv.AdaptConfig(engine="sv", eps_grad=1e-6, max_iter=args.iters)
    hsv.run_adapt(hsv.AdaptConfig(engine="sv", eps_grad=1e-6, max_iter=2), sysm, engine=eng)
    prof = cProfile.Profile()
    prof.enable()
    hsv.run_adapt(cfg, sysm, engine=eng)
    prof.disable()
    st = pstats.Stats(prof)
    st.sort_stats("tottime").print_stats(args.top)
    st.sort_stats("cumulative").print_stats(args.top)


if __name__ == "__main__":
    main()
