"""Reference ADAPT trace at H10 (adapt.py:570-664, unmodified reference) for the
replay-mode ADAPT iteration time of SURVEY.md 8(d) and its parity test.

Run in the build container (the reference is importable there, not on the GPU box):
    python tests/golden/make_golden_adapt_h10.py
Writes tests/golden/adapt_h10.npz (same layout as adapt_h4/h6 from make_golden.py).
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as mg  # noqa: E402  (puts the reference on sys.path)


def main():
    t0 = time.time()
    system = mg.MolecularSystem.from_fcidump(mg.bundled_fcidump("h10"))
    mg.adapt_trace("h10", system, 1e-6, 16)
    print(f"{time.time() - t0:.1f} s")


if __name__ == "__main__":
    main()
