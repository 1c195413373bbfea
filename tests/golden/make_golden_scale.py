"""Row-sampled H14 / H16 goldens from the CPU oracle (SURVEY.md section 8c,
"row-sampled oracle (H14/H16)").

For the S1 state (default_rng(20240811) standard normal over the sector,
normalized) and a deterministic sample of reference positions, store
(H psi)_b computed by oracle/sv_oracle.apply_h_rows (pull form of the
reference's per-x-group matrix elements, svengine.py:130-161).  The oracle
is pinned against the reference at H2..H10 (tests/test_oracle.py).

    python tests/golden/make_golden_scale.py
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import s1_values  # noqa: E402
from oracle import sv_oracle as O  # noqa: E402
from paper_2604_01176_b200.system import MolecularSystem  # noqa: E402

OUT = Path(__file__).resolve().parent


def main(names=("h14", "h16"), n_rows=48):
    for name in names:
        t0 = time.time()
        s = MolecularSystem.bundled(name)
        h = s.hamiltonian
        states = O.sector_states(s.n_qubits, s.n_alpha, s.n_beta)
        dim = len(states)
        psi = s1_values(dim)
        rng = np.random.default_rng(4242)
        rows = np.unique(np.concatenate([[0, dim - 1, int(np.searchsorted(states, s.hf.bits))],
                                         rng.integers(0, dim, n_rows)])).astype(np.int64)
        y = O.apply_h_rows(h.xs, h.zs, h.coeffs, states, psi, rows)
        np.savez_compressed(OUT / f"ref_{name}.npz", dim=dim, rows=rows, hpsi_rows=y,
                            psi_rows=psi[rows], keys=states[rows])
        print(f"{name}: dim={dim} rows={len(rows)} ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
