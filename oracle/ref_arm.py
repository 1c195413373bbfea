"""CPU REFERENCE ARM -- bench.py's `--impl reference` arm and `cpu_baseline` leg only.

Times the UNMODIFIED reference (`svmps`, staged byte for byte into
oracle/_ref by oracle/stage_reference.py) on its own public API: one step is
`SvAdaptEngine.energy(psi)` + `SvAdaptEngine.screen(psi, pool)`
(adapt.py:205-214) -- two `spmspv` calls plus `apply_generator` + `dot` per
pool operator -- on the S1 dense-in-sector state built exactly as the
reference tests build it (normalize(SparseVector.from_dense(
default_rng(20240811).standard_normal(dim)))).

* FULL (`stride == 1`): a genuine `SvAdaptEngine(system, AdaptConfig(threads=
  nproc))`, i.e. the reference's own CSR assembly (untimed setup, adapt.py:188).
  Feasible through H10 (28.2 M nnz, ~15 s assembly).
* SAMPLED (`stride = s > 1`, H12: its assembly needs ~63 GB and minutes):
  the engine's matrix is the reference `CsrMatrix` (built with its own
  `CsrMatrix.from_coo`) holding every s-th row of the Hamiltonian -- row r is
  column r (the matrix is exactly symmetric), computed with
  the reference's per-x-group sums in its term order (svengine.py:130-161,
  restated in oracle/sv_oracle.py and pinned bitwise against the reference's
  CSR).  `screen` gets every s-th pool operator (offset rotating per step).
  One timed step is therefore 1/s of the full step's work, and the reported
  throughput is the sample's own units over the sample's own measured time
  (no extrapolation of time).  Linearity is checked at H10, where the full
  and the sampled step both run (`validate_linearity`).

The reference code runs as shipped; this module only builds inputs and times.
"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
S1_SEED = 20240811


def load_svmps():
    """Import the staged reference package (oracle/_ref), or None if absent."""
    p = HERE / "_ref"
    if not (p / "svmps" / "__init__.py").exists():
        return None
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    import svmps  # noqa: F401
    import svmps.adapt
    import svmps.sparse
    import svmps.svengine
    import svmps.system
    return sys.modules["svmps"]


def host_info() -> dict:
    info = {"nproc": os.cpu_count()}
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        for line in Path("/proc/meminfo").read_text().splitlines():
            if line.startswith("MemTotal"):
                info["ram_gb"] = round(int(line.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return info


def sampled_rows_csr(svmps, system, stride: int, offset: int = 0):
    """Reference CsrMatrix (dim x dim) holding rows offset, offset+stride, ...
    of the subspace Hamiltonian, element values as svengine.py:130-161."""
    from . import sv_oracle as O
    h = system.hamiltonian
    states = np.asarray(system.basis.states)
    dim = len(states)
    rows = np.arange(offset, dim, stride, dtype=np.int64)
    b = states[rows]
    r_acc, c_acc, v_acc = [], [], []
    for x, terms in O.x_groups(np.asarray(h.xs), np.asarray(h.zs), np.asarray(h.coeffs)):
        amp = O.group_amp(b, terms)            # == amp_x(b ^ x): even-Y words
        if x == 0:
            keep = amp != 0.0
            r_acc.append(rows[keep]); c_acc.append(rows[keep]); v_acc.append(amp[keep])
            continue
        pos, found = O.try_positions(states, b ^ x)
        keep = found & (amp != 0.0)
        r_acc.append(rows[keep]); c_acc.append(pos[keep]); v_acc.append(amp[keep])
    return svmps.sparse.CsrMatrix.from_coo(dim, dim, np.concatenate(r_acc),
                                           np.concatenate(c_acc), np.concatenate(v_acc))


class ReferenceArm:
    """The reference's SvAdaptEngine.energy + .screen, full or row/op-sampled."""

    def __init__(self, name: str = "h12", stride: int = 1, threads: int | None = None):
        svmps = load_svmps()
        if svmps is None:
            raise FileNotFoundError("reference not staged: python oracle/stage_reference.py")
        self.svmps = svmps
        A, S = svmps.adapt, svmps.sparse
        self.threads = threads or os.cpu_count() or 1
        self.name, self.stride = name, int(stride)
        t0 = time.perf_counter()
        self.system = svmps.system.MolecularSystem.from_fcidump(svmps.system.bundled_fcidump(name))
        basis = self.system.basis
        self.dim = len(basis)
        self.n_terms = len(self.system.hamiltonian)
        self.pool = A.build_qeb_pool(self.system.n_qubits, self.system.integrals.nelec,
                                     self.system.ordering, self.system.integrals.ms2)
        rng = np.random.default_rng(S1_SEED)
        self.psi = svmps.svengine.SvState(basis, S.normalize(S.SparseVector.from_dense(
            rng.standard_normal(self.dim))))
        cfg = A.AdaptConfig(engine="sv", threads=self.threads)
        if self.stride == 1:
            self.engine = A.SvAdaptEngine(self.system, cfg)       # the reference's own assembly
        else:
            eng = A.SvAdaptEngine.__new__(A.SvAdaptEngine)       # skip only the full assembly
            eng.system, eng.basis, eng.threads = self.system, basis, self.threads
            eng.run_log, eng._drained = A.TruncationLog(), 0
            eng.matrix = sampled_rows_csr(svmps, self.system, self.stride)
            self.engine = eng
        self.nnz = int(self.engine.matrix.nnz)
        self.t_setup = time.perf_counter() - t0
        self.k = 0
        self.last = None

    def step(self) -> dict:
        """One (sampled) step; returns its wall time and units of work."""
        ops = list(self.pool.ops)
        if self.stride > 1:
            ops = ops[self.k % self.stride::self.stride]
        self.k += 1
        t0 = time.perf_counter()
        e = self.engine.energy(self.psi)
        g = self.engine.screen(self.psi, ops)
        t = time.perf_counter() - t0
        self.last = (e, g)
        frac = 1.0 / self.stride
        return {"t_s": t, "units": frac * self.n_terms * self.dim, "energy": e, "n_ops": len(ops)}

    def run(self, steps: int, warmup: int) -> dict:
        for _ in range(warmup):
            self.step()
        rs = [self.step() for _ in range(steps)]
        t = sum(r["t_s"] for r in rs)
        u = sum(r["units"] for r in rs)
        return {"value": u / t, "ms_per_step": t / steps * 1e3, "steps": steps,
                "t_step_s": [round(r["t_s"], 4) for r in rs]}

    def describe(self) -> str:
        if self.stride == 1:
            return (f"unmodified reference svmps, {self.name.upper()} full step: energy + screen "
                    f"of all {len(self.pool)} pool ops, CSR {self.nnz} nnz, {self.threads} threads")
        return (f"unmodified reference svmps, {self.name.upper()} 1/{self.stride} step sample: "
                f"energy + screen on every {self.stride}th CSR row ({self.nnz} nnz of the "
                f"full matrix's rows) and every {self.stride}th pool op (offset rotating), "
                f"{self.threads} threads; value = sampled units / measured time")


def validate_linearity(name: str = "h10", stride: int = 16, steps: int = 2,
                       threads: int | None = None) -> dict:
    """Full vs sampled reference step at a size where both run: the sampled
    throughput should equal the full one if the sample is representative."""
    full = ReferenceArm(name, 1, threads)
    rf = full.run(steps, 1)
    samp = ReferenceArm(name, stride, threads)
    rs = samp.run(steps * stride // 2 or 1, 1)
    return {"system": name, "stride": stride, "full_value": rf["value"],
            "full_ms_per_step": rf["ms_per_step"], "full_setup_s": full.t_setup,
            "sampled_value": rs["value"], "sampled_ms_per_step": rs["ms_per_step"],
            "sampled_over_full": rs["value"] / rf["value"]}
