"""ADAPT-VQE driver with the device SV engine (mirror of `svmps.adapt`).

The host loop -- screen, select (ties -> lowest index), append theta = 0,
L-BFGS-B re-optimization with analytic gradients, rebuild, record -- follows
adapt.py:570-664 and stays on the host.  `SvAdaptEngine` implements the
reference engine protocol (adapt.py:179-220) on libhsv:

* `screen`     -> one fused H|psi> + all-pool gradient launch (K1 + K4),
* `energy_and_gradient` -> one fused adjoint sweep (K3 forward, K1, K5),
* `rebuild`    -> in-place QEB rotations on one device buffer (K3).

Only the exact sparse engine is in scope; the tensor-train engines of the
reference (`mps`, `partitioned`) are Hyperion-2 and are rejected by
`make_engine` with NotImplementedError.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.optimize

from .cibasis import hartree_fock_configuration, qubit_spin
from .svengine import (DevicePool, ExcitationOperator, SvState, apply_ansatz,
                       apply_qeb_exponential, assemble_subspace_hamiltonian)

ENGINES = ("sv", "mps", "partitioned")


@dataclass(frozen=True)
class OperatorPool:
    ops: tuple

    @property
    def size(self) -> int:
        return len(self.ops)

    def __iter__(self):
        return iter(self.ops)

    def __len__(self):
        return len(self.ops)


def build_qeb_pool(n_qubits: int, n_electrons: int, ordering: str = "interleaved",
                   ms2: int = 0) -> OperatorPool:
    """Singles (same spin) then doubles (equal spin multiset) from HF occupied to
    virtual spin orbitals, each block sorted by (occ, virt) (adapt.py:78-108)."""
    hf = hartree_fock_configuration(n_electrons, n_qubits, ordering, ms2)
    occ = hf.occupied()
    virt = [q for q in range(n_qubits) if q not in occ]
    if not occ or not virt:
        raise ValueError("empty operator pool: no occupied/virtual orbitals")
    spin = [qubit_spin(q, n_qubits, ordering) for q in range(n_qubits)]
    singles = sorted((ExcitationOperator("single", (i,), (a,))
                      for i in occ for a in virt if spin[i] == spin[a]),
                     key=lambda op: (op.occ, op.virt))
    doubles = []
    for n1, i in enumerate(occ):
        for j in occ[n1 + 1:]:
            for n2, a in enumerate(virt):
                for b in virt[n2 + 1:]:
                    if sorted((spin[a], spin[b])) == sorted((spin[i], spin[j])):
                        doubles.append(ExcitationOperator("double", (i, j), (a, b)))
    doubles.sort(key=lambda op: (op.occ, op.virt))
    ops = tuple(singles + doubles)
    if len(set(ops)) != len(ops):
        raise AssertionError("duplicate pool operators")
    return OperatorPool(ops)


@dataclass
class AdaptConfig:
    engine: str = "sv"
    eps_grad: float = 1e-3
    max_iter: int = 500
    opt_tol: float = 1e-9
    opt_gtol: float = 1e-6
    opt_max_evals: int = 200_000
    opt_xtol: float = 1e-6
    opt_line: str = "golden"
    min_sweeps: int = 2
    delta: float = 1e-12
    trunc_rule: str = "value"
    eta: int = 1
    mpo_cap: int = 100
    max_bond: int = 1 << 16
    threads: int = 1
    seed: int = 0

    def validate(self):
        if self.engine not in ENGINES:
            raise ValueError(f"unknown engine {self.engine!r}")
        for name in ("eps_grad", "opt_tol", "opt_gtol", "opt_xtol"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be > 0")
        if self.delta < 0:
            raise ValueError("delta must be >= 0")
        if self.trunc_rule not in ("value", "tail"):
            raise ValueError(f"unknown truncation rule {self.trunc_rule!r}")

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in self.__dataclass_fields__}


@dataclass
class RunRecord:
    iteration: int
    selected_op: str | None
    grad_max: float
    energy: float
    abs_error: float | None
    nnz: int
    max_trunc_err: float
    wall_elapsed: float
    energy_evals: int

    CSV_HEADER = "iter,selected_op,grad_max,energy,abs_error,nnz,max_trunc_err,wall_s,energy_evals"

    def csv_row(self) -> str:
        err = "" if self.abs_error is None else f"{self.abs_error:.12e}"
        return (f"{self.iteration},{self.selected_op or ''},{self.grad_max:.12e},"
                f"{self.energy:.15e},{err},{self.nnz},{self.max_trunc_err:.12e},"
                f"{self.wall_elapsed:.6f},{self.energy_evals}")


@dataclass
class OptResult:
    thetas: np.ndarray
    energy: float
    n_evals: int
    warning: bool = False
    message: str = ""


class TruncationLog:
    """Exact engine: nothing is truncated (running max stays 0)."""

    def __init__(self):
        self.entries: list = []
        self.running_max = 0.0


class SvAdaptEngine:
    """Exact sparse engine on the device (engine protocol, adapt.py:179-220)."""

    name = "sv"
    uses_coordinate_search = False

    def __init__(self, system, config: AdaptConfig):
        self.system = system
        self.basis = system.basis
        self.matrix = assemble_subspace_hamiltonian(system.hamiltonian, self.basis)
        self.threads = config.threads
        self.run_log = TruncationLog()
        self._masks: dict = {}
        self._dpools: dict = {}
        self._dpool_last = None

    def _pool_masks(self, ops):
        # the L-BFGS evaluations of one iteration pass the same operators: an
        # identity check (~12 us at k = 400) before hashing the tuple (~58 us)
        last = getattr(self, "_mask_last", None)
        if (last is not None and len(last[0]) == len(ops)
                and all(a is b for a, b in zip(last[0], ops))):
            return last[1]
        key = tuple(ops)
        m = self._masks.get(key)
        if m is None:
            m = (np.array([o.occ_mask for o in key], dtype=np.uint64),
                 np.array([o.virt_mask for o in key], dtype=np.uint64))
            self._masks = {key: m} if len(self._masks) > 8 else {**self._masks, key: m}
        self._mask_last = (key, m)
        return m

    def initial_state(self) -> SvState:
        return SvState.from_configuration(self.basis, self.system.hf)

    def apply(self, state, op, theta, log=None):
        return apply_qeb_exponential(op, theta, state)

    def rebuild(self, ops, thetas):
        """apply_ansatz (svengine.py:240-244) with the evaluation's cached operator
        masks (the same fused device sweep)."""
        from . import _native as N
        from .svengine import DeviceState
        ops = list(ops)
        th = np.ascontiguousarray(thetas, dtype=np.float64)
        n = min(len(ops), th.size)
        if n != len(ops) or n != th.size:
            return apply_ansatz(self.basis, self.system.hf, ops, thetas)
        occ, virt = self._pool_masks(ops)
        cs, sn = N.as_f64(np.cos(th)), N.as_f64(np.sin(th))
        dev = DeviceState(self.basis)
        N.call("hsv_ansatz_state", self.basis.sector, int(self.system.hf.bits), N.ptr_u64(occ),
               N.ptr_u64(virt), N.ptr_f64(cs), N.ptr_f64(sn), n, dev.handle)
        return SvState(self.basis, _dev=dev)

    def energy(self, state) -> float:
        return self.matrix.expect(state)

    def energy_and_gradient(self, ops, thetas):
        """Adjoint energy + gradient (svengine.py:260-281) on two device states
        kept across L-BFGS evaluations (no per-call state allocation)."""
        from . import _native as N
        from .svengine import DeviceState
        occ, virt = self._pool_masks(ops)
        if getattr(self, "_eg_states", None) is None:
            self._eg_states = (DeviceState(self.basis), DeviceState(self.basis))
        psi, w = self._eg_states
        th = np.ascontiguousarray(thetas, dtype=np.float64)
        cs, sn = N.as_f64(np.cos(th)), N.as_f64(np.sin(th))
        na = self.basis._sector.n_alpha_strings
        N.call("hsv_eg_forward_async", self.matrix.handle, int(self.system.hf.bits),
               N.ptr_u64(occ), N.ptr_u64(virt), N.ptr_f64(cs), N.ptr_f64(sn), th.size,
               0, na, psi.handle, w.handle)
        g = np.empty(th.size)
        e = N.dbl()
        N.call("hsv_eg_backward", self.matrix.handle, psi.handle, w.handle, N.ptr_u64(occ),
               N.ptr_u64(virt), N.ptr_f64(cs), N.ptr_f64(sn), th.size, N.C.byref(e),
               N.ptr_f64(g))
        return float(e.value), g

    def _device_pool(self, pool):
        seq = getattr(pool, "ops", pool)
        last = self._dpool_last
        if last is not None and last[0] is seq and isinstance(seq, tuple):
            return last[1]                        # same immutable op tuple: skip hashing 1818 ops
        ops = tuple(seq)
        dp = self._dpools.get(ops)
        if dp is None:
            dp = DevicePool(self.basis, ops)
            self._dpools = {ops: dp} if len(self._dpools) > 4 else {**self._dpools, ops: dp}
        self._dpool_last = (seq, dp)
        return dp

    def screen(self, state, pool) -> np.ndarray:
        return self.matrix.energy_screen_pool(state, self._device_pool(pool))[1]

    def energy_and_screen(self, state, pool):
        return self.matrix.energy_screen_pool(state, self._device_pool(pool))

    def state_size(self, state) -> int:
        return state.nnz

    def drain_log(self):
        return []


def make_engine(system, config: AdaptConfig):
    config.validate()
    if config.engine != "sv":
        raise NotImplementedError(f"engine {config.engine!r} (Hyperion-2 tensor-train path) is "
                                  "outside this build's scope; use engine='sv'")
    return SvAdaptEngine(system, config)


def screen_gradients(engine, state, pool) -> list:
    return list(zip(pool.ops, engine.screen(state, pool)))


def select_operator(gradients, eps_grad: float):
    """argmax |g| with ties to the lowest index; None below eps_grad (adapt.py:369-381)."""
    vals = [g for _, g in gradients] if gradients and isinstance(gradients[0], tuple) else gradients
    mags = np.abs(np.asarray(vals, dtype=np.float64))
    if mags.size == 0:
        raise ValueError("empty gradient list")
    best = int(np.argmax(mags))
    return None if mags[best] < eps_grad else best


def _optimize_lbfgs(engine, ops, thetas0, cfg: AdaptConfig) -> OptResult:
    count = [0]

    def fun(t):
        count[0] += 1
        return engine.energy_and_gradient(ops, t)

    if len(ops) == 0:
        return OptResult(np.zeros(0), engine.energy(engine.initial_state()), 1)
    res = scipy.optimize.minimize(
        fun, np.asarray(thetas0, dtype=np.float64), jac=True, method="L-BFGS-B",
        options={"ftol": cfg.opt_tol, "gtol": cfg.opt_gtol, "maxfun": cfg.opt_max_evals})
    return OptResult(np.asarray(res.x), float(res.fun), count[0],
                     count[0] >= cfg.opt_max_evals, str(res.message))


def optimize_parameters(engine, ops, thetas0, config: AdaptConfig) -> OptResult:
    if engine.uses_coordinate_search:
        raise NotImplementedError("coordinate search belongs to the tensor-train engines")
    return _optimize_lbfgs(engine, ops, thetas0, config)


@dataclass
class RunResult:
    records: list
    status: str
    ansatz_ops: list = field(default_factory=list)
    thetas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    abort_reason: str = ""
    optimizer_warnings: int = 0


def run_adapt(config: AdaptConfig, system, *, pool: OperatorPool | None = None,
              reference_energy: float | None = None, csv_path=None, trunc_csv_path=None,
              progress=None, engine=None, replay=None, initial=None) -> RunResult:
    """screen -> select -> append -> optimize -> record (adapt.py:570-664).

    `replay` (optional list of pool indices) forces the operator sequence of a
    reference run, for parity checks where exact gradient ties make the free
    selection non-unique (hard part 2).  `initial`
    (optional (ops, thetas)) resumes a run from an ansatz of depth k: the loop
    starts at iteration k with that state (the deep-ADAPT benchmark leg).
    """
    config.validate()
    engine = engine or make_engine(system, config)
    if pool is None:
        pool = build_qeb_pool(system.n_qubits, system.integrals.nelec, system.ordering,
                              system.integrals.ms2)
    records: list[RunRecord] = []
    ansatz: list = []
    thetas = np.zeros(0)
    n_evals = n_warn = 0
    status = "max_iter"
    t0 = time.perf_counter()
    csv_file = open(csv_path, "w", encoding="ascii") if csv_path else None
    trunc_file = open(trunc_csv_path, "w", encoding="ascii") if trunc_csv_path else None
    if csv_file:
        csv_file.write(RunRecord.CSV_HEADER + "\n")
        csv_file.flush()
    if trunc_file:
        trunc_file.write("iteration,site,tail_norm,running_max\n")
        trunc_file.flush()

    def emit(rec: RunRecord):
        records.append(rec)
        if csv_file:
            csv_file.write(rec.csv_row() + "\n")
            csv_file.flush()
        if progress:
            progress(rec)

    try:
        if initial is not None:
            ansatz = list(initial[0])
            thetas = np.array(initial[1], dtype=np.float64)
            state = engine.rebuild(ansatz, thetas)
            selected = ansatz[-1].label() if ansatz else None
            it = len(ansatz)
        else:
            state = engine.initial_state()
            selected = None
            it = 0
        energy = engine.energy(state)
        n_evals += 1
        grads = engine.screen(state, pool)
        while True:
            emit(RunRecord(it, selected, float(np.max(np.abs(grads))), float(energy),
                           None if reference_energy is None else abs(energy - reference_energy),
                           engine.state_size(state), engine.run_log.running_max,
                           time.perf_counter() - t0, n_evals))
            pick = select_operator(list(grads), config.eps_grad)
            if replay is not None and pick is not None:
                pick = replay[it] if it < len(replay) else None
            if pick is None:
                status = "converged"
                break
            if it >= config.max_iter:
                status = "max_iter"
                break
            ansatz.append(pool.ops[pick])
            selected = pool.ops[pick].label()
            thetas = np.append(thetas, 0.0)
            opt = optimize_parameters(engine, ansatz, thetas, config)
            thetas, energy = opt.thetas, opt.energy
            n_evals += opt.n_evals
            n_warn += int(opt.warning)
            state = engine.rebuild(ansatz, thetas)
            grads = engine.screen(state, pool)
            it += 1
    finally:
        if csv_file:
            csv_file.close()
        if trunc_file:
            trunc_file.close()
    return RunResult(records, status, ansatz, thetas, "", n_warn)


def amortized_coefficient(records):
    """C~_j = j / sqrt(T_j) and the least-squares c of T = c j^2 (adapt.py:670-692)."""
    pairs = []
    for r in records:
        if hasattr(r, "iteration"):
            pairs.append((r.iteration, r.wall_elapsed))
        else:
            pairs.append((int(r[0]), float(r[1])))
    pairs = [(j, t) for j, t in pairs if j > 0 and t > 0]
    if len(pairs) < 2:
        raise ValueError("need at least 2 records with positive wall time")
    js = np.array([p[0] for p in pairs], dtype=np.float64)
    ts = np.array([p[1] for p in pairs])
    if np.any(np.diff(ts[np.argsort(js)]) < 0):
        raise ValueError("wall times are not monotone in the iteration index")
    return js.astype(int), js / np.sqrt(ts), float(np.sum(ts * js ** 2) / np.sum(js ** 4))
