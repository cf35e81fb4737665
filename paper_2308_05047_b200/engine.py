"""Host-side mirror of the reference's simulator API over the B200 engine.

Names, argument meaning and error behaviour follow the reference C++ API:

* ``IterativeShorEngine`` / ``run_iterative_shor`` —
  /root/reference/proj/include/shorsim/statevector.hpp:161-191
* ``ErrorConfig``, ``ErrorKind``, ``PauliProbs``, ``parse_error_config`` —
  /root/reference/proj/include/shorsim/noise.hpp:13-45, proj/src/noise.cpp:48-79
* ``FactoringProblem``, ``recommended_t`` — proj/include/shorsim/problems.hpp:15-32
* ``SimulatorOptions``, ``StageTrace``, ``BitString``, ``RunResult``, ``ErrorEvent``
  — proj/include/shorsim/statevector.hpp:109-159
* exceptions — proj/include/shorsim/errors.hpp:8-43

Every compute call goes through the C ABI (``libshorsim_b200.so``); nothing here
computes amplitudes.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

from . import _lib as L


# ----------------------------------------------------------------- errors
class Error(RuntimeError):
    """shorsim::Error (norm drift and the base of all simulator errors)."""


class NotInvertibleError(Error):
    def __init__(self, msg: str, gcd: int = 0):
        super().__init__(msg)
        self.gcd = gcd


class DegenerateBranchError(Error):
    pass


class BudgetExceededError(Error):
    pass


class CeilingExceededError(Error):
    pass


class ConfigError(Error):
    pass


class FactorizationTimeoutError(Error):
    """errors.hpp: Pollard rho ran out of its step budget (numtheory.cpp:137, 149)."""


class CudaError(Error):
    pass


def _raise(code: int) -> None:
    if code == L.SHS_OK:
        return
    msg = L.load().shs_last_error().decode(errors="replace")
    if code == L.SHS_NOT_INVERTIBLE:
        gcd = 0
        if "= " in msg:
            try:
                gcd = int(msg.rsplit("= ", 1)[1])
            except ValueError:
                pass
        raise NotInvertibleError(msg, gcd)
    raise {
        L.SHS_ERROR: Error,
        L.SHS_CONFIG_ERROR: ConfigError,
        L.SHS_CEILING_EXCEEDED: CeilingExceededError,
        L.SHS_DEGENERATE_BRANCH: DegenerateBranchError,
        L.SHS_BUDGET_EXCEEDED: BudgetExceededError,
        L.SHS_INVALID_ARGUMENT: ValueError,  # std::invalid_argument
        L.SHS_CUDA_ERROR: CudaError,
        L.SHS_FACTORIZATION_TIMEOUT: FactorizationTimeoutError,
    }.get(code, Error)(msg)


# ------------------------------------------------------------- data types
class ErrorKind(enum.IntEnum):
    none = 0
    amplitude_init = 1
    phase_init = 2
    classical_measure = 3
    quantum_measure = 4
    bitflip = 5


@dataclass
class PauliProbs:
    px: float = 0.0
    py: float = 0.0
    pz: float = 0.0


@dataclass
class ErrorConfig:
    kind: ErrorKind = ErrorKind.none
    delta: float = 0.0
    pauli: Optional[PauliProbs] = None

    @staticmethod
    def none_config() -> "ErrorConfig":
        return ErrorConfig()

    def to_c(self) -> L.shs_error:
        p = self.pauli or PauliProbs()
        return L.shs_error(int(self.kind), float(self.delta), p.px, p.py, p.pz,
                           1 if self.pauli is not None else 0)

    def validate(self) -> None:
        """ErrorConfig::validate, noise.cpp:13-25 (raises ConfigError)."""
        d = self.delta
        if d < 0.0 or d > 1.0:
            raise ConfigError("error config: delta outside [0, 1]")
        if self.kind == ErrorKind.quantum_measure:
            if self.pauli is None:
                raise ConfigError("quantum_measure requires px/py(/pz)")
            p = self.pauli
            if p.px < 0 or p.py < 0 or p.pz < 0 or p.px + p.py + p.pz > 1.0:
                raise ConfigError("error config: invalid Pauli probabilities")
            if abs((p.px + p.py) - d) > 1e-12:
                raise ConfigError("quantum_measure: delta != px + py")
        elif self.pauli is not None:
            raise ConfigError("error config: pauli probabilities only apply to quantum_measure")


def parse_error_config(text: str) -> ErrorConfig:
    """The CLI grammar of noise.cpp:48-79, e.g. "kind=quantum_measure,px=0.005,py=0.005"."""
    px = py = delta = -1.0
    pz = 0.0
    kind = ""
    for item in text.split(","):
        if "=" not in item:
            raise ConfigError("error config: expected key=value: " + item)
        key, value = item.split("=", 1)
        if key == "kind":
            kind = value
        elif key in ("delta", "px", "py", "pz"):
            v = float(value)
            if key == "delta":
                delta = v
            elif key == "px":
                px = v
            elif key == "py":
                py = v
            else:
                pz = v
        else:
            raise ConfigError("error config: unknown key: " + key)
    if not kind:
        raise ConfigError("error config: missing kind")
    try:
        k = ErrorKind[kind]
    except KeyError:
        raise ConfigError("unknown error kind: " + kind) from None
    cfg = ErrorConfig(kind=k)
    if k == ErrorKind.quantum_measure:
        if px < 0 or py < 0:
            raise ConfigError("quantum_measure: need px and py")
        cfg.pauli = PauliProbs(px, py, pz)
        cfg.delta = px + py
        if delta >= 0 and abs(delta - cfg.delta) > 1e-12:
            raise ConfigError("quantum_measure: delta != px + py")
    elif k != ErrorKind.none:
        if delta < 0:
            raise ConfigError("error config: missing delta")
        cfg.delta = delta
    cfg.validate()
    return cfg


def bit_length(n: int) -> int:
    return int(n).bit_length()


def recommended_t(n: int) -> int:
    """Smallest t with 2^t >= N^2 (problems.cpp:17-23)."""
    if n < 2:
        raise ValueError("recommended_t: N >= 2")
    t = 0
    while (1 << t) < n * n:
        t += 1
    return t


@dataclass
class FactoringProblem:
    N: int = 15
    a: int = 7
    L: int = 4
    t: int = 8
    p: Optional[int] = None
    q: Optional[int] = None
    seed: int = 0

    def qubits(self) -> int:
        return self.L + 1

    @staticmethod
    def make(N: int, a: int, t: Optional[int] = None, **kw) -> "FactoringProblem":
        return FactoringProblem(N=N, a=a, L=bit_length(N), t=t if t else recommended_t(N), **kw)


@dataclass
class SimulatorOptions:
    shard_count: int = 4
    workers: int = 1
    qubit_ceiling: int = 26
    check_norms: bool = True
    device: int = 0
    combine: str = "auto"  # "auto" | "kahan" | "exact" (see include/shorsim_b200.h)
    tiling: str = "auto"   # "auto" | "force" | "off"
    # multi-GPU (include/shorsim_b200.h shs_options.n_devices): None = one device;
    # a list of ordinals (repeats allowed: virtual shards) shards the state over
    # them; "auto" = as many devices as the state needs
    devices: Optional[object] = None

    def to_c(self) -> L.shs_options:
        o = L.shs_options(self.shard_count, self.workers, self.qubit_ceiling,
                          1 if self.check_norms else 0, self.device, L.COMBINE[self.combine],
                          L.TILING[self.tiling], 0, None)
        if self.devices == "auto":
            o.n_devices = -1
        elif self.devices is not None and len(self.devices) >= 2:
            arr = (L.i32 * len(self.devices))(*[int(d) for d in self.devices])
            o.n_devices = len(self.devices)
            o.devices = C.cast(arr, C.POINTER(L.i32))
            o.keep = arr  # the array lives as long as the struct
        return o


@dataclass
class ErrorEvent:
    classical_flip: bool = False
    quantum_error_branch: bool = False


@dataclass
class StageTrace:
    cbit: int
    p1: float
    sampled_bit: int
    observed_bit: int
    event: ErrorEvent = field(default_factory=ErrorEvent)


@dataclass
class BitString:
    t: int = 0
    j: int = 0


@dataclass
class RunResult:
    bits: BitString
    j_sampled: int
    trace: List[StageTrace]


# ----------------------------------------------------------------- engine
class IterativeShorEngine:
    """IterativeShorEngine(problem, error, options) — statevector.hpp:169-191.

    Owns the device state (one fp64 complex buffer of N amplitudes plus its
    double buffer) and the CUDA stream; ``run(seed, bitstring_index)`` replays
    exactly like the reference's (randomness addressed by seed / index / stage).
    """

    def __init__(self, problem: FactoringProblem, error: Optional[ErrorConfig] = None,
                 options: Optional[SimulatorOptions] = None):
        self._lib = L.load()
        self.problem = problem
        self.error = error if error is not None else ErrorConfig()
        self.options = options if options is not None else SimulatorOptions()
        self._h = L.vp()
        self._pr = L.shs_problem(problem.N, problem.a, problem.L, problem.t, problem.seed)
        self._er = self.error.to_c()
        self._op = self.options.to_c()
        _raise(self._lib.shs_engine_create(C.byref(self._pr), C.byref(self._er),
                                           C.byref(self._op), C.byref(self._h)))
        self.t = problem.t
        self._trace = (L.shs_stage_trace * self.t)()

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.shs_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- the reference API
    def run(self, seed: int, bitstring_index: int) -> RunResult:
        j = (L.u64 * 2)()
        js = (L.u64 * 2)()
        _raise(self._lib.shs_engine_run(self._h, seed, bitstring_index, j, js, self._trace))
        trace = [StageTrace(tr.cbit, tr.p1, tr.sampled_bit, tr.observed_bit,
                            ErrorEvent(bool(tr.classical_flip), bool(tr.quantum_error_branch)))
                 for tr in self._trace]
        return RunResult(BitString(self.t, j[0] | (j[1] << 64)), js[0] | (js[1] << 64), trace)

    def run_batch(self, seed: int, idx0: int, count: int) -> List[int]:
        """Bit strings of runs idx0 .. idx0+count-1 (whole runs on the device for
        small problems; see shs_engine_run_batch)."""
        out = (L.u64 * (2 * count))()
        _raise(self._lib.shs_engine_run_batch(self._h, seed, idx0, count, out))
        return [out[2 * i] | (out[2 * i + 1] << 64) for i in range(count)]

    def run_batch_array(self, seed: int, idx0: int, count: int, out=None):
        """As run_batch, into a numpy uint64 array of shape (count, 2) = (lo, hi)
        words of each bit string (no per-run Python objects)."""
        import numpy as np
        if out is None:
            out = np.empty((count, 2), dtype=np.uint64)
        ptr = out.ctypes.data_as(C.POINTER(L.u64))
        _raise(self._lib.shs_engine_run_batch(self._h, seed, idx0, count, ptr))
        return out

    def run_many(self, seed: int, idx0: int, count: int) -> List[RunResult]:
        """RunResult (with traces) for runs idx0 .. idx0+count-1 in one call."""
        t = self.t
        j = (L.u64 * (2 * count))()
        js = (L.u64 * (2 * count))()
        p1 = (L.dbl * (count * t))()
        bits = (L.i32 * (4 * count * t))()
        _raise(self._lib.shs_engine_run_many(self._h, seed, idx0, count, j, js, p1, bits))
        out = []
        for i in range(count):
            trace = []
            for s in range(t):
                b = bits[4 * (i * t + s):4 * (i * t + s) + 4]
                trace.append(StageTrace(s, p1[i * t + s], b[0], b[1],
                                        ErrorEvent(bool(b[2]), bool(b[3]))))
            out.append(RunResult(BitString(t, j[2 * i] | (j[2 * i + 1] << 64)),
                                 js[2 * i] | (js[2 * i + 1] << 64), trace))
        return out

    def run_sequential(self, seed: int, idx0: int, count: int) -> List[int]:
        out = (L.u64 * (2 * count))()
        _raise(self._lib.shs_engine_run_sequential(self._h, seed, idx0, count, out))
        return [out[2 * i] | (out[2 * i + 1] << 64) for i in range(count)]

    def stage_multipliers(self) -> List[int]:
        out = (L.u64 * self.t)()
        _raise(self._lib.shs_engine_stage_multipliers(self._h, out))
        return list(out)

    # -- step/measure API (forced sequences; amplitude parity)
    def state_init(self) -> None:
        _raise(self._lib.shs_state_init(self._h))

    def stage_probs(self, s: int, prefix: int = 0):
        p0, p1 = L.dbl(), L.dbl()
        _raise(self._lib.shs_stage_probs(self._h, s, prefix & (2**64 - 1), prefix >> 64,
                                         C.byref(p0), C.byref(p1)))
        return p0.value, p1.value

    def stage_collapse(self, src_group: int, p_source: float) -> None:
        _raise(self._lib.shs_stage_collapse(self._h, src_group, p_source))

    def stage_read(self, x: int, first: int, count: int):
        out = (L.dbl * (2 * count))()
        _raise(self._lib.shs_stage_read(self._h, x, first, count, out))
        return out

    def state_read(self, x: int, first: int, count: int):
        out = (L.dbl * (2 * count))()
        _raise(self._lib.shs_state_read(self._h, x, first, count, out))
        return out

    def state_gather(self, x: int, idx):
        """g_x at arbitrary indices (uint64 array-like) -> interleaved (re, im) doubles."""
        import numpy as np
        ix = np.ascontiguousarray(idx, dtype=np.uint64)
        out = np.empty(2 * ix.size, dtype=np.float64)
        _raise(self._lib.shs_state_gather(self._h, x, ix.ctypes.data_as(C.POINTER(L.u64)),
                                          ix.size, out.ctypes.data_as(C.POINTER(L.dbl))))
        return out

    def block_sums(self):
        nb = self._lib.shs_num_blocks(self._h)
        out = (L.dbl * (2 * nb))()
        _raise(self._lib.shs_stage_block_sums(self._h, out))
        return out[:nb], out[nb:]

    def index_map(self, s: int, first: int, count: int):
        out = (L.u64 * count)()
        _raise(self._lib.shs_index_map(self._h, s, first, count, out))
        return out

    def tile_plan(self, s: int):
        out = (L.u64 * 6)()
        _raise(self._lib.shs_stage_tile_plan(self._h, s, out))
        return dict(zip(("tiled", "H", "u", "v", "du", "dv"), list(out)))

    # -- instrumentation
    def set_timing(self, enable: bool) -> None:
        _raise(self._lib.shs_engine_set_timing(self._h, 1 if enable else 0))

    def kernel_times(self):
        ms = (L.dbl * 3)()
        n = (L.u64 * 3)()
        _raise(self._lib.shs_engine_kernel_times(self._h, ms, n))
        return {"probs": (ms[0], n[0]), "combine": (ms[1], n[1]), "collapse": (ms[2], n[2])}

    def stream_handle(self) -> int:
        return self._lib.shs_engine_stream(self._h) or 0

    def set_sparse(self, enable: bool) -> None:
        """Sparse prefix of run() (on by default where it applies): the first
        stages on the support of the state, bit-identical results."""
        _raise(self._lib.shs_engine_set_sparse(self._h, 1 if enable else 0))

    def sparse_stages(self) -> int:
        return self._lib.shs_engine_sparse_stages(self._h)

    def set_orbit(self, enable: bool) -> None:
        """Orbit-compressed stages (on by default from N >= 2^21): stages with
        whole-band tile plans store and sweep only the r = ord_N(a) members of
        <a>, bit-identical results. Toggling resets the state."""
        _raise(self._lib.shs_engine_set_orbit(self._h, 1 if enable else 0))

    def orbit_stages(self) -> List[int]:
        """1 for every stage that runs compressed"""
        out = (C.c_uint8 * self.problem.t)()
        _raise(self._lib.shs_engine_orbit_stages(self._h, out))
        return list(out)

    def orbit_info(self) -> dict:
        """{"r": orbit size (0: off), "stages": stages run compressed, "first": the first}"""
        out = (C.c_uint64 * 3)()
        _raise(self._lib.shs_engine_orbit_info(self._h, out))
        return {"r": int(out[0]), "stages": int(out[1]), "first": int(out[2])}

    def launch_count(self) -> int:
        return self._lib.shs_engine_launch_count(self._h)

    def device_bytes(self) -> int:
        return self._lib.shs_engine_device_bytes(self._h)

    def devices(self) -> List[int]:
        """CUDA ordinals the state lives on (several when the engine is sharded)."""
        out = (L.i32 * L.MAX_SHARDS)()
        n = self._lib.shs_engine_devices(self._h, out, L.MAX_SHARDS)
        return list(out[:n])


def run_iterative_shor(problem: FactoringProblem, error: ErrorConfig, seed: int,
                       bitstring_index: int, options: Optional[SimulatorOptions] = None
                       ) -> RunResult:
    """run_iterative_shor, statevector.cpp:414-418."""
    with IterativeShorEngine(problem, error, options) as engine:
        return engine.run(seed, bitstring_index)


def sample_measurement(p1: float, seed: int, idx: int, stage: int, error: ErrorConfig):
    """sample_measurement, statevector.cpp:236-256 (host side of the engine)."""
    out = (L.i32 * 4)()
    er = error.to_c()
    _raise(L.load().shs_sample_measurement(p1, seed, idx, stage, C.byref(er), out))
    return {"sampled_bit": out[0], "observed_bit": out[1], "error_branch": bool(out[2]),
            "classical_flip": bool(out[3])}


def exhaustive_joint_distribution(problem: FactoringProblem, error: Optional[ErrorConfig] = None,
                                  node_budget: int = 1 << 22, device: int = 0) -> List[float]:
    """exhaustive_joint_distribution, statevector.cpp:533-579: the exact distribution
    over observed bit strings (2^t values), computed on the device; raises
    BudgetExceededError past t > 14, n > 12 or the node budget, as the reference does."""
    error = error if error is not None else ErrorConfig()
    pr = L.shs_problem(problem.N, problem.a, problem.L, problem.t, problem.seed)
    er = error.to_c()
    out = (L.dbl * (1 << problem.t))()
    _raise(L.load().shs_exhaustive_distribution(C.byref(pr), C.byref(er), node_budget, device, out))
    return list(out)


def build_info() -> str:
    return L.load().shs_build_info().decode()
