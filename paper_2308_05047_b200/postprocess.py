"""Shor post-processing and the per-problem statistics (§8 f4), the step right
after the path.

* ``shor_postprocess_array`` — shor_standard_procedure
  (/root/reference/proj/src/postprocess.cpp:55-89) for a whole batch of bit
  strings on the device (``shs_shor_postprocess``, csrc/postprocess.cu).
* ``shor_standard_procedure`` — the same for one bit string, returning the
  reference's ``PostProcessOutcome`` fields.
* ``ekera_postprocess_array`` / ``ekera_postprocess`` — Ekerå's pipeline
  (postprocess.cpp:92-171: the ±B sweep, smooth-lift order recovery,
  factoring from the order with the shot's RngStream) on the device.
* ``multiplicative_order`` — ground-truth order from the known factors
  (numtheory.cpp:207-234), host integer code.
* ``run_problem`` — ``run_problem`` (proj/src/harness.cpp:109-148, simulator
  backend, Shor mode): M shots through the engine (whole runs on the device
  for small problems), post-processed on the device, tallied like
  ``note_outcome`` (harness.cpp:82-104).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import _lib as L
from .engine import (ErrorConfig, FactoringProblem, IterativeShorEngine, SimulatorOptions,
                     _raise)


class Classification(enum.IntEnum):  # postprocess.hpp:12
    success = 0
    lucky_ne = 1
    lucky_no = 2
    lucky_oo = 3
    fail = 4


class shs_shor_outcome(C.Structure):
    _fields_ = [("classification", C.c_int32), ("r_even", C.c_uint8), ("a_r_is_one", C.c_uint8),
                ("a_half_not_minus_one", C.c_uint8), ("order_match", C.c_uint8),
                ("k", C.c_uint64 * 2), ("r", C.c_uint64 * 2), ("n_factors", C.c_uint32),
                ("pad", C.c_uint32), ("factors", C.c_uint64 * 4)]


OUTCOME_DTYPE = np.dtype([("classification", np.int32), ("r_even", np.uint8),
                          ("a_r_is_one", np.uint8), ("a_half_not_minus_one", np.uint8),
                          ("order_match", np.uint8), ("k", np.uint64, 2), ("r", np.uint64, 2),
                          ("n_factors", np.uint32), ("pad", np.uint32), ("factors", np.uint64, 4)])
assert OUTCOME_DTYPE.itemsize == C.sizeof(shs_shor_outcome)


@dataclass
class StandardChecks:
    r_even: bool = False
    a_r_is_one: bool = False
    a_half_not_minus_one: bool = False

    def all(self) -> bool:
        return self.r_even and self.a_r_is_one and self.a_half_not_minus_one


@dataclass
class PostProcessOutcome:
    classification: Classification = Classification.fail
    convergent: Tuple[int, int] = (0, 1)  # (k, r)
    checks: StandardChecks = field(default_factory=StandardChecks)
    order_match: Optional[bool] = None
    factors: List[int] = field(default_factory=list)


def shor_postprocess_array(j: np.ndarray, t: int, N: int, a: int,
                           known_order: Optional[int] = None, device: int = 0) -> np.ndarray:
    """shor_standard_procedure for every row of j (uint64, shape (count, 2) =
    (lo, hi) words, as IterativeShorEngine.run_batch_array returns), on the
    device. Returns a structured array of OUTCOME_DTYPE."""
    j = np.ascontiguousarray(j, dtype=np.uint64).reshape(-1, 2)
    out = np.zeros(len(j), dtype=OUTCOME_DTYPE)
    _raise(L.load().shs_shor_postprocess(j.ctypes.data_as(C.POINTER(C.c_uint64)), len(j), t, N, a,
                                       known_order or 0, 0 if known_order is None else 1, device,
                                       out.ctypes.data))
    return out


@dataclass
class EkeraParams:  # postprocess.hpp:43-53
    B: int = 1
    c: int = 1
    k: int = 100
    varsigma: int = 1
    m: int = 1
    ell: int = 0
    rho_budget: int = 0  # recover_order's factorize() budget (0: the reference's 10^7)

    @staticmethod
    def for_problem(L: int, t: int) -> "EkeraParams":
        """(B, c, k, varsigma) = (L, 1, 100, 1), m = L, ell = t - L (postprocess.cpp:92-101)."""
        return EkeraParams(B=L, c=1, k=100, varsigma=1, m=L, ell=t - L if t > L else 0)


class shs_ekera_params(C.Structure):
    _fields_ = [("B", C.c_uint64), ("c", C.c_uint64), ("k", C.c_uint32),
                ("varsigma", C.c_uint32), ("m", C.c_uint32), ("ell", C.c_uint32),
                ("rho_budget", C.c_uint64)]


EKERA_DTYPE = np.dtype([("classification", np.int32), ("order_match", np.uint8),
                        ("has_recovered_order", np.uint8), ("has_offset", np.uint8),
                        ("timeout", np.uint8), ("k", np.uint64, 2), ("r", np.uint64, 2),
                        ("recovered_order", np.uint64), ("candidate_offset", np.int64),
                        ("n_factors", np.uint32), ("pad2", np.uint32), ("factors", np.uint64, 4)])


def ekera_postprocess_array(j: np.ndarray, t: int, N: int, a: int, params: EkeraParams,
                            seed: int, idx0: int = 0, known_order: Optional[int] = None,
                            device: int = 0) -> np.ndarray:
    """ekera_postprocess for every row of j (shot idx0 + row, its RngStream
    (seed, shot, 1, postprocess) as run_problem builds it), on the device."""
    j = np.ascontiguousarray(j, dtype=np.uint64).reshape(-1, 2)
    out = np.zeros(len(j), dtype=EKERA_DTYPE)
    prm = shs_ekera_params(params.B, params.c, params.k, params.varsigma, params.m, params.ell,
                           params.rho_budget)
    _raise(L.load().shs_ekera_postprocess(j.ctypes.data_as(C.POINTER(C.c_uint64)), len(j), t, N,
                                          a, C.byref(prm), seed, idx0, known_order or 0,
                                          0 if known_order is None else 1, device,
                                          out.ctypes.data))
    return out


@dataclass
class EkeraOutcome(PostProcessOutcome):
    recovered_order: Optional[int] = None
    candidate_offset: Optional[int] = None


def ekera_outcome_from_record(rec) -> EkeraOutcome:
    om = int(rec["order_match"])
    return EkeraOutcome(
        classification=Classification(int(rec["classification"])),
        convergent=(int(rec["k"][0]) | (int(rec["k"][1]) << 64),
                    int(rec["r"][0]) | (int(rec["r"][1]) << 64)),
        order_match=None if om == 2 else bool(om),
        factors=[int(x) for x in rec["factors"][:int(rec["n_factors"])]],
        recovered_order=int(rec["recovered_order"]) if rec["has_recovered_order"] else None,
        candidate_offset=int(rec["candidate_offset"]) if rec["has_offset"] else None)


def ekera_postprocess(j: int, t: int, N: int, a: int, params: EkeraParams, seed: int, idx: int,
                      known_order: Optional[int] = None, device: int = 0) -> EkeraOutcome:
    """postprocess.cpp:138-171 for one bit string (on the device)."""
    arr = np.array([[j & (2**64 - 1), j >> 64]], dtype=np.uint64)
    return ekera_outcome_from_record(
        ekera_postprocess_array(arr, t, N, a, params, seed, idx, known_order, device)[0])


def outcome_from_record(rec) -> PostProcessOutcome:
    om = int(rec["order_match"])
    return PostProcessOutcome(
        classification=Classification(int(rec["classification"])),
        convergent=(int(rec["k"][0]) | (int(rec["k"][1]) << 64),
                    int(rec["r"][0]) | (int(rec["r"][1]) << 64)),
        checks=StandardChecks(bool(rec["r_even"]), bool(rec["a_r_is_one"]),
                              bool(rec["a_half_not_minus_one"])),
        order_match=None if om == 2 else bool(om),
        factors=[int(x) for x in rec["factors"][:int(rec["n_factors"])]])


def shor_standard_procedure(j: int, t: int, N: int, a: int, known_order: Optional[int] = None,
                            device: int = 0) -> PostProcessOutcome:
    """postprocess.cpp:55-89 for one bit string (on the device)."""
    arr = np.array([[j & (2**64 - 1), j >> 64]], dtype=np.uint64)
    return outcome_from_record(shor_postprocess_array(arr, t, N, a, known_order, device)[0])


# ------------------------------------------------------------- ground truth
def _factorize(n: int) -> Dict[int, int]:
    """Prime factorisation by trial division (the multiplicative_order helper
    for lambda = lcm(p-1, q-1); fine for the moduli this engine holds)."""
    out: Dict[int, int] = {}
    d = 2
    while d * d <= n:
        while n % d == 0:
            out[d] = out.get(d, 0) + 1
            n //= d
        d += 1 if d == 2 else 2
    if n > 1:
        out[n] = out.get(n, 0) + 1
    return out


def multiplicative_order(a: int, N: int, known_factors: Optional[Tuple[int, int]] = None) -> int:
    """Exact order of a mod N (numtheory.cpp:207-234): brute force below 2^20,
    else among the divisors of lcm(p-1, q-1) from the known factors."""
    if N < 2:
        raise ValueError("multiplicative_order: modulus < 2")
    a %= N
    if math.gcd(a, N) != 1:
        raise ValueError("multiplicative_order: gcd(a, N) != 1")
    if a == 1:
        return 1
    if N < (1 << 20) and not known_factors:
        x, r = a, 1
        while x != 1:
            x = x * a % N
            r += 1
        return r
    if not known_factors:
        raise ValueError("multiplicative_order: large modulus needs known factors")
    p, q = known_factors
    if p * q != N:
        raise ValueError("multiplicative_order: p*q != N")
    lam = (p - 1) * (q - 1) // math.gcd(p - 1, q - 1)
    order = lam
    for prime, e in sorted(_factorize(lam).items()):
        for _ in range(e):
            if order % prime == 0 and pow(a, order // prime, N) == 1:
                order //= prime
            else:
                break
    return order


# ---------------------------------------------------------- run_problem
@dataclass
class RRatioHistogram:  # harness.hpp:39-44
    reciprocal: Dict[int, int] = field(default_factory=dict)
    overflow: int = 0
    other: int = 0
    total_lucky: int = 0


@dataclass
class ProblemResult:  # harness.hpp:46-61
    problem: FactoringProblem
    order: int = 1
    M: int = 0
    success: int = 0
    lucky_ne: int = 0
    lucky_no: int = 0
    lucky_oo: int = 0
    fail: int = 0
    first_factor_index: Optional[int] = None
    first_order_index: Optional[int] = None
    r_ratio: RRatioHistogram = field(default_factory=RRatioHistogram)
    order_solvable: bool = False

    def lucky_total(self) -> int:
        return self.lucky_ne + self.lucky_no + self.lucky_oo

    def success_fraction(self) -> float:
        return self.success / self.M

    def success_lucky_fraction(self) -> float:
        return (self.success + self.lucky_total()) / self.M


def tally(result: ProblemResult, outcomes: np.ndarray) -> ProblemResult:
    """note_outcome (harness.cpp:82-104) over a batch, in shot order."""
    cls = outcomes["classification"]
    counts = np.bincount(cls, minlength=5)
    result.success += int(counts[Classification.success])
    result.lucky_ne += int(counts[Classification.lucky_ne])
    result.lucky_no += int(counts[Classification.lucky_no])
    result.lucky_oo += int(counts[Classification.lucky_oo])
    result.fail += int(counts[Classification.fail])
    got = np.flatnonzero(outcomes["n_factors"] > 0)
    if len(got) and result.first_factor_index is None:
        result.first_factor_index = int(got[0]) + 1
    r = outcomes["r"][:, 0]  # r < N < 2^64: the low word
    hit = np.flatnonzero(r == np.uint64(result.order))
    if len(hit) and result.first_order_index is None:
        result.first_order_index = int(hit[0]) + 1
    lucky = (cls == Classification.lucky_ne) | (cls == Classification.lucky_no) | \
            (cls == Classification.lucky_oo)
    rl = r[lucky].astype(object)
    h = result.r_ratio
    h.total_lucky += len(rl)
    for rv in rl:
        rv = int(rv)
        if rv > result.order:
            h.overflow += 1
        elif rv != 0 and result.order % rv == 0:
            D = result.order // rv
            h.reciprocal[D] = h.reciprocal.get(D, 0) + 1
        else:
            h.other += 1
    return result


def run_problem(problem: FactoringProblem, M: int, error: Optional[ErrorConfig] = None,
                options: Optional[SimulatorOptions] = None,
                engine: Optional[IterativeShorEngine] = None,
                post_mode: str = "shor") -> ProblemResult:
    """run_problem (harness.cpp:109-148; simulator backend): shots m = 0 .. M-1
    are engine.run(problem.seed, m) — whole runs on the device for small
    problems — then shor_standard_procedure ("shor") or ekera_postprocess with
    EkeraParams.for_problem(L, t) and RngStream(seed, m, 1, postprocess)
    ("ekera"), with the known order, on the device, tallied in shot order."""
    if post_mode not in ("shor", "ekera"):
        raise ValueError(f"post_mode must be shor or ekera, not {post_mode!r}")
    if not problem.p or not problem.q:
        raise ValueError("campaign problems need known factors for verification labels")
    res = ProblemResult(problem=problem, M=M)
    res.order = multiplicative_order(problem.a, problem.N, (problem.p, problem.q))
    res.order_solvable = res.order % 2 == 0 and \
        pow(problem.a, res.order // 2, problem.N) != problem.N - 1
    own = engine is None
    if own:
        engine = IterativeShorEngine(problem, error or ErrorConfig(), options or SimulatorOptions())
    try:
        j = engine.run_batch_array(problem.seed, 0, M)
        dev = (options or SimulatorOptions()).device
        if post_mode == "shor":
            outcomes = shor_postprocess_array(j, problem.t, problem.N, problem.a, res.order, dev)
        else:
            outcomes = ekera_postprocess_array(j, problem.t, problem.N, problem.a,
                                               EkeraParams.for_problem(problem.L, problem.t),
                                               problem.seed, 0, res.order, dev)
    finally:
        if own:
            engine.close()
    return tally(res, outcomes)


def factorize(n: int, rho_budget: int = 10_000_000, device: int = 0):
    """factorize (numtheory.cpp:170-187) on the device: [(prime, exponent)]
    ascending; FactorizationTimeoutError once the Pollard-rho budget runs out."""
    primes = (C.c_uint64 * 64)()
    exps = (C.c_uint32 * 64)()
    cnt = C.c_uint32()
    _raise(L.load().shs_factorize(n, rho_budget, device, primes, exps, C.byref(cnt)))
    return [(primes[i], exps[i]) for i in range(cnt.value)]
