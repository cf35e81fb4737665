"""The reference's per-gate ("step/measure") API on a device-resident state
(SURVEY §8a rows A5, A6), mirroring /root/reference/proj/include/shorsim/
statevector.hpp:20-133 with the same names, argument meaning and errors:

    ShardLayout, make_shard_layout, ShardedState (amp / set_amp / amp_xy /
    group_base / norm_squared / group_norm_squared, value copies), init_state,
    apply_oracle, apply_phase, stage_phase, apply_hadamard_top, measure_top,
    reset_top, ExchangePlan / build_permutation_plan / plan_receive_lists /
    plan_send_lists.

The amplitudes live in device memory (shs_sv, csrc/sv.cu); every gate is a
kernel reproducing the reference's arithmetic bit for bit. measure_top samples
on the host from the device's group norm, as the reference does
(statevector.cpp:236-261)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

from . import _lib as L
from .engine import ErrorConfig, _raise, sample_measurement


@dataclass(frozen=True)
class ShardLayout:
    """ShardLayout, statevector.hpp:20-30 (group = most significant index bit)."""
    n: int = 2
    g: int = 1

    def shard_count(self) -> int:
        return 1 << self.g

    def shard_size(self) -> int:
        return 1 << (self.n - self.g)

    def group_size(self) -> int:
        return 1 << (self.n - 1)

    def group_shards(self) -> int:
        return 1 << (self.g - 1)

    def shard_of(self, glob: int) -> int:
        return glob >> (self.n - self.g)

    def offset_of(self, glob: int) -> int:
        return glob & (self.shard_size() - 1)


def make_shard_layout(n: int, shard_count: int) -> ShardLayout:
    """make_shard_layout, statevector.cpp:65-72 (ValueError = std::invalid_argument)."""
    if n < 2 or n > 33:
        raise ValueError("shard layout: need 2 <= n <= 33")
    if shard_count < 2 or shard_count & (shard_count - 1):
        raise ValueError("shard layout: shard count must be a power of two >= 2")
    g = shard_count.bit_length() - 1
    if g > n - 1:
        raise ValueError("shard layout: more shards than group states")
    return ShardLayout(n, g)


class ShardedState:
    """ShardedState, statevector.hpp:33-65, on the device (copy() = value copy)."""

    def __init__(self, n: int = 2, shard_count: int = 2, device: int = 0, _handle=None):
        self._lib = L.load()
        self.device = device
        if _handle is not None:
            self._h = _handle
        else:
            self._h = L.vp()
            _raise(self._lib.shs_sv_create(n, shard_count, device, C.byref(self._h)))
        lay = (L.u32 * 2)()
        _raise(self._lib.shs_sv_layout(self._h, lay))
        self._layout = ShardLayout(lay[0], lay[1])

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.shs_sv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def copy(self) -> "ShardedState":
        h = L.vp()
        _raise(self._lib.shs_sv_clone(self._h, C.byref(h)))
        return ShardedState(device=self.device, _handle=h)

    __copy__ = copy

    def layout(self) -> ShardLayout:
        return self._layout

    def qubits(self) -> int:
        return self._layout.n

    def group_base(self, x: int) -> int:
        return 0 if x == 0 else self._layout.group_size()

    def read(self, first: int, count: int) -> List[complex]:
        out = (L.dbl * (2 * count))()
        _raise(self._lib.shs_sv_read(self._h, first, count, out))
        return [complex(out[2 * i], out[2 * i + 1]) for i in range(count)]

    def read_array(self, first: int, count: int):
        import numpy as np
        out = np.empty(2 * count, dtype=np.float64)
        _raise(self._lib.shs_sv_read(self._h, first, count, out.ctypes.data_as(C.POINTER(L.dbl))))
        return out

    def write(self, first: int, values) -> None:
        vals = [complex(v) for v in values]
        arr = (L.dbl * (2 * len(vals)))(*[x for v in vals for x in (v.real, v.imag)])
        _raise(self._lib.shs_sv_write(self._h, first, len(vals), arr))

    def amp(self, glob: int) -> complex:
        return self.read(glob, 1)[0]

    def set_amp(self, glob: int, v: complex) -> None:
        self.write(glob, [v])

    def amp_xy(self, x: int, y: int) -> complex:
        return self.amp(self.group_base(x) + y)

    def group_norms(self) -> Tuple[float, float]:
        out = (L.dbl * 2)()
        _raise(self._lib.shs_sv_group_norms(self._h, out))
        return out[0], out[1]

    def group_norm_squared(self, x: int) -> float:
        return self.group_norms()[x]

    def norm_squared(self) -> float:
        p0, p1 = self.group_norms()
        return p0 + p1


def _pair(q) -> "C.Array":
    a0, a1 = complex(q[0]), complex(q[1])
    return (L.dbl * 4)(a0.real, a0.imag, a1.real, a1.imag)


def init_state(n: int, top_qubit_state, shard_count: int, device: int = 0) -> ShardedState:
    """init_state, statevector.cpp:126-131: |q>|0...01> with q = (a0, a1)."""
    st = ShardedState(n, shard_count, device)
    _raise(st._lib.shs_sv_init_state(st._h, _pair(top_qubit_state)))
    return st


def apply_oracle(state: ShardedState, a_pow: int, n_modulus: int) -> None:
    """apply_oracle, statevector.cpp:223-244 (NotInvertibleError as the reference)."""
    _raise(state._lib.shs_sv_apply_oracle(state._h, a_pow, n_modulus))


def stage_phase(cbit: int, measured_bits_so_far: int) -> float:
    """stage_phase, statevector.cpp:201-206 (glibc arithmetic, as the engine's host side)."""
    if cbit == 0:
        return 0.0
    return math.pi * float(measured_bits_so_far) * 2.0 ** (-cbit)


def apply_phase(state: ShardedState, cbit: int, measured_bits_so_far: int) -> None:
    """apply_phase, statevector.cpp:246-253."""
    p = measured_bits_so_far
    _raise(state._lib.shs_sv_apply_phase(state._h, cbit, p & (2**64 - 1), p >> 64))


def apply_hadamard_top(state: ShardedState) -> None:
    """apply_hadamard_top, statevector.cpp:255-270."""
    _raise(state._lib.shs_sv_apply_hadamard_top(state._h))


def measure_top(state: ShardedState, seed: int, idx: int, stage: int,
                error: Optional[ErrorConfig] = None) -> dict:
    """measure_top, statevector.cpp:258-261: sample_measurement(group_norm_squared(1))
    with RngStream(seed, idx, stage, measurement)."""
    p1 = state.group_norm_squared(1)
    m = sample_measurement(p1, seed, idx, stage, error if error is not None else ErrorConfig())
    m["p1"] = p1
    return m


def reset_top(state: ShardedState, bit: int, error_branch: bool, reinit, p_source: float) -> None:
    """reset_top(bit, branch, reinit, p_source), statevector.cpp:263-283
    (DegenerateBranchError below 1e-300)."""
    _raise(state._lib.shs_sv_reset_top(state._h, bit, 1 if error_branch else 0, _pair(reinit),
                                       p_source))


@dataclass
class ExchangePlan:
    """ExchangePlan, statevector.hpp:75-89 (computed on the device)."""
    modulus: int = 1
    a_pow: int = 1
    a_inv: int = 1
    y_limit: int = 0
    layout: ShardLayout = field(default_factory=ShardLayout)
    gather: List[int] = field(default_factory=list)
    identity: bool = False
    pair_counts: List[List[int]] = field(default_factory=list)


def build_permutation_plan(a_pow: int, n_modulus: int, layout: ShardLayout,
                           device: int = 0) -> ExchangePlan:
    """build_permutation_plan, statevector.cpp:133-154."""
    lib = L.load()
    inv, ident, ylim = L.u64(), L.i32(), L.u64()
    _raise(lib.shs_plan_build(a_pow, n_modulus, layout.n, layout.shard_count(), device,
                              C.byref(inv), C.byref(ident), C.byref(ylim), None, None))
    gs = layout.group_shards()
    gather = (L.u64 * max(ylim.value, 1))()
    pc = (L.u64 * (gs * gs))()
    _raise(lib.shs_plan_build(a_pow, n_modulus, layout.n, layout.shard_count(), device,
                              None, None, None, gather, pc))
    return ExchangePlan(n_modulus, a_pow % n_modulus, inv.value, ylim.value, layout,
                        list(gather[:ylim.value]), bool(ident.value),
                        [list(pc[s * gs:(s + 1) * gs]) for s in range(gs)])


@dataclass
class ShardIndexList:
    """ShardIndexList, statevector.hpp:91-94."""
    xrank: int
    local_index: List[int]


def _lists(plan: ExchangePlan, xrank: int, send: int, device: int) -> List[ShardIndexList]:
    lib = L.load()
    lay = plan.layout
    gs = lay.group_shards()
    counts = (L.u64 * gs)()
    idx = (L.u64 * max(lay.shard_size(), 1))()
    _raise(lib.shs_plan_lists(plan.a_pow, plan.modulus, lay.n, lay.shard_count(), xrank, send,
                              device, counts, idx))
    out, k = [], 0
    for peer in range(gs):
        c = counts[peer]
        if c:
            out.append(ShardIndexList(peer, list(idx[k:k + c])))
        k += c
    return out


def plan_receive_lists(plan: ExchangePlan, dst_xrank: int, device: int = 0) -> List[ShardIndexList]:
    """plan_receive_lists, statevector.cpp:156-168."""
    return _lists(plan, dst_xrank, 0, device)


def plan_send_lists(plan: ExchangePlan, src_xrank: int, device: int = 0) -> List[ShardIndexList]:
    """plan_send_lists, statevector.cpp:170-181."""
    return _lists(plan, src_xrank, 1, device)
