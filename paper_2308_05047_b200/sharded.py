"""Sharded iterative-Shor engine: one shard of the state per GPU.

The state `sel` is block-sharded over G shards (shard q owns global amplitude
indices [q*S, min(N, (q+1)*S)), S a multiple of 256). Per stage every shard runs
(include/shorsim_b200.h, "sharded engine"):

    exchange   P = sel o src (only stages with a real permutation): each rank
               pulls 256 B source runs from, and pushes 1 KB destination runs to,
               the owners' buffers (NVLink peer memory across GPUs)
    probs      shard-local h0/h1 and the reference's 256-block partials, folded
               into 80 exact integer digits -> allreduce (sum) over shards ->
               correctly rounded p0, p1 (identical for every G)
    measure    host sampling, identical on every rank (same Philox stream)
    collapse   shard-local, in place over P, which becomes the next sel

Two process layouts share this driver:
  * ``LocalGroup`` — every shard in this process (virtual shards on one GPU,
    or one shard per visible GPU); barrier = stream syncs, allreduce = host sum
  * ``DistGroup`` — one shard per ``torch.distributed`` rank (NCCL or gloo);
    shards see each other's buffers through CUDA IPC handles.
The driver only sequences C-ABI calls; all amplitude arithmetic is on device.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

from . import _lib as L
from .engine import (BitString, Error, ErrorConfig, ErrorEvent, FactoringProblem, RunResult,
                     SimulatorOptions, StageTrace, _raise, sample_measurement)

NORM_TOLERANCE = 1e-9  # statevector.cpp:18


def digits_to_probs(digits: Sequence[int]):
    """Correctly rounded (p0, p1) from summed exact digits (host, no device)."""
    arr = (L.u64 * L.SHS_DIGITS)(*[int(d) for d in digits])
    p0, p1 = L.dbl(), L.dbl()
    _raise(L.load().shs_digits_to_probs(arr, C.byref(p0), C.byref(p1)))
    return p0.value, p1.value


class Shard:
    """One shard of the state on one device (ctypes over shs_shard_*)."""

    def __init__(self, problem: FactoringProblem, error: ErrorConfig,
                 options: SimulatorOptions, rank: int, nshards: int):
        self._lib = L.load()
        self.rank, self.nshards, self.t = rank, nshards, problem.t
        self._h = L.vp()
        pr = L.shs_problem(problem.N, problem.a, problem.L, problem.t, problem.seed)
        er = error.to_c()
        op = options.to_c()
        _raise(self._lib.shs_shard_create(C.byref(pr), C.byref(er), C.byref(op), rank, nshards,
                                          C.byref(self._h)))
        rng = (L.u64 * 3)()
        _raise(self._lib.shs_shard_range(self._h, rng))
        self.lo, self.hi, self.S = rng[0], rng[1], rng[2]

    def close(self):
        if getattr(self, "_h", None):
            self._lib.shs_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def buffers(self):
        out = (L.vp * 2)()
        _raise(self._lib.shs_shard_buffers(self._h, out))
        return [out[0], out[1]]

    def ipc_handles(self) -> bytes:
        buf = C.create_string_buffer(L.SHS_SHARD_IPC_BYTES)
        _raise(self._lib.shs_shard_ipc_handles(self._h, buf))
        return buf.raw

    def attach(self, peer: int, bufs):
        arr = (L.vp * 2)(*bufs)
        _raise(self._lib.shs_shard_attach(self._h, peer, arr))

    def attach_ipc(self, peer: int, handles: bytes):
        buf = C.create_string_buffer(handles, L.SHS_SHARD_IPC_BYTES)
        _raise(self._lib.shs_shard_attach_ipc(self._h, peer, buf))

    def attach_local(self, peer: "Shard"):
        """a peer shard of this process: buffers, stage digits and ordering events"""
        _raise(self._lib.shs_shard_attach_local(self._h, peer._h))

    def set_barrier(self, name: str):
        _raise(self._lib.shs_shard_set_barrier(self._h, name.encode()))

    def init(self):
        _raise(self._lib.shs_shard_init(self._h))

    def needs_exchange(self, s: int) -> bool:
        return bool(self._lib.shs_shard_needs_exchange(self._h, s))

    def exchange(self, s: int):
        _raise(self._lib.shs_shard_exchange(self._h, s))

    def probs(self, s: int, prefix: int) -> List[int]:
        out = (L.u64 * L.SHS_DIGITS)()
        _raise(self._lib.shs_shard_probs(self._h, s, prefix & (2**64 - 1), prefix >> 64, out))
        return list(out)

    def collapse(self, src_group: int, p_source: float):
        _raise(self._lib.shs_shard_collapse(self._h, src_group, p_source))

    def sync(self):
        _raise(self._lib.shs_shard_sync(self._h))

    def set_sparse(self, enable: bool):
        _raise(self._lib.shs_shard_set_sparse(self._h, 1 if enable else 0))

    def sparse_stages(self) -> int:
        return self._lib.shs_shard_sparse_stages(self._h)

    def kahan(self) -> bool:
        """p0/p1 combined like the reference (sequential Kahan; small N under AUTO)"""
        return bool(self._lib.shs_shard_kahan(self._h))

    def kahan_probs(self):
        p0, p1 = L.dbl(), L.dbl()
        _raise(self._lib.shs_shard_kahan_probs(self._h, C.byref(p0), C.byref(p1)))
        return p0.value, p1.value

    def state_read(self, x: int, first: int, count: int):
        out = (L.dbl * (2 * count))()
        _raise(self._lib.shs_shard_state_read(self._h, x, first, count, out))
        return out

    def stage_read(self, x: int, first: int, count: int):
        out = (L.dbl * (2 * count))()
        _raise(self._lib.shs_shard_stage_read(self._h, x, first, count, out))
        return out

    def set_timing(self, enable: bool):
        _raise(self._lib.shs_shard_set_timing(self._h, 1 if enable else 0))

    def kernel_times(self):
        ms = (L.dbl * 5)()
        n = (L.u64 * 5)()
        _raise(self._lib.shs_shard_kernel_times(self._h, ms, n))
        return {k: (ms[i], n[i]) for i, k in enumerate(("probs", "exchange", "collapse", "pack",
                                                         "unpack"))}

    def launch_count(self) -> int:
        return self._lib.shs_shard_launch_count(self._h)

    def set_timeline(self, enable: bool):
        _raise(self._lib.shs_shard_set_timeline(self._h, 1 if enable else 0))

    def timeline(self):
        """[(kind, start_ms, end_ms)] of the last device-resident run's launches"""
        n = self._lib.shs_shard_timeline(self._h, None, 0)
        out = (L.dbl * (3 * max(n, 1)))()
        self._lib.shs_shard_timeline(self._h, out, n)
        kinds = ("probs", "exchange", "collapse", "pack", "unpack")
        return [(kinds[int(out[3 * i])], out[3 * i + 1], out[3 * i + 2]) for i in range(n)]

    def stream_handle(self) -> int:
        return self._lib.shs_shard_stream(self._h) or 0


class LocalGroup:
    """All shards live in this process: barrier = device syncs, allreduce = sum."""

    def __init__(self, shards: Sequence):
        self.shards = list(shards)
        for a in self.shards:
            for b in self.shards:
                if a is not b:
                    a.attach_local(b)

    def barrier(self):
        for sh in self.shards:
            sh.sync()

    def allreduce(self, digits: List[int]) -> List[int]:
        return digits


class DistGroup:
    """One shard per torch.distributed rank; peers attached through CUDA IPC."""

    def __init__(self, shard, attach_ipc: bool = True, device=None):
        import os
        import torch
        import torch.distributed as dist
        self.dist, self.torch = dist, torch
        self.shards = [shard]
        self.device = device
        if attach_ipc:
            handles = [None] * dist.get_world_size()
            dist.all_gather_object(handles, shard.ipc_handles())
            for q, h in enumerate(handles):
                if q != shard.rank:
                    shard.attach_ipc(q, h)
            # the node-local host barrier of device-resident runs (shs_shards_run)
            name = [f"/shs_{os.getpid()}_{os.urandom(6).hex()}" if dist.get_rank() == 0 else None]
            dist.broadcast_object_list(name, src=0)
            shard.set_barrier(name[0])
            dist.barrier()

    def barrier(self):
        for sh in self.shards:
            sh.sync()
        self.dist.barrier()

    def allreduce(self, digits: List[int]) -> List[int]:
        t = self.torch.tensor(digits, dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return [int(x) for x in t.tolist()]


class ShardedShorEngine:
    """IterativeShorEngine semantics (run(seed, bitstring_index)) over a sharded
    state. ``shards`` are this process's shards; ``group`` sequences them with
    the others (LocalGroup / DistGroup). With combine="exact" the results equal
    the single-GPU engine's bit for bit."""

    def __init__(self, problem: FactoringProblem, error: Optional[ErrorConfig],
                 options: Optional[SimulatorOptions], shards: Sequence, group):
        self.problem = problem
        self.error = error if error is not None else ErrorConfig()
        self.options = options if options is not None else SimulatorOptions()
        self.shards = list(shards)
        self.group = group
        self.t = problem.t

    @staticmethod
    def virtual(problem: FactoringProblem, error: Optional[ErrorConfig] = None,
                options: Optional[SimulatorOptions] = None, nshards: int = 2,
                devices: Optional[Sequence[int]] = None) -> "ShardedShorEngine":
        """G shards in this process (on one GPU, or spread over `devices`)."""
        import dataclasses
        error = error if error is not None else ErrorConfig()
        options = options if options is not None else SimulatorOptions()
        shards = []
        for r in range(nshards):
            o = dataclasses.replace(options, device=(devices[r % len(devices)] if devices
                                                     else options.device))
            shards.append(Shard(problem, error, o, r, nshards))
        return ShardedShorEngine(problem, error, options, shards, LocalGroup(shards))

    def close(self):
        for sh in self.shards:
            sh.close()

    def set_sparse(self, enable: bool):
        """sparse prefix of run() (on by default where it applies); results identical"""
        for sh in self.shards:
            sh.set_sparse(enable)

    def sparse_stages(self) -> int:
        return self.shards[0].sparse_stages()

    # -- step API (what run() is made of)
    def state_init(self):
        for sh in self.shards:
            sh.init()

    def stage_probs(self, s: int, prefix: int = 0):
        if any(sh.needs_exchange(s) for sh in self.shards):
            for sh in self.shards:
                sh.exchange(s)
            self.group.barrier()  # every P complete before anyone reads it
        digits = [0] * L.SHS_DIGITS
        for sh in self.shards:
            d = sh.probs(s, prefix)
            digits = [a + b for a, b in zip(digits, d)]
        digits = self.group.allreduce(digits)
        p0, p1 = digits_to_probs(digits)
        if self.shards[0].kahan():  # the reference's sequential Kahan over all partials
            self.group.barrier()  # (allreduce ordered the digits; partials are device-side)
            p0, p1 = self.shards[0].kahan_probs()
        if self.options.check_norms and abs(p0 + p1 - 1.0) > NORM_TOLERANCE:
            raise Error(f"statevector norm drifted beyond 1e-9 at stage {s}")
        return p0, p1

    def stage_collapse(self, src_group: int, p_source: float):
        for sh in self.shards:
            sh.collapse(src_group, p_source)
        self.group.barrier()  # the next exchange reads every shard's new sel

    def run(self, seed: int, bitstring_index: int) -> RunResult:
        """IterativeShorEngine::run, statevector.cpp:323-412, sharded and
        device-resident (shs_shards_run): per stage exchange, probs, the exact
        digit sum and the measurement run on every device, ordered across
        shards by (IPC) events; the host only enqueues. Collective over the
        group's processes."""
        arr = (L.vp * len(self.shards))(*[sh._h for sh in self.shards])
        j, js = (L.u64 * 2)(), (L.u64 * 2)()
        tr = (L.shs_stage_trace * self.t)()
        _raise(L.load().shs_shards_run(arr, len(self.shards), seed, bitstring_index, j, js, tr))
        trace = [StageTrace(x.cbit, x.p1, x.sampled_bit, x.observed_bit,
                            ErrorEvent(bool(x.classical_flip), bool(x.quantum_error_branch)))
                 for x in tr]
        return RunResult(BitString(self.t, j[0] | (j[1] << 64)), js[0] | (js[1] << 64), trace)

    def run_stepwise(self, seed: int, bitstring_index: int) -> RunResult:
        """The same run sequenced from the host through the per-stage calls
        (exchange / probs / digit allreduce / host sampling / collapse)."""
        self.state_init()
        observed = sampled = 0
        trace = []
        idx32 = bitstring_index & 0xFFFFFFFF
        for s in range(self.t):
            p0, p1 = self.stage_probs(s, observed)
            m = sample_measurement(p1, seed, idx32, s, self.error)
            trace.append(StageTrace(s, p1, m["sampled_bit"], m["observed_bit"],
                                    ErrorEvent(m["classical_flip"], m["error_branch"])))
            observed |= m["observed_bit"] << s
            sampled |= m["sampled_bit"] << s
            if s + 1 < self.t:
                src_group = 1 - m["sampled_bit"] if m["error_branch"] else m["sampled_bit"]
                self.stage_collapse(src_group, p1 if src_group == 1 else p0)
        j = observed
        if int(self.error.kind) == 5:  # ErrorKind::bitflip
            j = _bitflip(j, self.t, self.error.delta, seed, idx32)
        return RunResult(BitString(self.t, j), sampled, trace)


def _bitflip(j: int, t: int, delta: float, seed: int, idx: int) -> int:
    """bitflip_bitstring (statevector.cpp:404-409) through the library's host model."""
    arr = (L.u64 * 2)(j & (2**64 - 1), j >> 64)
    _raise(L.load().shs_bitflip(arr, t, delta, seed, idx))
    return arr[0] | (arr[1] << 64)
