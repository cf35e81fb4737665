"""TEST INFRASTRUCTURE: a numpy stand-in for one shard of the sharded engine,
with the same methods as paper_2308_05047_b200.sharded.Shard, so the product
driver (ShardedShorEngine + DistGroup) can run across gloo processes on a CPU.

Arithmetic restates the reference stage (statevector.cpp:339-401, Appendix A)
with numpy float64 elementwise ops (IEEE round-to-nearest, no contraction); block
partials are sequential (np.cumsum) inside the fixed 256-blocks; the exact
digits of Σ S_b follow the device format (value = F * 2^-1088, 40 x 32-bit)."""
from __future__ import annotations

import math

import numpy as np

K = 0.70710678118654752440
ANCHOR = 1088


def exact_digits(values) -> list:
    """40 x 32-bit digits of F = Σ v * 2^1088 (exact, v >= 0 doubles)."""
    F = 0
    for v in values:
        if v == 0.0:
            continue
        num, den = float(v).as_integer_ratio()
        F += num * ((1 << ANCHOR) // den)
    return [(F >> (32 * i)) & 0xFFFFFFFF for i in range(40)]


class CpuShard:
    def __init__(self, N, a, t, w, rank, nshards, dist):
        self.N, self.t, self.rank, self.nshards, self.dist = N, t, rank, nshards, dist
        per = -(-N // nshards)
        self.S = -(-per // 256) * 256
        self.lo = rank * self.S
        self.hi = min(N, self.lo + self.S)
        self.w = w  # (w0r, w0i, w1r, w1i)
        pows = [0] * t
        pows[t - 1] = a % N
        for s in range(t - 1, 0, -1):
            pows[s - 1] = pows[s] * pows[s] % N
        self.a_pows = pows
        self.a_invs = [pow(p, -1, N) if p != 1 else 1 for p in pows]
        self.init()

    # -- Shard interface
    def init(self):
        n = self.hi - self.lo
        self.sel = np.zeros((n, 2))
        if self.lo <= 1 < self.hi:
            self.sel[1 - self.lo, 0] = 1.0
        self.inv = 1.0
        self.e1 = True
        self.P = None
        self.pending = None

    def kahan(self):
        return False  # this stand-in combines exactly (digits); compared with the exact oracle

    def needs_exchange(self, s):
        return not self.e1 and self.a_pows[s] != 1

    def exchange(self, s):
        import torch
        n = self.hi - self.lo
        buf = np.zeros((self.S, 2))
        buf[:n] = self.sel
        parts = [torch.zeros(self.S, 2, dtype=torch.float64) for _ in range(self.nshards)]
        self.dist.all_gather(parts, torch.from_numpy(buf))
        full = np.concatenate([p.numpy() for p in parts])[: self.N]
        z = np.arange(self.lo, self.hi, dtype=object)
        src = np.array([(self.a_invs[s] * int(x)) % self.N for x in z], dtype=np.int64)
        self.P = full[src]

    def _h(self, s):
        x = self.sel
        if self.e1 or self.a_pows[s] == 1:
            xs = x
            if self.e1 and self.a_pows[s] != 1:  # implicit |1>: xs = e_1 at src(z) == 1
                xs = np.zeros_like(x)
                z = self.a_pows[s] % self.N  # src(z) = 1  <=>  z = a_pow
                if self.lo <= z < self.hi:
                    xs[z - self.lo, 0] = 1.0
        else:
            xs = self.P
        inv, (w0r, w0i, w1r, w1i) = self.inv, self.w
        xr, xi = x[:, 0] * inv, x[:, 1] * inv
        sr, si = xs[:, 0] * inv, xs[:, 1] * inv
        ur, ui = w0r * xr - w0i * xi, w0r * xi + w0i * xr
        vr, vi = w1r * sr - w1i * si, w1r * si + w1i * sr
        if self.phase_mul:
            vr, vi = vr * self.ph[0] - vi * self.ph[1], vr * self.ph[1] + vi * self.ph[0]
        return ((ur + vr) * K, (ui + vi) * K), ((ur - vr) * K, (ui - vi) * K)

    def probs(self, s, prefix):
        phi = 0.0 if s == 0 else math.pi * float(prefix) * 2.0 ** (-s)
        self.ph = (1.0 * math.cos(phi), 1.0 * math.sin(phi))
        self.phase_mul = self.a_pows[s] != 1 or phi != 0.0
        h0, h1 = self._h(s)
        self.pending = (s, h0, h1)
        digits = []
        for hr, hi in (h0, h1):
            nrm = hr * hr + hi * hi
            pad = (-len(nrm)) % 256
            blocks = np.concatenate([nrm, np.zeros(pad)]).reshape(-1, 256)
            sums = np.cumsum(blocks, axis=1)[:, -1]  # sequential in-block folds
            digits += exact_digits(sums.tolist())
        return digits

    def collapse(self, src_group, p_source):
        _, h0, h1 = self.pending
        hr, hi = h1 if src_group else h0
        self.sel = np.stack([hr, hi], axis=1)
        self.inv = 1.0 / math.sqrt(p_source)
        self.e1 = False
        self.pending = None

    def sync(self):
        pass
