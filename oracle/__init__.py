"""TEST INFRASTRUCTURE ONLY — CPU checkers for the GPU engine.

Two checkers live here:

* ``Oracle``: ctypes binding of ``shor_oracle.c``, our plain-C restatement of
  ``IterativeShorEngine`` (/root/reference/proj/src/statevector.cpp:285-412)
  on the compressed N-amplitude state.
* ``Reference``: ctypes binding of ``_ref/libshorsim_ref.so``, the UNMODIFIED
  reference library compiled from /root/reference/proj/src by ``Makefile`` plus
  the marshalling shim ``ref_shim.cpp``. Built in the dev container (where
  /root/reference exists); the built ``.so`` travels to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package, and only as the checker or the timed
reference. The product package ``paper_2308_05047_b200`` never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libshor_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libshorsim_ref.so")
REF_SO_NATIVE = os.path.join(HERE, "_ref", "native", "libshorsim_ref.so")


def native_reference_ok() -> bool:
    """The -march=native build runs here iff this CPU has every ISA flag of the
    machine it was built on (recorded at build time)."""
    try:
        need = set(open(os.path.join(HERE, "_ref", "native", "cpu_flags")).read().split())
        for line in open("/proc/cpuinfo"):
            if line.startswith("flags"):
                return need <= set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return False


def reference_build() -> dict:
    """Which reference build Reference() loads and with which flags."""
    flags = "-std=c++20 -O3 -DNDEBUG -ffp-contract=off -include cstdint"
    if os.path.exists(REF_SO_NATIVE) and native_reference_ok():
        try:
            march = open(os.path.join(HERE, "_ref", "native", "march")).read().strip()
        except OSError:
            march = "-march=native"
        return {"path": REF_SO_NATIVE, "variant": "native",
                "flags": f"{flags} -march=native ({march} of the build host; SHORSIM_NATIVE=ON)"}
    return {"path": REF_SO, "variant": "portable",
            "flags": f"{flags} (SHORSIM_NATIVE=OFF: this CPU lacks the build host's ISA)"}
REFERENCE_SRC = "/root/reference/proj/src"
SIMULATE_REF = os.path.join(HERE, "_ref", "simulate_ref")
SIMULATE_B200 = os.path.join(HERE, "_ref", "simulate_b200")
ACCEPTANCE_REF = os.path.join(HERE, "_ref", "acceptance_ref")
ACCEPTANCE_B200 = os.path.join(HERE, "_ref", "acceptance_b200")
# the reference's own unit tests / harness compiled against include/dropin
DROPIN_TESTS = {k: os.path.join(HERE, "_ref", f"test_{k}_b200")
                for k in ("statevector", "noise", "harness")}
SIMULATE_DROPIN = os.path.join(HERE, "_ref", "simulate_dropin")

u64 = C.c_uint64
u32 = C.c_uint32
i32 = C.c_int32
dbl = C.c_double

KIND = {"none": 0, "amplitude_init": 1, "phase_init": 2, "classical_measure": 3,
        "quantum_measure": 4, "bitflip": 5}


def build(ref: bool | None = None) -> None:
    """Compile the C restatement (always) and the reference library (when the
    reference sources are present, i.e. in the dev container)."""
    targets = ["oracle"]
    if ref is None:
        ref = os.path.isdir(REFERENCE_SRC)
    if ref:
        targets.append("ref")
        # the reference's own callers linked against the B200 engine (needs the lib built)
        if os.path.exists(os.path.join(HERE, "..", "paper_2308_05047_b200", "libshorsim_b200.so")):
            targets.append("link")
    subprocess.run(["make", "-s", "-j4", "-C", HERE] + targets, check=True)


class so_error(C.Structure):
    _fields_ = [("kind", i32), ("delta", dbl), ("px", dbl), ("py", dbl), ("pz", dbl),
                ("has_pauli", i32)]


def make_error(kind="none", delta=0.0, px=0.0, py=0.0, pz=0.0, has_pauli=None):
    k = KIND[kind] if isinstance(kind, str) else int(kind)
    if has_pauli is None:
        has_pauli = k == KIND["quantum_measure"]
    return so_error(k, delta, px, py, pz, 1 if has_pauli else 0)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"status {code} {msg}")
        self.code = code


def _check(rc, lib=None):
    if rc != 0:
        msg = ""
        if lib is not None and hasattr(lib, "ref_last_error"):
            msg = lib.ref_last_error().decode()
        raise OracleError(rc, msg)


class RunTrace:
    def __init__(self, t):
        self.j = (u64 * 2)()
        self.js = (u64 * 2)()
        self.p1 = (dbl * t)()
        self.ints = (i32 * (4 * t))()

    @property
    def bits(self):
        return self.j[0] | (self.j[1] << 64)

    @property
    def sampled(self):
        return self.js[0] | (self.js[1] << 64)

    def as_dict(self):
        t = len(self.p1)
        return {
            "j": self.bits, "j_sampled": self.sampled, "p1": list(self.p1),
            "sampled_bit": [self.ints[4 * s] for s in range(t)],
            "observed_bit": [self.ints[4 * s + 1] for s in range(t)],
            "classical_flip": [self.ints[4 * s + 2] for s in range(t)],
            "quantum_error_branch": [self.ints[4 * s + 3] for s in range(t)],
        }


class Oracle:
    """Our C restatement (compressed state)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        self.lib = L
        L.so_rng_u64.restype = u64
        L.so_rng_u64.argtypes = [u64, u32, u32, u32, u32]
        L.so_rng_double.restype = dbl
        L.so_rng_double.argtypes = [u64, u32, u32, u32, u32]
        L.so_mulmod.restype = u64
        L.so_mulmod.argtypes = [u64, u64, u64]
        L.so_mod_inverse.argtypes = [u64, u64, C.POINTER(u64), C.POINTER(u64)]
        L.so_recommended_t.restype = C.c_uint
        L.so_recommended_t.argtypes = [u64]
        L.so_bit_length.restype = C.c_uint
        L.so_bit_length.argtypes = [u64]
        L.so_index_map.argtypes = [u64, u64, u64, u64, C.POINTER(u64)]
        L.so_stage_phase.restype = dbl
        L.so_stage_phase.argtypes = [C.c_uint, u64, u64]
        L.so_sample_measurement.argtypes = [dbl, u64, u32, u32, C.POINTER(so_error),
                                            C.POINTER(i32)]
        L.so_reinit_state.argtypes = [C.POINTER(so_error), C.POINTER(dbl)]
        L.so_combine_blocks.restype = dbl
        L.so_combine_blocks.argtypes = [C.POINTER(dbl), u64]
        L.so_exact_sum.restype = dbl
        L.so_exact_sum.argtypes = [C.POINTER(dbl), u64]
        L.so_engine_create.argtypes = [u64, u64, C.c_uint, C.c_uint, C.POINTER(so_error),
                                       C.c_uint, C.c_uint, C.c_int, C.POINTER(C.c_void_p)]
        L.so_engine_destroy.argtypes = [C.c_void_p]
        L.so_engine_multipliers.argtypes = [C.c_void_p, C.POINTER(u64)]
        L.so_engine_run.argtypes = [C.c_void_p, u64, u64, C.c_int, C.POINTER(u64),
                                    C.POINTER(u64), C.POINTER(dbl), C.POINTER(i32)]
        L.so_state_init.argtypes = [C.c_void_p]
        L.so_stage_probs.argtypes = [C.c_void_p, C.c_uint, u64, u64, C.c_int,
                                     C.POINTER(dbl), C.POINTER(dbl)]
        L.so_stage_read.argtypes = [C.c_void_p, C.c_int, u64, u64, C.POINTER(dbl)]
        L.so_stage_collapse.argtypes = [C.c_void_p, C.c_int, dbl]
        L.so_state_read.argtypes = [C.c_void_p, C.c_int, u64, u64, C.POINTER(dbl)]
        L.so_stage_block_sums.argtypes = [C.c_void_p, C.POINTER(dbl)]
        L.so_num_blocks.restype = u64
        L.so_num_blocks.argtypes = [C.c_void_p]
        L.so_sparse_create.argtypes = [u64, u64, C.c_uint, C.c_uint, C.POINTER(so_error), C.c_int,
                                       C.POINTER(C.c_void_p)]
        L.so_sparse_destroy.argtypes = [C.c_void_p]
        L.so_sparse_init.argtypes = [C.c_void_p]
        L.so_sparse_stage_probs.argtypes = [C.c_void_p, C.c_uint, u64, u64, C.c_int,
                                            C.POINTER(dbl), C.POINTER(dbl)]
        L.so_sparse_stage_collapse.argtypes = [C.c_void_p, C.c_int, dbl]
        L.so_sparse_size.restype = u64
        L.so_sparse_size.argtypes = [C.c_void_p]
        L.so_sparse_state.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]

    # scalar helpers
    def philox(self, key, ctr):
        out = (u32 * 4)()
        self.lib.so_philox_block(u64(key), (u32 * 4)(*ctr), out)
        return list(out)

    def mod_inverse(self, a, n):
        inv, g = u64(), u64()
        rc = self.lib.so_mod_inverse(a, n, C.byref(inv), C.byref(g))
        if rc:
            raise OracleError(rc, f"gcd={g.value}")
        return inv.value

    def index_map(self, a_pow, n, first, count):
        out = (u64 * count)()
        _check(self.lib.so_index_map(a_pow, n, first, count, out))
        return list(out)

    def sample(self, p1, seed, idx, stage, err):
        out = (i32 * 4)()
        self.lib.so_sample_measurement(p1, seed, idx, stage, C.byref(err), out)
        return list(out)

    def exact_sum(self, values):
        arr = (dbl * len(values))(*values)
        return self.lib.so_exact_sum(arr, len(values))

    def kahan(self, values):
        arr = (dbl * len(values))(*values)
        return self.lib.so_combine_blocks(arr, len(values))

    def sparse(self, N, a, L, t, err=None, check_norms=True):
        return SparseOracle(self, N, a, L, t, err, check_norms)

    def engine(self, N, a, L, t, err=None, shard_count=4, qubit_ceiling=64, check_norms=True):
        return OracleEngine(self, N, a, L, t, err or make_error(), shard_count, qubit_ceiling,
                            check_norms)


class SparseOracle:
    """so_sparse: the stage recipe on the support of the state (config-4 sizes)."""

    def __init__(self, o, N, a, L, t, err=None, check_norms=True):
        self.o, self.t, self.N = o, t, N
        h = C.c_void_p()
        _check(o.lib.so_sparse_create(N, a, L, t, C.byref(err or make_error()),
                                      1 if check_norms else 0, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.so_sparse_destroy(self.h)
            self.h = None

    def state_init(self):
        _check(self.o.lib.so_sparse_init(self.h))

    def stage_probs(self, s, prefix=0, combine_mode=0):
        p0, p1 = dbl(), dbl()
        _check(self.o.lib.so_sparse_stage_probs(self.h, s, prefix & (2**64 - 1), prefix >> 64,
                                                combine_mode, C.byref(p0), C.byref(p1)))
        return p0.value, p1.value

    def collapse(self, src_group, p_src):
        _check(self.o.lib.so_sparse_stage_collapse(self.h, src_group, p_src))

    def state(self, x):
        """(sorted support as uint64 array, g_x there as interleaved float64 array)"""
        import numpy as np
        n = self.o.lib.so_sparse_size(self.h)
        z = np.empty(n, dtype=np.uint64)
        v = np.empty(2 * n, dtype=np.float64)
        _check(self.o.lib.so_sparse_state(self.h, x, z.ctypes.data, v.ctypes.data))
        return z, v


class OracleEngine:
    def __init__(self, o, N, a, L, t, err, shard_count, qubit_ceiling, check_norms):
        self.o, self.t, self.N = o, t, N
        self.err = err
        h = C.c_void_p()
        _check(o.lib.so_engine_create(N, a, L, t, C.byref(err), shard_count, qubit_ceiling,
                                      1 if check_norms else 0, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.so_engine_destroy(self.h)
            self.h = None

    def multipliers(self):
        out = (u64 * self.t)()
        self.o.lib.so_engine_multipliers(self.h, out)
        return list(out)

    def run(self, seed, idx, combine_mode=0):
        tr = RunTrace(self.t)
        _check(self.o.lib.so_engine_run(self.h, seed, idx, combine_mode, tr.j, tr.js, tr.p1,
                                        tr.ints))
        return tr.as_dict()

    def state_init(self):
        _check(self.o.lib.so_state_init(self.h))

    def stage_probs(self, s, prefix=0, combine_mode=0):
        p0, p1 = dbl(), dbl()
        rc = self.o.lib.so_stage_probs(self.h, s, prefix & (2**64 - 1), prefix >> 64, combine_mode,
                                       C.byref(p0), C.byref(p1))
        _check(rc)
        return p0.value, p1.value

    def stage_read(self, x, first, count):
        out = (dbl * (2 * count))()
        _check(self.o.lib.so_stage_read(self.h, x, first, count, out))
        return out

    def collapse(self, src_group, p_src):
        _check(self.o.lib.so_stage_collapse(self.h, src_group, p_src))

    def state_read(self, x, first, count):
        out = (dbl * (2 * count))()
        _check(self.o.lib.so_state_read(self.h, x, first, count, out))
        return out

    def block_sums(self):
        nb = self.o.lib.so_num_blocks(self.h)
        out = (dbl * (2 * nb))()
        _check(self.o.lib.so_stage_block_sums(self.h, out))
        return out[:nb], out[nb:]


class Reference:
    """The unmodified reference library (oracle/_ref)."""

    def __init__(self, path: str | None = None):
        self.build = reference_build() if path is None else {"path": path, "variant": "explicit",
                                                              "flags": ""}
        path = self.build["path"]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = C.CDLL(path)
        self.lib = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_u64.restype = u64
        L.ref_rng_u64.argtypes = [u64, u32, u32, u32, u32]
        L.ref_recommended_t.restype = C.c_uint
        L.ref_recommended_t.argtypes = [u64]
        L.ref_bit_length.restype = C.c_uint
        L.ref_bit_length.argtypes = [u64]
        L.ref_mod_inverse.argtypes = [u64, u64, C.POINTER(u64)]
        L.ref_stage_phase.restype = dbl
        L.ref_stage_phase.argtypes = [C.c_uint, u64, u64]
        L.ref_permutation_plan.argtypes = [u64, u64, C.c_uint, C.c_uint, C.POINTER(u32),
                                           C.POINTER(u64), C.POINTER(u64), C.POINTER(C.c_int)]
        L.ref_engine_create.argtypes = [u64, u64, C.c_uint, C.c_uint, C.c_int, dbl, dbl, dbl, dbl,
                                        C.c_int, C.c_uint, C.c_uint, C.c_uint, C.c_int,
                                        C.POINTER(C.c_void_p)]
        L.ref_engine_destroy.argtypes = [C.c_void_p]
        L.ref_engine_multipliers.argtypes = [C.c_void_p, C.POINTER(u64)]
        L.ref_engine_run.argtypes = [C.c_void_p, u64, u64, C.POINTER(u64), C.POINTER(u64),
                                     C.POINTER(dbl), C.POINTER(i32)]
        L.ref_engine_time_runs.argtypes = [C.c_void_p, u64, u64, C.c_uint, C.POINTER(dbl),
                                           C.POINTER(u64)]
        L.ref_state_create.argtypes = [C.c_uint, C.c_int, dbl, C.c_uint, C.POINTER(C.c_void_p)]
        L.ref_state_destroy.argtypes = [C.c_void_p]
        L.ref_state_set_amp.argtypes = [C.c_void_p, u64, dbl, dbl]
        L.ref_apply_oracle.argtypes = [C.c_void_p, u64, u64]
        L.ref_apply_phase.argtypes = [C.c_void_p, C.c_uint, u64, u64]
        L.ref_apply_hadamard.argtypes = [C.c_void_p]
        L.ref_group_norm.restype = dbl
        L.ref_group_norm.argtypes = [C.c_void_p, C.c_int]
        L.ref_reset_top.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, dbl, dbl]
        L.ref_state_read.argtypes = [C.c_void_p, u64, u64, C.POINTER(dbl)]
        L.ref_sample_measurement.argtypes = [dbl, u64, u32, u32, C.c_int, dbl, dbl, dbl, dbl,
                                             C.c_int, C.POINTER(i32)]
        L.ref_exhaustive.argtypes = [u64, u64, C.c_uint, C.c_uint, C.c_int, dbl, dbl, dbl, dbl,
                                     C.c_int, C.POINTER(dbl)]
        L.ref_shor_standard_procedure.argtypes = [u64, u64, C.c_uint, u64, u64, u64, C.c_int,
                                                  C.POINTER(i32), C.POINTER(u64), C.POINTER(u64)]
        L.ref_multiplicative_order.argtypes = [u64, u64, u64, u64, C.POINTER(u64)]
        L.ref_factorize.argtypes = [u64, u64, C.POINTER(u64), C.POINTER(u32), C.POINTER(u32)]
        L.ref_ekera_postprocess.argtypes = [u64, u64, C.c_uint, u64, u64, u64, u64, C.c_uint,
                                            C.c_uint, C.c_uint, C.c_uint, u64, u32, u64, C.c_int,
                                            C.POINTER(i32), C.POINTER(u64), C.POINTER(u64)]
        L.ref_run_problem.argtypes = [u64, u64, u64, u64, C.c_uint, C.c_uint, u64, C.c_uint,
                                      C.c_int, dbl, dbl, dbl, dbl, C.c_int, C.c_uint,
                                      C.POINTER(u64), C.POINTER(u64), C.c_uint, C.c_int]

    def philox(self, key, ctr):
        out = (u32 * 4)()
        self.lib.ref_philox_block(u64(key), (u32 * 4)(*ctr), out)
        return list(out)

    def plan(self, a_pow, N, n, shards):
        y_limit = min(N, 1 << (n - 1))
        gs = shards // 2
        gather = (u32 * y_limit)()
        pc = (u64 * (gs * gs))()
        inv, ident = u64(), C.c_int()
        _check(self.lib.ref_permutation_plan(a_pow, N, n, shards, gather, pc, C.byref(inv),
                                             C.byref(ident)), self.lib)
        return {"gather": list(gather), "a_inv": inv.value, "identity": bool(ident.value),
                "pair_counts": [list(pc[s * gs:(s + 1) * gs]) for s in range(gs)]}

    def engine(self, N, a, L, t, err=None, shard_count=4, workers=1, qubit_ceiling=33,
               check_norms=True):
        return RefEngine(self, N, a, L, t, err or make_error(), shard_count, workers,
                         qubit_ceiling, check_norms)

    def sample(self, p1, seed, idx, stage, err):
        out = (i32 * 4)()
        _check(self.lib.ref_sample_measurement(p1, seed, idx, stage, err.kind, err.delta, err.px,
                                               err.py, err.pz, err.has_pauli, out), self.lib)
        return list(out)

    def exhaustive(self, N, a, L, t, err=None):
        err = err or make_error()
        out = (dbl * (1 << t))()
        _check(self.lib.ref_exhaustive(N, a, L, t, err.kind, err.delta, err.px, err.py, err.pz,
                                       err.has_pauli, out), self.lib)
        return list(out)

    def state(self, n, err=None, shards=4):
        return RefState(self, n, err or make_error(), shards)

    def shor_standard_procedure(self, j, t, N, a, known_order=None):
        """proj/src/postprocess.cpp:55-89, fields as shs_shor_outcome."""
        ints, kr, f = (i32 * 6)(), (u64 * 4)(), (u64 * 4)()
        _check(self.lib.ref_shor_standard_procedure(
            j & (2**64 - 1), j >> 64, t, N, a, known_order or 0, 0 if known_order is None else 1,
            ints, kr, f), self.lib)
        return {"classification": ints[0], "r_even": ints[1], "a_r_is_one": ints[2],
                "a_half_not_minus_one": ints[3], "order_match": ints[4],
                "k": kr[0] | (kr[1] << 64), "r": kr[2] | (kr[3] << 64),
                "factors": list(f[:ints[5]])}

    def ekera_postprocess(self, j, t, N, a, params, seed, idx, known_order=None):
        """proj/src/postprocess.cpp:138-171 with RngStream(seed, idx, 1, postprocess);
        params = (B, c, k, varsigma, m, ell)."""
        ints, us, f = (i32 * 5)(), (u64 * 6)(), (u64 * 4)()
        B, c, k, vs, m, ell = params
        _check(self.lib.ref_ekera_postprocess(j & (2**64 - 1), j >> 64, t, N, a, B, c, k, vs, m,
                                              ell, seed, idx, known_order or 0,
                                              0 if known_order is None else 1, ints, us, f),
               self.lib)
        off = us[5] - (1 << 64) if us[5] >= (1 << 63) else us[5]
        return {"classification": ints[0], "order_match": ints[1],
                "recovered_order": us[4] if ints[2] else None,
                "candidate_offset": off if ints[3] else None,
                "k": us[0] | (us[1] << 64), "r": us[2] | (us[3] << 64),
                "factors": list(f[:ints[4]])}

    def factorize(self, n, budget=10_000_000):
        """[(prime, exponent)]; OracleError code 9 on FactorizationTimeoutError"""
        pr, ex, cnt = (u64 * 64)(), (u32 * 64)(), u32()
        _check(self.lib.ref_factorize(n, budget, pr, ex, C.byref(cnt)), self.lib)
        return [(pr[i], ex[i]) for i in range(cnt.value)]

    def multiplicative_order(self, a, N, p=0, q=0):
        out = u64()
        _check(self.lib.ref_multiplicative_order(a, N, p, q, C.byref(out)), self.lib)
        return out.value

    def run_problem(self, N, a, p, q, L, t, seed, M, err=None, qubit_ceiling=26, post_mode="shor"):
        """run_problem (proj/src/harness.cpp:109-148) on the reference engine."""
        err = err or make_error()
        counts, cap = (u64 * 13)(), 256
        recip = (u64 * (2 * cap))()
        _check(self.lib.ref_run_problem(N, a, p, q, L, t, seed, M, err.kind, err.delta, err.px,
                                        err.py, err.pz, err.has_pauli, qubit_ceiling, counts,
                                        recip, cap, 1 if post_mode == "ekera" else 0), self.lib)
        keys = ["order", "success", "lucky_ne", "lucky_no", "lucky_oo", "fail",
                "first_factor_index", "first_order_index", "r_overflow", "r_other",
                "r_total_lucky", "order_solvable"]
        out = {k: counts[i] for i, k in enumerate(keys)}
        for k in ("first_factor_index", "first_order_index"):
            out[k] = out[k] or None
        out["order_solvable"] = bool(out["order_solvable"])
        out["r_reciprocal"] = {recip[2 * i]: recip[2 * i + 1] for i in range(min(counts[12], cap))}
        return out


class RefEngine:
    def __init__(self, r, N, a, L, t, err, shard_count, workers, qubit_ceiling, check_norms):
        self.r, self.t = r, t
        h = C.c_void_p()
        _check(r.lib.ref_engine_create(N, a, L, t, err.kind, err.delta, err.px, err.py, err.pz,
                                       err.has_pauli, shard_count, workers, qubit_ceiling,
                                       1 if check_norms else 0, C.byref(h)), r.lib)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_engine_destroy(self.h)
            self.h = None

    def multipliers(self):
        out = (u64 * self.t)()
        self.r.lib.ref_engine_multipliers(self.h, out)
        return list(out)

    def run(self, seed, idx):
        tr = RunTrace(self.t)
        _check(self.r.lib.ref_engine_run(self.h, seed, idx, tr.j, tr.js, tr.p1, tr.ints),
               self.r.lib)
        return tr.as_dict()

    def time_runs(self, seed, idx0, count):
        sec, j = dbl(), u64()
        _check(self.r.lib.ref_engine_time_runs(self.h, seed, idx0, count, C.byref(sec),
                                               C.byref(j)), self.r.lib)
        return sec.value


class RefState:
    def __init__(self, r, n, err, shards):
        self.r, self.n, self.err = r, n, err
        h = C.c_void_p()
        _check(r.lib.ref_state_create(n, err.kind, err.delta, shards, C.byref(h)), r.lib)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.r.lib.ref_state_destroy(self.h)
            self.h = None

    def oracle(self, a_pow, N):
        _check(self.r.lib.ref_apply_oracle(self.h, a_pow, N), self.r.lib)

    def phase(self, cbit, prefix):
        _check(self.r.lib.ref_apply_phase(self.h, cbit, prefix & (2**64 - 1), prefix >> 64),
               self.r.lib)

    def hadamard(self):
        _check(self.r.lib.ref_apply_hadamard(self.h), self.r.lib)

    def group_norm(self, x):
        return self.r.lib.ref_group_norm(self.h, x)

    def reset(self, bit, error_branch, p_source):
        _check(self.r.lib.ref_reset_top(self.h, bit, 1 if error_branch else 0, self.err.kind,
                                        self.err.delta, p_source), self.r.lib)

    def read_group(self, x, first, count):
        out = (dbl * (2 * count))()
        base = x << (self.n - 1)
        _check(self.r.lib.ref_state_read(self.h, base + first, count, out), self.r.lib)
        return list(out)

    def set_amp(self, g, re, im):
        _check(self.r.lib.ref_state_set_amp(self.h, g, re, im), self.r.lib)
