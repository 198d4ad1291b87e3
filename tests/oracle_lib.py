"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/libmiso_oracle.so (the C restatement); `Ref` wraps
oracle/_ref/libmiso_ref.so (the unmodified reference headers behind a C shim). Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "libmiso_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libmiso_ref.so"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_i16p = np.ctypeslib.ndpointer(dtype=np.int16, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(dtype=np.int8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class OrcCatalog(C.Structure):
    _fields_ = [("n_entries", C.c_int), ("counts", (C.c_uint8 * 5) * 36)]


class OrcCandidates(C.Structure):
    _fields_ = [
        ("n", C.c_int),
        ("base", C.c_int * 9),
        ("entry", C.c_uint8 * 111),
        ("m", C.c_uint8 * 111),
        ("place", (C.c_uint8 * 7) * 111),
    ]


class RefSimOut(C.Structure):
    _fields_ = [
        ("completed", C.c_int), ("job_count", C.c_int), ("completed_count", C.c_int),
        ("repartitions", C.c_int), ("migrations", C.c_int), ("mps_sessions", C.c_int),
        ("avg_jct_s", C.c_double), ("makespan_s", C.c_double), ("stp_time_avg", C.c_double),
        ("queue_frac", C.c_double), ("mps_frac", C.c_double), ("checkpoint_frac", C.c_double),
        ("run_frac", C.c_double), ("idle_frac", C.c_double), ("stp_points", C.c_int64),
    ]


class Oracle:
    """The C restatement (oracle/miso_oracle.c)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(str(path))
        L.orc_build_catalog.argtypes = [C.POINTER(OrcCatalog)]
        L.orc_build_candidates.argtypes = [C.POINTER(OrcCandidates)]
        L.orc_optimize_batch.argtypes = [C.POINTER(OrcCatalog), _dp, _u32p, C.c_size_t, _i16p, _u8p, _dp]
        L.orc_gen_mixes.argtypes = [C.c_uint64, C.c_size_t, _dp, _u32p, C.c_size_t]
        L.orc_gen_mixes.restype = C.c_size_t
        L.orc_gen_profiles.argtypes = [C.c_uint64, C.c_size_t, _dp, C.c_void_p]
        L.orc_predict_batch.argtypes = [_dp, C.c_size_t, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                        C.c_double, _dp, _dp, _dp]
        L.orc_default_model.argtypes = [_dp, _dp]
        L.orc_perturb_speed.argtypes = [C.c_double, C.c_double, C.c_uint64]
        L.orc_perturb_speed.restype = C.c_double
        L.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_max_spare_slice_for.argtypes = [C.POINTER(OrcCatalog), _i32p, C.c_int]
        L.orc_build_spare_lut.argtypes = [C.POINTER(OrcCatalog), _i8p]
        L.orc_spare_key.argtypes = [_i32p, C.c_int]
        self.catalog = OrcCatalog()
        L.orc_build_catalog(C.byref(self.catalog))

    def catalog_counts(self) -> np.ndarray:
        n = self.catalog.n_entries
        return np.array([[self.catalog.counts[e][k] for k in range(5)] for e in range(n)], np.uint8)

    def candidates(self) -> OrcCandidates:
        c = OrcCandidates()
        self.lib.orc_build_candidates(C.byref(c))
        return c

    def gen_mixes(self, seed: int, n: int):
        cap = 7 * n
        speeds = np.zeros(cap * 5, np.float64)
        offs = np.zeros(n + 1, np.uint32)
        jobs = self.lib.orc_gen_mixes(seed, n, speeds, offs, cap)
        return speeds[: jobs * 5].copy(), offs

    def optimize_batch(self, speeds, offsets):
        n = len(offsets) - 1
        entry = np.zeros(n, np.int16)
        place = np.zeros(max(1, int(offsets[-1])), np.uint8)
        obj = np.zeros(n, np.float64)
        self.lib.orc_optimize_batch(C.byref(self.catalog), np.ascontiguousarray(speeds),
                                    np.ascontiguousarray(offsets), n, entry, place, obj)
        return entry, place, obj

    def gen_profiles(self, seed: int, n: int):
        t = np.zeros(3 * n, np.float64)
        s = np.zeros(2 * n, np.float64)
        self.lib.orc_gen_profiles(seed, n, t, s.ctypes.data)
        return t, s

    def default_model(self):
        w2 = np.zeros(4); w1 = np.zeros(4)
        self.lib.orc_default_model(w2, w1)
        return w2, w1

    def predict_batch(self, truth3, cpg, first_nonce, rng_seed, noisy, mae, w2=None, w1=None):
        if w2 is None:
            w2, w1 = self.default_model()
        n = len(truth3) // 3
        out = np.zeros(5 * n)
        self.lib.orc_predict_batch(np.ascontiguousarray(truth3), n, cpg, first_nonce, rng_seed,
                                   int(noisy), mae, w2, w1, out)
        return out

    def spare_lut(self) -> np.ndarray:
        lut = np.zeros(462, np.int8)
        self.lib.orc_build_spare_lut(C.byref(self.catalog), lut)
        return lut

    def max_spare(self, kinds) -> int:
        k = np.array(kinds, np.int32)
        return self.lib.orc_max_spare_slice_for(C.byref(self.catalog), k, len(kinds))


class Ref:
    """The unmodified reference (oracle/_ref/libmiso_ref.so)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(str(path))
        L.ref_catalog.argtypes = [_u8p]
        L.ref_optimize_batch.argtypes = [_dp, _u32p, C.c_size_t, C.c_int, _i16p, _u8p, _dp]
        L.ref_gen_mixes.argtypes = [C.c_uint64, C.c_size_t, _dp, _u32p, C.c_size_t]
        L.ref_gen_mixes.restype = C.c_size_t
        L.ref_gen_profiles.argtypes = [C.c_uint64, C.c_size_t, _dp, C.c_void_p]
        L.ref_default_model.argtypes = [_dp, _dp]
        L.ref_predict_batch.argtypes = [_dp, C.c_size_t, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                        C.c_double, C.c_int, _dp]
        L.ref_perturb_speed.argtypes = [C.c_double, C.c_double, C.c_uint64]
        L.ref_perturb_speed.restype = C.c_double
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_max_spare_slice_for.argtypes = [_i32p, C.c_int]
        L.ref_gen_trace.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_double,
                                    _dp, _dp, _dp, _i32p]
        L.ref_simulate.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                   C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                   C.c_double, C.c_int, C.POINTER(RefSimOut), C.c_char_p, C.c_int64]
        L.ref_simulate.restype = C.c_int64
        _ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
        L.ref_simulate_trace.argtypes = [C.c_int, _dp, _dp, _dp, _ip, _ip, C.c_uint64, C.c_int,
                                         C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_int, C.c_double, C.c_uint64, C.c_int,
                                         C.POINTER(RefSimOut), C.c_char_p, C.c_int64, C.c_void_p,
                                         C.c_int64]
        L.ref_trial.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_double, _dp]
        L.ref_best_static.argtypes = [C.c_int, _dp, _dp, _dp, _ip, C.c_int, C.c_double, C.c_double,
                                      C.c_double, C.c_double, _dp]
        L.ref_simulate_trace.restype = C.c_int64
        L.ref_rng_raw.argtypes = [C.c_uint64, C.c_size_t, np.ctypeslib.ndpointer(np.uint64)]
        L.ref_c1_chain.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                   _dp, _i32p, _dp, C.POINTER(C.c_int), _u8p,
                                   C.POINTER(C.c_double)]

    def rng_raw(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, np.uint64)
        self.lib.ref_rng_raw(seed, n, out)
        return out

    def trace_text(self, seed: int, job_count: int, lambda_s: float) -> str:
        """save_trace text of the reference's generate_trace (ref_trace_text)."""
        f = self.lib.ref_trace_text
        f.restype = C.c_size_t
        f.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_char_p, C.c_size_t]
        n = f(seed, job_count, lambda_s, None, 0)
        buf = C.create_string_buffer(n + 1)
        f(seed, job_count, lambda_s, buf, n)
        return buf.raw[:n].decode()

    def load_trace(self, text: str):
        """The reference's load_trace on `text`: (0, job_count, "") or (line, 0, what())."""
        f = self.lib.ref_load_trace
        f.restype = C.c_int
        f.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_char_p, C.c_size_t]
        jc = C.c_int(0)
        msg = C.create_string_buffer(512)
        r = f(text.encode(), C.byref(jc), msg, 512)
        return r, jc.value, msg.value.decode()

    def profile_record(self, line: str, lineno: int = 0):
        """The reference's parse_profile_record -> format_profile_record on `line`:
        (0, record text) or (ParseError line / -1 when 0 / -2 invalid_argument, what())."""
        f = self.lib.ref_profile_record
        f.restype = C.c_int
        f.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_size_t]
        out = C.create_string_buffer(1024)
        r = f(line.encode(), lineno, out, 1024)
        return r, out.value.decode()

    def c1_time(self, reps: int, seed=7, job_count=3, interference=0.8, target_mae=0.017):
        """Seconds for `reps` config-1 decisions on this thread (ref_c1_time) and the sum of
        their objectives (nonce 1..reps)."""
        cs = C.c_double()
        f = self.lib.ref_c1_time
        f.restype = C.c_double
        f.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double)]
        return f(seed, job_count, interference, target_mae, reps, C.byref(cs)), cs.value

    def c1_chain(self, seed=7, job_count=3, interference=0.8, target_mae=0.017, nonce=1):
        t = np.zeros(3 * job_count); mem = np.zeros(job_count, np.int32)
        est = np.zeros(5 * job_count); e = C.c_int(); pl = np.zeros(7, np.uint8); ob = C.c_double()
        ok = self.lib.ref_c1_chain(seed, job_count, interference, target_mae, nonce, t, mem, est,
                                   C.byref(e), pl, C.byref(ob))
        return dict(ok=ok, truth3=t, mem=mem, est5=est, entry=e.value, place=pl[:job_count].copy(),
                    obj=ob.value)

    def catalog_counts(self) -> np.ndarray:
        c = np.zeros(36 * 5, np.uint8)
        n = self.lib.ref_catalog(c)
        return c.reshape(36, 5)[:n].copy()

    def gen_mixes(self, seed: int, n: int):
        cap = 7 * n
        speeds = np.zeros(cap * 5, np.float64)
        offs = np.zeros(n + 1, np.uint32)
        jobs = self.lib.ref_gen_mixes(seed, n, speeds, offs, cap)
        return speeds[: jobs * 5].copy(), offs

    def optimize_batch(self, speeds, offsets, threads: int = 1):
        n = len(offsets) - 1
        entry = np.zeros(n, np.int16)
        place = np.zeros(max(1, int(offsets[-1])), np.uint8)
        obj = np.zeros(n, np.float64)
        self.lib.ref_optimize_batch(np.ascontiguousarray(speeds), np.ascontiguousarray(offsets), n,
                                    threads, entry, place, obj)
        return entry, place, obj

    def gen_profiles(self, seed: int, n: int):
        t = np.zeros(3 * n, np.float64)
        s = np.zeros(2 * n, np.float64)
        self.lib.ref_gen_profiles(seed, n, t, s.ctypes.data)
        return t, s

    def default_model(self):
        w2 = np.zeros(4); w1 = np.zeros(4)
        self.lib.ref_default_model(w2, w1)
        return w2, w1

    def predict_batch(self, truth3, cpg, first_nonce, rng_seed, noisy, mae, threads: int = 1):
        n = len(truth3) // 3
        out = np.zeros(5 * n)
        self.lib.ref_predict_batch(np.ascontiguousarray(truth3), n, cpg, first_nonce, rng_seed,
                                   int(noisy), mae, threads, out)
        return out

    def simulate_trace(self, arrival_s, duration_s, speeds5, mem_gb, qos_kind=None, seed=0,
                       cluster_size=8, policy=3, mig_reconfig_s=4.0, checkpoint_restart_s=30.0,
                       mps_window_s=10.0, interference=0.8, noisy=True, target_mae=0.017,
                       rng_seed=0, want_log=False, log_cap=1 << 26, stp_cap=0, static_entry=-1):
        n = len(arrival_s)
        qos = np.full(n, -1, np.int32) if qos_kind is None else np.asarray(qos_kind, np.int32)
        out = RefSimOut()
        buf = C.create_string_buffer(log_cap) if want_log else None
        stp = np.zeros(2 * stp_cap) if stp_cap else None
        r = self.lib.ref_simulate_trace(
            n, np.ascontiguousarray(arrival_s, np.float64), np.ascontiguousarray(duration_s, np.float64),
            np.ascontiguousarray(speeds5, np.float64).reshape(-1), np.ascontiguousarray(mem_gb, np.int32),
            qos, seed, cluster_size, policy, mig_reconfig_s, checkpoint_restart_s, mps_window_s,
            interference, int(noisy), target_mae, rng_seed, static_entry, C.byref(out), buf,
            log_cap if want_log else 0, None if stp is None else stp.ctypes.data, stp_cap)
        log = buf.raw[: min(r, log_cap)].decode() if (want_log and r >= 0) else None
        return out, log, stp

    def trial(self, seed, job_count=1000, lambda_s=10.0, cluster_size=100, target_mae=0.017):
        out = np.zeros(3)
        e = self.lib.ref_trial(seed, job_count, lambda_s, cluster_size, target_mae, out)
        return e, out

    def best_static(self, arrival_s, duration_s, speeds5, mem_gb, cluster_size=8,
                    mig_reconfig_s=4.0, checkpoint_restart_s=30.0, mps_window_s=10.0,
                    interference=0.8):
        table = np.zeros(36)
        e = self.lib.ref_best_static(len(arrival_s), np.ascontiguousarray(arrival_s, np.float64),
                                     np.ascontiguousarray(duration_s, np.float64),
                                     np.ascontiguousarray(speeds5, np.float64).reshape(-1),
                                     np.ascontiguousarray(mem_gb, np.int32), cluster_size,
                                     mig_reconfig_s, checkpoint_restart_s, mps_window_s,
                                     interference, table)
        return e, table

    def gen_trace(self, seed, job_count, lambda_s=60.0, max_duration_s=7200.0, sigma=1.5):
        arr = np.zeros(job_count); dur = np.zeros(job_count)
        sp = np.zeros(5 * job_count); mem = np.zeros(job_count, np.int32)
        self.lib.ref_gen_trace(seed, job_count, lambda_s, max_duration_s, sigma, arr, dur, sp, mem)
        return arr, dur, sp, mem

    def simulate(self, seed, job_count, lambda_s=60.0, cluster_size=8, policy=3,
                 mig_reconfig_s=4.0, checkpoint_restart_s=30.0, mps_window_s=10.0,
                 interference=0.8, noisy=True, target_mae=0.017, static_entry=-1,
                 max_duration_s=7200.0, sigma=1.5, want_log=False, log_cap=1 << 26):
        out = RefSimOut()
        buf = C.create_string_buffer(log_cap) if want_log else None
        n = self.lib.ref_simulate(seed, job_count, lambda_s, max_duration_s, sigma, cluster_size,
                                  policy, mig_reconfig_s, checkpoint_restart_s, mps_window_s,
                                  interference, int(noisy), target_mae, static_entry,
                                  C.byref(out), buf, log_cap if want_log else 0)
        log = buf.raw[: min(n, log_cap)].decode() if want_log else None
        return out, log


def have_ref() -> bool:
    return REF_SO.exists()


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class PyDetRng:
    """DetRng draws (common.hpp:85-119) over a precomputed raw mt19937_64 stream."""

    def __init__(self, raw: np.ndarray):
        self.raw = [int(x) for x in raw]
        self.i = 0

    def next(self) -> int:
        v = self.raw[self.i]
        self.i += 1
        return v

    def uniform01(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform01()

    def index(self, n: int) -> int:
        return self.next() % n
