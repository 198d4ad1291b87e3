"""Trace files ("miso-trace v1"), so GPU runs consume the traces the reference CLI writes.

Restates save_trace / load_trace (workload.hpp:122-245) with format_profile_body /
parse_profile_body (profiles.hpp:484-568) and validate_profile (profiles.hpp:67-87): the same
three header lines, 13 CSV fields per job, doubles as %.17g (fmt_exact, common.hpp:134-139)
and the same ParseError cases with 1-based line numbers. Host text I/O around the device path;
the C++ binding uses the reference's own reader.
"""
from __future__ import annotations

import ctypes
import io
from dataclasses import dataclass
from typing import List, Optional, Sequence, TextIO, Union

import numpy as np

from .sim import Trace

MAGIC = "miso-trace v1"
HEADER = ("job_id,arrival_s,base_duration_s,mem_demand_gb,qos_min_gpc,"
          "f7,f4,f3,f2,f1,mps100,mps50,mps14")
GPC = (1, 2, 3, 4, 7)
KIND_NAMES = ("1g", "2g", "3g", "4g", "7g")
SPEED_FLOOR = 1e-9  # profiles.hpp:33
DISTS = ("lognormal", "fixed", "uniform")


class ParseError(ValueError):
    """ParseError (common.hpp:30-39): message prefixed with 'line N: ' when N > 0."""

    def __init__(self, msg: str, line: int):
        super().__init__(f"line {line}: {msg}" if line > 0 else msg)
        self.line = line


@dataclass
class TraceSpec:
    """TraceSpec (workload.hpp:20-35)."""
    job_count: int = 100
    lambda_s: float = 60.0
    max_duration_s: float = 7200.0
    dist: str = "lognormal"
    sigma: float = 1.5
    fixed_s: float = 600.0
    lo_s: float = 60.0
    hi_s: float = 7200.0
    seed: int = 0

    def validate(self):
        """validate_trace_spec (workload.hpp:37-46)."""
        if self.job_count < 1:
            raise ValueError("job_count must be >= 1")
        if not self.lambda_s > 0:
            raise ValueError("lambda_s must be positive")
        if not self.max_duration_s > 0:
            raise ValueError("max_duration_s must be positive")
        if self.dist == "lognormal" and not self.sigma > 0:
            raise ValueError("lognormal sigma must be positive")
        if self.dist == "uniform" and not (self.lo_s > 0 and self.lo_s <= self.hi_s):
            raise ValueError("uniform bounds must satisfy 0 < lo_s <= hi_s")


@dataclass
class TraceFile:
    """A loaded trace: the simulator's Trace plus what the file also carries."""
    trace: Trace
    spec: TraceSpec
    job_ids: List[str]
    mps_rates: np.ndarray  # (n, 3): rates at MPS levels 100/50/14


def fmt_exact(v: float) -> str:
    """fmt_exact (common.hpp:134-139): printf("%.17g")."""
    return "%.17g" % v


def interp_speed(t: Sequence[float], gpc: float) -> float:
    """interp_speed (profiles.hpp:391-402), same operation order."""
    knots = (1.0, 2.0, 3.0, 4.0, 7.0)
    if gpc <= knots[0]:
        return t[0]
    if gpc >= knots[-1]:
        return t[-1]
    for i in range(1, 5):
        if gpc <= knots[i]:
            w = (gpc - knots[i - 1]) / (knots[i] - knots[i - 1])
            return t[i - 1] + w * (t[i] - t[i - 1])
    return t[-1]


def synthetic_mps_rates(speeds5: np.ndarray) -> np.ndarray:
    """make_synthetic_profile's placeholder solo-run rates (profiles.hpp:460-463)."""
    sp = np.asarray(speeds5, np.float64).reshape(-1, 5)
    out = np.empty((len(sp), 3))
    for i, row in enumerate(sp):
        out[i, 0] = 1.0
        out[i, 1] = min(max(interp_speed(row, 3.5), SPEED_FLOOR), 1.0)  # std::clamp
        out[i, 2] = row[0]
    return out


def _validate_profile(job_id, duration, mem, speeds, mps, line, instance_count=1):
    """validate_profile (profiles.hpp:67-87): ParseError when line > 0, else ValueError (the
    reference's std::invalid_argument)."""
    def fail(msg):
        if line > 0:
            raise ParseError(f"job '{job_id}': {msg}", line)
        raise ValueError(f"job '{job_id}': {msg}")
    if not job_id:
        fail("empty job id")
    if "," in job_id:
        fail("job id contains a comma")
    if not duration > 0:
        fail("base duration must be positive")
    if mem <= 0 or mem > 40:
        fail("memory demand must be in (0, 40] GB")
    for k in range(5):
        if not (speeds[k] > 0.0 and speeds[k] <= 1.0):
            fail(f"speed on {KIND_NAMES[k]} outside (0,1]")
    if speeds[4] != 1.0:
        fail("speed on 7g must be exactly 1")
    for k in range(1, 5):
        if speeds[k] < speeds[k - 1]:
            fail("speed table not monotone in gpc count")
    for r in mps:
        if not (r > 0.0 and r <= 1.0):
            fail("mps rate outside (0,1]")
    if instance_count < 1:
        fail("instance count must be >= 1")


_libc = ctypes.CDLL(None, use_errno=True)
_libc.strtod.restype = ctypes.c_double
_libc.strtod.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
_libc.strtol.restype = ctypes.c_long
_libc.strtol.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int]
_ERANGE = 34


def _c_convert(fn, tok: str, *base):
    """(value, characters consumed, ERANGE?) of libc strtod/strtol -- what std::stod/stoi call
    (hex floats, nan(...), leading whitespace and underflow/overflow as the reference sees them)."""
    raw = tok.encode()
    if b"\0" in raw:
        raw = raw[:raw.index(b"\0")]  # std::stod sees the C string
    buf = ctypes.create_string_buffer(raw)
    end = ctypes.c_char_p()
    ctypes.set_errno(0)
    v = fn(buf, ctypes.byref(end), *base)
    err = ctypes.get_errno()
    used = ctypes.cast(end, ctypes.c_void_p).value - ctypes.addressof(buf)
    return v, len(raw[:used].decode(errors="replace")), err == _ERANGE


def _parse_double(tok: str, what: str, line: int) -> float:
    """detail::parse_double (profiles.hpp:512-522): std::stod with the whole token consumed."""
    v, used, erange = _c_convert(_libc.strtod, tok)
    if used == 0 or erange or used != len(tok):
        raise ParseError(f"bad {what} '{tok}'", line)
    return v


def _parse_int(tok: str, what: str, line: int) -> int:
    """detail::parse_int (profiles.hpp:524-534): std::stoi (strtol, then the int range)."""
    v, used, erange = _c_convert(_libc.strtol, tok, 10)
    if used == 0 or erange or not (-2**31 <= v < 2**31) or used != len(tok):
        raise ParseError(f"bad {what} '{tok}'", line)
    return v


@dataclass
class ProfileRecord:
    """JobProfile (profiles.hpp:47-56) as a profile record carries it."""
    job_id: str
    base_duration_s: float
    mem_demand_gb: int
    qos_kind: int               # -1 = none, else kind index 0..4 (1g..7g)
    speeds5: np.ndarray         # kind order 1g..7g
    mps_rates: np.ndarray       # rates at MPS levels 100/50/14


def split_csv(line: str) -> List[str]:
    """detail::split_csv (profiles.hpp:497-510): split on ',', drop every '\\r'."""
    return [t.replace("\r", "") for t in line.split(",")]


def format_profile_body(p: ProfileRecord) -> str:
    """format_profile_body (profiles.hpp:484-491): base, mem, qos gpc (0 = none), f7..f1,
    mps100/50/14."""
    qg = GPC[int(p.qos_kind)] if p.qos_kind is not None and int(p.qos_kind) >= 0 else 0
    sp = np.asarray(p.speeds5, np.float64).reshape(5)
    out = [fmt_exact(float(p.base_duration_s)), str(int(p.mem_demand_gb)), str(qg)]
    out += [fmt_exact(float(sp[k])) for k in range(4, -1, -1)]
    out += [fmt_exact(float(r)) for r in np.asarray(p.mps_rates, np.float64).reshape(3)]
    return ",".join(out)


def format_profile_record(p: ProfileRecord) -> str:
    """format_profile_record (profiles.hpp:493-495)."""
    return p.job_id + "," + format_profile_body(p)


def parse_profile_body(job_id: str, tokens: Sequence[str], offset: int,
                       line: int) -> ProfileRecord:
    """parse_profile_body (profiles.hpp:539-562): the 11 fields after tokens[offset - 1],
    checked in the reference's order, then validate_profile."""
    if len(tokens) != offset + 11:
        raise ParseError(f"expected {offset + 11} fields, got {len(tokens)}", line)
    i = offset
    d = _parse_double(tokens[i], "duration", line)
    m = _parse_int(tokens[i + 1], "memory demand", line)
    qg = _parse_int(tokens[i + 2], "qos gpc", line)
    qk = -1
    if qg != 0:
        if qg not in GPC:
            raise ParseError(f"qos gpc {qg} is not a slice size", line)
        qk = GPC.index(qg)
    s5 = [0.0] * 5
    for j, k in enumerate(range(4, -1, -1)):
        s5[k] = _parse_double(tokens[i + 3 + j], "speed", line)
    r3 = [_parse_double(tokens[i + 8 + r], "mps rate", line) for r in range(3)]
    _validate_profile(job_id, d, m, s5, r3, line)
    return ProfileRecord(job_id, d, m, qk, np.asarray(s5), np.asarray(r3))


def parse_profile_record(line_text: str, line: int = 0) -> ProfileRecord:
    """parse_profile_record (profiles.hpp:564-568)."""
    tok = split_csv(line_text)
    if not tok or not tok[0]:
        raise ParseError("missing job id", line)
    return parse_profile_body(tok[0], tok, 1, line)


def save_trace(trace: Trace, spec: TraceSpec, out: Union[str, TextIO],
               job_ids: Optional[Sequence[str]] = None,
               mps_rates: Optional[np.ndarray] = None) -> None:
    """save_trace (workload.hpp:149-170). job_ids default to "j<i>" and mps_rates to the
    synthetic profile's (what generate_trace produces)."""
    n = trace.n
    ids = list(job_ids) if job_ids is not None else [f"j{i}" for i in range(n)]
    mps = synthetic_mps_rates(trace.speeds5) if mps_rates is None else np.asarray(mps_rates)
    qos = trace.qos_kind
    lines = [MAGIC,
             f"spec job_count={spec.job_count} lambda_s={fmt_exact(spec.lambda_s)} "
             f"max_duration_s={fmt_exact(spec.max_duration_s)} dist={spec.dist} "
             f"sigma={fmt_exact(spec.sigma)} fixed_s={fmt_exact(spec.fixed_s)} "
             f"lo_s={fmt_exact(spec.lo_s)} hi_s={fmt_exact(spec.hi_s)} seed={spec.seed}",
             HEADER]
    sp = np.asarray(trace.speeds5, np.float64).reshape(-1, 5)
    for i in range(n):
        qg = GPC[int(qos[i])] if qos is not None and int(qos[i]) >= 0 else 0
        body = [fmt_exact(float(trace.duration_s[i])), str(int(trace.mem_gb[i])), str(qg)]
        body += [fmt_exact(float(sp[i, k])) for k in range(4, -1, -1)]
        body += [fmt_exact(float(mps[i, r])) for r in range(3)]
        lines.append(",".join([ids[i], fmt_exact(float(trace.arrival_s[i]))] + body))
    text = "\n".join(lines) + "\n"
    if isinstance(out, str):
        with open(out, "w", newline="") as f:
            f.write(text)
    else:
        out.write(text)


def load_trace(src: Union[str, TextIO]) -> TraceFile:
    """load_trace (workload.hpp:172-243) from a path or an open text file."""
    if isinstance(src, str):
        try:
            with open(src, newline="") as f:
                text = f.read()
        except OSError:
            raise OSError(f"cannot open trace file: {src}") from None
        return loads(text)
    return loads(src.read())


def loads(text: str) -> TraceFile:
    """load_trace of a file's text: every check and message of the reference reader."""
    raw = text.split("\n")
    if raw and raw[-1] == "":
        raw.pop()
    lines = [ln[:-1] if ln.endswith("\r") else ln for ln in raw]
    if not lines or lines[0] != MAGIC:
        raise ParseError(f"expected '{MAGIC}'", 1)
    if len(lines) < 2 or not lines[1].startswith("spec "):
        raise ParseError("expected spec line", 2)
    spec = TraceSpec()
    ln = 2
    for kv in lines[1][5:].split():
        if "=" not in kv:
            raise ParseError(f"bad spec token '{kv}'", ln)
        key, val = kv.split("=", 1)
        if key == "job_count":
            spec.job_count = _parse_int(val, "job_count", ln)
        elif key in ("lambda_s", "max_duration_s", "sigma", "fixed_s", "lo_s", "hi_s"):
            setattr(spec, key, _parse_double(val, key, ln))
        elif key == "dist":
            if val not in DISTS:
                raise ParseError(f"unknown duration distribution '{val}'", ln)
            spec.dist = val
        elif key == "seed":
            spec.seed = int(val)
        else:
            raise ParseError(f"unknown spec key '{key}'", ln)
    try:
        spec.validate()
    except ValueError as e:
        raise ParseError(str(e), ln) from None
    if len(lines) < 3:
        raise ParseError("expected column header", ln + 1)
    ln = 3
    if lines[2] != HEADER:
        raise ParseError("expected column header", ln)
    ids, arr, dur, mem, qos, sp, mps = [], [], [], [], [], [], []
    seen = set()
    prev = 0.0
    for idx in range(3, len(lines)):
        ln = idx + 1
        line = lines[idx]
        if not line:
            continue
        tok = split_csv(line)
        if len(tok) != 13:
            raise ParseError(f"expected 13 fields, got {len(tok)}", ln)
        a = _parse_double(tok[1], "arrival", ln)
        pr = parse_profile_body(tok[0], tok, 2, ln)
        d, m, qk, s5, r3 = pr.base_duration_s, pr.mem_demand_gb, pr.qos_kind, pr.speeds5, pr.mps_rates
        if tok[0] in seen:
            raise ParseError(f"duplicate job id '{tok[0]}'", ln)
        seen.add(tok[0])
        if not ids:
            if a != 0:
                raise ParseError("first arrival must be at t=0", ln)
        elif a < prev:
            raise ParseError("arrival time regresses", ln)
        if d > spec.max_duration_s:
            raise ParseError("duration exceeds max_duration_s cap", ln)
        prev = a
        ids.append(tok[0]); arr.append(a); dur.append(d); mem.append(m); qos.append(qk)
        sp.append(list(s5)); mps.append(list(r3))
    if len(ids) != spec.job_count:
        raise ParseError(f"spec says {spec.job_count} jobs, file has {len(ids)}", ln)
    q = np.asarray(qos, np.int8)
    tr = Trace(np.asarray(arr), np.asarray(dur), np.asarray(sp).reshape(-1, 5),
               np.asarray(mem, np.int32), q if (q >= 0).any() else None, spec.seed)
    return TraceFile(tr, spec, ids, np.asarray(mps).reshape(-1, 3))


def dumps(trace: Trace, spec: TraceSpec, **kw) -> str:
    buf = io.StringIO()
    save_trace(trace, spec, buf, **kw)
    return buf.getvalue()
