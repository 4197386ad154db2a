"""The parity oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of the BubbleSpec hot path
(draft lookup, Alg. 1 verification step, commit), in C (``bs_oracle.c``) driven
from plain Python loops.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  It
shares no code with the CUDA path (``paper_2605_08862_b200``) and never imports it.

Parity pins (tests/test_oracle_pins.py): every function below is checked against
what the paper and mathematics fix; none is marked "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bs_oracle.c")
_LIB = os.path.join(_HERE, "libbs_oracle.so")

OK, ERR_INVALID, ERR_DEVICE = 0, 1, 7
ACCEPT, SAMPLE = 0, 1


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, -ffp-contract=off).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-ffp-contract=off", "-fPIC", "-shared",
             "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


class _RowStats(C.Structure):
    _fields_ = [("z", C.c_uint64), ("z_full", C.c_uint64), ("m", C.c_float),
                ("greedy", C.c_int32), ("norm_fp64", C.c_double), ("norm_r", C.c_float)]


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        L.orc_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.orc_draw_r128.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, P(C.c_uint32)]
        L.orc_uniform_floor.argtypes = [P(C.c_uint32), C.c_uint64]
        L.orc_uniform_floor.restype = C.c_uint64
        L.orc_exp2_poly.argtypes = [C.c_float]
        L.orc_exp2_poly.restype = C.c_float
        L.orc_mass_shift.argtypes = [C.c_int]
        L.orc_mass_of_y.argtypes = [C.c_float, C.c_int]
        L.orc_mass_of_y.restype = C.c_uint64
        L.orc_temp_scale.argtypes = [C.c_float]
        L.orc_temp_scale.restype = C.c_float
        L.orc_top_p_filter.argtypes = [P(C.c_uint64), C.c_int, C.c_float]
        L.orc_top_p_filter.restype = C.c_uint64
        L.orc_row_dist.argtypes = [P(C.c_uint16), C.c_int, C.c_float, C.c_float, P(C.c_uint64),
                                   P(_RowStats)]
        L.orc_row_dist_k.argtypes = [P(C.c_uint16), C.c_int, C.c_float, C.c_float, C.c_int,
                                     P(C.c_uint64), P(_RowStats)]
        L.orc_top_k_filter.argtypes = [P(C.c_uint64), C.c_int, C.c_int]
        L.orc_top_k_filter.restype = C.c_uint64
        L.orc_verify_one_k.argtypes = [
            P(P(C.c_uint16)), C.c_int, C.c_float, C.c_float, C.c_int32, C.c_uint64, C.c_uint64,
            C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_int32), C.c_int32, C.c_int32,
            P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_float), P(C.c_double), P(C.c_uint64),
            P(C.c_int32)]
        L.orc_sample_index.argtypes = [P(C.c_uint64), C.c_int, C.c_int32, C.c_uint64]
        L.orc_sample_index.restype = C.c_int32
        L.orc_verify_one.argtypes = [
            P(P(C.c_uint16)), C.c_int, C.c_float, C.c_float, C.c_uint64, C.c_uint64, C.c_int32,
            C.c_int32, C.c_int32, C.c_int32, P(C.c_int32), C.c_int32, C.c_int32, P(C.c_int32),
            P(C.c_int32), P(C.c_int32), P(C.c_float), P(C.c_double), P(C.c_uint64), P(C.c_int32)]
        L.orc_verify_one_r.argtypes = [
            P(P(C.c_uint16)), C.c_int, C.c_float, C.c_float, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
            C.c_int32, P(C.c_int32), C.c_int32, C.c_int32, P(C.c_uint32), P(C.c_uint32),
            P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_float), P(C.c_double), P(C.c_uint64),
            P(C.c_int32)]
        L.orc_lookup.argtypes = [P(C.c_int32), P(C.c_int64), C.c_int32, P(C.c_int32), C.c_int32,
                                 C.c_int32, C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32),
                                 P(C.c_int32)]
        L.orc_lookup_conf.argtypes = [P(C.c_int32), P(C.c_int64), C.c_int32, P(C.c_int32), C.c_int32,
                                      C.c_int32, C.c_int32, C.c_int32, C.c_uint64, P(C.c_int32),
                                      P(C.c_int32), P(C.c_int32)]
        L.orc_lookup_ngram.argtypes = [P(C.c_int32), P(C.c_int64), C.c_int32, P(C.c_int32),
                                       C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_int32),
                                       P(C.c_int32), P(C.c_int32)]
        _lib = L
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


# ---------------------------------------------------------------- primitives
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c, C.c_uint32), _ptr(k, C.c_uint32), _ptr(o, C.c_uint32))
    return [int(v) for v in o]


def draw_r128(seed: int, uid: int, position: int, purpose: int):
    o = np.zeros(4, dtype=np.uint32)
    lib().orc_draw_r128(seed, uid, position, purpose, _ptr(o, C.c_uint32))
    return [int(v) for v in o]


def uniform_floor(r, Z: int) -> int:
    a = np.asarray(r, dtype=np.uint32)
    return int(lib().orc_uniform_floor(_ptr(a, C.c_uint32), Z))


def exp2_poly(f: float) -> float:
    return float(lib().orc_exp2_poly(f))


def mass_shift(V: int) -> int:
    return int(lib().orc_mass_shift(V))


def mass_of_y(y: float, S: int) -> int:
    return int(lib().orc_mass_of_y(y, S))


def temp_scale(T: float) -> float:
    return float(lib().orc_temp_scale(T))


def top_k_filter(masses, top_k: int):
    m = np.ascontiguousarray(masses, dtype=np.uint64).copy()
    z = lib().orc_top_k_filter(_ptr(m, C.c_uint64), len(m), top_k)
    return m, int(z)


def top_p_filter(masses, top_p: float):
    m = np.ascontiguousarray(masses, dtype=np.uint64).copy()
    z = lib().orc_top_p_filter(_ptr(m, C.c_uint64), len(m), top_p)
    return m, int(z)


@dataclass
class RowDist:
    mass: np.ndarray  # uint64 [V], kept masses mass'_i
    z: int            # Z' (after top-p)
    z_full: int
    m: float
    greedy: int
    norm_fp64: float
    norm_r: float


def row_dist(row_bits: np.ndarray, T: float, top_p: float = 1.0, top_k: int = 0) -> RowDist:
    row = np.ascontiguousarray(row_bits, dtype=np.uint16)
    mass = np.zeros(len(row), dtype=np.uint64)
    st = _RowStats()
    rc = lib().orc_row_dist_k(_ptr(row, C.c_uint16), len(row), T, top_p, top_k, _ptr(mass, C.c_uint64),
                              C.byref(st))
    if rc != OK:
        raise OracleError(rc)
    return RowDist(mass, int(st.z), int(st.z_full), float(st.m), int(st.greedy),
                   float(st.norm_fp64), float(st.norm_r))


def sample_index(masses, excl: int, U: int) -> int:
    m = np.ascontiguousarray(masses, dtype=np.uint64)
    return int(lib().orc_sample_index(_ptr(m, C.c_uint64), len(m), excl, U))


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


# ---------------------------------------------------------------- one step
@dataclass
class StepOut:
    tokens: list
    accepted: int
    rows_used: int
    norm_r: list
    norm_fp64: list
    z: list


def verify_one(rows, T: float, top_p: float, seed: int, uid: int, pos: int, max_len: int,
               eos: int, finished: bool, draft, k: int, top_k: int = 0) -> StepOut:
    """Alg. 1 step for one rollout.  rows: list of q+1 bf16 rows (uint16 arrays)."""
    V = len(rows[0])
    nr = len(rows)
    keep = [np.ascontiguousarray(r, dtype=np.uint16) for r in rows]
    arr = (C.POINTER(C.c_uint16) * nr)(*[_ptr(r, C.c_uint16) for r in keep])
    d = np.ascontiguousarray(np.asarray(list(draft) + [0], dtype=np.int32))
    out = np.zeros(k + 1, dtype=np.int32)
    ol, oa, ru = C.c_int32(), C.c_int32(), C.c_int32()
    nrm = np.zeros(k + 1, dtype=np.float32)
    n64 = np.zeros(k + 1, dtype=np.float64)
    zz = np.zeros(k + 1, dtype=np.uint64)
    rc = lib().orc_verify_one_k(arr, V, T, top_p, top_k, seed, uid, pos, max_len, eos, int(finished),
                              _ptr(d, C.c_int32), len(draft), k, _ptr(out, C.c_int32),
                              C.byref(ol), C.byref(oa), _ptr(nrm, C.c_float),
                              _ptr(n64, C.c_double), _ptr(zz, C.c_uint64), C.byref(ru))
    if rc != OK:
        raise OracleError(rc)
    n = ru.value
    return StepOut([int(x) for x in out[: ol.value]], oa.value, n, [float(x) for x in nrm[:n]],
                   [float(x) for x in n64[:n]], [int(x) for x in zz[:n]])


def _r128_words(r: int):
    return [(r >> 96) & 0xFFFFFFFF, (r >> 64) & 0xFFFFFFFF, (r >> 32) & 0xFFFFFFFF, r & 0xFFFFFFFF]


def verify_one_r(rows, T: float, top_p: float, pos: int, max_len: int, eos: int, draft, k: int,
                 r_acc, r_smp, top_k: int = 0) -> StepOut:
    """Alg. 1 step with caller-chosen uniforms: r_acc[j] / r_smp[j] are the 128-bit integers
    r128 of the accept test on row j and of a sample from row j (j = 0..k)."""
    V = len(rows[0])
    keep = [np.ascontiguousarray(r, dtype=np.uint16) for r in rows]
    arr = (C.POINTER(C.c_uint16) * len(keep))(*[_ptr(r, C.c_uint16) for r in keep])
    d = np.ascontiguousarray(np.asarray(list(draft) + [0], dtype=np.int32))
    ra = np.asarray([w for r in r_acc for w in _r128_words(int(r))], dtype=np.uint32)
    rs = np.asarray([w for r in r_smp for w in _r128_words(int(r))], dtype=np.uint32)
    out = np.zeros(k + 1, dtype=np.int32)
    ol, oa, ru = C.c_int32(), C.c_int32(), C.c_int32()
    rc = lib().orc_verify_one_r(arr, V, T, top_p, top_k, pos, max_len, eos, 0, _ptr(d, C.c_int32), len(draft), k,
                                _ptr(ra, C.c_uint32), _ptr(rs, C.c_uint32), _ptr(out, C.c_int32),
                                C.byref(ol), C.byref(oa), None, None, None, C.byref(ru))
    if rc != OK:
        raise OracleError(rc)
    return StepOut([int(x) for x in out[: ol.value]], oa.value, ru.value, [], [], [])


# ---------------------------------------------------------------- lookup
def tau_fixed(min_token_prob: float) -> int:
    """Reading C1: the confidence threshold as the integer round(tau * 2^32) in [0, 2^32]."""
    return min(1 << 32, max(0, int(round(float(min_token_prob) * 4294967296.0))))


def lookup(pool_seqs, ctx, M: int, Lmin: int, K: int, min_token_prob: float = 0.0):
    """Brute-force draft lookup over one prompt's pool (list of token sequences).
    min_token_prob > 0: confidence-scored drafts (reading C1).  Returns (draft list, m_star)."""
    lens = [len(s) for s in pool_seqs]
    off = np.zeros(len(pool_seqs) + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    toks = (np.concatenate([np.asarray(s, dtype=np.int32) for s in pool_seqs])
            if pool_seqs and off[-1] > 0 else np.zeros(1, dtype=np.int32))
    c = np.ascontiguousarray(np.asarray(list(ctx) if len(ctx) else [0], dtype=np.int32))
    draft = np.zeros(max(K, 1), dtype=np.int32)
    q, ms = C.c_int32(), C.c_int32()
    rc = lib().orc_lookup_conf(_ptr(toks, C.c_int32), _ptr(off, C.c_int64), len(pool_seqs),
                               _ptr(c, C.c_int32), len(ctx), M, Lmin, K, tau_fixed(min_token_prob),
                               _ptr(draft, C.c_int32), C.byref(q), C.byref(ms))
    if rc != OK:
        raise OracleError(rc)
    return [int(x) for x in draft[: q.value]], ms.value


def lookup_ngram(pool_seqs, ctx, n_min: int, n_max: int, K: int):
    """n-gram linear-scan drafter (reading N1) over one prompt's pool.  Returns (draft, n)."""
    lens = [len(s) for s in pool_seqs]
    off = np.zeros(len(pool_seqs) + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    toks = (np.concatenate([np.asarray(s, dtype=np.int32) for s in pool_seqs])
            if pool_seqs and off[-1] > 0 else np.zeros(1, dtype=np.int32))
    c = np.ascontiguousarray(np.asarray(list(ctx) if len(ctx) else [0], dtype=np.int32))
    draft = np.zeros(max(K, 1), dtype=np.int32)
    q, nn = C.c_int32(), C.c_int32()
    rc = lib().orc_lookup_ngram(_ptr(toks, C.c_int32), _ptr(off, C.c_int64), len(pool_seqs),
                                _ptr(c, C.c_int32), len(ctx), n_min, n_max, K, _ptr(draft, C.c_int32),
                                C.byref(q), C.byref(nn))
    if rc != OK:
        raise OracleError(rc)
    return [int(x) for x in draft[: q.value]], nn.value


from .rollout import OracleRollout, run_rollouts  # noqa: E402,F401
