"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (ctypes wrapper around oracle/liboracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import this module.  It never imports the CUDA package and the CUDA package never
imports it.  The arithmetic lives in oracle.c (plain int64 full-matrix DP, cited there
against PAPER.md Eqs. (1)-(5), and the relax listing P:284-308).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")

KINDS = {"global": 0, "local": 1, "semi": 2, "semiglobal": 2}
GAPS = {"linear": 0, "affine": 1}
OPS = "MID"


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no SIMD intrinsics, no shared headers)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, SRC,
                               "-lpthread"])
        os.replace(tmp, LIB)
    return LIB


class _Params(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("gap", ctypes.c_int32), ("match", ctypes.c_int32),
                ("mismatch", ctypes.c_int32), ("gap_open", ctypes.c_int32),
                ("gap_extend", ctypes.c_int32), ("has_subst", ctypes.c_int32),
                ("subst", ctypes.c_int32 * 25)]


class _Result(ctypes.Structure):
    _fields_ = [("score", ctypes.c_int64), ("q_begin", ctypes.c_int64),
                ("s_begin", ctypes.c_int64), ("q_end", ctypes.c_int64),
                ("s_end", ctypes.c_int64), ("n_ops", ctypes.c_int64)]


_RESULT_DTYPE = np.dtype([("score", np.int64), ("q_begin", np.int64), ("s_begin", np.int64),
                          ("q_end", np.int64), ("s_end", np.int64), ("n_ops", np.int64)])

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_align.restype = ctypes.c_int
        _lib.oracle_align.argtypes = [ctypes.POINTER(_Params), ctypes.c_char_p, ctypes.c_int64,
                                      ctypes.c_char_p, ctypes.c_int64, ctypes.c_int,
                                      ctypes.POINTER(_Result), ctypes.c_void_p, ctypes.c_int64]
        _lib.oracle_score_rolling.restype = ctypes.c_int
        _lib.oracle_score_rolling.argtypes = [ctypes.POINTER(_Params), ctypes.c_char_p,
                                              ctypes.c_int64, ctypes.c_char_p, ctypes.c_int64,
                                              ctypes.POINTER(_Result)]
        _lib.oracle_batch.restype = ctypes.c_int
        _lib.oracle_batch.argtypes = [ctypes.POINTER(_Params), ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                      ctypes.c_void_p]
    return _lib


@dataclass(frozen=True)
class Scheme:
    """Alignment kind + scoring: kind, gap model, sigma, gap magnitudes."""
    kind: str = "global"
    gap: str = "linear"
    match: int = 2
    mismatch: int = -1
    gap_open: int = 0
    gap_extend: int = 1
    matrix: tuple = None  # optional 5x5 sigma over codes A,C,G,T,N (matrix scoring)

    def c(self) -> _Params:
        p = _Params(KINDS[self.kind], GAPS[self.gap], self.match, self.mismatch,
                    self.gap_open, self.gap_extend)
        if self.matrix is not None:
            p.has_subst = 1
            for a in range(5):
                for b in range(5):
                    p.subst[5 * a + b] = int(self.matrix[a][b])
        return p


@dataclass
class Alignment:
    score: int
    q_begin: int
    s_begin: int
    q_end: int
    s_end: int
    cigar: list  # list of (length, op) with op in "MID"

    def cigar_str(self) -> str:
        return "".join(f"{l}{o}" for l, o in self.cigar)


def _b(x) -> bytes:
    return x.encode() if isinstance(x, str) else bytes(x)


def align(scheme: Scheme, q, s, traceback: bool = True) -> Alignment:
    q, s = _b(q), _b(s)
    r = _Result()
    cap = len(q) + len(s) + 1
    buf = (ctypes.c_uint32 * cap)()
    rc = lib().oracle_align(ctypes.byref(scheme.c()), q, len(q), s, len(s), int(traceback),
                            ctypes.byref(r), ctypes.cast(buf, ctypes.c_void_p), cap)
    if rc != 0:
        raise ValueError(f"oracle_align failed rc={rc}")
    cig = [(int(buf[k]) >> 4, OPS[int(buf[k]) & 15]) for k in range(r.n_ops)]
    return Alignment(r.score, r.q_begin, r.s_begin, r.q_end, r.s_end, cig)


def score_rolling(scheme: Scheme, q, s) -> Alignment:
    """Linear-space score-only variant (Fig. 1 right); end cell included."""
    q, s = _b(q), _b(s)
    r = _Result()
    rc = lib().oracle_score_rolling(ctypes.byref(scheme.c()), q, len(q), s, len(s),
                                    ctypes.byref(r))
    if rc != 0:
        raise ValueError(f"oracle_score_rolling failed rc={rc}")
    return Alignment(r.score, r.q_begin, r.s_begin, r.q_end, r.s_end, [])


def batch(scheme: Scheme, q: np.ndarray, q_off: np.ndarray, s: np.ndarray, s_off: np.ndarray,
          traceback: bool = False, threads: int | None = None):
    """Plain per-pair oracle, parallel across pairs only (pthreads).

    q, s: uint8 ASCII CSR buffers; q_off, s_off: uint64 offsets (num_pairs + 1).
    Returns (results structured array, cigar uint32 array or None).  For traceback,
    pair k's ops start at q_off[k] + s_off[k] + k and there are results['n_ops'][k].
    """
    q = np.ascontiguousarray(q, dtype=np.uint8)
    s = np.ascontiguousarray(s, dtype=np.uint8)
    q_off = np.ascontiguousarray(q_off, dtype=np.uint64)
    s_off = np.ascontiguousarray(s_off, dtype=np.uint64)
    B = len(q_off) - 1
    res = np.zeros(B, dtype=_RESULT_DTYPE)
    cig = np.zeros(int(q_off[-1] + s_off[-1]) + B + 1, dtype=np.uint32) if traceback else None
    th = threads or os.cpu_count() or 1
    rc = lib().oracle_batch(ctypes.byref(scheme.c()), q.ctypes.data, q_off.ctypes.data,
                            s.ctypes.data, s_off.ctypes.data, B, th, int(traceback),
                            res.ctypes.data, cig.ctypes.data if cig is not None else None)
    if rc != 0:
        raise ValueError(f"oracle_batch failed rc={rc}")
    return res, cig


def batch_cigars(res, cig, q_off, s_off):
    """Decode the per-pair RLE words written by batch(traceback=True)."""
    out = []
    for k in range(len(res)):
        base = int(q_off[k] + s_off[k]) + k
        words = cig[base: base + int(res["n_ops"][k])]
        out.append([(int(w) >> 4, OPS[int(w) & 15]) for w in words])
    return out
