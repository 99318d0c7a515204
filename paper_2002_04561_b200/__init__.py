"""paper_2002_04561_b200 -- B200-native pairwise DNA alignment (AnySeq's DP relaxation hot path).

Thin Python binding over the C-ABI in include/anyseq.h (ctypes; argument marshalling only).
Every step of the path -- packing, planning, relaxation, optimum, traceback -- runs in the
CUDA kernels of libanyseq.so (paper_2002_04561_b200/csrc, sm_100a).  There is no CPU
fallback: importing this module raises if the library is missing, and creating a
Context raises if no CUDA device is present.

PyTorch (optional) is only used for device memory and streams in the *_device calls.
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ANYSEQ_LIB: another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("ANYSEQ_LIB") or os.path.join(HERE, "lib", "libanyseq.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "anyseq.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

KINDS = {"global": 0, "local": 1, "semi": 2, "semiglobal": 2}
GAPS = {"linear": 0, "affine": 1}
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_BADSEQ", 3: "E_NOMEM", 4: "E_CAPACITY", 5: "E_CUDA",
          6: "E_UNSUPPORTED", 7: "E_PEER", 8: "E_TIMEOUT"}
OPS = "MID"


class _Params(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("gap", ctypes.c_int32), ("match", ctypes.c_int32),
                ("mismatch", ctypes.c_int32), ("gap_open", ctypes.c_int32),
                ("gap_extend", ctypes.c_int32), ("has_subst", ctypes.c_int32),
                ("subst", ctypes.c_int32 * 25)]


class _Batch(ctypes.Structure):
    _fields_ = [("q", ctypes.c_void_p), ("q_off", ctypes.c_void_p), ("s", ctypes.c_void_p),
                ("s_off", ctypes.c_void_p), ("num_pairs", ctypes.c_uint64)]


ALIGNMENT_DTYPE = np.dtype([("score", np.int32), ("reserved", np.int32), ("q_begin", np.int64),
                            ("s_begin", np.int64), ("q_end", np.int64), ("s_end", np.int64),
                            ("cigar_offset", np.uint64), ("cigar_len", np.uint32),
                            ("reserved2", np.uint32)])
assert ALIGNMENT_DTYPE.itemsize == 56

_vp, _u64, _i64, _i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32
_sig = {
    "anyseq_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), _vp, ctypes.c_int]),
    "anyseq_destroy": (None, [_vp]),
    "anyseq_align_batch": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "anyseq_align_batch_device": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "anyseq_traceback": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _u64, _vp]),
    "anyseq_align_long": (ctypes.c_int, [_vp, _vp, ctypes.c_char_p, _u64, ctypes.c_char_p, _u64, _vp]),
    "anyseq_traceback_long": (ctypes.c_int, [_vp, _vp, ctypes.c_char_p, _u64, ctypes.c_char_p, _u64,
                                             _vp, _vp, _u64, _vp]),
    "anyseq_sync": (ctypes.c_int, [_vp]),
    "anyseq_kernel_launches": (ctypes.c_uint64, [_vp]),
    "anyseq_set_option": (ctypes.c_int, [_vp, ctypes.c_char_p, _i64]),
    "anyseq_get_stat": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double)]),
    "anyseq_reset_stats": (ctypes.c_int, [_vp]),
    "anyseq_status_str": (ctypes.c_char_p, [ctypes.c_int]),
    "anyseq_last_error": (ctypes.c_char_p, [_vp]),
    "anyseq_version": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def header_functions() -> list[str]:
    """Names of the functions declared in include/anyseq.h."""
    with open(HEADER) as f:
        txt = f.read()
    return sorted(set(re.findall(r"\b(anyseq_[a-z_0-9]+)\s*\(", txt)))


class AnyseqError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.status_name = STATUS.get(status, str(status))


@dataclass(frozen=True)
class Scheme:
    """Alignment kind and scoring: penalties are non-negative magnitudes."""
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


def version() -> str:
    return _lib.anyseq_version().decode()


def _u8(x) -> np.ndarray:
    if isinstance(x, (bytes, bytearray)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    return np.ascontiguousarray(x, dtype=np.uint8)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def decode_cigar(words) -> list:
    return [(int(w) >> 4, OPS[int(w) & 15]) for w in words]


class Context:
    """An anyseq context on one or more CUDA devices (all device work is in libanyseq.so)."""

    def __init__(self, devices=(0,)):
        h = ctypes.c_void_p()
        ids = (ctypes.c_int * len(devices))(*devices)
        st = _lib.anyseq_create(ctypes.byref(h), ids, len(devices))
        if st != 0:
            raise AnyseqError(st, "anyseq_create failed (no CUDA device?)")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _lib.anyseq_destroy(self._h)
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

    def _check(self, st: int):
        if st != 0:
            raise AnyseqError(st, _lib.anyseq_last_error(self._h).decode())

    @property
    def launches(self) -> int:
        return int(_lib.anyseq_kernel_launches(self._h))

    def set_option(self, name: str, value: int):
        self._check(_lib.anyseq_set_option(self._h, name.encode(), int(value)))

    @staticmethod
    def _batch(q, q_off, s, s_off):
        q, s = _u8(q), _u8(s)
        q_off = np.ascontiguousarray(q_off, dtype=np.uint64)
        s_off = np.ascontiguousarray(s_off, dtype=np.uint64)
        assert len(q_off) == len(s_off) and len(q_off) >= 1
        b = _Batch(_ptr(q), q_off.ctypes.data, _ptr(s), s_off.ctypes.data, len(q_off) - 1)
        return b, (q, s, q_off, s_off)

    def align_batch(self, scheme: Scheme, q, q_off, s, s_off, ends: bool = False, out=None):
        """Score-only batch (host buffers).  Returns scores, or (scores, alignments) if ends.
        `out`: optional preallocated int32 array of B scores (pinned memory avoids staging)."""
        b, keep = self._batch(q, q_off, s, s_off)
        B = int(b.num_pairs)
        if out is not None:
            if not (isinstance(out, np.ndarray) and out.dtype == np.int32 and out.shape == (B,)
                    and out.flags.c_contiguous):
                raise ValueError("out must be a contiguous int32 array of num_pairs scores")
            scores = out
        else:
            scores = np.empty(B, dtype=np.int32)
        aln = np.zeros(B, dtype=ALIGNMENT_DTYPE) if ends else None
        p = scheme.c()
        self._check(_lib.anyseq_align_batch(self._h, ctypes.byref(p), ctypes.byref(b),
                                            _ptr(scores), _ptr(aln) if ends else None))
        return (scores, aln) if ends else scores

    def traceback(self, scheme: Scheme, q, q_off, s, s_off, cigar_capacity: int | None = None,
                  out_aln=None, out_cigar=None):
        """Full alignments.  Returns (alignments structured array, cigar uint32 words).
        `out_aln` / `out_cigar`: optional preallocated outputs (ALIGNMENT_DTYPE[B] and uint32
        words; pinned memory avoids staging); out_cigar's length is the capacity."""
        b, keep = self._batch(q, q_off, s, s_off)
        B = int(b.num_pairs)
        q_off, s_off = keep[2], keep[3]
        if out_aln is not None:
            if not (isinstance(out_aln, np.ndarray) and out_aln.dtype == ALIGNMENT_DTYPE
                    and out_aln.shape == (B,) and out_aln.flags.c_contiguous):
                raise ValueError("out_aln must be a contiguous ALIGNMENT_DTYPE array of B entries")
            aln = out_aln
        else:
            aln = np.empty(B, dtype=ALIGNMENT_DTYPE)
        if out_cigar is not None:
            if not (isinstance(out_cigar, np.ndarray) and out_cigar.dtype == np.uint32
                    and out_cigar.ndim == 1 and out_cigar.flags.c_contiguous):
                raise ValueError("out_cigar must be a contiguous uint32 array")
            cig = out_cigar
            cap = len(cig) if cigar_capacity is None else min(cigar_capacity, len(cig))
        else:
            cap = int(q_off[-1] - q_off[0] + s_off[-1] - s_off[0]) if cigar_capacity is None \
                else cigar_capacity
            cig = np.empty(max(cap, 1), dtype=np.uint32)
        used = ctypes.c_uint64(0)
        p = scheme.c()
        st = _lib.anyseq_traceback(self._h, ctypes.byref(p), ctypes.byref(b), _ptr(aln),
                                   cig.ctypes.data, cap, ctypes.byref(used))
        if st != 0:
            err = AnyseqError(st, _lib.anyseq_last_error(self._h).decode())
            err.cigar_used = int(used.value)
            raise err
        return aln, cig[: used.value]

    def align_long(self, scheme: Scheme, q, s) -> dict:
        q = bytes(q) if not isinstance(q, bytes) else q
        s = bytes(s) if not isinstance(s, bytes) else s
        out = np.zeros(1, dtype=ALIGNMENT_DTYPE)
        p = scheme.c()
        self._check(_lib.anyseq_align_long(self._h, ctypes.byref(p), q, len(q), s, len(s),
                                           out.ctypes.data))
        r = out[0]
        return {"score": int(r["score"]), "q_end": int(r["q_end"]), "s_end": int(r["s_end"])}

    def traceback_long(self, scheme: Scheme, q, s, cigar_capacity: int | None = None) -> dict:
        """Linear-space long-pair traceback (anyseq_traceback_long): score, begin/end cells
        and the CIGAR as (length, op) tuples."""
        q = bytes(q) if not isinstance(q, bytes) else q
        s = bytes(s) if not isinstance(s, bytes) else s
        out = np.zeros(1, dtype=ALIGNMENT_DTYPE)
        cap = len(q) + len(s) + 1 if cigar_capacity is None else cigar_capacity
        cig = np.empty(max(cap, 1), dtype=np.uint32)
        used = ctypes.c_uint64(0)
        p = scheme.c()
        st = _lib.anyseq_traceback_long(self._h, ctypes.byref(p), q, len(q), s, len(s),
                                        out.ctypes.data, cig.ctypes.data, cap, ctypes.byref(used))
        if st != 0:
            err = AnyseqError(st, _lib.anyseq_last_error(self._h).decode())
            err.cigar_used = int(used.value)
            raise err
        r = out[0]
        return {"score": int(r["score"]), "q_begin": int(r["q_begin"]), "s_begin": int(r["s_begin"]),
                "q_end": int(r["q_end"]), "s_end": int(r["s_end"]),
                "cigar": decode_cigar(cig[: used.value])}

    def align_batch_device(self, scheme: Scheme, d_q, d_q_off, d_s, d_s_off, d_scores,
                           d_ends=None, stream=None):
        """Device-resident batch: arguments are torch CUDA tensors (uint8 sequences, int64
        offsets reinterpreted as uint64, int32 scores, optional uint8 [B*56] ends)."""
        B = d_q_off.numel() - 1
        b = _Batch(d_q.data_ptr() if d_q.numel() else None, d_q_off.data_ptr(),
                   d_s.data_ptr() if d_s.numel() else None, d_s_off.data_ptr(), B)
        p = scheme.c()
        st_ptr = stream.cuda_stream if stream is not None else None
        self._check(_lib.anyseq_align_batch_device(
            self._h, ctypes.byref(p), ctypes.byref(b), d_scores.data_ptr(),
            d_ends.data_ptr() if d_ends is not None else None, st_ptr))

    def stat(self, name: str) -> float:
        v = ctypes.c_double(0)
        self._check(_lib.anyseq_get_stat(self._h, name.encode(), ctypes.byref(v)))
        return float(v.value)

    def reset_stats(self):
        self._check(_lib.anyseq_reset_stats(self._h))

    def sync(self):
        self._check(_lib.anyseq_sync(self._h))


def cigars_of(aln: np.ndarray, cig: np.ndarray) -> list:
    """Per-pair decoded CIGARs [(len, op), ...] from traceback() output."""
    out = []
    for r in aln:
        o, n = int(r["cigar_offset"]), int(r["cigar_len"])
        out.append(decode_cigar(cig[o:o + n]))
    return out
