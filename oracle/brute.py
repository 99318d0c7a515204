"""oracle/brute.py -- TEST INFRASTRUCTURE ONLY: brute-force enumeration of alignments.

Independent of the DP: it enumerates every alignment path (every sequence of M/I/D
operations) between every admissible begin and end cell and scores each path by the
paper's definition of an alignment score -- the sum of sigma over aligned pairs
(simple_subst_scoring P:408-415) minus G_o + k*G_e per maximal gap run of length
k (linear: k*g, Eqs. (2)-(3)).  The admissible begin/end cells per kind are the
problem statements of P:259 (local: any substring pair, empty allowed), P:262 (global:
(0,0) -> (n,m)) and P:264 (semi-global: free leading/trailing gaps on both sequences;
begin on row 0 or column 0, end on row n or column m -- reading L5 in DESIGN.md).

Pure Python, exponential; only for lengths <= ~7.
"""
from __future__ import annotations

from functools import lru_cache

OPS = "MID"


def sigma(match: int, mismatch: int, a: str, b: str, matrix=None) -> int:
    a, b = a.upper(), b.upper()
    if matrix is not None:  # matrix scoring over A,C,G,T,N
        return int(matrix["ACGTN".index(a)]["ACGTN".index(b)])
    return match if (a == b and a in "ACGT") else mismatch


def rescore(scheme, q_sub: str, s_sub: str, ops: str) -> int:
    """Score of one alignment given as an op string over q_sub x s_sub."""
    go = scheme.gap_open if scheme.gap == "affine" else 0
    ge = scheme.gap_extend
    sc = 0
    i = j = 0
    prev = None
    for op in ops:
        if op == "M":
            sc += sigma(scheme.match, scheme.mismatch, q_sub[i], s_sub[j],
                        getattr(scheme, "matrix", None))
            i += 1
            j += 1
        elif op == "I":          # q_i against a gap (vertical, consumes q only)
            sc -= ge + (go if prev != "I" else 0)
            i += 1
        elif op == "D":          # s_j against a gap (horizontal, consumes s only)
            sc -= ge + (go if prev != "D" else 0)
            j += 1
        else:
            raise ValueError(op)
        prev = op
    assert i == len(q_sub) and j == len(s_sub)
    return sc


def rescore_cigar(scheme, q: str, s: str, qb: int, sb: int, cigar) -> int:
    ops = "".join(o * l for l, o in cigar)
    nq = sum(l for l, o in cigar if o in "MI")
    ns = sum(l for l, o in cigar if o in "MD")
    return rescore(scheme, q[qb:qb + nq], s[sb:sb + ns], ops)


@lru_cache(maxsize=None)
def paths(di: int, dj: int) -> tuple:
    """All op strings that consume exactly di query and dj subject symbols."""
    if di == 0 and dj == 0:
        return ("",)
    out = []
    if di > 0 and dj > 0:
        out += ["M" + p for p in paths(di - 1, dj - 1)]
    if di > 0:
        out += ["I" + p for p in paths(di - 1, dj)]
    if dj > 0:
        out += ["D" + p for p in paths(di, dj - 1)]
    return tuple(out)


def rle(ops: str):
    out = []
    for op in ops:
        if out and out[-1][1] == op:
            out[-1] = (out[-1][0] + 1, op)
        else:
            out.append((1, op))
    return tuple(out)


def _starts(kind: str, n: int, m: int):
    if kind == "global":
        return [(0, 0)]
    if kind in ("semi", "semiglobal"):
        return sorted({(i, 0) for i in range(n + 1)} | {(0, j) for j in range(m + 1)})
    if kind == "local":
        return [(i, j) for i in range(n + 1) for j in range(m + 1)]
    raise ValueError(kind)


def _is_end(kind: str, n: int, m: int, i: int, j: int) -> bool:
    if kind == "global":
        return i == n and j == m
    if kind in ("semi", "semiglobal"):
        return i == n or j == m
    return True  # local: any cell


def brute(scheme, q: str, s: str):
    """Return (best score, set of optimal (q_begin, s_begin, q_end, s_end, rle_cigar)).

    Depth-first enumeration of every op string from every admissible begin cell; every
    prefix that stops on an admissible end cell is a candidate alignment.  The running
    score is the same sum as rescore(): sigma per M, G_o + G_e for the first op of a gap
    run and G_e for each further op of the run."""
    n, m = len(q), len(s)
    go = scheme.gap_open if scheme.gap == "affine" else 0
    ge = scheme.gap_extend
    best = None
    opt = set()
    for (i0, j0) in _starts(scheme.kind, n, m):
        stack = [(i0, j0, "", 0)]
        while stack:
            i, j, ops, sc = stack.pop()
            if _is_end(scheme.kind, n, m, i, j):
                if best is None or sc > best:
                    best, opt = sc, set()
                if sc == best:
                    opt.add((i0, j0, i, j, rle(ops)))
            last = ops[-1] if ops else None
            if i < n and j < m:
                stack.append((i + 1, j + 1, ops + "M",
                              sc + sigma(scheme.match, scheme.mismatch, q[i], s[j],
                                    getattr(scheme, "matrix", None))))
            if i < n:
                stack.append((i + 1, j, ops + "I", sc - ge - (go if last != "I" else 0)))
            if j < m:
                stack.append((i, j + 1, ops + "D", sc - ge - (go if last != "D" else 0)))
    return best, opt
