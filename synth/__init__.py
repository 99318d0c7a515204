"""synth -- seeded synthetic DNA workloads shared by the oracle side and the CUDA side.

This module holds NO alignment arithmetic: it only draws bases.  Both tests/ (oracle
parity) and bench.py use it so that the two sides see identical inputs.  Recipes follow
SURVEY.md 8(d) ("Synthetic inputs") and are restated in DESIGN.md ("Input recipe"):

* C1  one pair, i.i.d. 1000 x 1000 bp, seed 1.
* C2  10 Mbp i.i.d. reference R; per pair pos ~ U, s = R[pos+d : pos+d+150] with
      d ~ U{-8..8}; q = R[pos:] mutated (substitutions rising linearly 0.2 % -> 1.0 % 5'->3',
      insertions 0.05 %, deletions 0.05 %, geometric length with mean 1.5) then truncated
      or extended from R to exactly 150 bp.  (The paper's Mason settings are not given,
      P:872.)
* C4  G1 = 5 Mbp i.i.d.; G2 = (a) mutated copy (1 % subs, 0.1 % indels, mean length 3),
      (b) independent i.i.d., (c) G2 = G1.
* C5  L ~ U{100..1000}; s = R window of length L; q = mutated copy of length L + U{-5..5}.

All draws use numpy's PCG64 with explicit seeds; 50 % GC, i.i.d. bases unless stated.
Sequences are returned as ASCII uint8 CSR buffers (data, offsets[num+1]).
"""
from __future__ import annotations

import numpy as np

ALPHA = np.frombuffer(b"ACGT", dtype=np.uint8)


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def iid_codes(rng, n: int) -> np.ndarray:
    return rng.integers(0, 4, size=n, dtype=np.uint8)


def iid(n: int, seed: int) -> bytes:
    return ALPHA[iid_codes(_rng(seed), n)].tobytes()


def csr(seqs) -> tuple[np.ndarray, np.ndarray]:
    """list of bytes -> (uint8 data, uint64 offsets)."""
    lens = np.fromiter((len(x) for x in seqs), dtype=np.uint64, count=len(seqs))
    off = np.zeros(len(seqs) + 1, dtype=np.uint64)
    np.cumsum(lens, out=off[1:])
    data = np.frombuffer(b"".join(seqs), dtype=np.uint8).copy() if len(seqs) else \
        np.zeros(0, np.uint8)
    return data, off


def uniform_csr(mat: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(B, L) uint8 matrix -> CSR with equal lengths."""
    B, L = mat.shape
    off = np.arange(B + 1, dtype=np.uint64) * np.uint64(L)
    return np.ascontiguousarray(mat).reshape(-1), off


def random_pairs(num: int, min_len: int, max_len: int, seed: int, alphabet: bytes = b"ACGT",
                 lower_frac: float = 0.0):
    """Independent random pairs with lengths ~ U{min_len..max_len} (test workloads)."""
    rng = _rng(seed)
    alpha = np.frombuffer(alphabet, dtype=np.uint8)
    out = []
    for _ in range(2):
        lens = rng.integers(min_len, max_len + 1, size=num)
        seqs = []
        for L in lens:
            x = alpha[rng.integers(0, len(alpha), size=int(L))]
            if lower_frac > 0:
                low = rng.random(int(L)) < lower_frac
                x = np.where(low & (x >= 65) & (x <= 90), x + 32, x).astype(np.uint8)
            seqs.append(x.tobytes())
        out.append(csr(seqs))
    (q, qo), (s, so) = out
    return q, qo, s, so


def _mutate(rng, src: np.ndarray, sub_rate, ins_rate: float, del_rate: float,
            mean_indel: float) -> np.ndarray:
    """Mutate a code array: per-position substitution rate (scalar or array), then
    geometric-length insertions/deletions (Illumina-/genome-like profile)."""
    x = src.copy()
    L = len(x)
    sub = rng.random(L) < sub_rate
    x[sub] = (x[sub] + rng.integers(1, 4, size=int(sub.sum()), dtype=np.uint8)) % 4
    p_geo = 1.0 / mean_indel
    ev_ins = np.flatnonzero(rng.random(L) < ins_rate)
    ev_del = np.flatnonzero(rng.random(L) < del_rate)
    if len(ev_ins) == 0 and len(ev_del) == 0:
        return x
    keep = np.ones(L, dtype=bool)
    for p in ev_del:
        k = int(rng.geometric(p_geo))
        keep[p:p + k] = False
    pieces = []
    last = 0
    for p in sorted(ev_ins):
        pieces.append(x[last:p][keep[last:p]])
        pieces.append(iid_codes(rng, int(rng.geometric(p_geo))))
        last = p
    pieces.append(x[last:][keep[last:]])
    return np.concatenate(pieces)


def _apply_indels(rng, x: np.ndarray, events: np.ndarray, mean_len: float) -> np.ndarray:
    """Each event position becomes an insertion or a deletion (coin flip) of geometric
    length with the given mean."""
    p_geo = 1.0 / mean_len
    keep = np.ones(len(x), dtype=bool)
    ins = []
    for p in events:
        k = int(rng.geometric(p_geo))
        if rng.random() < 0.5:
            keep[p:p + k] = False
        else:
            ins.append((int(p), iid_codes(rng, k)))
    pieces, last = [], 0
    for p, seg in ins:
        pieces.append(x[last:p][keep[last:p]])
        pieces.append(seg)
        last = p
    pieces.append(x[last:][keep[last:]])
    return np.concatenate(pieces)


def c1_pair(seed: int = 1) -> tuple[bytes, bytes]:
    """C1: one i.i.d. 1000 x 1000 bp pair."""
    rng = _rng(seed)
    return ALPHA[iid_codes(rng, 1000)].tobytes(), ALPHA[iid_codes(rng, 1000)].tobytes()


def c2_reads(num_pairs: int, seed: int = 2, read_len: int = 150, ref_len: int = 10_000_000):
    """C2/C3: Illumina-like read pairs (q = read, s = reference window), exactly read_len.

    Returns (q_mat, s_mat) uint8 ASCII matrices of shape (num_pairs, read_len)."""
    rng = _rng(seed)
    ref = iid_codes(rng, ref_len)
    margin = 64
    pos = rng.integers(margin, ref_len - read_len - 2 * margin, size=num_pairs)
    delta = rng.integers(-8, 9, size=num_pairs)
    cols = np.arange(read_len)
    s = ref[(pos + delta)[:, None] + cols[None, :]]
    span = read_len + margin
    src = ref[pos[:, None] + np.arange(span)[None, :]]
    # substitutions rising linearly 0.2 % -> 1.0 % along the read (5' -> 3')
    rate = 0.002 + 0.008 * (np.arange(span) / (read_len - 1))
    sub = rng.random((num_pairs, span)) < rate[None, :]
    shift = rng.integers(1, 4, size=(num_pairs, span), dtype=np.uint8)
    src = np.where(sub, (src + shift) % 4, src).astype(np.uint8)
    q = src[:, :read_len].copy()
    # indels (0.05 % each per base, geometric length mean 1.5) on the affected reads only
    ev = rng.random((num_pairs, read_len)) < 0.001
    rows = np.flatnonzero(ev.any(axis=1))
    for r in rows:
        y = _apply_indels(rng, src[r], np.flatnonzero(ev[r]), 1.5)
        if len(y) < read_len:  # extend from the reference
            p = int(pos[r]) + span
            y = np.concatenate([y, ref[p:p + read_len - len(y)]])
        q[r] = y[:read_len]
    return ALPHA[q], ALPHA[s]


def c4_genomes(n: int = 5_000_000, variant: str = "a", seed: int = 4) -> tuple[bytes, bytes]:
    """C4: two genome-sized sequences.  variant a = mutated copy, b = independent, c = same."""
    rng = _rng(seed)
    g1 = iid_codes(rng, n)
    if variant == "c":
        g2 = g1
    elif variant == "b":
        g2 = iid_codes(rng, n)
    elif variant == "a":
        g2 = _mutate(rng, g1, 0.01, 0.0005, 0.0005, 3.0)
    else:
        raise ValueError(variant)
    return ALPHA[g1].tobytes(), ALPHA[g2].tobytes()


def c5_mixed(num_pairs: int, seed: int = 5, lo: int = 100, hi: int = 1000,
             ref_len: int = 10_000_000):
    """C5: mixed-length pairs; s = reference window of length L ~ U{lo..hi}, q = mutated copy
    of length L + U{-5..5}.  Returns CSR (q, q_off, s, s_off)."""
    rng = _rng(seed)
    ref = iid_codes(rng, ref_len)
    L = rng.integers(lo, hi + 1, size=num_pairs)
    dl = rng.integers(-5, 6, size=num_pairs)
    pos = rng.integers(0, ref_len - hi - 64, size=num_pairs)
    qs, ss = [], []
    for k in range(num_pairs):
        p, l = int(pos[k]), int(L[k])
        ss.append(ALPHA[ref[p:p + l]].tobytes())
        y = _mutate(rng, ref[p:p + l + 32], 0.01, 0.0005, 0.0005, 1.5)
        ql = max(1, l + int(dl[k]))
        if len(y) < ql:
            y = np.concatenate([y, iid_codes(rng, ql - len(y))])
        qs.append(ALPHA[y[:ql]].tobytes())
    q, qo = csr(qs)
    s, so = csr(ss)
    return q, qo, s, so


def _ragged_gather(src: np.ndarray, starts: np.ndarray, lens: np.ndarray) -> np.ndarray:
    """Concatenation of src[starts[k] : starts[k] + lens[k]] over k (vectorised)."""
    lens = lens.astype(np.int32)
    tot = int(lens.sum())
    it = np.int32 if tot + len(src) < 2**31 else np.int64
    base = np.repeat((starts.astype(it) - (np.cumsum(lens, dtype=it) - lens)), lens)
    base += np.arange(tot, dtype=it)
    return src[base]


def c5_mixed_large(num_pairs: int, seed: int = 5, lo: int = 100, hi: int = 1000,
                   ref_len: int = 10_000_000, chunk: int = 50_000):
    """C5 at scale (vectorised; same recipe as c5_mixed, its own draw order): L ~ U{lo..hi};
    s = R window of length L; q = copy of R[pos : pos + L + 32] with 1 % substitutions, then
    indel events at 0.1 % of positions (insertion or deletion by coin flip, geometric length
    with mean 1.5, deletions clipped at the copy's end), cut or extended with i.i.d. bases to
    length L + U{-5..5} (at least 1).  Returns CSR (q, q_off, s, s_off)."""
    rng = _rng(seed)
    ref = iid_codes(rng, ref_len)
    qs, ss, qlens, slens = [], [], [], []
    for k0 in range(0, num_pairs, chunk):
        B = min(chunk, num_pairs - k0)
        L = rng.integers(lo, hi + 1, size=B)
        dl = rng.integers(-5, 6, size=B)
        pos = rng.integers(0, ref_len - hi - 64, size=B)
        ss.append(ALPHA[_ragged_gather(ref, pos, L)])
        slens.append(L)
        span = L + 32
        src = _ragged_gather(ref, pos, span)
        N = len(src)
        sub = rng.random(N) < 0.01
        src[sub] = (src[sub] + rng.integers(1, 4, size=int(sub.sum()), dtype=np.uint8)) % 4
        pair_end = np.repeat(np.cumsum(span), span)  # exclusive end of each element's pair
        ev = np.flatnonzero(rng.random(N) < 0.001)
        glen = rng.geometric(1.0 / 1.5, size=len(ev))
        is_del = rng.random(len(ev)) < 0.5
        keep = np.ones(N, dtype=np.int32)
        d0, dg = ev[is_del], glen[is_del]
        if len(d0):
            di = np.repeat(d0, dg) + (np.arange(int(dg.sum())) -
                                      np.repeat(np.cumsum(dg) - dg, dg))
            di = di[di < np.repeat(pair_end[d0], dg)]
            keep[di] = 0
        ins = np.zeros(N, dtype=np.int32)
        np.add.at(ins, ev[~is_del], glen[~is_del])
        cnt = ins + keep  # output symbols per source element: inserted bases, then the element
        tot = int(cnt.sum())
        grp = np.repeat(np.arange(N, dtype=np.int32), cnt)
        r = np.arange(tot, dtype=np.int32) - np.repeat(np.cumsum(cnt, dtype=np.int32) - cnt, cnt)
        y = np.where(r < ins[grp], iid_codes(rng, tot), src[grp]).astype(np.uint8)
        newlen = np.add.reduceat(cnt, np.concatenate([[0], np.cumsum(span)[:-1]]))
        ql = np.maximum(1, L + dl)
        take = np.minimum(newlen, ql)
        ystart = np.concatenate([[0], np.cumsum(newlen)[:-1]])
        qstart = np.concatenate([[0], np.cumsum(ql)[:-1]])
        out = iid_codes(rng, int(ql.sum()))  # the extension bases where a copy is too short
        out[_ragged_gather(np.arange(len(out), dtype=np.int32), qstart, take)] = \
            _ragged_gather(y, ystart, take)
        qs.append(ALPHA[out])
        qlens.append(ql)
    q = np.concatenate(qs)
    s = np.concatenate(ss)
    qo = np.zeros(num_pairs + 1, dtype=np.uint64)
    so = np.zeros(num_pairs + 1, dtype=np.uint64)
    np.cumsum(np.concatenate(qlens), out=qo[1:])
    np.cumsum(np.concatenate(slens), out=so[1:])
    return q, qo, s, so
