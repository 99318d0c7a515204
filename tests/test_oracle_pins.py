"""Pins for the CPU oracle (not gpu).

The oracle (oracle/oracle.c) is checked against things other than itself:
  * worked examples in tests/golden/*.tsv (SPEC.md examples derived from the paper and the
    tie-rule conventions of DESIGN.md), every row also re-derived by brute force here;
  * brute-force enumeration of all alignments (oracle/brute.py) -- exhaustively for tiny
    lengths, randomly up to length 6;
  * closed forms: LCS, Levenshtein distance (textbook Wagner-Fischer written in this file),
    identity, disjoint alphabets, empty sequences, affine(Go=0) == linear;
  * invariants: symmetry, local >= semi >= global, rescore(CIGAR) == score, local >= 0.
"""
import itertools
import os
import random

import pytest

from oracle import brute
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            yield line.rstrip("\n").split("\t")


def _parse_cigar(c):
    if c == "*":
        return []
    out, num = [], ""
    for ch in c:
        if ch.isdigit():
            num += ch
        else:
            out.append((int(num), ch))
            num = ""
    return out


PINS = list(_rows("pins.tsv"))


@pytest.mark.parametrize("row", PINS, ids=[f"{r[0]}-{r[1]}-{r[2]}-{r[3]}" for r in PINS])
def test_pin_oracle(row):
    q, s, kind, gap, ma, mi, go, ge, score, qb, sb, qe, se, cig, _src = row
    sch = O.Scheme(kind, gap, int(ma), int(mi), int(go), int(ge))
    a = O.align(sch, q, s)
    assert a.score == int(score)
    assert (a.q_begin, a.s_begin, a.q_end, a.s_end) == (int(qb), int(sb), int(qe), int(se))
    assert a.cigar == _parse_cigar(cig)
    r = O.score_rolling(sch, q, s)
    assert (r.score, r.q_end, r.s_end) == (int(score), int(qe), int(se))


@pytest.mark.parametrize("row", PINS, ids=[f"{r[0]}-{r[1]}-{r[2]}-{r[3]}" for r in PINS])
def test_pin_brute(row):
    """Each pin is itself consistent with exhaustive enumeration (score and membership)."""
    q, s, kind, gap, ma, mi, go, ge, score, qb, sb, qe, se, cig, _src = row
    if len(q) * len(s) > (30 if kind == "local" else 48):
        pytest.skip("too large for exhaustive enumeration; pinned by its golden values")
    sch = O.Scheme(kind, gap, int(ma), int(mi), int(go), int(ge))
    best, opt = brute.brute(sch, q, s)
    assert best == int(score)
    key = (int(qb), int(sb), int(qe), int(se), tuple(_parse_cigar(cig)))
    assert key in opt


def test_init_column():
    for gap, go, ge, vals in _rows("init_column.tsv"):
        want = [int(v) for v in vals.split(",")]
        sch = O.Scheme("global", gap, 2, -1, int(go), int(ge))
        for i, v in enumerate(want):
            assert O.align(sch, "ACG"[:i], "").score == v
            assert O.align(sch, "", "TTT"[:i]).score == v


SCHEMES = [
    O.Scheme(k, g, ma, mi, go, ge)
    for k in ("global", "local", "semi")
    for (g, go, ge) in (("linear", 0, 1), ("affine", 2, 1), ("affine", 5, 1), ("affine", 1, 2))
    for (ma, mi) in ((2, -1), (1, -3))
]


def _check_vs_brute(sch, q, s):
    a = O.align(sch, q, s)
    best, opt = brute.brute(sch, q, s)
    assert a.score == best, (sch, q, s)
    key = (a.q_begin, a.s_begin, a.q_end, a.s_end, tuple(a.cigar))
    assert key in opt, (sch, q, s, a, sorted(opt)[:5])
    r = O.score_rolling(sch, q, s)
    assert (r.score, r.q_end, r.s_end) == (a.score, a.q_end, a.s_end)


def test_brute_enumerators_agree():
    """The DFS enumerator and the explicit path list + rescore() agree (global, tiny)."""
    rng = random.Random(1)
    for _ in range(40):
        sch = O.Scheme("global", rng.choice(["linear", "affine"]), 2, -1, rng.randint(0, 3), 1)
        q = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 4)))
        s = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 4)))
        best = max(brute.rescore(sch, q, s, p) for p in brute.paths(len(q), len(s)))
        assert brute.brute(sch, q, s)[0] == best


def test_exhaustive_len_le_2():
    words = [""] + ["".join(w) for L in (1, 2) for w in itertools.product("ACGT", repeat=L)]
    for sch in SCHEMES[::2]:
        for q in words:
            for s in words:
                _check_vs_brute(sch, q, s)


def test_random_vs_brute():
    rng = random.Random(7)
    for t in range(600):
        sch = O.Scheme(rng.choice(["global", "local", "semi"]), rng.choice(["linear", "affine"]),
                       rng.randint(1, 5), rng.randint(-5, 0), rng.randint(0, 8), rng.randint(1, 4))
        lim = 5 if sch.kind == "local" else 6
        q = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, lim)))
        s = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, lim)))
        _check_vs_brute(sch, q, s)


def test_random_with_N_vs_brute():
    rng = random.Random(11)
    for t in range(80):
        sch = O.Scheme(rng.choice(["global", "local", "semi"]), rng.choice(["linear", "affine"]),
                       2, -1, 3, 1)
        q = "".join(rng.choice("ACGTN") for _ in range(rng.randint(0, 5)))
        s = "".join(rng.choice("ACGTN") for _ in range(rng.randint(0, 5)))
        _check_vs_brute(sch, q, s)


def _rand_matrix(rng):
    """A random 5x5 substitution matrix over A,C,G,T,N (matrix scoring)."""
    return tuple(tuple(rng.randint(-6, 6) for _ in range(5)) for _ in range(5))


def test_matrix_scoring_vs_brute():
    """Matrix scoring: the oracle against exhaustive enumeration (brute.sigma reads the
    matrix itself) on tiny pairs with N, all kinds x gap models."""
    rng = random.Random(13)
    for t in range(300):
        m = _rand_matrix(rng)
        sch = O.Scheme(rng.choice(["global", "local", "semi"]), rng.choice(["linear", "affine"]),
                       0, 0, rng.randint(0, 6), rng.randint(1, 3), matrix=m)
        lim = 5 if sch.kind == "local" else 6
        q = "".join(rng.choice("ACGTN") for _ in range(rng.randint(0, lim)))
        s = "".join(rng.choice("ACGTN") for _ in range(rng.randint(0, lim)))
        _check_vs_brute(sch, q, s)


def test_matrix_closed_forms():
    """A matrix with +1 on the diagonal and 0 elsewhere (N included) and zero gap cost is
    the LCS over the 5-letter alphabet; a matrix that spells the simple scheme gives the
    simple scheme's alignments."""
    rng = random.Random(17)
    ident = tuple(tuple(1 if a == b else 0 for b in range(5)) for a in range(5))
    simple = tuple(tuple(2 if (a == b and a < 4) else -1 for b in range(5)) for a in range(5))
    for _ in range(40):
        q = "".join(rng.choice("ACGTN") for _ in range(rng.randint(0, 50)))
        s = "".join(rng.choice("ACGTN") for _ in range(rng.randint(0, 50)))
        assert O.align(O.Scheme("global", "linear", 0, 0, 0, 0, matrix=ident), q, s).score == \
            _lcs(q, s)
        for kind in ("global", "local", "semi"):
            a = O.align(O.Scheme(kind, "affine", 2, -1, 3, 1), q, s)
            b = O.align(O.Scheme(kind, "affine", 0, 0, 3, 1, matrix=simple), q, s)
            assert (a.score, a.q_begin, a.s_begin, a.q_end, a.s_end, a.cigar) == \
                (b.score, b.q_begin, b.s_begin, b.q_end, b.s_end, b.cigar)


# ---------------- closed forms ----------------

def _lcs(a, b):
    """Textbook longest-common-subsequence length (CLRS 15.4)."""
    c = [[0] * (len(b) + 1) for _ in range(len(a) + 1)]
    for i in range(1, len(a) + 1):
        for j in range(1, len(b) + 1):
            c[i][j] = c[i - 1][j - 1] + 1 if a[i - 1] == b[j - 1] else max(c[i - 1][j], c[i][j - 1])
    return c[-1][-1]


def _levenshtein(a, b):
    """Textbook Wagner-Fischer edit distance."""
    prev = list(range(len(b) + 1))
    for i in range(1, len(a) + 1):
        cur = [i] + [0] * len(b)
        for j in range(1, len(b) + 1):
            cur[j] = min(prev[j] + 1, cur[j - 1] + 1, prev[j - 1] + (a[i - 1] != b[j - 1]))
        prev = cur
    return prev[-1]


def test_closed_forms_lcs_levenshtein():
    rng = random.Random(3)
    for _ in range(60):
        q = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 60)))
        s = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 60)))
        assert O.align(O.Scheme("global", "linear", 1, 0, 0, 0), q, s).score == _lcs(q, s)
        assert O.align(O.Scheme("global", "linear", 0, -1, 0, 1), q, s).score == \
            -_levenshtein(q, s)


def test_closed_forms_identity_disjoint_empty():
    rng = random.Random(5)
    for _ in range(30):
        L = rng.randint(1, 80)
        q = "".join(rng.choice("ACGT") for _ in range(L))
        for kind in ("global", "local", "semi"):
            for gap, go in (("linear", 0), ("affine", 5)):
                a = O.align(O.Scheme(kind, gap, 2, -1, go, 1), q, q)
                assert a.score == 2 * L and (a.q_end, a.s_end) == (L, L)
                assert a.cigar == [(L, "M")]
        a_ = "".join(rng.choice("AC") for _ in range(rng.randint(1, 40)))
        b_ = "".join(rng.choice("GT") for _ in range(rng.randint(1, 40)))
        loc = O.align(O.Scheme("local", "affine", 2, -1, 5, 1), a_, b_)
        assert loc.score == 0 and loc.cigar == [] and (loc.q_end, loc.s_end) == (0, 0)
    for kind in ("global", "local", "semi"):
        for gap, go in (("linear", 0), ("affine", 5)):
            sch = O.Scheme(kind, gap, 2, -1, go, 1)
            assert O.align(sch, "", "").score == 0
            e = O.align(sch, "ACGTA", "")
            f = O.align(sch, "", "ACG")
            if kind == "global":
                assert e.score == -(go + 5) and e.cigar == [(5, "I")]
                assert f.score == -(go + 3) and f.cigar == [(3, "D")]
            else:
                assert e.score == 0 and e.cigar == [] and f.score == 0 and f.cigar == []


def test_affine_zero_open_equals_linear():
    rng = random.Random(9)
    for _ in range(100):
        q = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 40)))
        s = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 40)))
        g = rng.randint(1, 4)
        for kind in ("global", "local", "semi"):
            assert O.align(O.Scheme(kind, "affine", 2, -1, 0, g), q, s).score == \
                O.align(O.Scheme(kind, "linear", 2, -1, 0, g), q, s).score


def test_invariants_random():
    rng = random.Random(13)
    for _ in range(150):
        q = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 50)))
        s = "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 50)))
        gap = rng.choice(["linear", "affine"])
        go = rng.randint(0, 6) if gap == "affine" else 0
        ge = rng.randint(1, 3)
        sc = {}
        for kind in ("global", "local", "semi"):
            sch = O.Scheme(kind, gap, 2, -1, go, ge)
            a = O.align(sch, q, s)
            sc[kind] = a.score
            # rescoring the emitted CIGAR reproduces the score (P:266 traceback)
            assert brute.rescore_cigar(sch, q, s, a.q_begin, a.s_begin, a.cigar) == a.score
            nq = sum(l for l, o in a.cigar if o in "MI")
            ns = sum(l for l, o in a.cigar if o in "MD")
            assert (a.q_begin + nq, a.s_begin + ns) == (a.q_end, a.s_end)
            # symmetry under swapping q and s (sigma symmetric)
            assert O.align(sch, s, q).score == a.score
            r = O.score_rolling(sch, q, s)
            assert (r.score, r.q_end, r.s_end) == (a.score, a.q_end, a.s_end)
        assert sc["local"] >= sc["semi"] >= sc["global"]
        assert sc["local"] >= 0
        if set(q) & set(s):
            assert sc["local"] >= 2


def test_batch_matches_single():
    import numpy as np
    from synth import random_pairs
    q, qo, s, so = random_pairs(200, 0, 60, seed=21)
    for kind in ("global", "local", "semi"):
        sch = O.Scheme(kind, "affine", 2, -1, 5, 1)
        res, cig = O.batch(sch, q, qo, s, so, traceback=True, threads=4)
        cigs = O.batch_cigars(res, cig, qo, so)
        for k in range(len(res)):
            a = O.align(sch, q[qo[k]:qo[k + 1]].tobytes(), s[so[k]:so[k + 1]].tobytes())
            assert res["score"][k] == a.score
            assert (res["q_end"][k], res["s_end"][k]) == (a.q_end, a.s_end)
            assert (res["q_begin"][k], res["s_begin"][k]) == (a.q_begin, a.s_begin)
            assert cigs[k] == a.cigar


def test_lowercase_branch_vs_brute():
    """oracle_code's lowercase branch (reading R12: ACGTN case-insensitive): mixed-case
    inputs, including lowercase n, scored against brute force (which maps case itself) and
    equal to the uppercase spelling -- score, cells and CIGAR."""
    rng = random.Random(13)
    for t in range(120):
        sch = O.Scheme(rng.choice(["global", "local", "semi"]), rng.choice(["linear", "affine"]),
                       2, -1, rng.randint(0, 4), 1)
        q = "".join(rng.choice("ACGTNacgtn") for _ in range(rng.randint(0, 5)))
        s = "".join(rng.choice("ACGTNacgtn") for _ in range(rng.randint(0, 5)))
        _check_vs_brute(sch, q, s)
        a, u = O.align(sch, q, s), O.align(sch, q.upper(), s.upper())
        assert (a.score, a.q_begin, a.s_begin, a.q_end, a.s_end, a.cigar) == \
               (u.score, u.q_begin, u.s_begin, u.q_end, u.s_end, u.cigar)


def test_invalid_bytes_rejected():
    """oracle_code's reject branch (R12): every byte outside ACGTNacgtn, at the first, a
    middle and the last position of q or of s, makes align, score_rolling and batch fail;
    every byte inside the alphabet is accepted."""
    import numpy as np
    ok = set(b"ACGTNacgtn")
    sch = O.Scheme("local", "affine", 2, -1, 5, 1)
    for byte in range(256):
        for pos in (0, 2, 4):
            bad = bytearray(b"ACGTA")
            bad[pos] = byte
            for q, s in ((bytes(bad), b"ACGTA"), (b"ACGTA", bytes(bad))):
                if byte in ok:
                    O.align(sch, q, s)
                    O.score_rolling(sch, q, s)
                    continue
                with pytest.raises(ValueError):
                    O.align(sch, q, s)
                with pytest.raises(ValueError):
                    O.score_rolling(sch, q, s)
        if byte not in ok:
            qa = np.frombuffer(b"ACGT" + bytes([byte]) + b"GG", np.uint8)
            sa = np.frombuffer(b"ACGTGG", np.uint8)
            with pytest.raises(ValueError):
                O.batch(sch, qa, np.array([0, 3, 7], np.uint64), np.concatenate([sa, sa]),
                        np.array([0, 6, 12], np.uint64))
