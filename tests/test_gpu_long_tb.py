"""GPU parity of the linear-space long-pair traceback (anyseq_traceback_long).

Checkpointed path (every kind, linear and affine gaps): the walk takes every decision from
exact full-matrix values, so score, begin cell, end cell and CIGAR are compared
ELEMENT BY ELEMENT with the oracle's full-matrix traceback (oracle.align), at checkpoint
geometries that put many tile boundaries on the path.  Larger pairs (beyond the oracle's
full matrix) are checked against the oracle's linear-space score (score and end cell) and
by rescoring the path.

Hirschberg fallback (linear gaps, subjects with N): several paths can be optimal, so those
tests compare what is unique -- the optimum score and end cell -- and check that the path
is valid and rescores to the optimum."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2002_04561_b200 as A
    c = A.Context([0])
    yield c
    c.close()


def _check_path(scheme_o, q, s, r):
    from oracle import brute
    cig = r["cigar"]
    nq = sum(l for l, o in cig if o in "MI")
    ns = sum(l for l, o in cig if o in "MD")
    assert (r["q_begin"] + nq, r["s_begin"] + ns) == (r["q_end"], r["s_end"])
    assert all(cig[k][1] != cig[k + 1][1] for k in range(len(cig) - 1))  # run-length encoded
    qs, ss = q.decode(), s.decode()
    assert brute.rescore_cigar(scheme_o, qs, ss, r["q_begin"], r["s_begin"], cig) == r["score"]


KINDS = ("global", "local", "semi")
GAPS = (("linear", 0), ("affine", 5), ("affine", 2))
# (long_band_rows, tb_ck_every, tb_kc_shift, walk_helpers): 512-row strips with tiles
# 512 x 256 (the walker alone) and 1024 x 512 (helper CTAs recomputing predicted tiles), and
# the automatic geometry with helpers
GEOMS = ((512, 1, 8, 0), (512, 2, 9, 96), (0, 0, 0, 96))


def _set_geom(ctx, geom):
    rows, every, kcs, helpers = geom
    ctx.set_option("long_band_rows", rows)
    ctx.set_option("tb_ck_every", every)
    ctx.set_option("tb_kc_shift", kcs)
    ctx.set_option("walk_helpers", helpers)


def _pairs():
    from synth import iid, c4_genomes
    g1, g2 = c4_genomes(9000, "a", seed=21)
    return [(iid(3000, 1), iid(2800, 2)),              # unrelated: gappy, many ties
            (g1[:3100], g2[:2900]),                    # mutated copy, indels
            (g1[5000:5400], g2[200:5200]),             # wide, a long free-end / gap run
            (iid(1, 3), iid(1, 4)), (iid(70, 5), iid(1, 6)), (iid(1, 7), iid(700, 8))]


@pytest.mark.parametrize("geom", GEOMS, ids=["512x256", "1024x512", "auto"])
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gap,go", GAPS, ids=["lin", "aff5", "aff2"])
def test_long_tb_ckpt_bit_exact(ctx, geom, kind, gap, go):
    """Checkpointed traceback == the oracle's full-matrix traceback: score, begin, end and
    CIGAR, for every kind and gap model, across checkpoint geometries."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    so = O.Scheme(kind, gap, 2, -1, go, 1)
    _set_geom(ctx, geom)
    try:
        for q, s in _pairs():
            r = ctx.traceback_long(A.Scheme(kind, gap, 2, -1, go, 1), q, s)
            assert ctx.stat("tb_method") == 1
            o = O.align(so, q, s)
            got = (r["score"], r["q_begin"], r["s_begin"], r["q_end"], r["s_end"])
            assert got == (o.score, o.q_begin, o.s_begin, o.q_end, o.s_end), (len(q), len(s))
            assert r["cigar"] == o.cigar, (len(q), len(s))
    finally:
        _set_geom(ctx, (0, 0, 0, 96))


@pytest.mark.parametrize("kind", KINDS)
def test_long_tb_ckpt_matrix_scoring(ctx, kind):
    """Matrix scoring through the checkpointed traceback, bit-exact."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import c4_genomes
    mat = ((3, -2, -1, -2, -1), (-2, 2, -2, -1, -1), (-1, -2, 3, -2, -1),
           (-2, -1, -2, 2, -1), (-1, -1, -1, -1, -1))
    g1, g2 = c4_genomes(4000, "a", seed=23)
    so = O.Scheme(kind, "affine", 0, 0, 4, 1, matrix=mat)
    ctx.set_option("tb_kc_shift", 8)
    try:
        r = ctx.traceback_long(A.Scheme(kind, "affine", 0, 0, 4, 1, matrix=mat), g1, g2)
    finally:
        ctx.set_option("tb_kc_shift", 0)
    o = O.align(so, g1, g2)
    assert (r["score"], r["q_begin"], r["s_begin"], r["q_end"], r["s_end"]) == \
           (o.score, o.q_begin, o.s_begin, o.q_end, o.s_end)
    assert r["cigar"] == o.cigar


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gap,go", [("affine", 5), ("linear", 0)])
def test_long_tb_ckpt_large(ctx, kind, gap, go):
    """30 kbp mutated pair (C4 variant-a shape): score and end cell equal the oracle's
    linear-space score; the path spans begin -> end and rescores to the optimum."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import c4_genomes
    g1, g2 = c4_genomes(30_000, "a", seed=24)
    so = O.Scheme(kind, gap, 2, -1, go, 1)
    r = ctx.traceback_long(A.Scheme(kind, gap, 2, -1, go, 1), g1, g2)
    assert ctx.stat("tb_method") == 1
    o = O.score_rolling(so, g1, g2)
    assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end)
    _check_path(so, g1, g2, r)


def _with_n(x: bytes) -> bytes:
    """The same sequence with one base replaced by N (sends the subject to the 32-bit kernel
    and the traceback to the Hirschberg fallback)."""
    b = bytearray(x)
    if b:
        b[len(b) // 2] = ord("N")
    return bytes(b)


@pytest.mark.parametrize("n,m,seed", [(1, 1, 1), (0, 9, 2), (7, 0, 3), (300, 280, 4),
                                      (3000, 2500, 5), (9000, 8700, 6), (1, 5000, 7),
                                      (6000, 3, 8)])
def test_long_tb_global_linear(ctx, n, m, seed):
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import iid
    q, s = iid(n, seed), _with_n(iid(m, seed + 100))
    r = ctx.traceback_long(A.Scheme("global", "linear", 2, -1, 0, 1), q, s)
    so = O.Scheme("global", "linear", 2, -1, 0, 1)
    o = O.score_rolling(so, q, s)
    assert r["score"] == o.score
    assert (r["q_begin"], r["s_begin"], r["q_end"], r["s_end"]) == (0, 0, n, m)
    _check_path(so, q, s, r)


def test_long_tb_global_matches_full_traceback_score(ctx):
    """Small case: the oracle's full-matrix traceback has the same score."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import iid
    q, s = iid(700, 11), iid(650, 12)
    so = O.Scheme("global", "linear", 1, -1, 0, 2)
    r = ctx.traceback_long(A.Scheme("global", "linear", 1, -1, 0, 2), q, s)
    assert r["score"] == O.align(so, q, s).score
    _check_path(so, q, s, r)


@pytest.mark.parametrize("length,seed", [(5000, 4), (30_000, 5)])
def test_long_tb_local_linear_mutated(ctx, length, seed):
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import c4_genomes
    g1, g2 = c4_genomes(length, "a", seed=seed)
    g2 = _with_n(g2)
    so = O.Scheme("local", "linear", 2, -1, 0, 1)
    r = ctx.traceback_long(A.Scheme("local", "linear", 2, -1, 0, 1), g1, g2)
    o = O.score_rolling(so, g1, g2)
    assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end)
    _check_path(so, g1, g2, r)


def test_long_tb_local_random_and_zero(ctx):
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import iid
    q, s = iid(2500, 21), _with_n(iid(2700, 22))
    so = O.Scheme("local", "linear", 2, -1, 0, 1)
    r = ctx.traceback_long(A.Scheme("local", "linear", 2, -1, 0, 1), q, s)
    o = O.align(so, q, s)
    assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end)
    _check_path(so, q, s, r)
    # no positive cell: the empty alignment
    r = ctx.traceback_long(A.Scheme("local", "linear", 2, -1, 0, 1), b"AAAA", b"CCCC")
    assert r["score"] == 0 and r["cigar"] == []


def test_long_tb_errors(ctx):
    import paper_2002_04561_b200 as A
    # affine gaps with an N in the subject: neither the 16-bit kernel nor Hirschberg (linear)
    with pytest.raises(A.AnyseqError) as e:
        ctx.traceback_long(A.Scheme("global", "affine", 2, -1, 5, 1), b"ACGT" * 300,
                           b"ACNT" * 300)
    assert e.value.status == 6
    with pytest.raises(A.AnyseqError) as e:
        ctx.traceback_long(A.Scheme("global", "linear", 2, -1, 0, 1), b"ACXT", b"ACGT")
    assert e.value.status == 2
    with pytest.raises(A.AnyseqError) as e:
        ctx.traceback_long(A.Scheme("global", "linear", 2, -1, 0, 1), b"ACGT" * 100,
                           b"TTGA" * 100, cigar_capacity=1)
    assert e.value.status == 4 and e.value.cigar_used > 1


@pytest.mark.parametrize("n,m,seed", [(1, 1, 31), (5, 0, 32), (2000, 2600, 33), (9000, 400, 34),
                                      (300, 7000, 35)])
def test_long_tb_semi_linear(ctx, n, m, seed):
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import iid
    q, s = iid(n, seed), _with_n(iid(m, seed + 100))
    so = O.Scheme("semi", "linear", 2, -1, 0, 1)
    r = ctx.traceback_long(A.Scheme("semi", "linear", 2, -1, 0, 1), q, s)
    o = O.score_rolling(so, q, s)
    assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end)
    assert r["q_begin"] == 0 or r["s_begin"] == 0          # begins on row 0 or column 0
    assert r["q_end"] == n or r["s_end"] == m              # ends on the last row or column
    _check_path(so, q, s, r)


def test_long_tb_semi_read_in_reference(ctx):
    """A 3 kbp read taken from a 40 kbp reference: semi-global places it with free end gaps."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import c4_genomes
    g1, g2 = c4_genomes(40_000, "a", seed=9)
    read = g2[12_000:15_000]
    g1 = _with_n(g1)
    so = O.Scheme("semi", "linear", 2, -1, 0, 1)
    r = ctx.traceback_long(A.Scheme("semi", "linear", 2, -1, 0, 1), read, g1)
    o = O.score_rolling(so, read, g1)
    assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end)
    _check_path(so, read, g1, r)


@pytest.mark.parametrize("leaf", [64, 4096, 1 << 24])
def test_long_tb_leaf_sizes(ctx, leaf):
    """Deep recursion (tiny leaves: many levels, one-row and one-column pieces) and no
    recursion at all give the same optimum and valid paths, for every kind."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import iid
    q, s = iid(1800, 41), _with_n(iid(1500, 42))
    ctx.set_option("tb_leaf_cells", leaf)
    try:
        for kind in ("global", "local", "semi"):
            so = O.Scheme(kind, "linear", 2, -1, 0, 1)
            r = ctx.traceback_long(A.Scheme(kind, "linear", 2, -1, 0, 1), q, s)
            o = O.score_rolling(so, q, s)
            assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end), kind
            _check_path(so, q, s, r)
    finally:
        ctx.set_option("tb_leaf_cells", 1 << 20)
