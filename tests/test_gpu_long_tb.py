"""GPU parity of the linear-space long-pair traceback (anyseq_traceback_long, SURVEY 8(f) f1;
global, local and semi-global kinds with linear gaps)
against the oracle.  Several paths can be optimal, so the test compares what is unique --
the optimum score (and, for local, the end cell under the tie rule of reading R10) -- with
the oracle, and checks that the returned path is valid: it spans exactly the reported
cells and rescoring it by P:241 (oracle/brute.rescore_cigar) gives the optimum."""
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


@pytest.mark.parametrize("n,m,seed", [(1, 1, 1), (0, 9, 2), (7, 0, 3), (300, 280, 4),
                                      (3000, 2500, 5), (9000, 8700, 6), (1, 5000, 7),
                                      (6000, 3, 8)])
def test_long_tb_global_linear(ctx, n, m, seed):
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import iid
    q, s = iid(n, seed), iid(m, seed + 100)
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
    so = O.Scheme("local", "linear", 2, -1, 0, 1)
    r = ctx.traceback_long(A.Scheme("local", "linear", 2, -1, 0, 1), g1, g2)
    o = O.score_rolling(so, g1, g2)
    assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end)
    _check_path(so, g1, g2, r)


def test_long_tb_local_random_and_zero(ctx):
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import iid
    q, s = iid(2500, 21), iid(2700, 22)
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
    with pytest.raises(A.AnyseqError) as e:
        ctx.traceback_long(A.Scheme("global", "affine", 2, -1, 5, 1), b"ACGT", b"ACGT")
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
    q, s = iid(n, seed), iid(m, seed + 100)
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
    q, s = iid(1800, 41), iid(1500, 42)
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
