"""GPU parity of the long-pair kernel (anyseq_align_long) against the oracle's linear-space
score variant, across virtual column strips (the multi-GPU boundary protocol on one
device), band progress granularity and all kinds."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2002_04561_b200 as A
    c = A.Context([0])
    yield c
    c.close()


def _orc(kind, gap, go, q, s):
    from oracle import oracle as O
    return O.score_rolling(O.Scheme(kind, gap, 2, -1, go, 1), q, s)


@pytest.mark.parametrize("kind", ["global", "local", "semi"])
@pytest.mark.parametrize("gap,go", [("linear", 0), ("affine", 5)])
@pytest.mark.parametrize("strips", [0, 1, 3])
def test_long_random_windows(ctx, kind, gap, go, strips):
    import paper_2002_04561_b200 as A
    from synth import iid, c4_genomes
    for (n, m, seed) in ((1, 1, 1), (37, 1200, 2), (1500, 20, 3), (2600, 2300, 4)):
        q, s = iid(n, seed), iid(m, seed + 100)
        ctx.set_option("long_strips", strips)
        ctx.set_option("long_chunk_cols", 64)
        r = ctx.align_long(A.Scheme(kind, gap, 2, -1, go, 1), q, s)
        o = _orc(kind, gap, go, q, s)
        assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end), (n, m)
    ctx.set_option("long_strips", 0)


def test_long_mutated_window(ctx):
    """C4 variant (a) shape: a 40 kbp window of a mutated genome pair, SW affine 5/1."""
    import paper_2002_04561_b200 as A
    from synth import c4_genomes
    g1, g2 = c4_genomes(40_000, "a", seed=4)
    for strips, chunk in ((1, 64), (4, 32), (7, 256)):
        ctx.set_option("long_strips", strips)
        ctx.set_option("long_chunk_cols", chunk)
        r = ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2)
        o = _orc("local", "affine", 5, g1, g2)
        assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end), strips
    ctx.set_option("long_strips", 0)
    ctx.set_option("long_chunk_cols", 64)


def test_long_identical_closed_form(ctx):
    """C4 variant (c): G2 = G1 -> local score 2n at (n, n) (closed form), 1 Mbp."""
    import paper_2002_04561_b200 as A
    from synth import c4_genomes
    g1, g2 = c4_genomes(1_000_000, "c", seed=4)
    for strips in (1, 2):
        ctx.set_option("long_strips", strips)
        r = ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2)
        assert (r["score"], r["q_end"], r["s_end"]) == (2_000_000, 1_000_000, 1_000_000)
    ctx.set_option("long_strips", 0)


def test_long_strip_invariance(ctx):
    """Result unchanged for G = auto/1/2/4/8 virtual strips (SURVEY 8(c) invariants)."""
    import paper_2002_04561_b200 as A
    from synth import c4_genomes
    g1, g2 = c4_genomes(200_000, "b", seed=8)
    outs = []
    for strips in (0, 1, 2, 4, 8):
        ctx.set_option("long_strips", strips)
        outs.append(tuple(ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2).values()))
    ctx.set_option("long_strips", 0)
    assert len(set(outs)) == 1, outs


def test_long_bad_byte(ctx):
    import paper_2002_04561_b200 as A
    with pytest.raises(A.AnyseqError) as e:
        ctx.align_long(A.Scheme("local"), b"ACGTQ", b"ACGT")
    assert e.value.status_name == "E_BADSEQ"


@pytest.mark.parametrize("kind,gap,go", [("local", "affine", 5), ("global", "linear", 0),
                                         ("semi", "affine", 2)])
def test_long_multi_device(kind, gap, go):
    """A multi-device context: one column strip per entry.  With several GPUs the boundary
    column goes over NVLink (peer stores + system-scope flags); on a one-GPU box the entries
    name GPU 0 repeatedly and form one device group whose strips run in ONE launch (kernels
    that wait on each other are never launched side by side on one GPU)."""
    import torch
    import paper_2002_04561_b200 as A
    from synth import c4_genomes
    n = torch.cuda.device_count()
    g1, g2 = c4_genomes(60_000, "a", seed=4)
    o = _orc(kind, gap, go, g1, g2)
    for devs in ([0, 0], [0, 0, 0, 0], list(range(n)) if n >= 2 else [0] * 8):
        with A.Context(devs) as c:
            r = c.align_long(A.Scheme(kind, gap, 2, -1, go, 1), g1, g2)
        assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end), devs


def test_long_kinds_and_gaps_small_strips(ctx):
    """All kinds x gaps with short strips and tiny progress chunks."""
    import paper_2002_04561_b200 as A
    from synth import iid
    q, s = iid(3000, 91), iid(2800, 92)
    ctx.set_option("long_chunk_cols", 8)
    ctx.set_option("long_strips", 5)
    try:
        for kind in ("global", "local", "semi"):
            for gap, go in (("linear", 0), ("affine", 3)):
                r = ctx.align_long(A.Scheme(kind, gap, 2, -1, go, 1), q, s)
                o = _orc(kind, gap, go, q, s)
                assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end), (kind, gap)
    finally:
        ctx.set_option("long_chunk_cols", 64)
        ctx.set_option("long_strips", 0)


def test_long_matrix_scoring(ctx):
    """Matrix scoring on the long kernel: windows with N against the oracle."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import iid
    m = ((3, -2, -1, -2, -1), (-2, 4, -2, -1, -1), (-1, -2, 3, -2, -1), (-2, -1, -2, 4, -1),
         (-1, -1, -1, -1, 1))
    q, s = bytearray(iid(2100, 61)), bytearray(iid(1900, 62))
    for k in range(0, len(q), 97):
        q[k] = ord("N")
    q, s = bytes(q), bytes(s)
    for kind in ("global", "local", "semi"):
        for gap, go in (("linear", 0), ("affine", 3)):
            r = ctx.align_long(A.Scheme(kind, gap, 0, 0, go, 1, matrix=m), q, s)
            o = O.score_rolling(O.Scheme(kind, gap, 0, 0, go, 1, matrix=m), q, s)
            assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end), (kind, gap)


@pytest.mark.parametrize("narrow", [1, 0])
def test_long_stalled_task_times_out(ctx, narrow):
    """Fault injection (every spin-wait bounded -> E_TIMEOUT): a warp skips one
    row-strip task, the tasks that depend on it exhaust their poll bound, the call returns
    ANYSEQ_E_TIMEOUT (score-only and traceback), and the same context then aligns
    correctly (C4 variant c closed form)."""
    import paper_2002_04561_b200 as A
    from synth import c4_genomes
    g1, g2 = c4_genomes(300_000, "c", seed=4)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    ctx.set_option("long_narrow", narrow)
    try:
        ctx.set_option("long_spin_limit", 1 << 14)
        ctx.set_option("long_stall_task", 2)
        with pytest.raises(A.AnyseqError) as e:
            ctx.align_long(sch, g1, g2)
        assert e.value.status_name == "E_TIMEOUT"
        if narrow:
            with pytest.raises(A.AnyseqError) as e:
                ctx.traceback_long(sch, g1, g2)
            assert e.value.status_name == "E_TIMEOUT"
    finally:
        ctx.set_option("long_stall_task", -1)
        ctx.set_option("long_spin_limit", 0)
    r = ctx.align_long(sch, g1, g2)
    assert (r["score"], r["q_end"], r["s_end"]) == (600_000, 300_000, 300_000)
    if narrow:
        t = ctx.traceback_long(sch, g1, g2)
        assert (t["score"], t["q_begin"], t["s_begin"]) == (600_000, 0, 0)
        assert t["cigar"] == [(300_000, "M")]
    ctx.set_option("long_narrow", 1)
