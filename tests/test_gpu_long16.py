"""GPU parity of the 16-bit differential long kernel (long16.cuh) against the
oracle's linear-space score variant: local affine alignment, both register layouts
(8 and 16 registers per lane: 512- and 1024-row tasks), virtual column strips, scores far
beyond the 16-bit range (the per-warp base), the local floor (unrelated sequences), N in the
query, and the s32 fallback (N in the subject)."""
import pytest

pytestmark = pytest.mark.gpu

SW = dict(kind="local", gap="affine", match=2, mismatch=-1, gap_open=5, gap_extend=1)


@pytest.fixture(scope="module")
def ctx():
    import paper_2002_04561_b200 as A
    c = A.Context([0])
    yield c
    c.close()


def _sch(**kw):
    import paper_2002_04561_b200 as A
    p = dict(SW, **kw)
    return A.Scheme(p["kind"], p["gap"], p["match"], p["mismatch"], p["gap_open"], p["gap_extend"])


def _orc(q, s, **kw):
    from oracle import oracle as O
    p = dict(SW, **kw)
    o = O.score_rolling(O.Scheme(p["kind"], p["gap"], p["match"], p["mismatch"], p["gap_open"],
                                 p["gap_extend"]), q, s)
    return (o.score, o.q_end, o.s_end)


def _run(ctx, q, s, rows=0, strips=0, chunk=64, narrow=1, **kw):
    ctx.set_option("long_band_rows", rows)
    ctx.set_option("long_strips", strips)
    ctx.set_option("long_chunk_cols", chunk)
    ctx.set_option("long_narrow", narrow)
    try:
        r = ctx.align_long(_sch(**kw), q, s)
        used = int(ctx.stat("long_narrow"))
    finally:
        ctx.set_option("long_band_rows", 0)
        ctx.set_option("long_strips", 0)
        ctx.set_option("long_narrow", 1)
    return (r["score"], r["q_end"], r["s_end"]), used


@pytest.mark.parametrize("rows", [0, 512])
@pytest.mark.parametrize("strips", [1, 3])
def test_long16_random_windows(ctx, rows, strips):
    """Unrelated i.i.d. sequences: small scores, the local floor active almost everywhere;
    ragged shapes (fewer rows than one task, fewer columns than the wavefront)."""
    from synth import iid
    for (n, m, seed) in ((1, 1, 1), (5, 70, 2), (37, 1200, 3), (1500, 20, 4), (2600, 2300, 5),
                         (4097, 999, 6)):
        q, s = iid(n, seed), iid(m, seed + 100)
        got, used = _run(ctx, q, s, rows=rows, strips=strips)
        assert used == 1
        assert got == _orc(q, s), (n, m)


@pytest.mark.parametrize("rows", [0, 512])
def test_long16_mutated_beyond_16bit(ctx, rows):
    """C4 variant (a) shape, 40 kbp: optimum ~ 78k (far outside s16) -- the per-warp base
    and its re-basing carry the absolute value; strips exercise the boundary column."""
    from synth import c4_genomes
    g1, g2 = c4_genomes(40_000, "a", seed=4)
    want = _orc(g1, g2)
    assert want[0] > 40_000
    for strips in (1, 4):
        got, used = _run(ctx, g1, g2, rows=rows, strips=strips)
        assert used == 1 and got == want, strips


def test_long16_identical_closed_form(ctx):
    """G2 = G1: local score 2n at (n, n) (closed form), 300 kbp."""
    from synth import c4_genomes
    g1, g2 = c4_genomes(300_000, "c", seed=5)
    for rows, strips in ((0, 1), (0, 3), (512, 2)):
        got, used = _run(ctx, g1, g2, rows=rows, strips=strips)
        assert used == 1 and got == (600_000, 300_000, 300_000)


def test_long16_equals_s32(ctx):
    """The 16-bit and the 32-bit kernels agree on a 300 kbp mutated pair (and on an
    unrelated one) for automatic and explicit column passes."""
    from synth import c4_genomes
    for variant in ("a", "b"):
        g1, g2 = c4_genomes(300_000, variant, seed=6)
        ref, used = _run(ctx, g1, g2, narrow=0)
        assert used == 0
        for rows, strips in ((0, 0), (512, 0), (0, 5)):
            got, used = _run(ctx, g1, g2, rows=rows, strips=strips)
            assert used == 1 and got == ref, (variant, rows, strips)


def test_long16_schemes(ctx):
    """Other affine schemes within the range guard (the paper's 2/1, larger sigma), N in the
    query (allowed), N in the subject (falls back to s32) -- all against the oracle."""
    from synth import iid, c4_genomes
    g1, g2 = c4_genomes(6000, "a", seed=7)
    for kw in (dict(gap_open=2, gap_extend=1), dict(match=5, mismatch=-4, gap_open=10, gap_extend=2),
               dict(match=1, mismatch=-3, gap_open=0, gap_extend=2)):
        got, used = _run(ctx, g1, g2, **kw)
        assert used == 1 and got == _orc(g1, g2, **kw), kw
    qn = bytearray(g1)
    for k in range(0, len(qn), 53):
        qn[k] = ord("N")
    qn = bytes(qn)
    got, used = _run(ctx, qn, g2)
    assert used == 1 and got == _orc(qn, g2)
    got, used = _run(ctx, g2, qn)
    assert used == 0 and got == _orc(g2, qn)
    # a scheme outside the 16-bit range guard runs the s32 kernel
    q, s = iid(900, 8), iid(800, 9)
    got, used = _run(ctx, q, s, gap_open=3000, gap_extend=1000)
    assert used == 0 and got == _orc(q, s, gap_open=3000, gap_extend=1000)
