"""C4 at full size: parity on three 100 kbp windows of the ACTUAL 5 Mbp
genomes against stored oracle values (tests/golden/c4_windows.tsv, written by
tools/make_c4_windows.py, which calls only oracle/ and synth/), the closed form of the
identical-genome variant at the full 5 Mbp, and the 16-bit differential kernel equal to the
32-bit kernel on the full 5 Mbp mutated pair."""
import hashlib
import os

import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "c4_windows.tsv")


@pytest.fixture(scope="module")
def ctx():
    import paper_2002_04561_b200 as A
    c = A.Context([0])
    yield c
    c.close()


@pytest.fixture(scope="module")
def genomes():
    from synth import c4_genomes
    return c4_genomes(5_000_000, "a", seed=4)


def _rows():
    with open(GOLD) as f:
        return [l.rstrip("\n").split("\t") for l in f if l.strip() and not l.startswith("#")]


def _window(g1, g2, name, W=100_000):
    n, m = len(g1), len(g2)
    if name == "start":
        return g1[:W], g2[:W]
    if name == "middle":
        a, b = n // 2 - W // 2, m // 2 - W // 2
        return g1[a:a + W], g2[b:b + W]
    return g1[n - W:], g2[m - W:]


@pytest.mark.parametrize("shrink", [False, True], ids=["default", "shrunk"])
def test_c4_windows_of_full_genomes(ctx, genomes, shrink):
    """Start, middle and end windows (100 kbp x 100 kbp) of the C4 genomes: score and end
    cell equal the oracle's.  'shrunk': 3 virtual column strips and 512-row tasks, so every
    boundary type (row hand-off, column edge, first/last strip, ragged last task) occurs."""
    import paper_2002_04561_b200 as A
    g1, g2 = genomes
    rows = _rows()
    assert len(rows) == 9
    if shrink:
        ctx.set_option("long_strips", 3)
        ctx.set_option("long_band_rows", 512)
    try:
        for name, hq, hs, kind, gap, ma, mi, go, ge, score, qe, se in rows:
            q, s = _window(g1, g2, name)
            assert hashlib.sha256(q).hexdigest()[:16] == hq, "synth generator drifted"
            assert hashlib.sha256(s).hexdigest()[:16] == hs, "synth generator drifted"
            r = ctx.align_long(A.Scheme(kind, gap, int(ma), int(mi), int(go), int(ge)), q, s)
            assert (r["score"], r["q_end"], r["s_end"]) == (int(score), int(qe), int(se)), \
                (name, kind, gap)
    finally:
        ctx.set_option("long_strips", 0)
        ctx.set_option("long_band_rows", 0)


def test_c4_full_identical_closed_form(ctx):
    """C4 variant c (G2 = G1, 5 Mbp): the local optimum is n * match = 10^7 at (n, n) -- the
    identity closed form of SURVEY 8(c) -- on the 16-bit kernel and on the 32-bit kernel."""
    import paper_2002_04561_b200 as A
    from synth import c4_genomes
    g1, g2 = c4_genomes(5_000_000, "c", seed=4)
    n = len(g1)
    for narrow in (1, 0):
        ctx.set_option("long_narrow", narrow)
        try:
            r = ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2)
        finally:
            ctx.set_option("long_narrow", 1)
        assert (r["score"], r["q_end"], r["s_end"]) == (2 * n, n, n), narrow


def test_c4_full_long16_equals_s32(ctx, genomes):
    """The full C4 pair (5 Mbp, mutated copy): the 16-bit differential kernel and the 32-bit
    kernel give the same score and end cell (invariant 'GPU s16 = GPU s32' of SURVEY 8(c))."""
    import paper_2002_04561_b200 as A
    g1, g2 = genomes
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    r16 = ctx.align_long(sch, g1, g2)
    assert ctx.stat("long_narrow") == 1
    ctx.set_option("long_narrow", 0)
    try:
        r32 = ctx.align_long(sch, g1, g2)
        assert ctx.stat("long_narrow") == 0
    finally:
        ctx.set_option("long_narrow", 1)
    assert r16 == r32
