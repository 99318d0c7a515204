"""Several long pairs in ONE launch (device-side form).

A score-only host batch whose long pairs (n·m >= batch_long_cells, both sides >= 2048) are
aligned by one launch of the 16-bit long kernel's MULTI instance: the row-strip tasks of all
pairs in one ticket queue.  Scores and end cells must equal the oracle's (linear-space
oracle, oracle/oracle.c `oracle_score_rolling`) for every pair, in pair order, and equal the
one-pair-at-a-time path (option long_multi = 0).  A pair whose subject holds an N is not
taken by the 16-bit kernel and must still come back right (per-pair s32 path).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2002_04561_b200 as A
    c = A.Context([0])
    yield c
    c.close()


def _batch(seed, with_n):
    from synth import c4_genomes, random_pairs, csr
    g1, g2 = c4_genomes(20000, "a", seed=seed)
    rng = np.random.default_rng(seed)
    q0, qo0, s0, so0 = random_pairs(30, 0, 300, seed=seed + 1)
    qs = [q0[qo0[k]:qo0[k + 1]].tobytes() for k in range(30)]
    ss = [s0[so0[k]:so0[k + 1]].tobytes() for k in range(30)]
    # long pairs of mixed shapes: square-ish, tall, wide, one side at the 2048 minimum,
    # lengths off the 512-row strip grid (SEMI top padding)
    shapes = [(2048, 6000), (6100, 2100), (3000, 3100), (4500, 4400), (2600, 2500),
              (5000, 5200), (2049, 2300), (3333, 2777)]
    longs = []
    for k, (n, m) in enumerate(shapes):
        a = int(rng.integers(0, 20000 - n))
        b = max(0, min(20000 - m, a + int(rng.integers(-300, 300))))
        longs.append((g1[a:a + n], g2[b:b + m]))
    if with_n:
        sN = bytearray(g2[100:3100])
        sN[1234] = ord("N")
        longs.append((g1[0:3000], bytes(sN)))
    for x, (a, b) in enumerate(longs):
        pos = (7 * x + 3) % (len(qs) + 1)
        qs.insert(pos, a)
        ss.insert(pos, b)
    q, qo = csr(qs)
    s, so = csr(ss)
    return q, qo, s, so, len(longs)


def _oracle_scores(kind, gap, go, q, qo, s, so):
    from oracle import oracle as O
    osch = O.Scheme(kind, gap, 2, -1, go, 1)
    B = len(qo) - 1
    sc = np.zeros(B, np.int32)
    qe = np.zeros(B, np.int64)
    se = np.zeros(B, np.int64)
    for k in range(B):
        r = O.score_rolling(osch, q[qo[k]:qo[k + 1]].tobytes(), s[so[k]:so[k + 1]].tobytes())
        sc[k], qe[k], se[k] = r.score, r.q_end, r.s_end
    return sc, qe, se


@pytest.mark.parametrize("kind", ["global", "semi", "local"])
@pytest.mark.parametrize("gap,go", [("linear", 0), ("affine", 5)])
def test_long_pairs_one_launch(ctx, kind, gap, go):
    import paper_2002_04561_b200 as A
    q, qo, s, so, nl = _batch(200 + len(kind) + go, with_n=(kind == "local"))
    osc, oqe, ose = _oracle_scores(kind, gap, go, q, qo, s, so)
    sch = A.Scheme(kind, gap, 2, -1, go, 1)
    ctx.set_option("batch_long_cells", 1 << 22)
    try:
        sc, ends = ctx.align_batch(sch, q, qo, s, so, ends=True)
        taken = ctx.stat("long_multi_pairs")
        bad = np.flatnonzero(sc != osc)
        assert len(bad) == 0, f"{kind} {gap}: score mismatches at {bad[:5]}"
        bi = np.flatnonzero((ends["q_end"] != oqe) | (ends["s_end"] != ose))
        assert len(bi) == 0, f"{kind} {gap}: end mismatches at {bi[:5]}"
        # every long pair but the one with N in its subject ran in the shared launch
        assert taken == (nl - 1 if kind == "local" else nl)
        assert ctx.stat("long_multi_ms") > 0
        # the one-pair-at-a-time path gives the same results
        ctx.set_option("long_multi", 0)
        sc1, ends1 = ctx.align_batch(sch, q, qo, s, so, ends=True)
        assert ctx.stat("long_multi_pairs") == 0
        assert np.array_equal(sc1, sc)
        assert np.array_equal(ends1["q_end"], ends["q_end"])
        assert np.array_equal(ends1["s_end"], ends["s_end"])
    finally:
        ctx.set_option("long_multi", 1)
        ctx.set_option("batch_long_cells", 1 << 22)


@pytest.mark.parametrize("kind", ["global", "semi", "local"])
def test_long_pairs_one_launch_1024_rows(ctx, kind):
    """The 1024-row MULTI instance (chosen automatically for batches with many long pairs;
    long_band_rows = 1024 forces it here) gives the oracle's results too."""
    import paper_2002_04561_b200 as A
    q, qo, s, so, nl = _batch(500 + len(kind), with_n=False)
    osc, oqe, ose = _oracle_scores(kind, "affine", 5, q, qo, s, so)
    sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
    ctx.set_option("batch_long_cells", 1 << 22)
    ctx.set_option("long_band_rows", 1024)
    try:
        sc, ends = ctx.align_batch(sch, q, qo, s, so, ends=True)
        assert ctx.stat("long_multi_pairs") == nl
        assert np.array_equal(sc, osc)
        assert np.array_equal(ends["q_end"], oqe) and np.array_equal(ends["s_end"], ose)
    finally:
        ctx.set_option("long_band_rows", 0)


def test_long_pairs_one_launch_column_passes(ctx):
    """Forced column passes (long_strips) inside the shared launch: every pair's
    tasks then wait on the pass to their left as well."""
    import paper_2002_04561_b200 as A
    q, qo, s, so, nl = _batch(321, with_n=False)
    osc, oqe, ose = _oracle_scores("local", "affine", 5, q, qo, s, so)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    ctx.set_option("batch_long_cells", 1 << 22)
    try:
        for vs in (2, 3, 7):
            ctx.set_option("long_strips", vs)
            sc, ends = ctx.align_batch(sch, q, qo, s, so, ends=True)
            assert ctx.stat("long_multi_pairs") == nl
            assert np.array_equal(sc, osc), vs
            assert np.array_equal(ends["q_end"], oqe) and np.array_equal(ends["s_end"], ose), vs
    finally:
        ctx.set_option("long_strips", 0)
        ctx.set_option("batch_long_cells", 1 << 22)


def test_long_pairs_one_launch_timeout(ctx):
    """A stalled task in the shared launch (fault injection) times out with E_TIMEOUT and
    the context stays usable."""
    import paper_2002_04561_b200 as A
    q, qo, s, so, nl = _batch(77, with_n=False)
    sch = A.Scheme("global", "linear", 2, -1, 0, 1)
    ctx.set_option("batch_long_cells", 1 << 22)
    ctx.set_option("long_stall_task", 0)  # strip 0 of the first segment: strip 1 waits on it
    ctx.set_option("long_spin_limit", 1 << 16)
    try:
        with pytest.raises(A.AnyseqError) as ei:
            ctx.align_batch(sch, q, qo, s, so)
        assert ei.value.status_name == "E_TIMEOUT"
    finally:
        ctx.set_option("long_stall_task", -1)
        ctx.set_option("long_spin_limit", 1 << 28)
    sc = ctx.align_batch(sch, q, qo, s, so)
    osc, _, _ = _oracle_scores("global", "linear", 0, q, qo, s, so)
    assert np.array_equal(sc, osc)
    ctx.set_option("batch_long_cells", 1 << 22)


@pytest.mark.parametrize("kind", ["global", "semi", "local"])
def test_batch_of_only_long_pairs(ctx, kind):
    """Every pair of the batch is long: the batch kernels' pass plans nothing (all pairs
    skipped by classify) and the shared launch aligns them all."""
    import paper_2002_04561_b200 as A
    from synth import c4_genomes, csr
    g1, g2 = c4_genomes(12000, "a", seed=41)
    shapes = [(2048, 2048), (2048, 2048), (3000, 2500), (2100, 4000), (2048, 2048), (2500, 2600)]
    qs = [g1[k * 1000:k * 1000 + n] for k, (n, m) in enumerate(shapes)]
    ss = [g2[k * 1000:k * 1000 + m] for k, (n, m) in enumerate(shapes)]
    q, qo = csr(qs)
    s, so = csr(ss)
    osc, oqe, ose = _oracle_scores(kind, "affine", 5, q, qo, s, so)
    sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
    ctx.set_option("batch_long_cells", 1 << 22)
    try:
        for multi in (1, 0):
            ctx.set_option("long_multi", multi)
            sc, ends = ctx.align_batch(sch, q, qo, s, so, ends=True)
            assert ctx.stat("long_multi_pairs") == (len(shapes) if multi else 0)
            assert np.array_equal(sc, osc), multi
            assert np.array_equal(ends["q_end"], oqe) and np.array_equal(ends["s_end"], ose)
            assert np.array_equal(ends["q_begin"], oqe) and np.array_equal(ends["s_begin"], ose)
    finally:
        ctx.set_option("long_multi", 1)
        ctx.set_option("batch_long_cells", 1 << 22)


def test_mixed_batch_two_entry_context():
    """A context naming GPU 0 twice: the batch kernels' pass shards the batch over the two
    entries with the long pairs skipped in each shard (ClassifyArgs::skip_cells copied into
    the per-entry contexts), and the long pairs run one at a time over the two-entry long
    path (one launch, two column strips).  Results equal the oracle's."""
    import paper_2002_04561_b200 as A
    q, qo, s, so, nl = _batch(611, with_n=True)
    osc, oqe, ose = _oracle_scores("local", "affine", 5, q, qo, s, so)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    with A.Context([0, 0]) as c:
        c.set_option("batch_long_cells", 1 << 22)
        sc, ends = c.align_batch(sch, q, qo, s, so, ends=True)
        assert c.stat("long_multi_pairs") == 0  # the shared launch is one-device only
        assert np.array_equal(sc, osc)
        assert np.array_equal(ends["q_end"], oqe) and np.array_equal(ends["s_end"], ose)


def _tb_batch(seed, with_n):
    from synth import c4_genomes, random_pairs, csr
    g1, g2 = c4_genomes(12000, "a", seed=seed)
    q0, qo0, s0, so0 = random_pairs(20, 0, 250, seed=seed + 1)
    qs = [q0[qo0[k]:qo0[k + 1]].tobytes() for k in range(20)]
    ss = [s0[so0[k]:so0[k + 1]].tobytes() for k in range(20)]
    shapes = [(2048, 2900), (2700, 2100), (2300, 2400), (2049, 2050), (2600, 2500)]
    longs = [(g1[k * 1500:k * 1500 + n], g2[k * 1500 + 20:k * 1500 + 20 + m])
             for k, (n, m) in enumerate(shapes)]
    if with_n:
        sN = bytearray(g2[9000:11100])
        sN[700] = ord("N")
        longs.append((g1[9000:11200], bytes(sN)))
    for x, (a, b) in enumerate(longs):
        pos = (5 * x + 2) % (len(qs) + 1)
        qs.insert(pos, a)
        ss.insert(pos, b)
    q, qo = csr(qs)
    s, so = csr(ss)
    return q, qo, s, so, len(shapes)


@pytest.mark.parametrize("kind", ["global", "semi", "local"])
@pytest.mark.parametrize("gap,go", [("linear", 0), ("affine", 5)])
def test_traceback_long_pairs_one_pass(ctx, kind, gap, go):
    """Traceback batches: the long pairs' checkpointing forward passes share one launch
    (MULTI + CKPT instance), then each pair's tile walk runs from its checkpoints.  Scores,
    begin/end cells and CIGARs equal the oracle's; cigar offsets stay contiguous."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    q, qo, s, so, nl = _tb_batch(700 + len(kind) + go, with_n=(kind == "global" and gap == "linear"))
    osch = O.Scheme(kind, gap, 2, -1, go, 1)
    res, cig = O.batch(osch, q, qo, s, so, traceback=True)
    ocig = O.batch_cigars(res, cig, qo, so)
    sch = A.Scheme(kind, gap, 2, -1, go, 1)
    ctx.set_option("batch_long_cells_tb", 1 << 22)
    try:
        aln, words = ctx.traceback(sch, q, qo, s, so)
        assert ctx.stat("long_multi_pairs") == nl
        assert np.array_equal(aln["score"], res["score"].astype(np.int32))
        for f in ("q_begin", "s_begin", "q_end", "s_end"):
            assert np.array_equal(aln[f], res[f]), f
        got = A.cigars_of(aln, words)
        bad = [k for k in range(len(got)) if got[k] != ocig[k]]
        assert not bad, f"CIGAR mismatches at {bad[:5]}"
        cl = aln["cigar_len"].astype(np.uint64)
        assert np.array_equal(aln["cigar_offset"], np.cumsum(cl) - cl)
    finally:
        ctx.set_option("batch_long_cells_tb", 1 << 22)


@pytest.mark.parametrize("tb", [False, True])
def test_bad_symbol_in_long_pair(ctx, tb):
    """An invalid byte inside a long pair of a mixed batch is reported as E_BADSEQ (no
    result is returned), and the context aligns the next batch normally."""
    import paper_2002_04561_b200 as A
    from synth import csr
    q, qo, s, so, nl = _batch(901, with_n=False)
    qs = [q[qo[k]:qo[k + 1]].tobytes() for k in range(len(qo) - 1)]
    ss = [s[so[k]:so[k + 1]].tobytes() for k in range(len(so) - 1)]
    k = max(range(len(qs)), key=lambda i: len(qs[i]) * len(ss[i]))  # a long pair
    bad = bytearray(ss[k])
    bad[1500] = ord("X")
    ss2 = list(ss)
    ss2[k] = bytes(bad)
    sb, sob = csr(ss2)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    ctx.set_option("batch_long_cells", 1 << 22)
    ctx.set_option("batch_long_cells_tb", 1 << 22)
    with pytest.raises(A.AnyseqError) as e:
        if tb:
            ctx.traceback(sch, q, qo, sb, sob)
        else:
            ctx.align_batch(sch, q, qo, sb, sob)
    assert e.value.status_name == "E_BADSEQ"
    sc = ctx.align_batch(sch, q, qo, s, so)
    osc, _, _ = _oracle_scores("local", "affine", 5, q, qo, s, so)
    assert np.array_equal(sc, osc)


def test_shared_launch_in_groups(ctx):
    """More long pairs than one launch takes (option long_multi_group, 2048 by default; 2
    here): score mode runs several launches and takes every pair; traceback takes the first
    group through the shared pass and the rest one by one.  Results equal the oracle's."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    q, qo, s, so, nl = _tb_batch(977, with_n=False)
    osch = O.Scheme("semi", "affine", 2, -1, 5, 1)
    res, cig = O.batch(osch, q, qo, s, so, traceback=True)
    ocig = O.batch_cigars(res, cig, qo, so)
    sch = A.Scheme("semi", "affine", 2, -1, 5, 1)
    ctx.set_option("long_multi_group", 2)
    try:
        sc, ends = ctx.align_batch(sch, q, qo, s, so, ends=True)
        assert ctx.stat("long_multi_pairs") == nl
        assert np.array_equal(sc, res["score"].astype(np.int32))
        assert np.array_equal(ends["q_end"], res["q_end"]) and np.array_equal(ends["s_end"], res["s_end"])
        aln, words = ctx.traceback(sch, q, qo, s, so)
        assert ctx.stat("long_multi_pairs") == 2
        assert np.array_equal(aln["score"], res["score"].astype(np.int32))
        for f in ("q_begin", "s_begin", "q_end", "s_end"):
            assert np.array_equal(aln[f], res[f]), f
        assert A.cigars_of(aln, words) == ocig
    finally:
        ctx.set_option("long_multi_group", 2048)
