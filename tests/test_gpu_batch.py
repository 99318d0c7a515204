"""GPU parity of the batch path (score-only, end cells, traceback) against the CPU oracle.

Every comparison is element by element and bit-exact (integers): score, end cell, begin
cell and CIGAR.  Inputs are seeded synthetic DNA (synth/), with lengths spanning several
strips of every kernel variant and ragged tails.  All calls go through the C-ABI.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KINDS = ("global", "local", "semi")
GAPS = (("linear", 0, 1), ("affine", 5, 1), ("affine", 2, 1), ("affine", 0, 2))


@pytest.fixture(scope="module")
def ctx():
    import paper_2002_04561_b200 as A
    c = A.Context([0])
    yield c
    c.close()


def _oracle(kind, gap, go, ge, q, qo, s, so, tb, ma=2, mi=-1):
    from oracle import oracle as O
    res, cig = O.batch(O.Scheme(kind, gap, ma, mi, go, ge), q, qo, s, so, traceback=tb)
    return res, (O.batch_cigars(res, cig, qo, so) if tb else None)


def _check_scores(ctx, sch, q, qo, s, so, res, ends=True):
    sc, aln = ctx.align_batch(sch, q, qo, s, so, ends=True)
    bad = np.flatnonzero(sc != res["score"].astype(np.int32))
    assert len(bad) == 0, f"{sch}: {len(bad)} score mismatches, first pair {bad[:5]}"
    if ends:
        bi = np.flatnonzero((aln["q_end"] != res["q_end"]) | (aln["s_end"] != res["s_end"]))
        assert len(bi) == 0, f"{sch}: end mismatches at {bi[:5]}"
    # score-only path without ends
    sc2 = ctx.align_batch(sch, q, qo, s, so)
    assert np.array_equal(sc2, sc)


def _check_tb(ctx, sch, q, qo, s, so, res, ocig):
    import paper_2002_04561_b200 as A
    aln, words = ctx.traceback(sch, q, qo, s, so)
    assert np.array_equal(aln["score"], res["score"].astype(np.int32)), sch
    for f in ("q_begin", "s_begin", "q_end", "s_end"):
        bad = np.flatnonzero(aln[f] != res[f])
        assert len(bad) == 0, f"{sch} {f} mismatch at {bad[:5]}"
    got = A.cigars_of(aln, words)
    bad = [k for k in range(len(got)) if got[k] != ocig[k]]
    assert not bad, f"{sch}: cigar mismatch at pairs {bad[:5]}: {got[bad[0]]} vs {ocig[bad[0]]}"


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gap", GAPS, ids=lambda g: f"{g[0]}{g[1]}_{g[2]}")
def test_random_pairs_all_variants(ctx, kind, gap):
    """Random pairs, lengths 0..330 (several strips of R=8/16/19 variants, ragged tails)."""
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    q, qo, s, so = random_pairs(300, 0, 330, seed=100 * KINDS.index(kind) + GAPS.index(gap))
    g, go, ge = gap
    res, ocig = _oracle(kind, g, go, ge, q, qo, s, so, tb=True)
    sch = A.Scheme(kind, g, 2, -1, go, ge)
    _check_scores(ctx, sch, q, qo, s, so, res)
    _check_tb(ctx, sch, q, qo, s, so, res, ocig)


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_forced_variants_score(ctx, variant):
    """Every score variant (s16x2 R=8/16/19, s32 R=8/16) on the same inputs."""
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    q, qo, s, so = random_pairs(200, 1, 420, seed=50 + variant)
    ctx.set_option("force_variant", variant)
    try:
        for kind in KINDS:
            for g, go, ge in (("linear", 0, 1), ("affine", 5, 1)):
                res, _ = _oracle(kind, g, go, ge, q, qo, s, so, tb=False)
                _check_scores(ctx, A.Scheme(kind, g, 2, -1, go, ge), q, qo, s, so, res)
    finally:
        ctx.set_option("force_variant", -1)


@pytest.mark.parametrize("variant", [5, 6])
def test_forced_variants_traceback(ctx, variant):
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    q, qo, s, so = random_pairs(150, 0, 300, seed=70 + variant)
    ctx.set_option("force_variant", variant)
    try:
        for kind in KINDS:
            for g, go, ge in (("linear", 0, 1), ("affine", 5, 1)):
                res, ocig = _oracle(kind, g, go, ge, q, qo, s, so, tb=True)
                _check_tb(ctx, A.Scheme(kind, g, 2, -1, go, ge), q, qo, s, so, res, ocig)
    finally:
        ctx.set_option("force_variant", -1)


def test_scoring_params_sweep(ctx):
    """Random valid schemes (match 1..5, mismatch -5..0, Go 0..8, Ge 1..4)."""
    import random
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    rng = random.Random(17)
    for t in range(12):
        kind = rng.choice(KINDS)
        g = rng.choice(["linear", "affine"])
        ma, mi, go, ge = rng.randint(1, 5), rng.randint(-5, 0), rng.randint(0, 8), rng.randint(1, 4)
        q, qo, s, so = random_pairs(80, 0, 200, seed=1000 + t)
        res, ocig = _oracle(kind, g, go, ge, q, qo, s, so, tb=True, ma=ma, mi=mi)
        sch = A.Scheme(kind, g, ma, mi, go, ge)
        _check_scores(ctx, sch, q, qo, s, so, res)
        _check_tb(ctx, sch, q, qo, s, so, res, ocig)


def test_N_and_lowercase(ctx):
    """N mismatches everything (reading R12) -> s32 path; lower case accepted."""
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    q, qo, s, so = random_pairs(120, 0, 180, seed=5, alphabet=b"ACGTNacgtn")
    for kind in KINDS:
        res, ocig = _oracle(kind, "affine", 3, 1, q, qo, s, so, tb=True)
        sch = A.Scheme(kind, "affine", 2, -1, 3, 1)
        _check_scores(ctx, sch, q, qo, s, so, res)
        _check_tb(ctx, sch, q, qo, s, so, res, ocig)


def test_edge_shapes(ctx):
    """n or m in {0, 1, 7, 8, 9, 31, 32, 33, 63, 64, 65, 151, 152, 153} against each other."""
    import paper_2002_04561_b200 as A
    from synth import csr, iid
    L = [0, 1, 7, 8, 9, 31, 32, 33, 63, 64, 65, 151, 152, 153]
    qs, ss = [], []
    for i, a in enumerate(L):
        for j, b in enumerate(L):
            qs.append(iid(a, 3 * i + 1))
            ss.append(iid(b, 7 * j + 2))
    q, qo = csr(qs)
    s, so = csr(ss)
    for kind in KINDS:
        for g, go, ge in (("linear", 0, 1), ("affine", 5, 1)):
            res, ocig = _oracle(kind, g, go, ge, q, qo, s, so, tb=True)
            sch = A.Scheme(kind, g, 2, -1, go, ge)
            _check_scores(ctx, sch, q, qo, s, so, res)
            _check_tb(ctx, sch, q, qo, s, so, res, ocig)


def test_golden_pins_on_gpu(ctx):
    import os
    import paper_2002_04561_b200 as A
    from synth import csr
    rows = []
    with open(os.path.join(os.path.dirname(__file__), "golden", "pins.tsv")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append(line.rstrip("\n").split("\t"))
    for r in rows:
        qq, ss_, kind, gap, ma, mi, go, ge, score, qb, sb, qe, se, cig, _ = r
        q, qo = csr([qq.encode()])
        s, so = csr([ss_.encode()])
        sch = A.Scheme(kind, gap, int(ma), int(mi), int(go), int(ge))
        aln, words = ctx.traceback(sch, q, qo, s, so)
        a = aln[0]
        assert int(a["score"]) == int(score), r
        assert (a["q_begin"], a["s_begin"], a["q_end"], a["s_end"]) == \
            (int(qb), int(sb), int(qe), int(se)), r
        got = "".join(f"{l}{o}" for l, o in A.decode_cigar(words[a["cigar_offset"]:
                                                                 a["cigar_offset"] + a["cigar_len"]]))
        assert (got or "*") == cig, r


def test_c1_nw_traceback(ctx):
    """C1: one 1000 x 1000 pair, global linear (2/-1/-1), score + traceback."""
    import paper_2002_04561_b200 as A
    from synth import c1_pair, csr
    a, b = c1_pair(1)
    q, qo = csr([a])
    s, so = csr([b])
    res, ocig = _oracle("global", "linear", 0, 1, q, qo, s, so, tb=True)
    _check_tb(ctx, A.Scheme("global", "linear", 2, -1, 0, 1), q, qo, s, so, res, ocig)


def test_c2_c3_shape_full_oracle(ctx):
    """C2/C3 workload shape (150 bp reads vs windows), 20k pairs, full oracle."""
    import paper_2002_04561_b200 as A
    from synth import c2_reads, uniform_csr
    qm, sm = c2_reads(20000, seed=2)
    q, qo = uniform_csr(qm)
    s, so = uniform_csr(sm)
    res, _ = _oracle("semi", "affine", 5, 1, q, qo, s, so, tb=False)
    _check_scores(ctx, A.Scheme("semi", "affine", 2, -1, 5, 1), q, qo, s, so, res)
    res, ocig = _oracle("local", "affine", 5, 1, q, qo, s, so, tb=True)
    _check_tb(ctx, A.Scheme("local", "affine", 2, -1, 5, 1), q, qo, s, so, res, ocig)


def test_c2_full_size_sampled(ctx):
    """C2 at BASELINE size (1M pairs, the launch configuration bench.py times); the oracle
    checks a fixed sample of 3000 pairs one by one."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import c2_reads, uniform_csr
    qm, sm = c2_reads(1_000_000, seed=2)
    q, qo = uniform_csr(qm)
    s, so = uniform_csr(sm)
    sc = ctx.align_batch(A.Scheme("semi", "affine", 2, -1, 5, 1), q, qo, s, so)
    idx = np.random.default_rng(0).choice(len(sc), 3000, replace=False)
    sch = O.Scheme("semi", "affine", 2, -1, 5, 1)
    for k in idx:
        assert sc[k] == O.align(sch, qm[k].tobytes(), sm[k].tobytes(), traceback=False).score, k
    # property at any size: semi-global >= 0 and <= 2 * 150
    assert sc.min() >= 0 and sc.max() <= 300


def test_c3_full_size_sampled(ctx):
    """C3 at BASELINE size (1M pairs, local affine, traceback + CIGAR; several H-store
    chunks): the oracle checks score, begin, end and CIGAR of a fixed sample of 1000 pairs,
    and every CIGAR is checked against its pair's coordinates (property at any size)."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import c2_reads, uniform_csr
    qm, sm = c2_reads(1_000_000, seed=2)
    q, qo = uniform_csr(qm)
    s, so = uniform_csr(sm)
    ctx.set_option("tb_scratch_bytes", 4 << 30)  # > 1 fill/walk chunk
    try:
        aln, words = ctx.traceback(A.Scheme("local", "affine", 2, -1, 5, 1), q, qo, s, so)
    finally:
        ctx.set_option("tb_scratch_bytes", 16 << 30)
    sch = O.Scheme("local", "affine", 2, -1, 5, 1)
    idx = np.random.default_rng(1).choice(len(aln), 1000, replace=False)
    cigs = A.cigars_of(aln[idx], words)
    for n, k in enumerate(idx):
        o = O.align(sch, qm[k].tobytes(), sm[k].tobytes())
        got = (int(aln["score"][k]), int(aln["q_begin"][k]), int(aln["s_begin"][k]),
               int(aln["q_end"][k]), int(aln["s_end"][k]))
        assert got == (o.score, o.q_begin, o.s_begin, o.q_end, o.s_end), k
        assert cigs[n] == o.cigar, k
    # every CIGAR spans exactly its alignment: M+I rows, M+D columns
    ops = words & 15
    lens = (words >> 4).astype(np.int64)
    off = aln["cigar_offset"].astype(np.int64)
    cnt = aln["cigar_len"].astype(np.int64)
    seg = np.repeat(np.arange(len(aln)), cnt)
    rows = np.bincount(seg, weights=lens * (ops != 2), minlength=len(aln))
    cols = np.bincount(seg, weights=lens * (ops != 1), minlength=len(aln))
    assert np.all(off[1:] == off[:-1] + cnt[:-1])
    assert np.array_equal(rows.astype(np.int64), aln["q_end"] - aln["q_begin"])
    assert np.array_equal(cols.astype(np.int64), aln["s_end"] - aln["s_begin"])


def _matrix(seed):
    rng = np.random.default_rng(seed)
    m = rng.integers(-5, 6, size=(5, 5))
    m[np.arange(4), np.arange(4)] = rng.integers(1, 6, size=4)  # matches score positive
    return tuple(tuple(int(x) for x in row) for row in m)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("gap", [("linear", 0, 1), ("affine", 4, 1)], ids=lambda g: g[0])
def test_matrix_scoring(ctx, kind, gap):
    """Matrix scoring: random 5x5 sigma, pairs with and without N (s16x2 and
    s32 paths), score + ends and traceback against the oracle."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import random_pairs
    g, go, ge = gap
    m = _matrix(200 + KINDS.index(kind))
    for with_n in (False, True):
        q, qo, s, so = random_pairs(250, 0, 240, seed=300 + with_n)
        if with_n:  # sprinkle N so those pairs take the s32 path
            rng = np.random.default_rng(5)
            q = q.copy()
            q[rng.choice(len(q), size=len(q) // 40, replace=False)] = ord("N")
        res, cig = O.batch(O.Scheme(kind, g, 0, 0, go, ge, matrix=m), q, qo, s, so, traceback=True)
        ocig = O.batch_cigars(res, cig, qo, so)
        sch = A.Scheme(kind, g, 0, 0, go, ge, matrix=m)
        _check_scores(ctx, sch, q, qo, s, so, res)
        _check_tb(ctx, sch, q, qo, s, so, res, ocig)


def test_c5_mixed_sample(ctx):
    """C5 shape (mixed 100..1000 bp), all kinds x modes, 600 pairs."""
    import paper_2002_04561_b200 as A
    from synth import c5_mixed
    q, qo, s, so = c5_mixed(600, seed=5)
    for kind in KINDS:
        res, ocig = _oracle(kind, "affine", 5, 1, q, qo, s, so, tb=True)
        sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
        _check_scores(ctx, sch, q, qo, s, so, res)
        _check_tb(ctx, sch, q, qo, s, so, res, ocig)


def test_s16_equals_s32_at_scale(ctx):
    """GPU s16x2 == GPU s32 on the same 200k C2 pairs (invariant of SURVEY 8(c))."""
    import paper_2002_04561_b200 as A
    from synth import c2_reads, uniform_csr
    qm, sm = c2_reads(200_000, seed=9)
    q, qo = uniform_csr(qm)
    s, so = uniform_csr(sm)
    for kind in KINDS:
        sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
        a16, e16 = ctx.align_batch(sch, q, qo, s, so, ends=True)
        ctx.set_option("allow16", 0)
        try:
            a32, e32 = ctx.align_batch(sch, q, qo, s, so, ends=True)
        finally:
            ctx.set_option("allow16", 1)
        assert np.array_equal(a16, a32)
        assert np.array_equal(e16["q_end"], e32["q_end"]) and np.array_equal(e16["s_end"], e32["s_end"])


def test_errors(ctx):
    import paper_2002_04561_b200 as A
    from synth import csr
    q, qo = csr([b"ACGT", b"ACXT"])
    s, so = csr([b"ACGT", b"ACGT"])
    with pytest.raises(A.AnyseqError) as e:
        ctx.align_batch(A.Scheme("global"), q, qo, s, so)
    assert e.value.status_name == "E_BADSEQ"
    assert "pair 1" in str(e.value) and "0x58" in str(e.value)
    with pytest.raises(A.AnyseqError) as e:
        ctx.align_batch(A.Scheme("global", "affine", 2, -1, -1, 1), q[:4], qo[:2], s[:4], so[:2])
    assert e.value.status_name == "E_INVALID"
    q, qo = csr([b"ACGTACGT", b"AAAA"])
    s, so = csr([b"TTTT", b"CCCCCC"])
    with pytest.raises(A.AnyseqError) as e:
        ctx.traceback(A.Scheme("global"), q, qo, s, so, cigar_capacity=1)
    assert e.value.status_name == "E_CAPACITY" and e.value.cigar_used > 1


def test_device_api_matches_oracle(ctx):
    """anyseq_align_batch_device on torch device tensors, on the caller's stream."""
    import torch
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    q, qo, s, so = random_pairs(400, 0, 300, seed=77)
    dev = torch.device("cuda", 0)
    d_q = torch.from_numpy(q).to(dev)
    d_s = torch.from_numpy(s).to(dev)
    d_qo = torch.from_numpy(qo.view(np.int64)).to(dev)
    d_so = torch.from_numpy(so.view(np.int64)).to(dev)
    B = len(qo) - 1
    for kind in KINDS:
        sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
        res, _ = _oracle(kind, "affine", 5, 1, q, qo, s, so, tb=False)
        d_sc = torch.empty(B, dtype=torch.int32, device=dev)
        d_ends = torch.empty(B * A.ALIGNMENT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            ctx.align_batch_device(sch, d_q, d_qo, d_s, d_so, d_sc, d_ends, stream=stream)
        stream.synchronize()
        assert np.array_equal(d_sc.cpu().numpy(), res["score"].astype(np.int32))
        ends = d_ends.cpu().numpy().view(A.ALIGNMENT_DTYPE)
        assert np.array_equal(ends["q_end"], res["q_end"]) and np.array_equal(ends["s_end"], res["s_end"])


def test_host_chunking_and_tb_scratch_chunks(ctx):
    """Tiny upload chunks (host pipeline) and tiny traceback scratch (several fill/walk
    chunks per variant) give the same results."""
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    q, qo, s, so = random_pairs(700, 0, 260, seed=78)
    res, ocig = _oracle("local", "affine", 5, 1, q, qo, s, so, tb=True)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    ctx.set_option("chunk_bytes", 1 << 16)
    ctx.set_option("tb_scratch_bytes", 1 << 20)
    try:
        _check_scores(ctx, sch, q, qo, s, so, res)
        _check_tb(ctx, sch, q, qo, s, so, res, ocig)
    finally:
        ctx.set_option("chunk_bytes", 64 << 20)
        ctx.set_option("tb_scratch_bytes", 16 << 30)


def test_host_pipeline_many_chunks_pinned_outputs(ctx):
    """Many upload chunks (4 KB), pinned and pageable outputs, cigar written straight into a
    caller buffer across chunks, and the capacity error when that buffer is one word short."""
    import torch
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    q, qo, s, so = random_pairs(900, 0, 200, seed=81)
    res, ocig = _oracle("semi", "affine", 5, 1, q, qo, s, so, tb=True)
    sch = A.Scheme("semi", "affine", 2, -1, 5, 1)
    pin = lambda a: torch.from_numpy(a.view(np.uint8)).pin_memory().numpy().view(a.dtype)
    B = len(qo) - 1
    ctx.set_option("chunk_bytes", 1 << 12)
    try:
        _check_scores(ctx, sch, q, qo, s, so, res)
        _check_tb(ctx, sch, q, qo, s, so, res, ocig)
        out = pin(np.full(B, -7, np.int32))
        ctx.align_batch(sch, pin(q), pin(qo), pin(s), pin(so), out=out)
        assert np.array_equal(out, res["score"].astype(np.int32))
        aln, cig = ctx.traceback(sch, q, qo, s, so)
        paln = pin(np.zeros(B, A.ALIGNMENT_DTYPE))
        pcig = pin(np.zeros(len(cig) + 5, np.uint32))
        aln2, cig2 = ctx.traceback(sch, pin(q), pin(qo), pin(s), pin(so), out_aln=paln,
                                   out_cigar=pcig)
        assert np.array_equal(aln2, aln) and np.array_equal(cig2, cig)
        with pytest.raises(A.AnyseqError) as e:
            ctx.traceback(sch, q, qo, s, so, out_cigar=np.zeros(len(cig) - 1, np.uint32))
        assert e.value.status_name == "E_CAPACITY" and e.value.cigar_used == len(cig)
    finally:
        ctx.set_option("chunk_bytes", 64 << 20)


def _multi_devices():
    """Every visible GPU, or -- on a one-GPU box -- GPU 0 listed three times: the context's
    G-device code (cell-balanced shards, one host thread, stream set and scratch per entry,
    per-shard result gather and CIGAR rebasing) then runs for real on one B200 (the shards
    are independent, so their kernels never wait on each other)."""
    import torch
    n = torch.cuda.device_count()
    return list(range(n)) if n >= 2 else [0, 0, 0]


@pytest.mark.parametrize("devices", ["all", "dup"])
def test_multi_device_context(devices):
    """A context over several devices shards the batch by cells; identical results."""
    import torch
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    devs = _multi_devices() if devices == "all" else [0, 0]
    q, qo, s, so = random_pairs(500, 0, 300, seed=79)
    with A.Context(devs) as c:
        for kind in KINDS:
            sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
            res, ocig = _oracle(kind, "affine", 5, 1, q, qo, s, so, tb=True)
            _check_scores(c, sch, q, qo, s, so, res)
            _check_tb(c, sch, q, qo, s, so, res, ocig)


def test_c5_one_percent_of_1m_mixed():
    """C5 at scale: a 1,000,000-pair mixed-length batch (100..1000 bp),
    every kind x both modes on the GPU over the WHOLE batch in one call each, checked against
    the oracle on a fixed 1 % sample (10,000 pairs): score, begin and end cells and CIGAR
    bit-exact; every other pair's CIGAR must span exactly its begin -> end cells."""
    import paper_2002_04561_b200 as A
    from oracle import oracle as O
    from synth import c5_mixed_large, csr
    q, qo, s, so = c5_mixed_large(1_000_000, seed=55)
    B = len(qo) - 1
    idx = np.sort(np.random.default_rng(5).choice(B, B // 100, replace=False))
    sq = csr([q[qo[k]:qo[k + 1]].tobytes() for k in idx])
    ss = csr([s[so[k]:so[k + 1]].tobytes() for k in idx])
    with A.Context([0]) as c:
        for kind in KINDS:
            sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
            res, ocig = _oracle(kind, "affine", 5, 1, sq[0], sq[1], ss[0], ss[1], tb=True)
            sc, ends = c.align_batch(sch, q, qo, s, so, ends=True)
            assert np.array_equal(sc[idx], res["score"].astype(np.int32)), kind
            assert np.array_equal(ends["q_end"][idx], res["q_end"]), kind
            assert np.array_equal(ends["s_end"][idx], res["s_end"]), kind
            aln, words = c.traceback(sch, q, qo, s, so, cigar_capacity=24 * B)
            assert np.array_equal(aln["score"], sc), kind
            for f in ("q_begin", "s_begin", "q_end", "s_end"):
                assert np.array_equal(aln[f][idx], res[f]), (kind, f)
            got = A.cigars_of(aln[idx], words)
            bad = [k for k in range(len(idx)) if got[k] != ocig[k]]
            assert not bad, (kind, bad[:5])
            # span property for all pairs: M+I = q extent, M+D = s extent
            cl = aln["cigar_len"].astype(np.uint64)
            assert np.array_equal(aln["cigar_offset"], np.cumsum(cl) - cl), kind
            w = words.astype(np.int64)
            ln, op = w >> 4, w & 15
            pair = np.repeat(np.arange(B), aln["cigar_len"].astype(np.int64))
            qspan = np.bincount(pair, weights=ln * (op != 2), minlength=B)
            sspan = np.bincount(pair, weights=ln * (op != 1), minlength=B)
            assert np.array_equal(qspan.astype(np.int64), aln["q_end"] - aln["q_begin"]), kind
            assert np.array_equal(sspan.astype(np.int64), aln["s_end"] - aln["s_begin"]), kind


def test_pack2_mixed_chunks(ctx):
    """The host API's 2-bit upload (a1): ACGT-only chunks (upper and lower case) go up as
    2-bit codes, chunks with an N -- or a bad byte -- take the byte path.  With small
    chunks the same batch mixes both; scores, ends and CIGARs equal the oracle's and the
    byte-path-only run (option pack2 = 0); a bad byte is still reported with its pair."""
    import paper_2002_04561_b200 as A
    from synth import random_pairs, csr
    q, qo, s, so = random_pairs(1200, 0, 300, seed=90, lower_frac=0.3)
    q = q.copy()
    # an N in pair 700's query and in pair 1100's subject: their chunks take the byte path
    for arr, off, k in ((q, qo, 700), (s, so, 1100)):
        if off[k + 1] > off[k]:
            arr[int(off[k])] = ord("N")
    res, ocig = _oracle("local", "affine", 5, 1, q, qo, s, so, tb=True)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    ctx.set_option("chunk_bytes", 1 << 16)
    try:
        for p2 in (1, 0):
            ctx.set_option("pack2", p2)
            _check_scores(ctx, sch, q, qo, s, so, res)
            _check_tb(ctx, sch, q, qo, s, so, res, ocig)
        ctx.set_option("pack2", 1)
        bad = q.copy()
        bad[int(qo[900]) + 1 if qo[901] - qo[900] > 1 else int(qo[901])] = ord("x")
        with pytest.raises(A.AnyseqError) as e:
            ctx.align_batch(sch, bad, qo, s, so)
        assert e.value.status_name == "E_BADSEQ"
    finally:
        ctx.set_option("pack2", 1)
        ctx.set_option("chunk_bytes", 64 << 20)


def test_pack2_all_lengths(ctx):
    """2-bit upload edge cases: every length 0..70 (partial last code byte, chunk ends
    mid-byte) in one uniform-free batch, global linear, against the oracle."""
    import paper_2002_04561_b200 as A
    from synth import csr
    rng = np.random.default_rng(3)
    qs = [rng.choice(list(b"ACGTacgt"), size=L).astype(np.uint8).tobytes() for L in range(71)]
    ss = [rng.choice(list(b"ACGT"), size=(L * 7) % 71).astype(np.uint8).tobytes()
          for L in range(71)]
    q, qo = csr(qs)
    s, so = csr(ss)
    res, ocig = _oracle("global", "linear", 0, 1, q, qo, s, so, tb=True)
    sch = A.Scheme("global", "linear", 2, -1, 0, 1)
    for cb in (1 << 12, 64 << 20):
        ctx.set_option("chunk_bytes", cb)
        try:
            _check_scores(ctx, sch, q, qo, s, so, res)
            _check_tb(ctx, sch, q, qo, s, so, res, ocig)
        finally:
            ctx.set_option("chunk_bytes", 64 << 20)


@pytest.mark.parametrize("kind", KINDS)
def test_tb8_low_byte_store(ctx, kind):
    """Traceback H store in low bytes: identical alignments to the full
    store and to the oracle, for s16x2 and s32 slots; a scheme whose neighbour differences
    can reach 128 (open 60 / extend 10) keeps the full store and is still exact."""
    import paper_2002_04561_b200 as A
    from synth import random_pairs
    q, qo, s, so = random_pairs(400, 0, 360, seed=91)
    for go, ge in ((5, 1), (60, 10)):
        res, ocig = _oracle(kind, "affine", go, ge, q, qo, s, so, tb=True)
        sch = A.Scheme(kind, "affine", 2, -1, go, ge)
        for allow16 in (1, 0):
            ctx.set_option("allow16", allow16)
            try:
                for tb8 in (1, 0):
                    ctx.set_option("tb8", tb8)
                    _check_tb(ctx, sch, q, qo, s, so, res, ocig)
            finally:
                ctx.set_option("tb8", 1)
                ctx.set_option("allow16", 1)


@pytest.mark.parametrize("kind", KINDS)
def test_mixed_batch_routes_long_pairs(ctx, kind):
    """Mixed batch (host-side form): pairs at or above batch_long_cells go
    to the long-pair path; scores, cells and CIGARs of every pair still equal the oracle's,
    in pair order, with cigar offsets contiguous."""
    import paper_2002_04561_b200 as A
    from synth import random_pairs, c4_genomes, csr
    q0, qo0, s0, so0 = random_pairs(40, 0, 300, seed=92)
    g1, g2 = c4_genomes(6000, "a", seed=93)
    qs = [q0[qo0[k]:qo0[k + 1]].tobytes() for k in range(40)]
    ss = [s0[so0[k]:so0[k + 1]].tobytes() for k in range(40)]
    for pos, (a, b) in ((3, (g1[:2500], g2[:2600])), (17, (g1[3000:5600], g2[3000:5500])),
                        (39, (g2[:2100], g1[:3000]))):
        qs.insert(pos, a)
        ss.insert(pos, b)
    q, qo = csr(qs)
    s, so = csr(ss)
    res, ocig = _oracle(kind, "affine", 5, 1, q, qo, s, so, tb=True)
    sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
    ctx.set_option("batch_long_cells", 1 << 22)
    ctx.set_option("batch_long_cells_tb", 1 << 22)
    try:
        _check_scores(ctx, sch, q, qo, s, so, res)
        _check_tb(ctx, sch, q, qo, s, so, res, ocig)
        aln, words = ctx.traceback(sch, q, qo, s, so)
        cl = aln["cigar_len"].astype(np.uint64)
        assert np.array_equal(aln["cigar_offset"], np.cumsum(cl) - cl)
    finally:
        ctx.set_option("batch_long_cells", 1 << 22)
        ctx.set_option("batch_long_cells_tb", 1 << 22)


@pytest.mark.parametrize("kind", ["global", "semi", "local"])
@pytest.mark.parametrize("gap,go", [("linear", 0), ("affine", 5)])
def test_small_batch_takes_long_path(ctx, kind, gap, go):
    """Batches of at most batch_long_small pairs send ACGT-only pairs with both sides >= 256
    to the long-pair path (one pair spread over many warps); the pair whose subject holds an
    N and the short pair stay on the batch kernel.  Scores, end/begin cells and CIGARs equal
    the oracle's either way."""
    import paper_2002_04561_b200 as A
    from synth import c4_genomes, csr
    g1, g2 = c4_genomes(4000, "a", seed=94)
    sN = bytearray(g2[1000:1700])
    sN[350] = ord("N")
    qs = [g1[:1000], g1[1000:1650], b"ACGTTGCA"]
    ss = [g2[:1050], bytes(sN), b"ACGTAGCA"]
    q, qo = csr(qs)
    s, so = csr(ss)
    res, ocig = _oracle(kind, gap, go, 1, q, qo, s, so, tb=True)
    sch = A.Scheme(kind, gap, 2, -1, go, 1)
    for small in (4, 0):  # long path (and fallback) vs the batch kernel alone
        ctx.set_option("batch_long_small", small)
        try:
            _check_scores(ctx, sch, q, qo, s, so, res)
            _check_tb(ctx, sch, q, qo, s, so, res, ocig)
        finally:
            ctx.set_option("batch_long_small", 4)
