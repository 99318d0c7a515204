"""Small runs of every kernel family for compute-sanitizer (one tool per invocation):
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize.py
batch fill (s16x2 and s32, score and traceback, every kind), long-pair kernels (16-bit with
virtual strips, 32-bit), the checkpointed long traceback and its walk, the Hirschberg
fallback (lastrow passes).  Results are checked against the oracle so a silent corruption
also fails."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2002_04561_b200 as A
from oracle import oracle as O
from synth import random_pairs, c4_genomes

ctx = A.Context([0])
q, qo, s, so = random_pairs(96, 0, 200, seed=5)
for kind in ("global", "local", "semi"):
    for allow16 in (1, 0):
        ctx.set_option("allow16", allow16)
        sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
        res, cig = O.batch(O.Scheme(kind, "affine", 2, -1, 5, 1), q, qo, s, so, traceback=True)
        sc = ctx.align_batch(sch, q, qo, s, so)
        assert np.array_equal(sc, res["score"].astype(np.int32)), (kind, allow16)
        aln, words = ctx.traceback(sch, q, qo, s, so)
        assert np.array_equal(aln["score"], res["score"].astype(np.int32)), (kind, allow16)
ctx.set_option("allow16", 1)
g1, g2 = c4_genomes(2500, "a", seed=4)
for kind, gap, go in (("local", "affine", 5), ("semi", "linear", 0), ("global", "affine", 5)):
    o = O.score_rolling(O.Scheme(kind, gap, 2, -1, go, 1), g1, g2)
    for narrow, strips in ((1, 3), (0, 2)):
        ctx.set_option("long_narrow", narrow)
        ctx.set_option("long_strips", strips)
        ctx.set_option("long_band_rows", 512)
        r = ctx.align_long(A.Scheme(kind, gap, 2, -1, go, 1), g1, g2)
        assert (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end), (kind, narrow)
    ctx.set_option("long_narrow", 1)
    ctx.set_option("long_strips", 0)
    ctx.set_option("tb_kc_shift", 8)
    t = ctx.traceback_long(A.Scheme(kind, gap, 2, -1, go, 1), g1, g2)
    oa = O.align(O.Scheme(kind, gap, 2, -1, go, 1), g1, g2)
    assert t["cigar"] == oa.cigar, kind
    ctx.set_option("tb_kc_shift", 0)
    ctx.set_option("long_band_rows", 0)
gn = bytearray(g2)
gn[100] = ord("N")
t = ctx.traceback_long(A.Scheme("global", "linear", 2, -1, 0, 1), g1, bytes(gn))
assert ctx.stat("tb_method") == 2
print("sanitize workload ok")
