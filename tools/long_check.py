"""Quick parity sweep of anyseq_align_long against the oracle's rolling score (debugging)."""
import sys
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A
from oracle import oracle as O
from synth import c4_genomes
ctx = A.Context([0])
bad = 0
for n, strips, rows in ((3000, 1, 0), (5000, 1, 0), (9000, 3, 512), (20000, 3, 512), (20000, 0, 0)):
    g1, g2 = c4_genomes(n, "a", seed=4)
    for kind, gap, go in (("local", "affine", 5), ("global", "affine", 5), ("semi", "linear", 0)):
        ctx.set_option("long_strips", strips)
        ctx.set_option("long_band_rows", rows)
        r = ctx.align_long(A.Scheme(kind, gap, 2, -1, go, 1), g1, g2)
        o = O.score_rolling(O.Scheme(kind, gap, 2, -1, go, 1), g1, g2)
        ok = (r["score"], r["q_end"], r["s_end"]) == (o.score, o.q_end, o.s_end)
        bad += not ok
        print(n, strips, rows, kind, gap, "OK" if ok else f"BAD got {r} want {(o.score, o.q_end, o.s_end)}", flush=True)
print("bad", bad)
