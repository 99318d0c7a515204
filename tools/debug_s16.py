import sys, numpy as np
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A
from oracle import oracle as O
from synth import csr, iid, random_pairs
ctx = A.Context([0])
def run(kind, gap, go, qs, ss, variant):
    q, qo = csr(qs); s, so = csr(ss)
    ctx.set_option("force_variant", variant)
    sc, aln = ctx.align_batch(A.Scheme(kind, gap, 2, -1, go, 1), q, qo, s, so, ends=True)
    sc2 = ctx.align_batch(A.Scheme(kind, gap, 2, -1, go, 1), q, qo, s, so)
    res, _ = O.batch(O.Scheme(kind, gap, 2, -1, go, 1), q, qo, s, so)
    for k in range(len(qs)):
        print(kind, gap, variant, len(qs[k]), len(ss[k]), "gpu", sc[k], sc2[k], aln["q_end"][k], aln["s_end"][k], "orc", res["score"][k], res["q_end"][k], res["s_end"][k])
for v in (0, 3):
    for kind in ("local", "semi", "global"):
        qs = [iid(n, n) for n in (5, 8, 20, 64, 70)] + [b"ACGT", b"GGGACGTGGG"]
        ss = [iid(m, m + 7) for m in (5, 8, 20, 64, 70)] + [b"ACGT", b"ACGT"]
        run(kind, "linear", 0, qs, ss, v)
