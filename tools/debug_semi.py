import sys, numpy as np
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A
from oracle import oracle as O
from synth import csr, iid
ctx = A.Context([0])
for v in (3, 0):
    for n, m in ((5, 5), (8, 8), (20, 17), (64, 64), (70, 70), (130, 40), (10, 100)):
        q, qo = csr([iid(n, n)]); s, so = csr([iid(m, m + 7)])
        ctx.set_option("force_variant", v)
        sc, aln = ctx.align_batch(A.Scheme("semi", "linear", 2, -1, 0, 1), q, qo, s, so, ends=True)
        sc2 = ctx.align_batch(A.Scheme("semi", "linear", 2, -1, 0, 1), q, qo, s, so)
        r = O.align(O.Scheme("semi", "linear", 2, -1, 0, 1), q.tobytes(), s.tobytes())
        print(v, n, m, "gpu", sc[0], sc2[0], aln["q_end"][0], aln["s_end"][0], "orc", r.score, r.q_end, r.s_end)
