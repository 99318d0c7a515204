import sys, time; sys.path.insert(0,'.')
import numpy as np
import paper_2002_04561_b200 as A, synth
from oracle import oracle as O
a, b = synth.c1_pair(1)
ctx = A.Context([0])
sch = A.Scheme("global", "linear", 2, -1, 0, 1)
for rep in range(4):
    t0 = time.perf_counter(); r = ctx.traceback_long(sch, a, b); w = time.perf_counter() - t0
    print("traceback_long", round(w*1e3, 3), "ms", ctx.stat("tb_method"), ctx.stat("tb_pass_ms"), ctx.stat("tb_walk_ms"))
q, qo = synth.csr([a]); s, so = synth.csr([b])
for rep in range(4):
    t0 = time.perf_counter(); aln, cig = ctx.traceback(sch, q, qo, s, so); w = time.perf_counter() - t0
    print("batch", round(w*1e3, 3), "ms")
o = O.align(O.Scheme("global", "linear", 2, -1, 0, 1), a, b)
print("long ok", r["score"] == o.score and r["cigar"] == o.cigar, "batch ok", A.cigars_of(aln, cig)[0] == o.cigar)
