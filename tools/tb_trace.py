import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2002_04561_b200 as A
from synth import c2_reads, uniform_csr
qm, sm = c2_reads(1_000_000, seed=2)
q, qo = uniform_csr(qm); s, so = uniform_csr(sm)
pin = lambda a: torch.from_numpy(a.view(np.uint8)).pin_memory().numpy().view(a.dtype)
pq, ps, pqo, pso = pin(q), pin(s), pin(qo), pin(so)
B = len(qo) - 1
paln = pin(np.zeros(B, A.ALIGNMENT_DTYPE)); pcig = pin(np.zeros(8 * B, np.uint32))
ctx = A.Context([0]); sch = A.Scheme("local", "affine", 2, -1, 5, 1)
ref_aln, ref_cig = ctx.traceback(sch, q, qo, s, so)
for label, args, kw in (("pageable", (q, qo, s, so), {}), ("pinned", (pq, pqo, ps, pso), {"out_aln": paln, "out_cigar": pcig})):
    for rep in range(2):
        t0 = time.perf_counter(); aln, cig = ctx.traceback(sch, *args, **kw); dt = time.perf_counter() - t0
        print(label, "tb wall ms", round(dt * 1e3, 2), "gcups", round(22.5e9 / dt / 1e9, 1), "cigar words", len(cig),
              "same", bool(np.array_equal(aln, ref_aln) and np.array_equal(cig, ref_cig)), flush=True)
ctx.set_option("timing", 2)
t0 = time.perf_counter(); ctx.traceback(sch, pq, pqo, ps, pso, out_aln=paln, out_cigar=pcig); dt = time.perf_counter() - t0
print("traced wall", round(dt * 1e3, 2), flush=True)
