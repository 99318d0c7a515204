"""One C3 traceback call (1M x 150 bp, local affine) from page-locked buffers, for profiling."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2002_04561_b200 as A, synth
npairs = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
qm, sm = synth.c2_reads(npairs, seed=2)
q, qo = synth.uniform_csr(qm); s, so = synth.uniform_csr(sm)
ctx = A.Context([0])
aln, cig = ctx.traceback(A.Scheme("local", "affine", 2, -1, 5, 1), q, qo, s, so)
print("pairs", npairs, "cigar words", len(cig), "score sum", int(aln["score"].sum()))
