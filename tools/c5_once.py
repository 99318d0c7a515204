"""One C5 score-only call (mixed 100-1000 bp, local affine) for profiling."""
import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2002_04561_b200 as A, synth
npairs = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000
kind = sys.argv[2] if len(sys.argv) > 2 else "local"
q, qo, s, so = synth.c5_mixed(npairs, seed=5)
ctx = A.Context([0])
sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
ctx.align_batch(sch, q, qo, s, so)
sc = ctx.align_batch(sch, q, qo, s, so)
n = np.diff(qo); m = np.diff(so)
print("pairs", npairs, "n range", n.min(), n.max(), "cells", float((n * m.astype(np.float64)).sum()), "checksum", int(sc.sum()))
