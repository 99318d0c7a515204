"""C3 (1M x 150 bp local affine traceback) with and without the fused walk, pinned buffers."""
import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2002_04561_b200 as A, synth
from oracle import oracle as O
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).pin_memory().numpy().view(a.dtype)
qm, sm = synth.c2_reads(1_000_000, seed=2)
q, qo = synth.uniform_csr(qm); s, so = synth.uniform_csr(sm)
q, qo, s, so = pin(q), pin(qo), pin(s), pin(so)
B = len(qo) - 1
paln = pin(np.zeros(B, A.ALIGNMENT_DTYPE)); pcig = pin(np.zeros(32 * B, np.uint32))
ctx = A.Context([0]); sch = A.Scheme("local", "affine", 2, -1, 5, 1)
ref = None
for fused in (1, 0, 1, 0):
    ctx.set_option("tb_fused_walk", fused)
    ctx.traceback(sch, q, qo, s, so, out_aln=paln, out_cigar=pcig)
    t0 = time.perf_counter()
    aln, cig = ctx.traceback(sch, q, qo, s, so, out_aln=paln, out_cigar=pcig)
    dt = time.perf_counter() - t0
    cur = (aln.copy(), cig.copy())
    same = ref is None or (np.array_equal(cur[0], ref[0]) and np.array_equal(cur[1], ref[1]))
    ref = ref or cur
    print("fused", fused, "ms", round(dt * 1e3, 2), "gcups", round(22.5e9 / dt / 1e9, 1), "same", same, flush=True)
