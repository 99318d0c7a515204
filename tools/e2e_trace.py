"""One host-API C2 call with the per-chunk host timeline (option timing = 2; device
events are skipped unless argv[2] == 'dev')."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2002_04561_b200 as A
from synth import c2_reads, uniform_csr
qm, sm = c2_reads(1_000_000, seed=2)
q, qo = uniform_csr(qm); s, so = uniform_csr(sm)
pin = lambda a: torch.from_numpy(a.view(np.uint8)).pin_memory().numpy().view(a.dtype)
pq, ps, pqo, pso = pin(q), pin(s), pin(qo), pin(so)
out = pin(np.zeros(len(qo) - 1, np.int32))
ctx = A.Context([0])
sch = A.Scheme("semi", "affine", 2, -1, 5, 1)
p2 = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx.set_option("pack2", p2)
for _ in range(3):
    ctx.align_batch(sch, pq, pqo, ps, pso, out=out)
ctx.set_option("timing", 2)
ctx.align_batch(sch, pq, pqo, ps, pso, out=out)
