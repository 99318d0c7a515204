"""e2e probe: host API C2 time with pack2 on/off and several chunk sizes (pinned buffers)."""
import sys, time
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
cells = (len(qo) - 1) * 150 * 150
for p2, pct in ((0, 0), (1, 100), (1, 40), (1, 50), (1, 60), (1, 70)):
    for cb in (16 << 20, 32 << 20, 64 << 20):
        ctx.set_option("pack2", p2); ctx.set_option("pack2_percent", pct); ctx.set_option("chunk_bytes", cb)
        ctx.align_batch(sch, pq, pqo, ps, pso, out=out)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); ctx.align_batch(sch, pq, pqo, ps, pso, out=out); ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"pack2={p2} pct={pct} chunk={cb>>20}MB: {t*1e3:.2f} ms  {cells/t/1e9:.0f} GCUPS", flush=True)
