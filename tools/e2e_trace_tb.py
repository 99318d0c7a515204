"""One host-API C3 traceback call (1M x 150 bp local affine, CIGAR out) with the per-chunk
host timeline (option timing = 2), after warm-up; then the plain wall time of 3 calls."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np, torch  # noqa: E401,E402
import paper_2002_04561_b200 as A  # noqa: E402
from synth import c2_reads, uniform_csr  # noqa: E402
qm, sm = c2_reads(1_000_000, seed=2)
q, qo = uniform_csr(qm); s, so = uniform_csr(sm)
pin = lambda a: torch.from_numpy(a.view(np.uint8)).pin_memory().numpy().view(a.dtype)  # noqa: E731
pq, ps, pqo, pso = pin(q), pin(s), pin(qo), pin(so)
paln = pin(np.zeros(len(qo) - 1, A.ALIGNMENT_DTYPE))
pcig = pin(np.zeros(32 * (len(qo) - 1), np.uint32))
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
for k, v in (a.split("=") for a in sys.argv[1:]):
    ctx.set_option(k, int(v))
for _ in range(3):
    ctx.traceback(sch, pq, pqo, ps, pso, out_aln=paln, out_cigar=pcig)
t0 = time.perf_counter()
for _ in range(3):
    ctx.traceback(sch, pq, pqo, ps, pso, out_aln=paln, out_cigar=pcig)
print(f"wall {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms", flush=True)
ctx.set_option("timing", 2)
ctx.traceback(sch, pq, pqo, ps, pso, out_aln=paln, out_cigar=pcig)
print({k: round(ctx.stat(k), 3) for k in ("fill_ms", "walk_ms", "h2d_bytes", "d2h_bytes")}, flush=True)
