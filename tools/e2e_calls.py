"""Per-call wall times of the C2 host-API call (defaults, pinned buffers), as bench.py's e2e
leg makes them; prints each call so outliers are visible."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np, torch  # noqa: E401,E402
import paper_2002_04561_b200 as A  # noqa: E402
from synth import c2_reads, uniform_csr  # noqa: E402
qm, sm = c2_reads(1_000_000, seed=2)
q, qo = uniform_csr(qm); s, so = uniform_csr(sm)
pq = torch.from_numpy(q).pin_memory().numpy()
ps = torch.from_numpy(s).pin_memory().numpy()
pqo = torch.from_numpy(qo.view(np.int64)).pin_memory().numpy().view(np.uint64)
pso = torch.from_numpy(so.view(np.int64)).pin_memory().numpy().view(np.uint64)
pout = torch.empty(len(qo) - 1, dtype=torch.int32).pin_memory().numpy()
ctx = A.Context([0])
sch = A.Scheme("semi", "affine", 2, -1, 5, 1)
for k, v in (a.split("=") for a in sys.argv[1:]):
    ctx.set_option(k, int(v))
cells = (len(qo) - 1) * 150 * 150
ts = []
for i in range(12):
    t0 = time.perf_counter()
    ctx.align_batch(sch, pq, pqo, ps, pso, out=pout)
    ts.append(time.perf_counter() - t0)
print(" ".join(f"{t*1e3:.2f}" for t in ts), flush=True)
print(f"mean(2:) {np.mean(ts[2:])*1e3:.2f} ms = {cells/np.mean(ts[2:])/1e9:.0f} GCUPS; min {min(ts)*1e3:.2f} ms", flush=True)
