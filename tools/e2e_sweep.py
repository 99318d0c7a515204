import sys, time, json; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2002_04561_b200 as A
from synth import c2_reads, uniform_csr
qm, sm = c2_reads(1_000_000, seed=2)
q, qo = uniform_csr(qm); s, so = uniform_csr(sm)
pq = torch.from_numpy(q).pin_memory().numpy(); ps = torch.from_numpy(s).pin_memory().numpy()
pqo = torch.from_numpy(qo.view(np.int64)).pin_memory().numpy().view(np.uint64)
pso = torch.from_numpy(so.view(np.int64)).pin_memory().numpy().view(np.uint64)
ctx = A.Context([0]); sch = A.Scheme("semi", "affine", 2, -1, 5, 1)
out = torch.empty(len(qo) - 1, dtype=torch.int32).pin_memory().numpy()
# raw H2D bandwidth
d = torch.empty(len(pq), dtype=torch.uint8, device="cuda")
tq = torch.from_numpy(pq)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(3): d.copy_(tq, non_blocking=True)
torch.cuda.synchronize(); print("raw H2D GB/s", round(3 * len(pq) / (time.perf_counter() - t0) / 1e9, 1))
for cb in (48, 64, 96, 128, 192):
    ctx.set_option("chunk_bytes", cb << 20)
    ctx.align_batch(sch, pq, pqo, ps, pso, out=out)
    t0 = time.perf_counter()
    for _ in range(3): ctx.align_batch(sch, pq, pqo, ps, pso, out=out)
    dt = (time.perf_counter() - t0) / 3
    print(json.dumps({"chunk_MB": cb, "ms": round(dt * 1e3, 2), "gcups": round(22.5e9 / dt / 1e9, 1)}), flush=True)
ctx.set_option("timing", 1); ctx.reset_stats()
ctx.set_option("chunk_bytes", 64 << 20)
t0 = time.perf_counter(); ctx.align_batch(sch, pq, pqo, ps, pso, out=out); dt = time.perf_counter() - t0
print("fill ms inside e2e call", round(ctx.stat("fill_ms"), 2), "wall", round(dt * 1e3, 2))
ctx.set_option("timing", 2)
t0 = time.perf_counter(); ctx.align_batch(sch, pq, pqo, ps, pso, out=out); dt = time.perf_counter() - t0
print("traced wall", round(dt * 1e3, 2), flush=True)
