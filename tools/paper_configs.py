"""The paper's own benchmark schemes (Fig. 5): GLOBAL alignment with
linear (+2/-1, gap 1) and affine (G_o = 2, G_e = 1) gaps, score-only and traceback, on
1M x 150 bp read pairs (C2 shape) and a long pair -- measured here to set beside the
paper's Titan V numbers (context, not targets).  Page-locked buffers as in bench.py e2e;
device time from the library's CUDA-event instrumentation."""
import json, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2002_04561_b200 as A, synth


def pin(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).pin_memory().numpy().view(a.dtype)


def timed(ctx, fn, reps=3):
    fn()
    ctx.set_option("timing", 1)
    ctx.reset_stats()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    wall = (time.perf_counter() - t0) / reps
    fill = ctx.stat("fill_ms") / reps
    walk = ctx.stat("walk_ms") / reps
    ctx.set_option("timing", 0)
    return wall, fill, walk


ctx = A.Context([0])
qm, sm = synth.c2_reads(1_000_000, seed=2)
q, qo = synth.uniform_csr(qm); s, so = synth.uniform_csr(sm)
q, qo, s, so = pin(q), pin(qo), pin(s), pin(so)
B = len(qo) - 1
out = pin(np.zeros(B, np.int32))
paln = pin(np.zeros(B, A.ALIGNMENT_DTYPE))
pcig = pin(np.zeros(16 * B, np.uint32))
cells = B * 150.0 * 150.0
for name, sch in (("linear 2/-1/-1", A.Scheme("global", "linear", 2, -1, 0, 1)),
                  ("affine 2/-1, Go=2 Ge=1", A.Scheme("global", "affine", 2, -1, 2, 1))):
    w, f, _ = timed(ctx, lambda: ctx.align_batch(sch, q, qo, s, so, out=out))
    print(json.dumps({"config": f"1M x 150 bp global {name} score-only", "fill_gcups": cells / f / 1e6,
                      "e2e_gcups": cells / w / 1e9}), flush=True)
    w, f, k = timed(ctx, lambda: ctx.traceback(sch, q, qo, s, so, out_aln=paln, out_cigar=pcig), 2)
    print(json.dumps({"config": f"1M x 150 bp global {name} traceback", "fill_walk_gcups": cells / (f + k) / 1e6,
                      "e2e_gcups": cells / w / 1e9}), flush=True)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
for name, sch in (("linear 2/-1/-1", A.Scheme("global", "linear", 2, -1, 0, 1)),
                  ("affine 2/-1, Go=2 Ge=1", A.Scheme("global", "affine", 2, -1, 2, 1))):
    ctx.align_long(sch, g1[:100000], g2[:100000])
    t0 = time.perf_counter(); r = ctx.align_long(sch, g1, g2); w = time.perf_counter() - t0
    kms = ctx.stat("long_kernel_ms")
    print(json.dumps({"config": f"{n} bp pair global {name} score-only",
                      "gcups_kernel": len(g1) * len(g2) / kms / 1e6,
                      "gcups_wall": len(g1) * len(g2) / w / 1e9, "score": r["score"]}), flush=True)
# the paper's long-genome traceback panels (Fig. 5a), here on a 1 Mbp pair (checkpointed walk)
t1, t2 = g1[:1_000_000], g2[:1_000_000]
for name, sch in (("linear 2/-1/-1", A.Scheme("global", "linear", 2, -1, 0, 1)),
                  ("affine 2/-1, Go=2 Ge=1", A.Scheme("global", "affine", 2, -1, 2, 1))):
    ctx.traceback_long(sch, t1, t2)
    t0 = time.perf_counter(); r = ctx.traceback_long(sch, t1, t2); w = time.perf_counter() - t0
    print(json.dumps({"config": f"1 Mbp pair global {name} traceback", "gcups_wall": len(t1) * len(t2) / w / 1e9,
                      "pass_ms": ctx.stat("tb_pass_ms"), "walk_ms": ctx.stat("tb_walk_ms"),
                      "score": r["score"]}), flush=True)
