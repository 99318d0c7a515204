import sys, os, time, json
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
for lag, chunk in ((64, 32), (96, 32), (160, 32), (96, 64)):
    ctx.set_option("long_start_lag", lag); ctx.set_option("long_chunk_cols", chunk)
    t0 = time.perf_counter(); r = ctx.align_long(sch, g1, g2); dt = time.perf_counter() - t0
    print(json.dumps({"n": n, "lag": lag, "chunk": chunk, "s": round(dt, 3), "gcups": round(len(g1) * len(g2) / dt / 1e9, 1), "r": r}), flush=True)
