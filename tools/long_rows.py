"""Long kernel: rows per lane 12 vs 16 (option long_band_rows 384 / 512), C4 shape, best of 2."""
import sys, time; sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
ctx.align_long(sch, g1[:200000], g2[:200000])
for rows in (384, 512, 384, 512):
    ctx.set_option("long_band_rows", rows)
    t0 = time.perf_counter(); r = ctx.align_long(sch, g1, g2); dt = time.perf_counter() - t0
    print("rows", rows, "s", round(dt, 3), "gcups", round(len(g1) * len(g2) / dt / 1e9, 1), r, flush=True)
