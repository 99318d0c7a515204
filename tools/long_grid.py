"""C4-style long pair: GCUPS over virtual column strips (task granularity) and grid size."""
import sys, time; sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
ref = None
for strips in [int(x) for x in sys.argv[2].split(",")]:
    ctx.set_option("long_strips", strips)
    t0 = time.perf_counter(); r = ctx.align_long(sch, g1, g2); dt = time.perf_counter() - t0
    ref = ref or r
    print("strips", strips, "s", round(dt, 3), "gcups", round(len(g1) * len(g2) / dt / 1e9, 1), r == ref, flush=True)
