"""C4-style long pair: GCUPS versus the persistent grid size (warps = 4 x blocks); best of 2."""
import sys, time; sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
ctx.align_long(sch, g1[:200000], g2[:200000])
for blocks in [int(x) for x in sys.argv[2].split(",")]:
    ctx.set_option("long_blocks", blocks)
    best = 1e9
    for _ in range(2):
        t0 = time.perf_counter(); r = ctx.align_long(sch, g1, g2); best = min(best, time.perf_counter() - t0)
    print("n", n, "blocks", blocks, "s", round(best, 3), "gcups", round(len(g1) * len(g2) / best / 1e9, 1), r, flush=True)
