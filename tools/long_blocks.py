"""C4-style long pair: GCUPS versus the persistent grid size (warps = 4 x blocks)."""
import sys, time; sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
ctx.align_long(sch, g1[:100000], g2[:100000])
for blocks in [int(x) for x in sys.argv[2].split(",")]:
    ctx.set_option("long_blocks", blocks)
    t0 = time.perf_counter(); r = ctx.align_long(sch, g1, g2); dt = time.perf_counter() - t0
    print("blocks", blocks, "s", round(dt, 3), "gcups", round(len(g1) * len(g2) / dt / 1e9, 1), r, flush=True)
