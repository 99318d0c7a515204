"""One long16 call for source-level profiling: n bp (C4 variant a shape), 1024-row tasks,
a grid capped so that every resident warp has strips to run (long_blocks)."""
import sys
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_200_000
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 148
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
ctx.set_option("long_band_rows", 1024)
ctx.set_option("long_blocks", blocks)
r = ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2)
print(r, ctx.stat("long_kernel_ms"), n * len(g2) / ctx.stat("long_kernel_ms") / 1e9)
