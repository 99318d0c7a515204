"""One long-pair call (C4 shape, local affine) with a given grid, for profiling.
usage: long_one.py [n] [blocks] [band_rows] [narrow]"""
import sys; sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = int(sys.argv[3]) if len(sys.argv) > 3 else 0
narrow = int(sys.argv[4]) if len(sys.argv) > 4 else 1
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
ctx.set_option("long_blocks", blocks)
ctx.set_option("long_band_rows", rows)
ctx.set_option("long_narrow", narrow)
print(ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2), ctx.stat("long_kernel_ms"))
