"""One long-pair call on a rectangular window of the C4 genomes (n rows x m columns, local
affine 5/1), for profiling the long kernel's steady state at C4's strip count without
C4's run time.  usage: long_rect.py [n] [m] [blocks] [band_rows]"""
import sys
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A  # noqa: E402
import synth  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 500_000
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rows = int(sys.argv[4]) if len(sys.argv) > 4 else 0
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
ctx.set_option("long_blocks", blocks)
ctx.set_option("long_band_rows", rows)
r = ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2[:m])
print(r, ctx.stat("long_kernel_ms"), "GCUPS", n * m / ctx.stat("long_kernel_ms") / 1e6)
