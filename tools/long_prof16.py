"""Wait share of the long kernels (in-kernel clock64 counters, option long_profile) at C4
shape: s32 and the 16-bit kernel (8 / 16 registers per lane)."""
import sys; sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
ctx.set_option("long_profile", 1)
for narrow, rows in ((0, 0), (1, 512), (1, 0)):
    ctx.set_option("long_narrow", narrow)
    ctx.set_option("long_band_rows", rows)
    r = ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2)
    print(narrow, rows, r, ctx.stat("long_kernel_ms"), flush=True)
