"""C4 shape, 16-bit long kernel: row hand-off poll back-off sweep (kernel ms, GCUPS)."""
import sys; sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
for ns in (64, 0, 16, 32, 128, 256):
    ctx.set_option("long_sleep_ns", ns)
    r = ctx.align_long(A.Scheme("local", "affine", 2, -1, 5, 1), g1, g2)
    ms = ctx.stat("long_kernel_ms")
    print(ns, r["score"], round(ms, 1), round(n * len(g2) / ms / 1e6, 1), flush=True)
