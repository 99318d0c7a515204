"""C4-shape long16 time vs the persistent grid size (blocks of 4 warps): latency- or
throughput-bound?  Prints kernel time, GCUPS and the in-kernel wait shares."""
import sys
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
ctx.set_option("long_profile", 1)
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
for blocks in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "148,296,444").split(",")]:
    ctx.set_option("long_blocks", blocks)
    r = ctx.align_long(sch, g1, g2)
    ms = ctx.stat("long_kernel_ms")
    print(f"blocks {blocks}: {ms:.1f} ms  {n * len(g2) / ms / 1e9:.0f} GCUPS", flush=True)
