"""C4 (5 Mbp local affine) long16 kernel time vs the start slack (option long_start_lag) and
the poll back-off; also prints the in-kernel wait share (option long_profile)."""
import sys
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
lags = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 128, 256, 512]
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
for lag in lags:
    ctx.set_option("long_start_lag", lag)
    r = ctx.align_long(sch, g1, g2)
    ms = ctx.stat("long_kernel_ms")
    print(f"lag {lag}: {ms:.1f} ms  {n * len(g2) / ms / 1e9:.0f} GCUPS  {r}", flush=True)
ctx.set_option("long_profile", 1)
ctx.set_option("long_start_lag", 0)
ctx.align_long(sch, g1, g2)
