"""C4 (5 Mbp x 5 Mbp, variant a, local affine 5/1) long-kernel time for several values of
one context option.  usage: long_opt_sweep.py OPTION v1,v2,... [n]"""
import sys
sys.path.insert(0, '.')
import paper_2002_04561_b200 as A  # noqa: E402
import synth  # noqa: E402
opt = sys.argv[1]
vals = [int(x) for x in sys.argv[2].split(",")]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 5_000_000
g1, g2 = synth.c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
for v in vals:
    ctx.set_option(opt, v)
    r = ctx.align_long(sch, g1, g2)
    ms = ctx.stat("long_kernel_ms")
    print(f"{opt}={v}: {ms:.1f} ms {len(g1) * len(g2) / ms / 1e6:.0f} GCUPS score {r['score']}", flush=True)
