"""C4 shape (local affine 5/1, 2/-1): the s32 long kernel vs the 16-bit differential kernel
(8 and 16 registers per lane) on one GPU -- score, end cell, kernel time, GCUPS."""
import sys; sys.path.insert(0, '.')
import json
import paper_2002_04561_b200 as A, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
variant = sys.argv[2] if len(sys.argv) > 2 else "a"
g1, g2 = synth.c4_genomes(n, variant, seed=4)
ctx = A.Context([0])
sch = A.Scheme("local", "affine", 2, -1, 5, 1)
for narrow, rows in ((0, 0), (1, 512), (1, 768), (1, 0)):
    ctx.set_option("long_narrow", narrow)
    ctx.set_option("long_band_rows", rows)
    r = ctx.align_long(sch, g1, g2)
    ms = ctx.stat("long_kernel_ms")
    print(json.dumps({"n": n, "variant": variant, "narrow": int(ctx.stat("long_narrow")), "rows": rows,
                      "score": r["score"], "end": [r["q_end"], r["s_end"]], "kernel_ms": round(ms, 2),
                      "gcups": round(len(g1) * len(g2) / ms / 1e6, 1)}), flush=True)
