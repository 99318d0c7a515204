import sys; sys.path.insert(0,'.')
import paper_2002_04561_b200 as A, synth
g1, g2 = synth.c4_genomes(1_000_000, "a", seed=4)
ctx = A.Context([0])
for kind, gap, go in (("global","linear",0), ("local","affine",5)):
    sch = A.Scheme(kind, gap, 2, -1, go, 1)
    for rep in range(2):
        r = ctx.align_long(sch, g1, g2); ms = ctx.stat("long_kernel_ms")
        t = ctx.traceback_long(sch, g1, g2)
        print(kind, gap, "score-only kernel", round(ms,1), "ms; tb pass", round(ctx.stat("tb_pass_ms"),1), "walk", round(ctx.stat("tb_walk_ms"),1), "ckpt GB", round(ctx.stat("tb_ckpt_bytes")/1e9,1), flush=True)
ctx.set_option("long_profile", 1)
ctx.align_long(A.Scheme("global","linear",2,-1,0,1), g1, g2)
ctx.traceback_long(A.Scheme("global","linear",2,-1,0,1), g1, g2)
