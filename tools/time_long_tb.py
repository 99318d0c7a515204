"""Times the linear-space long-pair traceback (anyseq_traceback_long) on
mutated genome pairs (C4 variant a shape) and prints one JSON line per size: wall time of
the call, the matrix cells n*m and GCUPS = n*m / time (the paper's long-traceback metric,
Fig. 5a; Hirschberg relaxes about 2*n*m cells in its passes plus the leaves)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_04561_b200 as A  # noqa: E402
from synth import c4_genomes  # noqa: E402


def main(sizes):
    import os
    ctx = A.Context([0])
    if os.environ.get("TB_LEAF_CELLS"):
        ctx.set_option("tb_leaf_cells", int(os.environ["TB_LEAF_CELLS"]))
    for kind in ("global", "local"):
        sch = A.Scheme(kind, "linear", 2, -1, 0, 1)
        for n in sizes:
            g1, g2 = c4_genomes(n, "a", seed=4)
            ctx.traceback_long(sch, g1[:2000], g2[:2000])  # warm-up
            ctx.traceback_long(sch, g1, g2)  # first full-size call: one-time allocations
            t0 = time.perf_counter()
            r = ctx.traceback_long(sch, g1, g2)
            dt = time.perf_counter() - t0
            cells = len(g1) * len(g2)
            print(json.dumps({"kind": kind, "n": len(g1), "m": len(g2), "score": r["score"],
                              "ops": len(r["cigar"]), "s": round(dt, 4),
                              "gcups": round(cells / dt / 1e9, 1),
                              "pass_gcups": round(ctx.stat("tb_pass_cells")
                                                  / ctx.stat("tb_pass_ms") / 1e6, 1),
                              "pass_ms": round(ctx.stat("tb_pass_ms"), 1),
                              "leaf_ms": round(ctx.stat("tb_leaf_ms"), 1)}),
                  flush=True)


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [100_000, 1_000_000])
