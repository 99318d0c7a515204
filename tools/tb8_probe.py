"""C3-shaped traceback (150 bp reads, local affine) at a reduced pair count: fill/walk device
time with the full H store (tb8=0) and the 1-byte store (tb8=1).  Probe, not a bench line."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_04561_b200 as A  # noqa: E402
import synth  # noqa: E402


def main():
    pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
    modes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,1").split(",")]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    qm, sm = synth.c2_reads(pairs, seed=2)
    q, qo = synth.uniform_csr(qm)
    s, so = synth.uniform_csr(sm)
    ctx = A.Context([0])
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    ctx.set_option("force_variant", int(os.environ.get("FORCE_VARIANT", "-1")))
    for t8 in modes:
        ctx.set_option("tb8", t8)
        ctx.traceback(sch, q, qo, s, so)
        ctx.set_option("timing", 1)
        ctx.reset_stats()
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.traceback(sch, q, qo, s, so)
        wall = (time.perf_counter() - t0) / reps
        f, w = ctx.stat("fill_ms") / reps, ctx.stat("walk_ms") / reps
        cells = pairs * 150 * 150
        print(f"tb8={t8}: wall {wall*1e3:.2f} ms fill {f:.2f} ms ({cells/f/1e6:.0f} GCUPS) "
              f"walk {w:.2f} ms", flush=True)
        ctx.set_option("timing", 0)


if __name__ == "__main__":
    main()
