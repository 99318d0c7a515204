"""1 Mbp long traceback (C4 variant a shape) with the host phase timeline (timing = 2):
usage: python tools/long_tb_phases.py [n] [kind] [gap] [go]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_04561_b200 as A  # noqa: E402
from synth import c4_genomes  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
kind = sys.argv[2] if len(sys.argv) > 2 else "local"
gap = sys.argv[3] if len(sys.argv) > 3 else "affine"
go = int(sys.argv[4]) if len(sys.argv) > 4 else 5
g1, g2 = c4_genomes(n, "a", seed=4)
ctx = A.Context([0])
sch = A.Scheme(kind, gap, 2, -1, go, 1)
for rep in range(5):
    if rep == 1:
        ctx.set_option("timing", 2)
    t0 = time.perf_counter()
    r = ctx.traceback_long(sch, g1, g2)
    wall = time.perf_counter() - t0
    print(f"rep {rep}: wall {wall*1e3:.1f} ms pass {ctx.stat('tb_pass_ms'):.1f} walk {ctx.stat('tb_walk_ms'):.1f} "
          f"score {r['score']} begin {r['q_begin']},{r['s_begin']}", flush=True)
