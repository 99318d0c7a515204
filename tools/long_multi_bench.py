"""Mixed batch with many long pairs: one shared launch (long_multi = 1) vs one launch per
long pair (long_multi = 0), score-only through the host API.

Workload: `--long` pairs of similar sequences (windows of a C4-style genome pair, lengths
U{lo..hi}) mixed into `--short` random 100-300 bp pairs.  Prints wall time, the shared
launch's kernel time and GCUPS for both settings, and checks the results agree.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--long", type=int, default=200)
    ap.add_argument("--lo", type=int, default=2048)
    ap.add_argument("--hi", type=int, default=20000)
    ap.add_argument("--short", type=int, default=100000)
    ap.add_argument("--kind", default="local")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cells", type=int, default=1 << 22, help="option batch_long_cells")
    ap.add_argument("--min", type=int, default=2048, help="option batch_long_min")
    ap.add_argument("--rows", type=int, default=0, help="option long_band_rows (512/1024 force)")
    ap.add_argument("--tb", action="store_true", help="traceback mode (anyseq_traceback)")
    ap.add_argument("--helpers", type=int, default=96, help="option walk_helpers")
    ap.add_argument("--only", type=int, default=-1, help="run only long_multi = this")
    args = ap.parse_args()
    import paper_2002_04561_b200 as A
    from synth import c4_genomes, random_pairs, csr
    rng = np.random.default_rng(5)
    g1, g2 = c4_genomes(2_000_000, "a", seed=6)
    q0, qo0, s0, so0 = random_pairs(args.short, 100, 300, seed=7)
    qs = [q0[qo0[k]:qo0[k + 1]].tobytes() for k in range(args.short)]
    ss = [s0[so0[k]:so0[k + 1]].tobytes() for k in range(args.short)]
    cells = float(np.sum((np.diff(qo0) + 0.0) * np.diff(so0)))
    for _ in range(args.long):
        n = int(rng.integers(args.lo, args.hi + 1))
        m = int(rng.integers(args.lo, args.hi + 1))
        a = int(rng.integers(0, len(g1) - max(n, m)))
        pos = int(rng.integers(0, len(qs) + 1))
        qs.insert(pos, g1[a:a + n])
        ss.insert(pos, g2[a:a + m])
        cells += float(n) * m
    q, qo = csr(qs)
    s, so = csr(ss)
    sch = A.Scheme(args.kind, "affine", 2, -1, 5, 1)
    out = {"long_pairs": args.long, "lengths": [args.lo, args.hi], "short_pairs": args.short,
           "kind": args.kind, "cells": cells}
    with A.Context([0]) as ctx:
        ctx.set_option("batch_long_cells", args.cells)
        ctx.set_option("batch_long_cells_tb", args.cells)
        out["mode"] = "traceback" if args.tb else "score"
        ctx.set_option("walk_helpers", args.helpers)
        out["walk_helpers"] = args.helpers
        out["batch_long_cells"] = args.cells
        ctx.set_option("batch_long_min", args.min)
        out["batch_long_min"] = args.min
        ctx.set_option("long_band_rows", args.rows)
        out["rows"] = args.rows
        res = {}
        for multi in ((1, 0) if args.only < 0 else (args.only,)):
            ctx.set_option("long_multi", multi)
            def call():
                if args.tb:
                    aln, words = ctx.traceback(sch, q, qo, s, so)
                    return np.concatenate([aln["score"].astype(np.int64), aln["q_begin"],
                                           aln["s_begin"], aln["cigar_len"].astype(np.int64),
                                           words.astype(np.int64)])
                return ctx.align_batch(sch, q, qo, s, so)
            sc = call()  # warm-up
            best = 1e30
            for _ in range(args.reps):
                t0 = time.perf_counter()
                sc = call()
                best = min(best, time.perf_counter() - t0)
            res[multi] = sc
            out[f"multi{multi}"] = {"wall_ms": round(best * 1e3, 2),
                                    "gcups": round(cells / best / 1e9, 1),
                                    "kernel_ms": round(ctx.stat("long_multi_ms"), 2),
                                    "pairs_in_shared_launch": int(ctx.stat("long_multi_pairs"))}
        if len(res) == 2:
            out["same_scores"] = bool(np.array_equal(res[0], res[1]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
