"""Measure the secondary configs (C1, C3, C4, C5) on one GPU: device time of the library's
kernels per call (CUDA events inside the library, option "timing") and host wall time of
the synchronous host-API call from page-locked buffers (as bench.py e2e), plus an oracle
parity sample.  Prints one JSON per config.
Not the driver's bench line (bench.py is); numbers go to BASELINE.md."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_04561_b200 as A  # noqa: E402
from oracle import oracle as O  # noqa: E402
import synth  # noqa: E402


def pin(a):
    """Copy into page-locked host memory (the host API's fast path, as in bench.py's e2e)."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).pin_memory().numpy().view(a.dtype)


def timed(ctx, fn, reps=3):
    fn()  # warm
    ctx.set_option("timing", 1)
    ctx.reset_stats()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    wall = (time.perf_counter() - t0) / reps
    fill = ctx.stat("fill_ms") / reps
    walk = ctx.stat("walk_ms") / reps
    ctx.set_option("timing", 0)
    return out, wall, fill, walk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c5,c4")
    ap.add_argument("--c4n", type=int, default=5_000_000)
    ap.add_argument("--c5pairs", type=int, default=1_000_000)
    args = ap.parse_args()
    ctx = A.Context([0])
    res = []
    printed = 0
    for c in args.configs.split(","):
        if c == "c1":
            a, b = synth.c1_pair(1)
            q, qo = synth.csr([a]); s, so = synth.csr([b])
            sch = A.Scheme("global", "linear", 2, -1, 0, 1)
            (aln, cig), wall, fill, walk = timed(ctx, lambda: ctx.traceback(sch, q, qo, s, so))
            o = O.align(O.Scheme("global", "linear", 2, -1, 0, 1), a, b)
            ok = int(aln["score"][0]) == o.score and A.cigars_of(aln, cig)[0] == o.cigar
            cells = 1e6
            # a one-pair batch takes the long-pair path (option batch_long_small): its
            # device times are the checkpointed pass and the tile walk of the last call
            res.append({"config": "C1 1000x1000 NW linear traceback", "cells": cells,
                        "wall_ms": wall * 1e3, "fill_ms": fill, "walk_ms": walk,
                        "tb_pass_ms": ctx.stat("tb_pass_ms"), "tb_walk_ms": ctx.stat("tb_walk_ms"),
                        "gcups_wall": cells / wall / 1e9, "parity": ok})
        elif c == "c3":
            qm, sm = synth.c2_reads(1_000_000, seed=2)
            q, qo = synth.uniform_csr(qm); s, so = synth.uniform_csr(sm)
            q, qo, s, so = pin(q), pin(qo), pin(s), pin(so)
            paln = pin(np.zeros(len(qo) - 1, A.ALIGNMENT_DTYPE))
            pcig = pin(np.zeros(32 * (len(qo) - 1), np.uint32))
            sch = A.Scheme("local", "affine", 2, -1, 5, 1)
            ctx.set_option("tb8", 0)  # the round-1 store (full H, 2 B per cell) for comparison
            _, wall16, fill16, walk16 = timed(
                ctx, lambda: ctx.traceback(sch, q, qo, s, so, out_aln=paln, out_cigar=pcig), 2)
            ctx.set_option("tb8", 1)
            (aln, cig), wall, fill, walk = timed(
                ctx, lambda: ctx.traceback(sch, q, qo, s, so, out_aln=paln, out_cigar=pcig), 2)
            idx = np.random.default_rng(0).choice(len(qm), 300, replace=False)
            osch = O.Scheme("local", "affine", 2, -1, 5, 1)
            cigs = A.cigars_of(aln[idx], cig)
            ok = all(int(aln["score"][k]) == O.align(osch, qm[k].tobytes(), sm[k].tobytes()).score and
                     cigs[n] == O.align(osch, qm[k].tobytes(), sm[k].tobytes()).cigar
                     for n, k in enumerate(idx))
            cells = 1e6 * 150 * 150
            res.append({"config": "C3 1M x 150bp SW affine traceback (CIGAR)", "cells": cells,
                        "wall_ms": wall * 1e3, "fill_ms": fill, "walk_ms": walk,
                        "fill_gcups": cells / (fill / 1e3) / 1e9,
                        "full_h_store": {"wall_ms": wall16 * 1e3, "fill_ms": fill16,
                                         "walk_ms": walk16},
                        "gcups_wall": cells / wall / 1e9,
                        "gcups_fill_walk": cells / ((fill + walk) / 1e3) / 1e9, "parity_300": ok})
        elif c == "c5":
            q, qo, s, so = synth.c5_mixed_large(args.c5pairs, seed=5)
            q, qo, s, so = pin(q), pin(qo), pin(s), pin(so)
            B = len(qo) - 1
            psc = pin(np.zeros(B, np.int32))
            paln = pin(np.zeros(B, A.ALIGNMENT_DTYPE))
            pcig = pin(np.zeros(24 * B, np.uint32))
            cells = float(np.sum(np.diff(qo).astype(np.float64) * np.diff(so).astype(np.float64)))
            for kind in ("global", "semi", "local"):
                sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
                sc, wall, fill, _ = timed(ctx, lambda: ctx.align_batch(sch, q, qo, s, so, out=psc))
                sc = sc.copy()
                (aln, cig), wall2, fill2, walk2 = timed(
                    ctx, lambda: ctx.traceback(sch, q, qo, s, so, out_aln=paln, out_cigar=pcig), 1)
                idx = np.random.default_rng(1).choice(len(qo) - 1, 100, replace=False)
                osch = O.Scheme(kind, "affine", 2, -1, 5, 1)
                ok = all(int(sc[k]) == O.align(osch, q[qo[k]:qo[k + 1]].tobytes(),
                                               s[so[k]:so[k + 1]].tobytes(), False).score for k in idx)
                res.append({"config": f"C5 {args.c5pairs} mixed 100-1000bp {kind} affine",
                            "cells": cells, "score_wall_ms": wall * 1e3, "score_fill_ms": fill,
                            "score_gcups_fill": cells / (fill / 1e3) / 1e9,
                            "score_gcups_wall": cells / wall / 1e9,
                            "tb_wall_ms": wall2 * 1e3, "tb_fill_ms": fill2, "tb_walk_ms": walk2,
                            "tb_gcups_wall": cells / wall2 / 1e9, "parity_100": ok})
        elif c == "c4":
            for variant in ("c", "a"):
                g1, g2 = synth.c4_genomes(args.c4n, variant, seed=4)
                sch = A.Scheme("local", "affine", 2, -1, 5, 1)
                t0 = time.perf_counter()
                r = ctx.align_long(sch, g1, g2)
                wall = time.perf_counter() - t0
                kms = ctx.stat("long_kernel_ms")
                cells = float(len(g1)) * len(g2)
                ok = (r["score"], r["q_end"], r["s_end"]) == (2 * len(g1), len(g1), len(g1)) \
                    if variant == "c" else None
                res.append({"config": f"C4 {args.c4n}bp x {len(g2)}bp SW affine variant {variant}",
                            "cells": cells, "wall_ms": wall * 1e3, "kernel_ms": kms,
                            "gcups_kernel": cells / (kms / 1e3) / 1e9,
                            "gcups_wall": cells / wall / 1e9, "result": r, "closed_form_ok": ok})
        while printed < len(res):
            print(json.dumps(res[printed]), flush=True)
            printed += 1


if __name__ == "__main__":
    main()
