"""C5 at the survey's full size (8 M mixed 100-1000 bp pairs, every kind,
score-only and traceback, affine 5/1, match 2 / mismatch -1) on one GPU through the host API
from page-locked buffers, with oracle parity on a 1 % sample (scores, end cells and, for
traceback, CIGARs element by element).  Prints one JSON line per kind.
usage: python tools/c5_full.py [pairs] [sample_fraction]"""
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
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).pin_memory().numpy().view(a.dtype)


def main():
    pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
    frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
    t0 = time.perf_counter()
    q, qo, s, so = synth.c5_mixed_large(pairs, seed=5)
    gen_s = time.perf_counter() - t0
    B = len(qo) - 1
    cells = float(np.sum(np.diff(qo).astype(np.float64) * np.diff(so).astype(np.float64)))
    pq, pqo, ps, pso = pin(q), pin(qo), pin(s), pin(so)
    psc = pin(np.zeros(B, np.int32))
    paln = pin(np.zeros(B, A.ALIGNMENT_DTYPE))
    pcig = pin(np.zeros(24 * B, np.uint32))
    idx = np.sort(np.random.default_rng(7).choice(B, max(1, int(B * frac)), replace=False))
    # the sample as its own CSR batch for the oracle
    ql, sl = np.diff(qo)[idx], np.diff(so)[idx]
    sq = np.concatenate([q[qo[k]:qo[k + 1]] for k in idx])
    ss_ = np.concatenate([s[so[k]:so[k + 1]] for k in idx])
    sqo = np.concatenate([[0], np.cumsum(ql)]).astype(np.uint64)
    sso = np.concatenate([[0], np.cumsum(sl)]).astype(np.uint64)
    ctx = A.Context([0])
    for kind in ("global", "semi", "local"):
        sch = A.Scheme(kind, "affine", 2, -1, 5, 1)
        osch = O.Scheme(kind, "affine", 2, -1, 5, 1)
        ctx.align_batch(sch, pq, pqo, ps, pso, out=psc)  # warm
        ctx.set_option("timing", 1)
        ctx.reset_stats()
        t0 = time.perf_counter()
        ctx.align_batch(sch, pq, pqo, ps, pso, out=psc)
        sw = time.perf_counter() - t0
        sfill = ctx.stat("fill_ms")
        ctx.set_option("timing", 0)
        sc = psc.copy()
        ctx.traceback(sch, pq, pqo, ps, pso, out_aln=paln, out_cigar=pcig)  # warm
        ctx.set_option("timing", 1)
        ctx.reset_stats()
        t0 = time.perf_counter()
        aln, cig = ctx.traceback(sch, pq, pqo, ps, pso, out_aln=paln, out_cigar=pcig)
        tw = time.perf_counter() - t0
        tfill, twalk = ctx.stat("fill_ms"), ctx.stat("walk_ms")
        ctx.set_option("timing", 0)
        t0 = time.perf_counter()
        ores, ocig = O.batch(osch, sq, sqo, ss_, sso, traceback=True)
        oracle_s = time.perf_counter() - t0
        ocigs = O.batch_cigars(ores, ocig, sqo, sso)
        gcigs = A.cigars_of(aln[idx], cig)
        bad_score = int(np.sum(sc[idx] != ores["score"]))
        bad_tb = 0
        for n, k in enumerate(idx):
            a = aln[k]
            if (int(a["score"]) != int(ores["score"][n]) or int(a["q_end"]) != int(ores["q_end"][n])
                    or int(a["s_end"]) != int(ores["s_end"][n])
                    or int(a["q_begin"]) != int(ores["q_begin"][n])
                    or int(a["s_begin"]) != int(ores["s_begin"][n]) or gcigs[n] != ocigs[n]):
                bad_tb += 1
        print(json.dumps({
            "config": f"C5 {B} mixed 100-1000 bp pairs, {kind} affine 5/1, 1 GPU, host API (pinned)",
            "cells": cells, "score_wall_ms": round(sw * 1e3, 1), "score_fill_ms": round(sfill, 1),
            "score_gcups_wall": round(cells / sw / 1e9, 1),
            "tb_wall_ms": round(tw * 1e3, 1), "tb_fill_ms": round(tfill, 1), "tb_walk_ms": round(twalk, 1),
            "tb_gcups_wall": round(cells / tw / 1e9, 1),
            "parity_sample": len(idx), "score_mismatches": bad_score, "tb_mismatches": bad_tb,
            "oracle_s": round(oracle_s, 1), "gen_s": round(gen_s, 1)}), flush=True)


if __name__ == "__main__":
    main()
