#!/usr/bin/env python
"""bench.py -- headline benchmark: GCUPS of batched 150 bp semi-global affine alignment (C2).

Workload (BASELINE.json configs[1], "C2"): 1,000,000 synthetic Illumina-like read pairs,
150 x 150 bp, semi-global, affine gap open 5 / extend 1 (magnitudes), match +2 /
mismatch -1, score-only, one B200 per rank.  One step = the whole hot path on one batch:
pack + validate (a1), plan (a2), fill with fused optimum (a3, a7) -- all on device through
the C-ABI (anyseq_align_batch_device), inputs resident in HBM (300 MB > 126 MB L2, so no
L2 flush is needed between steps).

  value  : total cells of all ranks / max-over-ranks device time, in GCUPS.
  e2e    : the same metric through the host API anyseq_align_batch with pinned host buffers
           (H2D of the ASCII batch and D2H of the scores inside the timed region).
  roofline: the fill kernel's cells/s (CUDA events around each launch, on its stream)
           against the integer-pipe roofline derived in DESIGN.md ("bound": "alu").
  cpu_baseline: the plain CPU oracle (oracle/) on a bounded sample of the same workload.

--impl reference runs the reference arm for this tier: the oracle itself on the host cores,
each step a bounded sample of the same workload.
Multi-GPU (torchrun): every rank aligns its own 1M pairs (seed per rank): weak scaling,
no data-path collective (batches shard by pair); timing is max over ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCHEME = dict(kind="semi", gap="affine", match=2, mismatch=-1, gap_open=5, gap_extend=1)
NUM_PAIRS = 1_000_000
READ_LEN = 150
METRIC = "GCUPS (batched 150bp semi-global affine, long-pair SW) at 1/2/4/8 B200"
# dram__bytes_read.sum + dram__bytes_write.sum of one fill launch on the full C2 batch, from
# the committed ncu --set full capture of the fill kernel at the full C2 size.
TRAFFIC_BYTES_PER_LAUNCH = 328_585_984  # 320.27 MB read + 8.32 MB write (profiles/r01_fill_ncu.txt)


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, nm in enumerate(names):
                if len(s) > 3 + k and s[3 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def cpu_oracle_baseline(qm, sm, budget_s: float = 12.0, threads=None):
    """Time the plain CPU oracle on a bounded sample (first k pairs) of the same workload."""
    import numpy as np
    from oracle import oracle as O
    from synth import uniform_csr
    th = threads or os.cpu_count() or 1
    sch = O.Scheme(SCHEME["kind"], SCHEME["gap"], SCHEME["match"], SCHEME["mismatch"],
                   SCHEME["gap_open"], SCHEME["gap_extend"])
    k = min(len(qm), 400 * th)
    q, qo = uniform_csr(qm[:k])
    s, so = uniform_csr(sm[:k])
    t0 = time.perf_counter()
    O.batch(sch, q, qo, s, so, traceback=False, threads=th)
    dt = time.perf_counter() - t0
    # scale the sample to the time budget
    k2 = int(min(len(qm), max(k, k * budget_s / max(dt, 1e-3))))
    q, qo = uniform_csr(qm[:k2])
    s, so = uniform_csr(sm[:k2])
    t0 = time.perf_counter()
    res, _ = O.batch(sch, q, qo, s, so, traceback=False, threads=th)
    dt = time.perf_counter() - t0
    cells = k2 * READ_LEN * READ_LEN
    return {"value": round(cells / dt / 1e9, 4), "unit": "GCUPS", "cores": th, "kind": "oracle",
            "sample": f"first {k2} of the {len(qm)} C2 pairs (150x150, semi-global affine 5/1), "
                      f"{dt:.1f} s on {th} threads"}, res["score"]


def measured_alu_peak():
    """Integer-pipe roofline of the shipped fill formulation.

    cells/clk/SM = 2 cells per s16x2 register / (ALU cycles per register), with the
    per-instruction lane rates MEASURED on a B200 by the DPX microbenchmark
    (paper_2002_04561_b200/csrc/dpx_bench.cu -> profiles/dpx_rates.json): per register
    the fill issues 1 PRMT + 3 VIADDMNMX.S16x2 + 1 VIMNMX.S16x2 on the ALU pipe (and 2
    IMAD on the FMA pipe, which is not binding).  All five run at ~64 lane-ops/clk/SM
    (16 lanes/clk per SM sub-partition), i.e. 25.6 cells/clk/SM.  Falls back to 64
    lane-ops/clk/SM for every ALU op when the file is absent."""
    import torch
    props = torch.cuda.get_device_properties(0)
    path = os.path.join(ROOT, "profiles", "dpx_rates.json")
    r = {}
    if os.path.exists(path):
        try:
            r = json.load(open(path))
        except Exception:
            r = {}
    prmt = r.get("prmt", 64.0)
    vadd = r.get("viaddmnmx_s16x2", 64.0)
    vmax = r.get("vimnmx_s16x2", 64.0)
    clk_per_reg = 1.0 / prmt + 3.0 / vadd + 1.0 / vmax  # SM-clocks per lane-register
    cells = 2.0 / clk_per_reg
    src = "measured dpx_bench rates" if r else "design 64 lane-ops/clk/SM"
    return props.multi_processor_count, cells, src


def arm_config(pairs_per_gpu: int, ws: int) -> dict:
    """The workload description both arms print (the reference arm times bounded samples of
    exactly this workload; its cpu_baseline.sample says how many pairs per step)."""
    return {"workload": "C2: 1M Illumina-like 150x150 bp pairs per GPU, semi-global, "
                        "affine open 5 / extend 1, match 2 / mismatch -1, score-only",
            "pairs_per_gpu": pairs_per_gpu, "cells_per_gpu": pairs_per_gpu * READ_LEN * READ_LEN,
            "l2": "inputs 300 MB > 126 MB L2 (no flush needed)",
            "parallelism": f"dp{ws} (pairs sharded, no collective)"}


def run_reference(args):
    """Reference arm of this tier: the CPU oracle (as it stands), timed on the host cores.
    Each step aligns a bounded sample of the C2 workload (calibrated once to about
    --ref-budget seconds); the value is the median GCUPS of the K timed steps."""
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import numpy as np
    from oracle import oracle as O
    from synth import c2_reads, uniform_csr
    th = os.cpu_count() or 1
    qm, sm = c2_reads(200_000, seed=2)
    sch = O.Scheme(SCHEME["kind"], SCHEME["gap"], SCHEME["match"], SCHEME["mismatch"],
                   SCHEME["gap_open"], SCHEME["gap_extend"])

    def run(k):
        q, qo = uniform_csr(qm[:k])
        s, so = uniform_csr(sm[:k])
        t0 = time.perf_counter()
        O.batch(sch, q, qo, s, so, traceback=False, threads=th)
        return time.perf_counter() - t0

    k = min(len(qm), 200 * th)
    dt = run(k)
    k = int(min(len(qm), max(1000, k * args.ref_budget / max(dt, 1e-3))))
    vals = []
    for it in range(args.warmup + args.steps):
        dt = run(k)
        if it >= args.warmup:
            vals.append(k * READ_LEN * READ_LEN / dt / 1e9)
    v = round(float(np.median(vals)), 4)
    sample = f"{k} of the C2 pairs (150x150, semi-global affine 5/1) per step on {th} threads"
    line = {"metric": METRIC, "value": v, "unit": "GCUPS", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(k * READ_LEN * READ_LEN / v / 1e6, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "impl": "reference",
            "config": arm_config(args.pairs, ws),
            "cpu_baseline": {"value": v, "unit": "GCUPS", "cores": th, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def long_pair_leg(ctx, A, n, n_sm, f_mhz, n_gpus=1):
    """The metric's second half: C4 (two n-bp genomes, G2 = mutated copy of G1, local affine
    5/1, +2/-1, score-only) through anyseq_align_long, once (one call is ~9 s at 5 Mbp on one
    GPU).  With n_gpus > 1 the context spans GPUs 0..n_gpus-1 and the pair runs as n_gpus
    column strips with the boundary column passed GPU to GPU over NVLink; rank
    0 drives every device from one process (the other ranks wait on a CPU barrier).
    GCUPS = n*m / kernel time (CUDA events around the long kernel, max over devices); wall
    includes the upload and pack of both genomes.  Not a bench step: the headline value is
    C2."""
    from synth import c4_genomes
    g1, g2 = c4_genomes(n, "a", seed=4)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    t0 = time.perf_counter()
    r = ctx.align_long(sch, g1, g2)
    wall = time.perf_counter() - t0
    ms = ctx.stat("long_kernel_ms")
    narrow = int(ctx.stat("long_narrow"))
    cells = len(g1) * len(g2)
    gcups = cells / (ms / 1e3) / 1e9
    # 5.5 ALU ops per two cells at 64 lane-ops/clk/SM (16-bit kernel);
    # 5 ALU ops per cell (s32 kernel, 5.4)
    cpc = 64 * 2 / 5.5 if narrow else 64 / 5.0
    peak = n_gpus * n_sm * f_mhz * 1e6 * cpc / 1e9
    return {"workload": f"C4: {len(g1)} bp x {len(g2)} bp (G2 = mutated copy of G1), local affine "
                        f"open 5 / extend 1, match 2 / mismatch -1, score-only, {n_gpus} GPU"
                        + ("s (column strips)" if n_gpus > 1 else ""),
            "n_gpus": n_gpus,
            "value": round(gcups, 1), "unit": "GCUPS", "kernel_ms": round(ms, 1),
            "wall_ms": round(wall * 1e3, 1),
            "kernel": "long16_kernel<16> (16-bit differential)" if narrow else "long_kernel<LOCAL,AFFINE,16> (s32)",
            "roofline": {"bound": "alu", "achieved": round(gcups, 1), "peak": round(peak, 1),
                         "unit": "GCUPS", "frac": round(gcups / peak, 4),
                         "peak_basis": f"{n_gpus} GPU x {n_sm} SM x {f_mhz:.0f} MHz (C2 median under load) x {cpc:.2f} cells/clk/SM"},
            "score": r["score"], "end": [r["q_end"], r["s_end"]]}


def mixed_sizes_leg(ctx, A, n_long, n_short, n_sm, f_mhz, reps=3):
    """a score-only batch of n_long similar pairs of
    2-20 kbp (windows of a mutated genome pair) mixed into n_short random 100-300 bp pairs,
    local affine 5/1, through the host API (anyseq_align_batch, pageable buffers): the long
    pairs share ONE launch of the 16-bit long kernel while the batch kernels align the short
    pairs in place.  value = all cells / best wall time of `reps` calls; the shared launch's
    own rate is over the long pairs' cells.  Checked against the one-long-call-per-pair path
    (option long_multi = 0) on the same batch."""
    import numpy as np
    from synth import c4_genomes, random_pairs, csr
    rng = np.random.default_rng(5)
    g1, g2 = c4_genomes(2_000_000, "a", seed=6)
    q0, qo0, s0, so0 = random_pairs(n_short, 100, 300, seed=7)
    qs = [q0[qo0[k]:qo0[k + 1]].tobytes() for k in range(n_short)]
    ss = [s0[so0[k]:so0[k + 1]].tobytes() for k in range(n_short)]
    short_cells = float(np.sum(np.diff(qo0).astype(np.float64) * np.diff(so0)))
    long_cells = 0.0
    for _ in range(n_long):
        n = int(rng.integers(2048, 20001))
        m = int(rng.integers(2048, 20001))
        a = int(rng.integers(0, len(g1) - max(n, m)))
        pos = int(rng.integers(0, len(qs) + 1))
        qs.insert(pos, g1[a:a + n])
        ss.insert(pos, g2[a:a + m])
        long_cells += float(n) * m
    q, qo = csr(qs)
    s, so = csr(ss)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    sc = ctx.align_batch(sch, q, qo, s, so)  # warm-up (workspace growth)
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        sc = ctx.align_batch(sch, q, qo, s, so)
        best = min(best, time.perf_counter() - t0)
    kms = ctx.stat("long_multi_ms")
    taken = int(ctx.stat("long_multi_pairs"))
    rows = int(ctx.stat("long_multi_rows"))
    ctx.set_option("long_multi", 0)
    t0 = time.perf_counter()
    sc1 = ctx.align_batch(sch, q, qo, s, so)
    per_pair = time.perf_counter() - t0
    ctx.set_option("long_multi", 1)
    cells = short_cells + long_cells
    kg = long_cells / (kms / 1e3) / 1e9 if kms > 0 else 0.0
    peak = n_sm * f_mhz * 1e6 * (64 * 2 / 5.5) / 1e9
    return {"workload": f"{n_long} pairs of 2-20 kbp (mutated genome windows) + {n_short} pairs of "
                        "100-300 bp, local affine open 5 / extend 1, match 2 / mismatch -1, "
                        "score-only, host API from pageable buffers, 1 GPU",
            "value": round(cells / best / 1e9, 1), "unit": "GCUPS", "wall_ms": round(best * 1e3, 2),
            "long_pairs_in_shared_launch": taken,
            "shared_launch": {"kernel": f"long16_kernel<{rows // 64}, LOCAL, MULTI> ({rows}-row tasks)",
                              "kernel_ms": round(kms, 2),
                              "gcups": round(kg, 1),
                              "roofline": {"bound": "alu", "achieved": round(kg, 1),
                                           "peak": round(peak, 1), "unit": "GCUPS",
                                           "frac": round(kg / peak, 4)}},
            "one_call_per_long_pair_wall_ms": round(per_pair * 1e3, 1),
            "same_scores_as_one_call_per_pair": bool(np.array_equal(sc, sc1))}


def mixed_sizes_traceback_leg(ctx, A, n_long=200, n_short=10_000, reps=3):
    """SURVEY 8(f) f4 in traceback mode: n_long similar pairs of 2-10 kbp
    mixed into n_short random 100-300 bp pairs, local affine 5/1, anyseq_traceback through
    the host API (pageable buffers): the long pairs' checkpointing forward passes share one
    launch (overlapped with the short pairs' batch traceback), then each long pair is walked
    from its checkpoints.  value = all cells / best wall time; checked (scores, cells and
    CIGARs) against the one-long-traceback-per-pair path (option long_multi = 0)."""
    import numpy as np
    from synth import c4_genomes, random_pairs, csr
    rng = np.random.default_rng(8)
    g1, g2 = c4_genomes(1_000_000, "a", seed=9)
    q0, qo0, s0, so0 = random_pairs(n_short, 100, 300, seed=10)
    qs = [q0[qo0[k]:qo0[k + 1]].tobytes() for k in range(n_short)]
    ss = [s0[so0[k]:so0[k + 1]].tobytes() for k in range(n_short)]
    cells = float(np.sum(np.diff(qo0).astype(np.float64) * np.diff(so0)))
    for _ in range(n_long):
        n = int(rng.integers(2048, 10001))
        m = int(rng.integers(2048, 10001))
        a = int(rng.integers(0, len(g1) - max(n, m)))
        pos = int(rng.integers(0, len(qs) + 1))
        qs.insert(pos, g1[a:a + n])
        ss.insert(pos, g2[a:a + m])
        cells += float(n) * m
    q, qo = csr(qs)
    s, so = csr(ss)
    sch = A.Scheme("local", "affine", 2, -1, 5, 1)
    aln, words = ctx.traceback(sch, q, qo, s, so)  # warm-up
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        aln, words = ctx.traceback(sch, q, qo, s, so)
        best = min(best, time.perf_counter() - t0)
    taken = int(ctx.stat("long_multi_pairs"))
    kms = ctx.stat("long_multi_ms")
    ctx.set_option("long_multi", 0)
    t0 = time.perf_counter()
    aln1, words1 = ctx.traceback(sch, q, qo, s, so)
    per_pair = time.perf_counter() - t0
    ctx.set_option("long_multi", 1)
    same = bool(np.array_equal(aln, aln1) and np.array_equal(words, words1))
    return {"workload": f"{n_long} pairs of 2-10 kbp (mutated genome windows) + {n_short} pairs of "
                        "100-300 bp, local affine open 5 / extend 1, match 2 / mismatch -1, "
                        "traceback + CIGAR, host API from pageable buffers, 1 GPU",
            "value": round(cells / best / 1e9, 1), "unit": "GCUPS", "wall_ms": round(best * 1e3, 2),
            "long_pairs_in_shared_pass": taken, "shared_pass_ms": round(kms, 2),
            "one_traceback_per_long_pair_wall_ms": round(per_pair * 1e3, 1),
            "same_alignments_as_one_per_pair": same}


def long_traceback_leg(ctx, A, n, kind="global", gap="linear", go=0):
    """linear-space traceback of a C4-shaped pair (n-bp genomes, G2 =
    mutated copy of G1), once, through anyseq_traceback_long with host buffers: one
    checkpointing forward pass of the 16-bit long kernel, then the tile-recompute walk
    (DESIGN.md 5.4c).  Schemes: global linear +2/-1/-1 (the paper's long traceback scheme,
    Fig. 5a) and local affine 5/1 (C4's scheme).  GCUPS = n*m / wall time of the call (the
    paper's convention: matrix cells over total time); pass_gcups = n*m / the forward pass's
    device time; walk_ms = the walk kernel's device time."""
    from synth import c4_genomes
    g1, g2 = c4_genomes(n, "a", seed=4)
    sch = A.Scheme(kind, gap, 2, -1, go, 1)
    ctx.traceback_long(sch, g1, g2)  # warm-up: one-time allocations
    t0 = time.perf_counter()
    r = ctx.traceback_long(sch, g1, g2)
    wall = time.perf_counter() - t0
    pass_ms, walk_ms = ctx.stat("tb_pass_ms"), ctx.stat("tb_walk_ms")
    cells = len(g1) * len(g2)
    return {"workload": f"{len(g1)} bp x {len(g2)} bp (C4 variant a shape), {kind} {gap}"
                        + (f" open {go} / extend 1" if gap == "affine" else " gap 1")
                        + ", match 2 / mismatch -1, traceback (checkpoints + tile walk), 1 GPU",
            "value": round(cells / wall / 1e9, 1), "unit": "GCUPS", "wall_ms": round(wall * 1e3, 1),
            "pass_ms": round(pass_ms, 1), "pass_gcups": round(cells / (pass_ms / 1e3) / 1e9, 1),
            "walk_ms": round(walk_ms, 1), "ckpt_bytes": int(ctx.stat("tb_ckpt_bytes")),
            "method": "checkpoints" if ctx.stat("tb_method") == 1 else "hirschberg",
            "score": r["score"], "begin": [r["q_begin"], r["s_begin"]],
            "end": [r["q_end"], r["s_end"]], "cigar_ops": len(r["cigar"])}


def time_device_steps(step, stream, steps):
    """CUDA events around `steps` calls of step() on `stream` (after a synchronize)."""
    import torch
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pairs", type=int, default=NUM_PAIRS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=3.0)
    ap.add_argument("--long-tb-bp", type=int, default=1_000_000,
                    help="linear-space long traceback leg (8(f) f1) genome length; 0 skips it")
    ap.add_argument("--long-bp", type=int, default=5_000_000,
                    help="C4 long pair (second half of the metric) genome length; 0 skips it")
    ap.add_argument("--mixed-long", type=int, default=200,
                    help="mixed-size leg (8(f) f4): long pairs of 2-20 kbp; 0 skips it")
    ap.add_argument("--mixed-short", type=int, default=100_000)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2002_04561_b200 as A
    from synth import c2_reads, uniform_csr

    ws, rank, local = _dist()
    if args.gpus != ws:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch N>1 under torchrun "
              f"(one rank per GPU) -- reporting n_gpus={ws}", file=sys.stderr)
    torch.cuda.set_device(local)
    cpu_group = None
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # CPU-side barrier for the legs where rank 0 alone drives every GPU (C4 column strips):
        # an NCCL barrier would park a kernel on the GPUs that leg needs
        cpu_group = dist.new_group(backend="gloo")

    def barrier():
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=torch.device("cuda", local))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    qm, sm = c2_reads(args.pairs, seed=2 + 1000 * rank)
    q, qo = uniform_csr(qm)
    s, so = uniform_csr(sm)
    B = len(qo) - 1
    cells = B * READ_LEN * READ_LEN
    dev = torch.device("cuda", local)
    d_q = torch.from_numpy(q).to(dev)
    d_s = torch.from_numpy(s).to(dev)
    d_qo = torch.from_numpy(qo.view(np.int64)).to(dev)
    d_so = torch.from_numpy(so.view(np.int64)).to(dev)
    d_sc = torch.empty(B, dtype=torch.int32, device=dev)
    sch = A.Scheme(**SCHEME)
    ctx = A.Context([local])
    stream = torch.cuda.current_stream()

    def step():
        ctx.align_batch_device(sch, d_q, d_qo, d_s, d_so, d_sc, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.set_option("timing", 1)
    ctx.reset_stats()
    launches0 = ctx.launches
    sampler = ClockSampler(local)
    sampler.start()
    barrier()
    ms = time_device_steps(step, stream, args.steps)
    barrier()
    clocks = sampler.stop()
    launches = ctx.launches - launches0
    fill_ms = ctx.stat("fill_ms")
    fill_launches = int(ctx.stat("fill_launches"))
    ctx.set_option("timing", 0)
    ms_max = max_over_ranks(ms)
    value = cells * ws * args.steps / (ms_max / 1e3) / 1e9
    got = d_sc.cpu().numpy()

    # generic scheme (no compile-time scoring constants: open 6 / extend 1 has no specialised
    # instance) on the same batch -- the rate of the fill without partial evaluation
    gsch = A.Scheme("semi", "affine", 2, -1, 6, 1)
    d_sc2 = torch.empty_like(d_sc)
    gstep = lambda: ctx.align_batch_device(gsch, d_q, d_qo, d_s, d_so, d_sc2, stream=stream)
    gstep()
    g_ms = max_over_ranks(time_device_steps(gstep, stream, max(3, args.steps // 2)))
    generic = {"scheme": "semi-global affine open 6 / extend 1, match 2 / mismatch -1 "
                         "(no specialised instance)",
               "value": round(cells * ws * max(3, args.steps // 2) / (g_ms / 1e3) / 1e9, 1),
               "unit": "GCUPS"}

    # strong scaling: the same 1M-pair batch split over the ranks
    strong = None
    if ws > 1:
        k0, k1 = B * rank // ws, B * (rank + 1) // ws
        sq, sqo = uniform_csr(qm[k0:k1])
        ss_, sso = uniform_csr(sm[k0:k1])
        t_q, t_s = torch.from_numpy(sq).to(dev), torch.from_numpy(ss_).to(dev)
        t_qo = torch.from_numpy(sqo.view(np.int64)).to(dev)
        t_so = torch.from_numpy(sso.view(np.int64)).to(dev)
        t_sc = torch.empty(k1 - k0, dtype=torch.int32, device=dev)
        sstep = lambda: ctx.align_batch_device(sch, t_q, t_qo, t_s, t_so, t_sc, stream=stream)
        for _ in range(args.warmup):
            sstep()
        barrier()
        s_ms = max_over_ranks(time_device_steps(sstep, stream, args.steps))
        strong = {"workload": f"C2 1M pairs total split over {ws} ranks",
                  "value": round(cells * args.steps / (s_ms / 1e3) / 1e9, 1), "unit": "GCUPS",
                  "ms_per_step": round(s_ms / args.steps, 4), "scaling": "strong"}

    # e2e through the host API from pinned buffers
    pq = torch.from_numpy(q).pin_memory().numpy()
    ps = torch.from_numpy(s).pin_memory().numpy()
    pqo = torch.from_numpy(qo.view(np.int64)).pin_memory().numpy().view(np.uint64)
    pso = torch.from_numpy(so.view(np.int64)).pin_memory().numpy().view(np.uint64)
    pout = torch.empty(B, dtype=torch.int32).pin_memory().numpy()
    e2e_steps = max(2, min(args.steps, 5))
    ctx.align_batch(sch, pq, pqo, ps, pso, out=pout)
    ctx.reset_stats()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ctx.align_batch(sch, pq, pqo, ps, pso, out=pout)
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    # bytes the host API actually moved (ACGT-only chunks go up as 2-bit codes, a1)
    h2d_step = int(ctx.stat("h2d_bytes") / e2e_steps)
    d2h_step = int(ctx.stat("d2h_bytes") / e2e_steps)
    e2e_value = cells * ws * e2e_steps / e2e_s / 1e9
    e2e_same = bool(np.array_equal(pout, got))

    # roofline of the dominant kernel (fill): cells per launch / mean launch time
    n_sm, cells_per_clk, rate_src = measured_alu_peak()
    f_mhz = clocks.get("sm_mhz") or 1965.0
    peak = n_sm * f_mhz * 1e6 * cells_per_clk / 1e9
    fill_gcups = cells * args.steps / (fill_ms / 1e3) / 1e9 if fill_ms > 0 else None
    roof = {"bound": "alu", "achieved": round(fill_gcups, 1) if fill_gcups else None,
            "peak": round(peak, 1), "unit": "GCUPS",
            "frac": round(fill_gcups / peak, 4) if fill_gcups else None,
            "traffic": TRAFFIC_BYTES_PER_LAUNCH,
            "kernel": "fill_kernel<VS16,SEMI,AFFINE,L=8,R=19>",
            "kernel_share_of_step": round(fill_ms / ms, 4) if ms > 0 else None,
            "peak_basis": f"{n_sm} SM x {f_mhz:.0f} MHz (median under load) x "
                          f"{cells_per_clk:.2f} cells/clk/SM ({rate_src}: 2 cells per "
                          f"PRMT + 3 VIADDMNMX.S16x2 + VIMNMX.S16x2)"}

    line = {"metric": METRIC, "value": round(value, 1), "unit": "GCUPS", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "s16x2",
            "data": "synthetic",
            "config": arm_config(B, ws),
            "e2e": {"value": round(e2e_value, 1), "unit": "GCUPS",
                    # counted by the library: 2-bit sequence codes (offsets only for
                    # non-uniform chunks) up, scores down
                    "h2d_bytes_per_step": h2d_step, "d2h_bytes_per_step": d2h_step,
                    "ascii_bytes_per_step": int(q.nbytes + s.nbytes),
                    "same_scores_as_device_api": e2e_same},
            "gpu_launches": int(launches),
            "fill_launches": fill_launches,
            "roofline": roof,
            "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "generic_scheme": generic}
    if strong:
        line["strong_scaling"] = strong

    from oracle import oracle as O
    osch = O.Scheme(SCHEME["kind"], SCHEME["gap"], SCHEME["match"], SCHEME["mismatch"],
                    SCHEME["gap_open"], SCHEME["gap_extend"])
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        # the oracle baseline aligns (up to) the whole batch: compare every score it computed
        cb, oscores = cpu_oracle_baseline(qm, sm)
        line["cpu_baseline"] = cb
        k = len(oscores)
        mism = int(np.count_nonzero(got[:k] != oscores.astype(np.int32)))
        line["parity"] = {"checked_pairs": k, "of": B, "mismatches": mism,
                          "parity_full": bool(k == B and mism == 0)}
    else:
        # parity spot check of this rank's output (oracle on 64 pairs) -- not timed
        idx = np.random.default_rng(rank).choice(B, 64, replace=False)
        mism = sum(int(got[k]) != O.align(osch, qm[k].tobytes(), sm[k].tobytes(), False).score
                   for k in idx)
        line["parity"] = {"checked_pairs": 64, "of": B, "mismatches": int(mism),
                          "parity_full": False}

    # C4 long pair: on N GPUs through one N-device context driven by rank 0
    if args.long_bp > 0:
        if ws > 1:
            dist.barrier(group=cpu_group)
        if rank == 0:
            lctx = ctx if ws == 1 else A.Context(list(range(ws)))
            line["long_pair"] = long_pair_leg(lctx, A, args.long_bp, n_sm, f_mhz, n_gpus=ws)
            if lctx is not ctx:
                lctx.close()
        if ws > 1:
            dist.barrier(group=cpu_group)
    if rank == 0 and args.mixed_long > 0:
        line["mixed_sizes"] = mixed_sizes_leg(ctx, A, args.mixed_long, args.mixed_short, n_sm, f_mhz)
        line["mixed_sizes_traceback"] = mixed_sizes_traceback_leg(ctx, A)
    if rank == 0 and args.long_tb_bp > 0:
        line["long_traceback"] = long_traceback_leg(ctx, A, args.long_tb_bp)
        line["long_traceback_local_affine"] = long_traceback_leg(ctx, A, args.long_tb_bp,
                                                                 "local", "affine", 5)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        dist.barrier(group=cpu_group)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
