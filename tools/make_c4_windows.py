"""Write tests/golden/c4_windows.tsv: the CPU oracle's result (oracle_score_rolling, the
linear-space variant of the full DP) on three 100 kbp x 100 kbp windows -- start,
middle and end -- of the actual C4 genomes (synth.c4_genomes(5_000_000, "a", seed=4): G2 is a
mutated copy of G1), for the long-pair kinds the GPU tests check.  Calls only oracle/ and
synth/; the SHA-256 of each window pins the generator so a drift fails the test instead of
comparing against stale values.  Run: python tools/make_c4_windows.py (about 100 s per
window per scheme on one core; the windows run in parallel threads).
"""
import concurrent.futures as cf
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from synth import c4_genomes  # noqa: E402

W = 100_000
SCHEMES = [("local", "affine", 5), ("global", "affine", 5), ("semi", "linear", 0)]


def windows():
    g1, g2 = c4_genomes(5_000_000, "a", seed=4)
    n, m = len(g1), len(g2)
    mid1, mid2 = n // 2 - W // 2, m // 2 - W // 2
    return [("start", g1[:W], g2[:W]), ("middle", g1[mid1:mid1 + W], g2[mid2:mid2 + W]),
            ("end", g1[n - W:], g2[m - W:])]


def main():
    wins = windows()
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        for name, q, s in wins:
            for kind, gap, go in SCHEMES:
                sch = O.Scheme(kind, gap, 2, -1, go, 1)
                jobs.append((name, q, s, kind, gap, go, ex.submit(O.score_rolling, sch, q, s)))
        rows = []
        for name, q, s, kind, gap, go, fut in jobs:
            r = fut.result()
            rows.append("\t".join(str(x) for x in (
                name, hashlib.sha256(q).hexdigest()[:16], hashlib.sha256(s).hexdigest()[:16],
                kind, gap, 2, -1, go, 1, r.score, r.q_end, r.s_end)))
    out = os.path.join(ROOT, "tests", "golden", "c4_windows.tsv")
    with open(out, "w") as f:
        f.write("# written by tools/make_c4_windows.py (oracle_score_rolling on 100 kbp windows of "
                "synth.c4_genomes(5e6, 'a', seed=4))\n")
        f.write("# window\tsha256(q)[:16]\tsha256(s)[:16]\tkind\tgap\tmatch\tmismatch\topen\textend"
                "\tscore\tq_end\ts_end\n")
        f.write("\n".join(rows) + "\n")
    print(out)


if __name__ == "__main__":
    main()
