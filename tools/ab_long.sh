# A/B of long-kernel builds on one box: tools/ab/libanyseq_A.so vs the in-tree library,
# alternating, C4 (5 Mbp local affine) kernel time.
for r in 1 2; do
  ANYSEQ_LIB=$PWD/tools/ab/libanyseq_A.so python tools/long_lag.py 5000000 0 2>&1 | head -1 | sed 's/^/A: /'
  python tools/long_lag.py 5000000 0 2>&1 | head -1 | sed 's/^/B: /'
done
