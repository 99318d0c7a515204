# A/B of long-kernel builds on one box, alternating: C4 (5 Mbp local affine) kernel time.
# usage: bash tools/ab_long.sh tools/ab/libX.so [tools/ab/libY.so ...]   (in-tree lib = "cur")
for r in 1 2; do
  for lib in "$@"; do
    ANYSEQ_LIB=$PWD/$lib python tools/long_lag.py 5000000 0 2>&1 | head -1 | sed "s#^#$(basename $lib): #"
  done
  python tools/long_lag.py 5000000 0 2>&1 | head -1 | sed 's/^/cur: /'
done
