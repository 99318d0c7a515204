# Build an A/B variant of libanyseq.so: recompile the listed sources with extra nvcc flags
# and link them with the in-tree objects of everything else.
# usage: bash tools/ab_build.sh NAME "FLAGS" src1.cu [src2.cu ...]  -> tools/ab/libanyseq_NAME.so
set -e
name=$1; flags=$2; shift 2
B=paper_2002_04561_b200/build; C=paper_2002_04561_b200/csrc
mkdir -p tools/ab /tmp/ab_$name
objs=""
for o in $B/*.o; do
  s=$(basename $o .o).cu
  if printf '%s\n' "$@" | grep -qx "$s"; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr -I include -I $C $flags -c $C/$s -o /tmp/ab_$name/$s.o
    objs="$objs /tmp/ab_$name/$s.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/ab/libanyseq_$name.so $objs -Xcompiler -fPIC
echo tools/ab/libanyseq_$name.so
