// csrc/long16_global.cu -- instances of the 16-bit differential long kernel
// (long16.cuh) for KGLOBAL alignments; one translation unit per kind so they compile in
// parallel.
#include "long_dev.cuh"

namespace anyseq {

#include "long16.cuh"

LongFn long16_fn_global(int nr, bool ckpt) {
  if (ckpt) return nr == 8 ? long16_kernel<8, KGLOBAL, true> : long16_kernel<16, KGLOBAL, true>;
  return nr == 8 ? long16_kernel<8, KGLOBAL> : long16_kernel<16, KGLOBAL>;
}

// several pairs in one launch (MULTI; CKPT: the traceback's forward pass)
LongFn long16_fn_global_multi(int nr, bool ckpt) {
  if (ckpt) return nr == 8 ? long16_kernel<8, KGLOBAL, true, true> : long16_kernel<16, KGLOBAL, true, true>;
  return nr == 8 ? long16_kernel<8, KGLOBAL, false, true> : long16_kernel<16, KGLOBAL, false, true>;
}

}  // namespace anyseq
