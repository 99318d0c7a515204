// csrc/long16_semi.cu -- instances of the 16-bit differential long kernel
// (long16.cuh) for KSEMI alignments; one translation unit per kind so they compile in
// parallel.
#include "long_dev.cuh"

namespace anyseq {

#include "long16.cuh"

LongFn long16_fn_semi(int nr, bool ckpt) {
  if (ckpt) return nr == 8 ? long16_kernel<8, KSEMI, true> : long16_kernel<16, KSEMI, true>;
  return nr == 8 ? long16_kernel<8, KSEMI> : long16_kernel<16, KSEMI>;
}

// several pairs in one launch (MULTI; CKPT: the traceback's forward pass)
LongFn long16_fn_semi_multi(int nr, bool ckpt) {
  if (ckpt) return nr == 8 ? long16_kernel<8, KSEMI, true, true> : long16_kernel<16, KSEMI, true, true>;
  return nr == 8 ? long16_kernel<8, KSEMI, false, true> : long16_kernel<16, KSEMI, false, true>;
}

}  // namespace anyseq
