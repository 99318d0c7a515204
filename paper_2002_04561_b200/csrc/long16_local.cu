// csrc/long16_local.cu -- instances of the 16-bit differential long kernel
// (long16.cuh) for KLOCAL alignments; one translation unit per kind so they compile in
// parallel.
#include "long_dev.cuh"

namespace anyseq {

#include "long16.cuh"

LongFn long16_fn_local(int nr, bool ckpt) {
  if (ckpt) return nr == 8 ? long16_kernel<8, KLOCAL, true> : long16_kernel<16, KLOCAL, true>;
  return nr == 8 ? long16_kernel<8, KLOCAL> : long16_kernel<16, KLOCAL>;
}

// several pairs in one launch (MULTI; CKPT: the traceback's forward pass)
LongFn long16_fn_local_multi(int nr, bool ckpt) {
  if (ckpt) return nr == 8 ? long16_kernel<8, KLOCAL, true, true> : long16_kernel<16, KLOCAL, true, true>;
  return nr == 8 ? long16_kernel<8, KLOCAL, false, true> : long16_kernel<16, KLOCAL, false, true>;
}

}  // namespace anyseq
