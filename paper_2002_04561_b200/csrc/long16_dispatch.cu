// csrc/long16_dispatch.cu -- 16-bit long kernel instance by kind (long_dev.cuh).
#include "long_dev.cuh"

namespace anyseq {

LongFn long16_fn_global(int nr, bool ckpt);
LongFn long16_fn_local(int nr, bool ckpt);
LongFn long16_fn_semi(int nr, bool ckpt);
LongFn long16_fn_global_multi(int nr, bool ckpt);
LongFn long16_fn_local_multi(int nr, bool ckpt);
LongFn long16_fn_semi_multi(int nr, bool ckpt);

LongFn long16_fn(int nr, int kind, bool ckpt) {
  return kind == KGLOBAL ? long16_fn_global(nr, ckpt)
       : kind == KLOCAL ? long16_fn_local(nr, ckpt) : long16_fn_semi(nr, ckpt);
}

LongFn long16_multi_fn(int kind, int nr, bool ckpt) {
  return kind == KGLOBAL ? long16_fn_global_multi(nr, ckpt)
       : kind == KLOCAL ? long16_fn_local_multi(nr, ckpt) : long16_fn_semi_multi(nr, ckpt);
}

}  // namespace anyseq
