// csrc/fill_inst.cuh -- explicit instantiation helpers for the fill kernel variants.
#pragma once
#include "fill_kernel.cuh"

namespace anyseq {

typedef void (*FillFn)(FillArgs);

template <class V, int L, int R, bool TB>
FillFn fill_fn(int kind, int gap) {
  if (kind == KGLOBAL) return gap == GAFFINE ? fill_kernel<V, KGLOBAL, GAFFINE, L, R, TB>
                                             : fill_kernel<V, KGLOBAL, GLINEAR, L, R, TB>;
  if (kind == KLOCAL) return gap == GAFFINE ? fill_kernel<V, KLOCAL, GAFFINE, L, R, TB>
                                            : fill_kernel<V, KLOCAL, GLINEAR, L, R, TB>;
  return gap == GAFFINE ? fill_kernel<V, KSEMI, GAFFINE, L, R, TB>
                        : fill_kernel<V, KSEMI, GLINEAR, L, R, TB>;
}

}  // namespace anyseq
