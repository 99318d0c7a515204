// csrc/fill_inst.cuh -- explicit instantiation helpers for the fill kernel variants.
#pragma once
#include "fill_kernel.cuh"

namespace anyseq {

typedef void (*FillFn)(FillArgs);

// compile-time scoring constants (the paper's partial evaluation of the scheme):
// GAP = affine with (G_o, G_e) = (CGO, CGE), or linear with g = CGE (CGO unused)
template <class V, int L, int R, bool POS, int GAP, int CGE, int CGO>
FillFn fill_fn_spec(int kind) {
  if (kind == KGLOBAL) return fill_kernel<V, KGLOBAL, GAP, L, R, false, POS, CGE, CGO>;
  if (kind == KLOCAL) return fill_kernel<V, KLOCAL, GAP, L, R, false, POS, CGE, CGO>;
  return fill_kernel<V, KSEMI, GAP, L, R, false, POS, CGE, CGO>;
}

template <class V, int L, int R, bool TB, bool POS>
FillFn fill_fn_p(int kind, int gap) {
  if (kind == KGLOBAL) return gap == GAFFINE ? fill_kernel<V, KGLOBAL, GAFFINE, L, R, TB, POS>
                                             : fill_kernel<V, KGLOBAL, GLINEAR, L, R, TB, POS>;
  if (kind == KLOCAL) return gap == GAFFINE ? fill_kernel<V, KLOCAL, GAFFINE, L, R, TB, POS>
                                            : fill_kernel<V, KLOCAL, GLINEAR, L, R, TB, POS>;
  return gap == GAFFINE ? fill_kernel<V, KSEMI, GAFFINE, L, R, TB, POS>
                        : fill_kernel<V, KSEMI, GLINEAR, L, R, TB, POS>;
}

// score-only instances come in two flavours: plain (POS = false) and with end cells
template <class V, int L, int R, bool TB>
FillFn fill_fn(int kind, int gap, bool pos) {
  if constexpr (TB) {
    return fill_fn_p<V, L, R, true, true>(kind, gap);
  } else {
    return pos ? fill_fn_p<V, L, R, false, true>(kind, gap) : fill_fn_p<V, L, R, false, false>(kind, gap);
  }
}

}  // namespace anyseq
