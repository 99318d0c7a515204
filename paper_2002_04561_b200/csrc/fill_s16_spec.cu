// csrc/fill_s16_spec.cu -- VS16 score-only instances with the paper's own schemes compiled in
// (Fig. 5): affine (G_o, G_e) = (2, 1) and linear g = 1.
#include "fill_inst.cuh"
namespace anyseq {
// spec 2: affine (2, 1)
FillFn fill_fn_s16_spec_a21(int v, int kind, bool pos) {
  switch (v) {
    case 0: return pos ? fill_fn_spec<VS16, 8, 8, true, GAFFINE, 1, 2>(kind) : fill_fn_spec<VS16, 8, 8, false, GAFFINE, 1, 2>(kind);
    case 1: return pos ? fill_fn_spec<VS16, 8, 16, true, GAFFINE, 1, 2>(kind) : fill_fn_spec<VS16, 8, 16, false, GAFFINE, 1, 2>(kind);
    case 2: return pos ? fill_fn_spec<VS16, 8, 19, true, GAFFINE, 1, 2>(kind) : fill_fn_spec<VS16, 8, 19, false, GAFFINE, 1, 2>(kind);
    default: return nullptr;
  }
}
// spec 3: linear g = 1
FillFn fill_fn_s16_spec_l1(int v, int kind, bool pos) {
  switch (v) {
    case 0: return pos ? fill_fn_spec<VS16, 8, 8, true, GLINEAR, 1, 0>(kind) : fill_fn_spec<VS16, 8, 8, false, GLINEAR, 1, 0>(kind);
    case 1: return pos ? fill_fn_spec<VS16, 8, 16, true, GLINEAR, 1, 0>(kind) : fill_fn_spec<VS16, 8, 16, false, GLINEAR, 1, 0>(kind);
    case 2: return pos ? fill_fn_spec<VS16, 8, 19, true, GLINEAR, 1, 0>(kind) : fill_fn_spec<VS16, 8, 19, false, GLINEAR, 1, 0>(kind);
    default: return nullptr;
  }
}
}  // namespace anyseq
