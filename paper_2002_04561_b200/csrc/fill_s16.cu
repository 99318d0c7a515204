// csrc/fill_s16.cu -- VS16 (two alignments per register) score-only instances.
#include "fill_inst.cuh"
namespace anyseq {
// spec 1: affine (G_o, G_e) = (5, 1), the C2-C5 scheme (readings R18/R19)
FillFn fill_fn_s16_spec(int v, int kind, bool pos) {
  switch (v) {
    case 0: return pos ? fill_fn_spec<VS16, 8, 8, true, GAFFINE, 1, 5>(kind) : fill_fn_spec<VS16, 8, 8, false, GAFFINE, 1, 5>(kind);
    case 1: return pos ? fill_fn_spec<VS16, 8, 16, true, GAFFINE, 1, 5>(kind) : fill_fn_spec<VS16, 8, 16, false, GAFFINE, 1, 5>(kind);
    case 2: return pos ? fill_fn_spec<VS16, 8, 19, true, GAFFINE, 1, 5>(kind) : fill_fn_spec<VS16, 8, 19, false, GAFFINE, 1, 5>(kind);
    default: return nullptr;
  }
}
FillFn fill_fn_s16(int v, int kind, int gap, bool pos) {
  switch (v) {
    case 0: return fill_fn<VS16, 8, 8, false>(kind, gap, pos);
    case 1: return fill_fn<VS16, 8, 16, false>(kind, gap, pos);
    case 2: return fill_fn<VS16, 8, 19, false>(kind, gap, pos);
    default: return nullptr;
  }
}
}  // namespace anyseq
