// csrc/fill_s16.cu -- VS16 (two alignments per register) score-only instances.
#include "fill_inst.cuh"
namespace anyseq {
FillFn fill_fn_s16_spec(int v, int kind, bool pos) {
  switch (v) {
    case 0: return pos ? fill_fn_spec<VS16, 8, 8, true>(kind) : fill_fn_spec<VS16, 8, 8, false>(kind);
    case 1: return pos ? fill_fn_spec<VS16, 8, 16, true>(kind) : fill_fn_spec<VS16, 8, 16, false>(kind);
    case 2: return pos ? fill_fn_spec<VS16, 8, 19, true>(kind) : fill_fn_spec<VS16, 8, 19, false>(kind);
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
