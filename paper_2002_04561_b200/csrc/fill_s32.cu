// csrc/fill_s32.cu -- VS32 score-only instances.
#include "fill_inst.cuh"
namespace anyseq {
FillFn fill_fn_s32(int v, int kind, int gap, bool pos) {
  switch (v) {
    case 3: return fill_fn<VS32, 8, 8, false>(kind, gap, pos);
    case 4: return fill_fn<VS32, 8, 16, false>(kind, gap, pos);
    default: return nullptr;
  }
}
}  // namespace anyseq
