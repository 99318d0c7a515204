// csrc/fill_tb.cu -- traceback instances (the fill stores every cell's H for the walk).
#include "fill_inst.cuh"
namespace anyseq {
FillFn fill_fn_tb(int v, int kind, int gap, bool pos) {
  switch (v) {
    case 5: return fill_fn<VS32, 8, 8, true>(kind, gap, pos);
    case 6: return fill_fn<VS16, 8, 8, true>(kind, gap, pos);
    case 7: return fill_fn<VS16, 8, 19, true>(kind, gap, pos);
    default: return nullptr;
  }
}
}  // namespace anyseq
