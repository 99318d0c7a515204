// csrc/nvtx.h -- NVTX ranges around the host API's phases (SURVEY §5 tracing): visible in
// Nsight Systems / ncu --nvtx; without an attached tool each push/pop is a no-op call.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace anyseq {

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace anyseq
