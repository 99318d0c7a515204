// csrc/long_tb.h -- checkpointed linear-space long-pair traceback.
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include "long.h"

namespace anyseq {

// Walks the traceback of a long pair from (end_i, end_j) back to its begin cell using the
// checkpoints of a CKPT forward pass (run_long with ck->want set).  ops receives the CIGAR in
// alignment order (BAM-style words, op 0 = M, 1 = I, 2 = D); *begin_i/*begin_j the begin
// cell; *walk_ms the device time of the walk; walk_helpers CTAs recompute predicted next
// tiles ahead of the walker (0 = the walker alone); *tiles / *hits count the tiles walked
// and those found precomputed.  Returns 0 or an anyseq_status.
int run_long_traceback(const LongDevice& dev, const DevParams& P, const int8_t sig[25],
                       const LongCkpt& ck, int64_t end_i, int64_t end_j, int64_t n, int64_t m,
                       std::vector<uint32_t>* ops, int64_t* begin_i, int64_t* begin_j,
                       double* walk_ms, std::string* err, uint64_t* launches,
                       int walk_helpers = 96, int64_t* tiles = nullptr, int64_t* hits = nullptr,
                       bool trace = false);

}  // namespace anyseq
