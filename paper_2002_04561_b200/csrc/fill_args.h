// csrc/fill_args.h -- argument block of the fill kernel (host + device).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace anyseq {

struct FillArgs {
  DevParams P;
  const uint8_t* qcode;
  const uint8_t* scode;
  const uint64_t* q_off;
  const uint64_t* s_off;
  const Slot* slots;          // this variant's slot array
  const int32_t* nslots_dev;  // if non-null: slot range is [0, *nslots_dev)
  int32_t slot_lo, slot_hi;   // otherwise [slot_lo, slot_hi)
  int32_t* ticket;            // if non-null (zeroed): warp-slots handed out dynamically
  int32_t pos;                // also produce end cells
  int32_t* scores;            // [num_pairs]
  int32_t* end_i;             // [num_pairs] (pos)
  int32_t* end_j;
  uint4* strip_scratch;       // per resident lane group: strip_stride entries (H, E, bits)
  int64_t strip_stride;
  uint32_t* dirs;             // TB: per-cell H store (one 32-bit word per lane, row, diagonal)
  int64_t dir_block_words;    // TB: words per slot block (fixed per launch)
  TbInfo* tb;                 // TB: per pair
  int32_t tb8;                // TB: store only the low byte of H per cell (the walk rebuilds
                              // H from neighbour differences, |dH| < 128: DESIGN.md 5.3)
  int32_t defer_row;          // TB local: the end row is resolved by the walk (TbInfo::end_span)
  int32_t one;                // = 1 at run time (keeps IMAD-based adds on the FMA pipe)
  uint32_t nge_s16;           // packed (-Ge, -Ge): read from the constant bank in the hot loop
  uint32_t koc_s16;           // -(Go+Ge)*65537 (biased VS16 Hop addend)
};

}  // namespace anyseq
