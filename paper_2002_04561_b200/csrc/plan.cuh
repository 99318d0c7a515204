// csrc/plan.cuh -- host/device shared plan definitions (variants, summary).
#pragma once
#include <cstdint>
#include "common.cuh"

namespace anyseq {

// A fill variant = register width x lane-group size x rows per lane x traceback.
// Kind and gap are orthogonal template parameters (one instance per kind x gap).
struct VariantDesc {
  int pairs;  // 2 = VS16 (two alignments per register), 1 = VS32
  int L;      // lanes per group
  int R;      // rows per lane
  int tb;     // 1 = traceback fill (stores every cell's H)
};

constexpr int NV = 8;
// Score-only variants: s16x2 with R in {8,16,19} (19*8 = 152 rows fits 150 bp reads with
// one strip), s32 with R in {8,16}; traceback variants: s32 / s16x2 with R = 8.
__host__ __device__ inline VariantDesc variant_desc(int v) {
  switch (v) {
    case 0: return {2, 8, 8, 0};
    case 1: return {2, 8, 16, 0};
    case 2: return {2, 8, 19, 0};
    case 3: return {1, 8, 8, 0};
    case 4: return {1, 8, 16, 0};
    case 5: return {1, 8, 8, 1};
    case 6: return {2, 8, 8, 1};
    case 7: return {2, 8, 19, 1};
    default: return {0, 0, 0, 0};
  }
}

// Per-call plan summary (device -> host once per call).
struct PlanSummary {
  unsigned long long err_pos;  // min global byte position of an invalid symbol (q then s)
  int32_t count[NV];           // pairs per variant
  int32_t maxn[NV], maxm[NV];
  unsigned long long kmin[NV], kmax[NV];
  int32_t range_err;           // a pair exceeds the 32-bit score range
  int32_t blocks_done;         // classify's last-block detection
};

// Planner inputs decided on the host.
struct PlanCfg {
  int32_t tb;          // traceback mode: only traceback variants are eligible
  int32_t allow16;     // s16x2 permitted (debug/tests can force s32)
  int32_t force_variant;  // -1 = auto
  int32_t bound_go, bound_ge, bound_match;  // for the range guards
  int32_t ascending;   // plan order smallest-first (debug; default largest-first)
};

}  // namespace anyseq
