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

// The plan of one non-empty pair (n, m >= 1): its variant, its sort key and whether it
// exceeds the 32-bit range.  Shared by the device planner (classify_kernel) and the host
// API's plan of uniform ACGT-only chunks, so that both decide identically.
struct PairPlan {
  int v;
  unsigned long long key;
  bool range_err;
};
__host__ __device__ inline PairPlan plan_pair(const PlanCfg& cfg, int64_t n, int64_t m, bool hasN) {
  PairPlan pp;
  pp.v = -1;
  // range guards (reading R11): |all intermediate values| bounded by the all-gap path
  const int64_t padded = n + 192;  // max strip padding of any variant
  const int64_t neg = 3 * (int64_t)cfg.bound_go + (padded + m + 2) * (int64_t)cfg.bound_ge + 256;
  const int64_t posb = (int64_t)(cfg.bound_match > 0 ? cfg.bound_match : 0) * (padded < m ? padded : m);
  // VS16 stores scores with a +2^14 bias; Hop = H - (Go+Ge) is a packed 32-bit IMAD that
  // must not borrow across halves -> biased values stay >= Go+Ge.
  const bool ok16 = cfg.allow16 && !hasN &&
                    neg + cfg.bound_go + cfg.bound_ge <= 16000 && posb <= 16000;
  const bool ok32 = neg <= (1ll << 30) - (1ll << 24) && posb <= (1ll << 30) - (1ll << 24);
  pp.range_err = !ok32;
  if (cfg.force_variant >= 0) {
    pp.v = cfg.force_variant;
    if (variant_desc(pp.v).pairs == 2 && !ok16) pp.v = cfg.tb ? 5 : 4;
  } else {
    int64_t best_rows = 0x7fffffff;
    int best_R = 0;
    for (int c = 0; c < NV; ++c) {
      const VariantDesc d = variant_desc(c);
      if (d.tb != cfg.tb) continue;
      if (d.pairs == 2 && !ok16) continue;
      if (d.pairs == 1 && ok16) continue;
      const int64_t hs = (int64_t)d.L * d.R;
      const int64_t rows = (n + hs - 1) / hs * hs;
      if (rows < best_rows || (rows == best_rows && d.R > best_R)) {
        best_rows = rows < 0x7fffffff ? rows : 0x7fffffff;
        best_R = d.R;
        pp.v = c;
      }
    }
  }
  // plan order: by variant, then largest (m, n) first (the fill hands out slots in this
  // order, so the tail of a launch is made of the smallest slots)
  constexpr int64_t KM = (1 << 29) - 1;
  const int64_t mk = m < KM ? m : KM, nk = n < KM ? n : KM;
  pp.key = ((unsigned long long)pp.v << 58) |
           ((unsigned long long)(cfg.ascending ? mk : KM - mk) << 29) |
           (unsigned long long)(cfg.ascending ? nk : KM - nk);
  return pp;
}

}  // namespace anyseq
