// csrc/kernels.h -- host-callable launchers of the device kernels (internal interface).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "common.cuh"
#include "plan.cuh"
#include "fill_args.h"

namespace anyseq {

// a1: ASCII -> byte codes (A,C,G,T -> 0..3, N -> 4), validation, per-pair N flags; q and s
// in one launch.
cudaError_t launch_pack(const char* d_q, uint64_t q_len, uint8_t* d_qcode, const uint64_t* d_qoff,
                        const char* d_s, uint64_t s_len, uint8_t* d_scode, const uint64_t* d_soff,
                        uint64_t num_pairs, uint32_t* d_flags, PlanSummary* d_sum,
                        cudaStream_t st, int num_sms);

// a1, 2-bit path (host API, ACGT-only chunks): expand 2-bit codes (base p in bits 2 (p % 4)
// of byte p / 4, packed on the host) into byte codes 0..3; q and s in one launch.  No
// validation is needed (the host packer admits only ACGTacgt) and no pair has an N.
cudaError_t launch_unpack2(const uint8_t* d_q2, uint64_t q_len, uint8_t* d_qcode,
                           const uint8_t* d_s2, uint64_t s_len, uint8_t* d_scode,
                           cudaStream_t st, int num_sms);

// per-call plan state: clear the per-pair flags, initialise the device summary and (host-API
// chunks, qoff != null) rebase the verbatim-uploaded offsets to the chunk's first byte
// fill-launch slot counters zeroed by prep (one per fill launch of a call; more launches
// than this fall back to static slot assignment)
constexpr int kNumTickets = 64;
cudaError_t launch_prep(uint32_t* flags, uint64_t n, PlanSummary* sum, uint64_t* qoff,
                        uint64_t* soff, uint64_t q0, uint64_t s0, int64_t gq, int64_t gs,
                        int32_t* tickets, cudaStream_t st, int num_sms);

struct ClassifyArgs {
  DevParams P;
  PlanCfg cfg;
  const uint64_t* q_off;
  const uint64_t* s_off;
  uint64_t num_pairs;
  const uint32_t* flags;
  PlanSummary* sum;
  PlanSummary* host_sum;     // host-mapped copy written by the last block
  Slot* slots;               // speculative uniform-case slots
  unsigned long long* keys;  // [num_pairs]
  int32_t* vals;             // [num_pairs]
  int32_t* scores;           // trivial pairs are finished here
  int32_t* end_i;
  int32_t* end_j;
  // traceback mode bookkeeping for trivial pairs
  uint32_t* ops;             // per-pair run region base q_off+s_off+k
  int32_t* n_ops;
  int32_t* beg_i;
  int32_t* beg_j;
  // > 0: pairs with n, m >= skip_min and n * m >= skip_cells are not planned (key ~0,
  // outputs untouched): the host API aligns them on the long-pair path (run_host_batch)
  int64_t skip_cells;
  int64_t skip_min;
};
// a2: plan -- variant choice, range guard, sort keys; finishes empty pairs.
cudaError_t launch_classify(const ClassifyArgs& a, cudaStream_t st, int num_sms);

// a2: slot formation from the (sorted) order
cudaError_t launch_slots(const int32_t* d_order, int64_t num, const int32_t* voff_host,
                         const int32_t* count_host, const int32_t* sbase_host, Slot* d_slots,
                         cudaStream_t st, int num_sms);

// radix sort (cub) of (key, pair) -- temp storage managed by the caller
cudaError_t sort_pairs(void* d_temp, size_t& temp_bytes, const unsigned long long* keys_in,
                       unsigned long long* keys_out, const int32_t* vals_in, int32_t* vals_out,
                       int64_t num, cudaStream_t st);
cudaError_t exclusive_scan_i32_to_u64(void* d_temp, size_t& temp_bytes, const int32_t* in,
                                      uint64_t* out, int64_t num, cudaStream_t st);

// a3/a4: fill (template dispatch)
cudaError_t launch_fill(int variant, int kind, int gap, const FillArgs& a, cudaStream_t st,
                        int num_sms, int* grid_out);

// a5: traceback walk of one chunk of slots of a variant
struct WalkArgs {
  int32_t kind, gap;
  DevParams P;
  const uint8_t* qcode;  // byte codes at the CSR positions (sigma of the DIAG test)
  const uint8_t* scode;
  const Slot* slots;
  int32_t slot_lo, slot_hi;
  int32_t pairs_per_slot;
  const TbInfo* tb;
  const uint32_t* dirs;
  int32_t tb8;     // the H store holds low bytes (FillArgs::tb8)
  const uint64_t* q_off;
  const uint64_t* s_off;
  uint32_t* ops;   // per-pair run region (reversed run order)
  int32_t* n_ops;
  int32_t* beg_i;
  int32_t* beg_j;
  int32_t* end_i;  // end rows resolved by the walk (TbInfo::end_span > 0)
};
cudaError_t launch_walk(const WalkArgs& a, cudaStream_t st, int num_sms);

// output assembly (anyseq_alignment layout, see include/anyseq.h)
struct FinalizeArgs {
  uint64_t num_pairs;
  const int32_t* scores;
  const int32_t* end_i;
  const int32_t* end_j;
  const int32_t* beg_i;   // null => begin = end
  const int32_t* beg_j;
  const int32_t* n_ops;   // null => no cigar
  const uint64_t* cig_off;
  const uint64_t* q_off;
  const uint64_t* s_off;
  const uint32_t* ops;
  void* out_aln;          // anyseq_alignment[num_pairs]
  uint32_t* cigar;        // compacted cigar (may be null)
  uint64_t cigar_cap;
  uint64_t cig_base;      // added to every output cigar_offset
};
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st, int num_sms);

}  // namespace anyseq
