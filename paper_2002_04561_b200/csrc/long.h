// csrc/long.h -- long-pair (genome x genome) score-only driver (internal interface).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <functional>
#include <string>
#include <vector>
#include "common.cuh"

namespace anyseq {

struct LongOptions {
  int band_rows = 0;       // 0 = default (rows per warp task = 32 * R)
  int blocks = 0;          // 0 = occupancy-derived persistent grid
  int virtual_strips = 0;  // column strips on one device (0 = auto from the round count;
                           // > 0 also tests the multi-GPU protocol)
  int chunk_cols = 256;    // progress publication period (a release = full memory barrier)
  int start_lag = 0;       // columns the strip above must be ahead before a strip starts
  int profile = 0;         // print wait/task cycle counters to stderr
  int sleep_ns = 64;       // long16: row hand-off poll back-off
  int narrow = 1;          // 1: 16-bit differential kernel where eligible (local affine)
  long long spin_limit = 1ll << 28;  // poll iterations before a wait gives up (E_TIMEOUT)
  int multi_group = 2048;  // run_long_multi: pairs per launch
  int stall_task = -1;     // fault injection (tests): the warp that draws this task skips
                           // it, so the tasks that depend on it must time out
};

// Device buffers of the long-pair path kept across calls (a context owns one per device):
// slot k grows on demand, so repeated calls skip cudaMalloc / cudaFree of the row buffer,
// the boundary columns and the traceback checkpoints (tens of GB for 1 Mbp pairs).
enum { WS_QA, WS_SA, WS_QC, WS_SC, WS_SUM, WS_FLG, WS_OFF, WS_ROWBUF, WS_PROG, WS_TICKET,
       WS_ABORT, WS_CB, WS_BPTR, WS_FPTR, WS_BCOL, WS_FLAGS, WS_PARTS, WS_PROF, WS_KEY,
       WS_ROWCK, WS_COLCK,
       // long traceback walk (long_tb.cu)
       WS_TB_SCRATCH, WS_TB_OPS, WS_TB_OUT, WS_TB_SLOTS, WS_TB_SYNC, WS_TB_JOBS,
       // several pairs in one launch (run_long_multi)
       WS_M_PAIRS, WS_M_TASKS, WS_M_SEGS, WS_M_RED, WS_COUNT };

struct LongWs {
  static constexpr int kSlots = WS_COUNT;
  void* p[kSlots] = {};
  size_t cap[kSlots] = {};
  cudaError_t get(int slot, size_t bytes, void** out) {
    if (cap[slot] < bytes) {
      if (p[slot]) cudaFree(p[slot]);
      p[slot] = nullptr;
      cap[slot] = 0;
      cudaError_t e = cudaMalloc(&p[slot], bytes < 256 ? 256 : bytes);
      if (e != cudaSuccess) return e;
      cap[slot] = bytes < 256 ? 256 : bytes;
    }
    *out = p[slot];
    return cudaSuccess;
  }
  void release() {
    for (int k = 0; k < kSlots; ++k) {
      if (p[k]) cudaFree(p[k]);
      p[k] = nullptr;
      cap[k] = 0;
    }
  }
  cudaStream_t stream = nullptr;  // run_long_multi's own stream (created on first use)
  ~LongWs() {
    release();
    if (stream) cudaStreamDestroy(stream);
  }
};

struct LongDevice {
  int id;
  cudaStream_t stream;
  int num_sms;
  LongWs* ws = nullptr;  // persistent buffers (nullptr: allocate per call)
};

struct LongResult {
  int32_t score;
  int64_t end_i, end_j;
  double kernel_ms;
  bool narrow;             // the 16-bit differential kernel ran
};

// Checkpoints for the linear-space traceback (long_tb.h): with want set, run_long runs the
// 16-bit kernel's CKPT instance on ONE device and hands back (owned here, freed by release()
// or the destructor) the device codes of q and s and the checkpoint rows / columns.
struct LongCkpt {
  int want = 0;
  int64_t budget = 0;         // max device bytes for the checkpoints (0 = 40 % of free)
  int force_kc_shift = 0;     // > 0: column block 2^k (tests); else chosen from the budget
  int force_ck_every = 0;     // > 0: row checkpoint every k strips (tests)
  // outputs
  uint8_t* qc = nullptr;
  uint8_t* sc = nullptr;
  int2* rowck = nullptr;
  int2* colck = nullptr;
  int HS = 0, ck_every = 1, kc_shift = 10, PT = 0, S = 0;
  size_t bytes = 0;           // checkpoint bytes allocated
  bool owns = true;           // false: the buffers live in a LongWs
  void release();
  ~LongCkpt() { release(); }
};

// Returns 0 or an anyseq_status code; err receives a message.
int run_long(std::vector<LongDevice>& devs, const DevParams& P, const char* q, uint64_t n,
             const char* s, uint64_t m, const LongOptions& opt, LongResult* out, std::string* err,
             uint64_t* launches, LongCkpt* ck = nullptr);

// Several long pairs in ONE launch of the 16-bit kernel (device-side form;
// DESIGN.md 5.4d): score-only, one device, the pairs' row-strip tasks in one ticket queue
// (column pass by column pass; within a pass the pairs with the widest tasks first), so the
// bands of many pairs run side by side and a pair's fill/drain is covered by the others.  A pair the
// 16-bit kernel cannot take (subject with N, range guard, empty) is left alone: taken[k] = 0
// and the caller runs it through run_long.  Results of taken pairs are bit-identical to
// run_long's (same kernel body, same optimum rules).  `during` (optional) runs on the host
// while the launch is in flight (it runs even when no pair is taken); the launch uses the
// workspace's own non-blocking stream, so work `during` enqueues elsewhere overlaps it.
// cks (optional): the pass is the traceback's checkpointing forward pass (CKPT instances,
// 512-column blocks, a row checkpoint after every strip) and (*cks)[k] receives pair k's
// checkpoint view (buffers in the workspace, owns = false) for run_long_traceback; when the
// checkpoints of all pairs exceed ck_budget (0 = 40 % of free memory) no pair is taken.
struct LongPairIn {
  const char* q;
  uint64_t n;
  const char* s;
  uint64_t m;
};
int run_long_multi(LongDevice& dev, const DevParams& P, const std::vector<LongPairIn>& pairs,
                   const LongOptions& opt, std::vector<LongResult>* out, std::vector<int>* taken,
                   std::string* err, uint64_t* launches, double* kernel_ms,
                   const std::function<int()>& during = {}, int* rows_out = nullptr,
                   std::vector<LongCkpt>* cks = nullptr, int64_t ck_budget = 0);

}  // namespace anyseq
