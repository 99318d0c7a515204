// csrc/api.cu -- the anyseq_* C-ABI (include/anyseq.h): context, validation, planner
// orchestration, host <-> device staging, multi-GPU sharding of batches.
//
// Control flow per call follows the paper's ten steps: allocate/read input
// (H2D of the caller's ASCII CSR), allocate output, build accessors (pack kernel -> byte
// codes), allocate temporaries (context-owned device buffers), relax (fill kernels),
// look up the optimum (fused into the fill epilogue), build alignments if needed (walk +
// compaction kernels), output (D2H).
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <functional>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/anyseq.h"
#include "kernels.h"
#include "long.h"
#include "hirschberg.h"
#include "hostpack.h"
#include "nvtx.h"
#include "long_tb.h"

using namespace anyseq;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Growable pinned host buffer (staging for device->host results into pageable memory).
struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMallocHost(&p, std::max<size_t>(bytes, 4096));
    if (e == cudaSuccess) cap = std::max<size_t>(bytes, 4096);
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

bool host_pinned(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

struct Device {
  int id = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  DevBuf q_ascii, s_ascii, q_code, s_code, q_off, s_off, flags, keys, keys2, vals, vals2, slots;
  DevBuf scores, end_i, end_j, beg_i, beg_j, n_ops, cig_off, ops, dirs, tb, strip, aln, cigar;
  DevBuf temp, sum, long_ws, tickets;
  DevBuf q_ascii2[2], s_ascii2[2], q_off2[2], s_off2[2];  // double-buffered host uploads
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_up[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  PlanSummary* h_sum = nullptr;  // pinned, mapped (written by the publish kernel)
  HostBuf h_stage;               // pinned staging of score-mode results
  HostBuf h_pack[3];             // pinned 2-bit packed chunks (host API, ACGT-only chunks)
  // score-mode variant launches of one plan run concurrently (each with its own strip
  // scratch): small per-variant launches of mixed-length batches then share the GPU
  DevBuf strip_v[NV], dirs_v[NV];
  cudaStream_t vstream[NV] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[NV] = {};
  uint64_t* h_small = nullptr;   // pinned scratch
};

}  // namespace

struct anyseq_ctx {
  std::vector<Device> devs;
  std::vector<std::unique_ptr<LongWs>> lws;  // per device entry: long-pair buffers kept across calls
  std::string err;
  std::atomic<uint64_t> launches{0};
  int64_t tb_scratch_bytes = 16ll << 30;  // traceback H store per fill/walk chunk
  int64_t chunk_bytes = 64ll << 20;  // host-API upload/compute pipelining granularity
  int64_t force_variant = -1;
  int64_t allow16 = 1;
  int64_t batch_long_cells = 1ll << 22;  // batch pairs this large take the long-pair path
  int64_t batch_long_min = 2048;         // ... when both sides are at least this long
  int64_t batch_long_cells_tb = 1ll << 22;  // traceback mode's threshold
  int64_t batch_long_small = 4;  // batches of at most this many pairs: every pair with both
                                 // sides >= 256 takes the long-pair path
  int64_t tb8 = 1;          // traceback: 1-byte H store where the range allows
  int64_t pack2 = 1;        // host API: upload ACGT-only chunks as 2-bit codes
  int64_t pack2_percent = 0;  // share of the bytes packed (0 = all)
  std::unique_ptr<PackPool> packpool;  // host packing threads (created on first use)
  PackPool* shared_pool = nullptr;  // per-device shard contexts use the parent's pool
  std::mutex pool_mu;
  PackPool* packer() {
    if (shared_pool) return shared_pool;
    std::lock_guard<std::mutex> lk(pool_mu);
    // one core stays with the thread that drives the device (it waits on the plan summary)
    if (!packpool)
      packpool.reset(new PackPool((int)std::max(1u, std::thread::hardware_concurrency() - 1)));
    return packpool.get();
  }
  int64_t tb_leaf_cells = 1 << 20;  // long traceback: Hirschberg leaf size (cells)
  double tb_leaf_ms = 0;            // last anyseq_traceback_long: host time of the leaves
  LongOptions long_opt;
  int64_t long_multi = 1;  // mixed batches: long pairs share one launch (run_long_multi)
  int64_t skip_cells = 0;  // set by run_host_batch for its batch-kernel pass (DeviceJob)
  int64_t long_multi_pairs = 0;   // ... pairs the last batch call ran that way
  double long_multi_ms = 0;       // ... and that launch's kernel time
  int long_multi_rows = 0;        // ... and its rows per warp task (512 or 1024)
  int long_narrow = 0;   // the last anyseq_align_long ran the 16-bit differential kernel
  double long_ms = 0;    // ... and its kernel time (max over devices)
  double tb_pass_ms = 0, tb_pass_cells = 0;  // last anyseq_traceback_long: forward pass(es)
  double tb_walk_ms = 0, tb_ckpt_bytes = 0;   // ... checkpointed walk time, checkpoint bytes
  double tb_tiles = 0, tb_hits = 0;           // ... tiles walked, found precomputed by helpers
  int64_t walk_helpers = 96;                  // helper CTAs of the walk
  int64_t tb_budget = 0, tb_kc_shift = 0, tb_ck_every = 0;  // options (0 = automatic)
  int tb_method = 0;  // last anyseq_traceback_long: 1 = checkpoints, 2 = Hirschberg
  int timing = 0;
  std::mutex ev_mu;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> fill_ev, walk_ev, pool;
  double fill_ms = 0, walk_ms = 0;
  std::atomic<uint64_t> h2d_bytes{0}, d2h_bytes{0};  // host API sequence / result traffic
  uint64_t fill_launches = 0;
  // timing >= 2: labelled events on the device streams, printed by the host API (debug)
  std::vector<std::pair<std::string, cudaEvent_t>> trace;
  void mark(cudaStream_t x, const std::string& label) {
    if (timing < 2) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, x);
    std::lock_guard<std::mutex> lk(ev_mu);
    trace.emplace_back(label, e);
  }
  void dump_trace() {
    if (trace.empty()) return;
    std::vector<std::pair<float, std::string>> rows;
    for (auto& t : trace) {
      float ms = 0;
      cudaEventSynchronize(t.second);
      cudaEventElapsedTime(&ms, trace[0].second, t.second);
      rows.emplace_back(ms, t.first);
    }
    std::stable_sort(rows.begin(), rows.end(),
                     [](const auto& x, const auto& y) { return x.first < y.first; });
    for (auto& r : rows) fprintf(stderr, "[trace] %8.3f ms  %s\n", r.first, r.second.c_str());
    for (auto& t : trace) cudaEventDestroy(t.second);
    trace.clear();
  }
};

namespace {

const char* kStatus[] = {"ok",          "invalid argument", "invalid sequence byte",
                         "out of memory", "cigar capacity too small", "CUDA error",
                         "unsupported",  "peer access unavailable", "timeout"};

anyseq_status fail(anyseq_ctx* c, anyseq_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) {
    try {
      c->err = buf;
    } catch (...) {  // no exception crosses the ABI, not even from the error path
    }
  }
  return s;
}

// Every extern "C" body runs inside abi_guard: a host allocation failure (std::bad_alloc
// from a vector, a string or a thread) becomes ANYSEQ_E_NOMEM and any other C++ exception
// ANYSEQ_E_CUDA, so nothing but a status code crosses the C ABI (include/anyseq.h).
template <class F>
anyseq_status abi_guard(anyseq_ctx* c, F&& body) {
  try {
    return body();
  } catch (const std::bad_alloc&) {
    return fail(c, ANYSEQ_E_NOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(c, ANYSEQ_E_CUDA, "internal error: %s", e.what());
  } catch (...) {
    return fail(c, ANYSEQ_E_CUDA, "internal error");
  }
}

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      if (e_ == cudaErrorMemoryAllocation)                                              \
        return fail(ctx, ANYSEQ_E_NOMEM, "%s: %s", #call, cudaGetErrorString(e_));      \
      return fail(ctx, ANYSEQ_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_));         \
    }                                                                                   \
  } while (0)

std::pair<cudaEvent_t, cudaEvent_t> take_events(anyseq_ctx* c) {
  std::lock_guard<std::mutex> lk(c->ev_mu);
  if (!c->pool.empty()) {
    auto e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  std::pair<cudaEvent_t, cudaEvent_t> e{nullptr, nullptr};
  cudaEventCreate(&e.first);
  cudaEventCreate(&e.second);
  return e;
}

void resolve_events(anyseq_ctx* c) {
  std::lock_guard<std::mutex> lk(c->ev_mu);
  for (int w = 0; w < 2; ++w) {
    auto& v = w == 0 ? c->fill_ev : c->walk_ev;
    for (auto& e : v) {
      cudaEventSynchronize(e.second);
      float ms = 0;
      cudaEventElapsedTime(&ms, e.first, e.second);
      (w == 0 ? c->fill_ms : c->walk_ms) += ms;
      c->pool.push_back(e);
    }
    v.clear();
  }
}

anyseq_status validate_params(anyseq_ctx* ctx, const anyseq_params* p) {
  if (!p) return fail(ctx, ANYSEQ_E_INVALID, "params is NULL");
  if (p->kind < 0 || p->kind > 2) return fail(ctx, ANYSEQ_E_INVALID, "kind %d invalid", p->kind);
  if (p->gap < 0 || p->gap > 1) return fail(ctx, ANYSEQ_E_INVALID, "gap %d invalid", p->gap);
  if (p->match < -128 || p->match > 127 || p->mismatch < -128 || p->mismatch > 127)
    return fail(ctx, ANYSEQ_E_INVALID, "match/mismatch must be in [-128,127]");
  if (p->has_subst)
    for (int k = 0; k < 25; ++k)
      if (p->subst[k] < -128 || p->subst[k] > 127)
        return fail(ctx, ANYSEQ_E_INVALID, "subst[%d] must be in [-128,127]", k);
  if (p->gap_extend < 0 || p->gap_extend > 32767)
    return fail(ctx, ANYSEQ_E_INVALID, "gap_extend must be in [0,32767]");
  if (p->gap == ANYSEQ_GAP_AFFINE && (p->gap_open < 0 || p->gap_open > 32767))
    return fail(ctx, ANYSEQ_E_INVALID, "gap_open must be in [0,32767]");
  return ANYSEQ_OK;
}

DevParams dev_params(const anyseq_params* p) {
  DevParams d;
  d.kind = p->kind;
  d.gap = p->gap;
  d.match = p->match;
  d.mismatch = p->mismatch;
  d.go = p->gap == ANYSEQ_GAP_AFFINE ? p->gap_open : 0;
  d.ge = p->gap_extend;
  // sigma tables: simple_subst_scoring(match, mismatch) with N mismatching everything
  // (reading R12) or the caller's 5x5 matrix
  d.smax = -1 << 30;
  for (int a = 0; a < 5; ++a) {
    d.prof[a] = 0;
    for (int b = 0; b < 5; ++b) {
      const int v = p->has_subst ? p->subst[5 * a + b] : ((a == b && a < 4) ? p->match : p->mismatch);
      d.smax = std::max(d.smax, v);
      if (b < 4) d.prof[a] |= ((uint32_t)(v & 0xff)) << (8 * b);
      else d.pn[a] = ((uint32_t)(v & 0xff)) * 0x01010101u;
    }
  }
  return d;
}


// Device-side batch job: offsets and sequences are already in device memory.
struct DeviceJob {
  const char* d_q;
  const uint64_t* d_qoff;
  const char* d_s;
  const uint64_t* d_soff;
  uint64_t B;
  uint64_t q_end, s_end;      // q_off[B], s_off[B] (absolute ends; codes are indexed absolutely)
  int tb;                     // traceback mode
  int want_ends;              // score mode: fill end cells + alignment structs
  uint64_t* rebase_qoff = nullptr;  // host-API chunk: offsets to rebase by (q0, s0) first
  uint64_t* rebase_soff = nullptr;
  uint64_t rebase_q0 = 0, rebase_s0 = 0;
  int64_t gen_q = -1, gen_s = -1;   // >= 0: offsets are k * gen (not uploaded), see prep
  int packed2 = 0;                  // d_q / d_s hold 2-bit codes (host-packed ACGT-only chunk)
  int64_t skip_cells = 0;           // score mode: pairs this large are left to the long path
  int64_t skip_min = 2048;          // ... when both sides have at least this many bases
  uint64_t cig_base = 0;            // traceback: added to every cigar_offset of this job
  int32_t* d_scores_out;      // score mode output (device) or null => ctx buffer
  anyseq_alignment* d_aln_out;  // alignment structs (device) or null => ctx buffer
  // traceback: cigar sizing results
  uint64_t cigar_total = 0;
  // traceback: called once the chunk's kernels are enqueued, before run_device blocks on
  // the CIGAR total (the host API issues the next chunk's upload here, so it overlaps this
  // chunk's fill and walk)
  std::function<anyseq_status()> before_sync;
};

anyseq_status run_device(anyseq_ctx* ctx, Device& D, const anyseq_params* prm, DeviceJob& J,
                         uint32_t* d_cigar_out_or_null, uint64_t cigar_cap) {
  NvtxRange nvtx(J.tb ? "enqueue traceback chunk" : "enqueue score chunk");
  cudaStream_t st = D.stream;
  const uint64_t B = J.B;
  const DevParams P = dev_params(prm);
  auto L = [&](uint64_t n) { ctx->launches += n; };

  CK(D.q_code.ensure(J.q_end + 16));
  CK(D.s_code.ensure(J.s_end + 16));
  CK(D.flags.ensure(B * 4 + 4));
  CK(D.keys.ensure(B * 8 + 8));
  CK(D.keys2.ensure(B * 8 + 8));
  CK(D.vals.ensure(B * 4 + 4));
  CK(D.vals2.ensure(B * 4 + 4));
  CK(D.slots.ensure(B * sizeof(Slot) + 16));
  CK(D.sum.ensure(sizeof(PlanSummary)));
  CK(D.end_i.ensure(B * 4 + 4));
  CK(D.end_j.ensure(B * 4 + 4));
  int32_t* d_scores = J.d_scores_out;
  if (!d_scores) {
    CK(D.scores.ensure(B * 4 + 4));
    d_scores = D.scores.as<int32_t>();
  }
  if (J.tb) {
    CK(D.beg_i.ensure(B * 4 + 4));
    CK(D.beg_j.ensure(B * 4 + 4));
    CK(D.n_ops.ensure(B * 4 + 4));
    CK(D.cig_off.ensure(B * 8 + 16));
    CK(D.ops.ensure((J.q_end + J.s_end + B + 1) * 4));
    CK(D.tb.ensure(B * sizeof(TbInfo) + 16));
  }

  // ---- a1: pack + validate ----
  CK(D.tickets.ensure(kNumTickets * 4));
  CK(launch_prep(D.flags.as<uint32_t>(), B + 1, D.sum.as<PlanSummary>(), J.rebase_qoff,
                 J.rebase_soff, J.rebase_q0, J.rebase_s0, J.gen_q, J.gen_s,
                 D.tickets.as<int32_t>(), st, D.num_sms));
  static const int dbg_asc = getenv("ANYSEQ_ASCENDING") ? 1 : 0;    // debug/tuning
  static const int dbg_static = getenv("ANYSEQ_STATIC_SLOTS") ? 1 : 0;
  int ticket_next = 0;
  auto take_ticket = [&]() -> int32_t* {
    return (!dbg_static && ticket_next < kNumTickets) ? D.tickets.as<int32_t>() + ticket_next++
                                                      : nullptr;
  };
  L(1);
  // byte codes are indexed by absolute CSR position; pack the whole [0, end) range the
  // caller's offsets cover (bytes before off[0] are never read by a pair)
  if (J.packed2)
    CK(launch_unpack2((const uint8_t*)J.d_q, J.q_end, D.q_code.as<uint8_t>(),
                      (const uint8_t*)J.d_s, J.s_end, D.s_code.as<uint8_t>(), st, D.num_sms));
  else
    CK(launch_pack(J.d_q, J.q_end, D.q_code.as<uint8_t>(), J.d_qoff, J.d_s, J.s_end,
                   D.s_code.as<uint8_t>(), J.d_soff, B, D.flags.as<uint32_t>(),
                   D.sum.as<PlanSummary>(), st, D.num_sms));
  L(1);
  ctx->mark(st, "packed");

  // ---- a2: classify ----
  ClassifyArgs ca;
  memset(&ca, 0, sizeof(ca));
  ca.P = P;
  ca.cfg.tb = J.tb;
  ca.cfg.allow16 = (int32_t)ctx->allow16;
  ca.cfg.force_variant = (int32_t)ctx->force_variant;
  ca.cfg.bound_go = P.go;
  ca.cfg.bound_ge = P.ge;
  ca.cfg.bound_match = P.smax;
  ca.cfg.ascending = dbg_asc;
  ca.q_off = J.d_qoff;
  ca.s_off = J.d_soff;
  ca.num_pairs = B;
  ca.flags = D.flags.as<uint32_t>();
  ca.sum = D.sum.as<PlanSummary>();
  ca.host_sum = D.h_sum;
  ca.slots = D.slots.as<Slot>();
  ca.keys = D.keys.as<unsigned long long>();
  ca.vals = D.vals.as<int32_t>();
  ca.scores = d_scores;
  ca.end_i = D.end_i.as<int32_t>();
  ca.end_j = D.end_j.as<int32_t>();
  if (J.tb) {
    ca.ops = D.ops.as<uint32_t>();
    ca.n_ops = D.n_ops.as<int32_t>();
    ca.beg_i = D.beg_i.as<int32_t>();
    ca.beg_j = D.beg_j.as<int32_t>();
  }
  ca.skip_cells = J.skip_cells;
  ca.skip_min = J.skip_min;
  CK(launch_classify(ca, st, D.num_sms));
  L(1);
  ctx->mark(st, "classified");
  // The plan summary normally comes back from classify (a stream synchronisation: the host
  // waits for the previous chunk's fill).  A host-API chunk of ACGT-only pairs of one common
  // length (2-bit upload, offsets generated on the device) has a plan the host can work out
  // with the same plan_pair() -- then nothing waits and the host enqueues the next chunk
  // while this one computes.
  PlanSummary S;
  bool host_plan = false;
  const bool skipped_all = J.skip_cells > 0 && J.gen_q >= J.skip_min && J.gen_s >= J.skip_min &&
                           J.gen_q * J.gen_s >= J.skip_cells;
  if (J.packed2 && J.gen_q > 0 && J.gen_s > 0 && B > 0 && !skipped_all) {
    const PairPlan pp = plan_pair(ca.cfg, J.gen_q, J.gen_s, false);
    if (!pp.range_err && pp.v >= 0) {
      memset(&S, 0, sizeof(S));
      S.err_pos = ~0ull;
      for (int v = 0; v < NV; ++v) {
        S.kmin[v] = ~0ull;
        S.kmax[v] = 0ull;
      }
      S.count[pp.v] = (int32_t)B;
      S.maxn[pp.v] = (int32_t)J.gen_q;
      S.maxm[pp.v] = (int32_t)J.gen_s;
      S.kmin[pp.v] = S.kmax[pp.v] = pp.key;
      host_plan = true;
    }
  }
  if (!host_plan) {
    CK(cudaStreamSynchronize(st));
    S = *D.h_sum;
  }
  ctx->mark(st, "host-planned");
  if (S.err_pos != ~0ull) {
    const bool in_s = S.err_pos >= (1ull << 62);
    return fail(ctx, ANYSEQ_E_BADSEQ, "invalid symbol at %s byte offset %llu", in_s ? "s" : "q",
                (unsigned long long)(in_s ? S.err_pos - (1ull << 62) : S.err_pos));
  }
  if (S.range_err)
    return fail(ctx, ANYSEQ_E_UNSUPPORTED, "score range exceeds 32-bit arithmetic");

  // ---- a2: order pairs by (variant, m, n) and form slots ----
  int32_t voff[NV + 1], sbase[NV], nslot[NV];
  int64_t nontriv = 0, total_slots = 0;
  int used = 0, used_v = -1;
  for (int v = 0; v < NV; ++v) {
    voff[v] = (int32_t)nontriv;
    nontriv += S.count[v];
    sbase[v] = (int32_t)total_slots;
    const int pp = variant_desc(v).pairs;
    nslot[v] = pp == 2 ? (S.count[v] + 1) / 2 : S.count[v];
    total_slots += nslot[v];
    if (S.count[v]) { ++used; used_v = v; }
  }
  voff[NV] = (int32_t)nontriv;
  const int32_t* order = D.vals.as<int32_t>();
  const bool uniform = used == 1 && (uint64_t)S.count[used_v] == B && S.kmin[used_v] == S.kmax[used_v];
  if (nontriv > 0 && !uniform) {
    size_t tb = 0;
    CK(sort_pairs(nullptr, tb, nullptr, nullptr, nullptr, nullptr, (int64_t)B, st));
    CK(D.temp.ensure(tb + 256));
    tb = D.temp.cap;
    CK(sort_pairs(D.temp.p, tb, D.keys.as<unsigned long long>(), D.keys2.as<unsigned long long>(),
                  D.vals.as<int32_t>(), D.vals2.as<int32_t>(), (int64_t)B, st));
    L(4);
    order = D.vals2.as<int32_t>();
  }
  if (nontriv > 0 && !uniform) {  // uniform: classify's speculative slots are the slots
    CK(launch_slots(order, nontriv, voff, S.count, sbase, D.slots.as<Slot>(), st, D.num_sms));
    L(1);
  }

  // Traceback H store in low bytes: the walk rebuilds H from neighbour
  // differences, exact when |H(x) - H(y)| < 128 for adjacent cells and a diagonal test
  // |H(i-1,j-1) - (H(i,j) - sigma)| < 256 -- both hold when 2 d + max |sigma| < 256, d =
  // G_o + G_e + max(sigma, 0) being the Lipschitz bound of the recurrence
  int tb8 = 0;
  if (J.tb && ctx->tb8) {
    int smaxabs = 0;
    for (int a = 0; a < 25; ++a) {
      const int v = prm->has_subst ? prm->subst[a] : ((a % 6 == 0 && a < 24) ? prm->match : prm->mismatch);
      smaxabs = std::max(smaxabs, std::abs(v));
    }
    const int64_t dl = (int64_t)P.go + P.ge + std::max(P.smax, 0);
    tb8 = (2 * dl + smaxabs < 256 && dl < 128) ? 1 : 0;
  }

  // ---- a3/a4: fill (+ a5 walk) per variant ----
  // score mode with several variants: fork the variant launches onto their own streams
  int nvar = 0;
  for (int v = 0; v < NV; ++v) nvar += S.count[v] ? 1 : 0;
  // (traceback too: each concurrent variant gets its own full H store -- at most the three
  // traceback variants, 3 x tb_scratch_bytes of device memory)
  const bool fork = nvar > 1;
  std::pair<cudaEvent_t, cudaEvent_t> fev{nullptr, nullptr};
  if (fork) {
    if (ctx->timing && !J.tb) { fev = take_events(ctx); CK(cudaEventRecord(fev.first, st)); }
    CK(cudaEventRecord(D.ev_fork, st));
  }
  for (int v = 0; v < NV; ++v) {
    if (!S.count[v]) continue;
    const VariantDesc d = variant_desc(v);
    cudaStream_t vst = fork ? D.vstream[v] : st;
    DevBuf& strip = fork ? D.strip_v[v] : D.strip;
    if (fork) CK(cudaStreamWaitEvent(vst, D.ev_fork, 0));
    FillArgs fa;
    memset(&fa, 0, sizeof(fa));
    fa.P = P;
    fa.qcode = D.q_code.as<uint8_t>();
    fa.scode = D.s_code.as<uint8_t>();
    fa.q_off = J.d_qoff;
    fa.s_off = J.d_soff;
    fa.slots = D.slots.as<Slot>();
    fa.nslots_dev = nullptr;
    fa.pos = J.want_ends || J.tb;
    fa.scores = d_scores;
    fa.end_i = D.end_i.as<int32_t>();
    fa.end_j = D.end_j.as<int32_t>();
    fa.one = 1;
    fa.nge_s16 = (uint32_t)(-P.ge & 0xffff) * 0x10001u;
    fa.koc_s16 = (uint32_t)(-(int)((P.go + P.ge) * 65537));
    const int HS = d.L * d.R;
    const int G = 32 / d.L;
    // strip row buffer only when some pair needs more than one strip
    int grid_est = D.num_sms * 16;  // upper bound of resident blocks (128 threads each)
    if (S.maxn[v] > HS) {
      fa.strip_stride = S.maxm[v] + 1;
      const int64_t groups = (int64_t)grid_est * 4 * G;
      CK(strip.ensure((size_t)groups * fa.strip_stride * sizeof(uint4)));
      fa.strip_scratch = strip.as<uint4>();
    } else {
      fa.strip_stride = 0;
      CK(strip.ensure(256));
      fa.strip_scratch = strip.as<uint4>();
    }
    if (!d.tb) {
      fa.slot_lo = sbase[v];
      fa.slot_hi = sbase[v] + nslot[v];
      int grid = 0;
      std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
      if (ctx->timing && !fork) { ev = take_events(ctx); CK(cudaEventRecord(ev.first, st)); }
      ctx->mark(vst, "fill-begin");
      fa.ticket = take_ticket();
      CK(launch_fill(v, prm->kind, prm->gap, fa, vst, D.num_sms, &grid));
      ctx->mark(vst, "fill-end");
      if (ctx->timing) {
        std::lock_guard<std::mutex> lk(ctx->ev_mu);
        if (!fork) {
          CK(cudaEventRecord(ev.second, st));
          ctx->fill_ev.push_back(ev);
        }
        ctx->fill_launches++;
      }
      if (grid > grid_est) return fail(ctx, ANYSEQ_E_CUDA, "occupancy above scratch estimate");
      L(1);
    } else {
      const int64_t ns = (S.maxn[v] + HS - 1) / HS;
      const int64_t dk = S.maxm[v] + d.L - 1 + d.R - 1;  // diagonals (step - row) per strip
      const int64_t block_words = ns * dk * d.R * d.L;    // one H element per (diag, row, lane)
      DevBuf& dirs = fork ? D.dirs_v[v] : D.dirs;
      // element size: the full H word (4 B), or -- when neighbouring H values provably
      // differ by less than 128 -- its low byte per alignment (2 B for s16x2, 1 B for s32)
      const int64_t esz = tb8 ? (d.pairs == 2 ? 2 : 1) : 4;
      const int64_t cap_words = std::max<int64_t>(ctx->tb_scratch_bytes / esz, block_words);
      int64_t chunk = std::max<int64_t>(1, cap_words / block_words);
      chunk = std::min<int64_t>(chunk, nslot[v]);
      // the G = 32 / L slots of a warp share one interleaved block (fill_kernel.cuh): the
      // last warp of a launch owns a whole block even when it holds fewer slots
      const int64_t gw = 32 / d.L;
      CK(dirs.ensure((size_t)(((chunk + gw - 1) / gw) * gw * block_words) * esz + 16));
      fa.dirs = dirs.as<uint32_t>();
      fa.dir_block_words = block_words;
      fa.tb8 = tb8;
      fa.tb = D.tb.as<TbInfo>();
      // local optimum rows resolved by the walk: the rows of a fill lane span at most
      // d (R - 1) below the lane's maximum, which the low byte must tell apart
      {
        const int64_t dl = (int64_t)P.go + P.ge + std::max(P.smax, 0);
        fa.defer_row = (prm->kind == ANYSEQ_LOCAL && (!tb8 || dl * (d.R - 1) < 256)) ? 1 : 0;
      }
      for (int64_t lo = 0; lo < nslot[v]; lo += chunk) {
        const int64_t hi = std::min<int64_t>(nslot[v], lo + chunk);
        fa.slot_lo = (int32_t)(sbase[v] + lo);
        fa.slot_hi = (int32_t)(sbase[v] + hi);
        int grid = 0;
        std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
        if (ctx->timing) { ev = take_events(ctx); CK(cudaEventRecord(ev.first, vst)); }
        fa.ticket = take_ticket();
        CK(launch_fill(v, prm->kind, prm->gap, fa, vst, D.num_sms, &grid));
        if (ctx->timing) {
          CK(cudaEventRecord(ev.second, vst));
          std::lock_guard<std::mutex> lk(ctx->ev_mu);
          ctx->fill_ev.push_back(ev);
          ctx->fill_launches++;
        }
        if (grid > grid_est) return fail(ctx, ANYSEQ_E_CUDA, "occupancy above scratch estimate");
        WalkArgs wa;
        wa.kind = prm->kind;
        wa.gap = prm->gap;
        wa.P = P;
        wa.qcode = D.q_code.as<uint8_t>();
        wa.scode = D.s_code.as<uint8_t>();
        wa.slots = D.slots.as<Slot>();
        wa.slot_lo = fa.slot_lo;
        wa.slot_hi = fa.slot_hi;
        wa.pairs_per_slot = d.pairs;
        wa.tb = D.tb.as<TbInfo>();
        wa.dirs = dirs.as<uint32_t>();
        wa.tb8 = tb8;
        wa.q_off = J.d_qoff;
        wa.s_off = J.d_soff;
        wa.ops = D.ops.as<uint32_t>();
        wa.n_ops = D.n_ops.as<int32_t>();
        wa.beg_i = D.beg_i.as<int32_t>();
        wa.beg_j = D.beg_j.as<int32_t>();
        wa.end_i = D.end_i.as<int32_t>();
        std::pair<cudaEvent_t, cudaEvent_t> ew{nullptr, nullptr};
        if (ctx->timing) { ew = take_events(ctx); CK(cudaEventRecord(ew.first, vst)); }
        CK(launch_walk(wa, vst, D.num_sms));
        if (ctx->timing) {
          CK(cudaEventRecord(ew.second, vst));
          std::lock_guard<std::mutex> lk(ctx->ev_mu);
          ctx->walk_ev.push_back(ew);
        }
        L(2);
      }
    }
    if (fork) {  // join this variant's stream back into the compute stream
      CK(cudaEventRecord(D.ev_join[v], vst));
      CK(cudaStreamWaitEvent(st, D.ev_join[v], 0));
    }
  }

  if (fork && ctx->timing && !J.tb) {  // one fill interval: fork to join (traceback: per launch)
    CK(cudaEventRecord(fev.second, st));
    std::lock_guard<std::mutex> lk(ctx->ev_mu);
    ctx->fill_ev.push_back(fev);
  }

  // ---- output assembly ----
  FinalizeArgs fz;
  memset(&fz, 0, sizeof(fz));
  fz.num_pairs = B;
  fz.scores = d_scores;
  fz.end_i = D.end_i.as<int32_t>();
  fz.end_j = D.end_j.as<int32_t>();
  fz.q_off = J.d_qoff;
  fz.s_off = J.d_soff;
  if (J.tb) {
    size_t tbytes = 0;
    CK(exclusive_scan_i32_to_u64(nullptr, tbytes, nullptr, nullptr, (int64_t)B + 1, st));
    CK(D.temp.ensure(tbytes + 256));
    tbytes = D.temp.cap;
    // n_ops[B] is a zero sentinel so cig_off[B] is the total
    CK(cudaMemsetAsync(D.n_ops.as<int32_t>() + B, 0, 4, st));
    CK(exclusive_scan_i32_to_u64(D.temp.p, tbytes, D.n_ops.as<int32_t>(), D.cig_off.as<uint64_t>(),
                                 (int64_t)B + 1, st));
    L(1);
    ctx->mark(st, "walked+scanned");
    CK(cudaMemcpyAsync(D.h_small, D.cig_off.as<uint64_t>() + B, 8, cudaMemcpyDeviceToHost, st));
    if (J.before_sync) {
      const anyseq_status u = J.before_sync();
      if (u != ANYSEQ_OK) return u;
    }
    CK(cudaStreamSynchronize(st));
    J.cigar_total = D.h_small[0];
    ctx->mark(st, "host-has-total");
    fz.beg_i = D.beg_i.as<int32_t>();
    fz.beg_j = D.beg_j.as<int32_t>();
    fz.n_ops = D.n_ops.as<int32_t>();
    fz.cig_off = D.cig_off.as<uint64_t>();
    fz.ops = D.ops.as<uint32_t>();
    fz.cigar = d_cigar_out_or_null;
    fz.cigar_cap = cigar_cap;
    fz.cig_base = J.cig_base;
  }
  if (J.tb || J.want_ends) {
    anyseq_alignment* out = J.d_aln_out;
    if (!out) {
      CK(D.aln.ensure(B * sizeof(anyseq_alignment) + 64));
      out = D.aln.as<anyseq_alignment>();
    }
    fz.out_aln = out;
    CK(launch_finalize(fz, st, D.num_sms));
    L(1);
    ctx->mark(st, "finalized");
  }
  return ANYSEQ_OK;
}

anyseq_status check_batch_host(anyseq_ctx* ctx, const anyseq_batch* b) {
  if (!b) return fail(ctx, ANYSEQ_E_INVALID, "batch is NULL");
  if (b->num_pairs == 0) return ANYSEQ_OK;
  if (!b->q_off || !b->s_off) return fail(ctx, ANYSEQ_E_INVALID, "offsets are NULL");
  if (b->num_pairs >= (1ull << 31)) return fail(ctx, ANYSEQ_E_INVALID, "too many pairs");
  if (b->q_off[b->num_pairs] < b->q_off[0] || b->s_off[b->num_pairs] < b->s_off[0])
    return fail(ctx, ANYSEQ_E_INVALID, "offsets decrease");
  if ((b->q_off[b->num_pairs] > b->q_off[0] && !b->q) ||
      (b->s_off[b->num_pairs] > b->s_off[0] && !b->s))
    return fail(ctx, ANYSEQ_E_INVALID, "sequence pointer is NULL");
  return ANYSEQ_OK;
}

// Per-pair offset checks of pairs [k0, k1), run by the host API on each chunk before its
// upload (off the critical path: the host thread checks chunk c+1 while chunk c computes).
// *uq / *us: the common q / s length when every pair of the range has the same lengths
// (then the chunk's offsets are generated on the device instead of uploaded), else -1.
anyseq_status check_pairs_host(anyseq_ctx* ctx, const anyseq_batch* b, uint64_t k0, uint64_t k1,
                               int tb, int64_t* uq, int64_t* us) {
  // traceback: a CIGAR word holds a run of at most 2^28 - 1 (len << 4 | op); an empty
  // partner makes one gap run of the whole other sequence, so longer sequences are refused
  const uint64_t lim = tb ? (1ull << 28) : (1ull << 31);
  const uint64_t lq = b->q_off[k0 + 1] - b->q_off[k0], ls = b->s_off[k0 + 1] - b->s_off[k0];
  bool uni = true;
  for (uint64_t k = k0; k < k1; ++k) {
    uni = uni && b->q_off[k + 1] - b->q_off[k] == lq && b->s_off[k + 1] - b->s_off[k] == ls;
    if (b->q_off[k + 1] < b->q_off[k] || b->s_off[k + 1] < b->s_off[k])
      return fail(ctx, ANYSEQ_E_INVALID, "pair %llu: offsets decrease", (unsigned long long)k);
    if (b->q_off[k + 1] - b->q_off[k] >= lim || b->s_off[k + 1] - b->s_off[k] >= lim)
      return fail(ctx, tb ? ANYSEQ_E_UNSUPPORTED : ANYSEQ_E_INVALID,
                  "pair %llu: sequence longer than %s", (unsigned long long)k,
                  tb ? "2^28-1 (traceback)" : "2^31-1");
  }
  *uq = uni ? (int64_t)lq : -1;
  *us = uni ? (int64_t)ls : -1;
  return ANYSEQ_OK;
}

// Map an error byte position back to (pair, offset) for the message.
void describe_badseq(anyseq_ctx* ctx, const anyseq_batch* b, uint64_t k0) {
  // ctx->err holds "invalid symbol at q byte offset X" relative to the shard
  unsigned long long pos = 0;
  char which = 0;
  if (sscanf(ctx->err.c_str(), "invalid symbol at %c byte offset %llu", &which, &pos) != 2) return;
  const uint64_t* off = which == 'q' ? b->q_off : b->s_off;
  const char* seq = which == 'q' ? b->q : b->s;
  const uint64_t abs = pos + off[k0];
  const uint64_t* it = std::upper_bound(off, off + b->num_pairs + 1, abs);
  const uint64_t k = (uint64_t)(it - off) - 1;
  char buf[256];
  snprintf(buf, sizeof(buf), "pair %llu: byte 0x%02x at %c offset %llu",
           (unsigned long long)k, (unsigned)(unsigned char)seq[abs], which,
           (unsigned long long)(abs - off[k]));
  ctx->err = buf;
}

// Host-memory batch on one device, pairs [k0, k1).  The shard is cut into chunks of about
// ctx->chunk_bytes of sequence; the upload of chunk c+1 (copy stream, double-buffered)
// overlaps the planning/relaxation of chunk c (compute stream).
// Traceback cigar words go straight into the caller's buffer when cig_direct is set (one
// device: offsets are final), else into *cig (multi-device: rebased after all shards finish).
// *cig_words receives the shard's total cigar words either way.
PackPool* pool_of(anyseq_ctx* ctx) { return ctx->packer(); }

anyseq_status run_host_shard(anyseq_ctx* ctx, Device& D, const anyseq_params* prm,
                             const anyseq_batch* b, uint64_t k0, uint64_t k1, int tb,
                             int32_t* scores, anyseq_alignment* aln, uint32_t* cig_direct,
                             uint64_t cig_cap, std::vector<uint32_t>* cig, uint64_t* cig_words) {
  CK(cudaSetDevice(D.id));
  cudaStream_t st = D.stream, cs = D.copy_stream;
  const auto t_call = std::chrono::steady_clock::now();  // timing >= 2: host timeline
  auto ms_since = [t_call]() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count();
  };
  // chunk boundaries by cumulative sequence bytes (offsets are monotone)
  std::vector<uint64_t> cb{k0};
  {
    // ramp-up: the first upload is not overlapped with anything, so the first chunks are
    // small (1/8, 1/4, 1/2 of chunk_bytes) and the compute stream starts early; ramp-down:
    // the last chunk's compute is not overlapped either, so the tail halves likewise
    const uint64_t full = (uint64_t)std::max<int64_t>(ctx->chunk_bytes, 1 << 12);
    const uint64_t end_bytes = b->q_off[k1] + b->s_off[k1];
    uint64_t k = k0;
    int c = 0;
    while (k < k1) {
      const uint64_t base = b->q_off[k] + b->s_off[k];
      const uint64_t left = end_bytes - base;
      uint64_t cap = c < 3 ? full >> (3 - c) : full;
      if (c >= 3 && left < 2 * full) cap = std::max<uint64_t>(full >> 3, left / 2);
      cap = std::max<uint64_t>(1 << 12, cap);
      ++c;
      uint64_t lo = k + 1, hi = k1;  // last index e in (k, k1] with bytes(k, e) <= cap
      while (lo < hi) {
        const uint64_t mid = lo + (hi - lo + 1) / 2;
        if (b->q_off[mid] + b->s_off[mid] - base <= cap) lo = mid; else hi = mid - 1;
      }
      k = lo;
      cb.push_back(k);
    }
  }
  const int NC = (int)cb.size() - 1;
  // Score-mode results go to the caller's buffers directly when those are pinned; a D2H copy
  // into pageable memory would block the host until the chunk finished and stall the upload
  // pipeline, so pageable outputs are staged in pinned memory and copied out one chunk late.
  const bool stage_s = !tb && !host_pinned(scores);
  const bool stage_a = aln && !host_pinned(aln);
  const uint64_t nloc = k1 - k0;
  const size_t st_a_off = stage_s ? ((nloc * 4 + 63) & ~63ull) : 0;
  if (stage_s || stage_a)
    CK(D.h_stage.ensure(st_a_off + (stage_a ? nloc * sizeof(anyseq_alignment) : 0)));
  int32_t* h_sc = stage_s ? (int32_t*)D.h_stage.p - k0 : scores;
  anyseq_alignment* h_al =
      stage_a ? (anyseq_alignment*)((char*)D.h_stage.p + st_a_off) - k0 : aln;
  auto copy_out = [&](int c) {  // chunk c's results are complete on the host side
    NvtxRange nvtx("copy out chunk");
    const uint64_t a0 = cb[c], B = cb[c + 1] - a0;
    if (stage_s) memcpy(scores + a0, h_sc + a0, B * 4);
    if (stage_a) memcpy(aln + a0, h_al + a0, B * sizeof(anyseq_alignment));
  };
  int64_t gen_q[2] = {-1, -1}, gen_s[2] = {-1, -1};  // per buffer set (see check_pairs_host)
  int packed[2] = {0, 0};       // per buffer set: the chunk went up as 2-bit codes
  uint64_t s2off[2] = {0, 0};   // ... and its s codes start at this byte of the blob
  // a1, 2-bit path: a pack-ahead thread packs chunk after chunk on the host pool (validation
  // fused) into a ring of three pinned staging slots while this thread drives the device;
  // chunk c waits only for its own packing, and the packer reuses a slot once the upload of
  // the chunk three back has completed.  A chunk with any byte outside ACGTacgt (N
  // included) goes up as ASCII instead; the device pack then validates it and flags N.
  PackPool* pool = ctx->pack2 ? pool_of(ctx) : nullptr;
  struct Ahead {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<int> state;   // per chunk: 0 pending, 1 packed, 2 take the ASCII path
    std::vector<char> issued; // per chunk: its upload was issued (slot event recorded)
    bool stop = false;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    std::thread th;
    ~Ahead() {
      {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
      }
      cv.notify_all();
      if (th.joinable()) th.join();
      for (auto e : ev) if (e) cudaEventDestroy(e);
    }
  } ahead;
  auto chunk_sizes = [&](int c, uint64_t* qb, uint64_t* sb) {
    const uint64_t qlen = b->q_off[cb[c + 1]] - b->q_off[cb[c]];
    const uint64_t slen = b->s_off[cb[c + 1]] - b->s_off[cb[c]];
    *qb = ((qlen + 3) / 4 + 15) & ~15ull;
    *sb = ((slen + 3) / 4 + 15) & ~15ull;
  };
  if (pool && NC > 0) {
    uint64_t need = 0;
    for (int c = 0; c < NC; ++c) {
      uint64_t qb, sb;
      chunk_sizes(c, &qb, &sb);
      need = std::max(need, qb + sb + 16);
    }
    for (int k = 0; k < 3; ++k) {
      CK(D.h_pack[k].ensure(need));
      CK(cudaEventCreateWithFlags(&ahead.ev[k], cudaEventDisableTiming));
    }
    ahead.state.assign(NC, 0);
    ahead.issued.assign(NC, 0);
    const int dev = D.id;
    // Share of the chunks (by bytes) packed on the host; the rest go up as ASCII DMA
    // (option pack2_percent; all by default: splitting between host packing and ASCII DMA
    // measured slower on B200 hosts -- both read host memory)
    const double share = ctx->pack2_percent > 0 ? std::min<int64_t>(ctx->pack2_percent, 100) / 100.0
                                                : 1.0;
    ahead.th = std::thread([&, dev, ms_since, share] {
      cudaSetDevice(dev);
      double packed_bytes = 0, all_bytes = 0;
      for (int c = 0; c < NC; ++c) {
        const double cbytes = (double)(b->q_off[cb[c + 1]] - b->q_off[cb[c]] +
                                       b->s_off[cb[c + 1]] - b->s_off[cb[c]]);
        all_bytes += cbytes;
        if (packed_bytes + cbytes > share * all_bytes + 1.0) {  // this one goes as ASCII
          std::lock_guard<std::mutex> lk(ahead.mu);
          ahead.state[c] = 2;
          ahead.cv.notify_all();
          continue;
        }
        packed_bytes += cbytes;
        const int slot = c % 3;
        if (c >= 3) {  // the slot's previous upload (chunk c - 3) must have completed
          std::unique_lock<std::mutex> lk(ahead.mu);
          ahead.cv.wait(lk, [&] { return ahead.stop || ahead.issued[c - 3]; });
          if (ahead.stop) return;
          lk.unlock();
          cudaEventSynchronize(ahead.ev[slot]);
        }
        uint64_t qb, sb;
        chunk_sizes(c, &qb, &sb);
        const uint64_t q0 = b->q_off[cb[c]], s0 = b->s_off[cb[c]];
        uint8_t* hp = (uint8_t*)D.h_pack[slot].p;
        bool ok2 = false;
        const double tp0 = ms_since();
        NvtxRange nvtx("pack2 chunk");
        try {
          ok2 = pool->pack2(b->q + q0, b->q_off[cb[c + 1]] - q0, hp) &&
                pool->pack2(b->s + s0, b->s_off[cb[c + 1]] - s0, hp + qb);
        } catch (...) {
          ok2 = false;  // (allocation failure in the pool) -> the ASCII path
        }
        if (ctx->timing >= 2)
          fprintf(stderr, "[host] pack %d: %.3f -> %.3f ms\n", c, tp0, ms_since());
        std::lock_guard<std::mutex> lk(ahead.mu);
        ahead.state[c] = ok2 ? 1 : 2;
        ahead.cv.notify_all();
        if (ahead.stop) return;
      }
    });
  }
  auto upload = [&](int c) -> anyseq_status {
    const int set = c & 1;
    const uint64_t a0 = cb[c], a1 = cb[c + 1], B = a1 - a0;
    const anyseq_status chk = check_pairs_host(ctx, b, a0, a1, tb, &gen_q[set], &gen_s[set]);
    if (chk != ANYSEQ_OK) return chk;
    const uint64_t q0 = b->q_off[a0], s0 = b->s_off[a0];
    const uint64_t qlen = b->q_off[a1] - q0, slen = b->s_off[a1] - s0;
    CK(D.q_ascii2[set].ensure(qlen + 64));
    CK(D.s_ascii2[set].ensure(slen + 16));
    CK(D.q_off2[set].ensure((B + 1) * 8));
    CK(D.s_off2[set].ensure((B + 1) * 8));
    // the previous user of this set (chunk c-2) is finished: its offsets are read up to the
    // last kernel of the chunk, not just by the pack kernels
    CK(cudaStreamWaitEvent(cs, D.ev_free[set], 0));
    packed[set] = 0;
    if (pool) {
      int stt;
      {
        std::unique_lock<std::mutex> lk(ahead.mu);
        ahead.cv.wait(lk, [&] { return ahead.state[c] != 0; });
        stt = ahead.state[c];
      }
      if (ctx->timing >= 2) fprintf(stderr, "[host] chunk %d packed-wait done %.3f ms\n", c, ms_since());
      const int slot = c % 3;
      if (stt == 1) {
        uint64_t qb, sb;
        chunk_sizes(c, &qb, &sb);
        packed[set] = 1;
        s2off[set] = qb;
        CK(cudaMemcpyAsync(D.q_ascii2[set].p, D.h_pack[slot].p, qb + sb, cudaMemcpyHostToDevice, cs));
        ctx->h2d_bytes += qb + sb;
      }
      CK(cudaEventRecord(ahead.ev[slot], cs));
      {
        std::lock_guard<std::mutex> lk(ahead.mu);
        ahead.issued[c] = 1;
      }
      ahead.cv.notify_all();
    }
    if (!packed[set]) {
      if (qlen) CK(cudaMemcpyAsync(D.q_ascii2[set].p, b->q + q0, qlen, cudaMemcpyHostToDevice, cs));
      if (slen) CK(cudaMemcpyAsync(D.s_ascii2[set].p, b->s + s0, slen, cudaMemcpyHostToDevice, cs));
      ctx->h2d_bytes += qlen + slen;
    }
    if (gen_q[set] < 0) {  // uniform chunks: offsets generated on the device (prep kernel)
      CK(cudaMemcpyAsync(D.q_off2[set].p, b->q_off + a0, (B + 1) * 8, cudaMemcpyHostToDevice, cs));
      CK(cudaMemcpyAsync(D.s_off2[set].p, b->s_off + a0, (B + 1) * 8, cudaMemcpyHostToDevice, cs));
      ctx->h2d_bytes += 2 * (B + 1) * 8;
    }
    CK(cudaEventRecord(D.ev_up[set], cs));
    return ANYSEQ_OK;
  };
  auto mark = [&](cudaStream_t x, const char* what, int c) {
    if (ctx->timing >= 2) ctx->mark(x, std::string(what) + " " + std::to_string(c));
  };
  mark(cs, "up-begin", 0);
  anyseq_status s = upload(0);
  if (s != ANYSEQ_OK) return s;
  mark(cs, "up-end", 0);
  uint64_t cig_base = 0;
  // ASCII path: the upload of chunk c+1 is issued before chunk c's compute (the copy engine
  // is the bottleneck); 2-bit path: after it, so that chunk c's kernels never wait for the
  // packing of chunk c+1 (the packer thread runs ahead on its own)
  auto upload_next = [&](int c) -> anyseq_status {
    if (c + 1 >= NC) return ANYSEQ_OK;
    mark(cs, "up-begin", c + 1);
    const anyseq_status u = upload(c + 1);
    if (u != ANYSEQ_OK) {
      cudaStreamSynchronize(cs);  // chunk c may be in flight: leave the device idle
      cudaStreamSynchronize(st);
      return u;
    }
    mark(cs, "up-end", c + 1);
    return ANYSEQ_OK;
  };
  for (int c = 0; c < NC; ++c) {
    const int set = c & 1;
    if (!pool && (s = upload_next(c)) != ANYSEQ_OK) return s;
    mark(st, "compute-begin", c);
    const uint64_t a0 = cb[c], a1 = cb[c + 1], B = a1 - a0;
    const uint64_t q0 = b->q_off[a0], s0 = b->s_off[a0];
    const uint64_t qlen = b->q_off[a1] - q0, slen = b->s_off[a1] - s0;
    CK(cudaStreamWaitEvent(st, D.ev_up[set], 0));
    mark(st, "compute-wait", c);

    DeviceJob J;
    J.d_q = D.q_ascii2[set].as<char>();
    J.d_qoff = D.q_off2[set].as<uint64_t>();
    J.d_s = packed[set] ? D.q_ascii2[set].as<char>() + s2off[set] : D.s_ascii2[set].as<char>();
    J.packed2 = packed[set];
    J.d_soff = D.s_off2[set].as<uint64_t>();
    J.rebase_qoff = D.q_off2[set].as<uint64_t>();
    J.rebase_soff = D.s_off2[set].as<uint64_t>();
    J.rebase_q0 = q0;
    J.rebase_s0 = s0;
    J.gen_q = gen_q[set];
    J.gen_s = gen_s[set];
    J.cig_base = cig_base;
    J.B = B;
    J.q_end = qlen;
    J.s_end = slen;
    J.tb = tb;
    J.skip_cells = tb ? 0 : ctx->skip_cells;
    J.skip_min = ctx->batch_long_min;
    J.want_ends = aln != nullptr;
    J.d_scores_out = nullptr;
    J.d_aln_out = nullptr;
    uint64_t cap_words = 0;
    if (tb) {
      cap_words = qlen + slen + 1;  // worst case sum(n+m); exact total known after the walk
      CK(D.cigar.ensure(cap_words * 4));
    }
    const double tr0 = ms_since();
    bool up_done = false;
    if (tb && pool)  // traceback: upload chunk c+1 while chunk c's fill and walk run
      J.before_sync = [&]() -> anyseq_status {
        up_done = true;
        return upload_next(c);
      };
    s = run_device(ctx, D, prm, J, tb ? D.cigar.as<uint32_t>() : nullptr, cap_words);
    if (ctx->timing >= 2) fprintf(stderr, "[host] chunk %d run_device %.3f -> %.3f ms\n", c, tr0, ms_since());
    if (s == ANYSEQ_OK && pool && !up_done) {
      const anyseq_status u = upload_next(c);
      if (u != ANYSEQ_OK) return u;
    }
    if (s == ANYSEQ_OK && c > 0) {
      // chunk c-1's results have landed once its last enqueued work has (run_device no
      // longer synchronises when the host planned chunk c itself)
      if (stage_s || stage_a) CK(cudaEventSynchronize(D.ev_free[(c - 1) & 1]));
      copy_out(c - 1);
    }
    if (s != ANYSEQ_OK) {
      if (s == ANYSEQ_E_BADSEQ) describe_badseq(ctx, b, a0);
      cudaStreamSynchronize(cs);
      cudaStreamSynchronize(st);
      return s;
    }
    if (!tb) {
      CK(cudaMemcpyAsync(h_sc + a0, D.scores.p, B * 4, cudaMemcpyDeviceToHost, st));
      ctx->d2h_bytes += B * 4 + (aln ? B * sizeof(anyseq_alignment) : 0);
      mark(st, "scores-d2h-issued", c);
      if (aln) CK(cudaMemcpyAsync(h_al + a0, D.aln.p, B * sizeof(anyseq_alignment), cudaMemcpyDeviceToHost, st));
    } else {
      // cigar offsets already include cig_base (finalize adds J.cig_base on the device)
      CK(cudaMemcpyAsync(h_al + a0, D.aln.p, B * sizeof(anyseq_alignment), cudaMemcpyDeviceToHost, st));
      ctx->d2h_bytes += B * sizeof(anyseq_alignment) + J.cigar_total * 4;
      if (J.cigar_total && cig_direct) {
        if (cig_base + J.cigar_total <= cig_cap)
          CK(cudaMemcpyAsync(cig_direct + cig_base, D.cigar.p, J.cigar_total * 4,
                             cudaMemcpyDeviceToHost, st));
      } else if (J.cigar_total) {
        // the vector may reallocate: its previous contents must have landed
        CK(cudaStreamSynchronize(st));
        cig->resize(cig_base + J.cigar_total);
        CK(cudaMemcpyAsync(cig->data() + cig_base, D.cigar.p, J.cigar_total * 4,
                           cudaMemcpyDeviceToHost, st));
      }
      mark(st, "tb-d2h-issued", c);
      cig_base += J.cigar_total;
    }
    CK(cudaEventRecord(D.ev_free[set], st));  // every kernel reading this set is enqueued
  }
  CK(cudaStreamSynchronize(st));
  if (NC > 0) copy_out(NC - 1);
  if (cig_words) *cig_words = cig_base;
  if (ctx->timing >= 2) {
    CK(cudaStreamSynchronize(cs));
    ctx->dump_trace();
  }
  return ANYSEQ_OK;
}

// Split [0, B) into G contiguous shards of ~equal cell count.
std::vector<uint64_t> shard_bounds(const anyseq_batch* b, int G) {
  std::vector<uint64_t> bounds(G + 1, b->num_pairs);
  bounds[0] = 0;
  if (G == 1) return bounds;
  long double total = 0;
  for (uint64_t k = 0; k < b->num_pairs; ++k)
    total += (long double)(b->q_off[k + 1] - b->q_off[k] + 1) * (b->s_off[k + 1] - b->s_off[k] + 1);
  long double acc = 0;
  int g = 1;
  for (uint64_t k = 0; k < b->num_pairs && g < G; ++k) {
    acc += (long double)(b->q_off[k + 1] - b->q_off[k] + 1) * (b->s_off[k + 1] - b->s_off[k] + 1);
    while (g < G && acc >= total * g / G) bounds[g++] = k + 1;
  }
  for (; g < G; ++g) bounds[g] = b->num_pairs;
  return bounds;
}

anyseq_status run_host_batch_core(anyseq_ctx* ctx, const anyseq_params* prm, const anyseq_batch* b,
                                  int tb, int32_t* scores, anyseq_alignment* aln, uint32_t* cigar,
                                  uint64_t cap, uint64_t* used) {
  const int G = (int)ctx->devs.size();
  std::vector<uint64_t> bounds = shard_bounds(b, G);
  std::vector<anyseq_status> st(G, ANYSEQ_OK);
  std::vector<std::string> errs(G);
  std::vector<std::vector<uint32_t>> cigs(G);
  std::vector<uint64_t> words(G, 0);
  if (G == 1) {
    st[0] = run_host_shard(ctx, ctx->devs[0], prm, b, 0, b->num_pairs, tb, scores, aln,
                           tb ? cigar : nullptr, cap, &cigs[0], &words[0]);
  } else {
    std::vector<anyseq_ctx*> sub(G);
    std::vector<std::thread> th;
    std::mutex mu;
    struct Joiner {  // a failed thread creation must not leave joinable threads behind
      std::vector<std::thread>& v;
      ~Joiner() { for (auto& t : v) if (t.joinable()) t.join(); }
    } joiner{th};
    for (int g = 0; g < G; ++g) {
      th.emplace_back([&, g] {
        anyseq_ctx local;  // per-thread error string
        local.tb_scratch_bytes = ctx->tb_scratch_bytes;
        local.force_variant = ctx->force_variant;
        local.allow16 = ctx->allow16;
        local.chunk_bytes = ctx->chunk_bytes;
        local.pack2 = ctx->pack2;
        local.tb8 = ctx->tb8;
        local.pack2_percent = ctx->pack2_percent;
        local.skip_cells = ctx->skip_cells;
        local.batch_long_min = ctx->batch_long_min;
        local.shared_pool = ctx->pack2 ? ctx->packer() : nullptr;
        anyseq_status s = ANYSEQ_OK;
        if (bounds[g + 1] > bounds[g])  // an exception must not escape a std::thread either
          s = abi_guard(&local, [&]() {
            return run_host_shard(&local, ctx->devs[g], prm, b, bounds[g], bounds[g + 1], tb,
                                  scores, aln, nullptr, 0, &cigs[g], &words[g]);
          });
        std::lock_guard<std::mutex> lk(mu);
        st[g] = s;
        errs[g] = local.err;
        ctx->launches += local.launches.load();
        ctx->h2d_bytes += local.h2d_bytes.load();
        ctx->d2h_bytes += local.d2h_bytes.load();
      });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < G; ++g)
      if (st[g] != ANYSEQ_OK) {
        ctx->err = "device " + std::to_string(ctx->devs[g].id) + ": " + errs[g];
        return st[g];
      }
  }
  if (st[0] != ANYSEQ_OK) return st[0];
  if (tb) {
    uint64_t total = 0;
    for (int g = 0; g < G; ++g) total += words[g];
    if (used) *used = total;
    if (total > cap) return fail(ctx, ANYSEQ_E_CAPACITY, "cigar needs %llu words, capacity %llu",
                                 (unsigned long long)total, (unsigned long long)cap);
    if (G > 1) {
      uint64_t base = 0;
      for (int g = 0; g < G; ++g) {
        if (!cigs[g].empty()) memcpy(cigar + base, cigs[g].data(), cigs[g].size() * 4);
        if (base)
          for (uint64_t k = bounds[g]; k < bounds[g + 1]; ++k) aln[k].cigar_offset += base;
        base += cigs[g].size();
      }
    }
  }
  return ANYSEQ_OK;
}

// ---- linear-space long-pair traceback: Hirschberg's divide and conquer.
// A problem (i0,i1) x (j0,j1) with more than kLeafCells cells is cut at mid = (i0+i1)/2:
// a forward last-row pass over q[i0,mid) x s[j0,j1) and a reverse pass over q[mid,i1) x
// s[j0,j1) (both on the GPU, all problems of one recursion level in one launch, every
// pass cut into pipelined 3072-row bands, one CTA each) give
// F(j) = H(mid, j) and B(j) = the best score of q[mid,i1) x s[j0+j,j1); the optimal path
// crosses row mid at the smallest j maximising F(j) + B(m'-j).  Leaves (in path order, so
// their q and s ranges tile the alignment) run as ONE batched global traceback
// (run_host_batch, the a4/a5 kernels); their CIGARs are concatenated.
// Linear gaps only: an affine split must carry the gap state across the cut
// (Myers-Miller), which the leaf traceback does not take as a boundary condition.
anyseq_status run_traceback_long(anyseq_ctx* ctx, const anyseq_params* prm, const char* q,
                                 uint64_t n, const char* s, uint64_t m, anyseq_alignment* out,
                                 uint32_t* cigar, uint64_t cap, uint64_t* used);

// Score mode of a mixed batch without copying it: the batch kernels skip the long pairs
// (classify leaves pairs of >= batch_long_cells cells unplanned, ClassifyArgs::skip_cells)
// and run while the long pairs share one launch of the long kernel (run_long_multi, one
// device); their results are then written into the caller's outputs.  Long pairs the shared
// launch does not take run one by one (anyseq_align_long, else the batch path alone).
static anyseq_status run_host_batch_inplace(anyseq_ctx* ctx, const anyseq_params* prm,
                                            const anyseq_batch* b,
                                            const std::vector<uint64_t>& longs, int32_t* scores,
                                            anyseq_alignment* aln) {
  const uint64_t BL = longs.size();
  struct SkipGuard {  // the batch pass skips the long pairs; nothing after it does
    anyseq_ctx* c;
    ~SkipGuard() { c->skip_cells = 0; }
  } guard{ctx};
  ctx->skip_cells = ctx->batch_long_cells;
  auto run_short = [&]() -> int {
    const anyseq_status r = run_host_batch_core(ctx, prm, b, 0, scores, aln, nullptr, 0, nullptr);
    ctx->skip_cells = 0;
    return r;
  };
  std::vector<int> done(BL, 0);
  auto put = [&](uint64_t k, int32_t score, int64_t ei, int64_t ej) {
    scores[k] = score;
    if (aln) {
      anyseq_alignment a;
      memset(&a, 0, sizeof(a));
      a.score = score;
      a.q_end = a.q_begin = ei;
      a.s_end = a.s_begin = ej;
      aln[k] = a;
    }
  };
  if (ctx->long_multi && BL >= 2 && ctx->devs.size() == 1) {
    std::vector<LongPairIn> in(BL);
    for (uint64_t x = 0; x < BL; ++x) {
      const uint64_t k = longs[x];
      in[x] = LongPairIn{b->q + b->q_off[k], b->q_off[k + 1] - b->q_off[k], b->s + b->s_off[k],
                         b->s_off[k + 1] - b->s_off[k]};
    }
    const Device& D = ctx->devs[0];
    LongDevice ld;
    ld.id = D.id;
    ld.stream = D.stream;
    ld.num_sms = D.num_sms;
    ld.ws = ctx->lws[0].get();
    std::vector<LongResult> lr;
    std::vector<int> took;
    std::string err;
    uint64_t launches = 0;
    double kms = 0;
    int rs = ANYSEQ_OK;
    const int rc = run_long_multi(ld, dev_params(prm), in, ctx->long_opt, &lr, &took, &err,
                                  &launches, &kms, [&]() { return rs = run_short(); },
                                  &ctx->long_multi_rows);
    ctx->launches += launches;
    if (rs != ANYSEQ_OK) return (anyseq_status)rs;
    if (rc != 0) return fail(ctx, (anyseq_status)rc, "long pairs (one launch): %s", err.c_str());
    for (uint64_t x = 0; x < BL; ++x)
      if (took[x]) {
        done[x] = 1;
        put(longs[x], lr[x].score, lr[x].end_i, lr[x].end_j);
        ++ctx->long_multi_pairs;
      }
    ctx->long_multi_ms = kms;
  } else {
    const anyseq_status r = (anyseq_status)run_short();
    if (r != ANYSEQ_OK) return r;
  }
  for (uint64_t x = 0; x < BL; ++x) {
    if (done[x]) continue;
    const uint64_t k = longs[x];
    const char* qk = b->q + b->q_off[k];
    const char* sk = b->s + b->s_off[k];
    const uint64_t n = b->q_off[k + 1] - b->q_off[k], m = b->s_off[k + 1] - b->s_off[k];
    anyseq_alignment a;
    anyseq_status r = anyseq_align_long(ctx, prm, qk, n, sk, m, &a);
    if (r == ANYSEQ_E_UNSUPPORTED) {  // not for the long path: this pair on the batch path
      const uint64_t qo1[2] = {0, n}, so1[2] = {0, m};
      const anyseq_batch b1{qk, qo1, sk, so1, 1};
      r = run_host_batch_core(ctx, prm, &b1, 0, scores + k, aln ? aln + k : nullptr, nullptr, 0,
                              nullptr);
      if (r == ANYSEQ_OK) continue;
    }
    if (r != ANYSEQ_OK) {
      ctx->err = "pair " + std::to_string(k) + " (long-pair path): " + ctx->err;
      return r;
    }
    put(k, a.score, a.q_end, a.s_end);
  }
  return ANYSEQ_OK;
}

// Mixed batches: a pair whose matrix is large (n·m >= option
// batch_long_cells -- batch_long_cells_tb in traceback mode -- both sides >= batch_long_min) would tie one 8-lane group of the batch
// kernel up for seconds; it goes to the long-pair path instead (the tiled wavefront over all
// SMs, §5.4 / §5.4c), the rest of the batch to the batch path, and the results are merged in
// pair order (both paths follow the same optimum and traceback rules, so the results are the
// ones the batch path would give).  A batch of only a few pairs (option batch_long_small)
// sends every pair with both sides >= 256 there too: the batch kernel gives a pair one
// 8-lane group, the long kernel spreads it over many warps (C1, one 1000 x 1000 pair:
// 1.3 ms instead of 5 ms with traceback).  A pair the long path cannot take (e.g. affine
// traceback of a subject with N) falls back to the batch path on its own.  Score mode
// (not a small batch) takes run_host_batch_inplace above.
anyseq_status run_host_batch(anyseq_ctx* ctx, const anyseq_params* prm, const anyseq_batch* b,
                             int tb, int32_t* scores, anyseq_alignment* aln, uint32_t* cigar,
                             uint64_t cap, uint64_t* used) {
  std::vector<uint64_t> longs;
  const bool small = b->num_pairs <= (uint64_t)ctx->batch_long_small;
  // small-batch routing only where the long path is the checkpointed 16-bit one (its
  // CIGARs follow the batch path's tie rules; a subject with N would take the s32 kernel
  // and, for traceback, the Hirschberg fallback)
  auto acgt_only = [](const char* p, uint64_t len) {
    for (uint64_t x = 0; x < len; ++x) {
      const char c = (char)(p[x] | 0x20);
      if (c != 'a' && c != 'c' && c != 'g' && c != 't') return false;
    }
    return true;
  };
  const int64_t thr = tb ? ctx->batch_long_cells_tb : ctx->batch_long_cells;
  if (thr > 0 || small)
    for (uint64_t k = 0; k < b->num_pairs; ++k) {
      const uint64_t n = b->q_off[k + 1] - b->q_off[k], m = b->s_off[k + 1] - b->s_off[k];
      if ((thr > 0 && n >= (uint64_t)ctx->batch_long_min && m >= (uint64_t)ctx->batch_long_min &&
           (long double)n * m >= (long double)thr) ||
          (small && n >= 256 && m >= 256 && acgt_only(b->s + b->s_off[k], m)))
        longs.push_back(k);
    }
  if (longs.empty()) return run_host_batch_core(ctx, prm, b, tb, scores, aln, cigar, cap, used);
  ctx->long_multi_pairs = 0;
  ctx->long_multi_ms = 0;
  if (!tb && !small) return run_host_batch_inplace(ctx, prm, b, longs, scores, aln);
  // the other pairs, compacted
  const uint64_t B = b->num_pairs, BL = longs.size(), BS = B - BL;
  std::vector<uint64_t> rest;
  rest.reserve(BS);
  {
    size_t x = 0;
    for (uint64_t k = 0; k < B; ++k) {
      if (x < BL && longs[x] == k) { ++x; continue; }
      rest.push_back(k);
    }
  }
  std::string cq, cs;
  std::vector<uint64_t> qo{0}, so{0};
  for (uint64_t k : rest) {
    cq.append(b->q + b->q_off[k], (size_t)(b->q_off[k + 1] - b->q_off[k]));
    cs.append(b->s + b->s_off[k], (size_t)(b->s_off[k + 1] - b->s_off[k]));
    qo.push_back(cq.size());
    so.push_back(cs.size());
  }
  const anyseq_batch b2{cq.data(), qo.data(), cs.data(), so.data(), BS};
  std::vector<int32_t> sc2(BS);
  std::vector<anyseq_alignment> al2((aln || tb) ? BS : 0);
  std::vector<uint32_t> cg2;
  uint64_t used2 = 0;
  auto run_short = [&]() -> int {
    if (!BS) return ANYSEQ_OK;
    if (tb) cg2.resize(std::max<uint64_t>(cq.size() + cs.size() + BS, 1));
    return run_host_batch_core(ctx, prm, &b2, tb, sc2.data(), al2.empty() ? nullptr : al2.data(),
                               tb ? cg2.data() : nullptr, cg2.size(), &used2);
  };
  // the long pairs: score-only on one device -> the bands of all of them in ONE launch
  // (run_long_multi, the device-side queue of SURVEY 8(f) f4) on the workspace's own
  // stream, and the short pairs' batch pipeline runs while it is in flight (its kernels
  // take the SMs the long launch's blocks leave as its queue drains); pairs the shared
  // launch does not take (subject with N, range guard) and traceback go one by one below
  std::vector<anyseq_alignment> al3(BL);
  std::vector<std::vector<uint32_t>> cg3(BL);
  std::vector<int> done(BL, 0);
  const bool multi = ctx->long_multi && BL >= 2 && ctx->devs.size() == 1;
  if (!multi) {
    const int r = run_short();
    if (r != ANYSEQ_OK) return (anyseq_status)r;
  } else {
    std::vector<uint64_t> ord(BL);
    for (uint64_t x = 0; x < BL; ++x) ord[x] = x;
    auto cells = [&](uint64_t x) {
      const uint64_t k = longs[x];
      return (long double)(b->q_off[k + 1] - b->q_off[k]) * (long double)(b->s_off[k + 1] - b->s_off[k]);
    };
    std::stable_sort(ord.begin(), ord.end(), [&](uint64_t u, uint64_t v) { return cells(u) > cells(v); });
    std::vector<LongPairIn> in(BL);
    for (uint64_t y = 0; y < BL; ++y) {
      const uint64_t k = longs[ord[y]];
      in[y] = LongPairIn{b->q + b->q_off[k], b->q_off[k + 1] - b->q_off[k], b->s + b->s_off[k],
                         b->s_off[k + 1] - b->s_off[k]};
    }
    const Device& D = ctx->devs[0];
    LongDevice ld;
    ld.id = D.id;
    ld.stream = D.stream;
    ld.num_sms = D.num_sms;
    ld.ws = ctx->lws[0].get();
    std::vector<LongResult> lr;
    std::vector<int> took;
    std::string err;
    uint64_t launches = 0;
    double kms = 0;
    int rs = ANYSEQ_OK;
    // traceback: the shared launch is the checkpointing forward pass of every pair, then
    // each pair's tile walk (run_long_traceback) from its checkpoints
    std::vector<LongCkpt> cks;
    const DevParams dp = dev_params(prm);
    const int rc = run_long_multi(ld, dp, in, ctx->long_opt, &lr, &took, &err, &launches, &kms,
                                  [&]() { return rs = run_short(); }, &ctx->long_multi_rows,
                                  tb ? &cks : nullptr, ctx->tb_budget);
    ctx->launches += launches;
    if (rs != ANYSEQ_OK) return (anyseq_status)rs;
    if (rc != 0) return fail(ctx, (anyseq_status)rc, "long pairs (one launch): %s", err.c_str());
    int8_t sig[25];
    for (int a = 0; a < 5; ++a)
      for (int c = 0; c < 5; ++c)
        sig[5 * a + c] = (int8_t)(prm->has_subst ? prm->subst[5 * a + c]
                                                 : ((a == c && a < 4) ? prm->match : prm->mismatch));
    for (uint64_t y = 0; y < BL; ++y) {
      if (!took[y]) continue;
      const uint64_t x = ord[y];
      memset(&al3[x], 0, sizeof(al3[x]));
      al3[x].score = lr[y].score;
      al3[x].q_end = al3[x].q_begin = lr[y].end_i;
      al3[x].s_end = al3[x].s_begin = lr[y].end_j;
      if (tb) {
        int64_t bi = 0, bj = 0;
        double wms = 0;
        uint64_t wl = 0;
        const int rw = run_long_traceback(ld, dp, sig, cks[y], lr[y].end_i, lr[y].end_j,
                                          (int64_t)in[y].n, (int64_t)in[y].m, &cg3[x], &bi, &bj,
                                          &wms, &err, &wl, (int)ctx->walk_helpers);
        ctx->launches += wl;
        if (rw != 0)
          return fail(ctx, (anyseq_status)rw, "pair %llu (long-pair walk): %s",
                      (unsigned long long)longs[x], err.c_str());
        al3[x].q_begin = bi;
        al3[x].s_begin = bj;
        al3[x].cigar_len = (uint32_t)cg3[x].size();
      }
      done[x] = 1;
      ++ctx->long_multi_pairs;
    }
    ctx->long_multi_ms = kms;
  }
  for (uint64_t x = 0; x < BL; ++x) {
    if (done[x]) continue;
    const uint64_t k = longs[x];
    const char* qk = b->q + b->q_off[k];
    const char* sk = b->s + b->s_off[k];
    const uint64_t n = b->q_off[k + 1] - b->q_off[k], m = b->s_off[k + 1] - b->s_off[k];
    anyseq_status r;
    if (tb) {
      cg3[x].resize(n + m + 1);
      uint64_t u = 0;
      r = run_traceback_long(ctx, prm, qk, n, sk, m, &al3[x], cg3[x].data(), cg3[x].size(), &u);
      cg3[x].resize(u);
    } else {
      r = anyseq_align_long(ctx, prm, qk, n, sk, m, &al3[x]);
    }
    if (r == ANYSEQ_E_UNSUPPORTED) {  // not for the long path: this pair on the batch path
      const uint64_t qo1[2] = {0, n}, so1[2] = {0, m};
      const anyseq_batch b1{qk, qo1, sk, so1, 1};
      int32_t sc1 = 0;
      uint64_t u1 = 0;
      if (tb) cg3[x].resize(n + m + 1);
      r = run_host_batch_core(ctx, prm, &b1, tb, &sc1, &al3[x], tb ? cg3[x].data() : nullptr,
                              tb ? cg3[x].size() : 0, &u1);
      if (tb) cg3[x].resize(u1);
      if (r == ANYSEQ_OK && !tb) al3[x].score = sc1;
    }
    if (r != ANYSEQ_OK) {
      ctx->err = "pair " + std::to_string(k) + " (long-pair path): " + ctx->err;
      return r;
    }
  }
  // merge in pair order
  uint64_t off = 0;
  size_t xl = 0, xs = 0;
  for (uint64_t k = 0; k < B; ++k) {
    const bool isl = xl < BL && longs[xl] == k;
    anyseq_alignment a;
    memset(&a, 0, sizeof(a));
    const uint32_t* ops = nullptr;
    if (isl) {
      a = al3[xl];
      ops = cg3[xl].data();
      ++xl;
    } else {
      if (!al2.empty()) a = al2[xs];
      if (!tb) a.score = sc2[xs];  // (traceback mode: the score is in the alignment struct)
      if (tb) ops = cg2.data() + al2[xs].cigar_offset;
      ++xs;
    }
    scores[k] = a.score;
    if (tb) {
      const uint32_t len = a.cigar_len;
      if (off + len <= cap && len) memcpy(cigar + off, ops, (size_t)len * sizeof(uint32_t));
      a.cigar_offset = off;
      off += len;
    }
    if (aln) aln[k] = a;
  }
  if (tb) {
    if (used) *used = off;
    if (off > cap)
      return fail(ctx, ANYSEQ_E_CAPACITY, "cigar needs %llu words, capacity %llu",
                  (unsigned long long)off, (unsigned long long)cap);
  }
  return ANYSEQ_OK;
}

// Append a run of `len` ops to a CIGAR, merging with the last word when the op repeats;
// a word holds at most 2^28 - 1 (len << 4 | op), so longer runs split into several words.
void push_run(std::vector<uint32_t>& ops, uint32_t op, uint64_t len) {
  constexpr uint64_t kMax = (1u << 28) - 1;
  if (!ops.empty() && (ops.back() & 15) == op) {
    const uint64_t room = kMax - (ops.back() >> 4), add = std::min(room, len);
    ops.back() += (uint32_t)(add << 4);
    len -= add;
  }
  for (; len > 0;) {
    const uint64_t k = std::min(kMax, len);
    ops.push_back((uint32_t)(k << 4) | op);
    len -= k;
  }
}

struct HbNode {
  int64_t i0, i1, j0, j1;
};

anyseq_status run_traceback_long_hirschberg(anyseq_ctx* ctx, const anyseq_params* prm, const char* q,
                                 uint64_t n, const char* s, uint64_t m, anyseq_alignment* out,
                                 uint32_t* cigar, uint64_t cap, uint64_t* used) {
  Device& D = ctx->devs[0];
  CK(cudaSetDevice(D.id));
  cudaStream_t st = D.stream;
  const DevParams dp = dev_params(prm);
  LrParams P;
  P.g = prm->gap_extend;
  for (int a = 0; a < 5; ++a)
    for (int b = 0; b < 5; ++b)
      P.sig[5 * a + b] = (int8_t)(prm->has_subst ? prm->subst[5 * a + b]
                                                 : ((a == b && a < 4) ? prm->match : prm->mismatch));
  (void)dp;
  // range guard: |H| <= (n + m) * max(g, |sigma|) must stay inside int32
  int64_t amax = P.g;
  for (int k = 0; k < 25; ++k) amax = std::max<int64_t>(amax, std::abs((int)P.sig[k]));
  if ((int64_t)(n + m + 2) * amax >= (1ll << 30))
    return fail(ctx, ANYSEQ_E_UNSUPPORTED, "score range of the long traceback exceeds int32");
  DevBuf asc, codes, bad, taskbuf, rows, best, sync;
  struct Guard {
    DevBuf* b[7];
    ~Guard() { for (auto* x : b) x->release(); }
  } guard{{&asc, &codes, &bad, &taskbuf, &rows, &best, &sync}};
  CK(asc.ensure(n + m + 16));
  CK(codes.ensure(n + m + 16));
  CK(bad.ensure(sizeof(int)));
  CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  if (n) CK(cudaMemcpyAsync(asc.as<char>(), q, n, cudaMemcpyHostToDevice, st));
  if (m) CK(cudaMemcpyAsync(asc.as<char>() + n, s, m, cudaMemcpyHostToDevice, st));
  launch_encode_codes(asc.as<char>(), codes.as<uint8_t>(), n + m, bad.as<int>(), st);
  ctx->launches += n + m ? 1 : 0;
  int h_bad = 0;
  CK(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h_bad) return fail(ctx, ANYSEQ_E_BADSEQ, "long traceback: byte outside ACGTNacgtn");
  const uint8_t* dq = codes.as<uint8_t>();
  const uint8_t* ds = codes.as<uint8_t>() + n;

  // region of the alignment: the whole matrix (global) or [begin, end) of a local optimum
  int64_t qb = 0, sb = 0, qe = (int64_t)n, se = (int64_t)m;
  int32_t want = 0;
  if (prm->kind != ANYSEQ_GLOBAL) {
    anyseq_alignment e;
    anyseq_status r = anyseq_align_long(ctx, prm, q, n, s, m, &e);
    if (r != ANYSEQ_OK) return r;
    want = e.score;
    qe = e.q_end;
    se = e.s_end;
    qb = qe;
    sb = se;
    const bool local = prm->kind == ANYSEQ_LOCAL;
    if (local ? e.score > 0 : (qe > 0 && se > 0)) {
      // anchored reverse pass over the prefixes ending at the end cell: its optimum is the
      // score of the best alignment ending there (= the local optimum), its cell the begin;
      // semi-global: the best over begins on row 0 / column 0 (the pass's last row / column)
      CK(cudaSetDevice(D.id));
      const int nb = lastrow_bands((int)qe);
      CK(rows.ensure((se + 1) * sizeof(int32_t)));
      CK(best.ensure(3 * (size_t)nb * sizeof(int32_t)));
      CK(sync.ensure((2 + (size_t)nb) * sizeof(int)));
      CK(cudaMemsetAsync(sync.p, 0, (2 + (size_t)nb) * sizeof(int), st));
      LrTask t{dq, ds, (int32_t)qe, (int32_t)se, 1, 1, rows.as<int32_t>(), best.as<int32_t>()};
      CK(taskbuf.ensure(sizeof(LrTask) + sizeof(int)));
      struct {
        LrTask t;
        int bs;
      } up{t, 0};
      CK(cudaMemcpyAsync(taskbuf.p, &up, sizeof(up), cudaMemcpyHostToDevice, st));
      const int* bstart = reinterpret_cast<const int*>(taskbuf.as<char>() + sizeof(LrTask));
      if (local) launch_lastrow_anchored(taskbuf.as<LrTask>(), bstart, 1, nb, sync.as<int>(), P, st);
      else launch_lastrow_edges(taskbuf.as<LrTask>(), bstart, 1, nb, sync.as<int>(), P, st);
      ctx->launches += 1;
      std::vector<int32_t> hbb(3 * (size_t)nb);
      CK(cudaMemcpyAsync(hbb.data(), best.p, hbb.size() * sizeof(int32_t),
                         cudaMemcpyDeviceToHost, st));
      int h_abort = 0;
      CK(cudaMemcpyAsync(&h_abort, sync.as<int>() + 1 + nb, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      CK(cudaGetLastError());
      if (h_abort) return fail(ctx, ANYSEQ_E_TIMEOUT, "long traceback: a band wait exceeded its bound");
      int32_t hb[3] = {hbb[0], hbb[1], hbb[2]};  // key: score desc, j asc, i asc (R10)
      for (int b = 1; b < nb; ++b) {
        const int32_t* x = hbb.data() + 3 * b;
        if (x[0] > hb[0] || (x[0] == hb[0] && (x[2] < hb[2] || (x[2] == hb[2] && x[1] < hb[1]))))
          hb[0] = x[0], hb[1] = x[1], hb[2] = x[2];
      }
      if (!local) {  // border cells of the pass: all of q against nothing, or all of s
        const int64_t cand[2][3] = {{-qe * (int64_t)P.g, qe, 0}, {-se * (int64_t)P.g, 0, se}};
        for (auto& c : cand)
          if (c[0] > hb[0] || (c[0] == hb[0] && (c[2] < hb[2] || (c[2] == hb[2] && c[1] < hb[1]))))
            hb[0] = (int32_t)c[0], hb[1] = (int32_t)c[1], hb[2] = (int32_t)c[2];
      }
      if (hb[0] != e.score)
        return fail(ctx, ANYSEQ_E_CUDA, "anchored pass optimum %d != long-kernel optimum %d", hb[0],
                    e.score);
      qb = qe - hb[1];
      sb = se - hb[2];
    }
  }

  // Hirschberg levels; nodes stay in path order
  ctx->tb_pass_ms = ctx->tb_pass_cells = 0;
  cudaEvent_t ev0, ev1;
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() { cudaEventDestroy(a); cudaEventDestroy(b); }
  } evg{ev0, ev1};
  const int64_t kLeafCells = ctx->tb_leaf_cells;
  std::vector<HbNode> nodes{{qb, qe, sb, se}};
  std::vector<char> leaf(1, 0);
  std::vector<int32_t> hrows;
  for (;;) {
    std::vector<LrTask> tasks;
    std::vector<size_t> split_nodes, row_off;
    size_t total = 0;
    for (size_t k = 0; k < nodes.size(); ++k) {
      if (leaf[k]) continue;
      const HbNode& x = nodes[k];
      const int64_t r = x.i1 - x.i0, c = x.j1 - x.j0;
      if (r <= 1 || c <= 1 || r * c <= kLeafCells) {
        leaf[k] = 1;
        continue;
      }
      const int64_t mid = (x.i0 + x.i1) / 2;
      split_nodes.push_back(k);
      row_off.push_back(total);
      tasks.push_back(LrTask{dq + x.i0, ds + x.j0, (int32_t)(mid - x.i0), (int32_t)c, 0, 0,
                             nullptr, nullptr});
      tasks.push_back(LrTask{dq + mid, ds + x.j0, (int32_t)(x.i1 - mid), (int32_t)c, 1, 0,
                             nullptr, nullptr});
      total += 2 * (size_t)(c + 1);
    }
    if (tasks.empty()) break;
    CK(rows.ensure(total * sizeof(int32_t)));
    for (size_t t = 0; t < split_nodes.size(); ++t) {
      const int64_t c = nodes[split_nodes[t]].j1 - nodes[split_nodes[t]].j0;
      tasks[2 * t].row = rows.as<int32_t>() + row_off[t];
      tasks[2 * t + 1].row = rows.as<int32_t>() + row_off[t] + c + 1;
    }
    // task array, then the first band of every task
    const size_t tb = tasks.size() * sizeof(LrTask);
    std::vector<char> up(tb + tasks.size() * sizeof(int));
    memcpy(up.data(), tasks.data(), tb);
    int nb = 0;
    for (size_t k = 0; k < tasks.size(); ++k) {
      memcpy(up.data() + tb + k * sizeof(int), &nb, sizeof(int));
      nb += lastrow_bands(tasks[k].n1);
    }
    CK(taskbuf.ensure(up.size()));
    CK(cudaMemcpyAsync(taskbuf.p, up.data(), up.size(), cudaMemcpyHostToDevice, st));
    CK(sync.ensure((2 + (size_t)nb) * sizeof(int)));
    CK(cudaMemsetAsync(sync.p, 0, (2 + (size_t)nb) * sizeof(int), st));
    CK(cudaEventRecord(ev0, st));
    launch_lastrow(taskbuf.as<LrTask>(), reinterpret_cast<const int*>(taskbuf.as<char>() + tb),
                   (int)tasks.size(), nb, sync.as<int>(), P, st);
    CK(cudaEventRecord(ev1, st));
    ctx->launches += 1;
    CK(cudaGetLastError());
    hrows.resize(total);
    CK(cudaMemcpyAsync(hrows.data(), rows.p, total * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    int h_abort = 0;
    CK(cudaMemcpyAsync(&h_abort, sync.as<int>() + 1 + nb, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h_abort) return fail(ctx, ANYSEQ_E_TIMEOUT, "long traceback: a band wait exceeded its bound");
    float lvl_ms = 0;
    CK(cudaEventElapsedTime(&lvl_ms, ev0, ev1));
    ctx->tb_pass_ms += lvl_ms;
    for (const LrTask& x : tasks) ctx->tb_pass_cells += (double)x.n1 * x.m1;
    std::vector<HbNode> nn;
    std::vector<char> nl;
    size_t t = 0;
    for (size_t k = 0; k < nodes.size(); ++k) {
      if (t < split_nodes.size() && split_nodes[t] == k) {
        const HbNode x = nodes[k];
        const int64_t c = x.j1 - x.j0, mid = (x.i0 + x.i1) / 2;
        const int32_t* F = hrows.data() + row_off[t];
        const int32_t* B = F + c + 1;
        const int64_t top = mid - x.i0, bot = x.i1 - mid;
        int64_t bj = 0, bv = INT64_MIN;
        for (int64_t j = 0; j <= c; ++j) {
          const int64_t f = j == 0 ? -top * (int64_t)P.g : F[j];
          const int64_t b = j == c ? -bot * (int64_t)P.g : B[c - j];
          if (f + b > bv) {
            bv = f + b;
            bj = j;
          }
        }
        nn.push_back({x.i0, mid, x.j0, x.j0 + bj});
        nn.push_back({mid, x.i1, x.j0 + bj, x.j1});
        nl.push_back(0);
        nl.push_back(0);
        ++t;
      } else {
        nn.push_back(nodes[k]);
        nl.push_back(leaf[k]);
      }
    }
    nodes.swap(nn);
    leaf.swap(nl);
  }

  // leaves: one batched global traceback over consecutive q / s ranges.  One-row and
  // one-column leaves (a long indel crossing a cut) can be arbitrarily long and would size
  // the batch's per-variant scratch by their length: they are solved here in closed form
  // (global, linear gaps: the best single match plus gaps, or the all-gap path).
  const uint64_t L = nodes.size();
  auto code_of = [](char ch) -> int {
    const int x = ch | 0x20;
    return x == 'a' ? 0 : x == 'c' ? 1 : x == 'g' ? 2 : x == 't' ? 3 : 4;
  };
  auto sig_of = [&](int a, int b) -> int64_t {
    return prm->has_subst ? prm->subst[5 * a + b] : ((a == b && a < 4) ? prm->match : prm->mismatch);
  };
  const int64_t g = prm->gap_extend;
  std::vector<char> thin(L, 0);
  std::vector<uint64_t> thick;
  for (uint64_t k = 0; k < L; ++k) {
    const HbNode& x = nodes[k];
    if (x.i1 - x.i0 <= 1 || x.j1 - x.j0 <= 1) thin[k] = 1;
    else thick.push_back(k);
  }
  std::vector<anyseq_alignment> la(thick.size());
  std::vector<uint32_t> lc;
  uint64_t lused = 0;
  const auto tl0 = std::chrono::steady_clock::now();
  if (!thick.empty()) {
    // the thick leaves' ranges, copied back to back into one CSR batch (thin leaves between
    // them leave gaps in q and s, so the original buffers cannot serve as the CSR)
    std::vector<uint64_t> bq{0}, bs{0};
    std::string cq, cs;
    for (uint64_t k : thick) {
      const HbNode& x = nodes[k];
      cq.append(q + x.i0, (size_t)(x.i1 - x.i0));
      cs.append(s + x.j0, (size_t)(x.j1 - x.j0));
      bq.push_back(cq.size());
      bs.push_back(cs.size());
    }
    const uint64_t B = thick.size();
    anyseq_batch lb{cq.data(), bq.data(), cs.data(), bs.data(), B};
    anyseq_params gp = *prm;
    gp.kind = ANYSEQ_GLOBAL;
    const uint64_t lcap = cq.size() + cs.size() + B;
    lc.resize(std::max<uint64_t>(lcap, 1));
    std::vector<int32_t> lsc(B);
    // leaves stay on the batch kernel (the routing wrapper could send a few large leaves back
    // to the long-pair path, i.e. into this recursion again)
    anyseq_status r = run_host_batch_core(ctx, &gp, &lb, 1, lsc.data(), la.data(), lc.data(), lcap, &lused);
    if (r != ANYSEQ_OK) return r;
  }
  ctx->tb_leaf_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl0).count();
  int64_t score = 0;
  std::vector<uint32_t> ops;
  size_t tk = 0;
  for (uint64_t k = 0; k < L; ++k) {
    const HbNode& x = nodes[k];
    if (!thin[k]) {
      const anyseq_alignment& a = la[tk++];
      score += a.score;
      for (uint32_t w = 0; w < a.cigar_len; ++w) {
        const uint32_t word = lc[a.cigar_offset + w];
        push_run(ops, word & 15, word >> 4);
      }
      continue;
    }
    const int64_t r = x.i1 - x.i0, c = x.j1 - x.j0;
    if (r == 0 || c == 0) {  // one gap run
      if (r) push_run(ops, 1u, (uint64_t)r);
      if (c) push_run(ops, 2u, (uint64_t)c);
      score -= (r + c) * g;
      continue;
    }
    // r == 1 or c == 1: the best single match (first maximiser) or the all-gap path
    const bool row = r == 1;
    const int64_t len = row ? c : r;
    int64_t bv = INT64_MIN, bk = 0;
    for (int64_t k2 = 0; k2 < len; ++k2) {
      const int64_t v = row ? sig_of(code_of(q[x.i0]), code_of(s[x.j0 + k2]))
                            : sig_of(code_of(q[x.i0 + k2]), code_of(s[x.j0]));
      if (v > bv) { bv = v; bk = k2; }
    }
    const uint32_t gapop = row ? 2u : 1u;  // the long side's gaps
    if (bv - (len - 1) * g >= -(len + 1) * g) {
      push_run(ops, gapop, (uint64_t)bk);
      push_run(ops, 0u, 1);
      push_run(ops, gapop, (uint64_t)(len - 1 - bk));
      score += bv - (len - 1) * g;
    } else {
      push_run(ops, row ? 1u : 2u, 1);
      push_run(ops, gapop, (uint64_t)len);
      score -= (len + 1) * g;
    }
  }
  if (prm->kind != ANYSEQ_GLOBAL && score != want)
    return fail(ctx, ANYSEQ_E_CUDA, "long traceback: path score %lld != optimum %d",
                (long long)score, want);
  if (used) *used = ops.size();
  if (ops.size() > cap)
    return fail(ctx, ANYSEQ_E_CAPACITY, "cigar needs %llu words, capacity %llu",
                (unsigned long long)ops.size(), (unsigned long long)cap);
  if (!ops.empty()) memcpy(cigar, ops.data(), ops.size() * sizeof(uint32_t));
  memset(out, 0, sizeof(*out));
  out->score = (int32_t)score;
  out->q_begin = qb;
  out->s_begin = sb;
  out->q_end = qe;
  out->s_end = se;
  out->cigar_offset = 0;
  out->cigar_len = (uint32_t)ops.size();
  return ANYSEQ_OK;
}

// Linear-space long traceback from checkpoints (long_tb.cu): ONE forward pass of the 16-bit
// long kernel keeps the DP rows at row-block and the DP columns at column-block boundaries
// (and finds the optimum); the walk recomputes one tile at a time from them, so every
// decision is the full-matrix one (bit-exact with the oracle's traceback), for every kind
// and both gap models.  Falls back to Hirschberg (linear gaps only) when the 16-bit kernel
// cannot run the pair (an N in the subject, or the range guard).
anyseq_status run_traceback_long(anyseq_ctx* ctx, const anyseq_params* prm, const char* q,
                                 uint64_t n, const char* s, uint64_t m, anyseq_alignment* out,
                                 uint32_t* cigar, uint64_t cap, uint64_t* used) {
  ctx->tb_pass_ms = ctx->tb_pass_cells = ctx->tb_walk_ms = ctx->tb_ckpt_bytes = 0;
  ctx->tb_leaf_ms = 0;
  ctx->tb_method = 1;
  const DevParams dp = dev_params(prm);
  memset(out, 0, sizeof(*out));
  std::vector<uint32_t> ops;
  if (n == 0 || m == 0) {  // one gap run (global) or the empty alignment
    if (prm->kind == ANYSEQ_GLOBAL && n + m) {
      push_run(ops, n ? 1u : 2u, n + m);
      out->score = (int32_t)(-(dp.go + (int64_t)(n + m) * dp.ge));
      out->q_end = (int64_t)n;
      out->s_end = (int64_t)m;
    }
  } else {
    Device& D = ctx->devs[0];
    CK(cudaSetDevice(D.id));
    LongDevice ld{D.id, D.stream, D.num_sms, ctx->lws[0].get()};
    std::vector<LongDevice> one{ld};
    LongCkpt ck;
    ck.want = 1;
    ck.budget = ctx->tb_budget;
    ck.force_kc_shift = (int)ctx->tb_kc_shift;
    ck.force_ck_every = (int)ctx->tb_ck_every;
    LongResult r;
    std::string err;
    uint64_t launches = 0;
    const auto tl0 = std::chrono::steady_clock::now();
    auto tl_ms = [&]() {
      return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl0).count();
    };
    int rc;
    {
      NvtxRange nvtx("checkpointed forward pass");
      rc = run_long(one, dp, q, n, s, m, ctx->long_opt, &r, &err, &launches, &ck);
    }
    ctx->launches += launches;
    if (ctx->timing >= 2)
      fprintf(stderr, "[tb-long] pass done %.1f ms (kernel %.1f ms)\n", tl_ms(), r.kernel_ms);
    if (rc == ANYSEQ_E_UNSUPPORTED && prm->gap == ANYSEQ_GAP_LINEAR) {
      ctx->tb_method = 2;
      return run_traceback_long_hirschberg(ctx, prm, q, n, s, m, out, cigar, cap, used);
    }
    if (rc != 0) return fail(ctx, (anyseq_status)rc, "%s", err.c_str());
    ctx->tb_pass_ms = r.kernel_ms;
    ctx->tb_pass_cells = (double)n * (double)m;
    ctx->tb_ckpt_bytes = (double)ck.bytes;
    int8_t sig[25];
    for (int a = 0; a < 5; ++a)
      for (int b = 0; b < 5; ++b)
        sig[5 * a + b] = (int8_t)(prm->has_subst ? prm->subst[5 * a + b]
                                                 : ((a == b && a < 4) ? prm->match : prm->mismatch));
    int64_t bi = 0, bj = 0;
    double wms = 0;
    launches = 0;
    int64_t tiles = 0, hits = 0;
    NvtxRange nvtx_walk("checkpoint tile walk");
    rc = run_long_traceback(ld, dp, sig, ck, r.end_i, r.end_j, (int64_t)n, (int64_t)m, &ops, &bi,
                            &bj, &wms, &err, &launches, (int)ctx->walk_helpers, &tiles, &hits,
                            ctx->timing >= 2);
    if (ctx->timing >= 2)
      fprintf(stderr, "[tb-long] walk done %.1f ms (kernel %.1f ms, tiles %lld)\n", tl_ms(), wms,
              (long long)tiles);
    ctx->tb_tiles = (double)tiles;
    ctx->tb_hits = (double)hits;
    ctx->launches += launches;
    if (rc != 0) return fail(ctx, (anyseq_status)rc, "%s", err.c_str());
    ctx->tb_walk_ms = wms;
    out->score = r.score;
    out->q_begin = bi;
    out->s_begin = bj;
    out->q_end = r.end_i;
    out->s_end = r.end_j;
  }
  if (used) *used = ops.size();
  if (ops.size() > cap)
    return fail(ctx, ANYSEQ_E_CAPACITY, "cigar needs %llu words, capacity %llu",
                (unsigned long long)ops.size(), (unsigned long long)cap);
  if (!ops.empty()) memcpy(cigar, ops.data(), ops.size() * sizeof(uint32_t));
  out->cigar_offset = 0;
  out->cigar_len = (uint32_t)ops.size();
  return ANYSEQ_OK;
}

}  // namespace

// =========================================================================== C-ABI
extern "C" {

static anyseq_status create_impl(anyseq_ctx** out, const int* device_ids, int num_devices);

anyseq_status anyseq_create(anyseq_ctx** out, const int* device_ids, int num_devices) {
  if (!out) return ANYSEQ_E_INVALID;
  *out = nullptr;
  try {
    return create_impl(out, device_ids, num_devices);
  } catch (const std::bad_alloc&) {
    return ANYSEQ_E_NOMEM;
  } catch (...) {
    return ANYSEQ_E_CUDA;
  }
}

static anyseq_status create_impl(anyseq_ctx** out, const int* device_ids, int num_devices) {
  if (num_devices < 1) return ANYSEQ_E_INVALID;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return ANYSEQ_E_CUDA;
  }
  anyseq_ctx* c = new (std::nothrow) anyseq_ctx();
  if (!c) return ANYSEQ_E_NOMEM;
  for (int g = 0; g < num_devices; ++g) {
    const int id = device_ids ? device_ids[g] : g;
    if (id < 0 || id >= ndev) {
      anyseq_destroy(c);
      return ANYSEQ_E_INVALID;
    }
    Device D;
    D.id = id;
    if (cudaSetDevice(id) != cudaSuccess ||
        cudaStreamCreateWithFlags(&D.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaDeviceGetAttribute(&D.num_sms, cudaDevAttrMultiProcessorCount, id) != cudaSuccess ||
        cudaHostAlloc((void**)&D.h_sum, sizeof(PlanSummary), cudaHostAllocMapped) != cudaSuccess ||
        cudaMallocHost(&D.h_small, 64) != cudaSuccess ||
        cudaStreamCreateWithFlags(&D.copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&D.ev_up[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&D.ev_up[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&D.ev_free[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&D.ev_free[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&D.ev_fork, cudaEventDisableTiming) != cudaSuccess) {
      c->devs.push_back(D);
      anyseq_destroy(c);
      return ANYSEQ_E_CUDA;
    }
    bool vok = true;
    for (int v = 0; v < NV && vok; ++v)
      vok = cudaStreamCreateWithFlags(&D.vstream[v], cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&D.ev_join[v], cudaEventDisableTiming) == cudaSuccess;
    c->devs.push_back(D);
    if (!vok) {
      anyseq_destroy(c);
      return ANYSEQ_E_CUDA;
    }
  }
  for (size_t d = 0; d < c->devs.size(); ++d) c->lws.emplace_back(new LongWs());
  cudaSetDevice(c->devs[0].id);
  *out = c;
  return ANYSEQ_OK;
}

static void destroy_impl(anyseq_ctx* c);

void anyseq_destroy(anyseq_ctx* c) {
  if (!c) return;
  try {
    destroy_impl(c);
  } catch (...) {  // nothing crosses the ABI; the context memory is released regardless
  }
}

static void destroy_impl(anyseq_ctx* c) {
  resolve_events(c);
  for (size_t d = 0; d < c->lws.size(); ++d) {
    cudaSetDevice(c->devs[d].id);
    c->lws[d]->release();
  }
  for (auto& e : c->pool) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (auto& D : c->devs) {
    cudaSetDevice(D.id);
    DevBuf* bufs[] = {&D.q_ascii, &D.s_ascii, &D.q_code, &D.s_code, &D.q_off, &D.s_off,
                      &D.flags,   &D.keys,    &D.keys2,  &D.vals,   &D.vals2, &D.slots,
                      &D.scores,  &D.end_i,   &D.end_j,  &D.beg_i,  &D.beg_j, &D.n_ops,
                      &D.cig_off, &D.ops,     &D.dirs,   &D.tb,     &D.strip, &D.aln,
                      &D.cigar,   &D.temp,    &D.sum,    &D.long_ws, &D.tickets};
    for (DevBuf* b : bufs) b->release();
    D.h_stage.release();
    for (auto& hp : D.h_pack) hp.release();
    if (D.h_sum) cudaFreeHost(D.h_sum);
    if (D.h_small) cudaFreeHost(D.h_small);
    for (int i = 0; i < 2; ++i) {
      D.q_ascii2[i].release();
      D.s_ascii2[i].release();
      D.q_off2[i].release();
      D.s_off2[i].release();
      if (D.ev_up[i]) cudaEventDestroy(D.ev_up[i]);
      if (D.ev_free[i]) cudaEventDestroy(D.ev_free[i]);
    }
    for (int v = 0; v < NV; ++v) {
      D.strip_v[v].release();
      D.dirs_v[v].release();
      if (D.vstream[v]) cudaStreamDestroy(D.vstream[v]);
      if (D.ev_join[v]) cudaEventDestroy(D.ev_join[v]);
    }
    if (D.ev_fork) cudaEventDestroy(D.ev_fork);
    if (D.copy_stream) cudaStreamDestroy(D.copy_stream);
    if (D.stream) cudaStreamDestroy(D.stream);
  }
  delete c;
}

anyseq_status anyseq_align_batch(anyseq_ctx* ctx, const anyseq_params* params,
                                 const anyseq_batch* batch, int32_t* scores,
                                 anyseq_alignment* ends) {
  if (!ctx) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    NvtxRange nvtx("anyseq_align_batch");
    anyseq_status s = validate_params(ctx, params);
    if (s != ANYSEQ_OK) return s;
    if ((s = check_batch_host(ctx, batch)) != ANYSEQ_OK) return s;
    if (batch->num_pairs == 0) return ANYSEQ_OK;
    if (!scores) return fail(ctx, ANYSEQ_E_INVALID, "scores is NULL");
    return run_host_batch(ctx, params, batch, 0, scores, ends, nullptr, 0, nullptr);
  });
}

anyseq_status anyseq_traceback(anyseq_ctx* ctx, const anyseq_params* params,
                               const anyseq_batch* batch, anyseq_alignment* out, uint32_t* cigar,
                               uint64_t cigar_capacity, uint64_t* cigar_used) {
  if (!ctx) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    NvtxRange nvtx("anyseq_traceback");
    anyseq_status s = validate_params(ctx, params);
    if (s != ANYSEQ_OK) return s;
    if ((s = check_batch_host(ctx, batch)) != ANYSEQ_OK) return s;
    if (cigar_used) *cigar_used = 0;
    if (batch->num_pairs == 0) return ANYSEQ_OK;
    if (!out) return fail(ctx, ANYSEQ_E_INVALID, "out is NULL");
    if (!cigar && cigar_capacity) return fail(ctx, ANYSEQ_E_INVALID, "cigar is NULL");
    std::vector<int32_t> scores(batch->num_pairs);
    return run_host_batch(ctx, params, batch, 1, scores.data(), out, cigar, cigar_capacity,
                          cigar_used);
  });
}

anyseq_status anyseq_align_batch_device(anyseq_ctx* ctx, const anyseq_params* params,
                                        const anyseq_batch* d_batch, int32_t* d_scores,
                                        anyseq_alignment* d_ends, void* stream) {
  if (!ctx) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    NvtxRange nvtx("anyseq_align_batch_device");
    anyseq_status s = validate_params(ctx, params);
    if (s != ANYSEQ_OK) return s;
    if (!d_batch) return fail(ctx, ANYSEQ_E_INVALID, "batch is NULL");
    if (d_batch->num_pairs == 0) return ANYSEQ_OK;
    if (!d_batch->q_off || !d_batch->s_off || !d_scores)
      return fail(ctx, ANYSEQ_E_INVALID, "NULL device pointer");
    if (d_batch->num_pairs >= (1ull << 31)) return fail(ctx, ANYSEQ_E_INVALID, "too many pairs");
    Device& D = ctx->devs[0];
    CK(cudaSetDevice(D.id));
    cudaStream_t user = (cudaStream_t)stream;
    // order the context stream after the caller's stream, run, then order the caller after us
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, user));
    CK(cudaStreamWaitEvent(D.stream, ev, 0));
    // absolute ends of the CSR ranges
    CK(cudaMemcpyAsync(D.h_small, d_batch->q_off + d_batch->num_pairs, 8, cudaMemcpyDeviceToHost, D.stream));
    CK(cudaMemcpyAsync(D.h_small + 1, d_batch->s_off + d_batch->num_pairs, 8, cudaMemcpyDeviceToHost, D.stream));
    CK(cudaStreamSynchronize(D.stream));
    DeviceJob J;
    J.d_q = d_batch->q;
    J.d_qoff = d_batch->q_off;
    J.d_s = d_batch->s;
    J.d_soff = d_batch->s_off;
    J.B = d_batch->num_pairs;
    J.q_end = D.h_small[0];
    J.s_end = D.h_small[1];
    J.tb = 0;
    J.want_ends = d_ends != nullptr;
    J.d_scores_out = d_scores;
    J.d_aln_out = d_ends;
    s = run_device(ctx, D, params, J, nullptr, 0);
    CK(cudaEventRecord(ev, D.stream));
    CK(cudaStreamWaitEvent(user, ev, 0));
    cudaEventDestroy(ev);
    return s;
  });
}

anyseq_status anyseq_sync(anyseq_ctx* ctx) {
  if (!ctx) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    for (auto& D : ctx->devs) {
      CK(cudaSetDevice(D.id));
      CK(cudaStreamSynchronize(D.stream));
    }
    return ANYSEQ_OK;
  });
}

uint64_t anyseq_kernel_launches(const anyseq_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

anyseq_status anyseq_set_option(anyseq_ctx* ctx, const char* name, int64_t value) {
  if (!ctx || !name) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    std::string n(name);
    if (n == "tb_scratch_bytes") { ctx->tb_scratch_bytes = std::max<int64_t>(value, 1 << 20); return ANYSEQ_OK; }
    if (n == "timing") { ctx->timing = (int)value; return ANYSEQ_OK; }
    if (n == "force_variant") { ctx->force_variant = value; return ANYSEQ_OK; }
    if (n == "chunk_bytes") { ctx->chunk_bytes = std::max<int64_t>(value, 1 << 16); return ANYSEQ_OK; }
    if (n == "allow16") { ctx->allow16 = value ? 1 : 0; return ANYSEQ_OK; }
    if (n == "pack2") { ctx->pack2 = value ? 1 : 0; return ANYSEQ_OK; }
    if (n == "tb8") { ctx->tb8 = value ? 1 : 0; return ANYSEQ_OK; }
    if (n == "batch_long_cells") { ctx->batch_long_cells = std::max<int64_t>(value, 0); return ANYSEQ_OK; }
    if (n == "batch_long_cells_tb") { ctx->batch_long_cells_tb = std::max<int64_t>(value, 0); return ANYSEQ_OK; }
    if (n == "batch_long_min") { ctx->batch_long_min = std::max<int64_t>(value, 1); return ANYSEQ_OK; }
    if (n == "long_multi") { ctx->long_multi = value ? 1 : 0; return ANYSEQ_OK; }
    if (n == "batch_long_small") { ctx->batch_long_small = std::max<int64_t>(value, 0); return ANYSEQ_OK; }
    if (n == "pack2_percent") {
      if (value < 0 || value > 100) return fail(ctx, ANYSEQ_E_INVALID, "pack2_percent in [0, 100]");
      ctx->pack2_percent = value;
      return ANYSEQ_OK;
    }
    if (n == "tb_ckpt_bytes") { ctx->tb_budget = std::max<int64_t>(value, 0); return ANYSEQ_OK; }
    if (n == "walk_helpers") { ctx->walk_helpers = std::max<int64_t>(value, 0); return ANYSEQ_OK; }
    if (n == "tb_kc_shift") {
      if (value != 0 && (value < 8 || value > 12))
        return fail(ctx, ANYSEQ_E_INVALID, "tb_kc_shift must be 0 or in [8, 12]");
      ctx->tb_kc_shift = value;
      return ANYSEQ_OK;
    }
    if (n == "tb_ck_every") {
      if (value < 0 || value > 8) return fail(ctx, ANYSEQ_E_INVALID, "tb_ck_every must be in [0, 8]");
      ctx->tb_ck_every = value;
      return ANYSEQ_OK;
    }
    if (n == "tb_leaf_cells") {
      if (value < 1) return fail(ctx, ANYSEQ_E_INVALID, "tb_leaf_cells must be >= 1");
      ctx->tb_leaf_cells = value;
      return ANYSEQ_OK;
    }
    if (n == "long_band_rows") { ctx->long_opt.band_rows = (int)value; return ANYSEQ_OK; }
    if (n == "long_blocks") { ctx->long_opt.blocks = (int)value; return ANYSEQ_OK; }
    if (n == "long_strips") { ctx->long_opt.virtual_strips = (int)value; return ANYSEQ_OK; }
    if (n == "long_profile") { ctx->long_opt.profile = (int)value; return ANYSEQ_OK; }
    if (n == "long_start_lag") { ctx->long_opt.start_lag = (int)value; return ANYSEQ_OK; }
    if (n == "long_sleep_ns") { ctx->long_opt.sleep_ns = (int)value; return ANYSEQ_OK; }
    if (n == "long_narrow") { ctx->long_opt.narrow = (int)value; return ANYSEQ_OK; }
    if (n == "long_spin_limit") {
      ctx->long_opt.spin_limit = value > 0 ? (long long)value : (1ll << 28);
      return ANYSEQ_OK;
    }
    if (n == "long_multi_group") { ctx->long_opt.multi_group = (int)std::max<int64_t>(value, 1); return ANYSEQ_OK; }
    if (n == "long_stall_task") { ctx->long_opt.stall_task = (int)value; return ANYSEQ_OK; }
    if (n == "long_chunk_cols") { ctx->long_opt.chunk_cols = (int)value; return ANYSEQ_OK; }
    return fail(ctx, ANYSEQ_E_INVALID, "unknown option %s", name);
  });
}

anyseq_status anyseq_align_long(anyseq_ctx* ctx, const anyseq_params* params, const char* q,
                                uint64_t n, const char* s, uint64_t m, anyseq_alignment* out) {
  if (!ctx) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    NvtxRange nvtx("anyseq_align_long");
    anyseq_status st = validate_params(ctx, params);
    if (st != ANYSEQ_OK) return st;
    if (!out) return fail(ctx, ANYSEQ_E_INVALID, "out is NULL");
    if ((n && !q) || (m && !s)) return fail(ctx, ANYSEQ_E_INVALID, "sequence pointer is NULL");
    if (n >= (1ull << 31) || m >= (1ull << 31))
      return fail(ctx, ANYSEQ_E_UNSUPPORTED, "long sequences must be shorter than 2^31");
    std::vector<LongDevice> ld;
    for (size_t d = 0; d < ctx->devs.size(); ++d) {
      const Device& D = ctx->devs[d];
      LongDevice x;
      x.id = D.id;
      x.stream = D.stream;
      x.num_sms = D.num_sms;
      x.ws = ctx->lws[d].get();
      ld.push_back(x);
    }
    std::string err;
    uint64_t launches = 0;
    LongResult r;
    const int rc = run_long(ld, dev_params(params), q, n, s, m, ctx->long_opt, &r, &err, &launches);
    ctx->launches += launches;
    if (rc != 0) return fail(ctx, (anyseq_status)rc, "%s", err.c_str());
    ctx->long_narrow = r.narrow ? 1 : 0;
    ctx->long_ms = r.kernel_ms;
    memset(out, 0, sizeof(*out));
    out->score = r.score;
    out->q_end = out->q_begin = r.end_i;
    out->s_end = out->s_begin = r.end_j;
    return ANYSEQ_OK;
  });
}

anyseq_status anyseq_traceback_long(anyseq_ctx* ctx, const anyseq_params* params, const char* q,
                                    uint64_t n, const char* s, uint64_t m, anyseq_alignment* out,
                                    uint32_t* cigar, uint64_t cigar_capacity,
                                    uint64_t* cigar_used) {
  if (!ctx) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    NvtxRange nvtx("anyseq_traceback_long");
    anyseq_status st = validate_params(ctx, params);
    if (st != ANYSEQ_OK) return st;
    if (cigar_used) *cigar_used = 0;
    if (!out) return fail(ctx, ANYSEQ_E_INVALID, "out is NULL");
    if (!cigar && cigar_capacity) return fail(ctx, ANYSEQ_E_INVALID, "cigar is NULL");
    if ((n && !q) || (m && !s)) return fail(ctx, ANYSEQ_E_INVALID, "sequence pointer is NULL");
    if (n >= (1ull << 31) || m >= (1ull << 31))
      return fail(ctx, ANYSEQ_E_UNSUPPORTED, "long sequences must be shorter than 2^31");
    return run_traceback_long(ctx, params, q, n, s, m, out, cigar, cigar_capacity, cigar_used);
  });
}

anyseq_status anyseq_get_stat(anyseq_ctx* ctx, const char* name, double* value) {
  if (!ctx || !name || !value) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    for (auto& D : ctx->devs) {
      cudaSetDevice(D.id);
    }
    resolve_events(ctx);
    std::string n(name);
    if (n == "fill_ms") { *value = ctx->fill_ms; return ANYSEQ_OK; }
    if (n == "walk_ms") { *value = ctx->walk_ms; return ANYSEQ_OK; }
    if (n == "long_narrow") { *value = ctx->long_narrow; return ANYSEQ_OK; }
    if (n == "long_multi_pairs") { *value = (double)ctx->long_multi_pairs; return ANYSEQ_OK; }
    if (n == "long_multi_ms") { *value = ctx->long_multi_ms; return ANYSEQ_OK; }
    if (n == "long_multi_rows") { *value = ctx->long_multi_rows; return ANYSEQ_OK; }
    if (n == "long_kernel_ms") { *value = ctx->long_ms; return ANYSEQ_OK; }
    if (n == "tb_pass_ms") { *value = ctx->tb_pass_ms; return ANYSEQ_OK; }
    if (n == "tb_pass_cells") { *value = ctx->tb_pass_cells; return ANYSEQ_OK; }
    if (n == "tb_leaf_ms") { *value = ctx->tb_leaf_ms; return ANYSEQ_OK; }
    if (n == "tb_walk_ms") { *value = ctx->tb_walk_ms; return ANYSEQ_OK; }
    if (n == "tb_ckpt_bytes") { *value = ctx->tb_ckpt_bytes; return ANYSEQ_OK; }
    if (n == "tb_method") { *value = ctx->tb_method; return ANYSEQ_OK; }
    if (n == "tb_tiles") { *value = ctx->tb_tiles; return ANYSEQ_OK; }
    if (n == "tb_hits") { *value = ctx->tb_hits; return ANYSEQ_OK; }
    if (n == "fill_launches") { *value = (double)ctx->fill_launches; return ANYSEQ_OK; }
    if (n == "h2d_bytes") { *value = (double)ctx->h2d_bytes.load(); return ANYSEQ_OK; }
    if (n == "d2h_bytes") { *value = (double)ctx->d2h_bytes.load(); return ANYSEQ_OK; }
    return fail(ctx, ANYSEQ_E_INVALID, "unknown stat %s", name);
  });
}

anyseq_status anyseq_reset_stats(anyseq_ctx* ctx) {
  if (!ctx) return ANYSEQ_E_INVALID;
  return abi_guard(ctx, [&]() -> anyseq_status {
    resolve_events(ctx);
    ctx->fill_ms = ctx->walk_ms = 0;
    ctx->fill_launches = 0;
    ctx->h2d_bytes = 0;
    ctx->d2h_bytes = 0;
    return ANYSEQ_OK;
  });
}

const char* anyseq_status_str(anyseq_status s) {
  const int i = (int)s;
  return (i >= 0 && i < (int)(sizeof(kStatus) / sizeof(kStatus[0]))) ? kStatus[i] : "unknown status";
}

const char* anyseq_last_error(const anyseq_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

const char* anyseq_version(void) { return "anyseq-b200 0.1 (sm_100a)"; }

}  // extern "C"
