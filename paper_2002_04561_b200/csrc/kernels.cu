// csrc/kernels.cu -- pack (a1), plan (a2), traceback walk (a5), output assembly.
//
//  * pack: "Sequence" accessor storage of the paper as byte codes on the device;
//    validation of the alphabet (reading R12).
//  * classify/slots: per-pair variant choice (register width by the 16-bit range guard,
//    the paper's narrow differential-score argument P:498 applied to absolute scores --
//    reading R11), sort by (variant, m, n) so that pairs sharing a warp have similar shape.
//  * walk: the predecessor walk of the traceback.
#include <climits>
#include <cub/cub.cuh>
#include "kernels.h"
#include "walk.cuh"
#include "../../include/anyseq.h"

namespace anyseq {

static inline int grid_for(int64_t work, int threads, int num_sms, int per_sm = 8) {
  int64_t g = (work + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// ------------------------------------------------------------------------------- pack
__device__ __forceinline__ uint32_t code_of(uint32_t c) {
  const uint32_t x = c | 0x20u;  // lower case
  return x == 'a' ? 0u : x == 'c' ? 1u : x == 'g' ? 2u : x == 't' ? 3u : x == 'n' ? 4u : 0xFFu;
}

__device__ int64_t find_pair(const uint64_t* off, uint64_t num_pairs, uint64_t pos) {
  // largest k with off[k] <= pos
  int64_t lo = 0, hi = (int64_t)num_pairs;  // off[hi] > pos for pos < off[num]
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= pos) lo = mid; else hi = mid;
  }
  return lo;
}

struct PackSeg {
  const uint8_t* in;
  uint64_t len;
  uint8_t* out;
  uint64_t pos_base;
  const uint64_t* off;
};

// One launch packs both sequence sets: units [0, u0) are q's 16-byte units, [u0, u0+u1) s's.
__global__ void __launch_bounds__(256) pack_kernel(PackSeg q, PackSeg s, uint64_t num_pairs,
                                                   uint32_t* flags, PlanSummary* sum) {
  __shared__ uint8_t lut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = (uint8_t)code_of((uint32_t)i);
  __syncthreads();
  const uint64_t u0 = (q.len + 15) / 16, units = u0 + (s.len + 15) / 16;
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const bool isq = u < u0;
    const PackSeg& g = isq ? q : s;
    const uint64_t b = (isq ? u : u - u0) * 16, len = g.len;
    const uint8_t* in = g.in;
    uint8_t* out = g.out;
    const bool vec = (b + 16 <= len) && ((((uintptr_t)(in + b)) & 15) == 0) &&
                     ((((uintptr_t)(out + b)) & 15) == 0);
    uint32_t w[4] = {0, 0, 0, 0};
    int cnt = 16;
    if (vec) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(in + b));  // streamed once
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
      cnt = (int)((len - b) < 16 ? (len - b) : 16);
      for (int k = 0; k < cnt; ++k) w[k >> 2] |= (uint32_t)in[b + k] << (8 * (k & 3));
    }
    uint32_t o[4];
    uint32_t bad = 0, nn = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      uint32_t r = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t x = lut[(w[t] >> (8 * k)) & 0xffu];
        r |= x << (8 * k);
        const bool in_range = (t * 4 + k) < cnt;
        bad |= (in_range && x == 0xFFu) ? (1u << (t * 4 + k)) : 0u;
        nn |= (in_range && x == 4u) ? 1u : 0u;
      }
      o[t] = r;
    }
    if (vec) {
      *reinterpret_cast<uint4*>(out + b) = make_uint4(o[0], o[1], o[2], o[3]);
    } else {
      for (int k = 0; k < cnt; ++k) out[b + k] = (uint8_t)(o[k >> 2] >> (8 * (k & 3)));
    }
    if (bad) atomicMin(&sum->err_pos, (unsigned long long)(g.pos_base + b + __ffs(bad) - 1));
    if (nn) {  // rare: mark every pair that owns an N in this unit
      for (int k = 0; k < cnt; ++k)
        if (((o[k >> 2] >> (8 * (k & 3))) & 0xffu) == 4u)
          atomicOr(&flags[find_pair(g.off, num_pairs, b + k)], 1u);
    }
  }
}

cudaError_t launch_pack(const char* d_q, uint64_t q_len, uint8_t* d_qcode, const uint64_t* d_qoff,
                        const char* d_s, uint64_t s_len, uint8_t* d_scode, const uint64_t* d_soff,
                        uint64_t num_pairs, uint32_t* d_flags, PlanSummary* d_sum,
                        cudaStream_t st, int num_sms) {
  const uint64_t units = (q_len + 15) / 16 + (s_len + 15) / 16;
  if (units == 0) return cudaSuccess;
  PackSeg q{(const uint8_t*)d_q, q_len, d_qcode, 0, d_qoff};
  PackSeg s{(const uint8_t*)d_s, s_len, d_scode, 1ull << 62, d_soff};
  pack_kernel<<<grid_for((int64_t)units, 256, num_sms, 16), 256, 0, st>>>(q, s, num_pairs, d_flags,
                                                                           d_sum);
  return cudaGetLastError();
}

// One thread per 16 bases: a 32-bit word of 2-bit codes -> 16 byte codes (one 16-byte store).
__global__ void __launch_bounds__(256) unpack2_kernel(const uint8_t* __restrict__ q2, uint64_t qn,
                                                      uint8_t* __restrict__ qc,
                                                      const uint8_t* __restrict__ s2, uint64_t sn,
                                                      uint8_t* __restrict__ sc) {
  const uint64_t u0 = (qn + 15) / 16, units = u0 + (sn + 15) / 16;
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const bool isq = u < u0;
    const uint64_t b = (isq ? u : u - u0) * 16, len = isq ? qn : sn;
    const uint8_t* in = isq ? q2 : s2;
    uint8_t* out = isq ? qc : sc;
    // the packed buffers are padded to a 4-byte multiple by the host API
    const uint32_t w = __ldcs(reinterpret_cast<const uint32_t*>(in + b / 4));
    uint32_t o[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t x = w >> (8 * t);  // bases 4t .. 4t+3
      o[t] = (x & 3u) | ((x << 6) & 0x300u) | ((x << 12) & 0x30000u) | ((x << 18) & 0x3000000u);
    }
    if (b + 16 <= len) {
      *reinterpret_cast<uint4*>(out + b) = make_uint4(o[0], o[1], o[2], o[3]);
    } else {
      for (uint64_t k = 0; b + k < len; ++k) out[b + k] = (uint8_t)(o[k >> 2] >> (8 * (k & 3)));
    }
  }
}

cudaError_t launch_unpack2(const uint8_t* d_q2, uint64_t q_len, uint8_t* d_qcode,
                           const uint8_t* d_s2, uint64_t s_len, uint8_t* d_scode,
                           cudaStream_t st, int num_sms) {
  const uint64_t units = (q_len + 15) / 16 + (s_len + 15) / 16;
  if (units == 0) return cudaSuccess;
  unpack2_kernel<<<grid_for((int64_t)units, 256, num_sms, 16), 256, 0, st>>>(d_q2, q_len, d_qcode,
                                                                             d_s2, s_len, d_scode);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------ prep / publish
__global__ void prep_kernel(uint32_t* flags, uint64_t n, PlanSummary* sum, uint64_t* qoff,
                            uint64_t* soff, uint64_t q0, uint64_t s0, int64_t gq, int64_t gs,
                            int32_t* tickets) {
  if (blockIdx.x == 0 && threadIdx.x < kNumTickets) tickets[threadIdx.x] = 0;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    flags[k] = 0;
    if (qoff && gq >= 0) {  // host-API uniform chunk: offsets were not uploaded
      qoff[k] = k * (uint64_t)gq;
      soff[k] = k * (uint64_t)gs;
    } else if (qoff) {  // host-API chunk: offsets were uploaded verbatim
      qoff[k] -= q0;
      soff[k] -= s0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < NV) {
    const int v = threadIdx.x;
    sum->count[v] = 0;
    sum->maxn[v] = 0;
    sum->maxm[v] = 0;
    sum->kmin[v] = ~0ull;
    sum->kmax[v] = 0ull;
    if (v == 0) {
      sum->err_pos = ~0ull;
      sum->range_err = 0;
      sum->blocks_done = 0;
    }
  }
}

cudaError_t launch_prep(uint32_t* flags, uint64_t n, PlanSummary* sum, uint64_t* qoff,
                        uint64_t* soff, uint64_t q0, uint64_t s0, int64_t gq, int64_t gs,
                        int32_t* tickets, cudaStream_t st, int num_sms) {
  prep_kernel<<<grid_for((int64_t)n, 256, num_sms), 256, 0, st>>>(flags, n, sum, qoff, soff, q0,
                                                                  s0, gq, gs, tickets);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------- classify
__global__ void classify_kernel(ClassifyArgs a) {
  // per-block plan summary (warp-aggregated, then one set of global atomics per block:
  // the naive per-pair global atomics serialise on a handful of addresses)
  __shared__ int s_cnt[NV], s_maxn[NV], s_maxm[NV];
  __shared__ unsigned long long s_kmin[NV], s_kmax[NV];
  if (threadIdx.x < NV) {
    s_cnt[threadIdx.x] = 0;
    s_maxn[threadIdx.x] = 0;
    s_maxm[threadIdx.x] = 0;
    s_kmin[threadIdx.x] = ~0ull;
    s_kmax[threadIdx.x] = 0ull;
  }
  __syncthreads();
  const DevParams& P = a.P;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < a.num_pairs; base += stride) {
    const uint64_t k = base + threadIdx.x;
    int v = -1;
    int64_t n = 0, m = 0;
    unsigned long long key = 0;
    if (k < a.num_pairs) {
      n = (int64_t)(a.q_off[k + 1] - a.q_off[k]);
      m = (int64_t)(a.s_off[k + 1] - a.s_off[k]);
      if (n == 0 || m == 0) {
        // empty sequences (SURVEY 8(b) "Empty sequences"): global = one gap run, else 0
        int32_t sc = 0, ei = 0, ej = 0;
        if (P.kind == KGLOBAL) {
          const int64_t len = n + m;
          sc = len ? (int32_t)(-(P.go + len * P.ge)) : 0;
          ei = (int32_t)n; ej = (int32_t)m;
          if (a.ops && len) {
            const uint64_t obase = a.q_off[k] + a.s_off[k] + k;
            a.ops[obase] = ((uint32_t)len << 4) | (n ? 1u : 2u);
            a.n_ops[k] = 1;
          } else if (a.ops) {
            a.n_ops[k] = 0;
          }
        } else if (a.ops) {
          a.n_ops[k] = 0;
        }
        a.scores[k] = sc;
        if (a.end_i) { a.end_i[k] = ei; a.end_j[k] = ej; }
        if (a.beg_i) { a.beg_i[k] = 0; a.beg_j[k] = 0; }
        a.keys[k] = ~0ull;
        a.vals[k] = (int32_t)k;
      } else if (a.skip_cells > 0 && n >= a.skip_min && m >= a.skip_min && n * m >= a.skip_cells) {
        a.keys[k] = ~0ull;  // left to the long-pair path
        a.vals[k] = (int32_t)k;
      } else {
        const PairPlan pp = plan_pair(a.cfg, n, m, (a.flags[k] & 1u) != 0);
        v = pp.v;
        if (pp.range_err) atomicExch(&a.sum->range_err, 1);
        // speculative slots for the uniform case (every pair in one variant, identity
        // order); the host re-forms slots from the sorted order otherwise
        if (variant_desc(v).pairs == 2) {
          if (!(k & 1)) {
            Slot sl;
            sl.pair[0] = (int32_t)k;
            sl.pair[1] = k + 1 < a.num_pairs ? (int32_t)(k + 1) : -1;
            a.slots[k >> 1] = sl;
          }
        } else {
          Slot sl;
          sl.pair[0] = (int32_t)k;
          sl.pair[1] = -1;
          a.slots[k] = sl;
        }
        key = pp.key;
        a.keys[k] = key;
        a.vals[k] = (int32_t)k;
      }
    }
    const unsigned grp = __match_any_sync(0xffffffffu, v);
    if (v >= 0) {
      const int mxn = __reduce_max_sync(grp, (int)n);
      const int mxm = __reduce_max_sync(grp, (int)m);
      if ((threadIdx.x & 31) == __ffs(grp) - 1) {
        atomicAdd(&s_cnt[v], __popc(grp));
        atomicMax(&s_maxn[v], mxn);
        atomicMax(&s_maxm[v], mxm);
      }
      atomicMin(&s_kmin[v], key);
      atomicMax(&s_kmax[v], key);
    }
  }
  __syncthreads();
  if (threadIdx.x < NV && s_cnt[threadIdx.x] > 0) {
    const int v = threadIdx.x;
    atomicAdd(&a.sum->count[v], s_cnt[v]);
    atomicMax(&a.sum->maxn[v], s_maxn[v]);
    atomicMax(&a.sum->maxm[v], s_maxm[v]);
    atomicMin(&a.sum->kmin[v], s_kmin[v]);
    atomicMax(&a.sum->kmax[v], s_kmax[v]);
  }
  // the last block to finish publishes the summary into host-mapped memory (no copy-engine
  // transfer: the host API's uploads keep the copy engine and the PCIe link busy)
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&a.sum->blocks_done, 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    static_assert(sizeof(PlanSummary) % 8 == 0, "summary is copied in 8-byte words");
    const volatile uint64_t* src = reinterpret_cast<const volatile uint64_t*>(a.sum);
    volatile uint64_t* dst = reinterpret_cast<volatile uint64_t*>(a.host_sum);
    for (int i = threadIdx.x; i < (int)(sizeof(PlanSummary) / 8); i += blockDim.x) dst[i] = src[i];
  }
}

cudaError_t launch_classify(const ClassifyArgs& a, cudaStream_t st, int num_sms) {
  const int threads = 256;
  classify_kernel<<<grid_for((int64_t)a.num_pairs, threads, num_sms), threads, 0, st>>>(a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------ slots
struct SlotTables {
  int32_t voff[NV + 1];
  int32_t count[NV];
  int32_t sbase[NV];
  int32_t pairs[NV];
};

__global__ void slots_kernel(const int32_t* __restrict__ order, int64_t num, SlotTables T,
                             Slot* __restrict__ slots) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < num;
       p += (int64_t)gridDim.x * blockDim.x) {
    int v = -1;
#pragma unroll
    for (int c = 0; c < NV; ++c)
      if (p >= T.voff[c] && p < T.voff[c] + T.count[c]) v = c;
    if (v < 0) continue;
    const int64_t local = p - T.voff[v];
    if (T.pairs[v] == 2) {
      if (local & 1) continue;
      Slot s;
      s.pair[0] = order[p];
      s.pair[1] = (local + 1 < T.count[v]) ? order[p + 1] : -1;
      slots[T.sbase[v] + local / 2] = s;
    } else {
      Slot s;
      s.pair[0] = order[p];
      s.pair[1] = -1;
      slots[T.sbase[v] + local] = s;
    }
  }
}

cudaError_t launch_slots(const int32_t* d_order, int64_t num, const int32_t* voff_host,
                         const int32_t* count_host, const int32_t* sbase_host, Slot* d_slots,
                         cudaStream_t st, int num_sms) {
  if (num == 0) return cudaSuccess;
  SlotTables T;
  for (int c = 0; c < NV; ++c) {
    T.voff[c] = voff_host[c];
    T.count[c] = count_host[c];
    T.sbase[c] = sbase_host[c];
    T.pairs[c] = variant_desc(c).pairs;
  }
  T.voff[NV] = voff_host[NV];
  slots_kernel<<<grid_for(num, 256, num_sms), 256, 0, st>>>(d_order, num, T, d_slots);
  return cudaGetLastError();
}

cudaError_t sort_pairs(void* d_temp, size_t& temp_bytes, const unsigned long long* keys_in,
                       unsigned long long* keys_out, const int32_t* vals_in, int32_t* vals_out,
                       int64_t num, cudaStream_t st) {
  return cub::DeviceRadixSort::SortPairs(d_temp, temp_bytes, keys_in, keys_out, vals_in,
                                         vals_out, (int)num, 0, 64, st);
}

struct I32ToU64 {
  __host__ __device__ uint64_t operator()(int32_t x) const { return (uint64_t)(x < 0 ? 0 : x); }
};

cudaError_t exclusive_scan_i32_to_u64(void* d_temp, size_t& temp_bytes, const int32_t* in,
                                      uint64_t* out, int64_t num, cudaStream_t st) {
  cub::TransformInputIterator<uint64_t, I32ToU64, const int32_t*> it(in, I32ToU64());
  return cub::DeviceScan::ExclusiveSum(d_temp, temp_bytes, it, out, (int)num, st);
}

// ------------------------------------------------------------------------------- walk
__global__ void walk_kernel(WalkArgs a) {
  const int64_t total = (int64_t)(a.slot_hi - a.slot_lo) * a.pairs_per_slot;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int slot = a.slot_lo + (int)(w / a.pairs_per_slot);
    const int half = (int)(w % a.pairs_per_slot);
    const int pair = a.slots[slot].pair[half];
    if (pair < 0) continue;
    const TbInfo ti = a.tb[pair];
    const uint64_t base = a.q_off[pair] + a.s_off[pair] + (uint64_t)pair;
    const uint8_t* qc = a.qcode + a.q_off[pair] - 1;
    const uint8_t* sc = a.scode + a.s_off[pair] - 1;
    switch (ti.R) {  // the traceback variants' rows per lane (plan.cuh)
      case 8:
        walk_pair<8>(a.P, a.dirs, ti, qc, sc, a.ops + base, a.n_ops + pair, a.beg_i + pair,
                     a.beg_j + pair, a.end_i + pair, a.tb8 != 0);
        break;
      case 16:
        walk_pair<16>(a.P, a.dirs, ti, qc, sc, a.ops + base, a.n_ops + pair, a.beg_i + pair,
                      a.beg_j + pair, a.end_i + pair, a.tb8 != 0);
        break;
      default:
        walk_pair<19>(a.P, a.dirs, ti, qc, sc, a.ops + base, a.n_ops + pair, a.beg_i + pair,
                      a.beg_j + pair, a.end_i + pair, a.tb8 != 0);
        break;
    }
  }
}

cudaError_t launch_walk(const WalkArgs& a, cudaStream_t st, int num_sms) {
  const int64_t total = (int64_t)(a.slot_hi - a.slot_lo) * a.pairs_per_slot;
  if (total <= 0) return cudaSuccess;
  walk_kernel<<<grid_for(total, 128, num_sms, 16), 128, 0, st>>>(a);
  return cudaGetLastError();
}

// --------------------------------------------------------------------------- finalize
__global__ void finalize_kernel(FinalizeArgs a) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < a.num_pairs;
       k += (uint64_t)gridDim.x * blockDim.x) {
    anyseq_alignment o;
    o.score = a.scores[k];
    o.reserved = 0;
    o.q_end = a.end_i ? a.end_i[k] : 0;
    o.s_end = a.end_j ? a.end_j[k] : 0;
    o.q_begin = a.beg_i ? a.beg_i[k] : o.q_end;
    o.s_begin = a.beg_j ? a.beg_j[k] : o.s_end;
    o.cigar_offset = 0;
    o.cigar_len = 0;
    o.reserved2 = 0;
    if (a.n_ops) {
      const int nops = a.n_ops[k];
      const uint64_t off = a.cig_off[k];
      o.cigar_offset = a.cig_base + off;
      o.cigar_len = (uint32_t)nops;
      if (a.cigar && off + nops <= a.cigar_cap) {
        const uint32_t* src = a.ops + a.q_off[k] + a.s_off[k] + k;
        for (int r = 0; r < nops; ++r) a.cigar[off + r] = src[nops - 1 - r];  // reverse runs
      }
    }
    reinterpret_cast<anyseq_alignment*>(a.out_aln)[k] = o;
  }
}

cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st, int num_sms) {
  if (a.num_pairs == 0) return cudaSuccess;
  finalize_kernel<<<grid_for((int64_t)a.num_pairs, 256, num_sms), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace anyseq
