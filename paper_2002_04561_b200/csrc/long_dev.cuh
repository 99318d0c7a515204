// csrc/long_dev.cuh -- device-side shared definitions of the long-pair kernels (the 32-bit
// long_kernel in long.cu and the 16-bit long16_kernel instances in long16_*.cu): task
// arguments, per-warp partial optimum, hand-off loads/stores and bounded waits.
#pragma once
#include <cstdint>
#include <type_traits>
#include "common.cuh"

namespace anyseq {

struct LongPart {
  int32_t lv, li, lj;  // local best (value, i, j)
  int32_t rv, rj;      // semi: best on row n, j in [0, m-1]
  int32_t cv, ci;      // semi: best on column m, i in [0, n]
  int32_t gv, gset;    // global H(n,m)
  int32_t pad_;
};

struct LongArgs {
  DevParams P;
  const uint8_t* qc;
  const uint8_t* sc;
  int32_t n, m;
  int32_t Gtot, g_first, g_count;
  const int32_t* cb;  // [Gtot+1]
  int32_t S;
  int32_t* ticket;
  int32_t* rowprog;   // [Gtot * S]
  int32_t* const* bflag;  // [Gtot+1] per-edge flag arrays of S ints (on the consumer)
  int2* const* bcol;  // [Gtot+1] column buffers: (H(i, cb[g]), F(i, cb[g])), i = 0..n
  int4* rowbuf;       // [m+1]: (H, tag, E, tag) of the last completed row at column j
  LongPart* parts;
  int32_t* abort_flag;
  int32_t chunk;
  int32_t one;
  int32_t lag;
  int32_t keyed;  // local: 32 * (max score) fits in 31 bits -> packed (value, row) tracking
  int32_t sleep_ns;  // long16: back-off of the row hand-off poll
  int32_t hopc;    // long16: packed -(G_o+G_e) for both halves, low-half borrow compensated
  int32_t neg16;   // long16: relative "-inf" (below every real relative value)
  int32_t margin;  // long16: the warp maximum is re-based to -margin
  int32_t bspan;   // long16: bound on |H(x) - H(y)| over one task window (Lipschitz, d * dist)
  int32_t pad_top; // long16 SEMI: pad rows above row 1 (the last strip then ends at row n)
  // CKPT instances (linear-space traceback): checkpoint rows and columns (absolute values)
  int2* rowck;      // [((S-1) / ck_every) x (m+1)]: (H, E) of row strip k*ck_every-1's last row
  int2* colck;      // [((m-1) >> kc_shift) x (n+1)]: (H, F) at column (k+1) << kc_shift
  int32_t ck_every, kc_shift;
  unsigned long long* prof;  // optional: [0] cycles waiting, [1] cycles in tasks, [2] tasks
  long long spin_limit;
  int32_t stall_task;  // fault injection: this task is skipped (-1: none)
  // long16 MULTI instances (several pairs in one launch): per-pair arguments (device array),
  // ticket segments (pair, column pass) and the inclusive prefix of their task counts
  const LongArgs* pairs;
  const int2* segs;
  const int32_t* task_end;
  int32_t task_total;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Row hand-off words: (value, tag) pairs in one 8-byte access each, so a reader that sees
// the tag of the strip it waits for also sees the value (single-copy atomicity of aligned
// 8-byte accesses) -- no fences, no progress counters (the LL idea of NCCL's protocols).
__device__ __forceinline__ void st_row(int4* p, int h, int e, int tag) {
  asm volatile("st.relaxed.gpu.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(h), "r"(tag),
               "r"(e), "r"(tag)
               : "memory");
}
__device__ __forceinline__ int4 ld_row(const int4* p) {
  int4 v;
  asm volatile("ld.relaxed.gpu.global.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// 16-byte global -> shared copy that bypasses L1 (cp.async.cg), committed as a group
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ bool lkey_better(int v, int i, int j, int bv, int bi, int bj) {
  return v > bv || (v == bv && (j < bj || (j == bj && i < bi)));
}

__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_sys(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// lane 0 polls *p >= need with relaxed loads (no L1 invalidation per poll) and closes with
// one acquire fence; returns false on timeout/abort (warp-uniform).
template <bool SYS>
__device__ __forceinline__ bool warp_wait(const int* p, int need, const LongArgs& a) {
  int ok = 1;
  if ((threadIdx.x & 31) == 0) {
    const long long t0 = a.prof ? clock64() : 0;
    long long spins = 0;
    // relaxed polls, then one acquire load once the value is there (no full fence)
    while (true) {
      if ((SYS ? ld_relaxed_sys(p) : ld_relaxed_gpu(p)) >= need &&
          (SYS ? ld_acquire_sys(p) : ld_acquire_gpu(p)) >= need)
        break;
      if ((++spins & 255) == 0 && (spins > a.spin_limit || *(volatile int*)a.abort_flag)) {
        atomicExch(a.abort_flag, 1);
        ok = 0;
        break;
      }
      __nanosleep(32);
    }
    if (a.prof) atomicAdd(&a.prof[4], (unsigned long long)(clock64() - t0));  // [4]: flags
  }
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

__device__ __forceinline__ int imad_add_s(int x, uint32_t one, int k) {
  int d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(one), "r"(k));
  return d;
}

typedef void (*LongFn)(LongArgs);
// long16_*.cu: the 16-bit differential kernel instance for (rows per lane, kind, checkpoints)
LongFn long16_fn(int nr, int kind, bool ckpt);
LongFn long16_multi_fn(int kind, int nr, bool ckpt = false);  // MULTI instances (nr 8 or 16)

}  // namespace anyseq
