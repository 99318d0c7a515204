// csrc/common.cuh -- shared device definitions of the CUDA path (NOT shared with oracle/).
//
// Score arithmetic follows PAPER.md Eqs. (1)-(5) with the per-kind
// initialisation and optimum of P:257-264.  Two register widths:
//   VS32  : one alignment per 32-bit register (int32, -inf = -2^30)
//   VS16  : two alignments per 32-bit register (s16x2 DPX lanes, -inf = -2^14), used only
//           when the range guard of DESIGN.md (reading R11) proves no 16-bit overflow.
// This mirrors the paper's own narrow-score idea for SIMD lanes on
// Blackwell's DPX instructions (VIADDMNMX / VIMNMX .S16x2).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Debug builds (-DANYSEQ_CHECKS, tools/checks_build.sh): device-side bounds checks on the
// index computations of the long-pair kernels and the traceback walk; a failed check traps
// the kernel (the call then reports ANYSEQ_E_CUDA).  compute-sanitizer is not available on
// the GPU pool, so this is the memory-safety run of the test workload.
#ifdef ANYSEQ_CHECKS
#define ANY_CHECK(c) do { if (!(c)) __trap(); } while (0)
#else
#define ANY_CHECK(c) do { } while (0)
#endif

namespace anyseq {

enum Kind : int { KGLOBAL = 0, KLOCAL = 1, KSEMI = 2 };
enum Gap : int { GLINEAR = 0, GAFFINE = 1 };

constexpr int32_t NEG32 = -(1 << 30);
constexpr int32_t NEG16 = -(1 << 14);
constexpr uint8_t CODE_N = 4;
constexpr uint8_t CODE_BAD = 0xFF;

// Run-time scheme, already validated on the host.
struct DevParams {
  int32_t kind, gap;
  int32_t match, mismatch;
  int32_t go;       // effective gap open (0 for linear)
  int32_t ge;       // gap extend (linear: g)
  int32_t smax;     // max sigma (range guards, walk bounds)
  uint32_t prof[5]; // query profile of code c: bytes sigma(c, A..T) (simple or matrix scoring)
  uint32_t pn[5];   // byte 0: sigma(c, N) (the s32 profile's fifth byte)
};

// ---------------------------------------------------------------------------------------
// byte permute with sign replication (PRMT default mode).  __byte_perm masks the selector
// with 0x7777 and drops the sign-replicate bit, so use PTX directly.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// profile word of a query symbol c: byte k = sigma(c, k) for subject codes k = 0..3
// (simple_subst_scoring).  N (code 4) mismatches everything (reading R12).
// (P should refer to the kernel parameter itself: the index then becomes one constant-bank
// load with a register offset instead of a local-memory copy of DevParams)
__device__ __forceinline__ uint32_t prof4(const DevParams& P, uint32_t c) {
  return P.prof[c < 4 ? c : 4];
}
__device__ __forceinline__ uint32_t pn_of(const DevParams& P, uint32_t c) {
  return P.pn[c < 4 ? c : 4];
}
// sigma(a, b) for codes 0..4 (traceback walk)
__device__ __forceinline__ int sigma_of(const DevParams& P, uint32_t a, uint32_t b) {
  const uint32_t aa = a < 4 ? a : 4;
  return b < 4 ? (int)(int8_t)(prof4(P, aa) >> (8 * b)) : (int)(int8_t)pn_of(P, aa);
}

// ---------------------------------------------------------------------------------------
// Register-width traits.
struct VS32 {
  static constexpr int P = 1;
  typedef int32_t T;
  static __device__ __forceinline__ T addmax(T a, T b, T c) { return __viaddmax_s32(a, b, c); }
  static __device__ __forceinline__ T addmax_relu(T a, T b, T c) {
    return __viaddmax_s32_relu(a, b, c);
  }
  static __device__ __forceinline__ T vmax(T a, T b) { return max(a, b); }
  static __device__ __forceinline__ T vmax3(T a, T b, T c) { return __vimax3_s32(a, b, c); }
  static __device__ __forceinline__ T vmax_relu(T a, T b) { return __vimax_s32_relu(a, b); }
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
  static __device__ __forceinline__ T splat(int32_t v) { return v; }
  static __device__ __forceinline__ T make(int32_t a, int32_t) { return a; }
  static __device__ __forceinline__ int32_t get(T x, int) { return x; }
  static __device__ __forceinline__ T neg() { return NEG32; }
  // max with predicate bits: bit h set iff a >= b in half h (a wins ties)
  static __device__ __forceinline__ T bmax(T a, T b, uint32_t& p) {
    bool q;
    T r = __vibmax_s32(a, b, &q);
    p = q ? 1u : 0u;
    return r;
  }
  static __device__ __forceinline__ T sigma(uint32_t p0, uint32_t p1, uint32_t sel) {
    return (T)prmt(p0, p1, sel);
  }
  // selector: sign-extend byte c (c in 0..4: byte 4 lives in p1)
  static __device__ __forceinline__ uint32_t selector(uint32_t c0, uint32_t) {
    return c0 * 0x1111u + 0x8880u;
  }
  static __device__ __forceinline__ T shfl_up(T v, int width) {
    return __shfl_up_sync(0xffffffffu, v, 1, width);
  }
  static __device__ __forceinline__ T shfl(T v, int src, int width) {
    return __shfl_sync(0xffffffffu, v, src, width);
  }
  // keep lanes whose mask bit (per half) is set, others -> v
  static __device__ __forceinline__ T select_mask(T x, uint32_t keep, T other) {
    return (keep & 1u) ? x : other;
  }
};

struct VS16 {
  static constexpr int P = 2;
  typedef uint32_t T;
  static __device__ __forceinline__ T addmax(T a, T b, T c) { return __viaddmax_s16x2(a, b, c); }
  static __device__ __forceinline__ T addmax_relu(T a, T b, T c) {
    return __viaddmax_s16x2_relu(a, b, c);
  }
  static __device__ __forceinline__ T vmax(T a, T b) { return __vmaxs2(a, b); }
  static __device__ __forceinline__ T vmax3(T a, T b, T c) { return __vimax3_s16x2(a, b, c); }
  static __device__ __forceinline__ T vmax_relu(T a, T b) { return __vimax_s16x2_relu(a, b); }
  static __device__ __forceinline__ T add(T a, T b) { return __vadd2(a, b); }
  static __device__ __forceinline__ T splat(int32_t v) { return (uint32_t)(v & 0xffff) * 0x10001u; }
  static __device__ __forceinline__ T make(int32_t a, int32_t b) {
    return (uint32_t)(a & 0xffff) | ((uint32_t)(b & 0xffff) << 16);
  }
  static __device__ __forceinline__ int32_t get(T x, int h) {
    return (int32_t)(int16_t)(uint16_t)(h ? (x >> 16) : (x & 0xffff));
  }
  static __device__ __forceinline__ T neg() { return splat(NEG16); }
  // NOTE: the CUDA 12.9 header __vibmax_s16x2 lets its output alias input `a` and then
  // compares the max with itself (predicates always true); this version keeps the max in a
  // private register until both predicates are formed.
  static __device__ __forceinline__ T bmax(T a, T b, uint32_t& p) {
    T r;
    uint32_t plo, phi;
    asm("{.reg .pred p, q;\n\t"
        ".reg .s16 a0, a1, m0, m1;\n\t"
        ".reg .b32 t;\n\t"
        "max.s16x2 t, %3, %4;\n\t"
        "mov.b32 {a0, a1}, %3;\n\t"
        "mov.b32 {m0, m1}, t;\n\t"
        "setp.eq.s16 p, m0, a0;\n\t"
        "setp.eq.s16 q, m1, a1;\n\t"
        "selp.b32 %1, 1, 0, p;\n\t"
        "selp.b32 %2, 2, 0, q;\n\t"
        "mov.b32 %0, t;}"
        : "=r"(r), "=r"(plo), "=r"(phi)
        : "r"(a), "r"(b));
    p = plo | phi;
    return r;
  }
  static __device__ __forceinline__ T sigma(uint32_t p0, uint32_t p1, uint32_t sel) {
    return prmt(p0, p1, sel);
  }
  // half 0 <- sign-extended byte cA of p0; half 1 <- sign-extended byte cB of p1
  static __device__ __forceinline__ uint32_t selector(uint32_t cA, uint32_t cB) {
    return cA * 0x11u + cB * 0x1100u + 0xC480u;
  }
  static __device__ __forceinline__ T shfl_up(T v, int width) {
    return __shfl_up_sync(0xffffffffu, v, 1, width);
  }
  static __device__ __forceinline__ T shfl(T v, int src, int width) {
    return __shfl_sync(0xffffffffu, v, src, width);
  }
  static __device__ __forceinline__ T select_mask(T x, uint32_t keep, T other) {
    uint32_t m = ((keep & 1u) ? 0xffffu : 0u) | ((keep & 2u) ? 0xffff0000u : 0u);
    return (x & m) | (other & ~m);
  }
};

// ---------------------------------------------------------------------------------------
// Device-side plan structures.
struct Slot {
  int32_t pair[2];  // pair indices; pair[1] = -1 for s32 slots or an odd tail
};

// Per-pair traceback bookkeeping written by the fill kernel, read by the walk kernel.
struct TbInfo {
  int64_t dir_base;  // element offset of the pair's warp-slot block in the H store
  int32_t slot_M;    // columns of the warp-slot (max m over the warp's slots)
  int32_t ns;        // strips
  int16_t half, L, R, P;
  int32_t pad;       // top padding rows of this pair (0 for global)
  int32_t score;
  int32_t end_i, end_j;
  int32_t grp;       // lane group of the slot within its warp (interleaved store)
  int32_t end_span;  // > 0: end_i is the first row of the fill lane holding the optimum; the
                     // end row is the first of rows end_i .. end_i + end_span - 1 whose H at
                     // column end_j equals the score (resolved by the walk)
};

}  // namespace anyseq
