// csrc/walk.cuh -- the traceback walk of one pair over the fill's H store (shared by the
// stand-alone walk kernel and the fill kernel's fused walk).
//
// The predecessor walk re-derives every decision of the
// relax listing from H: DIAG iff H = H(i-1,j-1) + sigma (DIAG first, R7);
// else UP iff H = E(i,j) = max_k H(i-k,j) - Go - k Ge (E before F, R7), the gap being the
// LARGEST maximising k (extension wins ties at every cell, R8); else LEFT likewise along
// the row; local STOP at H <= 0 (R9); global boundary runs (R16).  Linear gaps: k = 1.
#pragma once
#include <climits>
#include "common.cuh"

namespace anyseq {

// H(i, j) of a pair from the traceback H store (fill_kernel.cuh, traceback mode): one
// element per (strip, diagonal d = step - row, row, lane group, lane) of the warp-slot -- a
// diagonal run of the walk steps back G * L elements per cell.  Full store: 32-bit words with both
// alignments of an s16x2 slot in their halves (s16x2 values biased by 2^14).
// Low-byte store (tb8): 16-bit elements holding the low byte of each alignment's H (s16x2)
// or bytes (s32); the walk rebuilds exact values from neighbour differences (see below).
// Row 0 / column 0 are the initial values of P:259-264, always exact.
__device__ __forceinline__ int hbound(const DevParams& P, int i, int j) {
  if (P.kind != KGLOBAL || (i == 0 && j == 0)) return 0;
  return -(P.go + (i + j) * P.ge);
}

__device__ __forceinline__ int hraw(const DevParams& P, const uint32_t* __restrict__ dirs,
                                    const TbInfo& ti, int i, int j, bool tb8) {
  const int L = ti.L, R = ti.R;
  const int ip = i - 1 + ti.pad;
  int st, tt, r;
  // R is one of the traceback variants' row counts: constant divisors
  switch (R) {
    case 19: st = ip / 152; r = ip - st * 152; tt = r / 19; r -= tt * 19; break;
    case 16: st = ip / 128; r = ip - st * 128; tt = r / 16; r -= tt * 16; break;
    default: st = ip / 64; r = ip - st * 64; tt = r / 8; r -= tt * 8; break;  // R = 8
  }
  const int k = (j - 1) + tt;                 // wavefront step of the cell
  const int DK = ti.slot_M + L - 1 + R - 1;   // diagonal index range per strip
  const int G = 32 / L;                        // lane groups per warp (interleaved)
  const int64_t w =
      ti.dir_base + (((((int64_t)st * DK + (k - r + R - 1)) * R + r) * G + ti.grp) * L + tt);
  if (tb8) {
    if (ti.P == 2)
      return (int)((__ldg(reinterpret_cast<const unsigned short*>(dirs) + w) >> (8 * ti.half)) & 0xffu);
    return (int)__ldg(reinterpret_cast<const unsigned char*>(dirs) + w);
  }
  const uint32_t word = dirs[w];
  if (ti.P == 2) {
    const int v = (int)(int16_t)(uint16_t)(ti.half ? (word >> 16) : (word & 0xffffu));
    return v - (1 << 14);  // every kind's s16x2 values carry the +2^14 bias
  }
  return (int)word;
}

// Does cell (i, j) hold the value `want`?  Exact for the full store; for the low-byte store
// exact whenever |H(i,j) - want| < 256 (the host admits tb8 only then).
__device__ __forceinline__ bool hmatch(int raw, int want, bool tb8) {
  return tb8 ? (raw == (want & 0xff)) : (raw == want);
}
// The exact value of cell (i, j) from its stored element and the exact value `ref` of an
// adjacent cell (|difference| < 128 for the low-byte store).
__device__ __forceinline__ int hnear(int raw, int ref, bool tb8) {
  return tb8 ? ref + (int)(int8_t)(uint8_t)(raw - (ref & 0xff)) : raw;
}

struct RunWriter {
  uint32_t* out;
  int n;
  uint32_t op, len;
  __device__ void push(uint32_t o, uint32_t l) {
    if (l == 0) return;
    if (len && o == op) { len += l; return; }
    if (len) out[n++] = (len << 4) | op;
    op = o; len = l;
  }
  __device__ void flush() {
    if (len) out[n++] = (len << 4) | op;
    len = 0;
  }
};

// Walk one pair from its end cell; runs in walk order (reversed) at ops_out, the number of
// runs and the begin cell to the pointers.  qc / sc: 1-based code pointers of the pair.
// The walk keeps the exact H of its current cell (starting from the optimum's score) and
// takes every other value either as a test against an expected value (hmatch) or rebuilt
// from the adjacent cell just visited (hnear): both exact for either store format.
static __device__ __noinline__ void walk_pair(const DevParams& P, const uint32_t* __restrict__ dirs,
                                       const TbInfo& ti, const uint8_t* qc, const uint8_t* sc,
                                       uint32_t* ops_out, int32_t* n_ops, int32_t* beg_i,
                                       int32_t* beg_j, bool tb8) {
  const int go = P.go, ge = P.ge;
  const int kind = P.kind;
  RunWriter rw{ops_out, 0, 0, 0};
  int i = ti.end_i, j = ti.end_j;
  int h = ti.score;
  const bool linear = P.gap == GLINEAR;
  // the exact value of (i2, j2) given the exact value ref of an adjacent cell
  auto hget = [&](int i2, int j2, int ref) -> int {
    if (i2 == 0 || j2 == 0) return hbound(P, i2, j2);
    return hnear(hraw(P, dirs, ti, i2, j2, tb8), ref, tb8);
  };
  // does (i2, j2) hold `want`
  auto hhas = [&](int i2, int j2, int want) -> bool {
    if (i2 == 0 || j2 == 0) return hbound(P, i2, j2) == want;
    return hmatch(hraw(P, dirs, ti, i2, j2, tb8), want, tb8);
  };
  for (;;) {
    if (i == 0 || j == 0) {
      if (kind == KGLOBAL) {  // reading R16: boundary runs
        rw.push(1u, (uint32_t)i);
        rw.push(2u, (uint32_t)j);
        i = 0; j = 0;
      }
      break;
    }
    if (kind == KLOCAL && h <= 0) break;  // STOP (reading R9)
    {  // diagonal runs: the next DW diagonal cells are loaded together (memory-level
       // parallelism for the dependent walk), then verified in order
      constexpr int DW = 8;
      const int lim = min(DW, min(i, j));
      int hv[DW], sg[DW];
      // the 8 query / subject codes of the run: two aligned 8-byte loads each (the code
      // buffers carry 16 bytes of slack), instead of 16 scattered byte loads
      uint64_t vq = 0, vs = 0;
      const bool vec = i > DW && j > DW;
      if (vec) {
        auto load8 = [](const uint8_t* p) -> uint64_t {  // bytes p[0..7], p unaligned
          const uintptr_t a = (uintptr_t)p & ~(uintptr_t)7;
          const uint64_t lo = __ldg((const unsigned long long*)a);
          const uint64_t hi = __ldg((const unsigned long long*)(a + 8));
          const int sh = (int)((uintptr_t)p - a) * 8;
          return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
        };
        vq = load8(qc + i - (DW - 1));  // byte 7 - l = code of row i - l
        vs = load8(sc + j - (DW - 1));
      }
#pragma unroll
      for (int l = 0; l < DW; ++l) {
        if (l < lim) {
          const int i2 = i - 1 - l, j2 = j - 1 - l;
          hv[l] = (i2 == 0 || j2 == 0) ? hbound(P, i2, j2) : hraw(P, dirs, ti, i2, j2, tb8);
          const uint32_t cq = vec ? (uint32_t)(vq >> (8 * (DW - 1 - l))) & 0xffu : qc[i - l];
          const uint32_t cs = vec ? (uint32_t)(vs >> (8 * (DW - 1 - l))) & 0xffu : sc[j - l];
          sg[l] = sigma_of(P, cq, cs);
        }
      }
      int taken = 0;
#pragma unroll
      for (int l = 0; l < DW; ++l) {
        if (l == taken && l < lim && !(kind == KLOCAL && h <= 0)) {
          const int want = h - sg[l];  // DIAG iff H(i-1-l, j-1-l) = H - sigma
          const bool bnd = (i - 1 - l == 0) || (j - 1 - l == 0);
          if (bnd ? hv[l] == want : hmatch(hv[l], want, tb8)) {
            h = want;
            ++taken;
          }
        }
      }
      if (taken) {
        rw.push(0u, (uint32_t)taken);
        i -= taken;
        j -= taken;
        continue;  // re-examine (i, j): boundary, STOP or the next run
      }
    }
    const int sig = sigma_of(P, qc[i], sc[j]);
    if (hhas(i - 1, j - 1, h - sig)) {  // DIAG
      rw.push(0u, 1);
      --i; --j;
      h -= sig;
      continue;
    }
    if (linear) {
      if (hhas(i - 1, j, h + ge)) { rw.push(1u, 1); --i; h += ge; continue; }
      rw.push(2u, 1);  // LEFT: H(i, j-1) = H(i, j) + g
      --j;
      h += ge;
      continue;
    }
    // UP iff E(i,j) = h, E(i,j) = max_k H(i-k,j) - Go - k Ge <= h; the gap is the largest
    // k with H(i-k,j) - Go - k Ge = h.  H(i',j') <= match * min(i',j') bounds the scan
    // (no k with match * min(i-k, j) - Go - k Ge < h can reach h); loads go in batches and
    // values are rebuilt cell by cell up the column.
    int kb = 0, hb = 0;
    {
      constexpr int SB = 8;
      const int mt = max(P.smax, 0);
      int ref = h;  // exact value of (i - k0 + 1, j)
      for (int k0 = 1; k0 <= i; k0 += SB) {
        if (mt * min(i - k0, j) - go - k0 * ge < h) break;
        int hv[SB];
#pragma unroll
        for (int l = 0; l < SB; ++l)
          if (k0 + l <= i) {
            const int i2 = i - k0 - l;
            hv[l] = (i2 == 0) ? hbound(P, 0, j) : hraw(P, dirs, ti, i2, j, tb8);
          }
#pragma unroll
        for (int l = 0; l < SB; ++l)
          if (k0 + l <= i) {
            const int i2 = i - k0 - l;
            ref = (i2 == 0) ? hv[l] : hnear(hv[l], ref, tb8);
            if (ref - go - (k0 + l) * ge == h) { kb = k0 + l; hb = ref; }
          }
      }
    }
    if (kb) {
      rw.push(1u, (uint32_t)kb);
      i -= kb;
      h = hb;
      continue;
    }
    {  // LEFT: F(i,j) = h, the largest such k along the row
      constexpr int SB = 8;
      const int mt = max(P.smax, 0);
      int ref = h;
      for (int k0 = 1; k0 <= j; k0 += SB) {
        if (mt * min(i, j - k0) - go - k0 * ge < h) break;
        int hv[SB];
#pragma unroll
        for (int l = 0; l < SB; ++l)
          if (k0 + l <= j) {
            const int j2 = j - k0 - l;
            hv[l] = (j2 == 0) ? hbound(P, i, 0) : hraw(P, dirs, ti, i, j2, tb8);
          }
#pragma unroll
        for (int l = 0; l < SB; ++l)
          if (k0 + l <= j) {
            const int j2 = j - k0 - l;
            ref = (j2 == 0) ? hv[l] : hnear(hv[l], ref, tb8);
            if (ref - go - (k0 + l) * ge == h) { kb = k0 + l; hb = ref; }
          }
      }
    }
    if (!kb) break;  // unreachable for a consistent H store (no predecessor found)
    rw.push(2u, (uint32_t)kb);
    j -= kb;
    h = hb;
  }
  (void)hget;
  rw.flush();
  *n_ops = rw.n;
  *beg_i = i;
  *beg_j = j;
}

}  // namespace anyseq
