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
// 32-bit word per (strip, diagonal d = step - row, row, lane) of the slot -- a diagonal
// run of the walk reads consecutive 32-byte sectors -- both alignments of an s16x2 slot
// in its halves (global/semi s16x2 values biased by 2^14); row 0 / column 0 are the
// initial values of P:259-264.
__device__ __forceinline__ int hval(const DevParams& P, const uint32_t* __restrict__ dirs,
                                    const TbInfo& ti, int i, int j) {
  if (i == 0 || j == 0) {
    if (P.kind != KGLOBAL || (i == 0 && j == 0)) return 0;
    return -(P.go + (i + j) * P.ge);
  }
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
  const int64_t w =
      ti.dir_base + ((((int64_t)st * DK + (k - r + R - 1)) * R + r) * L + tt);
  const uint32_t word = dirs[w];
  if (ti.P == 2) {
    const int v = (int)(int16_t)(uint16_t)(ti.half ? (word >> 16) : (word & 0xffffu));
    return P.kind == KLOCAL ? v : v - (1 << 14);
  }
  return (int)word;
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
static __device__ __noinline__ void walk_pair(const DevParams& P, const uint32_t* __restrict__ dirs,
                                       const TbInfo& ti, const uint8_t* qc, const uint8_t* sc,
                                       uint32_t* ops_out, int32_t* n_ops, int32_t* beg_i,
                                       int32_t* beg_j) {
  const int go = P.go, ge = P.ge;
  const int kind = P.kind;
  RunWriter rw{ops_out, 0, 0, 0};
  int i = ti.end_i, j = ti.end_j;
  int h = hval(P, dirs, ti, i, j);
  const bool linear = P.gap == GLINEAR;
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
          hv[l] = hval(P, dirs, ti, i - 1 - l, j - 1 - l);
          const uint32_t cq = vec ? (uint32_t)(vq >> (8 * (DW - 1 - l))) & 0xffu : qc[i - l];
          const uint32_t cs = vec ? (uint32_t)(vs >> (8 * (DW - 1 - l))) & 0xffu : sc[j - l];
          sg[l] = sigma_of(P, cq, cs);
        }
      }
      int taken = 0;
#pragma unroll
      for (int l = 0; l < DW; ++l) {
        if (l == taken && l < lim && !(kind == KLOCAL && h <= 0) && h == hv[l] + sg[l]) {
          h = hv[l];
          ++taken;
        }
      }
      if (taken) {
        rw.push(0u, (uint32_t)taken);
        i -= taken;
        j -= taken;
        continue;  // re-examine (i, j): boundary, STOP or the next run
      }
    }
    const int hd = hval(P, dirs, ti, i - 1, j - 1);
    const int sig = sigma_of(P, qc[i], sc[j]);
    if (h == hd + sig) {  // DIAG
      rw.push(0u, 1);
      --i; --j;
      h = hd;
      continue;
    }
    if (linear) {
      const int hu = hval(P, dirs, ti, i - 1, j);
      if (h == hu - ge) { rw.push(1u, 1); --i; h = hu; continue; }
      rw.push(2u, 1);
      --j;
      h = hval(P, dirs, ti, i, j);
      continue;
    }
    // UP iff E(i,j) = h, E(i,j) = max_k H(i-k,j) - Go - k Ge <= h; the gap is the largest
    // k with H(i-k,j) - Go - k Ge = h.  H(i',j') <= match * min(i',j') bounds the scan
    // (no k with match * min(i-k, j) - Go - k Ge < h can reach h); loads go in batches.
    int kb = 0, hb = 0;
    {
      constexpr int SB = 8;
      const int mt = max(P.smax, 0);
      for (int k0 = 1; k0 <= i; k0 += SB) {
        if (mt * min(i - k0, j) - go - k0 * ge < h) break;
        int hv[SB];
#pragma unroll
        for (int l = 0; l < SB; ++l)
          if (k0 + l <= i) hv[l] = hval(P, dirs, ti, i - k0 - l, j);
#pragma unroll
        for (int l = 0; l < SB; ++l)
          if (k0 + l <= i && hv[l] - go - (k0 + l) * ge == h) { kb = k0 + l; hb = hv[l]; }
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
      for (int k0 = 1; k0 <= j; k0 += SB) {
        if (mt * min(i, j - k0) - go - k0 * ge < h) break;
        int hv[SB];
#pragma unroll
        for (int l = 0; l < SB; ++l)
          if (k0 + l <= j) hv[l] = hval(P, dirs, ti, i, j - k0 - l);
#pragma unroll
        for (int l = 0; l < SB; ++l)
          if (k0 + l <= j && hv[l] - go - (k0 + l) * ge == h) { kb = k0 + l; hb = hv[l]; }
      }
    }
    if (!kb) break;  // unreachable for a consistent H store (no predecessor found)
    rw.push(2u, (uint32_t)kb);
    j -= kb;
    h = hb;
  }
  rw.flush();
  *n_ops = rw.n;
  *beg_i = i;
  *beg_j = j;
}

}  // namespace anyseq
