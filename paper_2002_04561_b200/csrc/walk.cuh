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

// Element addressing of one pair: R (rows per lane) and L = 8 (lanes per group, every batch
// variant) are compile-time; the warp-slot base and the diagonal count are computed once per
// pair.  raw(i, j) is the stored element of cell (i, j): the exact H (full store; s16x2
// halves unbiased) or its low byte (tb8).
template <int R>
struct HView {
  static constexpr int L = 8, G = 4, HS = L * R;
  const uint8_t* base;  // byte address of the warp-slot block's element 0
  int DK, pad, grp, half;
  bool p2, tb8;
  __device__ __forceinline__ HView(const uint32_t* dirs, const TbInfo& ti, bool t8) {
    p2 = ti.P == 2;
    tb8 = t8;
    const int esz = tb8 ? (p2 ? 2 : 1) : 4;
    base = reinterpret_cast<const uint8_t*>(dirs) + ti.dir_base * esz;
    DK = ti.slot_M + L - 1 + R - 1;
    pad = ti.pad;
    grp = ti.grp;
    half = ti.half;
  }
  __device__ __forceinline__ int raw(int i, int j) const {
    const int ip = i - 1 + pad;
    const int st = ip / HS;
    int r = ip - st * HS;
    const int tt = r / R;
    r -= tt * R;
    const int d = (j - 1) + tt - r + R - 1;  // diagonal (wavefront step - row) of the cell
    const uint64_t e = (uint64_t)(uint32_t)(st * DK + d) * (uint32_t)(R * G * L) +
                       (uint32_t)((r * G + grp) * L + tt);
    if (tb8) {
      if (p2) return (int)((__ldg(reinterpret_cast<const unsigned short*>(base) + e) >> (8 * half)) & 0xffu);
      return (int)__ldg(base + e);
    }
    const uint32_t word = __ldg(reinterpret_cast<const unsigned int*>(base) + e);
    if (p2) return (int)(int16_t)(uint16_t)(half ? (word >> 16) : (word & 0xffffu)) - (1 << 14);
    return (int)word;
  }
};

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
//
// Decisions, in the relax listing's order (readings R7-R9, R16):
//   (i, j) on row 0 / column 0: global -> boundary runs (R16), else stop; local H <= 0: stop;
//   DIAG iff H(i-1, j-1) = H - sigma (tested for up to 8 diagonal cells per batch);
//   linear: UP iff H(i-1, j) = H + g, else LEFT;
//   affine: UP iff H = E(i, j) = max_k H(i-k, j) - Go - k Ge, the gap being the LARGEST such k
//   (extension wins ties, R8), scanned 8 rows per batch while match * min(i-k, j) - Go - k Ge
//   could still reach H; else LEFT likewise along the row.
// One thread walks one pair, and the warp's 32 walks are kept convergent: every iteration of
// the loop is one batch of at most 8 loads in the thread's current mode (diagonal run, linear
// up-test, up scan, left scan), so threads in different modes only split inside one short
// batch body instead of running whole walks one after another.
template <int R>
__device__ __forceinline__ void walk_pair(const DevParams& P, const uint32_t* __restrict__ dirs,
                                          const TbInfo& ti, const uint8_t* qc, const uint8_t* sc,
                                          uint32_t* ops_out, int32_t* n_ops, int32_t* beg_i,
                                          int32_t* beg_j, int32_t* end_i_out, bool tb8) {
  constexpr int B = 8;  // cells per batch
  const HView<R> hs(dirs, ti, tb8);
  enum { TOP = 0, LINUP = 1, UP = 2, LEFT = 3, DONE = 4 };
  const int go = P.go, ge = P.ge;
  const int kind = P.kind;
  const bool linear = P.gap == GLINEAR;
  const int mt = max(P.smax, 0);
  RunWriter rw{ops_out, 0, 0, 0};
  int i = ti.end_i, j = ti.end_j;
  int h = ti.score;
  if (ti.end_span > 0) {
    // the fill recorded the first row of the lane holding the optimum at column j: the end
    // cell is the lane's first row with H = score (the lane's rows lie within d (R-1) < 256
    // of the maximum, so equal low bytes mean equal values; host check)
    int found = i;
    bool got = false;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i2 = ti.end_i + r;
      const int raw = i2 >= 1 ? hs.raw(i2, j) : -1;
      if (!got && i2 >= 1 && hmatch(raw, h, tb8)) { found = i2; got = true; }
    }
    i = found;
    *end_i_out = i;
  }
  int mode = TOP;
  int k0 = 1, ref = 0, kb = 0, hb = 0;  // gap scans: next k, exact value of the last cell, best
  while (mode != DONE) {
    if (mode == TOP) {
      if (i == 0 || j == 0) {
        if (kind == KGLOBAL) {  // reading R16: boundary runs
          rw.push(1u, (uint32_t)i);
          rw.push(2u, (uint32_t)j);
          i = 0; j = 0;
        }
        mode = DONE;
        continue;
      }
      if (kind == KLOCAL && h <= 0) { mode = DONE; continue; }  // STOP (reading R9)
      // diagonal run: the next B diagonal cells are loaded together, then verified in order
      const int lim = min(B, min(i, j));
      int hv[B], sg[B];
      uint64_t vq = 0, vs = 0;
      const bool vec = i > B && j > B;
      if (vec) {  // the B query / subject codes: two aligned 8-byte loads each (16 B slack)
        auto load8 = [](const uint8_t* p) -> uint64_t {
          const uintptr_t a = (uintptr_t)p & ~(uintptr_t)7;
          const uint64_t lo = __ldg((const unsigned long long*)a);
          const uint64_t hi = __ldg((const unsigned long long*)(a + 8));
          const int sh = (int)((uintptr_t)p - a) * 8;
          return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
        };
        vq = load8(qc + i - (B - 1));  // byte B-1-l = code of row i - l
        vs = load8(sc + j - (B - 1));
      }
#pragma unroll
      for (int l = 0; l < B; ++l) {
        hv[l] = 0;
        sg[l] = 0;
        if (l < lim) {
          const int i2 = i - 1 - l, j2 = j - 1 - l;
          hv[l] = (i2 == 0 || j2 == 0) ? hbound(P, i2, j2) : hs.raw(i2, j2);
          const uint32_t cq = vec ? (uint32_t)(vq >> (8 * (B - 1 - l))) & 0xffu : qc[i - l];
          const uint32_t cs = vec ? (uint32_t)(vs >> (8 * (B - 1 - l))) & 0xffu : sc[j - l];
          sg[l] = sigma_of(P, cq, cs);
        }
      }
      int taken = 0;
#pragma unroll
      for (int l = 0; l < B; ++l) {
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
      } else if (linear) {
        mode = LINUP;
      } else {
        mode = UP; k0 = 1; ref = h; kb = 0;
      }
      continue;
    }
    if (mode == LINUP) {  // linear gaps: UP iff H(i-1, j) = H + g, else LEFT
      const bool up = (i - 1 == 0) ? hbound(P, 0, j) == h + ge
                                   : hmatch(hs.raw(i - 1, j), h + ge, tb8);
      if (up) { rw.push(1u, 1); --i; } else { rw.push(2u, 1); --j; }
      h += ge;
      mode = TOP;
      continue;
    }
    // affine gap scans (mode UP: along column j; LEFT: along row i)
    const bool upm = mode == UP;
    const int len = upm ? i : j;              // k runs 1..len
    const int other = upm ? j : i;
    bool fin = k0 > len || mt * min(len - k0, other) - go - k0 * ge < h;
    if (!fin) {
      int hv[B];
#pragma unroll
      for (int l = 0; l < B; ++l) {
        hv[l] = 0;
        if (k0 + l <= len) {
          const int x = len - k0 - l;  // i2 (UP) or j2 (LEFT)
          hv[l] = (x == 0) ? (upm ? hbound(P, 0, j) : hbound(P, i, 0))
                           : (upm ? hs.raw(x, j) : hs.raw(i, x));
        }
      }
#pragma unroll
      for (int l = 0; l < B; ++l) {
        if (k0 + l <= len) {
          const int x = len - k0 - l;
          ref = (x == 0) ? hv[l] : hnear(hv[l], ref, tb8);
          if (ref - go - (k0 + l) * ge == h) { kb = k0 + l; hb = ref; }
        }
      }
      k0 += B;
      fin = k0 > len || mt * min(len - k0, other) - go - k0 * ge < h;
    }
    if (fin) {
      if (kb) {
        rw.push(upm ? 1u : 2u, (uint32_t)kb);
        if (upm) i -= kb; else j -= kb;
        h = hb;
        mode = TOP;
      } else if (upm) {
        mode = LEFT; k0 = 1; ref = h; kb = 0;
      } else {
        mode = DONE;  // unreachable for a consistent H store (no predecessor found)
      }
    }
  }
  rw.flush();
  *n_ops = rw.n;
  *beg_i = i;
  *beg_j = j;
}

}  // namespace anyseq
