// csrc/fill_kernel.cuh -- batched DP relaxation ("fill") kernel.
//
// What it computes: Eq. (1) H = max{H_diag + sigma, E, F, nu},
// linear gaps Eqs. (2)-(3), affine gaps Eqs. (4)-(5), the per-kind
// initialisation and optimum, max-tracking only where needed, and
// optionally (traceback) every cell's H for the walk that re-derives the predecessor
// decisions of the relax listing from it.
//
// How (B200 design):
//  * A lane group of L lanes (L | 32) relaxes one "slot" = one alignment (VS32) or two
//    alignments packed in the 16-bit halves of every register (VS16).  Lane t owns R
//    consecutive rows of a strip of L*R rows; the group sweeps the columns with a skew of
//    one column per lane, i.e. an anti-diagonal wavefront inside the warp (the paper's
//    minor-diagonal parallelism).  H, E (vertical) of the lane's bottom row go to
//    the next lane with __shfl_up_sync; H_left, Hop and F stay in registers per row.
//  * sigma comes from one PRMT per register: per-row query profile bytes sigma(q_i, .)
//    selected (with sign replication) by a per-column selector built from the subject
//    symbol(s) -- one instruction for two cells in VS16.
//  * Cell ops per register: PRMT, VIADDMNMX (E), VIADDMNMX (F), VIMNMX (E|F), VIADDMNMX (H;
//    local: a 3-input max with the floor nu = 0) on the integer pipe, and Hop = H - Go - Ge
//    (shared by E below and F right) as an IMAD on the FMA pipe: VS16 scores are stored with
//    a +2^14 bias so that the packed subtraction can never borrow across the halves.
//  * H lives in two register arrays used in ping-pong across steps (step k reads HA and
//    writes HB, step k+1 the reverse), so the diagonal value H(i-1,j-1) never needs a copy.
//  * Rows longer than one strip are handled strip after strip; the bottom row (H, E) of a
//    strip is kept in a per-group global row buffer (the paper's tile border stripe,
//    P:275, Fig. 2) and read back by lane 0 of the next strip.
//  * Local/semi-global pad rows at the TOP of the first strip (sigma = 0 rows reproduce
//    the H = 0 initial row exactly), global pads at the BOTTOM (rows below n never
//    influence H(n,m)); see DESIGN.md "padding".
#pragma once
#include "common.cuh"
#include "fill_args.h"
#include <type_traits>

namespace anyseq {

// (value desc, j asc, i asc) merge used by the local end-cell rule (reading R10)
__device__ __forceinline__ bool key_better(int v, int i, int j, int bv, int bi, int bj) {
  return v > bv || (v == bv && (j < bj || (j == bj && i < bi)));
}

// x * one + k with `one` opaque to the compiler -> IMAD (FMA pipe), not IADD3 (ALU pipe)
__device__ __forceinline__ uint32_t imad_add(uint32_t x, uint32_t one, uint32_t k) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(one), "r"(k));
  return d;
}

// CGE/CGO > 0: the gap extend / open values are compile-time constants (the paper's partial
// evaluation of the scoring scheme): the packed constants then become
// instruction immediates and the 3-source DPX/IMAD ops read one register less.
#ifndef FILL_MINB_SCORE
#define FILL_MINB_SCORE 4  // resident 128-thread blocks per SM the score kernels are built for
#endif
#ifndef FILL_MINB_TBWIDE
#define FILL_MINB_TBWIDE 3  // traceback kernels with R > 8 rows per lane: 168 registers, no spills
#endif
template <class V, int KIND, int GAP, int L, int R, bool TB, bool POS, int CGE = 0, int CGO = 0>
__global__ void __launch_bounds__(128, (TB && R > 8) ? FILL_MINB_TBWIDE : FILL_MINB_SCORE)
    fill_kernel(FillArgs a) {
  using T = typename V::T;
  constexpr int PP = V::P;
  constexpr int G = 32 / L;
  constexpr int HS = L * R;  // strip height
  // biased VS16 representation (every kind): stored = value + 2^14, so every H stays above
  // Go + Ge and Hop = H - Go - Ge is one packed IMAD (FMA pipe) without a borrow between
  // the halves; local's floor nu = 0 (Eq. 1) becomes the biased zero ZB
  constexpr bool BIAS = (PP == 2);
  constexpr int B0 = BIAS ? (1 << 14) : 0;
  const int lane = threadIdx.x & 31;
  const int g = lane / L, t = lane % L;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int slot_lo = a.nslots_dev ? 0 : a.slot_lo;
  const int slot_hi = a.nslots_dev ? *a.nslots_dev : a.slot_hi;
  const int nsl = slot_hi - slot_lo;
  const int nws = (nsl + G - 1) / G;
  const DevParams& P = a.P;
  constexpr bool pos = TB || POS;
  constexpr bool FAST = (GAP == GAFFINE);  // reassociated affine recurrence (score and TB)
  const uint32_t one = (uint32_t)a.one;
  constexpr bool SPEC = CGE > 0;
  const int cop = SPEC ? ((GAP == GAFFINE) ? CGO + CGE : CGE)
                       : ((GAP == GAFFINE) ? (P.go + P.ge) : P.ge);  // H -> Hop
  const T NEG = (PP == 2) ? V::splat(NEG16 + B0) : V::splat(NEG32);
  // packed constants straight from the kernel-parameter bank (no register-file bank reads)
  const T NGE = SPEC ? V::splat(-CGE) : ((PP == 2) ? (T)a.nge_s16 : V::splat(-P.ge));
  const T NOC = V::splat(-cop);
  const uint32_t KOC = (!SPEC && PP == 2 && GAP == GAFFINE) ? a.koc_s16
                                                            : (uint32_t)(-(int)(cop * ((PP == 2) ? 65537 : 1)));
  auto hop = [&](T h) -> T {  // Hop = H - Go - Ge (or H - g)
    if (PP == 1 || BIAS) return (T)imad_add((uint32_t)h, one, KOC);
    return V::add(h, NOC);
  };
  auto enc = [&](int v0, int v1) -> T { return V::make(v0 + B0, v1 + B0); };
  const T ZB = V::splat(B0);  // the local floor (biased zero)
  // H(., m) of every lane at its last column (odd row stride R keeps banks distinct)
  __shared__ uint32_t capbuf[KIND != KLOCAL ? PP : 1][128][KIND != KLOCAL ? R : 1];
  // rarely touched per-lane state lives in shared memory, not in registers
  struct LaneTrack { int nn[2], pad[2], cv[2], ci[2], gv[2]; };
  __shared__ LaneTrack track[128];
  // per-group column selectors of the current slot (built once per slot, read by every lane
  // at its own column: no selector shuffle, no per-step global loads)
  constexpr int SELCAP = 512;
  constexpr int SELMIR = 128;  // mirror of the first 128 slots after the end
  __shared__ uint16_t seltab[4 * G][SELCAP + SELMIR];
  const int gb = (threadIdx.x >> 5) * G + g;
  auto dec = [&](T x, int X) -> int { return V::get(x, X) - B0; };

  // warp-slots in plan order (largest first): handed out by ticket when the launch has a
  // zeroed counter (balances mixed lengths), else statically round-robin
  auto next_ws = [&](int stat) -> int {
    if (!a.ticket) return stat;
    int v = 0;
    if (lane == 0) v = atomicAdd(a.ticket, 1);
    return __shfl_sync(0xffffffffu, v, 0);
  };
  for (int ws = next_ws(warp); ws < nws; ws = next_ws(ws + nwarps)) {
    const int sidx = ws * G + g;
    const bool valid = (g < G) && (sidx < nsl);
    int pr[PP], nn[PP], mm[PP];
    uint64_t qo[PP], so[PP];
    {
      Slot sl;
      sl.pair[0] = sl.pair[1] = -1;
      if (valid) sl = a.slots[slot_lo + sidx];
#pragma unroll
      for (int X = 0; X < PP; ++X) {
        pr[X] = sl.pair[X];
        if (pr[X] >= 0) {
          qo[X] = a.q_off[pr[X]];
          nn[X] = (int)(a.q_off[pr[X] + 1] - qo[X]);
          so[X] = a.s_off[pr[X]];
          mm[X] = (int)(a.s_off[pr[X] + 1] - so[X]);
        } else {
          qo[X] = so[X] = 0;
          nn[X] = mm[X] = 0;
        }
      }
    }
    int M = 0, nmax = 0;
#pragma unroll
    for (int X = 0; X < PP; ++X) {
      M = max(M, mm[X]);
      nmax = max(nmax, nn[X]);
    }
    // a "uniform" slot: every present pair has M columns -> captures after the sweep
    const bool uni = (PP == 1) || pr[PP - 1] < 0 || mm[0] == mm[PP - 1];
    const int NS = (M > 0) ? (nmax + HS - 1) / HS : 0;
    const int Mw = __reduce_max_sync(0xffffffffu, M);
    const int NSw = __reduce_max_sync(0xffffffffu, NS);
    const int npad = NS * HS;
    int pad[PP];
#pragma unroll
    for (int X = 0; X < PP; ++X) pad[X] = (KIND == KGLOBAL) ? 0 : npad - nn[X];
    uint4* scr = a.strip_scratch + (int64_t)(warp * G + g) * a.strip_stride;
    // traceback H store: one block per warp-slot, the G slots of the warp interleaved at
    // lane-group granularity (a warp's store covers G x L contiguous elements: whole
    // 32-byte sectors for every element size)
    int64_t dbase = 0;
    if (TB) dbase = (int64_t)ws * G * a.dir_block_words;

    // column selectors of this slot in a 512-entry shared ring: columns [0, 384) now, then
    // 128 more every 128 steps (a lane at step k reads column k - t, t < L <= 8)
    auto fill_sel = [&](int c0, int c1) {
      constexpr int U = 4;  // loads in flight per lane before the first use
      for (int cb = c0 + t; cb < c1; cb += L * U) {
        uint32_t x0[U], x1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = cb + u * L;
          x0[u] = (c < c1 && c < mm[0]) ? a.scode[so[0] + c] : 0u;
          x1[u] = (PP == 2 && c < c1 && c < mm[PP - 1]) ? a.scode[so[PP - 1] + c] : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = cb + u * L;
          if (c < c1) {
            const uint16_t sv = (uint16_t)V::selector(x0[u], x1[u]);
            seltab[gb][c & (SELCAP - 1)] = sv;
            if ((c & (SELCAP - 1)) < SELMIR) seltab[gb][SELCAP + (c & (SELCAP - 1))] = sv;
          }
        }
      }
    };
    if (Mw <= SELCAP) {  // the whole slot fits: built once for all strips
      fill_sel(0, M);
      __syncwarp();
    }

    // ---- optimum trackers (readings R5, R10) ----
    T best = enc(0, 0);             // local running max / semi bottom-row max ((n,0) = 0)
    T bfin = enc(0, 0);             // semi (plain score): bottom-row max at column m
    int bv[PP], bi[PP], bj[PP];      // local (POS) overall best per half
    int rj[PP];                      // semi bottom-row best column
#pragma unroll
    for (int X = 0; X < PP; ++X) {
      bv[X] = 0; bi[X] = 0; bj[X] = 0; rj[X] = 0;
      // semi column-m best (value, i) starts at H(0,m) = 0; global H(n,m)
      track[threadIdx.x].cv[X] = 0;
      track[threadIdx.x].ci[X] = 0;
      track[threadIdx.x].gv[X] = 0;
      track[threadIdx.x].nn[X] = nn[X];
      track[threadIdx.x].pad[X] = pad[X];
    }

    // one strip of the sweep; MULTI = the warp has more than one strip (strip scratch rows
    // are read and written): single-strip warps (short reads) compile without any of it
    auto strip = [&](auto multi, const int st) {
      constexpr bool MULTI = decltype(multi)::value;
      const bool sact = st < NS;
      if (Mw > SELCAP) {  // ring restarts with every strip
        fill_sel(0, min(M, 384));
        __syncwarp();
      }
      const bool last_strip = (st == NS - 1);
      const int ip0 = st * HS + t * R;  // first physical row of this lane
      uint32_t p0[R], p1[R];
      T HA[R], HB[R], Ff[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int ip = ip0 + r;
        int iv[PP];
        uint32_t pf[PP];
        bool rl[PP];
        uint32_t c0 = 0;
#pragma unroll
        for (int X = 0; X < PP; ++X) {
          const int i = (KIND == KGLOBAL) ? ip + 1 : ip - pad[X] + 1;  // real row, 1-based
          rl[X] = sact && i >= 1 && i <= nn[X];
          const uint32_t c = rl[X] ? a.qcode[qo[X] + i - 1] : 0u;
          if (X == 0) c0 = c;
          pf[X] = rl[X] ? prof4(P, c) : 0u;  // pad rows: sigma = 0
          iv[X] = (KIND == KGLOBAL && i >= 1) ? -(P.go + i * P.ge) : 0;  // H(i,0)
        }
        if (PP == 1) {
          p0[r] = pf[0];
          p1[r] = rl[0] ? pn_of(P, c0) : 0u;  // byte 4 = sigma(q_i, N)
        } else {
          p0[r] = pf[0];
          p1[r] = pf[PP - 1];
        }
        HA[r] = enc(iv[0], iv[PP - 1]);
        HB[r] = HA[r];
        Ff[r] = NEG;
      }
      // H of the row above this lane's first row at column 0
      T diag;
      {
        int dv = 0;
        if (KIND == KGLOBAL && ip0 >= 1) dv = -(P.go + ip0 * P.ge);
        diag = enc(dv, dv);
      }
      T Hbot = NEG, Ebot = NEG;
      // per-strip local trackers (merged by key at strip end)
      int sv[PP], si[PP], sj[PP];
#pragma unroll
      for (int X = 0; X < PP; ++X) { sv[X] = 0; si[X] = 0; sj[X] = 0; }
      T sbest = ZB;

      const int K = Mw + L - 1;
      // H(i, 0) of row ip (initial column, P:259 / P:262)
      auto init_col = [&](int ip) -> T {
        if (KIND == KGLOBAL) {
          const int v = -(P.go + (ip + 1) * P.ge);
          return enc(v, v);
        }
        return enc(0, 0);
      };
      // Every lane relaxes its rows in every step (no divergent "active" region: a lane
      // outside its column range computes values nobody reads).  A lane loads its initial
      // column when it reaches column 0 and hands over captures at its last column.
      // CHK = this step may contain a lane's column 0 (initial column) or a pair's column m
      // (captures); the steady-state steps in between run without those checks.
      const uint32_t selbase = (uint32_t)__cvta_generic_to_shared(&seltab[gb][0]);
      uint32_t selo = 0, selv = 0;  // selv = selector of the next step (loaded one step ahead)
      auto lds16 = [&](uint32_t addr) -> uint32_t {
        unsigned short v16;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v16) : "r"(addr));
        return v16;
      };
      auto rebase = [&](int kk) {
        selo = selbase + (uint32_t)(((kk - t) & (SELCAP - 1)) * 2);
        selv = lds16(selo);
      };
      // strips after the first: lane 0's input row (H, E of the strip above) is prefetched
      // two steps ahead from the strip scratch (L2) in two registers used alternately
      uint4 pfA = make_uint4(0, 0, 0, 0), pfB = pfA;
      if (MULTI && st > 0 && t == 0 && sact) {
        pfA = scr[0];
        if (M > 1) pfB = scr[1];
      }
      auto step = [&](auto chk, const int k, T (&Hi)[R], T (&Hq)[R], uint4& pf) {
        constexpr bool CHK = decltype(chk)::value;
        T hin = V::shfl_up(Hbot, L);
        T ein = (GAP == GAFFINE) ? V::shfl_up(Ebot, L) : NEG;
        const int col = k - t;
        // selector of this lane's column: a shared-memory pointer that advances by one slot
        // per step (IMAD, FMA pipe) and is re-based every 128 steps (the mirror covers the
        // wrap in between), so the hot loop spends no ALU instruction on addressing
        const uint32_t sel = selv;
        selo = imad_add(selo, one, 2u);
        selv = lds16(selo);  // prefetch: the load latency overlaps this step's rows
        const bool act = CHK ? (sact && col >= 0 && col < M) : sact;
        if (CHK && col == 0 && sact) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            Hi[r] = init_col(ip0 + r);
            Ff[r] = NEG;  // F(i,0) = -inf
          }
          diag = (KIND == KGLOBAL && ip0 >= 1) ? init_col(ip0 - 1) : enc(0, 0);
          if (KIND == KLOCAL && !pos) sbest = ZB;
          if (KIND == KSEMI) {
            best = enc(0, 0);  // H(n,0) = 0 (first row candidate)
#pragma unroll
            for (int X = 0; X < PP; ++X) rj[X] = 0;
          }
        }
        if (!MULTI || st == 0) {  // the initial row (P:259 / P:262): no load, no branch
          const int h0 = (KIND == KGLOBAL) ? -(P.go + (col + 1) * P.ge) : 0;  // H(0,j)
          const T h0v = enc(h0, h0);
          if (t == 0) {
            hin = h0v;
            // E-below convention (FAST): E(1,j) = H(0,j) - Go - Ge; else E(0,j)
            ein = FAST ? hop(h0v) : NEG;
          }
        } else if (t == 0 && act) {
          const uint4 v = pf;
          hin = (T)v.x;
          ein = (T)v.y;
        }
        if (MULTI && st > 0 && t == 0 && sact && col + 2 < M) pf = scr[col + 2];
        // FAST = affine score-only: the reassociated recurrence
        //   F  = max(F - Ge, H_left - Go - Ge)          Eq. (5)
        //   DF = max(H_diag + sigma, F)
        //   H  = max(DF, E)        (.RELU: nu = 0)      Eq. (1)
        //   E' = max(E - Ge, DF - Go - Ge)              Eq. (4) for the row below, exact since
        //        H - Go - Ge = max(DF, E) - Go - Ge and E - Go - Ge <= E - Ge
        // so the only dependency from row to row is one VIADDMNMX on E.  In this mode the
        // value handed down the lanes / strips is E of the row BELOW the bottom row.
        T hup = FAST ? NEG : hop(hin);  // Hop of the row above (other modes)
        T e = ein;
        if (FAST) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const T hd = (r == 0) ? diag : Hi[r - 1];
            const T sig = V::sigma(p0[r], p1[r], sel);
            Ff[r] = V::addmax(Ff[r], NGE, hop(Hi[r]));
            const T df = V::addmax(hd, sig, Ff[r]);
            const T h = (KIND != KLOCAL) ? V::vmax(df, e)
                                         : (BIAS ? V::vmax3(df, e, ZB) : V::vmax_relu(df, e));
            e = V::addmax(e, NGE, hop(df));
            Hq[r] = h;
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const T hd = (r == 0) ? diag : Hi[r - 1];
            const T sig = V::sigma(p0[r], p1[r], sel);
            const T hleft = hop(Hi[r]);  // Hop(i, j-1), recomputed on the FMA pipe
            // Eqs. (2)-(3): H_up - g, H_left - g (biased local: and the floor)
            const T tm = (KIND == KLOCAL && BIAS) ? V::vmax3(hup, hleft, ZB) : V::vmax(hup, hleft);
            const T h = (KIND == KLOCAL && !BIAS) ? V::addmax_relu(hd, sig, tm) : V::addmax(hd, sig, tm);
            Hq[r] = h;
            hup = hop(h);
          }
        }
        // Traceback mode: the score recurrence above plus every cell's H, stored packed
        // (both alignments of an s16x2 register in one word, 2 B per cell) step-major and
        // lane-contiguous per slot; the walk re-derives each decision of the relax listing
        // (R7-R9) from H alone (walk_kernel).  Storing H instead of direction
        // bits keeps the fill at the score-only instruction count.
        if (TB && valid && sact && k < M + L - 1) {
          // element (((st * DK + k - r + R - 1) * R + r) * G + g) * L + t, DK from the warp's
          // widest slot: diagonal-major (the walk's diagonal runs are sequential), the lane
          // groups of the warp side by side, so one store instruction writes G * L
          // contiguous elements (128 B full store, 64 B / 32 B low-byte store)
          const int64_t w0 = ((((int64_t)st * (Mw + L - 1 + R - 1) + k + R - 1) * R) * G + g) * L + t;
          if (a.tb8) {
            // 1 B per cell: the low byte of H of each alignment (both halves of an s16x2
            // register in one 16-bit store); same element order, elements of 2 B (s16x2)
            // or 1 B (s32) instead of 4 B words
            if (V::P == 2) {
              uint16_t* bp = reinterpret_cast<uint16_t*>(a.dirs) + dbase + w0;
#pragma unroll
              for (int r = 0; r < R; ++r)
                bp[-(int64_t)r * (R - 1) * G * L] = (uint16_t)prmt((uint32_t)Hq[r], 0u, 0x0020u);
            } else {
              uint8_t* bp = reinterpret_cast<uint8_t*>(a.dirs) + dbase + w0;
#pragma unroll
              for (int r = 0; r < R; ++r) bp[-(int64_t)r * (R - 1) * G * L] = (uint8_t)Hq[r];
            }
          } else {
            uint32_t* wp = a.dirs + dbase + w0;
#pragma unroll
            for (int r = 0; r < R; ++r) wp[-(int64_t)r * (R - 1) * G * L] = (uint32_t)Hq[r];
          }
        }
        diag = hin;
        Hbot = Hq[R - 1];
        Ebot = e;
        if (MULTI && act && t == L - 1 && st + 1 < NS)
          scr[col] = make_uint4((uint32_t)Hq[R - 1], (uint32_t)e, 0u, 0u);

        // ---- optimum bookkeeping ----
        // Plain score mode tracks maxima in every lane and every step without masks: the
        // trackers restart when a lane enters column 0 and are snapshotted when it leaves
        // a pair's column m, so columns outside the pair never count.
        if (KIND == KLOCAL) {
          T cm = Hq[0];
#pragma unroll
          for (int r = 1; r + 1 < R; r += 2) cm = V::vmax3(cm, Hq[r], Hq[r + 1]);
          if ((R % 2) == 0) cm = V::vmax(cm, Hq[R - 1]);
          if (!pos) {
            sbest = V::vmax(sbest, cm);
          } else {
            uint32_t keep = 0;
            if (act) {
#pragma unroll
              for (int X = 0; X < PP; ++X) keep |= (uni || col < mm[X] ? 1u : 0u) << X;
            }
            cm = V::select_mask(cm, keep, ZB);
            uint32_t pb;
            const T nb = V::bmax(sbest, cm, pb);  // bit: sbest >= cm
            if (TB && PP == 2 && a.defer_row && ((~pb) & 3u)) {
              // traceback: record the lane's first row only; the walk finds the row of the
              // lane holding the maximum in the H store (TbInfo::end_span)
#pragma unroll
              for (int X = 0; X < PP; ++X) {
                if (!((pb >> X) & 1u)) {
                  sv[X] = dec(cm, X);
                  si[X] = ip0 - pad[X] + 1;
                  sj[X] = col + 1;
                }
              }
            } else if (PP == 2 && ((~pb) & 3u)) {
              // the smallest row holding the new maximum, both alignments at once: on a
              // kept half 0 <= Hq[r] <= cm (local), so e = max(Hq[r] + 1 - cm, 0) is 1 iff
              // Hq[r] == cm, and key = 64 e + 63 - r is largest for the first such row
              // (one DPX op + one IMAD per row instead of a compare-select per row and half)
              const T om = __vsub2(V::splat(1), cm);
              const uint32_t k64 = one << 6;
              T kmax = 0;
#pragma unroll
              for (int r = 0; r < R; r += 2) {
                const T ka = (T)imad_add((uint32_t)__viaddmax_s16x2(Hq[r], om, 0u), k64,
                                         (uint32_t)(63 - r) * 0x10001u);
                if (r + 1 < R) {
                  const T kb = (T)imad_add((uint32_t)__viaddmax_s16x2(Hq[r + 1], om, 0u), k64,
                                           (uint32_t)(62 - r) * 0x10001u);
                  kmax = V::vmax3(kmax, ka, kb);
                } else {
                  kmax = V::vmax(kmax, ka);
                }
              }
#pragma unroll
              for (int X = 0; X < PP; ++X) {
                if (!((pb >> X) & 1u)) {
                  sv[X] = dec(cm, X);
                  si[X] = ip0 + (63 - (V::get(kmax, X) & 63)) - pad[X] + 1;
                  sj[X] = col + 1;
                }
              }
            } else if (PP == 1 && ((~pb) & 1u)) {
#pragma unroll
              for (int X = 0; X < PP; ++X) {
                if (!((pb >> X) & 1u)) {
                  const int v = V::get(cm, X);
                  int rr = R - 1;
#pragma unroll
                  for (int r = R - 1; r >= 0; --r)
                    if (V::get(Hq[r], X) == v) rr = r;
                  sv[X] = v;
                  si[X] = ip0 + rr - pad[X] + 1;
                  sj[X] = col + 1;
                }
              }
            }
            sbest = nb;
          }
        } else if (KIND == KSEMI) {
          // bottom row n (row candidates j = 1..m-1 precede column m, reading R5); only
          // lane L-1 of the last strip holds row n, the others' values are ignored.
          if (!pos) {
            best = V::vmax(best, Hq[R - 1]);  // j = m may join: it is also a column candidate
          } else if (last_strip) {
            uint32_t keep = 0;
            if (act) {
#pragma unroll
              for (int X = 0; X < PP; ++X) keep |= (col < mm[X] - 1 ? 1u : 0u) << X;
            }
            uint32_t pb;
            const T nb = V::bmax(best, V::select_mask(Hq[R - 1], keep, NEG), pb);
#pragma unroll
            for (int X = 0; X < PP; ++X)
              if (!((pb >> X) & 1u)) rj[X] = col + 1;
            best = nb;
          }
        }
        // a pair's last column m: park this lane's H(., m) in shared memory (semi: column
        // candidates, global: H(n,m)); evaluated after the sweep, off the hot path
        if (CHK && act && (col == mm[0] - 1 || (PP == 2 && col == mm[PP - 1] - 1))) {
#pragma unroll
        for (int X = 0; X < PP; ++X) {
          if (col == mm[X] - 1) {
            if (KIND != KLOCAL) {
#pragma unroll
              for (int r = 0; r < R; ++r) capbuf[X][threadIdx.x][r] = (uint32_t)Hq[r];
            }
            if (KIND == KLOCAL && !pos) best = V::select_mask(V::vmax(best, sbest), 1u << X, best);
            if (KIND == KSEMI && !pos && last_strip) bfin = V::select_mask(best, 1u << X, bfin);
          }
        }
        }
      };

      // phases: [0, kA) checked (lanes enter column 0), [kA, kB) plain, [kB, K) checked
      // (lanes leave a pair's last column); kA, kB even and warp-uniform.
      const std::integral_constant<bool, true> CHK_ON{};
      const std::integral_constant<bool, false> CHK_OFF{};
      int mmin = 0x7fffffff;  // smallest pair width in the warp (captures start there)
#pragma unroll
      for (int X = 0; X < PP; ++X)
        if (valid && pr[X] >= 0) mmin = min(mmin, mm[X]);
      const int Mmin = __reduce_min_sync(0xffffffffu, mmin);
      const int kA = min(K & ~1, (L + 1) & ~1);
      const int kB = max(kA, min(K, Mmin - 1) & ~1);
      int k = 0;
      rebase(0);
      for (; k < kA; k += 2) {
        step(CHK_ON, k, HA, HB, pfA);
        step(CHK_ON, k + 1, HB, HA, pfB);
      }
      // every 128 steps (warp-uniform): selector ring refill (long rows) and pointer rebase
      auto block_start = [&](int kk) {
        if ((kk & 127) == 0) {
          if (Mw > SELCAP && kk > 0) {
            fill_sel(kk + 256, min(M, kk + 384));
            __syncwarp();
          }
          rebase(kk);
        }
      };
      while (k < kB) {
        block_start(k);
        const int kend = min(kB, (k & ~127) + 128);
        for (; k < kend; k += 2) {
          step(CHK_OFF, k, HA, HB, pfA);
          step(CHK_OFF, k + 1, HB, HA, pfB);
        }
      }
      for (; k + 1 < K; k += 2) {
        block_start(k);
        step(CHK_ON, k, HA, HB, pfA);
        step(CHK_ON, k + 1, HB, HA, pfB);
      }
      if (k < K) {
        block_start(k);
        step(CHK_ON, k, HA, HB, pfA);
      }

      __syncwarp();  // capbuf writes of this strip are visible (all lanes participate)
      if (KIND != KLOCAL && sact) {
        LaneTrack& tr = track[threadIdx.x];
#pragma unroll 1
        for (int X = 0; X < PP; ++X) {
          const int nX = tr.nn[X], pX = tr.pad[X];
          if (KIND == KSEMI && !pos) {
            // score only: the column-m maximum without its row (pad rows hold H = 0, which
            // is the H(0,m) candidate anyway)
            T cmx = (T)capbuf[X][threadIdx.x][0];
#pragma unroll
            for (int r = 1; r < R; ++r) cmx = V::vmax(cmx, (T)capbuf[X][threadIdx.x][r]);
            tr.cv[X] = max(tr.cv[X], dec(cmx, X));
          } else if (KIND == KSEMI) {  // column m candidates i = 1..n of this strip (R5)
            int cvx = tr.cv[X], cix = tr.ci[X];
#pragma unroll 1
            for (int r = 0; r < R; ++r) {
              const int i = ip0 + r - pX + 1;
              const int v = dec((T)capbuf[X][threadIdx.x][r], X);
              if (i >= 1 && i <= nX && v > cvx) { cvx = v; cix = i; }
            }
            tr.cv[X] = cvx;
            tr.ci[X] = cix;
          } else {
            const int ipn = nX - 1;
            if (ipn >= 0 && st == ipn / HS && t == (ipn % HS) / R)
              tr.gv[X] = dec((T)capbuf[X][threadIdx.x][ipn % R], X);
          }
        }
      }
      if (KIND == KLOCAL) {
        if (pos) {
#pragma unroll
          for (int X = 0; X < PP; ++X)
            if (key_better(sv[X], si[X], sj[X], bv[X], bi[X], bj[X])) {
              bv[X] = sv[X]; bi[X] = si[X]; bj[X] = sj[X];
            }
        }
      }
      __syncwarp();
    };  // strip
    if (NSw == 1) {
      strip(std::false_type{}, 0);
    } else {
      for (int st = 0; st < NSw; ++st) strip(std::true_type{}, st);
    }

    // ---- reduce across the lane group and write results (P:424-436 steps 8, 10) ----
    int osc[PP], oi[PP], oj[PP];
#pragma unroll
    for (int X = 0; X < PP; ++X) {
      if (KIND == KLOCAL) {
        int v = pos ? bv[X] : dec(best, X), i = bi[X], j = bj[X];
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
          const int v2 = __shfl_xor_sync(0xffffffffu, v, o, L);
          const int i2 = __shfl_xor_sync(0xffffffffu, i, o, L);
          const int j2 = __shfl_xor_sync(0xffffffffu, j, o, L);
          if (key_better(v2, i2, j2, v, i, j)) { v = v2; i = i2; j = j2; }
        }
        osc[X] = v; oi[X] = i; oj[X] = j;
      } else if (KIND == KSEMI) {
        int v = track[threadIdx.x].cv[X], i = track[threadIdx.x].ci[X];
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
          const int v2 = __shfl_xor_sync(0xffffffffu, v, o, L);
          const int i2 = __shfl_xor_sync(0xffffffffu, i, o, L);
          if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
        }
        const int rv = __shfl_sync(0xffffffffu, dec(pos ? best : bfin, X), L - 1, L);
        const int rjj = __shfl_sync(0xffffffffu, rj[X], L - 1, L);
        if (rv >= v) { osc[X] = rv; oi[X] = nn[X]; oj[X] = rjj; }
        else { osc[X] = v; oi[X] = i; oj[X] = mm[X]; }
      } else {
        const int ipn = max(nn[X] - 1, 0);
        const int owner = (ipn % HS) / R;
        osc[X] = __shfl_sync(0xffffffffu, track[threadIdx.x].gv[X], owner, L);
        oi[X] = nn[X];
        oj[X] = mm[X];
      }
    }
    if (valid && t == 0) {
#pragma unroll
      for (int X = 0; X < PP; ++X) {
        if (pr[X] < 0) continue;
        a.scores[pr[X]] = osc[X];
        if (pos && a.end_i) { a.end_i[pr[X]] = oi[X]; a.end_j[pr[X]] = oj[X]; }
        if (TB) {
          TbInfo ti;
          ti.dir_base = dbase;
          ti.slot_M = Mw;
          ti.grp = g;
          ti.ns = NS;
          ti.half = (int16_t)X;
          ti.L = (int16_t)L;
          ti.R = (int16_t)R;
          ti.P = (int16_t)PP;
          ti.pad = pad[X];
          ti.score = osc[X];
          ti.end_i = oi[X];
          ti.end_j = oj[X];
          ti.end_span = (KIND == KLOCAL && PP == 2 && a.defer_row && osc[X] > 0) ? R : 0;
          a.tb[pr[X]] = ti;
        }
      }
    }
  }  // slots
}

}  // namespace anyseq
