// csrc/fill_kernel.cuh -- batched DP relaxation ("fill") kernel.
//
// What it computes: Eq. (1) H = max{H_diag + sigma, E, F, nu},
// linear gaps Eqs. (2)-(3), affine gaps Eqs. (4)-(5), the per-kind
// initialisation and optimum, max-tracking only where needed, and
// optionally the predecessor information of the relax listing as a packed
// direction nibble per cell for the traceback walk.
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
//  * Cells per register: PRMT, VIADDMNMX (E), VIADDMNMX (F), VIMNMX (E|F), VIADDMNMX (H,
//    .RELU for local: nu = 0), VIADD (Hop = H - Go - Ge shared by E below and F right).
//  * Rows longer than one strip are handled strip after strip; the bottom row (H, E) of a
//    strip is kept in a per-group global row buffer (the paper's tile border stripe,
//    P:275, Fig. 2) and read back by lane 0 of the next strip.
//  * Local/semi-global pad rows at the TOP of the first strip (sigma = 0 rows reproduce
//    the H = 0 initial row exactly), global pads at the BOTTOM (rows below n never
//    influence H(n,m)); see DESIGN.md "padding".
#pragma once
#include "common.cuh"
#include "fill_args.h"

namespace anyseq {



template <int L>
__device__ __forceinline__ int group_max(int v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o, L));
  return v;
}

// (value desc, j asc, i asc) merge used by the local end-cell rule (reading R10)
__device__ __forceinline__ bool key_better(int v, int i, int j, int bv, int bi, int bj) {
  return v > bv || (v == bv && (j < bj || (j == bj && i < bi)));
}

template <class V, int KIND, int GAP, int L, int R, bool TB>
__global__ void __launch_bounds__(128) fill_kernel(FillArgs a) {
  using T = typename V::T;
  constexpr int PP = V::P;
  constexpr int G = 32 / L;
  constexpr int HS = L * R;  // strip height
  const int lane = threadIdx.x & 31;
  const int g = lane / L, t = lane % L;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int slot_lo = a.nslots_dev ? 0 : a.slot_lo;
  const int slot_hi = a.nslots_dev ? *a.nslots_dev : a.slot_hi;
  const int nsl = slot_hi - slot_lo;
  const int nws = (nsl + G - 1) / G;
  const DevParams P = a.P;
  const bool pos = TB || a.pos;
  const T NEG = V::neg();
  const T NGE = V::splat(-P.ge);
  const T NOC = V::splat(GAP == GAFFINE ? -(P.go + P.ge) : -P.ge);  // H -> Hop ("H - Go - Ge")

  for (int ws = warp; ws < nws; ws += nwarps) {
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
    const int NS = (M > 0) ? (nmax + HS - 1) / HS : 0;
    const int Mw = __reduce_max_sync(0xffffffffu, M);
    const int NSw = __reduce_max_sync(0xffffffffu, NS);
    const int npad = NS * HS;
    int pad[PP];
#pragma unroll
    for (int X = 0; X < PP; ++X) pad[X] = (KIND == KGLOBAL) ? 0 : npad - nn[X];
    uint2* scr = a.strip_scratch + (int64_t)(warp * G + g) * a.strip_stride;
    int64_t dbase = 0;
    int S8 = 0;
    if (TB && valid) {
      dbase = (int64_t)sidx * a.dir_block_words;
      S8 = (M + L - 1 + 7) >> 3;
    }

    // ---- optimum trackers (readings R5, R10) ----
    T best = V::splat(0);           // local running max / semi bottom-row max (j=0 -> H(n,0)=0)
    int bv[PP], bi[PP], bj[PP];      // local (POS) overall best per half
    int cv[PP], ci[PP];              // semi column-m best per half (value, i); starts H(0,m)=0
    int rj[PP];                      // semi bottom-row best column
    int gv[PP];                      // global H(n,m)
#pragma unroll
    for (int X = 0; X < PP; ++X) {
      bv[X] = 0; bi[X] = 0; bj[X] = 0;
      cv[X] = 0; ci[X] = 0; rj[X] = 0; gv[X] = 0;
    }

    for (int st = 0; st < NSw; ++st) {
      const bool sact = st < NS;
      const int ip0 = st * HS + t * R;  // first physical row of this lane
      uint32_t p0[R], p1[R];
      T Hh[R], Ho[R], Ff[R];
      uint32_t acc[TB ? R * PP : 1];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int ip = ip0 + r;
        int iv[PP];
        uint32_t pf[PP];
        bool rl[PP];
#pragma unroll
        for (int X = 0; X < PP; ++X) {
          const int i = (KIND == KGLOBAL) ? ip + 1 : ip - pad[X] + 1;  // real row, 1-based
          rl[X] = sact && i >= 1 && i <= nn[X];
          const uint32_t c = rl[X] ? a.qcode[qo[X] + i - 1] : 0u;
          pf[X] = rl[X] ? prof4(P, c) : 0u;  // pad rows: sigma = 0
          iv[X] = (KIND == KGLOBAL && i >= 1) ? -(P.go + i * P.ge) : 0;  // H(i,0)
        }
        if (PP == 1) {
          p0[r] = pf[0];
          p1[r] = rl[0] ? P.mism4 : 0u;  // byte 4 = sigma(q_i, N) = mismatch
        } else {
          p0[r] = pf[0];
          p1[r] = pf[PP - 1];
        }
        Hh[r] = V::make(iv[0], iv[PP - 1]);
        Ho[r] = V::add(Hh[r], NOC);
        Ff[r] = NEG;  // F(i,0) = -inf
        if (TB) {
#pragma unroll
          for (int X = 0; X < PP; ++X) acc[r * PP + X] = 0;
        }
      }
      // H of the row above this lane's first row at column 0
      T diag;
      {
        int dv = 0;
        if (KIND == KGLOBAL && ip0 >= 1) dv = -(P.go + ip0 * P.ge);
        diag = V::splat(dv);
      }
      T Hbot = NEG, Ebot = NEG;
      uint32_t selb = 0;
      // per-strip local trackers (merged by key at strip end)
      int sv[PP], si[PP], sj[PP];
#pragma unroll
      for (int X = 0; X < PP; ++X) { sv[X] = 0; si[X] = 0; sj[X] = 0; }
      T sbest = V::splat(0);

      const int K = Mw + L - 1;
      for (int k = 0; k < K; ++k) {
        T hin = V::shfl_up(Hbot, L);
        T ein = (GAP == GAFFINE) ? V::shfl_up(Ebot, L) : NEG;
        uint32_t sel = __shfl_up_sync(0xffffffffu, selb, 1, L);
        const int col = k - t;
        const bool act = sact && col >= 0 && col < M;
        if (t == 0 && act) {
          if (st == 0) {
            hin = V::splat((KIND == KGLOBAL) ? -(P.go + (col + 1) * P.ge) : 0);  // H(0,j)
            ein = NEG;                                                             // E(0,j)
          } else {
            const uint2 v = scr[col];
            hin = (T)v.x;
            ein = (T)v.y;
          }
          uint32_t c0 = 0, c1 = 0;
          if (col < mm[0]) c0 = a.scode[so[0] + col];
          if (PP == 2 && col < mm[PP - 1]) c1 = a.scode[so[PP - 1] + col];
          sel = V::selector(c0, c1);
        }
        if (act) {
          T hup = V::add(hin, NOC);  // Hop of the row above
          T e = ein;
          T hd = diag;
          if (!TB) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const T sig = V::sigma(p0[r], p1[r], sel);
              T tm;
              if (GAP == GAFFINE) {
                e = V::addmax(e, NGE, hup);           // Eq. (4)
                Ff[r] = V::addmax(Ff[r], NGE, Ho[r]);  // Eq. (5)
                tm = V::vmax(e, Ff[r]);
              } else {
                tm = V::vmax(hup, Ho[r]);  // Eqs. (2)-(3): H_up - g, H_left - g
              }
              const T h = (KIND == KLOCAL) ? V::addmax_relu(hd, sig, tm) : V::addmax(hd, sig, tm);
              hd = Hh[r];
              Hh[r] = h;
              Ho[r] = V::add(h, NOC);
              hup = Ho[r];
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const T sig = V::sigma(p0[r], p1[r], sel);
              uint32_t pe = 0, pf = 0, pef, pd;
              T tm;
              if (GAP == GAFFINE) {
                e = V::bmax(V::add(e, NGE), hup, pe);              // eext: extend >= open (R8)
                Ff[r] = V::bmax(V::add(Ff[r], NGE), Ho[r], pf);    // fext
                tm = V::bmax(e, Ff[r], pef);                       // E before F (R7)
              } else {
                tm = V::bmax(hup, Ho[r], pef);
              }
              T h = V::bmax(V::add(hd, sig), tm, pd);              // DIAG first (R7)
              uint32_t stop = 0;
              if (KIND == KLOCAL) {
                // STOP where H <= 0 (nu wins ties, reading R9).  Not via bmax(0, h): ptxas
                // 12.9 swaps the operands of a VIMNMX-with-predicates against a constant
                // zero and the predicates then mean h >= 0.
                h = V::vmax_relu(h, h);
#pragma unroll
                for (int X = 0; X < PP; ++X) stop |= (V::get(h, X) == 0 ? 1u : 0u) << X;
              }
#pragma unroll
              for (int X = 0; X < PP; ++X) {
                uint32_t src = ((pd >> X) & 1u) ? 0u : (((pef >> X) & 1u) ? 1u : 2u);
                if ((stop >> X) & 1u) src = 3u;
                const uint32_t nib = src | (((pe >> X) & 1u) << 2) | (((pf >> X) & 1u) << 3);
                acc[r * PP + X] = (acc[r * PP + X] >> 4) | (nib << 28);
              }
              hd = Hh[r];
              Hh[r] = h;
              Ho[r] = V::add(h, NOC);
              hup = Ho[r];
            }
          }
          diag = hin;
          Hbot = Hh[R - 1];
          Ebot = e;
          selb = sel;
          if (t == L - 1 && st + 1 < NS) scr[col] = make_uint2((uint32_t)Hh[R - 1], (uint32_t)e);

          // ---- optimum bookkeeping ----
          if (KIND == KLOCAL) {
            T cm = Hh[0];
#pragma unroll
            for (int r = 1; r + 1 < R; r += 2) cm = V::vmax3(cm, Hh[r], Hh[r + 1]);
            if ((R % 2) == 0) cm = V::vmax(cm, Hh[R - 1]);
            uint32_t keep = 0;
#pragma unroll
            for (int X = 0; X < PP; ++X) keep |= (col < mm[X] ? 1u : 0u) << X;
            cm = V::select_mask(cm, keep, V::splat(0));
            if (!pos) {
              sbest = V::vmax(sbest, cm);
            } else {
              uint32_t pb;
              const T nb = V::bmax(sbest, cm, pb);  // bit: sbest >= cm
              if ((~pb) & ((1u << PP) - 1u)) {
#pragma unroll
                for (int X = 0; X < PP; ++X) {
                  if (!((pb >> X) & 1u)) {
                    const int v = V::get(cm, X);
                    int rr = R - 1;
#pragma unroll
                    for (int r = R - 1; r >= 0; --r)
                      if (V::get(Hh[r], X) == v) rr = r;
                    sv[X] = v;
                    si[X] = ip0 + rr - pad[X] + 1;
                    sj[X] = col + 1;
                  }
                }
              }
              sbest = nb;
            }
          } else if (KIND == KSEMI) {
            // bottom row n, columns j = 1..m-1 (row candidates precede column m, R5)
            uint32_t keep = 0;
            if (st == NS - 1) {
#pragma unroll
              for (int X = 0; X < PP; ++X) keep |= (col < mm[X] - 1 ? 1u : 0u) << X;
            }
            const T cand = V::select_mask(Hh[R - 1], keep, NEG);
            uint32_t pb;
            const T nb = V::bmax(best, cand, pb);
            if (pos) {
#pragma unroll
              for (int X = 0; X < PP; ++X)
                if (!((pb >> X) & 1u)) rj[X] = col + 1;
            }
            best = nb;
            // column m: rows i = 1..n at the step where this lane reaches column m
#pragma unroll
            for (int X = 0; X < PP; ++X) {
              if (col == mm[X] - 1) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                  const int i = ip0 + r - pad[X] + 1;
                  const int v = V::get(Hh[r], X);
                  if (i >= 1 && i <= nn[X] && v > cv[X]) { cv[X] = v; ci[X] = i; }
                }
              }
            }
          } else {  // global: H(n,m)
#pragma unroll
            for (int X = 0; X < PP; ++X) {
              if (col == mm[X] - 1) {
                const int ipn = nn[X] - 1;
                if (ipn >= 0 && st == ipn / HS && t == (ipn % HS) / R) {
                  const int rr = ipn % R;
                  int v = 0;
#pragma unroll
                  for (int r = 0; r < R; ++r)
                    if (r == rr) v = V::get(Hh[r], X);
                  gv[X] = v;
                }
              }
            }
          }
        } else if (TB) {
#pragma unroll
          for (int r = 0; r < R * PP; ++r) acc[r] >>= 4;
        }
        if (TB && valid && sact) {
          const int Kslot = M + L - 1;
          if (k < Kslot && ((k & 7) == 7 || k == Kslot - 1)) {
            const int sh = 4 * (7 - (k & 7));
            uint32_t* wp = a.dirs + dbase + ((((int64_t)st * S8 + (k >> 3)) * R) * L + t) * PP;
#pragma unroll
            for (int r = 0; r < R; ++r) {
#pragma unroll
              for (int X = 0; X < PP; ++X) wp[((int64_t)r * L) * PP + X] = acc[r * PP + X] >> sh;
            }
          }
        }
      }  // steps

      if (KIND == KLOCAL) {
        if (!pos) {
          best = V::vmax(best, sbest);
        } else {
#pragma unroll
          for (int X = 0; X < PP; ++X)
            if (key_better(sv[X], si[X], sj[X], bv[X], bi[X], bj[X])) {
              bv[X] = sv[X]; bi[X] = si[X]; bj[X] = sj[X];
            }
        }
      }
      __syncwarp();
    }  // strips

    // ---- reduce across the lane group and write results (P:424-436 steps 8, 10) ----
    int osc[PP], oi[PP], oj[PP];
#pragma unroll
    for (int X = 0; X < PP; ++X) {
      if (KIND == KLOCAL) {
        int v = pos ? bv[X] : V::get(best, X), i = bi[X], j = bj[X];
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
          const int v2 = __shfl_xor_sync(0xffffffffu, v, o, L);
          const int i2 = __shfl_xor_sync(0xffffffffu, i, o, L);
          const int j2 = __shfl_xor_sync(0xffffffffu, j, o, L);
          if (key_better(v2, i2, j2, v, i, j)) { v = v2; i = i2; j = j2; }
        }
        osc[X] = v; oi[X] = i; oj[X] = j;
      } else if (KIND == KSEMI) {
        int v = cv[X], i = ci[X];
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
          const int v2 = __shfl_xor_sync(0xffffffffu, v, o, L);
          const int i2 = __shfl_xor_sync(0xffffffffu, i, o, L);
          if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
        }
        const int rv = __shfl_sync(0xffffffffu, V::get(best, X), L - 1, L);
        const int rjj = __shfl_sync(0xffffffffu, rj[X], L - 1, L);
        if (rv >= v) { osc[X] = rv; oi[X] = nn[X]; oj[X] = rjj; }
        else { osc[X] = v; oi[X] = i; oj[X] = mm[X]; }
      } else {
        const int ipn = max(nn[X] - 1, 0);
        const int owner = (ipn % HS) / R;
        osc[X] = __shfl_sync(0xffffffffu, gv[X], owner, L);
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
          ti.slot_M = M;
          ti.ns = NS;
          ti.half = (int16_t)X;
          ti.L = (int16_t)L;
          ti.R = (int16_t)R;
          ti.P = (int16_t)PP;
          ti.pad = pad[X];
          ti.score = osc[X];
          ti.end_i = oi[X];
          ti.end_j = oj[X];
          a.tb[pr[X]] = ti;
        }
      }
    }
  }  // slots
}

}  // namespace anyseq
