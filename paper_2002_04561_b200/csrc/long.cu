// csrc/long.cu -- long-pair score-only alignment: persistent tiled wavefront.
//
// Paper: tiles relaxed along anti-diagonals, borders handed to the right/below neighbours
// (Fig. 2), GPU tiles split into stripes whose last row is kept and
// reused (Fig. 4 caption P:531-537), dynamic scheduling of ready tiles
// (P:492).
//
// B200 design: the matrix is cut into row strips of 32*R rows
// (one warp: lane t owns R rows, anti-diagonal wavefront across lanes as in the batch
// kernel) and G column strips.  Warps take tasks (row strip s, column strip g) in ticket
// order (s-major), so every task waits only on lower tickets held by resident warps:
// deadlock-free.  Handoffs:
//   * row strip s -> s+1 (same column strip): an O(m) in-place row buffer (H,E) in global
//     memory (L2-resident for 5 Mbp) plus a per-task progress counter published every
//     `chunk` columns with st.release.gpu and polled with ld.acquire.gpu;
//   * column strip g -> g+1: the right-edge column (H,F) for all rows of the task plus a
//     per-(edge, row strip) flag published with a system-scope fence, so the same code
//     runs with the consumer on another GPU (peer pointer over NVLink) or on the same GPU
//     ("virtual strips" -- the multi-GPU protocol exercised on one device).
// Every spin-wait is bounded and raises an abort flag (-> ANYSEQ_E_TIMEOUT).
#include <algorithm>
#include <chrono>
#include <cstring>
#include <cstdio>
#include <type_traits>
#include "../../include/anyseq.h"
#include "kernels.h"
#include "long.h"
#include "long_dev.cuh"

namespace anyseq {

template <int KIND, int GAP, int R>
__global__ void __launch_bounds__(128) long_kernel(LongArgs a) {
  typedef VS32 V;
  constexpr int L = 32;
  constexpr int HS = L * R;
  constexpr bool FAST = GAP == GAFFINE;  // reassociated affine recurrence (see fill_kernel.cuh)
  constexpr int RING = 256;              // per-warp ring of lane-0 inputs and selectors
  constexpr int PER = 32;                // refill period (steps)
  __shared__ int2 ring_he[4][RING];
  __shared__ uint16_t ring_sel[4][RING];
  const int t = threadIdx.x & 31;
  const int wb = threadIdx.x >> 5;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const DevParams P = a.P;  // copy: hot-loop constants in registers
  const int NEG = NEG32;
  const int NGE = -P.ge;
  const int cop = (GAP == GAFFINE) ? (P.go + P.ge) : P.ge;
  const uint32_t one = (uint32_t)a.one;
  const uint32_t k32 = one << 5;  // 32, opaque to the compiler: key = H * 32 + row stays an IMAD
  auto hop = [&](int h) -> int { return imad_add_s(h, one, -cop); };  // FMA pipe
  const int n = a.n, m = a.m;
  // semi/global: where row n lives inside the last row strip
  const int tn = ((n - 1) % HS) / R, rn = (n - 1) % R;

  LongPart part;
  part.lv = 0; part.li = 0; part.lj = 0;
  part.rv = 0; part.rj = 0;  // (n, 0) = 0 is the first semi-global candidate
  part.cv = 0; part.ci = 0;  // (0, m) = 0
  part.gv = 0; part.gset = 0; part.pad_ = 0;

  for (;;) {
    int task = 0;
    if (t == 0) task = atomicAdd(a.ticket, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= a.S * a.g_count) break;
    if (*(volatile int*)a.abort_flag) break;
    if (task == a.stall_task) continue;  // fault injection (option long_stall_task)
    const long long task_t0 = (a.prof && t == 0) ? clock64() : 0;
    // column-strip major: task (s, g) waits on (s-1, g) (row hand-off) and (s, g-1) (left
    // edge, finished a whole pass earlier) -- both lower tickets held by resident warps
    const int s = task % a.S;
    const int g = a.g_first + task / a.S;
    const int c_lo = a.cb[g], c_hi = a.cb[g + 1], W = c_hi - c_lo;
    const bool last_strip = (s == a.S - 1), last_col = (c_hi == m);
    const int ip0 = s * HS + t * R;
    const int2* bl = a.bcol[g];
    int2* br = (g + 1 < a.Gtot) ? a.bcol[g + 1] : nullptr;

    if (g > 0) {  // left boundary of this row strip (and the previous one: diag of row 0)
      if (!warp_wait<true>(&a.bflag[g][s], 1, a)) break;
      if (s > 0 && !warp_wait<true>(&a.bflag[g][s - 1], 1, a)) break;
    }
    uint32_t p0[R], p1[R];
    int HA[R], HB[R], Ff[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int ip = ip0 + r;
      const bool real = ip < n;
      const uint32_t c = real ? a.qc[ip] : 0u;
      p0[r] = real ? prof4(a.P, c) : 0u;  // indexed from the parameter bank, not the copy
      p1[r] = real ? pn_of(a.P, c) : 0u;  // byte 4 of the profile: sigma(q_i, N)
      HA[r] = HB[r] = 0;
      Ff[r] = NEG;
    }
    // lane-0 inputs and selectors of columns [c0, c1) (c1 - c0 <= 32: one per lane) into
    // the warp's ring; the row entries are polled until they carry this strip's tag s
    // (written by strip s-1), bounded like every wait (-> abort, ANYSEQ_E_TIMEOUT)
    auto refill = [&](int c0, int c1) -> bool {
      const int c = c0 + t;
      const bool mine = c < c1;
      if (mine) ring_sel[wb][c & (RING - 1)] = (uint16_t)V::selector(a.sc[c_lo + c], 0);
      if (s == 0) return true;
      const int4* src = a.rowbuf + c_lo + c + 1;
      int4 v = mine ? ld_row(src) : make_int4(0, s, 0, s);
      long long spins = 0;
      while (!__all_sync(0xffffffffu, v.y == s && v.w == s)) {
        const long long t0 = (a.prof && t == 0) ? clock64() : 0;
        __nanosleep(64);
        if (v.y != s || v.w != s) v = ld_row(src);
        if ((++spins & 255) == 0 &&
            __any_sync(0xffffffffu, spins > a.spin_limit || *(volatile int*)a.abort_flag)) {
          if (t == 0) atomicExch(a.abort_flag, 1);
          return false;
        }
        if (a.prof && t == 0) atomicAdd(&a.prof[0], (unsigned long long)(clock64() - t0));
      }
      if (mine) ring_he[wb][c & (RING - 1)] = make_int2(v.x, v.z);
      return true;
    };
    if (!refill(0, min(W, PER)) || !refill(PER, min(W, 2 * PER))) break;
    __syncwarp();

    int diag = 0, Hbot = NEG, Ebot = NEG;
    int sv = 0, si = 0, sj = 0;  // local per task
    int skey = 0;                // keyed local tracking: best (H << 5 | 31 - r) of this lane

    // FIRST: the task's row strip is the matrix's first (lane 0 reads H(0, j) directly);
    // KEYED: local maximum tracked as one packed key per lane (value, first row) -- no
    // per-step row search (host sets a.keyed when 32 * max score fits in 31 bits).
    auto sweep = [&](auto first_c, auto keyed_c) -> bool {
      constexpr bool FIRST = decltype(first_c)::value;
      constexpr bool KEYED = decltype(keyed_c)::value;
      uint32_t sel_nx = 0;
      int2 he_nx = make_int2(0, 0);
      auto step = [&](auto chk, const int k, int (&Hi)[R], int (&Hq)[R]) {
        constexpr bool CHK = decltype(chk)::value;
        int hin = V::shfl_up(Hbot, L);
        int ein = V::shfl_up(Ebot, L);
        const int lc = k - t;
        // this step's selector / lane-0 input were loaded one step ahead (the ring holds
        // columns up to the next refill point, see maybe_refill)
        const uint32_t sel = sel_nx;
        const int2 he = he_nx;
        sel_nx = ring_sel[wb][(lc + 1) & (RING - 1)];
        if (!FIRST) he_nx = ring_he[wb][(lc + 1) & (RING - 1)];
        const bool act = !CHK || (lc >= 0 && lc < W);
        if (CHK && lc == 0) {  // the left boundary column H(i, c_lo), F(i, c_lo)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int ip = ip0 + r;
            int2 b = make_int2(0, NEG);
            if (ip < n) b = bl[ip + 1];
            Hi[r] = b.x;
            Ff[r] = b.y;
          }
          diag = (ip0 <= n) ? bl[ip0].x : 0;
        }
        if (t == 0) {
          if (FIRST) {
            const int h0 = (KIND == KGLOBAL) ? -(P.go + (c_lo + lc + 1) * P.ge) : 0;  // H(0,j)
            hin = h0;
            ein = FAST ? hop(h0) : NEG;
          } else {
            hin = he.x;
            ein = he.y;
          }
        }
        int e = ein;
        if (FAST) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int hd = (r == 0) ? diag : Hi[r - 1];
            const int sig = V::sigma(p0[r], p1[r], sel);
            Ff[r] = V::addmax(Ff[r], NGE, hop(Hi[r]));
            const int df = V::addmax(hd, sig, Ff[r]);
            Hq[r] = (KIND == KLOCAL) ? V::vmax_relu(df, e) : max(df, e);
            e = V::addmax(e, NGE, hop(df));
          }
        } else {
          int hup = hop(hin);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int hd = (r == 0) ? diag : Hi[r - 1];
            const int sig = V::sigma(p0[r], p1[r], sel);
            const int tm = max(hup, hop(Hi[r]));
            Hq[r] = (KIND == KLOCAL) ? V::addmax_relu(hd, sig, tm) : V::addmax(hd, sig, tm);
            hup = hop(Hq[r]);
          }
          e = NEG;
        }
        diag = hin;
        Hbot = Hq[R - 1];
        Ebot = e;
        if (t == L - 1 && act) st_row(a.rowbuf + c_lo + lc + 1, Hq[R - 1], e, s + 1);  // strip s+1
        const int j = c_lo + lc + 1;  // real column
        if (KIND == KLOCAL && KEYED) {
          // rows below n (last strip) never win: their values come from real cells of an
          // earlier column (sigma = 0 diagonal) or are strictly smaller (gaps), and the
          // (value, j, i) order prefers the earlier column / smaller row (reading R10)
          int key = imad_add_s(Hq[0], k32, 31);
#pragma unroll
          for (int r = 1; r + 1 < R; r += 2)
            key = V::vmax3(key, imad_add_s(Hq[r], k32, 31 - r), imad_add_s(Hq[r + 1], k32, 30 - r));
          if ((R % 2) == 0) key = max(key, imad_add_s(Hq[R - 1], k32, 32 - R));
          if (CHK && !act) key = 0;
          // a strictly larger value (the key's row part only orders rows of one column)
          if (key > (skey | 31)) { skey = key; sj = j; }
        } else if (KIND == KLOCAL) {
          int cm = 0;
          if (!last_strip) {
            cm = Hq[0];
#pragma unroll
            for (int r = 1; r + 1 < R; r += 2) cm = V::vmax3(cm, Hq[r], Hq[r + 1]);
            if ((R % 2) == 0) cm = max(cm, Hq[R - 1]);
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (ip0 + r < n) cm = max(cm, Hq[r]);
          }
          if (CHK && !act) cm = 0;
          if (cm > sv) {
            int rr = R - 1;
#pragma unroll
            for (int r = R - 1; r >= 0; --r)
              if (Hq[r] == cm && ip0 + r < n) rr = r;
            sv = cm;
            si = ip0 + rr + 1;
            sj = j;
          }
        } else if (KIND == KSEMI) {
          if (last_strip && t == tn && act && j <= m - 1) {
            int v = 0;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (r == rn) v = Hq[r];
            if (v > part.rv || (v == part.rv && j < part.rj)) { part.rv = v; part.rj = j; }
          }
        }
        if (CHK && lc == W - 1) {  // a lane's last column of this task
          if (KIND == KSEMI && last_col) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int i = ip0 + r + 1;
              if (i <= n && (Hq[r] > part.cv || (Hq[r] == part.cv && i < part.ci))) {
                part.cv = Hq[r];
                part.ci = i;
              }
            }
          }
          if (KIND == KGLOBAL && last_strip && last_col && t == tn) {
            int v = 0;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (r == rn) v = Hq[r];
            part.gv = v;
            part.gset = 1;
          }
          if (br) {
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (ip0 + r < n) br[ip0 + r + 1] = make_int2(Hq[r], Ff[r]);
          }
        }
      };

      const std::integral_constant<bool, true> ON{};
      const std::integral_constant<bool, false> OFF{};
      const int K = W + L - 1;
      sel_nx = ring_sel[wb][(0 - t) & (RING - 1)];
      if (!FIRST) he_nx = ring_he[wb][(0 - t) & (RING - 1)];
      const int kA = min(K & ~1, L);               // every lane has reached column 0
      const int kB = max(kA, (W - 1) & ~1);        // no lane has reached column W-1 yet
      int k = 0;
      auto maybe_refill = [&](int kk) -> bool {  // warp-uniform, every PER steps
        if ((kk % PER) == 0 && kk > 0 && kk + PER < W) {
          if (!refill(kk + PER, min(W, kk + 2 * PER))) return false;
          __syncwarp();
        }
        return true;
      };
      for (; k < kA; k += 2) {
        if (!maybe_refill(k)) return false;
        step(ON, k, HA, HB);
        step(ON, k + 1, HB, HA);
      }
      for (; k < kB; k += 2) {
        if (!maybe_refill(k)) return false;
        step(OFF, k, HA, HB);
        step(OFF, k + 1, HB, HA);
      }
      for (; k + 1 < K; k += 2) {
        if (!maybe_refill(k)) return false;
        step(ON, k, HA, HB);
        step(ON, k + 1, HB, HA);
      }
      if (k < K) step(ON, k, HA, HB);
      if (KIND == KLOCAL && KEYED && skey > 0) {
        sv = skey >> 5;
        si = ip0 + (31 - (skey & 31)) + 1;
      }
      return true;
    };
    bool done;
    if (s == 0) {
      done = (KIND == KLOCAL && a.keyed) ? sweep(std::true_type{}, std::true_type{})
                                          : sweep(std::true_type{}, std::false_type{});
    } else {
      done = (KIND == KLOCAL && a.keyed) ? sweep(std::false_type{}, std::true_type{})
                                          : sweep(std::false_type{}, std::false_type{});
    }
    if (!done) break;
    if (KIND == KLOCAL && lkey_better(sv, si, sj, part.lv, part.li, part.lj)) {
      part.lv = sv; part.li = si; part.lj = sj;
    }
    if (a.prof && t == 0) {
      atomicAdd(&a.prof[1], (unsigned long long)(clock64() - task_t0));
      atomicAdd(&a.prof[2], 1ull);
    }
    __syncwarp();
    if (br) {
      if (t == 0) {
        __threadfence_system();
        st_release_sys(&a.bflag[g + 1][s], 1);
      }
    }
  }
  // reduce the warp's lanes (keys per reading R10 / R5) and publish
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int lv = __shfl_xor_sync(0xffffffffu, part.lv, o);
    const int li = __shfl_xor_sync(0xffffffffu, part.li, o);
    const int lj = __shfl_xor_sync(0xffffffffu, part.lj, o);
    if (lkey_better(lv, li, lj, part.lv, part.li, part.lj)) { part.lv = lv; part.li = li; part.lj = lj; }
    const int rv = __shfl_xor_sync(0xffffffffu, part.rv, o);
    const int rj = __shfl_xor_sync(0xffffffffu, part.rj, o);
    if (rv > part.rv || (rv == part.rv && rj < part.rj)) { part.rv = rv; part.rj = rj; }
    const int cv = __shfl_xor_sync(0xffffffffu, part.cv, o);
    const int ci = __shfl_xor_sync(0xffffffffu, part.ci, o);
    if (cv > part.cv || (cv == part.cv && ci < part.ci)) { part.cv = cv; part.ci = ci; }
    const int gv = __shfl_xor_sync(0xffffffffu, part.gv, o);
    const int gs = __shfl_xor_sync(0xffffffffu, part.gset, o);
    if (gs && !part.gset) { part.gv = gv; part.gset = 1; }
  }
  if (t == 0) a.parts[wg] = part;
}



// SEMI optimum after a 16-bit long kernel (reading R5): candidates (n, j) for j in
// [j0, j1) ∩ [1, m-1] from the row buffer (the last row strip's published row = row n),
// then -- on the device owning column m -- (i, m) for i = 0..n from the boundary column the
// last strip wrote.  Key = (value, then the earliest candidate: seq = j for row n, m + i for
// column m); strict '>' in that order = the largest key with the smallest seq.  (n, 0) = 0
// is merged on the host.
__global__ void semi_reduce_kernel(const int4* __restrict__ rowbuf, int j0, int j1, int m,
                                   const int2* __restrict__ colm, int n,
                                   unsigned long long* out) {
  unsigned long long best = 0;
  const int64_t nrow = j1 > j0 ? j1 - j0 : 0;
  const int64_t tot = nrow + (colm ? (int64_t)n + 1 : 0);
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < tot;
       x += (int64_t)gridDim.x * blockDim.x) {
    int v;
    uint32_t seq;
    if (x < nrow) {
      const int j = j0 + (int)x;
      v = rowbuf[j].x;
      seq = (uint32_t)j;
    } else {
      const int i = (int)(x - nrow);
      v = colm[i].x;
      seq = (uint32_t)m + (uint32_t)i;
    }
    const unsigned long long key =
        ((unsigned long long)((uint32_t)v ^ 0x80000000u) << 32) | (0xFFFFFFFFu - seq);
    best = key > best ? key : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y > best ? y : best;
  }
  if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

__global__ void long_init_kernel(DevParams P, int n, int m, int4* rowbuf, int2* bcol0,
                                 int2* const* bcol, const int* cb, int Gtot, int g_first,
                                 int g_count) {
  const int NEG = NEG32;
  const bool glob = P.kind == KGLOBAL;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x <= (int64_t)max(n, m);
       x += (int64_t)gridDim.x * blockDim.x) {
    if (x <= m) rowbuf[x] = make_int4(0, 0, NEG, 0);  // tag 0: no strip has written yet
    if (bcol0 && x <= n) bcol0[x] = make_int2(glob && x > 0 ? -(P.go + (int)x * P.ge) : 0, NEG);  // H(i,0), F(i,0)
    if (x == 0) {
      for (int g = g_first; g <= g_first + g_count; ++g) {
        // the group's own edges; plus column m (edge Gtot) when the group keeps it (SEMI)
        if (g == 0 || (g == g_first + g_count && !(g == Gtot && bcol[g]))) continue;
        const int c = cb[g];
        bcol[g][0] = make_int2(glob ? -(P.go + c * P.ge) : 0, NEG);  // H(0, c_g)
      }
    }
  }
}

template <int R>
static LongFn long_fn(int kind, int gap) {
  if (kind == KGLOBAL) return gap ? long_kernel<KGLOBAL, GAFFINE, R> : long_kernel<KGLOBAL, GLINEAR, R>;
  if (kind == KLOCAL) return gap ? long_kernel<KLOCAL, GAFFINE, R> : long_kernel<KLOCAL, GLINEAR, R>;
  return gap ? long_kernel<KSEMI, GAFFINE, R> : long_kernel<KSEMI, GLINEAR, R>;
}

namespace {
struct Buf {
  void* p = nullptr;
  bool own = true;
  ~Buf() { if (p && own) cudaFree(p); }
};
// a buffer from the device's persistent workspace slot, or a call-local allocation
cudaError_t get_buf(Buf& b, LongWs* ws, int slot, size_t bytes) {
  if (ws) {
    b.own = false;
    return ws->get(slot, bytes, &b.p);
  }
  b.own = true;
  return cudaMalloc(&b.p, bytes < 256 ? 256 : bytes);
}
#define LK(call)                                                      \
  do {                                                                \
    cudaError_t e_ = (call);                                          \
    if (e_ != cudaSuccess) {                                          \
      *err = std::string(#call) + ": " + cudaGetErrorString(e_);      \
      return e_ == cudaErrorMemoryAllocation ? ANYSEQ_E_NOMEM : ANYSEQ_E_CUDA; \
    }                                                                 \
  } while (0)
}  // namespace

void LongCkpt::release() {
  if (owns)
    for (void* p : {(void*)qc, (void*)sc, (void*)rowck, (void*)colck})
      if (p) cudaFree(p);
  qc = sc = nullptr;
  rowck = colck = nullptr;
  bytes = 0;
}

int run_long(std::vector<LongDevice>& devs, const DevParams& P, const char* q, uint64_t n,
             const char* s, uint64_t m, const LongOptions& opt, LongResult* out, std::string* err,
             uint64_t* launches, LongCkpt* ck) {
  out->kernel_ms = 0;
  out->narrow = false;
  if (n == 0 || m == 0) {  // empty sequences: one gap run (global) or the empty alignment
    const int64_t len = (int64_t)(n + m);
    out->score = (P.kind == KGLOBAL && len) ? (int32_t)(-(P.go + len * P.ge)) : 0;
    out->end_i = P.kind == KGLOBAL ? (int64_t)n : 0;
    out->end_j = P.kind == KGLOBAL ? (int64_t)m : 0;
    return 0;
  }
  {  // 32-bit range guard (reading R11)
    const long double neg = 3.0L * P.go + ((long double)n + m + 2) * P.ge + 256;
    const long double pos = (long double)std::max(P.smax, 0) * std::min(n, m);
    if (neg > (1u << 30) - (1u << 24) || pos > (1u << 30) - (1u << 24)) {
      *err = "score range exceeds 32-bit arithmetic";
      return ANYSEQ_E_UNSUPPORTED;
    }
  }
  // Devices: one column strip per context entry; consecutive entries naming the same GPU
  // form one group that runs its strips in ONE launch (column-strip-major tickets, the
  // virtual-strip protocol) -- kernels that wait on each other are never launched side by
  // side on one GPU (they need not be co-scheduled).  A GPU named twice non-adjacently is
  // rejected for the same reason.
  const int NE = (int)devs.size();
  std::vector<int> gfirst, gcount;  // per group: first entry (= first strip), entries
  for (int e = 0; e < NE; ++e) {
    if (e > 0 && devs[e].id == devs[e - 1].id) { ++gcount.back(); continue; }
    for (int f = 0; f < e; ++f)
      if (devs[f].id == devs[e].id) {
        *err = "long pairs: device " + std::to_string(devs[e].id) +
               " is listed twice non-adjacently (its strips must run in one launch)";
        return ANYSEQ_E_INVALID;
      }
    gfirst.push_back(e);
    gcount.push_back(1);
  }
  const int ND = (int)gfirst.size();  // distinct devices (groups)
  // rows per lane: 16 (168 registers, 3 blocks/SM; default) or 12 (128 registers, 4
  // blocks/SM; option long_band_rows = 384) -- measured equal within noise on C4
  const int R = opt.band_rows == 384 ? 12 : 16;
  int HS = 32 * R;
  LongFn fn = R == 16 ? long_fn<16>(P.kind, P.gap) : long_fn<12>(P.kind, P.gap);
  // 16-bit differential kernel (long16.cuh): local affine, subject without
  // N (the s16x2 selector has no fifth byte), and the relative frame of DESIGN.md §5.4b:
  // every value of a task window within bspan = (rows + 66) * d of one reference cell
  // (d = G_o + G_e + max sigma bounds |H(x) - H(y)| per unit of Manhattan distance),
  // 2 bspan + margin (drift over 96 steps between re-basings) + slack inside the s16 range
  // above the relative -inf.
  const int64_t d16 = (int64_t)P.go + P.ge + std::max(P.smax, 0);
  const int64_t margin16 = 100 * d16 + 16;
  const int NEG16C = -24576;
  auto fits16 = [&](int nr) {
    return 2 * (int64_t)(64 * nr + 66) * d16 + margin16 + 96 * d16 + P.go + P.ge + 256 < -NEG16C;
  };
  // 1024-row tasks by default, 512 if the range guard needs it -- or across >= 4 devices:
  // a device keeps (resident warps x rows per task) rows in flight, and the last of G
  // devices trails the first by G - 1 such pipelines (tools/scaling_model.py)
  int NR16 = (opt.band_rows == 512 || (opt.band_rows == 0 && NE >= 4)) ? 8 : 16;  // (range
  if (NR16 > 8 && !fits16(NR16)) NR16 = 8;    // guard needs it
  if (NR16 > 8 && opt.band_rows == 0) {
    // short pairs: fewer 1024-row strips than ~1.5x the resident warps leave warps idle
    // through the first pass of every column strip -- 512-row strips double the strips
    int nb = 0;
    cudaSetDevice(devs[0].id);
    LK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, long16_fn(16, P.kind, ck && ck->want), 128, 0));
    const double warps = 4.0 * devs[0].num_sms * std::max(nb, 1);
    if ((double)((n + 1023) / 1024) < 1.5 * warps) NR16 = 8;
  }
  const int64_t bspan16 = (int64_t)(64 * NR16 + 66) * d16;
  // every kind and gap model (linear = affine with G_o = 0, exact for scores); the subject's
  // selector has four codes, so a subject with N takes the 32-bit kernel
  bool narrow = opt.narrow != 0 && fits16(NR16) && (int64_t)P.go + 2 * P.ge < 4096;
  if (narrow)
    for (uint64_t x = 0; x < m && narrow; ++x) narrow = (s[x] | 0x20) != 'n';
  if (narrow) {
    HS = 64 * NR16;
    fn = long16_fn(NR16, P.kind, ck && ck->want);
  }
  out->narrow = narrow;
  if (ck && ck->want && (!narrow || NE != 1)) {
    *err = narrow ? "long traceback: one device only"
                  : "long traceback: needs the 16-bit kernel (subject without N, range guard)";
    return ANYSEQ_E_UNSUPPORTED;
  }
  const int S = (int)((n + HS - 1) / HS);
  int Gtot = NE > 1 ? NE : std::max(1, opt.virtual_strips);
  if (NE == 1 && opt.virtual_strips <= 0) {
    // Auto: every task spans its column strip, so the last round of S*G tasks over W
    // resident warps idles the rest; G column passes (tickets column-strip major, so a
    // task's left edge was finished a pass earlier) shrink that round's share.
    int nb = 0;
    cudaSetDevice(devs[0].id);
    LK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 128, 0));
    int grid = devs[0].num_sms * std::max(nb, 1);
    if (opt.blocks > 0) grid = std::min(grid, opt.blocks);
    const double W = 4.0 * grid;
    double best = -1;
    for (int G = 1; G <= 8; ++G) {
      const double rounds = S * (double)G / W;
      const double score = rounds / std::ceil(rounds) - 0.005 * (G - 1);
      if (score > best + 1e-9) { best = score; Gtot = G; }
    }
  }
  if (NE > 1 && (uint64_t)Gtot > m) {
    *err = "long pairs: more devices than subject columns";
    return ANYSEQ_E_INVALID;
  }
  Gtot = (int)std::min<uint64_t>(Gtot, m);
  std::vector<int32_t> cb(Gtot + 1);
  for (int g = 0; g <= Gtot; ++g) cb[g] = (int32_t)((m * (uint64_t)g) / Gtot);
  int chunk = 8;  // power of two (the kernel masks with chunk - 1)
  while (chunk < opt.chunk_cols && chunk < (1 << 20)) chunk <<= 1;  // publication period

  struct PerDev {
    Buf qa, sa, qc, sc, rowbuf, bcol_own, prog, flags, ticket, abort_, parts, cbuf, bptr, fptr, sum, flg, profbuf;
    int g_first = 0, g_count = 0, grid = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
  };
  std::vector<PerDev> pd(ND);
  std::vector<int2*> bcol_ptr(Gtot + 1, nullptr);  // edge g buffer lives on its consumer device
  const int pad_top = (narrow && P.kind == KSEMI) ? (int)((uint64_t)S * HS - n) : 0;
  // checkpoint geometry: row checkpoints every ck_every strips (row blocks of HS * ck_every
  // <= 4096 rows), column checkpoints every 2^kc_shift columns (<= 4096), the finest that
  // fits the budget (the traceback's tile recompute shrinks with the tile)
  if (ck && ck->want) {
    size_t fr = 0, tot = 0;
    LK(cudaSetDevice(devs[0].id));
    LK(cudaMemGetInfo(&fr, &tot));
    const int64_t budget = ck->budget > 0 ? ck->budget : (int64_t)(0.4 * (double)fr);
    auto bytes_of = [&](int every, int kcs) -> int64_t {
      const int64_t rows = (int64_t)(S - 1) / every, cols = (int64_t)(m - 1) >> kcs;
      return (rows * (int64_t)(m + 1) + cols * (int64_t)(n + 1)) * (int64_t)sizeof(int2);
    };
    // the walk's tiles are recomputed by helper CTAs (~(n·KC + m·TH)/2 cells), the pass
    // writes the checkpoints (bytes ~ n·m·8·(1/TH + 1/KC)): 512-column blocks balance the
    // two (1 Mbp, 512-row strips: KC 256 / 512 / 1024 / 2048 -> 1095 / 726 / 728 / 876 ms)
    const int cands[][2] = {{1, 9}, {1, 10}, {1, 11}, {2, 11}, {2, 12}, {4, 12}, {8, 12}};
    int every = 0, kcs = 0;
    for (auto& c : cands) {
      if (HS * c[0] > 4096) continue;
      if (bytes_of(c[0], c[1]) <= budget) { every = c[0]; kcs = c[1]; break; }
    }
    if (ck->force_ck_every > 0) every = ck->force_ck_every;
    if (ck->force_kc_shift > 0) kcs = ck->force_kc_shift;
    if (every == 0) {
      *err = "long traceback: checkpoints exceed the device memory budget";
      return ANYSEQ_E_NOMEM;
    }
    ck->release();
    ck->HS = HS;
    ck->ck_every = every;
    ck->kc_shift = kcs;
    ck->PT = pad_top;
    ck->S = S;
    const int64_t rows = (int64_t)(S - 1) / every, cols = (int64_t)(m - 1) >> kcs;
    ck->bytes = (size_t)bytes_of(every, kcs);
    LongWs* ws = devs[0].ws;
    ck->owns = ws == nullptr;
    if (rows > 0) {
      void* p = nullptr;
      LK(ws ? ws->get(WS_ROWCK, (size_t)rows * (m + 1) * sizeof(int2), &p)
            : cudaMalloc(&p, (size_t)rows * (m + 1) * sizeof(int2)));
      ck->rowck = (int2*)p;
    }
    if (cols > 0) {
      void* p = nullptr;
      LK(ws ? ws->get(WS_COLCK, (size_t)cols * (n + 1) * sizeof(int2), &p)
            : cudaMalloc(&p, (size_t)cols * (n + 1) * sizeof(int2)));
      ck->colck = (int2*)p;
    }
  }
  std::vector<int32_t*> flag_ptr(Gtot + 1, nullptr);
  // column strips per device group (one strip per entry; a single entry: all Gtot strips)
  std::vector<LongDevice> gdev(ND);
  for (int d = 0; d < ND; ++d) {
    gdev[d] = devs[gfirst[d]];
    pd[d].g_first = NE > 1 ? gfirst[d] : 0;
    pd[d].g_count = NE > 1 ? gcount[d] : Gtot;
  }
  // peer access between neighbouring groups (distinct devices by construction): the producer
  // of edge g stores into the consumer's column buffer and flags
  for (int d = 0; d + 1 < ND; ++d) {
    int ok = 0;
    LK(cudaDeviceCanAccessPeer(&ok, gdev[d].id, gdev[d + 1].id));
    if (!ok) {
      *err = "peer access unavailable between devices " + std::to_string(gdev[d].id) + " and " +
             std::to_string(gdev[d + 1].id);
      return ANYSEQ_E_PEER;
    }
    cudaSetDevice(gdev[d].id);
    cudaError_t e = cudaDeviceEnablePeerAccess(gdev[d + 1].id, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) LK(e);
    cudaGetLastError();
  }
  // allocation + upload + pack
  for (int d = 0; d < ND; ++d) {
    PerDev& D = pd[d];
    LK(cudaSetDevice(gdev[d].id));
    cudaStream_t st = gdev[d].stream;
    LK(get_buf(D.qa, gdev[d].ws, WS_QA, n + 16));
    LK(get_buf(D.sa, gdev[d].ws, WS_SA, m + 16));
    LK(get_buf(D.qc, gdev[d].ws, WS_QC, n + 16));
    LK(get_buf(D.sc, gdev[d].ws, WS_SC, m + 16));
    LK(get_buf(D.sum, gdev[d].ws, WS_SUM, sizeof(PlanSummary)));
    LK(get_buf(D.flg, gdev[d].ws, WS_FLG, 16));
    LK(cudaMemcpyAsync(D.qa.p, q, n, cudaMemcpyHostToDevice, st));
    LK(cudaMemcpyAsync(D.sa.p, s, m, cudaMemcpyHostToDevice, st));
    PlanSummary hs;
    memset(&hs, 0, sizeof(hs));
    hs.err_pos = ~0ull;
    LK(cudaMemcpyAsync(D.sum.p, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));
    LK(cudaStreamSynchronize(st));
    uint64_t offs[4] = {0, n, 0, m};
    Buf off;
    LK(get_buf(off, gdev[d].ws, WS_OFF, 32));
    LK(cudaMemcpy(off.p, offs, 32, cudaMemcpyHostToDevice));
    LK(launch_pack((const char*)D.qa.p, n, (uint8_t*)D.qc.p, (const uint64_t*)off.p,
                   (const char*)D.sa.p, m, (uint8_t*)D.sc.p, (const uint64_t*)off.p + 2, 1,
                   (uint32_t*)D.flg.p, (PlanSummary*)D.sum.p, st, gdev[d].num_sms));
    *launches += 1;
    LK(cudaMemcpyAsync(&hs, D.sum.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    LK(cudaStreamSynchronize(st));
    if (hs.err_pos != ~0ull) {
      const bool in_s = hs.err_pos >= (1ull << 62);
      *err = std::string("invalid symbol at ") + (in_s ? "s" : "q") + " offset " +
             std::to_string(in_s ? hs.err_pos - (1ull << 62) : hs.err_pos);
      return ANYSEQ_E_BADSEQ;
    }
    LK(get_buf(D.rowbuf, gdev[d].ws, WS_ROWBUF, (m + 1) * sizeof(int4)));
    LK(get_buf(D.prog, gdev[d].ws, WS_PROG, (size_t)Gtot * S * 4));
    LK(get_buf(D.ticket, gdev[d].ws, WS_TICKET, 4));
    LK(get_buf(D.abort_, gdev[d].ws, WS_ABORT, 4));
    LK(get_buf(D.cbuf, gdev[d].ws, WS_CB, (Gtot + 1) * 4));
    LK(get_buf(D.bptr, gdev[d].ws, WS_BPTR, (Gtot + 1) * sizeof(int2*)));
    LK(get_buf(D.fptr, gdev[d].ws, WS_FPTR, (Gtot + 1) * sizeof(int32_t*)));
    LK(cudaMemsetAsync(D.prog.p, 0, (size_t)Gtot * S * 4, st));
    LK(cudaMemsetAsync(D.ticket.p, 0, 4, st));
    LK(cudaMemsetAsync(D.abort_.p, 0, 4, st));
    LK(cudaMemcpyAsync(D.cbuf.p, cb.data(), (Gtot + 1) * 4, cudaMemcpyHostToDevice, st));
    // column buffers consumed on this device: edges g_first .. g_first+g_count-1 (edge 0 = init)
    if (D.g_count > 0) {
      // 16-bit SEMI: the group owning the last column strip also keeps column m (H(i, m),
      // written by the last strip's right edge) for the optimum's column candidates
      const int extra = (narrow && P.kind == KSEMI && D.g_first + D.g_count == Gtot) ? 1 : 0;
      const size_t bytes = (size_t)(D.g_count + extra) * (n + 1) * sizeof(int2);
      LK(get_buf(D.bcol_own, gdev[d].ws, WS_BCOL, bytes));
      for (int k = 0; k < D.g_count + extra; ++k)
        bcol_ptr[D.g_first + k] = (int2*)D.bcol_own.p + (size_t)k * (n + 1);
      LK(get_buf(D.flags, gdev[d].ws, WS_FLAGS, (size_t)D.g_count * S * 4));
      LK(cudaMemsetAsync(D.flags.p, 0, (size_t)D.g_count * S * 4, st));
      for (int k = 0; k < D.g_count; ++k) flag_ptr[D.g_first + k] = (int32_t*)D.flags.p + (size_t)k * S;
    }
    int nb = 0;
    LK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 128, 0));
    D.grid = gdev[d].num_sms * std::max(nb, 1);
    if (opt.blocks > 0) D.grid = std::min(D.grid, opt.blocks);
    LK(get_buf(D.parts, gdev[d].ws, WS_PARTS, (size_t)D.grid * 4 * sizeof(LongPart)));
  }
  // In multi-GPU mode edge g (g >= 1) is produced on device g-1 and consumed on device g;
  // flags of edge g live on the consumer as well (producer stores over NVLink).
  for (int d = 0; d < ND; ++d) {
    PerDev& D = pd[d];
    LK(cudaSetDevice(gdev[d].id));
    LK(cudaMemcpyAsync(D.bptr.p, bcol_ptr.data(), (Gtot + 1) * sizeof(int2*), cudaMemcpyHostToDevice,
                       gdev[d].stream));
    LK(cudaMemcpyAsync(D.fptr.p, flag_ptr.data(), (Gtot + 1) * sizeof(int32_t*), cudaMemcpyHostToDevice,
                       gdev[d].stream));
    long_init_kernel<<<gdev[d].num_sms * 4, 256, 0, gdev[d].stream>>>(
        P, (int)n, (int)m, (int4*)D.rowbuf.p, D.g_first == 0 && D.g_count > 0 ? bcol_ptr[0] : nullptr,
        (int2* const*)D.bptr.p, (const int*)D.cbuf.p, Gtot, D.g_first, D.g_count);
    LK(cudaGetLastError());
    *launches += 1;
    LK(cudaStreamSynchronize(gdev[d].stream));
  }
  // launch (all devices concurrently; their kernels wait on each other only via flags)
  for (int d = 0; d < ND; ++d) {
    PerDev& D = pd[d];
    if (D.g_count == 0) continue;
    LK(cudaSetDevice(gdev[d].id));
    LongArgs a;
    a.P = P;
    a.qc = (const uint8_t*)D.qc.p;
    a.sc = (const uint8_t*)D.sc.p;
    a.n = (int)n;
    a.m = (int)m;
    a.Gtot = Gtot;
    a.g_first = D.g_first;
    a.g_count = D.g_count;
    a.cb = (const int32_t*)D.cbuf.p;
    a.S = S;
    a.ticket = (int32_t*)D.ticket.p;
    a.rowprog = (int32_t*)D.prog.p;
    a.bflag = (int32_t* const*)D.fptr.p;  // edge g flags live on the consumer of edge g
    a.bcol = (int2* const*)D.bptr.p;
    a.rowbuf = (int4*)D.rowbuf.p;
    a.parts = (LongPart*)D.parts.p;
    a.abort_flag = (int32_t*)D.abort_.p;
    a.chunk = chunk;
    a.one = 1;
    a.lag = opt.start_lag > 0 ? opt.start_lag : chunk + 2 * 32 + 64;
    a.keyed = (long double)std::max(P.smax, 0) * std::min(n, m) < (long double)(1 << 25) ? 1 : 0;
    {
      const int c = P.go + P.ge;  // low half always borrows (values < 0): pre-add 1 to the high half
      a.hopc = c == 0 ? 0 : (int32_t)((((uint32_t)(-c - 1) & 0xffffu) << 16) | (uint32_t)((65536 - c) & 0xffff));
    }
    a.neg16 = NEG16C;
    a.sleep_ns = opt.sleep_ns;
    a.margin = (int32_t)margin16;
    a.bspan = (int32_t)bspan16;
    a.pad_top = pad_top;
    a.rowck = ck && ck->want ? ck->rowck : nullptr;
    a.colck = ck && ck->want ? ck->colck : nullptr;
    a.ck_every = ck && ck->want ? ck->ck_every : 1;
    a.kc_shift = ck && ck->want ? ck->kc_shift : 30;
    if (narrow) a.lag = opt.start_lag;  // 16-bit kernel: start slack off unless asked for
    a.prof = nullptr;
    if (opt.profile) {
      LK(get_buf(D.profbuf, gdev[d].ws, WS_PROF, 64));
      LK(cudaMemset(D.profbuf.p, 0, 64));
      a.prof = (unsigned long long*)D.profbuf.p;
    }
    a.spin_limit = opt.spin_limit;
    a.stall_task = opt.stall_task;
    LK(cudaEventCreate(&D.e0));
    LK(cudaEventCreate(&D.e1));
    LK(cudaEventRecord(D.e0, gdev[d].stream));
    fn<<<D.grid, 128, 0, gdev[d].stream>>>(a);
    LK(cudaGetLastError());
    LK(cudaEventRecord(D.e1, gdev[d].stream));
    *launches += 1;
  }
  // gather
  bool have_g = false;
  LongPart best;
  memset(&best, 0, sizeof(best));
  int32_t lv = 0, li = 0, lj = 0, rv = 0, rj = 0, cv = 0, ci = 0, gv = 0;
  int aborted = 0;
  for (int d = 0; d < ND; ++d) {
    PerDev& D = pd[d];
    if (D.g_count == 0) continue;
    LK(cudaSetDevice(gdev[d].id));
    LK(cudaStreamSynchronize(gdev[d].stream));
    float ms = 0;
    cudaEventElapsedTime(&ms, D.e0, D.e1);
    out->kernel_ms = std::max(out->kernel_ms, (double)ms);
    cudaEventDestroy(D.e0);
    cudaEventDestroy(D.e1);
    int ab = 0;
    LK(cudaMemcpy(&ab, D.abort_.p, 4, cudaMemcpyDeviceToHost));
    if (opt.profile && D.profbuf.p) {
      unsigned long long pr[5];
      LK(cudaMemcpy(pr, D.profbuf.p, sizeof(pr), cudaMemcpyDeviceToHost));
      const double tc = pr[1] ? (double)pr[1] : 1.0;
      fprintf(stderr, "[anyseq long] device %d: task cycles %llu, tasks %llu, grid %d; wait share: "
              "mid-task refills %.3f, task-start refills %.3f, column-edge flags %.3f\n",
              gdev[d].id, pr[1], pr[2], D.grid, pr[0] / tc, pr[3] / tc, pr[4] / tc);
    }
    aborted |= ab;
    std::vector<LongPart> parts((size_t)D.grid * 4);
    LK(cudaMemcpy(parts.data(), D.parts.p, parts.size() * sizeof(LongPart), cudaMemcpyDeviceToHost));
    for (const LongPart& p : parts) {
      if (p.lv > lv || (p.lv == lv && (p.lj < lj || (p.lj == lj && p.li < li)))) { lv = p.lv; li = p.li; lj = p.lj; }
      if (p.rv > rv || (p.rv == rv && p.rj < rj)) { rv = p.rv; rj = p.rj; }
      if (p.cv > cv || (p.cv == cv && p.ci < ci)) { cv = p.cv; ci = p.ci; }
      if (p.gset) { gv = p.gv; have_g = true; }
    }
  }
  auto handoff = [&]() {  // CKPT: the traceback walk reads the codes after this returns
    if (ck && ck->want) {
      ck->qc = (uint8_t*)pd[0].qc.p;
      ck->sc = (uint8_t*)pd[0].sc.p;
      if (pd[0].qc.own) pd[0].qc.p = pd[0].sc.p = nullptr;  // ownership moves to ck
    }
  };
  if (aborted) {
    *err = "long kernel: a boundary wait exceeded its bound";
    return ANYSEQ_E_TIMEOUT;
  }
  if (narrow && P.kind == KSEMI) {
    // row n from each group's row buffer (its own column strips), column m from the last
    // group's extra boundary column; (n, 0) = 0 is the first candidate (seq 0)
    unsigned long long key = ((unsigned long long)0x80000000u << 32) | 0xFFFFFFFFu;
    for (int d = 0; d < ND; ++d) {
      PerDev& D = pd[d];
      if (D.g_count == 0) continue;
      LK(cudaSetDevice(gdev[d].id));
      Buf kb;
      LK(get_buf(kb, gdev[d].ws, WS_KEY, 8));
      LK(cudaMemsetAsync(kb.p, 0, 8, gdev[d].stream));
      const int j0 = std::max(1, cb[D.g_first]), j1 = std::min<int>((int)m, cb[D.g_first + D.g_count]);
      const bool lastg = D.g_first + D.g_count == Gtot;
      semi_reduce_kernel<<<gdev[d].num_sms * 4, 256, 0, gdev[d].stream>>>(
          (const int4*)D.rowbuf.p, j0, j1, (int)m, lastg ? bcol_ptr[Gtot] : nullptr, (int)n,
          (unsigned long long*)kb.p);
      LK(cudaGetLastError());
      *launches += 1;
      unsigned long long kd = 0;
      LK(cudaMemcpyAsync(&kd, kb.p, 8, cudaMemcpyDeviceToHost, gdev[d].stream));
      LK(cudaStreamSynchronize(gdev[d].stream));
      key = std::max(key, kd);
    }
    handoff();
    const uint32_t seq = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu);
    out->score = (int32_t)((uint32_t)(key >> 32) ^ 0x80000000u);
    if (seq < m) { out->end_i = (int64_t)n; out->end_j = seq; }
    else { out->end_i = (int64_t)(seq - m); out->end_j = (int64_t)m; }
    return 0;
  }
  if (P.kind == KLOCAL) {
    out->score = lv; out->end_i = li; out->end_j = lj;
  } else if (P.kind == KSEMI) {
    if (rv >= cv) { out->score = rv; out->end_i = (int64_t)n; out->end_j = rj; }
    else { out->score = cv; out->end_i = ci; out->end_j = (int64_t)m; }
  } else {
    if (!have_g) {
      *err = "long kernel: global end cell not produced";
      return ANYSEQ_E_CUDA;
    }
    out->score = gv; out->end_i = (int64_t)n; out->end_j = (int64_t)m;
  }
  handoff();
  return 0;
}


// run_long_multi: one block per pair folds the warps' partial optima of that pair (the
// host-side fold of run_long, on the device: K pairs x resident warps entries)
__global__ void parts_reduce_kernel(const LongPart* __restrict__ parts, int nw, LongPart* out) {
  __shared__ LongPart sh[256];
  const LongPart* p = parts + (size_t)blockIdx.x * nw;
  LongPart b;
  memset(&b, 0, sizeof(b));
  for (int x = threadIdx.x; x < nw; x += blockDim.x) {
    const LongPart q = p[x];
    if (q.lv > b.lv || (q.lv == b.lv && (q.lj < b.lj || (q.lj == b.lj && q.li < b.li)))) {
      b.lv = q.lv; b.li = q.li; b.lj = q.lj;
    }
    if (q.gset) { b.gv = q.gv; b.gset = 1; }
  }
  sh[threadIdx.x] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int x = 1; x < (int)blockDim.x; ++x) {
      const LongPart& q = sh[x];
      if (q.lv > b.lv || (q.lv == b.lv && (q.lj < b.lj || (q.lj == b.lj && q.li < b.li)))) {
        b.lv = q.lv; b.li = q.li; b.lj = q.lj;
      }
      if (q.gset) { b.gv = q.gv; b.gset = 1; }
    }
    out[blockIdx.x] = b;
  }
}

// run_long_multi: long_init_kernel for every pair of the launch in one grid (y = pair)
__global__ void long_init_multi_kernel(DevParams P, const LongArgs* __restrict__ pairs, int K) {
  const int NEG = NEG32;
  const bool glob = P.kind == KGLOBAL;
  for (int p = blockIdx.y; p < K; p += gridDim.y) {
    const LongArgs& a = pairs[p];
    const int n = a.n, m = a.m, G = a.Gtot;
    int4* rowbuf = a.rowbuf;
    int2* bcol0 = a.bcol[0];
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x <= max(n, m); x += gridDim.x * blockDim.x) {
      if (x <= m) rowbuf[x] = make_int4(0, 0, NEG, 0);  // tag 0: no strip has written yet
      if (x <= n) bcol0[x] = make_int2(glob && x > 0 ? -(P.go + x * P.ge) : 0, NEG);
      if (x == 0)  // the pair's inner edges, and column m (edge G) when it keeps it (SEMI)
        for (int g = 1; g <= G; ++g) {
          int2* bc = a.bcol[g];
          if (g == G && (P.kind != KSEMI || !bc)) continue;
          bc[0] = make_int2(glob ? -(P.go + a.cb[g] * P.ge) : 0, NEG);  // H(0, c_g)
        }
    }
  }
}

// run_long_multi: semi_reduce_kernel for every pair of the launch in one grid (y = pair)
__global__ void semi_reduce_multi_kernel(const LongArgs* __restrict__ pairs, int K,
                                         unsigned long long* out) {
  for (int p = blockIdx.y; p < K; p += gridDim.y) {
    const LongArgs& a = pairs[p];
    const int n = a.n, m = a.m;
    const int4* rowbuf = a.rowbuf;
    const int2* colm = a.bcol[a.Gtot];
    unsigned long long best = 0;
    const int64_t nrow = m > 1 ? m - 1 : 0;  // j in [1, m - 1]
    const int64_t tot = nrow + (int64_t)n + 1;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < tot;
         x += (int64_t)gridDim.x * blockDim.x) {
      int v;
      uint32_t seq;
      if (x < nrow) {
        const int j = 1 + (int)x;
        v = rowbuf[j].x;
        seq = (uint32_t)j;
      } else {
        const int i = (int)(x - nrow);
        v = colm[i].x;
        seq = (uint32_t)m + (uint32_t)i;
      }
      const unsigned long long key =
          ((unsigned long long)((uint32_t)v ^ 0x80000000u) << 32) | (0xFFFFFFFFu - seq);
      best = key > best ? key : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
      best = y > best ? y : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out + p, best);
  }
}

static int run_long_multi_group(LongDevice& dev, const DevParams& P,
                                const std::vector<LongPairIn>& pairs, const LongOptions& opt,
                                std::vector<LongResult>* out, std::vector<int>* taken,
                                std::string* err, uint64_t* launches, double* kernel_ms,
                                const std::function<int()>& during, int* rows_out,
                                std::vector<LongCkpt>* cks, int64_t ck_budget);

// Launches of at most opt.multi_group pairs each (per-launch device state, e.g. the per-warp
// optimum slots of every pair, stays bounded: 2048 pairs x resident warps x 40 B ~ 0.2 GB).  With
// checkpoints (traceback) only the first group is taken: its checkpoints live in the
// workspace until the caller has walked them; the rest are left to the caller.
int run_long_multi(LongDevice& dev, const DevParams& P, const std::vector<LongPairIn>& pairs,
                   const LongOptions& opt, std::vector<LongResult>* out, std::vector<int>* taken,
                   std::string* err, uint64_t* launches, double* kernel_ms,
                   const std::function<int()>& during, int* rows_out,
                   std::vector<LongCkpt>* cks, int64_t ck_budget) {
  const size_t kGroup = (size_t)std::max(1, opt.multi_group);
  const size_t K0 = pairs.size();
  if (K0 <= kGroup)
    return run_long_multi_group(dev, P, pairs, opt, out, taken, err, launches, kernel_ms, during,
                                rows_out, cks, ck_budget);
  out->assign(K0, LongResult{0, 0, 0, 0.0, true});
  taken->assign(K0, 0);
  *kernel_ms = 0;
  if (cks) {
    cks->clear();
    cks->resize(K0);
    for (LongCkpt& c : *cks) c.owns = false;
  }
  for (size_t g0 = 0; g0 < K0; g0 += kGroup) {
    const size_t g1 = std::min(K0, g0 + kGroup);
    const std::vector<LongPairIn> sub(pairs.begin() + g0, pairs.begin() + g1);
    std::vector<LongResult> so;
    std::vector<int> st;
    std::vector<LongCkpt> sc;
    double ms = 0;
    const int rc = run_long_multi_group(dev, P, sub, opt, &so, &st, err, launches, &ms,
                                        g0 == 0 ? during : std::function<int()>(), rows_out,
                                        cks ? &sc : nullptr, ck_budget);
    if (rc != 0) return rc;
    *kernel_ms += ms;
    for (size_t k = 0; k < sub.size(); ++k) {
      (*out)[g0 + k] = so[k];
      (*taken)[g0 + k] = st[k];
      if (cks && st[k]) {
        LongCkpt& c = (*cks)[g0 + k];
        c = sc[k];  // a view (owns = false): copying it moves no buffer
        sc[k].qc = sc[k].sc = nullptr;
        sc[k].rowck = sc[k].colck = nullptr;
      }
    }
    if (cks) break;  // traceback: one group (see above)
  }
  return 0;
}

static int run_long_multi_group(LongDevice& dev, const DevParams& P,
                                const std::vector<LongPairIn>& pairs, const LongOptions& opt,
                                std::vector<LongResult>* out, std::vector<int>* taken,
                                std::string* err, uint64_t* launches, double* kernel_ms,
                                const std::function<int()>& during, int* rows_out,
                                std::vector<LongCkpt>* cks, int64_t ck_budget) {
  const size_t K0 = pairs.size();
  out->assign(K0, LongResult{0, 0, 0, 0.0, true});
  taken->assign(K0, 0);
  const bool want_ck = cks != nullptr;
  if (want_ck) {
    cks->clear();
    cks->resize(K0);
    for (LongCkpt& c : *cks) c.owns = false;
  }
  *kernel_ms = 0;
  // the eligibility rules of run_long's 16-bit path (at 512-row tasks, NR = 8)
  const int64_t d16 = (int64_t)P.go + P.ge + std::max(P.smax, 0);
  const int64_t margin16 = 100 * d16 + 16;
  const int NEG16C = -24576;
  auto fits16 = [&](int nr) {
    return 2 * (int64_t)(64 * nr + 66) * d16 + margin16 + 96 * d16 + P.go + P.ge + 256 < -NEG16C;
  };
  const bool fits = fits16(8) && (int64_t)P.go + 2 * P.ge < 4096;
  std::vector<size_t> sel;
  for (size_t k = 0; k < K0 && fits; ++k) {
    const uint64_t n = pairs[k].n, m = pairs[k].m;
    if (n == 0 || m == 0 || n >= (1ull << 31) || m >= (1ull << 31)) continue;
    const long double neg = 3.0L * P.go + ((long double)n + m + 2) * P.ge + 256;
    const long double pos = (long double)std::max(P.smax, 0) * std::min(n, m);
    if (neg > (1u << 30) - (1u << 24) || pos > (1u << 30) - (1u << 24)) continue;
    bool ok = true;
    for (uint64_t x = 0; x < m && ok; ++x) ok = (pairs[k].s[x] | 0x20) != 'n';
    if (ok) sel.push_back(k);
  }
  const int K = (int)sel.size();
  if (K == 0) return during ? during() : 0;
  LK(cudaSetDevice(dev.id));
  cudaStream_t st = dev.stream;
  if (dev.ws && during) {
    if (!dev.ws->stream) LK(cudaStreamCreateWithFlags(&dev.ws->stream, cudaStreamNonBlocking));
    st = dev.ws->stream;
  }
  // 1024-row tasks (NR = 16, the faster step) when the pairs give at least one task per
  // resident warp at that height, else 512-row tasks (twice the tasks, shorter ramps);
  // measured: 200 pairs of 2-20 kbp (1.2 tasks per warp) 14.5 -> 12.5 ms, 100 such pairs
  // (0.6 per warp) 9.7 -> 10.7 ms (tools/long_multi_bench.py --rows)
  int NR = 8;
  if (fits16(16) && opt.band_rows != 512) {
    int nb16 = 0;
    LK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb16, long16_multi_fn(P.kind, 16, want_ck), 128, 0));
    double T16 = 0;
    for (size_t k : sel) T16 += (double)((pairs[k].n + 1023) / 1024);
    if (T16 >= 4.0 * dev.num_sms * std::max(nb16, 1) || opt.band_rows == 1024) NR = 16;
  }
  const int HS = 64 * NR;
  if (rows_out) *rows_out = HS;
  const int64_t bspan16 = (int64_t)(64 * NR + 66) * d16;
  LongFn fn = long16_multi_fn(P.kind, NR, want_ck);
  int nb = 0;
  LK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 128, 0));
  int grid = dev.num_sms * std::max(nb, 1);
  if (opt.blocks > 0) grid = std::min(grid, opt.blocks);
  const int nw = grid * 4;
  // column passes per pair: tasks no wider than a quarter of the launch's mean work per
  // warp (>= 4096 columns), so the last tasks handed out are short; option long_strips
  // forces the count.  Tickets: pass by pass over the pairs, widest tasks first (LPT).
  std::vector<int> S(K), G(K);
  double Tw = 0;
  for (int x = 0; x < K; ++x) {
    S[x] = (int)((pairs[sel[x]].n + HS - 1) / HS);
    Tw += (double)S[x] * ((double)pairs[sel[x]].m + 64);
  }
  Tw /= nw;
  static const double wmin = [] {  // tuning: ANYSEQ_MULTI_WMIN (columns), ANYSEQ_MULTI_WDIV
    const char* e = getenv("ANYSEQ_MULTI_WMIN");
    return e ? atof(e) : 4096.0;
  }();
  static const double wdiv = [] {
    const char* e = getenv("ANYSEQ_MULTI_WDIV");
    return e ? atof(e) : 4.0;
  }();
  const double Wt = std::max(wmin, Tw / wdiv);
  int Gmax = 1;
  for (int x = 0; x < K; ++x) {
    const uint64_t m = pairs[sel[x]].m;
    const int g = opt.virtual_strips > 0 ? opt.virtual_strips
                                         : (int)std::min(16.0, std::ceil((double)m / Wt));
    G[x] = (int)std::min<uint64_t>((uint64_t)std::max(g, 1), m);
    Gmax = std::max(Gmax, G[x]);
  }
  std::vector<int> ord(K);
  for (int x = 0; x < K; ++x) ord[x] = x;
  std::stable_sort(ord.begin(), ord.end(), [&](int u, int v) {
    return (double)pairs[sel[u]].m / G[u] > (double)pairs[sel[v]].m / G[v];
  });
  std::vector<int2> segs;
  std::vector<int32_t> task_end;
  int64_t tasks = 0;
  for (int g = 0; g < Gmax; ++g)
    for (int x : ord)
      if (G[x] > g) {
        segs.push_back(make_int2(x, g));
        tasks += S[x];
        if (tasks >= (1ll << 31)) {
          *err = "long pairs: too many tasks in one launch";
          return ANYSEQ_E_UNSUPPORTED;
        }
        task_end.push_back((int32_t)tasks);
      }
  const int NS = (int)segs.size();
  // per-pair offsets into the launch-wide buffers
  std::vector<uint64_t> qo(K + 1, 0), so(K + 1, 0);
  std::vector<int64_t> rowo(K + 1, 0), bco(K + 1, 0), flo(K + 1, 0), cbo(K + 1, 0);
  for (int x = 0; x < K; ++x) {
    const uint64_t n = pairs[sel[x]].n, m = pairs[sel[x]].m;
    qo[x + 1] = qo[x] + n;
    so[x + 1] = so[x] + m;
    rowo[x + 1] = rowo[x] + (int64_t)m + 1;
    const int extra = P.kind == KSEMI ? 1 : 0;  // SEMI keeps column m (edge G)
    bco[x + 1] = bco[x] + (int64_t)(G[x] + extra) * (int64_t)(n + 1);
    flo[x + 1] = flo[x] + (int64_t)G[x] * S[x];
    cbo[x + 1] = cbo[x] + G[x] + 1;
  }
  // traceback: checkpoint rows after every strip, columns every 2^9 (the single-pair
  // path's finest geometry), one workspace buffer for all pairs
  constexpr int kCkShift = 9;
  std::vector<int64_t> cko(K + 1, 0);
  if (want_ck) {
    for (int x = 0; x < K; ++x) {
      const int64_t n = (int64_t)pairs[sel[x]].n, m = (int64_t)pairs[sel[x]].m;
      cko[x + 1] = cko[x] + (int64_t)(S[x] - 1) * (m + 1) + ((m - 1) >> kCkShift) * (n + 1);
    }
    size_t fr = 0, tot = 0;
    LK(cudaMemGetInfo(&fr, &tot));
    const int64_t budget = ck_budget > 0 ? ck_budget : (int64_t)(0.4 * (double)fr);
    if (cko[K] * (int64_t)sizeof(int2) > budget) return during ? during() : 0;  // none taken
  }
  LongWs* ws = dev.ws;
  Buf qa, sa, qc, sc, sum, flg, off, rowbuf, bcol, flags, cbuf, bptr, fptr, ticket, abort_, parts,
      mp, mt, ms_, red, kb, ckb;
  // ASCII upload + pack (all pairs in one pack launch)
  std::string cq, cs;
  cq.reserve(qo[K]);
  cs.reserve(so[K]);
  for (int x = 0; x < K; ++x) {
    cq.append(pairs[sel[x]].q, pairs[sel[x]].n);
    cs.append(pairs[sel[x]].s, pairs[sel[x]].m);
  }
  LK(get_buf(qa, ws, WS_QA, qo[K] + 16));
  LK(get_buf(sa, ws, WS_SA, so[K] + 16));
  LK(get_buf(qc, ws, WS_QC, qo[K] + 16));
  LK(get_buf(sc, ws, WS_SC, so[K] + 16));
  LK(get_buf(sum, ws, WS_SUM, sizeof(PlanSummary)));
  LK(get_buf(flg, ws, WS_FLG, (size_t)K * 4 + 16));
  LK(get_buf(off, ws, WS_OFF, (size_t)2 * (K + 1) * 8));
  LK(cudaMemcpyAsync(qa.p, cq.data(), qo[K], cudaMemcpyHostToDevice, st));
  LK(cudaMemcpyAsync(sa.p, cs.data(), so[K], cudaMemcpyHostToDevice, st));
  LK(cudaMemcpyAsync(off.p, qo.data(), (K + 1) * 8, cudaMemcpyHostToDevice, st));
  LK(cudaMemcpyAsync((uint64_t*)off.p + K + 1, so.data(), (K + 1) * 8, cudaMemcpyHostToDevice, st));
  PlanSummary hs;
  memset(&hs, 0, sizeof(hs));
  hs.err_pos = ~0ull;
  LK(cudaMemcpyAsync(sum.p, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));
  LK(launch_pack((const char*)qa.p, qo[K], (uint8_t*)qc.p, (const uint64_t*)off.p,
                 (const char*)sa.p, so[K], (uint8_t*)sc.p, (const uint64_t*)off.p + K + 1,
                 (uint64_t)K, (uint32_t*)flg.p, (PlanSummary*)sum.p, st, dev.num_sms));
  *launches += 1;
  LK(cudaMemcpyAsync(&hs, sum.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
  LK(cudaStreamSynchronize(st));
  if (hs.err_pos != ~0ull) {  // offsets into the concatenated sequences -> pair and offset
    const bool in_s = hs.err_pos >= (1ull << 62);
    const uint64_t pos = in_s ? hs.err_pos - (1ull << 62) : hs.err_pos;
    const std::vector<uint64_t>& o = in_s ? so : qo;
    int x = 0;
    while (x + 1 < K && o[x + 1] <= pos) ++x;
    *err = std::string("invalid symbol at ") + (in_s ? "s" : "q") + " offset " +
           std::to_string(pos - o[x]) + " of long pair " + std::to_string(sel[x]);
    return ANYSEQ_E_BADSEQ;
  }
  // DP state of every pair
  LK(get_buf(rowbuf, ws, WS_ROWBUF, (size_t)rowo[K] * sizeof(int4)));
  LK(get_buf(bcol, ws, WS_BCOL, (size_t)bco[K] * sizeof(int2)));
  LK(get_buf(flags, ws, WS_FLAGS, (size_t)flo[K] * 4));
  LK(get_buf(cbuf, ws, WS_CB, (size_t)cbo[K] * 4));
  LK(get_buf(bptr, ws, WS_BPTR, (size_t)cbo[K] * sizeof(int2*)));
  LK(get_buf(fptr, ws, WS_FPTR, (size_t)cbo[K] * sizeof(int32_t*)));
  LK(get_buf(ticket, ws, WS_TICKET, 4));
  LK(get_buf(abort_, ws, WS_ABORT, 4));
  LK(get_buf(parts, ws, WS_PARTS, (size_t)K * nw * sizeof(LongPart)));
  LK(get_buf(mp, ws, WS_M_PAIRS, (size_t)K * sizeof(LongArgs)));
  LK(get_buf(mt, ws, WS_M_TASKS, (size_t)NS * 4));
  LK(get_buf(ms_, ws, WS_M_SEGS, (size_t)NS * sizeof(int2)));
  LK(get_buf(red, ws, WS_M_RED, (size_t)K * sizeof(LongPart)));
  if (P.kind == KSEMI) LK(get_buf(kb, ws, WS_KEY, (size_t)K * 8));
  if (want_ck) LK(get_buf(ckb, ws, WS_ROWCK, (size_t)std::max<int64_t>(cko[K], 1) * sizeof(int2)));
  LK(cudaMemsetAsync(flags.p, 0, (size_t)flo[K] * 4, st));
  LK(cudaMemsetAsync(ticket.p, 0, 4, st));
  LK(cudaMemsetAsync(abort_.p, 0, 4, st));
  LK(cudaMemsetAsync(parts.p, 0, (size_t)K * nw * sizeof(LongPart), st));
  if (P.kind == KSEMI) LK(cudaMemsetAsync(kb.p, 0, (size_t)K * 8, st));
  std::vector<int32_t> cb_h(cbo[K]);
  std::vector<int2*> bp_h(cbo[K], nullptr);
  std::vector<int32_t*> fp_h(cbo[K], nullptr);
  std::vector<LongArgs> la(K);
  const int c = P.go + P.ge;
  const int32_t hopc =
      c == 0 ? 0 : (int32_t)((((uint32_t)(-c - 1) & 0xffffu) << 16) | (uint32_t)((65536 - c) & 0xffff));
  for (int x = 0; x < K; ++x) {
    const uint64_t n = pairs[sel[x]].n, m = pairs[sel[x]].m;
    const int Gx = G[x];
    for (int g = 0; g <= Gx; ++g) cb_h[cbo[x] + g] = (int32_t)((m * (uint64_t)g) / Gx);
    int2* bc = (int2*)bcol.p + bco[x];
    for (int g = 0; g < Gx + (P.kind == KSEMI ? 1 : 0); ++g) bp_h[cbo[x] + g] = bc + (size_t)g * (n + 1);
    for (int g = 0; g < Gx; ++g) fp_h[cbo[x] + g] = (int32_t*)flags.p + flo[x] + (size_t)g * S[x];
    LongArgs& a = la[x];
    memset(&a, 0, sizeof(a));
    a.P = P;
    a.qc = (const uint8_t*)qc.p + qo[x];
    a.sc = (const uint8_t*)sc.p + so[x];
    a.n = (int)n;
    a.m = (int)m;
    a.Gtot = Gx;
    a.g_first = 0;
    a.g_count = Gx;
    a.cb = (const int32_t*)cbuf.p + cbo[x];
    a.S = S[x];
    a.ticket = (int32_t*)ticket.p;
    a.rowprog = nullptr;
    a.bflag = (int32_t* const*)fptr.p + cbo[x];
    a.bcol = (int2* const*)bptr.p + cbo[x];
    a.rowbuf = (int4*)rowbuf.p + rowo[x];
    a.parts = (LongPart*)parts.p + (size_t)x * nw;
    a.abort_flag = (int32_t*)abort_.p;
    a.chunk = 256;
    a.one = 1;
    a.lag = opt.start_lag;
    a.keyed = (long double)std::max(P.smax, 0) * std::min(n, m) < (long double)(1 << 25) ? 1 : 0;
    a.hopc = hopc;
    a.neg16 = NEG16C;
    a.sleep_ns = opt.sleep_ns;
    a.margin = (int32_t)margin16;
    a.bspan = (int32_t)bspan16;
    a.pad_top = P.kind == KSEMI ? (int)((uint64_t)S[x] * HS - n) : 0;
    a.ck_every = 1;
    a.kc_shift = 30;
    if (want_ck) {
      int2* base = (int2*)ckb.p + cko[x];
      a.rowck = S[x] > 1 ? base : nullptr;
      a.colck = ((m - 1) >> kCkShift) > 0 ? base + (size_t)(S[x] - 1) * (m + 1) : nullptr;
      a.kc_shift = kCkShift;
    }
    a.spin_limit = opt.spin_limit;
    a.stall_task = -1;
  }
  LK(cudaMemcpyAsync(cbuf.p, cb_h.data(), cb_h.size() * 4, cudaMemcpyHostToDevice, st));
  LK(cudaMemcpyAsync(bptr.p, bp_h.data(), bp_h.size() * sizeof(int2*), cudaMemcpyHostToDevice, st));
  LK(cudaMemcpyAsync(fptr.p, fp_h.data(), fp_h.size() * sizeof(int32_t*), cudaMemcpyHostToDevice, st));
  LK(cudaMemcpyAsync(mp.p, la.data(), (size_t)K * sizeof(LongArgs), cudaMemcpyHostToDevice, st));
  LK(cudaMemcpyAsync(mt.p, task_end.data(), (size_t)NS * 4, cudaMemcpyHostToDevice, st));
  LK(cudaMemcpyAsync(ms_.p, segs.data(), (size_t)NS * sizeof(int2), cudaMemcpyHostToDevice, st));
  uint64_t maxnm = 0;
  for (int x = 0; x < K; ++x) maxnm = std::max(maxnm, std::max(pairs[sel[x]].n, pairs[sel[x]].m));
  const dim3 gi((unsigned)std::min<uint64_t>((maxnm + 256) / 256, 64), (unsigned)std::min(K, 65535));
  long_init_multi_kernel<<<gi, 256, 0, st>>>(P, (const LongArgs*)mp.p, K);
  LK(cudaGetLastError());
  *launches += 1;
  LongArgs a0 = la[0];
  a0.pairs = (const LongArgs*)mp.p;
  a0.task_end = (const int32_t*)mt.p;
  a0.segs = (const int2*)ms_.p;
  a0.task_total = (int32_t)tasks;
  a0.stall_task = opt.stall_task;
  a0.prof = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  LK(cudaEventCreate(&e0));
  LK(cudaEventCreate(&e1));
  LK(cudaEventRecord(e0, st));
  fn<<<grid, 128, 0, st>>>(a0);
  LK(cudaGetLastError());
  LK(cudaEventRecord(e1, st));
  *launches += 1;
  parts_reduce_kernel<<<K, 256, 0, st>>>((const LongPart*)parts.p, nw, (LongPart*)red.p);
  LK(cudaGetLastError());
  *launches += 1;
  if (P.kind == KSEMI) {
    const dim3 gs((unsigned)std::min<uint64_t>((2 * maxnm + 256) / 256, 64), (unsigned)std::min(K, 65535));
    semi_reduce_multi_kernel<<<gs, 256, 0, st>>>((const LongArgs*)mp.p, K, (unsigned long long*)kb.p);
    LK(cudaGetLastError());
    *launches += 1;
  }
  // the caller's work in the shadow of the launch (results are read after it: pageable
  // device-to-host copies would block the host until the kernel ends)
  const int rd = during ? during() : 0;
  std::vector<LongPart> rp(K);
  std::vector<unsigned long long> keys(P.kind == KSEMI ? K : 0);
  int ab = 0;
  LK(cudaMemcpyAsync(rp.data(), red.p, (size_t)K * sizeof(LongPart), cudaMemcpyDeviceToHost, st));
  if (P.kind == KSEMI)
    LK(cudaMemcpyAsync(keys.data(), kb.p, (size_t)K * 8, cudaMemcpyDeviceToHost, st));
  LK(cudaMemcpyAsync(&ab, abort_.p, 4, cudaMemcpyDeviceToHost, st));
  LK(cudaStreamSynchronize(st));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *kernel_ms = ms;
  if (rd != 0) return rd;
  if (ab) {
    *err = "long kernel: a boundary wait exceeded its bound";
    return ANYSEQ_E_TIMEOUT;
  }
  for (int x = 0; x < K; ++x) {
    const size_t k = sel[x];
    const int64_t n = (int64_t)pairs[k].n, m = (int64_t)pairs[k].m;
    LongResult& r = (*out)[k];
    r.narrow = true;
    r.kernel_ms = ms;
    if (P.kind == KLOCAL) {
      r.score = rp[x].lv; r.end_i = rp[x].li; r.end_j = rp[x].lj;
    } else if (P.kind == KSEMI) {
      // (n, 0) = 0 is the first candidate (seq 0), as in run_long
      unsigned long long key = ((unsigned long long)0x80000000u << 32) | 0xFFFFFFFFu;
      key = std::max(key, keys[x]);
      const uint32_t seq = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu);
      r.score = (int32_t)((uint32_t)(key >> 32) ^ 0x80000000u);
      if (seq < (uint64_t)m) { r.end_i = n; r.end_j = seq; }
      else { r.end_i = (int64_t)(seq - m); r.end_j = m; }
    } else {
      if (!rp[x].gset) {
        *err = "long kernel: global end cell not produced";
        return ANYSEQ_E_CUDA;
      }
      r.score = rp[x].gv; r.end_i = n; r.end_j = m;
    }
    (*taken)[k] = 1;
    if (want_ck) {
      LongCkpt& c = (*cks)[k];
      c.owns = false;
      c.qc = (uint8_t*)la[x].qc;
      c.sc = (uint8_t*)la[x].sc;
      c.rowck = la[x].rowck;
      c.colck = la[x].colck;
      c.HS = HS;
      c.ck_every = 1;
      c.kc_shift = kCkShift;
      c.PT = la[x].pad_top;
      c.S = S[x];
      c.bytes = (size_t)(cko[x + 1] - cko[x]) * sizeof(int2);
    }
  }
  return 0;
}

}  // namespace anyseq
