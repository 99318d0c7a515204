// csrc/long_tb.cu -- linear-space long-pair traceback from checkpoints.
//
// The forward pass (long16_kernel<.., CKPT = true>, one pass over the whole matrix, which
// also finds the optimum of Eqs. (1)-(5)) keeps the DP rows at every row-block
// boundary and the DP columns at every column-block boundary.  The traceback then walks
// the path of the relax listing (the oracle's walk of SURVEY 8(c) step 7) from
// the end cell back, one tile (row block x column block) at a time: the tile region
// up-left of the current cell is recomputed from its top checkpoint row and left
// checkpoint column into per-cell direction bytes (H source DIAG/UP/LEFT/STOP with the tie
// order DIAG > E > F, plus the E / F extension bits with extension winning ties -- readings
// R7-R9), and one warp walks them with 32-cell lookahead until the path leaves the tile.
// Every decision is taken from exact full-matrix values, so the CIGAR is the one the
// full-matrix traceback (the oracle) produces: bit-exact, affine or linear, every kind.
//
// The recompute: thread t of 256 owns TR consecutive rows of the tile and sweeps its
// columns with a skew of one step per thread (the anti-diagonal wavefront of P:274); the
// row above a thread's first row arrives from thread t-1 through a double-buffered shared
// slot (one barrier per step).  Direction bytes go to a global scratch in step-major order
// (word (step * 256 + t) holds the thread's TR rows), so every step's stores are one
// coalesced row of words and the walk reads a diagonal run as consecutive words.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/anyseq.h"
#include "common.cuh"
#include "long.h"
#include "long_tb.h"

namespace anyseq {

namespace {

constexpr int NT = 256;  // recompute threads (rows: NT * TR per tile)
constexpr int NEGI = -(1 << 29);

struct WalkArgs {
  int32_t kind, affine;
  int32_t go, ge, cop;
  int8_t sig[25];
  const uint8_t* qc;  // codes of q (rows), s (columns)
  const uint8_t* sc;
  int32_t n, m;
  const int2* rowck;  // (H, E) of checkpoint rows
  const int2* colck;  // (H, F) of checkpoint columns
  int32_t TH;         // rows per row block (padded coordinates)
  int32_t PT;         // pad rows above row 1 (SEMI)
  int32_t kc_shift;   // columns per column block = 1 << kc_shift
  int32_t end_i, end_j;
  uint8_t* scratch;   // direction bytes of one tile, (kc + NT) * NT * TR
  uint32_t* ops;      // reversed RLE words (len << 4 | op)
  uint64_t ops_cap;
  unsigned long long* out;  // [0] ops written, [1] begin i, [2] begin j, [3] tiles, [4] hits
  uint8_t* slots;     // NSLOT helper scratches, slot_bytes each (whole tiles)
  size_t slot_bytes;
  int* sync;          // [0] jobs queued (walker), [1] jobs taken (helpers), [2] done, [3] abort
  int* slot_job;      // [NSLOT]: the job whose bytes the slot holds (-1: none yet)
  int2* jobs;         // [JMAX]: tile (row block, column block) of each job
  int32_t nrowck, ncolck;  // checkpoint rows / columns stored (bounds checks)
};

__device__ __forceinline__ int h_row0(const WalkArgs& a, int j) {  // H(0, j)
  return a.kind == KGLOBAL ? (j ? -(a.go + j * a.ge) : 0) : 0;
}
__device__ __forceinline__ int h_col0(const WalkArgs& a, int i) {  // H(i, 0)
  return a.kind == KGLOBAL ? (i ? -(a.go + i * a.ge) : 0) : 0;
}

constexpr int KC_MAX = 4096;  // widest column block
constexpr int NSLOT = 64;     // tile scratch slots of the helper CTAs
constexpr int JMAX = 1 << 20; // job queue entries (a job = one tile)

__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Shared memory of one CTA's recompute.
struct RecompSmem {
  int xh[2][NT], xe[2][NT];
  uint8_t scode[KC_MAX];
  int sig[25];
};

// Recompute rows (R, R + nr] x columns (C, C + nc] of tile (b, kb) into direction bytes at
// `dirs` (word (step * NT + t) * WPT + r/4 holds the thread's rows r), block-wide.  `top`
// (dynamic shared memory, nc entries) receives the tile's top boundary row.
template <int TR>
__device__ void recompute(const WalkArgs& a, int b, int kb, int R, int C, int nr, int nc,
                          uint8_t* dirs, RecompSmem& sm, int2* top) {
  const int t = threadIdx.x;
  const int row0 = R + t * TR;  // the row above this thread's first row
  const bool tact = t * TR < nr;
  int h[TR], f[TR];
  int qcode[TR];
#pragma unroll
  for (int r = 0; r < TR; ++r) {
    const int ii = row0 + r + 1;
    const bool real = ii <= R + nr;
    int2 lb = make_int2(h_col0(a, ii), NEGI);  // column 0: H(i, 0), F = -inf
    ANY_CHECK(!real || ii <= a.n);
    ANY_CHECK(kb == 0 || kb - 1 < a.ncolck);
    if (real && kb > 0) lb = a.colck[(size_t)(kb - 1) * (a.n + 1) + ii];
    h[r] = lb.x;
    f[r] = lb.y;
    qcode[r] = real ? 5 * (int)a.qc[ii - 1] : 0;
  }
  // the diagonal of the first row at the first column: H(row0, C)
  int hprev;
  if (t == 0) {
    hprev = R == 0 ? h_row0(a, C)
                   : (kb == 0 ? h_col0(a, R) : a.rowck[(size_t)(b - 1) * (a.m + 1) + C].x);
  } else {
    hprev = (kb == 0) ? h_col0(a, row0) : a.colck[(size_t)(kb - 1) * (a.n + 1) + row0].x;
  }
  const int nthreads = (nr + TR - 1) / TR;
  const int steps = nc + nthreads - 1;
  ANY_CHECK(nc <= KC_MAX && nr <= NT * TR && (R == 0 || b - 1 < a.nrowck));
  for (int c = t; c < nc; c += NT) {
    const int jj = C + 1 + c;
    top[c] = R == 0 ? make_int2(h_row0(a, jj), NEGI) : a.rowck[(size_t)(b - 1) * (a.m + 1) + jj];
    sm.scode[c] = a.sc[jj - 1];
  }
  __syncthreads();
  for (int k = 0; k < steps; ++k) {
    const int c = k - t;  // column index in the region (jj = C + 1 + c)
    if (tact && c >= 0 && c < nc) {
      int hup, eup;  // H(row0, jj), E(row0, jj)
      if (t == 0) {
        const int2 v = top[c];
        hup = v.x;
        eup = v.y;
      } else {
        hup = sm.xh[(k - 1) & 1][t - 1];
        eup = sm.xe[(k - 1) & 1][t - 1];
      }
      const int scode = sm.scode[c];
      int dg = hprev;
      hprev = hup;
      uint32_t word = 0;
#pragma unroll
      for (int r = 0; r < TR; ++r) {
        int E, F;
        uint32_t eext = 0, fext = 0;
        if (a.affine) {  // Eqs. (4)-(5): extension first, extension wins ties (R8)
          const int ex = eup - a.ge, eo = hup - a.cop;
          E = max(ex, eo);
          eext = ex >= eo;
          const int fx = f[r] - a.ge, fo = h[r] - a.cop;
          F = max(fx, fo);
          fext = fx >= fo;
        } else {  // Eqs. (2)-(3)
          E = hup - a.ge;
          F = h[r] - a.ge;
        }
        // Eq. (1) in the relax listing's order: strict '>' replacement, DIAG > E > F (R7)
        int H = dg + sm.sig[qcode[r] + scode];
        uint32_t src = 0;
        if (E > H) { H = E; src = 1; }
        if (F > H) { H = F; src = 2; }
        if (a.kind == KLOCAL && H <= 0) { H = 0; src = 3; }  // nu = 0 wins ties at 0 (R9)
        word |= (src | (eext << 2) | (fext << 3)) << (8 * (r & 3));
        if ((r & 3) == 3 || r == TR - 1) {
          ANY_CHECK(((size_t)k * NT + t) * ((TR + 3) / 4) * 4 < a.slot_bytes);
          reinterpret_cast<uint32_t*>(dirs)[((size_t)k * NT + t) * ((TR + 3) / 4) + (r >> 2)] = word;
          word = 0;
        }
        dg = h[r];
        h[r] = H;
        f[r] = F;
        hup = H;
        eup = E;
      }
      sm.xh[k & 1][t] = hup;
      sm.xe[k & 1][t] = eup;
    }
    __syncthreads();
  }
}

// Block 0 walks; blocks 1.. are helpers that recompute whole tiles the walker is predicted
// to enter next (the path is monotone: up, left or up-left), so the walker mostly finds its
// next tile's direction bytes ready instead of recomputing them on one SM.
template <int TR>
__global__ void __launch_bounds__(NT) tile_walk_kernel(WalkArgs a) {
  __shared__ RecompSmem sm;
  extern __shared__ int2 top[];  // [KC_MAX]
  __shared__ int sh_i, sh_j, sh_st, sh_done, sh_slot, sh_job;
  __shared__ unsigned long long sh_nops, sh_hits;
  __shared__ uint32_t sh_run;  // the RLE word being accumulated (len << 4 | op), 0 = none
  __shared__ long long sched_tile[NSLOT];  // walker: tile (b << 32 | kb) of the slot's last job
  __shared__ int sched_job[NSLOT];
  __shared__ int sh_tail;
  const int t = threadIdx.x;
  if (t < 25) sm.sig[t] = a.sig[t];
  const int kc = 1 << a.kc_shift;
  const size_t wpt_bytes = ((TR + 3) / 4) * 4;
  if (blockIdx.x > 0) {  // ---------------------------------------------------- helper
    __shared__ int hj, hexit;
    for (;;) {
      __syncthreads();
      if (t == 0) {
        hexit = 0;
        hj = atomicAdd(&a.sync[1], 1);
        long long spins = 0;
        while (ld_acq(&a.sync[0]) <= hj) {
          if (*(volatile int*)&a.sync[2]) { hexit = 1; break; }
          __nanosleep(256);
          if (++spins > (1ll << 26)) { atomicExch(&a.sync[3], 1); hexit = 1; break; }
        }
        if (!hexit && hj >= NSLOT) {  // the slot's previous job must be complete
          const int s = hj % NSLOT;
          while (ld_acq(&a.slot_job[s]) != hj - NSLOT) {
            if (*(volatile int*)&a.sync[3]) { hexit = 1; break; }
            __nanosleep(128);
          }
        }
      }
      __syncthreads();
      if (hexit) return;
      const int j = hj, s = j % NSLOT;
      const int2 tile = a.jobs[j];
      const int b = tile.x, kb = tile.y;
      const int R = max(0, b * a.TH - a.PT);
      const int R1 = min(a.n, (b + 1) * a.TH - a.PT);
      const int C = kb << a.kc_shift;
      const int C1 = min(a.m, C + kc);
      recompute<TR>(a, b, kb, R, C, R1 - R, C1 - C, a.slots + (size_t)s * a.slot_bytes, sm, top);
      if (t == 0) {
        __threadfence();
        st_rel(&a.slot_job[s], j);
      }
    }
  }
  // ------------------------------------------------------------------------- walker
  if (t == 0) {
    sh_i = a.end_i;
    sh_j = a.end_j;
    sh_st = 0;  // 0 = H, 1 = E (vertical, I), 2 = F (horizontal, D)
    sh_done = 0;
    sh_nops = 0;
    sh_hits = 0;
    sh_run = 0;
    sh_tail = 0;
  }
  if (t < NSLOT) {
    sched_tile[t] = -1;
    sched_job[t] = -1;
  }
  __syncthreads();
  unsigned long long tiles = 0;
  // append a run of ops (walk order = reversed alignment order); warp 0 lane 0 only
  auto emit = [&](uint32_t op, uint64_t len) {
    while (len > 0) {
      uint32_t r = sh_run;
      if (r && (r & 15) == op && (r >> 4) < (1u << 28) - 1) {
        const uint64_t room = ((1u << 28) - 1) - (r >> 4), add = len < room ? len : room;
        sh_run = r + (uint32_t)(add << 4);
        len -= add;
      } else {
        if (r) {
          if (sh_nops < a.ops_cap) a.ops[sh_nops] = r;
          ++sh_nops;
        }
        const uint64_t add = len < (1u << 28) - 1 ? len : (1u << 28) - 1;
        sh_run = (uint32_t)(add << 4) | op;
        len -= add;
      }
    }
  };
  const bool helpers = gridDim.x > 1;

  for (;;) {
    __syncthreads();
    if (sh_done) break;
    const int i = sh_i, j = sh_j;
    if (i == 0 || j == 0) {  // boundary: global emits the leading gap run (R16), else stop
      if (t == 0) {
        if (a.kind == KGLOBAL) {
          if (i) emit(1, (uint64_t)i);
          if (j) emit(2, (uint64_t)j);
          sh_i = 0;
          sh_j = 0;
        }
        sh_done = 1;
      }
      continue;
    }
    // the tile holding (i, j): row block b (padded rows [b TH, (b+1) TH)), column block k
    const int b = (i - 1 + a.PT) / a.TH;
    const int R = max(0, b * a.TH - a.PT);  // top boundary row of the tile
    const int kb = (j - 1) >> a.kc_shift;
    const int C = kb << a.kc_shift;         // left boundary column
    ++tiles;
    if (t == 0) {
      sh_slot = -1;
      if (helpers) {
        const long long key = ((long long)b << 32) | (unsigned)kb;
        int found = -1;
        for (int x = 0; x < NSLOT; ++x)
          if (sched_tile[x] == key) found = x;
        // predict the next tiles (up, left, up-left and the diagonal band two and three
        // tiles ahead) and queue those not yet queued; a slot is reused only when its
        // tile lies behind the walker (not up-left of or equal to the current tile)
        const int pred[9][2] = {{1, 1}, {1, 0}, {0, 1}, {2, 2}, {2, 1}, {1, 2}, {3, 3}, {3, 2}, {2, 3}};
        for (int x = 0; x < 9; ++x) {
          const int tb = b - pred[x][0], tk = kb - pred[x][1];
          if (tb < 0 || tk < 0) continue;
          const long long k2 = ((long long)tb << 32) | (unsigned)tk;
          bool have = false;
          for (int y = 0; y < NSLOT; ++y) have |= sched_tile[y] == k2;
          if (have) continue;
          const int jn = sh_tail;
          if (jn >= JMAX) break;
          const int sl = jn % NSLOT;
          const long long old = sched_tile[sl];
          if (old >= 0 && (int)(old >> 32) <= b && (int)(old & 0xffffffff) <= kb) continue;
          a.jobs[jn] = make_int2(tb, tk);
          sched_tile[sl] = k2;
          sched_job[sl] = jn;
          sh_tail = jn + 1;
          st_rel(&a.sync[0], jn + 1);
        }
        if (found >= 0) {  // its bytes are (or will be) in slot `found`
          const int jf = sched_job[found];
          long long spins = 0;
          while (ld_acq(&a.slot_job[found]) != jf) {
            __nanosleep(64);
            if (++spins > (1ll << 26)) { atomicExch(&a.sync[3], 1); break; }
          }
          sh_slot = found;
          ++sh_hits;
        }
      }
    }
    __syncthreads();
    const int slot = sh_slot;
    const uint8_t* dirs;
    if (slot >= 0) {
      dirs = a.slots + (size_t)slot * a.slot_bytes;
    } else {  // not predicted: recompute the region up-left of (i, j) here
      recompute<TR>(a, b, kb, R, C, i - R, j - C, a.scratch, sm, top);
      dirs = a.scratch;
    }
    // ---- walk the region (warp 0) until the path leaves it ----
    if (t < 32) {
      const int lane = t;
      int ci = i, cj = j, st = sh_st;
      auto dir_at = [&](int ii, int jj) -> uint32_t {  // direction byte of cell (ii, jj)
        const int rr = ii - R - 1, tt = rr / TR, step = (jj - C - 1) + tt;
        ANY_CHECK(rr >= 0 && step >= 0 && ((size_t)step * NT + tt) * wpt_bytes < a.slot_bytes);
        return dirs[((size_t)step * NT + tt) * wpt_bytes + (rr % TR)];
      };
      bool done = false;
      while (!done && ci > R && cj > C) {
        if (st == 0) {  // H state: a diagonal run, then the first non-DIAG cell
          // 4 x 32 cells of the diagonal are read at once (independent loads, one L2 round
          // trip): similar sequences have DIAG runs of hundreds of cells
          uint32_t dv[4];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int ii = ci - lane - 32 * g, jj = cj - lane - 32 * g;
            dv[g] = (ii > R && jj > C) ? dir_at(ii, jj) : 0xFFu;
          }
          int l = 128;
          uint32_t d = 0;
#pragma unroll
          for (int g = 3; g >= 0; --g) {
            const uint32_t m = __ballot_sync(0xffffffffu, (dv[g] & 3) != 0);
            if (m) { l = 32 * g + __ffs(m) - 1; d = __shfl_sync(0xffffffffu, dv[g], __ffs(m) - 1); }
          }
          // cells [0, l) are DIAG
          if (l > 0 && lane == 0) emit(0, (uint64_t)l);
          ci -= l;
          cj -= l;
          if (l < 128) {
            const uint32_t dl = d;
            const bool inl = (ci > R && cj > C);
            if (inl) {
              const uint32_t src = dl & 3;
              if (src == 3) done = true;           // local STOP
              else st = (int)src;                  // UP -> E state, LEFT -> F state
            }
          }
        } else if (st == 1) {  // E state: I ops up the column while E extends
          const int ii = ci - lane;
          const bool in = ii > R;
          const uint32_t d = in ? dir_at(ii, cj) : 0;
          const uint32_t endm = __ballot_sync(0xffffffffu, in && !((d >> 2) & 1));
          const uint32_t outm = __ballot_sync(0xffffffffu, !in);
          const int le = endm ? __ffs(endm) - 1 : 32, lo = outm ? __ffs(outm) - 1 : 32;
          if (le < lo) {  // the run ends inside: cells [0, le] emit I, then the H state
            if (lane == 0) emit(1, (uint64_t)le + 1);
            ci -= le + 1;
            st = 0;
          } else {        // all extend up to the region's edge (or 32 cells): stay in E
            if (lane == 0) emit(1, (uint64_t)lo);
            ci -= lo;
          }
        } else {  // F state: D ops along the row while F extends
          const int jj = cj - lane;
          const bool in = jj > C;
          const uint32_t d = in ? dir_at(ci, jj) : 0;
          const uint32_t endm = __ballot_sync(0xffffffffu, in && !((d >> 3) & 1));
          const uint32_t outm = __ballot_sync(0xffffffffu, !in);
          const int le = endm ? __ffs(endm) - 1 : 32, lo = outm ? __ffs(outm) - 1 : 32;
          if (le < lo) {
            if (lane == 0) emit(2, (uint64_t)le + 1);
            cj -= le + 1;
            st = 0;
          } else {
            if (lane == 0) emit(2, (uint64_t)lo);
            cj -= lo;
          }
        }
      }
      if (lane == 0) {
        sh_i = ci;
        sh_j = cj;
        sh_st = st;
        if (done) sh_done = 1;
      }
    }
  }
  if (t == 0) {
    if (helpers) st_rel(&a.sync[2], 1);  // helpers: no more jobs
    if (sh_run) {
      if (sh_nops < a.ops_cap) a.ops[sh_nops] = sh_run;
      ++sh_nops;
    }
    a.out[0] = sh_nops;
    a.out[1] = (unsigned long long)sh_i;
    a.out[2] = (unsigned long long)sh_j;
    a.out[3] = tiles;
    a.out[4] = sh_hits;
  }
}

// a walk buffer: from the context's persistent workspace when there is one (repeated calls
// skip cudaMalloc / cudaFree), else allocated for this call
struct DBuf {
  void* p = nullptr;
  bool own = false;
  cudaError_t get(LongWs* ws, int slot, size_t bytes) {
    if (ws) return ws->get(slot, bytes, &p);
    own = true;
    return cudaMalloc(&p, bytes);
  }
  ~DBuf() { if (own && p) cudaFree(p); }
};

}  // namespace

#define TK(call)                                                        \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) {                                            \
      *err = std::string(#call) + ": " + cudaGetErrorString(e_);        \
      return e_ == cudaErrorMemoryAllocation ? ANYSEQ_E_NOMEM : ANYSEQ_E_CUDA; \
    }                                                                   \
  } while (0)

int run_long_traceback(const LongDevice& dev, const DevParams& P, const int8_t sig[25],
                       const LongCkpt& ck, int64_t end_i, int64_t end_j, int64_t n, int64_t m,
                       std::vector<uint32_t>* ops, int64_t* begin_i, int64_t* begin_j,
                       double* walk_ms, std::string* err, uint64_t* launches, int walk_helpers,
                       int64_t* tiles, int64_t* hits, bool trace) {
  const auto t0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (trace)
      fprintf(stderr, "[tb-walk] %s %.1f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  TK(cudaSetDevice(dev.id));
  cudaStream_t st = dev.stream;
  ops->clear();
  *begin_i = end_i;
  *begin_j = end_j;
  if (end_i == 0 && end_j == 0) return 0;
  const int TH = ck.HS * ck.ck_every;
  const int TR = TH / NT;
  if (TR != 2 && TR != 4 && TR != 8 && TR != 16) {
    *err = "long traceback: unsupported row block height";
    return ANYSEQ_E_UNSUPPORTED;
  }
  WalkArgs a;
  memset(&a, 0, sizeof(a));
  a.kind = P.kind;
  a.affine = P.gap == GAFFINE;
  a.go = P.go;
  a.ge = P.ge;
  a.cop = P.go + P.ge;
  memcpy(a.sig, sig, 25);
  a.qc = ck.qc;
  a.sc = ck.sc;
  a.n = (int)n;
  a.m = (int)m;
  a.rowck = ck.rowck;
  a.colck = ck.colck;
  a.TH = TH;
  a.PT = ck.PT;
  a.kc_shift = ck.kc_shift;
  a.end_i = (int)end_i;
  a.end_j = (int)end_j;
  const size_t scratch = ((size_t)(1 << ck.kc_shift) + NT) * NT * (((TR + 3) / 4) * 4);
  DBuf sb, ob, outb, slotb, syncb, jobb;
  TK(sb.get(dev.ws, WS_TB_SCRATCH, scratch));
  const uint64_t cap = (uint64_t)(n + m + 2);
  TK(ob.get(dev.ws, WS_TB_OPS, cap * sizeof(uint32_t)));
  TK(outb.get(dev.ws, WS_TB_OUT, 8 * sizeof(unsigned long long)));
  TK(cudaMemsetAsync(outb.p, 0, 8 * sizeof(unsigned long long), st));
  // helper CTAs: whole-tile recomputes of the predicted next tiles (option walk_helpers)
  const int helpers = std::max(0, std::min(walk_helpers, dev.num_sms - 1));
  if (helpers > 0) {
    TK(slotb.get(dev.ws, WS_TB_SLOTS, (size_t)NSLOT * scratch));
    TK(syncb.get(dev.ws, WS_TB_SYNC, (4 + NSLOT) * sizeof(int)));
    TK(cudaMemsetAsync(syncb.p, 0, 4 * sizeof(int), st));
    TK(cudaMemsetAsync((int*)syncb.p + 4, 0xFF, NSLOT * sizeof(int), st));
    TK(jobb.get(dev.ws, WS_TB_JOBS, (size_t)JMAX * sizeof(int2)));
  }
  a.slots = (uint8_t*)slotb.p;
  a.slot_bytes = scratch;
  a.nrowck = (ck.S - 1) / ck.ck_every;
  a.ncolck = (int)((m - 1) >> ck.kc_shift);
  a.sync = (int*)syncb.p;
  a.slot_job = helpers > 0 ? (int*)syncb.p + 4 : nullptr;
  a.jobs = (int2*)jobb.p;
  a.scratch = (uint8_t*)sb.p;
  a.ops = (uint32_t*)ob.p;
  a.ops_cap = cap;
  a.out = (unsigned long long*)outb.p;
  mark("buffers");
  cudaEvent_t e0, e1;
  TK(cudaEventCreate(&e0));
  TK(cudaEventCreate(&e1));
  TK(cudaEventRecord(e0, st));
  const size_t smem = (size_t)KC_MAX * sizeof(int2);
  switch (TR) {
    case 2:
      TK(cudaFuncSetAttribute(tile_walk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      tile_walk_kernel<2><<<1 + helpers, NT, smem, st>>>(a);
      break;
    case 4:
      TK(cudaFuncSetAttribute(tile_walk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      tile_walk_kernel<4><<<1 + helpers, NT, smem, st>>>(a);
      break;
    case 8:
      TK(cudaFuncSetAttribute(tile_walk_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      tile_walk_kernel<8><<<1 + helpers, NT, smem, st>>>(a);
      break;
    default:
      TK(cudaFuncSetAttribute(tile_walk_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      tile_walk_kernel<16><<<1 + helpers, NT, smem, st>>>(a);
      break;
  }
  TK(cudaGetLastError());
  TK(cudaEventRecord(e1, st));
  *launches += 1;
  unsigned long long out[8];
  TK(cudaMemcpyAsync(out, outb.p, sizeof(out), cudaMemcpyDeviceToHost, st));
  TK(cudaStreamSynchronize(st));
  mark("kernel synced");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *walk_ms = ms;
  if (out[0] > cap) {
    *err = "long traceback: walk overflowed its op buffer";
    return ANYSEQ_E_CUDA;
  }
  ops->resize(out[0]);
  if (out[0]) TK(cudaMemcpy(ops->data(), ob.p, out[0] * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  // walk order is end -> begin: reverse into alignment order
  for (size_t x = 0, y = ops->size(); x + 1 < y; ++x, --y) std::swap((*ops)[x], (*ops)[y - 1]);
  mark("ops copied");
  *begin_i = (int64_t)out[1];
  *begin_j = (int64_t)out[2];
  if (tiles) *tiles = (int64_t)out[3];
  if (hits) *hits = (int64_t)out[4];
  if (helpers > 0) {
    int ab = 0;
    TK(cudaMemcpy(&ab, (int*)syncb.p + 3, sizeof(int), cudaMemcpyDeviceToHost));
    if (ab) {
      *err = "long traceback: a walk wait exceeded its bound";
      return ANYSEQ_E_TIMEOUT;
    }
  }
  return 0;
}

}  // namespace anyseq
