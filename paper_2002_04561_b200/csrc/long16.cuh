// csrc/long16.cuh -- long-pair score-only kernel in 16-bit differential arithmetic, every
// kind and gap model (included inside namespace anyseq by the
// long16_*.cu instance files after long_dev.cuh).
//
// Paper: 16-bit scores where the value range allows (SIMD lanes of half
// width double the cells per instruction).  Long pairs exceed 16 bits absolutely, so the
// kernel keeps every value relative to a per-warp base: the DP only compares sums of
// neighbouring cells, and neighbouring H values differ by at most d = G_o + G_e + max(σ,0)
// (the Lipschitz bound holds for the local, global and semi-global
// recurrences alike), so the cells a warp holds at one step fit in s16.
//
// Same task shell as long_kernel (tickets, tagged row hand-off, boundary columns, flags,
// bounded waits).  What changes is the warp's inner layout: lane t owns 2·NR rows of the
// task; rows [0, NR) live in the low halves of its NR registers, rows [NR, 2NR) in the high
// halves, and the high half runs ONE COLUMN BEHIND the low half (at step k the low half
// relaxes column k − 2t, the high half column k − 2t − 1).  That makes the two halves 64
// "virtual lanes" of one anti-diagonal wavefront: the high half's upper neighbour is its own
// low half of the previous step, the low half's is lane t−1's high half (one shuffle), so
// every s16x2 instruction relaxes two independent cells.
//
// Values are kept strictly negative (rel = abs − base ∈ [−24576, −1]): then H − (G_o+G_e)
// can be formed on the FMA pipe as one 32-bit IMAD on the packed register (the low half
// always borrows, the constant pre-compensates the high half), leaving the ALU pipe per two
// cells: PRMT (σ of both halves), 3 VIADDMNMX.S16x2 and one max (VIMNMX3.S16x2 with the
// local floor, VIMNMX.S16x2 otherwise).  Linear gaps run as affine with G_o = 0: the
// reassociated recurrence below is then exactly Eqs. (2)-(3) (E = H_up − g, F = H_left − g).
// The base is re-chosen every 32 steps once all virtual lanes are active (warp max of H →
// −margin).
//
// Optimum (readings R5/R10): LOCAL tracks a packed running maximum per half (one
// VIMNMX3 per two registers) resolved to (value, i, j) in a rare branch.  SEMI places its
// pad rows at the TOP of the first strip (σ = 0 rows that reproduce the zero row 0
// exactly), so the matrix's last row n is the last row strip's published row: after the
// kernel the row buffer holds H(n, j) for every j, the last column strip writes H(i, m) to
// one more boundary column, and semi_reduce_kernel scans both in the candidate order of
// R5.  GLOBAL reads H(n, m) at the last task's last column.
#pragma once

__device__ __forceinline__ uint32_t h16_set(uint32_t x, int h, int v) {
  return h ? ((x & 0xffffu) | ((uint32_t)v << 16)) : ((x & 0xffff0000u) | ((uint32_t)v & 0xffffu));
}
__device__ __forceinline__ int h16_get(uint32_t x, int h) {
  return (int)(int16_t)(uint16_t)(h ? (x >> 16) : (x & 0xffffu));
}
__device__ __forceinline__ uint32_t h16_pack(int lo, int hi) {
  return ((uint32_t)lo & 0xffffu) | ((uint32_t)hi << 16);
}

// CKPT (linear-space traceback): the pass also keeps the
// checkpoints the traceback's tile recompute starts from -- every ck_every-th row strip's
// last row, (H, E) of that row (a.rowck), and every 2^kc_shift-th column, (H, F) of every
// row (a.colck) -- in absolute 32-bit values.
#ifndef LONG16_MINB
#define LONG16_MINB 3  // resident blocks per SM asked of ptxas for 1024-row tasks (A/B builds: 4)
#endif
// MULTI: one launch over the tasks of several pairs (same
// scheme and kind): a_.pairs[p] holds pair p's arguments; tickets run through segments
// a_.segs[k] = (pair, column pass) -- every pair's pass 0, then every pair's pass 1, ... --
// with a_.task_end the inclusive prefix of the segments' S, so a task is handed out only
// after every task of the passes to its left.  A warp merges its partial optimum into the
// pair's parts entry when its next ticket belongs to another pair.  Every task still waits
// only on lower tickets of its own pair, so the deadlock argument of one pair carries over.
template <int NR, int KIND, bool CKPT = false, bool MULTI = false>
__global__ void __launch_bounds__(128, (NR <= 12 || (LONG16_MINB > 3 && !CKPT)) ? 4 : 3)
    long16_kernel(LongArgs a_) {
  constexpr int HS = 64 * NR;  // rows per task: 32 lanes x 2 halves x NR
  constexpr int RING = 256;
  constexpr int PER = 32;
  __shared__ int2 ring_he[4][RING];
  // full PRMT selector of a column c for the two halves: codes of c (low half) and c - 1
  // (high half, one column behind), sign-replicating (VS16::selector)
  // (each ring has a mirror of its first MIR entries after the end: the steady-state step
  // reads through a pointer advanced by an IMAD and re-based once per period)
  constexpr int MIR = 64;
  __shared__ uint32_t ring_sel[4][RING + MIR];
  // OFF-phase steps: lane 0's input (H, E of the row above) already in the warp's relative
  // frame, packed (h | e << 16), converted once per refill period right after re-basing
  __shared__ uint32_t ring_rel[4][RING + MIR];
  __shared__ int2 ring_out[4][64];        // the task's last row (H, E) awaiting publication
  __shared__ int ring_eck[CKPT ? 4 : 1][64];  // CKPT: E of that row itself (not of the next)
  __shared__ int4 ring_pf[4][64];  // row hand-off entries fetched (cp.async) ahead of need
  const int t = threadIdx.x & 31;
  const int wb = threadIdx.x >> 5;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const DevParams P = a_.P;
  const int cop = P.go + P.ge;
  const uint32_t NGE2 = VS16::splat(-P.ge);
  const uint32_t one = (uint32_t)a_.one;
  const int hopc = a_.hopc;  // packed (-cop, -cop) with the low half's borrow pre-compensated
  auto hop = [&](uint32_t h) -> uint32_t { return (uint32_t)imad_add_s((int)h, one, hopc); };
  const int NEGc = a_.neg16;
  // subject codes of columns past a task's end are read (and ignored) by the warp's last
  // steps: keep every ring entry a valid code so the active half's selector stays intact
  for (int x = t; x < RING + MIR; x += 32) {
    ring_sel[wb][x] = 0xC480u;
    if (x < RING) ring_he[wb][x] = make_int2(0, 0);
    ring_rel[wb][x] = 0;
  }
  const uint32_t sel_smem = (uint32_t)__cvta_generic_to_shared(&ring_sel[wb][0]);
  const uint32_t rel_smem = (uint32_t)__cvta_generic_to_shared(&ring_rel[wb][0]);
  const uint32_t out_smem = (uint32_t)__cvta_generic_to_shared(&ring_out[wb][0]);
  auto lds32 = [](uint32_t addr) -> uint32_t {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
  };
  __syncwarp();

  LongPart part;
  part.lv = 0; part.li = 0; part.lj = 0;
  part.rv = 0; part.rj = 0; part.cv = 0; part.ci = 0; part.gv = 0; part.gset = 0; part.pad_ = 0;

  // the warp's partial optimum -> its entry in parts (warp-collective)
  auto flush_part = [&](LongPart* parts, bool merge) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int lv = __shfl_xor_sync(0xffffffffu, part.lv, o);
      const int li = __shfl_xor_sync(0xffffffffu, part.li, o);
      const int lj = __shfl_xor_sync(0xffffffffu, part.lj, o);
      if (lkey_better(lv, li, lj, part.lv, part.li, part.lj)) { part.lv = lv; part.li = li; part.lj = lj; }
      const int gv = __shfl_xor_sync(0xffffffffu, part.gv, o);
      const int gs = __shfl_xor_sync(0xffffffffu, part.gset, o);
      if (gs && !part.gset) { part.gv = gv; part.gset = 1; }
    }
    if (t == 0) {
      if (merge) {  // MULTI: the warp's earlier passes over the same pair
        const LongPart q = parts[wg];
        if (lkey_better(q.lv, q.li, q.lj, part.lv, part.li, part.lj)) { part.lv = q.lv; part.li = q.li; part.lj = q.lj; }
        if (q.gset && !part.gset) { part.gv = q.gv; part.gset = 1; }
      }
      parts[wg] = part;
    }
  };
  int cur = 0;     // MULTI: segment of the warp's last ticket
  int cpair = -1;  // MULTI: pair of the warp's last task
  for (;;) {
    int task = 0;
    if (t == 0) task = atomicAdd(a_.ticket, 1);
    task = __shfl_sync(0xffffffffu, task, 0);
    if (task >= (MULTI ? a_.task_total : a_.S * a_.g_count)) break;
    if (*(volatile int*)a_.abort_flag) break;
    if (task == a_.stall_task) continue;  // fault injection (option long_stall_task)
    LongArgs am;  // MULTI: this task's pair
    if constexpr (MULTI) {
      while (task >= a_.task_end[cur]) ++cur;
      const int2 sg = a_.segs[cur];  // (pair, column pass)
      if (sg.x != cpair) {
        if (cpair >= 0) flush_part(a_.pairs[cpair].parts, true);
        part.lv = 0; part.li = 0; part.lj = 0; part.gv = 0; part.gset = 0;
        cpair = sg.x;
      }
      am = a_.pairs[sg.x];
      task = sg.y * am.S + task - (cur > 0 ? a_.task_end[cur - 1] : 0);
      ANY_CHECK(sg.y < am.g_count && task >= sg.y * am.S && task < (sg.y + 1) * am.S);
    }
    const LongArgs& a = MULTI ? am : a_;
    const int n = a.n;
    const long long task_t0 = (a.prof && t == 0) ? clock64() : 0;
    const int s = task % a.S;
    const int g = a.g_first + task / a.S;
    const int c_lo = a.cb[g], c_hi = a.cb[g + 1], W = c_hi - c_lo;
    // real row of the lane's first row, minus 1 (SEMI: a.pad_top pad rows above row 1)
    const int ip0 = s * HS + t * 2 * NR - a.pad_top;
    const int2* bl = a.bcol[g];
    // right edge: the next strip's left boundary; SEMI's last strip: column m (candidates)
    int2* br = (g + 1 < a.Gtot || KIND == KSEMI) ? a.bcol[g + 1] : nullptr;

    if (g > 0) {
      if (!warp_wait<true>(&a.bflag[g][s], 1, a)) break;
      if (s > 0 && !warp_wait<true>(&a.bflag[g][s - 1], 1, a)) break;
    }
    uint32_t p0[NR], p1[NR], H[NR], Ff[NR];  // H: the lane's rows at its last column (in place)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int iA = ip0 + r + 1, iB = ip0 + NR + r + 1;  // real rows (1-based)
      p0[r] = (iA >= 1 && iA <= n) ? prof4(a_.P, a.qc[iA - 1]) : 0u;  // sigma rows, low half
      p1[r] = (iB >= 1 && iB <= n) ? prof4(a_.P, a.qc[iB - 1]) : 0u;  // ... and high half
      H[r] = VS16::splat(NEGc);
      Ff[r] = VS16::splat(NEGc);
    }
    int last_code = 0;  // subject code of the column before the next refill's first
    // subject codes of columns [c0, c1) -> full selectors in the ring (first strip: lane 0's
    // input row 0 as well)
    auto codes = [&](int c0, int c1) {
      const int c = c0 + t;
      const bool mine = c < c1;
      const int code = mine ? a.sc[c_lo + c] : 0;
      int pcode = __shfl_up_sync(0xffffffffu, code, 1);
      if (t == 0) pcode = last_code;
      last_code = __shfl_sync(0xffffffffu, code, (c1 - 1 - c0) & 31);  // code of column c1 - 1
      if (mine) {
        const uint32_t v = (uint32_t)code * 0x11u + (uint32_t)pcode * 0x1100u + 0xC480u;
        ring_sel[wb][c & (RING - 1)] = v;
        if ((c & (RING - 1)) < MIR) ring_sel[wb][RING + (c & (RING - 1))] = v;
      }
      // the high half relaxes column W - 1 one step after the low half left the task: its
      // selector (entry W) carries code(W - 1) in the high nibbles
      if (c1 == W && t == 0) {
        const uint32_t v = (uint32_t)last_code * 0x1100u + 0xC480u;
        ring_sel[wb][W & (RING - 1)] = v;
        if ((W & (RING - 1)) < MIR) ring_sel[wb][RING + (W & (RING - 1))] = v;
      }
      if (s == 0 && mine) {
        const int h0 = KIND == KGLOBAL ? -(P.go + (c_lo + c + 1) * P.ge) : 0;
        ring_he[wb][c & (RING - 1)] = make_int2(h0, h0 - cop);
      }
    };
    // the hand-off entries of [c0, c1) (s > 0): poll until every entry carries tag s
    auto handoff = [&](int c0, int c1, int4 v) -> bool {
      const int c = c0 + t;
      const bool mine = c < c1;
      if (!mine) v = make_int4(0, s, 0, s);
      const int4* src = a.rowbuf + c_lo + c + 1;
      long long spins = 0;
      while (!__all_sync(0xffffffffu, v.y == s && v.w == s)) {
        const long long t0 = (a.prof && t == 0) ? clock64() : 0;
        if (v.y != s || v.w != s) v = ld_row(src);
        if (!__all_sync(0xffffffffu, v.y == s && v.w == s)) __nanosleep(a.sleep_ns);
        if ((++spins & 255) == 0 &&
            __any_sync(0xffffffffu, spins > a.spin_limit || *(volatile int*)a.abort_flag)) {
          if (t == 0) atomicExch(a.abort_flag, 1);
          return false;
        }
        if (a.prof && t == 0)  // [0]: mid-task waits, [3]: the task's first two refills
          atomicAdd(&a.prof[c0 < 2 * PER ? 3 : 0], (unsigned long long)(clock64() - t0));
      }
      if (mine) ring_he[wb][c & (RING - 1)] = make_int2(v.x, v.z);
      return true;
    };
    auto refill = [&](int c0, int c1) -> bool {  // synchronous (the task's first two periods)
      if (c0 >= c1) return true;  // (the task's second initial refill when W <= 32)
      codes(c0, c1);
      if (s == 0) return true;
      const int c = c0 + t;
      return handoff(c0, c1, c < c1 ? ld_row(a.rowbuf + c_lo + c + 1) : make_int4(0, s, 0, s));
    };
    // Non-blocking hand-off for the rest of the task: the next period's 32 entries are
    // requested (cp.async into ring_pf) two periods before lane 0 needs them and checked every
    // other step; entries the strip above has not published yet are requested again, and
    // the warp blocks (polls) only when the batch is due.  A strip that runs close behind
    // the strip above thereby keeps computing instead of spinning on the hand-off.
    int pf_next = 2 * PER;  // first column of the next batch to request
    int pf_b0 = -1;         // first column of the batch in flight (-1: none)
    auto pump = [&](int kk) -> bool {
      // a batch in flight is looked at every 8 steps until it is due (each look costs a
      // shared-memory pass over the entries, a vote and possibly a new request)
      if (pf_b0 >= 0 && ((kk & 7) == 0 || kk + 2 >= pf_b0)) {
        const int c1 = min(W, pf_b0 + PER), c = pf_b0 + t;
        cp_async_wait_all();
        int4 v = c < c1 ? ring_pf[wb][c & 63] : make_int4(0, s, 0, s);
        const bool ok = __all_sync(0xffffffffu, v.y == s && v.w == s);
        if (ok || kk + 2 >= pf_b0) {  // complete, or due: finish it (polling if needed)
          if (!handoff(pf_b0, c1, v)) return false;
          pf_next = pf_b0 + PER;
          pf_b0 = -1;
        } else if (c < c1 && (v.y != s || v.w != s)) {  // ask again for the missing ones
          cp_async16(&ring_pf[wb][c & 63], a.rowbuf + c_lo + c + 1);
          cp_async_commit();
        }
      }
      if (pf_b0 < 0 && pf_next < W && pf_next <= kk + 2 * PER) {
        const int c1 = min(W, pf_next + PER), c = pf_next + t;
        codes(pf_next, c1);
        if (s == 0) {
          pf_next += PER;
        } else {
          if (c < c1) cp_async16(&ring_pf[wb][c & 63], a.rowbuf + c_lo + c + 1);
          cp_async_commit();
          pf_b0 = pf_next;
        }
      }
      __syncwarp();
      return true;
    };
    // start slack (option long_start_lag, columns): tickets are taken in strip order, so the
    // strips of a round start one after the other and would run at the minimum distance the
    // hand-off allows (~4 refill periods) -- any hiccup of a strip then stalls the chain
    // below it.  Starting `lag` columns further behind gives every strip that much slack.
    if (s > 0 && a.lag > 0 && W > a.lag) {
      const int4* p = a.rowbuf + c_lo + a.lag;
      int ok = 1;
      if (t == 0) {
        long long spins = 0;
        while (ok) {
          const int4 v = ld_row(p);
          if (v.y == s && v.w == s) break;
          if ((++spins & 255) == 0 && (spins > a.spin_limit || *(volatile int*)a.abort_flag)) {
            atomicExch(a.abort_flag, 1);
            ok = 0;
          }
          __nanosleep(256);
        }
      }
      if (!__shfl_sync(0xffffffffu, ok, 0)) break;
    }
    if (!refill(0, min(W, PER)) || !refill(PER, min(W, 2 * PER))) break;
    __syncwarp();

    // frame: every value of the task lies within a.bspan of H(ip0, c_lo + 1) (the row
    // above, first column), so base = that + bspan puts them all in [-2 bspan, -margin]
    const int h00 = (s > 0) ? ring_he[wb][0].x
                            : (KIND == KGLOBAL ? -(P.go + (c_lo + 1) * P.ge) : 0);
    int base = h00 + a.bspan;
    auto cv = [&](int x) -> int { return max(x - base, NEGc); };  // absolute -> relative
    int bv0 = 0, bi0 = 0, bj0 = 0, bv1 = 0, bi1 = 0, bj1 = 0;   // per-half best (absolute)
    uint32_t Z = 0, best = 0;  // LOCAL: the floor (absolute 0) and the running maxima, relative
    auto frame_consts = [&]() {
      if (KIND == KLOCAL) {
        Z = VS16::splat(max(-base, NEGc));
        best = h16_pack(min(max(bv0 - base, -32768), 32767), min(max(bv1 - base, -32768), 32767));
      }
    };
    frame_consts();
    uint32_t diag = VS16::splat(NEGc), Hbot = VS16::splat(NEGc), Ebot = VS16::splat(NEGc);

    auto sweep = [&]() -> bool {
      uint32_t sel_nx = ring_sel[wb][(0 - 2 * t) & (RING - 1)];
      int2 he_nx = ring_he[wb][0];
      uint32_t rel_nx = 0;
      uint32_t psel = 0, prel = 0;  // OFF steps: addresses of the next selector / input entries
      uint32_t pout = 0;            // OFF steps: staging slot of the task's last row
      uint32_t peck = 0;            // CKPT, OFF steps: staging slot of its E
      // LOCAL, OFF steps: track the running maximum in this period?  Skipped when no cell
      // of the period can exceed it (see convert).  Only the 1024-row instances: in the
      // 512-row ones (128 registers) the extra live state cost more than the skip saved
      // (1 Mbp local affine 0.64 -> 0.87 s)
      constexpr bool SKIPTRK = NR >= 16;
      bool trk = true;
      int kck = -8;  // CKPT, OFF steps: the step whose low half (this step) or high half
                     // (next step) is at a checkpoint column, found once per period
      auto step = [&](auto chk, const int k) {
        uint32_t (&Hi)[NR] = H;
        uint32_t (&Hq)[NR] = H;
        constexpr bool CHK = decltype(chk)::value;
        const int lc = k - 2 * t;  // low half's column (task-relative); high half: lc - 1
        const uint32_t sel = sel_nx;
        if (CHK) {
          sel_nx = ring_sel[wb][(lc + 1) & (RING - 1)];
        } else {
          sel_nx = lds32(psel);
          psel = (uint32_t)imad_add_s((int)psel, one, 4);
        }
        uint32_t hin, ein;
        int2 he = make_int2(0, 0);
        if (CHK) {
          const uint32_t hs = __shfl_up_sync(0xffffffffu, Hbot, 1);
          const uint32_t es = __shfl_up_sync(0xffffffffu, Ebot, 1);
          // low half <- lane t-1's high half (row above, same column); high half <- own
          // low half of the previous step (row above, one column behind)
          hin = __byte_perm(hs, Hbot, 0x5432);
          ein = __byte_perm(es, Ebot, 0x5432);
          he = he_nx;
          he_nx = ring_he[wb][(k + 1) & (RING - 1)];  // lane 0's next column
        } else {
          // lane 31's high half is nobody's input: it carries lane 0's input (pre-converted
          // ring entry) through the same rotating shuffle, so lane 0 needs no select
          const uint32_t rel = rel_nx;
          rel_nx = lds32(prel);
          prel = (uint32_t)imad_add_s((int)prel, one, 4);
          const uint32_t vh = prmt(Hbot, rel, t == 31 ? 0x5410u : 0x3210u);
          const uint32_t ve = prmt(Ebot, rel, t == 31 ? 0x7610u : 0x3210u);
          const uint32_t hs = __shfl_sync(0xffffffffu, vh, (t + 31) & 31);
          const uint32_t es = __shfl_sync(0xffffffffu, ve, (t + 31) & 31);
          hin = __byte_perm(hs, Hbot, 0x5432);
          ein = __byte_perm(es, Ebot, 0x5432);
        }
        const bool act0 = !CHK || (lc >= 0 && lc < W);
        const bool act1 = !CHK || (lc >= 1 && lc <= W);
        if (CHK && (lc == 0 || lc == 1)) {  // half h reaches the left boundary column
          const int h = lc;
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            const int i = ip0 + h * NR + r + 1;  // real row; pad rows: H = 0 (SEMI), F = -inf
            int2 b = make_int2(0, NEG32);
            // (SEMI pad rows read bl[0] = (H(0, c_lo), F) = (0, -inf): their own boundary)
            if (i <= n) b = bl[KIND == KSEMI ? max(i, 0) : i];
            Hi[r] = h16_set(Hi[r], h, cv(b.x));
            Ff[r] = h16_set(Ff[r], h, cv(b.y));
          }
          const int id = ip0 + h * NR;  // the row above the half's first row
          diag = h16_set(diag, h, cv(id <= n ? bl[KIND == KSEMI ? max(id, 0) : id].x : 0));
        }
        if (CHK) {  // lane 0's low half: the row above the task, H(ip0, j), E(ip0 + 1, j)
          const uint32_t hl = prmt((uint32_t)cv(he.x), hin, 0x7610u);
          const uint32_t el = prmt((uint32_t)cv(he.y), ein, 0x7610u);
          hin = t == 0 ? hl : hin;
          ein = t == 0 ? el : ein;
        }
        uint32_t e = ein;
        uint32_t hd = diag;
        uint32_t elast = 0;  // CKPT: E of the last row
#pragma unroll
        for (int r = 0; r < NR; ++r) {  // in place: row r's previous column is row r+1's diagonal
          if (CKPT && r == NR - 1) elast = e;
          const uint32_t old = Hi[r];
          const uint32_t sig = prmt(p0[r], p1[r], sel);
          Ff[r] = __viaddmax_s16x2(Ff[r], NGE2, hop(old));
          const uint32_t df = __viaddmax_s16x2(hd, sig, Ff[r]);
          Hq[r] = KIND == KLOCAL ? __vimax3_s16x2(df, e, Z) : __vmaxs2(df, e);
          e = __viaddmax_s16x2(e, NGE2, hop(df));
          hd = old;
        }
        diag = hin;
        Hbot = Hq[NR - 1];
        Ebot = e;
        // the task's last row (high half), column c = lc - 1: staged in shared memory slot
        // (c + 63) & 63 (= k & 63: a period's 32 steps never wrap), published 32 columns at
        // a time; OFF steps store through a pointer advanced by an IMAD
        if (CHK) {
          if (t == 31 && act1)
            ring_out[wb][(lc + 62) & 63] = make_int2(h16_get(Hq[NR - 1], 1) + base, h16_get(e, 1) + base);
        } else {
          if (t == 31) {
            asm volatile("st.shared.v2.s32 [%0], {%1, %2};" ::"r"(pout),
                         "r"(h16_get(Hq[NR - 1], 1) + base), "r"(h16_get(e, 1) + base)
                         : "memory");
            if (CKPT)
              asm volatile("st.shared.s32 [%0], %1;" ::"r"(peck), "r"(h16_get(elast, 1) + base)
                           : "memory");
          }
          pout = (uint32_t)imad_add_s((int)pout, one, 8);
          if (CKPT) peck = (uint32_t)imad_add_s((int)peck, one, 4);
        }
        if (CKPT && CHK && t == 31 && act1) ring_eck[wb][(lc + 62) & 63] = h16_get(elast, 1) + base;
        if (CKPT) {  // column checkpoints: (H, F) of every real row at columns j = k 2^kc_shift
          const int jl = c_lo + lc + 1;  // the low half's column; the high half's is jl - 1
          int h = -1;                    // the half at a checkpoint column this step
          if (CHK) {
            const int kcm = (1 << a.kc_shift) - 1;
            h = (((jl & kcm) == 0) && act0) ? 0 : ((((jl - 1) & kcm) == 0) && act1) ? 1 : -1;
          } else {  // OFF steps: the step was found once per period (convert)
            const unsigned dk = (unsigned)(k - kck);
            if (dk < 2u) h = (int)dk;
          }
          if (h >= 0) {
            const int jj = jl - h;
            if (jj < a.m) {
              ANY_CHECK(jj >= (1 << a.kc_shift) && ((jj >> a.kc_shift) - 1) < ((a.m - 1) >> a.kc_shift));
              int2* dst = a.colck + (size_t)((jj >> a.kc_shift) - 1) * (a.n + 1);
#pragma unroll
              for (int r = 0; r < NR; ++r) {
                const int i = ip0 + h * NR + r + 1;
                if (i >= 1 && i <= n)
                  dst[i] = make_int2(h16_get(Hq[r], h) + base, h16_get(Ff[r], h) + base);
              }
            }
          }
        }
        if (KIND == KLOCAL && (CHK || !SKIPTRK || trk)) {
          // local optimum: packed running maximum per half; strictly larger values only.
          // cmB = max over the half's rows but its first: when the first row holds the new
          // maximum (the common case where H falls down the rows, e.g. left of a similar
          // pair's diagonal, where a new maximum appears at every step) its row is known
          // without searching the others.
          uint32_t cm, cmB;
          if (CHK) {
            const uint32_t keep = (act0 ? 1u : 0u) | (act1 ? 2u : 0u);
            uint32_t mx = Hq[1];
#pragma unroll
            for (int r = 2; r + 1 < NR; r += 2) mx = __vimax3_s16x2(mx, Hq[r], Hq[r + 1]);
            if ((NR % 2) == 1) mx = __vmaxs2(mx, Hq[NR - 1]);
            cmB = VS16::select_mask(mx, keep, VS16::splat(-32768));
            cm = __vimax3_s16x2(VS16::select_mask(Hq[0], keep, VS16::splat(-32768)), cmB, best);
          } else {
            cmB = Hq[1];
#pragma unroll
            for (int r = 2; r + 1 < NR; r += 2) cmB = __vimax3_s16x2(cmB, Hq[r], Hq[r + 1]);
            if ((NR % 2) == 1) cmB = __vmaxs2(cmB, Hq[NR - 1]);
            cm = __vimax3_s16x2(Hq[0], cmB, best);
          }
          if (cm != best) {  // resolve (value, first row, column) of the improved half(s)
            // first row holding the new maximum, both halves at once (unless row 0 holds it
            // in every improved half): t = clamp(Hq[r] + 1 - cm, 0, 1) is 1 iff Hq[r] == cm
            // (Hq[r] <= cm), key = 64 t + 63 - r, and the largest key names the first such
            // row -- one DPX op and one IMAD per row instead of a compare-select per row and
            // half (the clamp keeps halves that did not improve from carrying into the other)
            const uint32_t ne = __vcmpne2(cm, best), first = __vcmpeq2(Hq[0], cm);
            uint32_t kmax = VS16::splat(127);  // row 0 in both halves
            if (ne & ~first) {
              const uint32_t om = __vsub2(VS16::splat(1), cm), k64 = one << 6;
              kmax = 0;
#pragma unroll
              for (int r = 0; r < NR; r += 2) {
                const uint32_t ka = (uint32_t)imad_add_s(
                    (int)__viaddmin_s16x2_relu(Hq[r], om, VS16::splat(1)), k64, (63 - r) * 0x10001);
                if (r + 1 < NR) {
                  const uint32_t kb = (uint32_t)imad_add_s(
                      (int)__viaddmin_s16x2_relu(Hq[r + 1], om, VS16::splat(1)), k64, (62 - r) * 0x10001);
                  kmax = __vimax3_s16x2(kmax, ka, kb);
                } else {
                  kmax = __vmaxs2(kmax, ka);
                }
              }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int v = h16_get(cm, h);
              if (v != h16_get(best, h)) {
                const int rr = 63 - (h16_get(kmax, h) & 63);
                if (h == 0) { bv0 = v + base; bi0 = ip0 + rr + 1; bj0 = c_lo + lc + 1; }
                else { bv1 = v + base; bi1 = ip0 + NR + rr + 1; bj1 = c_lo + lc; }
              }
            }
            best = cm;
          }
        }
        if (CHK && (lc == W - 1 || lc == W)) {  // half h's last column
          const int h = lc - (W - 1);
          if (br) {  // right edge (H, F) of the half's real rows
#pragma unroll
            for (int r = 0; r < NR; ++r) {
              const int i = ip0 + h * NR + r + 1;
              if ((KIND != KSEMI || i >= 1) && i <= n)
                br[i] = make_int2(h16_get(Hq[r], h) + base, h16_get(Ff[r], h) + base);
            }
          }
          if (KIND == KGLOBAL && s == a.S - 1 && c_hi == a.m) {  // H(n, m): the global optimum
            const int rr = n - 1 - ip0 - h * NR;
            if (rr >= 0 && rr < NR) {
              int v = 0;
#pragma unroll
              for (int r = 0; r < NR; ++r)
                if (r == rr) v = h16_get(Hq[r], h);
              part.gv = v + base;
              part.gset = 1;
            }
          }
        }
      };
      // re-choose the base: warp max of H over the (all active) halves -> -margin
      auto reframe = [&]() {
        uint32_t mx = H[0];
#pragma unroll
        for (int r = 1; r + 1 < NR; r += 2) mx = __vimax3_s16x2(mx, H[r], H[r + 1]);
        if ((NR % 2) == 0) mx = __vmaxs2(mx, H[NR - 1]);
        const int ml = max(h16_get(mx, 0), h16_get(mx, 1));
        const int M = __reduce_max_sync(0xffffffffu, ml);
        const int dl = M + a.margin;
        const uint32_t sub = VS16::splat(-dl);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          H[r] = __vadd2(H[r], sub);
          Ff[r] = __vadd2(Ff[r], sub);
        }
        Hbot = __vadd2(Hbot, sub);
        Ebot = __vadd2(Ebot, sub);
        diag = __vadd2(diag, sub);
        base += dl;
        frame_consts();
      };
      // lane 0's inputs of columns [c0, c0 + 32) in the current frame, packed (h | e << 16)
      auto convert = [&](int c0) {
        const int x = (c0 + t) & (RING - 1);
        const int2 v = ring_he[wb][x];
        const uint32_t r = h16_pack(cv(v.x), cv(v.y));
        ring_rel[wb][x] = r;
        if (x < MIR) ring_rel[wb][RING + x] = r;
        if (KIND == KLOCAL && SKIPTRK) {
          // every H of the coming period derives from the warp's current cells (max -margin
          // right after the re-base), the previous column's diagonal inputs and the input
          // row of columns [c0, c0 + 32), gaining at most max(sigma) per column along a
          // diagonal (gaps only lose, and E, F <= H): if that bound cannot pass the running
          // maximum of either half, the period needs no tracking
          const int top = __reduce_max_sync(
              0xffffffffu, max((int)(int16_t)(uint16_t)(r & 0xffffu),
                               max(h16_get(diag, 0), h16_get(diag, 1))));
          const int bound = max(top, -a.margin) + (PER + 4) * max(P.smax, 0);
          trk = bound > min(h16_get(best, 0), h16_get(best, 1));
        }
        __syncwarp();
        rel_nx = ring_rel[wb][c0 & (RING - 1)];
        // the OFF steps from c0 on read entries c0 + 1 ... (inputs) and k - 2t + 1 ...
        // (selectors) linearly: at most PER + 1 past the re-base, inside the mirror
        prel = rel_smem + 4u * (uint32_t)((c0 + 1) & (RING - 1));
        pout = out_smem + 8u * (uint32_t)(c0 & 63);
        if (CKPT) peck = (uint32_t)__cvta_generic_to_shared(&ring_eck[wb][c0 & 63]);
        // checkpoint columns are 2^kc_shift >= 512 apart: at most one per period and half;
        // the low half is at column c_lo + (k - 2t) + 1 (high half: one step later)
        if (CKPT) {
          const int kcm = (1 << a.kc_shift) - 1;
          kck = (c0 - 1) + ((2 * t - 1 - c_lo - (c0 - 1)) & kcm);
        }
        psel = sel_smem + 4u * (uint32_t)((c0 - 2 * t + 1) & (RING - 1));
      };

      // publish staged columns [flushed, c_end) (at most 32) to the row buffer for strip s+1
      int flushed = 0;
      const int ck_slot =
          (CKPT && s + 1 < a.S && ((s + 1) % a.ck_every) == 0) ? (s + 1) / a.ck_every - 1 : -1;
      auto flush = [&](int c_end) {
        __syncwarp();
        const int c = flushed + t;
        if (c < c_end) {
          const int2 v = ring_out[wb][(c + 63) & 63];
          ANY_CHECK(c_lo + c + 1 <= a.m);
          st_row(a.rowbuf + c_lo + c + 1, v.x, v.y, s + 1);
          ANY_CHECK(!CKPT || ck_slot < (a.S - 1) / a.ck_every);
          if (CKPT && ck_slot >= 0)  // row checkpoint: (H, E) of the strip's last row
            a.rowck[(size_t)ck_slot * (a.m + 1) + c_lo + c + 1] = make_int2(v.x, ring_eck[wb][(c + 63) & 63]);
        }
        flushed = c_end;
        __syncwarp();
      };
      const std::integral_constant<bool, true> ON{};
      const std::integral_constant<bool, false> OFF{};
      const int K = W + 63;
      const int kA = min(K & ~1, 64);          // every virtual lane has reached column 0
      const int kB = max(kA, (W - 1) & ~1);    // no virtual lane has reached column W-1
      int k = 0;
      for (; k < kA; k += 2) {
        if (!pump(k)) return false;
        step(ON, k);
        step(ON, k + 1);
      }
      for (; k < kB; k += 2) {
        // steady state: the hand-off pump runs every 8 steps and when a batch falls due (a
        // new batch is then requested at most 6 steps later, still ~2 periods ahead)
        if (((k & 7) == 0 || (pf_b0 >= 0 && k + 2 >= pf_b0)) && !pump(k)) return false;
        if ((k % PER) == 0) {
          reframe();
          convert(k);
          flush(min(W, k - 63));  // columns <= k - 64 are complete
        }
        step(OFF, k);
        step(OFF, k + 1);
      }
      he_nx = ring_he[wb][k & (RING - 1)];  // the CHK path's lane-0 input again
      for (; k + 1 < K; k += 2) {
        if (!pump(k)) return false;
        if ((k % PER) == 0 && k >= 64) flush(min(W, k - 63));
        step(ON, k);
        step(ON, k + 1);
      }
      if (k < K) step(ON, k);
      while (flushed < W) flush(min(W, flushed + 32));
      return true;
    };
    const bool done = sweep();
    if (!done) break;
    if (KIND == KLOCAL) {
      if (lkey_better(bv0, bi0, bj0, part.lv, part.li, part.lj)) { part.lv = bv0; part.li = bi0; part.lj = bj0; }
      if (lkey_better(bv1, bi1, bj1, part.lv, part.li, part.lj)) { part.lv = bv1; part.li = bi1; part.lj = bj1; }
    }
    if (a.prof && t == 0) {
      atomicAdd(&a.prof[1], (unsigned long long)(clock64() - task_t0));
      atomicAdd(&a.prof[2], 1ull);
    }
    __syncwarp();
    if (br && g + 1 < a.Gtot) {
      if (t == 0) {
        __threadfence_system();
        st_release_sys(&a.bflag[g + 1][s], 1);
      }
    }
  }
if (MULTI) {
    if (cpair >= 0) flush_part(a_.pairs[cpair].parts, true);
  } else {
    flush_part(a_.parts, false);
  }
}
