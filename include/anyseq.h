/*
 * include/anyseq.h -- C-ABI of the B200-native pairwise alignment library.
 *
 * The library relaxes the dynamic-programming matrix of AnySeq (arXiv 2002.04561):
 *   H(i,j) = max{ H(i-1,j-1) + sigma(q_i,s_j), E(i,j), F(i,j), nu }        Eq. (1)
 *   linear gaps  E = H(i-1,j) - g,  F = H(i,j-1) - g                       Eqs. (2)-(3)
 *   affine gaps  E = max{E(i-1,j) - Ge, H(i-1,j) - Go - Ge}, F alike      Eqs. (4)-(5)
 *   local (nu = 0), global (nu = -inf), semi-global (local init, optimum in last row/col)
 *                                                                           P:257-264
 * The entry points follow the paper's C wrapper (construct_global_alignment)
 * and its control flow (allocate / read input, build accessors, relax, look up optimum,
 * build alignment, output -- P:424-436).  Parameters select the algorithmic variant at
 * run time (the paper selects it by partial evaluation).
 *
 * Conventions:
 *  - gap_open / gap_extend are NON-NEGATIVE MAGNITUDES that are subtracted;
 *    a gap of length k costs gap_open + k*gap_extend.  "open -5 / extend -1"
 *    means gap_open = 5, gap_extend = 1.  For LINEAR, gap_extend is g and gap_open is
 *    ignored.
 *  - rows are the query q (i = 1..n), columns the subject s (j = 1..m).
 *  - CIGAR ops are BAM-style words (len << 4 | op) with op 0 = M (q_i vs s_j, match or
 *    mismatch), 1 = I (q_i vs gap, vertical / E), 2 = D (s_j vs gap, horizontal / F).
 *  - ties: H source DIAG > E > F; gap extension beats opening; local traceback stops at
 *    the first cell with H <= 0; end cell = maximum with smallest j, then smallest i
 *    (semi-global candidates: row n for j < m, then column m).
 *  - alphabet: A C G T N (case-insensitive).  N mismatches everything, N included.
 *
 * Ownership: the caller owns every input and output buffer; the library keeps no pointer
 * after a call returns.  The context owns device memory, streams and peer mappings.
 * Host-pointer calls are synchronous.  One call at a time per context.
 * Errors: every function returns anyseq_status; no exceptions, aborts or exits cross the
 * ABI.  Validation happens before any result is written; on error, outputs are
 * unspecified and anyseq_last_error() names the failing pair / byte / CUDA call.
 * There is NO CPU fallback: without a CUDA device anyseq_create returns ANYSEQ_E_CUDA.
 */
#ifndef ANYSEQ_H
#define ANYSEQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct anyseq_ctx anyseq_ctx; /* opaque: devices, streams, scratch, peers */

typedef enum {
  ANYSEQ_OK = 0,
  ANYSEQ_E_INVALID = 1,     /* bad enum, penalty, pointer, size */
  ANYSEQ_E_BADSEQ = 2,      /* byte outside ACGTNacgtn */
  ANYSEQ_E_NOMEM = 3,       /* device or host allocation failed */
  ANYSEQ_E_CAPACITY = 4,    /* cigar buffer too small (*cigar_used = words required) */
  ANYSEQ_E_CUDA = 5,        /* CUDA runtime error (message names the call) */
  ANYSEQ_E_UNSUPPORTED = 6, /* score range exceeds 32-bit arithmetic, etc. */
  ANYSEQ_E_PEER = 7,        /* peer access between devices unavailable */
  ANYSEQ_E_TIMEOUT = 8      /* a device-side wait exceeded its bound */
} anyseq_status;

typedef enum { ANYSEQ_GLOBAL = 0, ANYSEQ_LOCAL = 1, ANYSEQ_SEMIGLOBAL = 2 } anyseq_kind;
typedef enum { ANYSEQ_GAP_LINEAR = 0, ANYSEQ_GAP_AFFINE = 1 } anyseq_gap;

/* Alignment scheme. */
typedef struct {
  int32_t kind;       /* anyseq_kind */
  int32_t gap;        /* anyseq_gap */
  int32_t match;      /* sigma(a,a), a in ACGT; [-128, 127] */
  int32_t mismatch;   /* sigma(a,b), a != b, and every pair involving N; [-128, 127] */
  int32_t gap_open;   /* G_o >= 0 (ignored for LINEAR); <= 32767 */
  int32_t gap_extend; /* G_e >= 0 (LINEAR: g); <= 32767 */
  /* Matrix scoring: if has_subst != 0, sigma(a, b) = subst[5*a + b] for codes
     A,C,G,T,N = 0..4 (each in [-128, 127]) and match / mismatch are ignored. */
  int32_t has_subst;
  int32_t subst[25];
} anyseq_params;

/* CSR batch: pair k is q[q_off[k] .. q_off[k+1]) vs s[s_off[k] .. s_off[k+1]).
   Offsets have num_pairs + 1 entries, non-decreasing; each length < 2^31. */
typedef struct {
  const char* q;
  const uint64_t* q_off;
  const char* s;
  const uint64_t* s_off;
  uint64_t num_pairs;
} anyseq_batch;

/* One alignment.  Aligned q = [q_begin, q_end), aligned s = [s_begin, s_end), 0-based
   (equivalently the begin and end DP cells (q_begin, s_begin) -> (q_end, s_end)). */
typedef struct {
  int32_t score;
  int32_t reserved;
  int64_t q_begin, s_begin;
  int64_t q_end, s_end;
  uint64_t cigar_offset; /* index of the first op word in the caller's cigar[] */
  uint32_t cigar_len;    /* number of op words */
  uint32_t reserved2;
} anyseq_alignment;

/* Create a context on the given CUDA devices (device_ids may be NULL => device 0).
   num_devices >= 1.  A context with G > 1 devices shards batches by cumulative cells
   and long pairs as column strips. */
anyseq_status anyseq_create(anyseq_ctx** out, const int* device_ids, int num_devices);
void anyseq_destroy(anyseq_ctx* ctx);

/* Score-only batch alignment (step 7-8 of P:424-436 + output).  All pointers are HOST
   memory (pinned memory gives the fastest upload).  scores[num_pairs] receives the
   optimum; if ends != NULL, ends[k] also receives score and END cell (q_end, s_end);
   its begin/cigar fields are set to the end cell / 0. */
anyseq_status anyseq_align_batch(anyseq_ctx* ctx, const anyseq_params* params,
                                 const anyseq_batch* batch, int32_t* scores,
                                 anyseq_alignment* ends);

/* Same computation on DEVICE memory of the context's first device, enqueued on the
   caller's CUDA stream (cudaStream_t passed as void*; NULL = legacy default stream).
   d_batch points to a HOST struct whose q, q_off, s, s_off are DEVICE pointers.
   d_scores / d_ends are DEVICE pointers (d_ends may be NULL).  Asynchronous: returns
   after enqueueing; validation errors in the sequence bytes are reported by the NEXT
   call to anyseq_sync(ctx) (returns ANYSEQ_E_BADSEQ) or by the host API. */
anyseq_status anyseq_align_batch_device(anyseq_ctx* ctx, const anyseq_params* params,
                                        const anyseq_batch* d_batch, int32_t* d_scores,
                                        anyseq_alignment* d_ends, void* stream);

/* Full alignment with traceback (predecessor walk) for a batch.
   out[num_pairs] (host), cigar[cigar_capacity] (host).  cigar_capacity >= sum(n_k + m_k)
   always suffices; if smaller, returns ANYSEQ_E_CAPACITY with *cigar_used = words
   required.  Otherwise *cigar_used = words written.  Pairs of >= "batch_long_cells_tb"
   cells (both sides >= "batch_long_min") take the long-pair traceback (SURVEY 8(f) f1/f4:
   one shared checkpointing pass on one device, then a tile walk per pair); the results are
   the same alignments (same optimum and tie rules). */
anyseq_status anyseq_traceback(anyseq_ctx* ctx, const anyseq_params* params,
                               const anyseq_batch* batch, anyseq_alignment* out,
                               uint32_t* cigar, uint64_t cigar_capacity, uint64_t* cigar_used);

/* Long-pair score-only alignment (tiled wavefront) of host
   sequences q[0..n) and s[0..m).  out receives score and end cell (cigar_len = 0).
   Every kind and gap model runs the 16-bit differential kernel (reading
   R21/R24: values relative to a per-warp frame, exact by the Lipschitz bound) unless the
   subject holds N or option "long_narrow" = 0; those take the 32-bit kernel.
   ANYSEQ_E_UNSUPPORTED if the score range could exceed int32 (R11); ANYSEQ_E_TIMEOUT if a
   bounded inter-warp wait expires (device state stays valid). */
anyseq_status anyseq_align_long(anyseq_ctx* ctx, const anyseq_params* params, const char* q,
                                uint64_t n, const char* s, uint64_t m, anyseq_alignment* out);

/* Long-pair alignment WITH traceback in linear space (the paper's long
   genome traceback workload, Fig. 5a), every kind, linear and affine gaps.
   Default method: one forward pass of the 16-bit long kernel (Eqs. (1)-(5),
   P:224-255) that also writes checkpoints -- (H, E) of every ck_every-th strip's last row
   and (H, F) of every 2^kc_shift-th column -- within the "tb_ckpt_bytes" budget (default:
   a share of free device memory); then a walk kernel that starts at the optimum's cell,
   recomputes one checkpoint tile at a time in shared memory (helper CTAs recompute the
   predicted next tiles ahead of it) and re-derives every decision of the relax listing
   (readings R7-R9) -- the same tie rules as anyseq_traceback, so the CIGAR is
   the oracle's bit for bit.  Fallback when no 16-bit pass applies (subject with N, range
   guard): Hirschberg's divide and conquer with GPU last-row passes for linear gaps.
   out receives score, begin/end cells, cigar_offset 0 and cigar_len; cigar[] (host)
   receives the ops.  Host inputs as anyseq_align_long.
   Errors: ANYSEQ_E_UNSUPPORTED for affine gaps on the fallback path and when the score
   range could exceed int32; ANYSEQ_E_NOMEM if even the coarsest checkpoint geometry
   exceeds the budget; ANYSEQ_E_CAPACITY with *cigar_used = words required;
   ANYSEQ_E_BADSEQ for a byte outside ACGTNacgtn; ANYSEQ_E_TIMEOUT if a bounded wait
   expires. */
anyseq_status anyseq_traceback_long(anyseq_ctx* ctx, const anyseq_params* params, const char* q,
                                    uint64_t n, const char* s, uint64_t m, anyseq_alignment* out,
                                    uint32_t* cigar, uint64_t cigar_capacity,
                                    uint64_t* cigar_used);

/* Wait for all device work of the context; reports deferred device-side errors. */
anyseq_status anyseq_sync(anyseq_ctx* ctx);

/* Number of kernels the context launched since creation (instrumentation). */
uint64_t anyseq_kernel_launches(const anyseq_ctx* ctx);

/* Instrumentation: with option "timing" = 1 the context brackets every fill (relaxation)
   launch with CUDA events (score mode with several concurrent variant launches: one
   interval from the first start to the last end).  anyseq_get_stat reads "fill_ms"
   (summed device time of fill intervals), "fill_launches", "walk_ms"; anyseq_reset_stats
   clears them.  "timing" = 2 also prints a per-chunk event timeline of the host API to
   stderr (debug).  After anyseq_align_long: "long_kernel_ms" (device time of the long
   kernel, max over devices) and "long_narrow" (1 if the 16-bit differential kernel ran).
   After anyseq_align_batch: "long_multi_pairs" (long pairs the shared launch aligned) and
   "long_multi_ms" (its device time), "long_multi_rows" (rows per warp task, 512 or 1024).
   After anyseq_traceback_long: "tb_method" (1 checkpoints, 2 Hirschberg), "tb_pass_ms"
   (device time of the forward pass; Hirschberg: of the last-row passes summed over
   levels), "tb_pass_cells" (cells those passes relaxed), "tb_walk_ms" (device time of the
   walk kernel), "tb_ckpt_bytes", "tb_tiles" / "tb_hits" (tiles walked / found
   precomputed by the helper CTAs) and "tb_leaf_ms" (Hirschberg: host time of the batched
   leaf traceback).
   "h2d_bytes" / "d2h_bytes": bytes the host API copied host -> device (sequences as
   2-bit codes or ASCII, offsets) and device -> host (results) since the last reset.
   Returns ANYSEQ_E_INVALID for unknown names. */
anyseq_status anyseq_get_stat(anyseq_ctx* ctx, const char* name, double* value);
anyseq_status anyseq_reset_stats(anyseq_ctx* ctx);

/* Tunables; returns ANYSEQ_E_INVALID for unknown names.
     "chunk_bytes"       host API: bytes of sequence per upload chunk (default 64 MiB;
                         the first and last chunks are smaller)
     "pack2"             host API: 1 (default) packs ACGT-only chunks to 2-bit codes on
                         host threads and uploads those (a quarter of the bytes; the device
                         expands them); chunks with N or other bytes go up as ASCII.  0 =
                         always ASCII
     "pack2_percent"     share (by bytes) of the chunks that are packed; the rest go up as
                         ASCII DMA in parallel (0 = 100, the default)
     "tb_scratch_bytes"  traceback: device bytes of the per-cell H store per fill/walk
                         chunk (default 16 GiB; 1 B per cell with "tb8", else 2 B per cell
                         for s16x2 slots and 4 B for s32)
     "allow16"           0 forces 32-bit arithmetic (debug); "force_variant" (debug)
     "long_strips"       long pairs on one device: column passes (0 = automatic from the
                         round count; > 0 also exercises the multi-GPU boundary protocol)
     "long_blocks"       long pairs: cap on the persistent grid (0 = occupancy)
     "long_profile"      long pairs: print wait / task cycle counters to stderr
     "long_narrow"       long pairs: 1 (default) runs local affine alignments whose scheme
                         passes the range guard and whose subject has no N on the 16-bit
                         differential kernel; 0 forces the 32-bit kernel
     "long_band_rows"    long pairs, rows per warp task: 32-bit kernel 512 (default) or
                         384; 16-bit kernel 1024 (default), 768 or 512
     "long_sleep_ns"     long pairs (16-bit kernel): back-off of the row hand-off poll
     "long_spin_limit"   long pairs: poll iterations (each with a short back-off) before a
                         bounded wait raises the abort flag -> ANYSEQ_E_TIMEOUT (default
                         2^28; <= 0 restores it)
     "long_stall_task"   fault injection (tests): the warp that draws this task index skips
                         it, so every task depending on it must time out (default -1)
     "tb_leaf_cells"     long traceback, Hirschberg fallback: recursion stops at <= this
                         many cells per sub-problem (default 2^20)
     "tb_ckpt_bytes"     long traceback: device memory budget of the checkpoints (default
                         0 = 40 % of free memory); "tb_kc_shift" (8..12) / "tb_ck_every"
                         (1..8) force the column / row checkpoint spacing (tests)
     "tb8"               batch traceback: 1 (default) stores the low byte of H per cell when
                         the scheme allows it exactly (R23); 0 = full H
     "batch_long_cells"  a batch pair with n*m >= this (and n, m >= batch_long_min) is
                         aligned by the long-pair path instead of the batch kernel (default
                         2^22; 0 = never).  Score mode, one device: all such pairs of the call
                         share ONE launch of the long kernel (their row-strip tasks in one
                         device queue) while the batch kernels
                         align the other pairs in place
     "batch_long_cells_tb"  the same threshold for anyseq_traceback (default 2^22): one
                         device -> one shared checkpointing forward pass over all such pairs,
                         then each pair's tile walk
     "batch_long_min"    minimum length of both sides for that routing (default 2048)
     "long_multi"        1 (default): the shared launch above; 0: one long-pair call per pair
     "long_multi_group"  pairs per shared launch (default 2048; more pairs: several launches
                         in score mode, the rest one at a time in traceback mode)
     "batch_long_small"  batches of at most this many pairs send every pair with n, m >= 256
                         to the long-pair path (default 4; 0 = never); pairs that path cannot
                         take stay on the batch kernel
     "timing"            see above */
anyseq_status anyseq_set_option(anyseq_ctx* ctx, const char* name, int64_t value);

const char* anyseq_status_str(anyseq_status st);
const char* anyseq_last_error(const anyseq_ctx* ctx);
/* Library version string. */
const char* anyseq_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ANYSEQ_H */
