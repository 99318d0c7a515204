/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the pairwise alignment
 * DP that AnySeq (arXiv 2002.04561) relaxes.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2002_04561_b200/csrc) and neither side includes the other.
 *
 * Everything is int64 with -inf = -2^62, full (n+1) x (m+1) matrices H, E, F and a
 * uint8 direction matrix, relaxed row-major exactly in the order of the paper's
 * equations.  Citations (PAPER.md line numbers, section / equation):
 *   Eq. (1)  H(i,j) = max{H(i-1,j-1)+sigma(q_i,s_j), E(i,j), F(i,j), nu}   P:224-232 (Sec. III-A)
 *   Eq. (2,3) linear gaps: E = H(i-1,j) - g,  F = H(i,j-1) - g
 *   Eq. (4,5) affine gaps: E = max(E(i-1,j)-Ge, H(i-1,j)-Go-Ge), F alike P:241-255
 *             "a gap of length k is penalized with G_o + k*G_e"
 *   local init / nu = 0 / optimum anywhere
 *   global init / nu = -inf / optimum H(n,m)
 *   semi-global: local init, optimum in last row or column
 *   predecessor with strict '>' replacement, no-gap first               P:284-308 (listing relax_global)
 *   traceback over predecessor information
 *   simple substitution scoring simple_subst_scoring(2,-1)
 * Readings where the paper is silent (DESIGN.md "Readings" R1..R20, = SURVEY L1..L20):
 *   penalties are non-negative magnitudes that are subtracted (L1); linear == Go=0,Ge=g
 *   in the init formulas (L3); semi-global nu = -inf (L4); semi-global candidates are
 *   row n (j=0..m-1) then column m (i=0..n) (L5); E is vertical = 'I', F horizontal =
 *   'D' (L6); H source tie order DIAG > E(up) > F(left) (L7); extend beats open on ties
 *   (L8); local traceback stops at H <= 0 (L9); end cell = first maximum in column-major
 *   order (smallest j, then smallest i) (L10); 'N' mismatches everything incl. N (L12);
 *   global boundary runs are emitted at (i,0)/(0,j) (L16).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ONEG (-(((int64_t)1) << 62))

enum { OK_GLOBAL = 0, OK_LOCAL = 1, OK_SEMI = 2 };
enum { OG_LINEAR = 0, OG_AFFINE = 1 };
/* direction bits of the oracle's own matrix (independent of any GPU encoding) */
enum { SRC_DIAG = 0, SRC_UP = 1, SRC_LEFT = 2, SRC_STOP = 3 };
enum { OP_M = 0, OP_I = 1, OP_D = 2 };

typedef struct {
  int32_t kind;      /* 0 global, 1 local, 2 semi-global */
  int32_t gap;       /* 0 linear, 1 affine */
  int32_t match;     /* sigma(a,a), a in ACGT */
  int32_t mismatch;  /* sigma(a,b), a != b, and anything involving N */
  int32_t gap_open;  /* G_o (ignored for linear) */
  int32_t gap_extend;/* G_e (linear: g) */
  int32_t has_subst; /* 1: sigma from subst (P:416-419 matrix scoring), else match/mismatch */
  int32_t subst[25]; /* sigma(a, b) = subst[5*a + b], codes A,C,G,T,N = 0..4 */
} oracle_params;

typedef struct {
  int64_t score;
  int64_t q_begin, s_begin, q_end, s_end;
  int64_t n_ops;     /* number of RLE cigar words written */
} oracle_result;

/* symbol code: A,C,G,T -> 0..3, N -> 4, anything else -> -1 (L12) */
static int oracle_code(char c) {
  switch (c) {
    case 'A': case 'a': return 0;
    case 'C': case 'c': return 1;
    case 'G': case 'g': return 2;
    case 'T': case 't': return 3;
    case 'N': case 'n': return 4;
    default: return -1;
  }
}

/* simple_subst_scoring(match, mismatch); N mismatches everything (L12);
   or a full substitution matrix over {A,C,G,T,N} (matrix scoring) */
static int64_t oracle_sigma(const oracle_params* p, int a, int b) {
  if (p->has_subst) return p->subst[5 * a + b];
  if (a == b && a < 4) return p->match;
  return p->mismatch;
}

int oracle_check_seq(const char* x, int64_t len) {
  for (int64_t i = 0; i < len; ++i)
    if (oracle_code(x[i]) < 0) return (int)(i < 0x7fffffff ? i : 0x7fffffff);
  return -1;
}

static int64_t gap_open_eff(const oracle_params* p) { return p->gap == OG_AFFINE ? p->gap_open : 0; }

/*
 * Full-matrix alignment.  want_tb != 0 also produces the CIGAR (BAM-style
 * len<<4|op, op M=0, I=1, D=2) into cigar[0..cigar_cap).  Returns 0 on success,
 * -1 bad input, -2 out of memory, -3 cigar capacity too small.
 */
int oracle_align(const oracle_params* p, const char* qs, int64_t n, const char* ss, int64_t m,
                 int want_tb, oracle_result* out, uint32_t* cigar, int64_t cigar_cap) {
  if (oracle_check_seq(qs, n) >= 0 || oracle_check_seq(ss, m) >= 0) return -1;
  const int64_t W = m + 1;
  const int64_t cells = (n + 1) * W;
  int64_t* H = (int64_t*)malloc(sizeof(int64_t) * cells);
  int64_t* E = (int64_t*)malloc(sizeof(int64_t) * cells);
  int64_t* F = (int64_t*)malloc(sizeof(int64_t) * cells);
  uint8_t* dir = (uint8_t*)malloc((size_t)cells);
  int* qc = (int*)malloc(sizeof(int) * (n + 1));
  int* sc = (int*)malloc(sizeof(int) * (m + 1));
  if (!H || !E || !F || !dir || !qc || !sc) {
    free(H); free(E); free(F); free(dir); free(qc); free(sc);
    return -2;
  }
  for (int64_t i = 1; i <= n; ++i) qc[i] = oracle_code(qs[i - 1]);
  for (int64_t j = 1; j <= m; ++j) sc[j] = oracle_code(ss[j - 1]);

  const int64_t Go = gap_open_eff(p), Ge = p->gap_extend;
  const int64_t nu = (p->kind == OK_LOCAL) ? 0 : ONEG;

  /* ---- initialisation, P:259 / P:262 / P:264 ---- */
  H[0] = 0; E[0] = ONEG; F[0] = ONEG; dir[0] = SRC_STOP;
  for (int64_t i = 1; i <= n; ++i) {
    int64_t* c = &H[i * W];
    c[0] = (p->kind == OK_GLOBAL) ? -Go - i * Ge : 0;
    E[i * W] = c[0];  /* dead value, never read (L15) */
    F[i * W] = ONEG;
    dir[i * W] = SRC_STOP;
  }
  for (int64_t j = 1; j <= m; ++j) {
    H[j] = (p->kind == OK_GLOBAL) ? -Go - j * Ge : 0;
    E[j] = ONEG;
    F[j] = H[j];      /* dead value, never read (L15) */
    dir[j] = SRC_STOP;
  }

  /* ---- relaxation, row-major, Eqs. (1)-(5) in the listing's order ---- */
  for (int64_t i = 1; i <= n; ++i) {
    for (int64_t j = 1; j <= m; ++j) {
      const int64_t up = (i - 1) * W + j, left = i * W + j - 1, diag = (i - 1) * W + j - 1,
                    cur = i * W + j;
      int64_t e, f;
      int eext = 0, fext = 0;
      if (p->gap == OG_AFFINE) {
        int64_t ex = E[up] - Ge, eo = H[up] - Go - Ge;       /* Eq. (4) */
        e = ex >= eo ? ex : eo; eext = ex >= eo;               /* L8: extend wins ties */
        int64_t fx = F[left] - Ge, fo = H[left] - Go - Ge;   /* Eq. (5) */
        f = fx >= fo ? fx : fo; fext = fx >= fo;
      } else {
        e = H[up] - Ge;                                       /* Eq. (2) */
        f = H[left] - Ge;                                     /* Eq. (3) */
      }
      int64_t h = H[diag] + oracle_sigma(p, qc[i], sc[j]);    /* Eq. (1), no gap */
      int src = SRC_DIAG;
      if (e > h) { h = e; src = SRC_UP; }                      /* strict '>' */
      if (f > h) { h = f; src = SRC_LEFT; }                    /* strict '>' */
      if (p->kind == OK_LOCAL && h <= nu) { h = nu; src = SRC_STOP; } /* nu = 0, L9 */
      H[cur] = h; E[cur] = e; F[cur] = f;
      dir[cur] = (uint8_t)(src | (eext << 2) | (fext << 3));
    }
  }

  /* ---- optimum, P:259-264, L5, L10 ---- */
  int64_t bi = 0, bj = 0, best = 0;
  if (p->kind == OK_GLOBAL) {
    bi = n; bj = m; best = H[n * W + m];
  } else if (p->kind == OK_SEMI) {
    int have = 0;
    for (int64_t j = 0; j < m; ++j) {            /* (n,0) .. (n,m-1) */
      int64_t v = H[n * W + j];
      if (!have || v > best) { best = v; bi = n; bj = j; have = 1; }
    }
    for (int64_t i = 0; i <= n; ++i) {           /* (0,m) .. (n,m) */
      int64_t v = H[i * W + m];
      if (!have || v > best) { best = v; bi = i; bj = m; have = 1; }
    }
  } else {
    int have = 0;
    for (int64_t j = 0; j <= m; ++j)             /* column-major, L10 */
      for (int64_t i = 0; i <= n; ++i) {
        int64_t v = H[i * W + j];
        if (!have || v > best) { best = v; bi = i; bj = j; have = 1; }
      }
  }
  out->score = best; out->q_end = bi; out->s_end = bj;
  out->q_begin = bi; out->s_begin = bj; out->n_ops = 0;

  int rc = 0;
  if (want_tb) {
    /* ---- traceback walk, SURVEY 8(c) step 7 ---- */
    int64_t cap_ops = n + m + 1;
    uint8_t* ops = (uint8_t*)malloc((size_t)cap_ops);
    int64_t nops = 0;
    int64_t i = bi, j = bj;
    int state = 0; /* 0 = H, 1 = E, 2 = F */
    for (;;) {
      if (state == 0) {
        if (i == 0 || j == 0) {
          if (p->kind == OK_GLOBAL) {           /* L16 */
            while (i > 0) { ops[nops++] = OP_I; --i; }
            while (j > 0) { ops[nops++] = OP_D; --j; }
          }
          break;
        }
        int src = dir[i * W + j] & 3;
        if (src == SRC_STOP) break;
        if (src == SRC_DIAG) { ops[nops++] = OP_M; --i; --j; }
        else if (src == SRC_UP) state = 1;
        else state = 2;
      } else if (state == 1) {
        int ext = (dir[i * W + j] >> 2) & 1;
        ops[nops++] = OP_I; --i;
        if (!ext || p->gap == OG_LINEAR) state = 0;
      } else {
        int ext = (dir[i * W + j] >> 3) & 1;
        ops[nops++] = OP_D; --j;
        if (!ext || p->gap == OG_LINEAR) state = 0;
      }
    }
    out->q_begin = i; out->s_begin = j;
    /* reverse + run-length encode */
    int64_t w = 0;
    for (int64_t k = nops - 1; k >= 0;) {
      int op = ops[k];
      int64_t len = 0;
      while (k >= 0 && ops[k] == op) { ++len; --k; }
      if (w < cigar_cap) cigar[w] = (uint32_t)((len << 4) | op);
      ++w;
    }
    out->n_ops = w;
    if (w > cigar_cap) rc = -3;
    free(ops);
  }
  free(H); free(E); free(F); free(dir); free(qc); free(sc);
  return rc;
}

/*
 * Score-only variant in linear space (Fig. 1 right): keeps one H row and
 * one E row; identical recurrences and the same optimum rules.  Used for long windows
 * (config C4) where the full matrix does not fit.  Returns end cell.
 */
int oracle_score_rolling(const oracle_params* p, const char* qs, int64_t n, const char* ss,
                         int64_t m, oracle_result* out) {
  if (oracle_check_seq(qs, n) >= 0 || oracle_check_seq(ss, m) >= 0) return -1;
  int64_t* Hrow = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
  int64_t* Erow = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
  int* sc = (int*)malloc(sizeof(int) * (m + 1));
  if (!Hrow || !Erow || !sc) { free(Hrow); free(Erow); free(sc); return -2; }
  for (int64_t j = 1; j <= m; ++j) sc[j] = oracle_code(ss[j - 1]);
  const int64_t Go = gap_open_eff(p), Ge = p->gap_extend;
  const int64_t nu = (p->kind == OK_LOCAL) ? 0 : ONEG;
  Hrow[0] = 0; Erow[0] = ONEG;
  for (int64_t j = 1; j <= m; ++j) {
    Hrow[j] = (p->kind == OK_GLOBAL) ? -Go - j * Ge : 0;
    Erow[j] = ONEG;
  }
  /* optimum bookkeeping in the order of L5/L10 */
  int64_t best = 0, bi = 0, bj = 0;
  int have = 0;
  /* local: column-major order over all cells.  While sweeping rows we remember, per
     column, the first row reaching that column's maximum; then pick the column. */
  int64_t* colbest = NULL; int64_t* colbesti = NULL;
  if (p->kind == OK_LOCAL) {
    colbest = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
    colbesti = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
    for (int64_t j = 0; j <= m; ++j) { colbest[j] = Hrow[j]; colbesti[j] = 0; }
  }
  int64_t colm_best = Hrow[m], colm_i = 0; /* semi: column m, i = 0.. */
  for (int64_t i = 1; i <= n; ++i) {
    const int qi = oracle_code(qs[i - 1]);
    int64_t diag = Hrow[0];
    Hrow[0] = (p->kind == OK_GLOBAL) ? -Go - i * Ge : 0;
    int64_t f = ONEG;
    if (p->kind == OK_LOCAL && Hrow[0] > colbest[0]) { colbest[0] = Hrow[0]; colbesti[0] = i; }
    for (int64_t j = 1; j <= m; ++j) {
      int64_t e;
      if (p->gap == OG_AFFINE) {
        int64_t ex = Erow[j] - Ge, eo = Hrow[j] - Go - Ge;
        e = ex >= eo ? ex : eo;
        int64_t fx = f - Ge, fo = Hrow[j - 1] - Go - Ge;
        f = fx >= fo ? fx : fo;
      } else {
        e = Hrow[j] - Ge;
        f = Hrow[j - 1] - Ge;
      }
      int64_t h = diag + oracle_sigma(p, qi, sc[j]);
      if (e > h) h = e;
      if (f > h) h = f;
      if (p->kind == OK_LOCAL && h <= nu) h = nu;
      diag = Hrow[j];
      Hrow[j] = h; Erow[j] = e;
      if (p->kind == OK_LOCAL && h > colbest[j]) { colbest[j] = h; colbesti[j] = i; }
    }
    if (p->kind == OK_SEMI && Hrow[m] > colm_best) { colm_best = Hrow[m]; colm_i = i; }
  }
  if (p->kind == OK_GLOBAL) {
    best = Hrow[m]; bi = n; bj = m;
  } else if (p->kind == OK_SEMI) {
    for (int64_t j = 0; j < m; ++j)
      if (!have || Hrow[j] > best) { best = Hrow[j]; bi = n; bj = j; have = 1; }
    if (!have || colm_best > best) { best = colm_best; bi = colm_i; bj = m; have = 1; }
  } else {
    for (int64_t j = 0; j <= m; ++j)
      if (!have || colbest[j] > best) { best = colbest[j]; bi = colbesti[j]; bj = j; have = 1; }
  }
  out->score = best; out->q_end = bi; out->s_end = bj;
  out->q_begin = bi; out->s_begin = bj; out->n_ops = 0;
  free(Hrow); free(Erow); free(sc); free(colbest); free(colbesti);
  return 0;
}

/* ---------------- batch driver: plain per-pair code, parallel across pairs only ------- */
typedef struct {
  const oracle_params* p;
  const char* q; const uint64_t* q_off;
  const char* s; const uint64_t* s_off;
  int64_t num_pairs;
  int want_tb;
  oracle_result* res;
  uint32_t* cigar;         /* pair k writes at cigar[q_off[k] + s_off[k] ...], capacity n+m+1 */
  int64_t next;
  pthread_mutex_t mu;
  int err;
} oracle_batch_job;

static void* oracle_worker(void* arg) {
  oracle_batch_job* J = (oracle_batch_job*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int64_t k0 = J->next;
    J->next += 64;
    pthread_mutex_unlock(&J->mu);
    if (k0 >= J->num_pairs) break;
    int64_t k1 = k0 + 64 < J->num_pairs ? k0 + 64 : J->num_pairs;
    for (int64_t k = k0; k < k1; ++k) {
      int64_t n = (int64_t)(J->q_off[k + 1] - J->q_off[k]);
      int64_t m = (int64_t)(J->s_off[k + 1] - J->s_off[k]);
      uint32_t* cg = J->want_tb ? J->cigar + J->q_off[k] + J->s_off[k] + k : NULL;
      int rc = oracle_align(J->p, J->q + J->q_off[k], n, J->s + J->s_off[k], m, J->want_tb,
                            &J->res[k], cg, n + m + 1);
      if (rc != 0) J->err = rc;
    }
  }
  return NULL;
}

/* cigar (if want_tb) must hold sum(n_k + m_k + 1) words; pair k's ops start at
   q_off[k] + s_off[k] + k.  Returns 0 or the first error code. */
int oracle_batch(const oracle_params* p, const char* q, const uint64_t* q_off, const char* s,
                 const uint64_t* s_off, int64_t num_pairs, int nthreads, int want_tb,
                 oracle_result* res, uint32_t* cigar) {
  oracle_batch_job J;
  J.p = p; J.q = q; J.q_off = q_off; J.s = s; J.s_off = s_off; J.num_pairs = num_pairs;
  J.want_tb = want_tb; J.res = res; J.cigar = cigar; J.next = 0; J.err = 0;
  pthread_mutex_init(&J.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, oracle_worker, &J);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&J.mu);
  return J.err;
}
