// hirschberg.h -- last-row score passes for the linear-space long-pair traceback
// (Hirschberg's divide and conquer over the relaxation of Eqs. (1)-(3),
// PAPER.md P:224-239, with the paper's linear-space score variant P:266-270 as the pass).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// One score pass of a global, linear-gap DP over a[0..n1) (rows) x b[0..m1) (columns),
// both as codes 0..4 (A,C,G,T,N).  rev != 0 reads both sequences back to front (the
// reverse pass of Hirschberg).  n1 >= 1 and m1 >= 1.
//  mode 0: row[j] = H(n1, j) for j = 1..m1 (row[0] is left to the host: -n1*g).
//          row[] doubles as the band-to-band row buffer of the pass, so it needs m1+1 entries.
//  mode 1: additionally best[0..2] = (max over all cells incl. row/col 0, i, j) with ties
//          to the smallest j, then the smallest i (the anchored pass of a local alignment:
//          reversed prefixes ending at the optimum's end cell).
struct LrTask {
  const uint8_t* a;
  const uint8_t* b;
  int32_t n1, m1;
  int32_t rev, mode;
  int32_t* row;
  int32_t* best;
};

struct LrParams {
  int32_t g;       // linear gap penalty magnitude (Eq. 2-3)
  int8_t sig[25];  // sigma(a, b) = sig[5a + b]
};

// Encodes ASCII ACGTN (either case) to codes 0..4; any other byte sets *bad = 1.
void launch_encode_codes(const char* ascii, uint8_t* codes, uint64_t len, int* bad,
                         cudaStream_t st);
// Row bands of one task (3072 rows each); band b of a task waits for band b-1's published
// columns.  d_band_start[num_tasks] = first band of each task (exclusive prefix sum of
// lastrow_bands), num_bands the total; d_sync = 2 + num_bands zeroed ints (ticket counter,
// per-band progress, then an abort flag set when a band-to-band wait exceeds its bound).  MODE 1 (anchored) writes best[3*band .. 3*band+2] per band.
int lastrow_bands(int n1);
void launch_lastrow(const LrTask* d_tasks, const int* d_band_start, int num_tasks,
                    int num_bands, int* d_sync, const LrParams& P, cudaStream_t st);
// MODE 2: best over the cells of row n1 and column m1 only (the anchored pass of a
// semi-global alignment, whose begin lies on row 0 or column 0); border cells (n1, 0) and
// (0, m1) are left to the host.
void launch_lastrow_edges(const LrTask* d_tasks, const int* d_band_start, int num_tasks,
                          int num_bands, int* d_sync, const LrParams& P, cudaStream_t st);
void launch_lastrow_anchored(const LrTask* d_tasks, const int* d_band_start, int num_tasks,
                             int num_bands, int* d_sync, const LrParams& P, cudaStream_t st);
