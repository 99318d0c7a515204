// hirschberg.cu -- device passes of the linear-space long-pair traceback.
//
// A last-row pass (hirschberg.h) is cut into row bands of NT*R rows, one CTA each: threads
// own R consecutive rows and sweep the columns with a skew of one step per thread; the
// bottom row of a thread is handed to the next thread through a double-buffered
// shared-memory slot (one barrier per step), and band to band through row[] in global
// memory, updated in place (a band's thread 0 reads column j at step j-1, before the last
// thread of the same band overwrites it at step j+NT-2) and published 32 columns at a time
// through a per-band progress word (release / acquire), so the bands of a pass run as a
// pipelined wavefront over the SMs (the tiled wavefront of P:488).  Recurrence: Eq. (1) with nu = -inf and the linear
// gaps of Eqs. (2)-(3), H(i,0) = -i*g, H(0,j) = -j*g.  32-bit scores.
#include "hirschberg.h"

#include <climits>

namespace {

#ifndef HB_NT
#define HB_NT 128
#endif
#ifndef HB_R
#define HB_R 24
#endif
#ifndef HB_PUB
#define HB_PUB 32
#endif
constexpr int NT = HB_NT;  // threads per CTA
constexpr int R = HB_R;    // rows per thread

__global__ void encode_kernel(const char* __restrict__ ascii, uint8_t* __restrict__ codes,
                              uint64_t len, int* bad) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < len;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned c = (unsigned char)ascii[k] & 0xDFu;  // upper case
    uint8_t v = c == 'A' ? 0 : c == 'C' ? 1 : c == 'G' ? 2 : c == 'T' ? 3 : c == 'N' ? 4 : 0xff;
    if (v == 0xff) {
      *bad = 1;
      v = 4;
    }
    codes[k] = v;
  }
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One CTA per row band of NT*R rows; bands are taken by atomic ticket in (task, band)
// order, so the band a CTA waits on always belongs to a CTA that is already running.
template <int MODE>
__global__ void __launch_bounds__(NT) lastrow_kernel(const LrTask* __restrict__ tasks,
                                                     const int* __restrict__ band_start,
                                                     int num_tasks, int* ticket, int* prog,
                                                     int num_bands_total, LrParams P) {
  __shared__ int32_t xch[2][NT];
  __shared__ int32_t ssig[25];
  __shared__ int32_t rs[NT], ri[NT], rj[NT];
  __shared__ int sh_ticket;
  const int t = threadIdx.x;
  if (t == 0) sh_ticket = atomicAdd(ticket, 1);
  if (t < 25) ssig[t] = P.sig[t];
  __syncthreads();
  const int tk = sh_ticket;
  int lo = 0, hi = num_tasks - 1;  // task: the last one with band_start <= tk
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (band_start[mid] <= tk) lo = mid;
    else hi = mid - 1;
  }
  const LrTask T = tasks[lo];
  const int band = tk - band_start[lo];
  const int g = P.g, n1 = T.n1, m1 = T.m1;
  // running optimum of MODE 1: cell (0,0) holds 0 and beats every other border cell
  // MODE 2 (semi-global begin): only cells of the last row or column count
  int bs = MODE == 2 ? INT_MIN : 0, bi = 0, bj = 0;
  const int base = band * NT * R;
  const bool last_band = base + NT * R >= n1;
  const int i0 = base + t * R + 1;  // first row of this thread (1-based)
  int ra[R], h[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int i = i0 + k;
    ra[k] = i <= n1 ? 5 * (int)(T.rev ? T.a[n1 - i] : T.a[i - 1]) : 0;
    h[k] = -i * g;  // H(i, 0)
  }
  int updiag = -(i0 - 1) * g;  // H(i0-1, 0)
  const int own = last_band ? n1 - i0 : -1;  // row n1 sits in h[own] of one thread
  const int* wait_on = band ? prog + tk - 1 : nullptr;
  int ready = 0;  // columns of the band above known to be published
  const int nsteps = m1 + NT - 1;
  for (int s = 0; s < nsteps; ++s) {
    const int j = s - t + 1;
    if (j >= 1 && j <= m1) {
      int up;  // H(i0-1, j)
      if (t == 0) {
        if (band == 0) {
          up = -j * g;
        } else {
          long long spins = 0;  // bounded like every device-side wait (-> ANYSEQ_E_TIMEOUT)
          while (ready < j) {
            ready = ld_acquire(wait_on);
            if (ready < j) {
              __nanosleep(64);
              if ((++spins & 1023) == 0 &&
                  (spins > (1ll << 26) || *(volatile int*)(prog - 1 + num_bands_total + 1))) {
                atomicExch((int*)(prog - 1 + num_bands_total + 1), 1);
                ready = j;  // abandon the band: the host discards the pass
              }
            }
          }
          up = __ldcg(T.row + j);
        }
      } else {
        up = xch[(s - 1) & 1][t - 1];
      }
      const int bcode = T.rev ? T.b[m1 - j] : T.b[j - 1];
      int diag = updiag, above = up;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        // Eq. (1) reassociated: the off-chain part max(H_left - g, diag + sigma) first, so
        // the dependency down the column is one VIADDMNMX per row (exact: max is associative)
        const int x = __viaddmax_s32(h[k], -g, diag + ssig[ra[k] + bcode]);
        const int nh = __viaddmax_s32(above, -g, x);
        diag = h[k];
        h[k] = nh;
        above = nh;
        if (MODE != 0 && nh > bs && i0 + k <= n1 &&  // strict >: smallest j, then i
            (MODE == 1 || i0 + k == n1 || j == m1)) {
          bs = nh;
          bi = i0 + k;
          bj = j;
        }
      }
      updiag = up;
      xch[s & 1][t] = h[R - 1];
      if (last_band) {
        if (own >= 0 && own < R) {
          int v = h[0];
#pragma unroll
          for (int k = 1; k < R; ++k) v = own == k ? h[k] : v;
          T.row[j] = v;
        }
      } else if (t == NT - 1) {
        __stcg(T.row + j, h[R - 1]);
        if ((j & (HB_PUB - 1)) == 0 || j == m1) {  // publish HB_PUB columns at a time
          __threadfence();
          atomicExch(prog + tk, j);
        }
      }
    }
    __syncthreads();
  }
  if (MODE != 0) {
    rs[t] = bs;
    ri[t] = bi;
    rj[t] = bj;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
      if (t < w) {
        const int s2 = rs[t + w], i2 = ri[t + w], j2 = rj[t + w];
        const bool take = s2 > rs[t] || (s2 == rs[t] && (j2 < rj[t] || (j2 == rj[t] && i2 < ri[t])));
        if (take) {
          rs[t] = s2;
          ri[t] = i2;
          rj[t] = j2;
        }
      }
      __syncthreads();
    }
    if (t == 0) {
      T.best[3 * band + 0] = rs[0];
      T.best[3 * band + 1] = ri[0];
      T.best[3 * band + 2] = rj[0];
    }
  }
}

}  // namespace

void launch_encode_codes(const char* ascii, uint8_t* codes, uint64_t len, int* bad,
                         cudaStream_t st) {
  if (!len) return;
  const uint64_t blocks = (len + 255) / 256;
  encode_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(ascii, codes,
                                                                                   len, bad);
}

int lastrow_bands(int n1) { return (n1 + NT * R - 1) / (NT * R); }

void launch_lastrow(const LrTask* d_tasks, const int* d_band_start, int num_tasks,
                    int num_bands, int* d_sync, const LrParams& P, cudaStream_t st) {
  if (num_tasks <= 0) return;
  lastrow_kernel<0><<<num_bands, NT, 0, st>>>(d_tasks, d_band_start, num_tasks, d_sync,
                                              d_sync + 1, num_bands, P);
}

void launch_lastrow_anchored(const LrTask* d_tasks, const int* d_band_start, int num_tasks,
                             int num_bands, int* d_sync, const LrParams& P, cudaStream_t st) {
  if (num_tasks <= 0) return;
  lastrow_kernel<1><<<num_bands, NT, 0, st>>>(d_tasks, d_band_start, num_tasks, d_sync,
                                              d_sync + 1, num_bands, P);
}

void launch_lastrow_edges(const LrTask* d_tasks, const int* d_band_start, int num_tasks,
                          int num_bands, int* d_sync, const LrParams& P, cudaStream_t st) {
  if (num_tasks <= 0) return;
  lastrow_kernel<2><<<num_bands, NT, 0, st>>>(d_tasks, d_band_start, num_tasks, d_sync,
                                              d_sync + 1, num_bands, P);
}
