// csrc/dpx_bench.cu -- integer/DPX pipe microbenchmark (the roofline denominator).
//
// Measures, on the box, how many lane-operations per clock one SM sustains for each SASS
// instruction the fill kernel is built from (VIADDMNMX[.S16x2], VIMNMX[.S16x2], PRMT,
// VIADD.16x2 / IADD3) and for the fill kernel's exact per-register mix
// (1 PRMT + 3 VIADDMNMX + 1 VIMNMX + 1 VIADD per two cells in s16x2).  Each thread runs 8
// independent dependency chains, no memory traffic, full occupancy; cycles come from
// clock64() on the SM.  Output: one JSON object on stdout.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define ITERS 4096
#define CH 8

__device__ __forceinline__ uint32_t prmt_(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}

template <int OP>
__global__ void __launch_bounds__(256) bench(uint32_t seed, uint32_t one, uint32_t* sink,
                                             unsigned long long* cyc) {
  uint32_t x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    x[c] = seed * (threadIdx.x + 1) + c;
    y[c] = seed ^ (c * 0x9e3779b9u);
  }
  const uint32_t k1 = seed | 0x00010001u, k2 = seed >> 3;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) x[c] = __viaddmax_s16x2(x[c], k1, y[c]);
      if (OP == 1) {  // dependent pair: ptxas cannot fuse two maxes into one VIMNMX3
        x[c] = __vmaxs2(x[c], y[c]);
        y[c] = __vmaxs2(y[c], x[c] ^ k2);  // (+1 LOP3, same pipe: counted)
      }
      if (OP == 2) x[c] = (uint32_t)__viaddmax_s32((int)x[c], (int)k1, (int)y[c]);
      if (OP == 3) x[c] = prmt_(x[c], y[c], k2);
      if (OP == 4) x[c] = __vadd2(x[c], k1);
      if (OP == 5) x[c] = x[c] + y[c] + k1;  // IADD3
      if (OP == 7) x[c] = __vimax3_s16x2(x[c], y[c], k1);
      if (OP == 8) {  // IMAD with a run-time multiplier of 1 (Hop on the FMA pipe)
        uint32_t d;
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x[c]), "r"(one), "r"(k2));
        x[c] = d;
      }
      if (OP == 9) {  // shipped fill mix per register: PRMT + 3 VIADDMNMX + VIMNMX (+2 IMAD)
        const uint32_t sig = prmt_(k1, k2, x[c]);
        uint32_t hl, X;
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hl) : "r"(x[c]), "r"(one), "r"(k2));
        const uint32_t f = __viaddmax_s16x2(y[c], k1, hl);
        const uint32_t df = __viaddmax_s16x2(x[c], sig, f);
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(X) : "r"(df), "r"(one), "r"(k2));
        const uint32_t h = __vmaxs2(df, y[c]);
        y[c] = __viaddmax_s16x2(f, k1, X);
        x[c] = h;
      }
      if (OP == 6) {  // fill-kernel mix for one register (2 cells): 6 instructions
        const uint32_t sig = prmt_(k1, k2, x[c]);
        uint32_t e = __viaddmax_s16x2(y[c], k1, x[c]);
        uint32_t f = __viaddmax_s16x2(x[c], k1, y[c]);
        uint32_t t = __vmaxs2(e, f);
        uint32_t h = __viaddmax_s16x2(y[c], sig, t);
        y[c] = e;
        x[c] = __vadd2(h, k1);
        (void)f;
      }
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= x[c] ^ y[c];
  if (acc == 0x12345678u) sink[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
double run(int sms, int instr_per_iter) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bench<OP>, 256, 0);
  const int grid = sms * nb;
  uint32_t* sink;
  unsigned long long* cyc;
  cudaMalloc(&sink, 4);
  cudaMalloc(&cyc, grid * 8);
  bench<OP><<<grid, 256>>>(12345u, 1u, sink, cyc);  // warm
  bench<OP><<<grid, 256>>>(54321u, 1u, sink, cyc);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  cudaFree(sink);
  cudaFree(cyc);
  // lane-ops per SM per clock: (blocks per SM) * 256 threads * ITERS * CH * instr / cycles
  return (double)nb * 256.0 * ITERS * CH * instr_per_iter / (double)mx;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double r0 = run<0>(sms, 1), r1 = run<1>(sms, 3), r2 = run<2>(sms, 1), r3 = run<3>(sms, 1),
               r4 = run<4>(sms, 1), r5 = run<5>(sms, 1), r6 = run<6>(sms, 6), r7 = run<7>(sms, 1),
               r8 = run<8>(sms, 1), r9 = run<9>(sms, 7);
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"viaddmnmx_s16x2\": %.2f, \"vimnmx_s16x2\": %.2f, "
         "\"viaddmnmx_s32\": %.2f, \"prmt\": %.2f, \"viadd_16x2\": %.2f, \"iadd3\": %.2f, "
         "\"mix_lane_ops_per_clk_per_sm\": %.2f, \"vimnmx3_s16x2\": %.2f, \"imad\": %.2f, "
         "\"fill_mix_lane_ops_per_clk_per_sm\": %.2f, \"fill_mix_instr_per_register\": 7, "
         "\"unit\": \"lane-ops per clock per SM\"}\n",
         sms, clk, r0, r1, r2, r3, r4, r5, r6, r7, r8, r9);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : 1;
}
