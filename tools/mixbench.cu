// instruction-mix microbenchmark for the fill kernel's per-register op mix
#include <cstdio>
#include <cstdint>
#include <vector>
#define ITERS 2048
#define CH 8
__device__ __forceinline__ uint32_t prmt_(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d; asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s)); return d; }
__device__ __forceinline__ uint32_t imad_(uint32_t x, uint32_t one, uint32_t k) {
  uint32_t d; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "r"(one), "r"(k)); return d; }
__device__ __forceinline__ uint32_t imadi_(uint32_t x, uint32_t one) {
  uint32_t d; asm volatile("mad.lo.u32 %0, %1, %2, 0xFFF9FFFA;" : "=r"(d) : "r"(x), "r"(one)); return d; }
template <int MIX>
__global__ void __launch_bounds__(128) bench(uint32_t seed, uint32_t one, uint32_t* sink, unsigned long long* cyc) {
  uint32_t x[CH], y[CH], f[CH];
  for (int c = 0; c < CH; ++c) { x[c] = seed * (threadIdx.x + 1) + c; y[c] = seed ^ (c * 0x9e3779b9u); f[c] = y[c] + 7; }
  const uint32_t k1 = seed | 0x00010001u, k2 = seed >> 3, k3 = seed * 3;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MIX == 1) {  // 5 ALU, register b operands
        const uint32_t sig = prmt_(k1, k2, x[c]);
        f[c] = __viaddmax_s16x2(f[c], k3, x[c]);
        const uint32_t df = __viaddmax_s16x2(y[c], sig, f[c]);
        const uint32_t h = __vmaxs2(df, y[c]);
        y[c] = __viaddmax_s16x2(y[c], k3, df);
        x[c] = h;
      }
      if (MIX == 2) {  // 5 ALU, immediate b
        const uint32_t sig = prmt_(k1, k2, x[c]);
        f[c] = __viaddmax_s16x2(f[c], 0xffffffffu, x[c]);
        const uint32_t df = __viaddmax_s16x2(y[c], sig, f[c]);
        const uint32_t h = __vmaxs2(df, y[c]);
        y[c] = __viaddmax_s16x2(y[c], 0xffffffffu, df);
        x[c] = h;
      }
      if (MIX == 3) {  // shipped: 5 ALU (imm) + 2 IMAD (imm addend)
        const uint32_t sig = prmt_(k1, k2, x[c]);
        f[c] = __viaddmax_s16x2(f[c], 0xffffffffu, imadi_(x[c], one));
        const uint32_t df = __viaddmax_s16x2(y[c], sig, f[c]);
        const uint32_t h = __vmaxs2(df, y[c]);
        y[c] = __viaddmax_s16x2(y[c], 0xffffffffu, imadi_(df, one));
        x[c] = h;
      }
      if (MIX == 4) {  // VIADDMNMX only (imm)
        f[c] = __viaddmax_s16x2(f[c], 0xffffffffu, x[c]);
        x[c] = __viaddmax_s16x2(x[c], 0xffffffffu, y[c]);
        y[c] = __viaddmax_s16x2(y[c], 0xffffffffu, f[c]);
      }
      if (MIX == 5) {  // VIMNMX only
        f[c] = __vmaxs2(f[c], x[c]); x[c] = __vmaxs2(x[c], y[c]); y[c] = __vmaxs2(y[c], f[c]);
      }
      if (MIX == 6) {  // PRMT only
        f[c] = prmt_(f[c], x[c], k1); x[c] = prmt_(x[c], y[c], k2); y[c] = prmt_(y[c], f[c], k3);
      }
      if (MIX == 7) {  // IMAD only
        f[c] = imadi_(f[c], one); x[c] = imadi_(x[c], one); y[c] = imadi_(y[c], one);
      }
      if (MIX == 8) {  // VIADDMNMX (imm) + IMAD interleaved 1:1
        f[c] = __viaddmax_s16x2(f[c], 0xffffffffu, x[c]); x[c] = imadi_(x[c], one);
        y[c] = __viaddmax_s16x2(y[c], 0xffffffffu, f[c]); f[c] = imadi_(f[c], one);
      }
    }
  }
  unsigned long long t1 = clock64();
  uint32_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= x[c] ^ y[c] ^ f[c];
  if (acc == 0x12345678u) sink[0] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MIX>
double run(int sms, int instr, int threads_per_sm) {
  int nb = threads_per_sm / 128;
  int grid = sms * nb;
  uint32_t* sink; unsigned long long* cyc;
  cudaMalloc(&sink, 4); cudaMalloc(&cyc, grid * 8);
  bench<MIX><<<grid, 128>>>(12345u, 1u, sink, cyc);
  bench<MIX><<<grid, 128>>>(54321u, 1u, sink, cyc);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
  cudaFree(sink); cudaFree(cyc);
  return (double)nb * 128.0 * ITERS * CH * instr / (double)mx;  // lane-instr per clk per SM
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int tps : {256, 512, 1024}) {
    printf("{\"threads_per_sm\": %d, \"mix1_5alu_regb\": %.1f, \"mix2_5alu_immb\": %.1f, \"mix3_shipped\": %.1f, "
           "\"viaddmnmx\": %.1f, \"vimnmx\": %.1f, \"prmt\": %.1f, \"imad\": %.1f, \"viaddmnmx_imad\": %.1f}\n", tps,
           run<1>(sms, 5, tps), run<2>(sms, 5, tps), run<3>(sms, 7, tps), run<4>(sms, 3, tps), run<5>(sms, 3, tps),
           run<6>(sms, 3, tps), run<7>(sms, 3, tps), run<8>(sms, 4, tps));
  }
  return 0;
}
