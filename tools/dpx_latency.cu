// Dependent-chain latency (cycles per op) of the ops on the long kernels' critical path,
// one warp alone on the GPU: VIADDMNMX.S16x2, VIMNMX3.S16x2, VIMNMX.S16x2, PRMT, IMAD,
// IADD3, SHFL, and the s32 forms.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d; asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s)); return d;
}
template <int OP>
__global__ void chain(uint32_t* out, uint32_t x, uint32_t y, int n, long long* cyc) {
  uint32_t v = x + threadIdx.x;
  const uint32_t w = y;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) v = __viaddmax_s16x2(v, w, v ^ 1);          // VIADDMNMX.S16x2
      if (OP == 1) v = __vimax3_s16x2(v, w, v + 3);            // VIMNMX3.S16x2 (+IADD)
      if (OP == 2) v = __vmaxs2(v, w);                         // VIMNMX.S16x2
      if (OP == 3) v = prmt(v, w, 0x3210 + (v & 1));           // PRMT (+LOP)
      if (OP == 4) { asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(v) : "r"(1u), "r"(w)); }  // IMAD
      if (OP == 5) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31);  // SHFL
      if (OP == 6) v = (uint32_t)__viaddmax_s32((int)v, (int)w, (int)(v ^ 1));  // VIADDMNMX s32
      if (OP == 7) v = __viaddmax_s16x2(v, w, w);              // VIADDMNMX.S16x2, one dependency
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  uint32_t* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  const char* names[] = {"VIADDMNMX.S16x2(a,b,f(a))", "VIMNMX3.S16x2", "VIMNMX.S16x2", "PRMT", "IMAD", "SHFL",
                         "VIADDMNMX s32", "VIADDMNMX.S16x2(a,b,c)"};
  const int n = 4096;
  for (int op = 0; op < 8; ++op) {
    long long h = 0;
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 32>>>(o, 1, 2, n, c); break;
        case 1: chain<1><<<1, 32>>>(o, 1, 2, n, c); break;
        case 2: chain<2><<<1, 32>>>(o, 1, 2, n, c); break;
        case 3: chain<3><<<1, 32>>>(o, 1, 2, n, c); break;
        case 4: chain<4><<<1, 32>>>(o, 1, 2, n, c); break;
        case 5: chain<5><<<1, 32>>>(o, 1, 2, n, c); break;
        case 6: chain<6><<<1, 32>>>(o, 1, 2, n, c); break;
        case 7: chain<7><<<1, 32>>>(o, 1, 2, n, c); break;
      }
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-28s %.2f cycles per chained op (incl. any helper op)\n", names[op], (double)h / (16.0 * n));
  }
  return 0;
}
