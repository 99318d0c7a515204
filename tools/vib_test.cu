#include <cstdio>
__global__ void k(const unsigned* a, const unsigned* b, unsigned* o, int* p, int n) {
  int t = threadIdx.x;
  if (t >= n) return;
  bool hi, lo;
  unsigned r = __vibmax_s16x2(a[t], b[t], &hi, &lo);
  o[t] = r;
  p[t] = (lo ? 1 : 0) | (hi ? 2 : 0);
  bool q;
  int r2 = __vibmax_s32((int)a[t], (int)b[t], &q);
  p[t] |= (q ? 4 : 0);
  (void)r2;
}
int main() {
  const int n = 6;
  unsigned ha[n] = {0x00050003u, 0x00030005u, 0x00040004u, 0xFFFF0001u, 0x0001FFFFu, 0x00000000u};
  unsigned hb[n] = {0x00030005u, 0x00050003u, 0x00040004u, 0x0001FFFFu, 0xFFFF0001u, 0x00010001u};
  unsigned *a, *b, *o; int* p;
  cudaMalloc(&a, 64); cudaMalloc(&b, 64); cudaMalloc(&o, 64); cudaMalloc(&p, 64);
  cudaMemcpy(a, ha, sizeof(ha), cudaMemcpyHostToDevice);
  cudaMemcpy(b, hb, sizeof(hb), cudaMemcpyHostToDevice);
  k<<<1, 32>>>(a, b, o, p, n);
  unsigned ho[n]; int hp[n];
  cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
  cudaMemcpy(hp, p, sizeof(hp), cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i) printf("a=%08x b=%08x max=%08x lo=%d hi=%d s32ge=%d\n", ha[i], hb[i], ho[i], hp[i] & 1, (hp[i] >> 1) & 1, (hp[i] >> 2) & 1);
  return 0;
}
