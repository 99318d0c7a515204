// Host-side 2-bit packing throughput (ASCII ACGT -> 2 bits, with validation), threads sweep.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <vector>
#include <thread>
#include <immintrin.h>
__attribute__((target("avx2"))) static uint32_t pack_avx2(const uint8_t* in, uint8_t* out, size_t n32) {
  __m256i bad = _mm256_setzero_si256();
  const __m256i m20 = _mm256_set1_epi8(0x20), ca = _mm256_set1_epi8('a'), cc = _mm256_set1_epi8('c'),
                cg = _mm256_set1_epi8('g'), ct = _mm256_set1_epi8('t'), m3 = _mm256_set1_epi8(3);
  for (size_t i = 0; i < n32; ++i) {
    __m256i x = _mm256_loadu_si256((const __m256i*)(in + 32 * i));
    __m256i l = _mm256_or_si256(x, m20);
    __m256i ok = _mm256_or_si256(_mm256_or_si256(_mm256_cmpeq_epi8(l, ca), _mm256_cmpeq_epi8(l, cc)),
                                 _mm256_or_si256(_mm256_cmpeq_epi8(l, cg), _mm256_cmpeq_epi8(l, ct)));
    bad = _mm256_or_si256(bad, _mm256_xor_si256(ok, _mm256_set1_epi8(-1)));
    // code = ((x >> 1) ^ (x >> 2)) & 3  (16-bit shifts are fine: masked per byte)
    __m256i c = _mm256_and_si256(_mm256_xor_si256(_mm256_srli_epi16(x, 1), _mm256_srli_epi16(x, 2)), m3);
    // pack 4 codes per byte: maddubs with (1,4) then madd with (1,16)
    __m256i p2 = _mm256_maddubs_epi16(c, _mm256_set1_epi16(0x0401));
    __m256i p4 = _mm256_madd_epi16(p2, _mm256_set1_epi32(0x00100001));
    // bytes 0 of each 32-bit lane hold the packed byte
    __m256i sh = _mm256_shuffle_epi8(p4, _mm256_setr_epi8(0,4,8,12,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,
                                                           0,4,8,12,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1,-1));
    uint32_t lo = (uint32_t)_mm256_extract_epi32(sh, 0), hi = (uint32_t)_mm256_extract_epi32(sh, 4);
    memcpy(out + 8 * i, &lo, 4);
    memcpy(out + 8 * i + 4, &hi, 4);
  }
  return (uint32_t)_mm256_movemask_epi8(bad);
}
int main() {
  unsigned hc = std::thread::hardware_concurrency();
  printf("hardware threads %u, avx2 %d\n", hc, __builtin_cpu_supports("avx2"));
  const size_t N = 300u << 20;
  std::vector<uint8_t> in(N), out(N / 4);
  for (size_t i = 0; i < N; ++i) in[i] = "ACGT"[(i * 2654435761u >> 7) & 3];
  for (unsigned T : {1u, 4u, 8u, 16u, 32u, 64u}) {
    if (T > 2 * hc) break;
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (unsigned t = 0; t < T; ++t) th.emplace_back([&, t] {
        size_t lo = N / 32 * t / T, hi = N / 32 * (t + 1) / T;
        pack_avx2(in.data() + 32 * lo, out.data() + 8 * lo, hi - lo);
      });
      for (auto& x : th) x.join();
      best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    printf("threads %u: %.1f GB/s\n", T, N / best / 1e9);
  }
}
