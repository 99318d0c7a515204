// Host-side 2-bit packer (csrc/hostpack.cu): codes of every ACGTacgt
// string of length 0..699 checked base by base, a bad byte anywhere detected, throughput.
#include "hostpack.h"
#include <chrono>
#include <cstdio>
#include <vector>
#include <random>
#include <cstring>
int main() {
  // correctness: random ACGTacgt strings of every length 0..300 and every offset vs scalar codes
  std::mt19937 rng(1);
  const char* al = "ACGTacgt";
  anyseq::PackPool pool(4);
  for (int n = 0; n < 700; ++n) {
    std::vector<char> in(n); for (auto& c : in) c = al[rng() % 8];
    std::vector<uint8_t> out((n + 3) / 4 + 8, 0xEE);
    bool ok = pool.pack2(in.data(), n, out.data());
    if (!ok) { printf("false negative n=%d\n", n); return 1; }
    for (int p = 0; p < n; ++p) {
      char c = in[p] | 0x20; int want = c == 'a' ? 0 : c == 'c' ? 1 : c == 'g' ? 2 : 3;
      if (((out[p >> 2] >> (2 * (p & 3))) & 3) != want) { printf("bad code n=%d p=%d\n", n, p); return 1; }
    }
    for (int b = 0; b < 256 && n > 0; b += 7) {  // a bad byte anywhere is detected
      std::vector<char> x = in; int pos = rng() % n; x[pos] = (char)b;
      char l = (char)(b | 0x20);
      bool valid = l == 'a' || l == 'c' || l == 'g' || l == 't';
      if (pool.pack2(x.data(), n, out.data()) != valid) { printf("validation n=%d b=%d\n", n, b); return 1; }
    }
  }
  const size_t N = 16u << 20;
  std::vector<char> in(N); std::vector<uint8_t> out(N / 4 + 64);
  for (size_t i = 0; i < N; ++i) in[i] = "ACGT"[(i * 2654435761u >> 7) & 3];
  anyseq::PackPool big(0);
  for (int rep = 0; rep < 4; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    bool ok = big.pack2(in.data(), N, out.data());
    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("threads %d ok %d  %.1f GB/s\n", big.threads(), ok, N / dt / 1e9);
  }
  printf("all ok\n");
}
