// csrc/hostpack.cu -- host side of the 2-bit sequence path.
//
// The paper's Sequence accessor stores DNA as symbol codes; for an ACGT-only
// chunk the host API uploads them as 2-bit codes (4 bases per byte: a quarter of the ASCII
// bytes over PCIe) and the device expands them to byte codes (unpack2_kernel in
// kernels.cu).  Packing runs on a pool of host threads with AVX2 (validation fused: any
// byte outside ACGTacgt -- N included -- sends the chunk down the ASCII/byte-code path,
// whose device pack kernel reports bad bytes and marks pairs with N).
//
// Host code only: this file holds no device code and no alignment arithmetic.
#include <immintrin.h>

#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hostpack.h"

namespace anyseq {

namespace {

// 2-bit code of an ASCII base: ((x >> 1) ^ (x >> 2)) & 3 maps A/a -> 0, C/c -> 1, G/g -> 2,
// T/t -> 3 (the same codes as the device's byte path).
inline uint32_t code2(uint8_t x) { return ((x >> 1) ^ (x >> 2)) & 3u; }
inline bool is_acgt(uint8_t x) {
  const uint8_t l = x | 0x20;
  return l == 'a' || l == 'c' || l == 'g' || l == 't';
}

// Scalar form: n bases (n % 4 == 0 or the tail of a range) -> out[n / 4] (+ partial byte).
bool pack_scalar(const uint8_t* in, size_t n, uint8_t* out) {
  bool ok = true;
  for (size_t i = 0; i < n; i += 4) {
    uint32_t b = 0;
    for (size_t k = 0; k < 4 && i + k < n; ++k) {
      ok &= is_acgt(in[i + k]);
      b |= code2(in[i + k]) << (2 * k);
    }
    out[i >> 2] = (uint8_t)b;
  }
  return ok;
}

// Per byte x (either case): the low nibble of 'a','c','g','t' is 1, 3, 7, 4; a 16-entry
// table indexed by the low nibble gives the lowercase letter that nibble must come from
// (0 = none) and a second one its 2-bit code, so validation is one table lookup and one
// compare of (x | 0x20) and the code one more lookup.  Four codes per byte: maddubs
// (c0 + 4 c1), madd (p0 + 16 p1), then the low byte of every 32-bit lane.
__attribute__((target("avx2"))) bool pack_avx2(const uint8_t* in, size_t n, uint8_t* out) {
  const size_t n32 = n / 32;
  const __m256i lowtab = _mm256_setr_epi8(0, 'a', 0, 'c', 't', 0, 0, 'g', 0, 0, 0, 0, 0, 0, 0, 0,
                                          0, 'a', 0, 'c', 't', 0, 0, 'g', 0, 0, 0, 0, 0, 0, 0, 0);
  const __m256i codetab = _mm256_setr_epi8(0, 0, 0, 1, 3, 0, 0, 2, 0, 0, 0, 0, 0, 0, 0, 0,
                                           0, 0, 0, 1, 3, 0, 0, 2, 0, 0, 0, 0, 0, 0, 0, 0);
  const __m256i m0f = _mm256_set1_epi8(0x0f), m20 = _mm256_set1_epi8(0x20);
  const __m256i w2 = _mm256_set1_epi16(0x0401), w4 = _mm256_set1_epi32(0x00100001);
  const __m256i gather = _mm256_setr_epi8(0, 4, 8, 12, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1,
                                          -1, -1, 0, 4, 8, 12, -1, -1, -1, -1, -1, -1, -1, -1,
                                          -1, -1, -1, -1);
  uint32_t bad = 0;
  for (size_t i = 0; i < n32; ++i) {
    const __m256i x = _mm256_loadu_si256((const __m256i*)(in + 32 * i));
    const __m256i lo = _mm256_and_si256(x, m0f);
    const __m256i ok = _mm256_cmpeq_epi8(_mm256_or_si256(x, m20), _mm256_shuffle_epi8(lowtab, lo));
    bad |= ~(uint32_t)_mm256_movemask_epi8(ok);
    const __m256i c = _mm256_shuffle_epi8(codetab, lo);
    const __m256i p4 = _mm256_madd_epi16(_mm256_maddubs_epi16(c, w2), w4);
    const __m256i sh = _mm256_shuffle_epi8(p4, gather);
    const uint32_t a0 = (uint32_t)_mm256_extract_epi32(sh, 0);
    const uint32_t a1 = (uint32_t)_mm256_extract_epi32(sh, 4);
    memcpy(out + 8 * i, &a0, 4);
    memcpy(out + 8 * i + 4, &a1, 4);
  }
  bool okall = bad == 0;
  if (n32 * 32 < n) okall &= pack_scalar(in + n32 * 32, n - n32 * 32, out + n32 * 8);
  return okall;
}

__attribute__((target("avx512f,avx512bw"))) bool pack_avx512(const uint8_t* in, size_t n,
                                                                uint8_t* out) {
  const size_t n64 = n / 64;
  const __m512i lowtab = _mm512_broadcast_i32x4(
      _mm_setr_epi8(0, 'a', 0, 'c', 't', 0, 0, 'g', 0, 0, 0, 0, 0, 0, 0, 0));
  const __m512i codetab = _mm512_broadcast_i32x4(
      _mm_setr_epi8(0, 0, 0, 1, 3, 0, 0, 2, 0, 0, 0, 0, 0, 0, 0, 0));
  const __m512i m0f = _mm512_set1_epi8(0x0f), m20 = _mm512_set1_epi8(0x20);
  const __m512i w2 = _mm512_set1_epi16(0x0401), w4 = _mm512_set1_epi32(0x00100001);
  __mmask64 bad = 0;
  for (size_t i = 0; i < n64; ++i) {
    const __m512i x = _mm512_loadu_si512((const void*)(in + 64 * i));
    const __m512i lo = _mm512_and_si512(x, m0f);
    bad |= _mm512_cmpneq_epi8_mask(_mm512_or_si512(x, m20), _mm512_shuffle_epi8(lowtab, lo));
    const __m512i c = _mm512_shuffle_epi8(codetab, lo);
    const __m512i p4 = _mm512_madd_epi16(_mm512_maddubs_epi16(c, w2), w4);
    _mm_storeu_si128((__m128i*)(out + 16 * i), _mm512_cvtepi32_epi8(p4));  // low byte of each lane
  }
  bool okall = bad == 0;
  if (n64 * 64 < n) okall &= pack_scalar(in + n64 * 64, n - n64 * 64, out + n64 * 16);
  return okall;
}

const bool kHaveAvx2 = __builtin_cpu_supports("avx2");
const bool kHaveAvx512 = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");

bool pack_range(const uint8_t* in, size_t n, uint8_t* out) {
  if (kHaveAvx512) return pack_avx512(in, n, out);
  return kHaveAvx2 ? pack_avx2(in, n, out) : pack_scalar(in, n, out);
}

}  // namespace

// A fixed pool of worker threads for parallel-for jobs issued by one caller at a time.
struct PackPool::Impl {
  std::vector<std::thread> th;
  std::mutex call_mu;  // one parallel_for at a time (shard threads of a multi-device call)
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::function<void(int)> job;
  int parts = 0, next = 0, done = 0;
  uint64_t gen = 0;
  bool stop = false;
  void worker() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu);
    for (;;) {
      cv.wait(lk, [&] { return stop || (gen != seen && next < parts); });
      if (stop) return;
      while (next < parts) {
        const int p = next++;
        lk.unlock();
        job(p);
        lk.lock();
        if (++done == parts) done_cv.notify_all();
      }
      seen = gen;
    }
  }
};

PackPool::PackPool(int threads) : impl_(new Impl) {
  if (threads < 1) threads = (int)std::max(1u, std::thread::hardware_concurrency());
  nthreads_ = threads;
  for (int t = 1; t < threads; ++t) impl_->th.emplace_back([this] { impl_->worker(); });
}

PackPool::~PackPool() {
  {
    std::lock_guard<std::mutex> lk(impl_->mu);
    impl_->stop = true;
  }
  impl_->cv.notify_all();
  for (auto& t : impl_->th) t.join();
  delete impl_;
}

void PackPool::parallel_for(int parts, const std::function<void(int)>& f) {
  if (parts <= 0) return;
  std::lock_guard<std::mutex> call(impl_->call_mu);
  std::unique_lock<std::mutex> lk(impl_->mu);
  impl_->job = f;
  impl_->parts = parts;
  impl_->next = 0;
  impl_->done = 0;
  ++impl_->gen;
  impl_->cv.notify_all();
  // the caller works too
  while (impl_->next < impl_->parts) {
    const int p = impl_->next++;
    lk.unlock();
    f(p);
    lk.lock();
    ++impl_->done;
  }
  impl_->done_cv.wait(lk, [&] { return impl_->done == impl_->parts; });
  impl_->parts = 0;
}

bool PackPool::pack2(const char* in, uint64_t n, uint8_t* out) {
  if (n == 0) return true;
  // pieces of whole 128-base blocks (32 output bytes): no two pieces share an output byte
  const uint64_t blocks = (n + 127) / 128;
  const int parts = (int)std::min<uint64_t>(blocks, (uint64_t)nthreads_ * 4);
  std::vector<char> ok(parts, 1);
  parallel_for(parts, [&](int p) {
    const uint64_t b0 = blocks * p / parts, b1 = blocks * (p + 1) / parts;
    const uint64_t lo = b0 * 128, hi = std::min<uint64_t>(n, b1 * 128);
    if (lo < hi) ok[p] = pack_range((const uint8_t*)in + lo, hi - lo, out + lo / 4);
  });
  for (char x : ok)
    if (!x) return false;
  return true;
}

}  // namespace anyseq
