// csrc/hostpack.h -- host-side 2-bit packing of ACGT-only chunks.
#pragma once
#include <cstdint>
#include <functional>

namespace anyseq {

class PackPool {
 public:
  explicit PackPool(int threads = 0);  // 0 = hardware concurrency (the caller is one of them)
  ~PackPool();
  PackPool(const PackPool&) = delete;
  PackPool& operator=(const PackPool&) = delete;
  int threads() const { return nthreads_; }
  // Packs ASCII bases in[0, n) into 2-bit codes: base p -> bits 2 (p % 4) of out[p / 4]
  // (A/a 0, C/c 1, G/g 2, T/t 3); out needs ceil(n / 4) bytes.  Returns false if any byte
  // is not one of ACGTacgt (out is then unspecified and the caller takes the byte path).
  bool pack2(const char* in, uint64_t n, uint8_t* out);
  void parallel_for(int parts, const std::function<void(int)>& f);

 private:
  struct Impl;
  Impl* impl_;
  int nthreads_ = 1;
};

}  // namespace anyseq
