// csrc/fill_dispatch.cu -- variant -> kernel instance, persistent grid sizing.
#include <cstdlib>
#include <mutex>
#include "kernels.h"
#include "fill_inst.cuh"

namespace anyseq {
FillFn fill_fn_s16(int v, int kind, int gap, bool pos);
FillFn fill_fn_s32(int v, int kind, int gap, bool pos);
FillFn fill_fn_tb(int v, int kind, int gap, bool pos);
FillFn fill_fn_s16_spec(int v, int kind, bool pos);
FillFn fill_fn_s16_spec_a21(int v, int kind, bool pos);
FillFn fill_fn_s16_spec_l1(int v, int kind, bool pos);

static FillFn pick(int v, int kind, int gap, bool pos) {
  if (v <= 2) return fill_fn_s16(v, kind, gap, pos);
  if (v <= 4) return fill_fn_s32(v, kind, gap, pos);
  return fill_fn_tb(v, kind, gap, pos);
}

cudaError_t launch_fill(int variant, int kind, int gap, const FillArgs& a, cudaStream_t st,
                        int num_sms, int* grid_out) {
  static std::mutex mu;
  static int occ[NV][3][2][2][4][16];  // per device up to 16
  static bool init = false;
  const int pos = a.pos ? 1 : 0;
  // compile-time-specialised instances: affine (5, 1) (C2-C5), the paper's affine (2, 1) and
  // linear g = 1 (Fig. 5); everything else takes its constants from the parameter bank
  int spec = 0;
  if (variant <= 2 && a.P.ge == 1) {
    if (gap == GAFFINE && a.P.go == 5) spec = 1;
    else if (gap == GAFFINE && a.P.go == 2) spec = 2;
    else if (gap == GLINEAR) spec = 3;
  }
  FillFn fn = spec == 1 ? fill_fn_s16_spec(variant, kind, pos != 0)
            : spec == 2 ? fill_fn_s16_spec_a21(variant, kind, pos != 0)
            : spec == 3 ? fill_fn_s16_spec_l1(variant, kind, pos != 0)
                        : pick(variant, kind, gap, pos != 0);
  if (!fn) return cudaErrorInvalidValue;
  int dev = 0;
  cudaGetDevice(&dev);
  int nb;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!init) { memset(occ, 0, sizeof(occ)); init = true; }
    nb = occ[variant][kind][gap][pos][spec][dev & 15];
    if (nb == 0) {
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, 128, 0);
      if (e != cudaSuccess) return e;
      if (nb < 1) nb = 1;
      occ[variant][kind][gap][pos][spec][dev & 15] = nb;
    }
  }
  // debug/tuning: ANYSEQ_FILL_BPS caps the resident blocks per SM of the persistent grid
  static const int bps_cap = [] {
    const char* e = getenv("ANYSEQ_FILL_BPS");
    return e ? atoi(e) : 0;
  }();
  if (bps_cap > 0 && nb > bps_cap) nb = bps_cap;
  const int grid = num_sms * nb;
  if (grid_out) *grid_out = grid;
  // dynamic slot hand-out pays off only with several warp-slots per warp: with fewer, the
  // static order (warp-slot w -> warp w, i.e. spread over the blocks and so over the SMs)
  // keeps the few busy warps on separate sub-partitions
  FillArgs b = a;
  const int64_t nws = ((int64_t)a.slot_hi - a.slot_lo + 3) / 4;  // L = 8: 4 slots per warp
  if (b.ticket && (a.nslots_dev || nws < 2ll * grid * 4)) b.ticket = nullptr;
  fn<<<grid, 128, 0, st>>>(b);
  return cudaGetLastError();
}
}  // namespace anyseq
