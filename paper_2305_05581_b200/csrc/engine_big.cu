// engine_big.cu — a second instance of the engine (engine.cuh) with 128 x 128
// tiles, 16 DMMA warps and 2 producer warps per CTA, one CTA per SM, for the
// phase-2 σ blocks of 65..128 rows and columns: one CTA loads each shared
// row (A) and column (B) operand panel once for all four 64 x 64 quadrants
// instead of four CTAs streaming two copies of each (L=50 D=4096: 76% of the
// phase-2 FLOPs sit in such blocks; phase 2 moved ~3.3x its compulsory
// bytes through DRAM, profiles/r2_notes.md).  Descriptor layouts (TileRec,
// Seg, Bases) are the same as the default instance's.
#define SDMRG_BIG 1
#define SDMRG_TILE 128
#define sdmrg sdmrg_big
#include "engine.cuh"
#undef sdmrg

#include <algorithm>
#include <map>
#include <mutex>

namespace {

template <bool TB, bool ONE>
int big_grid() {
  static std::mutex mu;
  static std::map<int, int> grids;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = grids.find(dev);
  if (it != grids.end()) return it->second;
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto* k = sdmrg_big::seg_gemm_kernel<false, TB, true, ONE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       sdmrg_big::smem_bytes<false, TB>());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, sdmrg_big::THREADS,
                                                sdmrg_big::smem_bytes<false, TB>());
  grids[dev] = sms * std::max(per, 1);
  return grids[dev];
}

template <bool TB, bool ONE>
void launch(const sdmrg_big::TileRec* t, int ntiles, const sdmrg_big::Seg* sg, int* counter,
            const sdmrg_big::Bases& b, cudaStream_t st) {
  const int grid = std::min(big_grid<TB, ONE>(), ntiles);
  sdmrg_big::seg_gemm_kernel<false, TB, true, ONE>
      <<<grid, sdmrg_big::THREADS, sdmrg_big::smem_bytes<false, TB>(), st>>>(t, ntiles, sg, counter,
                                                                            b);
}

}  // namespace

// Launch the big-tile instance (BULK operands, TA = false; trans_b: the
// phase-1 form T = A B^T, else phase 2's C += A B) over an uploaded tile /
// segment list; tiles must be <= 128 x 128.
extern "C" int sdmrg_internal_launch_big(const void* tiles, int ntiles, const void* segs,
                                         int* counter, const void* bases, void* stream,
                                         int one_body, int trans_b) {
  if (ntiles <= 0) return 0;
  const auto& b = *static_cast<const sdmrg_big::Bases*>(bases);
  const auto* t = static_cast<const sdmrg_big::TileRec*>(tiles);
  const auto* sg = static_cast<const sdmrg_big::Seg*>(segs);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (trans_b) launch<true, false>(t, ntiles, sg, counter, b, st);
  else if (one_body) launch<false, true>(t, ntiles, sg, counter, b, st);
  else launch<false, false>(t, ntiles, sg, counter, b, st);
  return static_cast<int>(cudaGetLastError());
}

extern "C" int sdmrg_internal_big_grid() { return big_grid<false, false>(); }
