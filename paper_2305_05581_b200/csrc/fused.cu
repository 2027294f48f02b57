// fused.cu — host side of the fused small-sector H_eff·ψ kernel (fused.cuh):
// tile emission, LPT order, upload, launch.
#include <algorithm>
#include <map>
#include <mutex>
#include <numeric>

#define SDMRG_FUSED_KERNEL 1
#include "../../include/sdmrg_b200.h"
#include "runtime.h"
#include "fused.cuh"

namespace sdmrg {

void FusedBatch::add_problem(uint64_t c, int ldc, int q, int r, int beta, int32_t seg_begin) {
  const int32_t seg_end = static_cast<int32_t>(segs.size());
  if (seg_end <= seg_begin) return;
  // DMMA work of the problem per 8-column block of σ (step 1 + step 2)
  const int qb = (q + 7) / 8;
  double kcost = 0.0;
  for (int s = seg_begin; s < seg_end; ++s) {
    const FSeg& sg = segs[s];
    const int mb = (sg.m + 7) / 8;
    kcost += double(mb) * (sg.ident ? 1.0 : (sg.n + 3) / 4) + double(mb) * 2.0 * qb;
  }
  // column tiles of 4 blocks, the remainder as 2 + 1 (fused_tile_blocks):
  // every tile keeps the CTA's four DMMA warps busy
  const int rb = (r + 7) / 8;
  for (int b0 = 0; b0 < rb;) {
    const int w = fused_tile_blocks(rb - b0);
    const int r0 = 8 * b0, rt = std::min(8 * w, r - r0);
    FTileRec t{};
    t.c = c + static_cast<uint64_t>(r0);
    t.ldc = ldc;
    t.beta = beta;
    t.seg_begin = seg_begin;
    t.seg_end = seg_end;
    t.q = static_cast<int16_t>(q);
    t.rt = static_cast<int16_t>(rt);
    t.r0 = r0;
    tiles.push_back(t);
    tile_cost.push_back(kcost * w / 4.0 * 4.0 + 64.0);  // per-warp work: the tile's blocks / 4 warps
    b0 += w;
  }
}

void FusedBatch::finalize() {
  std::vector<int64_t> idx(tiles.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(),
                   [&](int64_t a, int64_t b) { return tile_cost[a] > tile_cost[b]; });
  std::vector<FTileRec> t2(tiles.size());
  std::vector<double> c2(tiles.size());
  for (size_t i = 0; i < idx.size(); ++i) {
    t2[i] = tiles[idx[i]];
    c2[i] = tile_cost[idx[i]];
  }
  tiles.swap(t2);
  tile_cost.swap(c2);
}

int FusedBatch::upload() {
  int rc = SDMRG_OK;
  ntiles = static_cast<int64_t>(tiles.size());
  if (!tiles.empty()) {
    rc = cuda_check(cudaMalloc(&d_tiles, tiles.size() * sizeof(FTileRec)), "cudaMalloc ftiles");
    if (!rc)
      rc = cuda_check(cudaMemcpy(d_tiles, tiles.data(), tiles.size() * sizeof(FTileRec),
                                 cudaMemcpyHostToDevice), "upload ftiles");
  }
  if (!rc && !segs.empty()) {
    rc = cuda_check(cudaMalloc(&d_segs, segs.size() * sizeof(FSeg)), "cudaMalloc fsegs");
    if (!rc)
      rc = cuda_check(cudaMemcpy(d_segs, segs.data(), segs.size() * sizeof(FSeg),
                                 cudaMemcpyHostToDevice), "upload fsegs");
  }
  tiles = std::vector<FTileRec>();
  tile_cost = std::vector<double>();
  segs = std::vector<FSeg>();
  return rc;
}

void FusedBatch::release() {
  if (d_tiles) cudaFree(d_tiles);
  if (d_segs) cudaFree(d_segs);
  d_tiles = nullptr;
  d_segs = nullptr;
  ntiles = 0;
}

// persistent grid per device (smem opt-in is a per-device attribute)
static int fused_grid() {
  static std::mutex mu;
  static std::map<int, int> grids;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = grids.find(dev);
  if (it != grids.end()) return it->second;
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(fused_heff_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       fused_smem_bytes());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fused_heff_kernel, F_THREADS,
                                                fused_smem_bytes());
  grids[dev] = sms * std::max(per, 1);
  return grids[dev];
}

int fused_grid_size() { return fused_grid(); }

int launch_fused(const FusedBatch& b, const Bases& bases, int* counter, cudaStream_t stream) {
  if (b.ntiles == 0) return SDMRG_OK;
  const int grid = static_cast<int>(std::min<int64_t>(fused_grid(), b.ntiles));
  fused_heff_kernel<<<grid, F_THREADS, fused_smem_bytes(), stream>>>(
      b.d_tiles, static_cast<int>(b.ntiles), b.d_segs, counter, bases);
  count_launch();
  return cuda_check(cudaGetLastError(), "fused_heff_kernel launch");
}

}  // namespace sdmrg
