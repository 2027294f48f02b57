// runtime.h — host-side plumbing shared by the C-ABI entry points: error
// slot, launch accounting, and GemmBatch (host staging of a grouped GEMM
// descriptor list that is uploaded once and launched on the engine).
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "engine.cuh"

namespace sdmrg {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);
void count_launch(int n = 1);

// Persistent-grid size for the engine (148 SMs x resident CTAs).
int engine_grid(bool ta, bool tb);

// Device-side copy of a descriptor list.
struct DeviceBatch {
  TileRec* tiles = nullptr;
  Seg* segs = nullptr;
  int64_t ntiles = 0, nprobs = 0, nsegs = 0;
  void release();
};

// Host staging of problems/segments; tiles derived per problem.
struct GemmBatch {
  int cap = 0;          // tile edge (0: the default instance's BM x BN)
  std::vector<Prob> probs;
  std::vector<Seg> segs;
  std::vector<Tile> tiles;
  std::vector<double> tile_cost;
  int begin_prob(uint64_t c, int ldc, int m, int n, int beta);
  // move another batch's problems, segments and tiles behind this one's
  void append(GemmBatch&& other);
  void add_seg(uint64_t a, int lda, uint64_t b, int ldb, int k, double scale, int btile = 0);
  // the column-tile width end_prob uses for an n-column problem
  static int col_tile_width(int n);
  void end_prob();
  // order tiles by descending cost (longest-processing-time first)
  // octaves > 0: costs bucketed to 1/octaves of a power of two (emission
  // order kept inside a bucket) instead of exact distinct costs
  // by_problem: order by each problem's largest tile cost, a problem's tiles
  // kept together (sibling tiles share operand panels in L2)
  void finalize_tiles(int octaves = 0, bool by_problem = false);
  int upload(DeviceBatch* out, cudaStream_t stream) const;
  int64_t flops() const;  // useful (unpadded) FLOPs
};

// Launch the engine over an uploaded batch.  counter must point at one
// zeroed device int (reset by the caller or by this function when reset=1).
// bulk: every operand row 16-byte aligned, even leading dimensions, zero
// pads (engine.cuh BULK) — the H_eff plan's padded layouts only.
// one_body: (!ta && !tb && bulk only) the single always-scaling consumer body
int launch_engine(bool ta, bool tb, const DeviceBatch& b, const Bases& bases, int* counter,
                  cudaStream_t stream, bool bulk = false, bool one_body = false);

}  // namespace sdmrg

#include "fused.cuh"

namespace sdmrg {

// Host staging of the fused small-sector work list (fused.cuh): one σ
// problem = products (FSeg) + column tiles of <= F_RT 8-blocks.
struct FusedBatch {
  std::vector<FTileRec> tiles;
  std::vector<double> tile_cost;
  std::vector<FSeg> segs;
  FTileRec* d_tiles = nullptr;
  FSeg* d_segs = nullptr;
  int64_t ntiles = 0;
  // σ problem at handle c (q x r, ld ldc) over segs [seg_begin, segs.size())
  void add_problem(uint64_t c, int ldc, int q, int r, int beta, int32_t seg_begin);
  void finalize();         // descending-cost order (LPT)
  int upload();
  void release();
};
int launch_fused(const FusedBatch& b, const Bases& bases, int* counter, cudaStream_t stream);
int fused_grid_size();  // persistent fused-kernel grid on the current device

}  // namespace sdmrg
