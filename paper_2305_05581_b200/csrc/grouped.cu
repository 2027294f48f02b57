// grouped.cu — the generic grouped, segmented FP64 GEMM entry point on the
// engine, stream-ordered (no host synchronisation).
//
// The device sweep (paper_2305_05581_b200/blockops.py) expresses every block
// algebra step that follows a two-site diagonalisation through it:
//   * complementary-operator formation (blocks.py:331 materialize_aux) and
//     the enlarged-Hamiltonian cross sums (blocks.py:262 _enlarged_hamiltonian):
//     coefficient-matrix x operator-stack products and Σ_i C_i · M_i
//     segment sums for three-factor strings (blocks.py:104 resolve);
//   * enlargement fused with the truncation rotation (blocks.py:190
//     enlarge_block + dmrg.py:254 _transform_tree): W^T (X ⊗ s) W as
//     T = X · W_c, new += s · W_r^T · T with the Kronecker placements as
//     segments (the enlarged operators are never materialised);
//   * White's prediction (driver.py:200 _predict_right / :228 _predict_left).
#include <algorithm>
#include <vector>

#include "../../include/sdmrg_b200.h"
#include "runtime.h"

using namespace sdmrg;

namespace {

static bool aligned_batch(const GemmBatch& gb, const Bases& bases) {
  for (const Seg& sg : gb.segs) {
    const uint64_t a = reinterpret_cast<uint64_t>(bases.p[sg.a >> kHandleShift] + (sg.a & kHandleMask));
    const uint64_t b = reinterpret_cast<uint64_t>(bases.p[sg.b >> kHandleShift] + (sg.b & kHandleMask));
    if ((a & 15) || (b & 15) || (sg.lda & 1) || (sg.ldb & 1)) return false;
  }
  return true;
}

}  // namespace

extern "C" {

int sdmrg_grouped_gemm(int trans_a, int trans_b, int64_t nprob, const int64_t* c_h,
                       const int32_t* ldc, const int32_t* m, const int32_t* n,
                       const int32_t* beta, const int64_t* seg_begin, const int64_t* a_h,
                       const int32_t* lda, const int64_t* b_h, const int32_t* ldb,
                       const int32_t* k, const double* scale, double* const* bases,
                       int nbases, void* stream_) {
  if (nprob < 0) return fail(SDMRG_EINVAL, "grouped_gemm: negative problem count");
  if (nbases < 1 || nbases > kMaxBases)
    return fail(SDMRG_EINVAL, "grouped_gemm: 1..8 base pointers");
  if (nprob == 0) return SDMRG_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  Bases b{};
  for (int i = 0; i < nbases; ++i) b.p[i] = bases[i];
  const uint64_t top = uint64_t(nbases) << kHandleShift;
  GemmBatch gb;
  gb.probs.reserve(nprob);
  gb.segs.reserve(seg_begin[nprob] - seg_begin[0]);
  for (int64_t p = 0; p < nprob; ++p) {
    if (m[p] < 0 || n[p] < 0) return fail(SDMRG_EINVAL, "grouped_gemm: negative extent");
    if (beta[p] != 0 && beta[p] != 1) return fail(SDMRG_EINVAL, "grouped_gemm: beta must be 0 or 1");
    if (seg_begin[p + 1] < seg_begin[p]) return fail(SDMRG_EINVAL, "grouped_gemm: segment ranges");
    if (uint64_t(c_h[p]) >= top) return fail(SDMRG_EINVAL, "grouped_gemm: C handle base");
    if (m[p] == 0 || n[p] == 0) continue;
    if (ldc[p] < n[p]) return fail(SDMRG_EINVAL, "grouped_gemm: ldc < n (row-major C)");
    gb.begin_prob(uint64_t(c_h[p]), ldc[p], m[p], n[p], beta[p]);
    for (int64_t s = seg_begin[p]; s < seg_begin[p + 1]; ++s) {
      if (k[s] < 0) return fail(SDMRG_EINVAL, "grouped_gemm: negative k");
      if (uint64_t(a_h[s]) >= top || uint64_t(b_h[s]) >= top)
        return fail(SDMRG_EINVAL, "grouped_gemm: operand handle base");
      gb.add_seg(uint64_t(a_h[s]), lda[s], uint64_t(b_h[s]), ldb[s], k[s], scale[s]);
    }
    gb.end_prob();
  }
  if (gb.tiles.empty()) return SDMRG_OK;
  gb.finalize_tiles();
  const bool bulk = aligned_batch(gb, b);
  // stream-ordered upload of the descriptors (pageable sources are staged
  // before cudaMemcpyAsync returns) and stream-ordered frees: no host sync
  std::vector<TileRec> recs(gb.tiles.size());
  for (size_t i = 0; i < gb.tiles.size(); ++i) {
    const Tile& t = gb.tiles[i];
    const Prob& p = gb.probs[t.prob];
    recs[i] = TileRec{p.c, p.ldc, p.beta, p.seg_begin, p.seg_end, t.row0, t.col0, t.tm, t.tn, t.colw};
  }
  DeviceBatch db;
  int* counter = nullptr;
  int rc = cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&db.tiles), recs.size() * sizeof(TileRec), stream),
                      "grouped_gemm tiles alloc");
  if (!rc && !gb.segs.empty())
    rc = cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&db.segs), gb.segs.size() * sizeof(Seg), stream),
                    "grouped_gemm segs alloc");
  if (!rc) rc = cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&counter), sizeof(int), stream),
                           "grouped_gemm counter alloc");
  if (!rc) rc = cuda_check(cudaMemcpyAsync(db.tiles, recs.data(), recs.size() * sizeof(TileRec),
                                           cudaMemcpyHostToDevice, stream), "grouped_gemm tiles upload");
  if (!rc && !gb.segs.empty())
    rc = cuda_check(cudaMemcpyAsync(db.segs, gb.segs.data(), gb.segs.size() * sizeof(Seg),
                                    cudaMemcpyHostToDevice, stream), "grouped_gemm segs upload");
  if (!rc) rc = cuda_check(cudaMemsetAsync(counter, 0, sizeof(int), stream), "grouped_gemm counter");
  db.ntiles = static_cast<int64_t>(gb.tiles.size());
  db.nprobs = static_cast<int64_t>(gb.probs.size());
  db.nsegs = static_cast<int64_t>(gb.segs.size());
  if (!rc) rc = launch_engine(trans_a != 0, trans_b != 0, db, b, counter, stream, bulk);
  // the staged copies above completed into device memory before the kernel
  // reads them (same stream); pageable host vectors may now go out of scope
  if (db.tiles) cudaFreeAsync(db.tiles, stream);
  if (db.segs) cudaFreeAsync(db.segs, stream);
  if (counter) cudaFreeAsync(counter, stream);
  db.tiles = nullptr;
  db.segs = nullptr;
  return rc;
}

}  // extern "C"
