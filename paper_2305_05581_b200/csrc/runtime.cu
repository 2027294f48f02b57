#include <cmath>
// runtime.cu — engine launch plumbing and the GEMM-level C-ABI entry points
// (gemm.py backend contract and sbmm4s.py Alg. 2).
#include <algorithm>
#include <functional>
#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>

#include "../../include/sdmrg_b200.h"
#include "runtime.h"

namespace sdmrg {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SDMRG_OK;
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? SDMRG_ENOMEM : SDMRG_ECUDA;
}
void count_launch(int n) { g_launches += n; }

// Persistent grid per (device, TA, TB): the dynamic shared-memory opt-in is a
// per-device function attribute, so it is set once on every device the
// process launches on (a process-wide static broke device 1+).
template <bool TA, bool TB>
static int grid_for() {
  static std::mutex mu;
  static std::map<int, int> grids;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = grids.find(dev);
  if (it != grids.end()) return it->second;
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(seg_gemm_kernel<TA, TB, false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<TA, TB>());
  cudaFuncSetAttribute(seg_gemm_kernel<TA, TB, true>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<TA, TB>());
  if (!TA && !TB)
    cudaFuncSetAttribute(seg_gemm_kernel<false, false, true, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<TA, TB>());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, seg_gemm_kernel<TA, TB, true>, THREADS,
                                                smem_bytes<TA, TB>());
  const int grid = sms * std::max(per, 1);
  grids[dev] = grid;
  return grid;
}

int engine_grid(bool ta, bool tb) {
  if (!ta && !tb) return grid_for<false, false>();
  if (!ta && tb) return grid_for<false, true>();
  if (ta && !tb) return grid_for<true, false>();
  return grid_for<true, true>();
}

void DeviceBatch::release() {
  if (tiles) cudaFree(tiles);
  if (segs) cudaFree(segs);
  tiles = nullptr;
  segs = nullptr;
  ntiles = nprobs = nsegs = 0;
}

int GemmBatch::begin_prob(uint64_t c, int ldc, int m, int n, int beta) {
  Prob p{};
  p.c = c;
  p.ldc = ldc;
  p.m = m;
  p.n = n;
  p.seg_begin = p.seg_end = static_cast<int32_t>(segs.size());
  p.beta = beta;
  probs.push_back(p);
  return static_cast<int>(probs.size()) - 1;
}

void GemmBatch::add_seg(uint64_t a, int lda, uint64_t b, int ldb, int k, double scale,
                        int btile) {
  if (k <= 0) return;  // the engine requires non-empty segments
  Seg s{};
  s.a = a;
  s.b = b;
  s.lda = lda;
  s.ldb = ldb;
  s.k = k;
  s.btile = btile;
  s.scale = scale;
  segs.push_back(s);
  probs.back().seg_end = static_cast<int32_t>(segs.size());
}

int GemmBatch::col_tile_width(int n) {
  const int nt = (n + BN - 1) / BN;
  return std::max(((n + nt - 1) / nt + 7) / 8 * 8, 8);
}

void GemmBatch::end_prob() {
  const int pi = static_cast<int>(probs.size()) - 1;
  const Prob& p = probs[pi];
  int64_t ksum = 0;
  for (int s = p.seg_begin; s < p.seg_end; ++s) ksum += (segs[s].k + 3) / 4 * 4;
  // balanced tiles: ceil(extent/64) tiles per dimension of equal size
  // (rounded up to the 8-row DMMA granularity), e.g. 138 -> 48+48+42
  auto split = [](int extent, int cap) {
    const int nt = (extent + cap - 1) / cap;
    const int per = ((extent + nt - 1) / nt + 7) / 8 * 8;
    return std::max(per, 8);
  };
  const int tm = split(p.m, cap > 0 ? cap : BM), tn = split(p.n, cap > 0 ? cap : BN);
  for (int r0 = 0; r0 < p.m; r0 += tm)
    for (int c0 = 0; c0 < p.n; c0 += tn) {
      const int mm = std::min(tm, p.m - r0), nn = std::min(tn, p.n - c0);
      Tile t{pi, r0, c0, static_cast<int16_t>(mm), static_cast<int16_t>(nn), tn};
      tiles.push_back(t);
      tile_cost.push_back(double(ksum) * ((mm + 7) / 8 * 8) * ((nn + 7) / 8 * 8) + 4096.0);
    }
}

void GemmBatch::append(GemmBatch&& o) {
  const int32_t pbase = static_cast<int32_t>(probs.size());
  const int32_t sbase = static_cast<int32_t>(segs.size());
  for (Prob p : o.probs) {
    p.seg_begin += sbase;
    p.seg_end += sbase;
    probs.push_back(p);
  }
  segs.insert(segs.end(), o.segs.begin(), o.segs.end());
  for (Tile t : o.tiles) {
    t.prob += pbase;
    tiles.push_back(t);
  }
  tile_cost.insert(tile_cost.end(), o.tile_cost.begin(), o.tile_cost.end());
  o = GemmBatch();
}

void GemmBatch::finalize_tiles(int octaves, bool by_problem) {
  // stable descending-cost order by bucketing on the (few) distinct costs:
  // O(n + u log u) instead of a comparison sort of millions of tiles
  if (octaves > 0)
    for (double& c : tile_cost) c = std::exp2(std::floor(std::log2(c) * octaves) / octaves);
  std::vector<double> own;
  if (by_problem) {  // sort keys: the problem's largest tile cost
    own = tile_cost;
    std::vector<double> pmax(probs.size(), 0.0);
    for (size_t i = 0; i < tiles.size(); ++i)
      pmax[tiles[i].prob] = std::max(pmax[tiles[i].prob], tile_cost[i]);
    for (size_t i = 0; i < tiles.size(); ++i) tile_cost[i] = pmax[tiles[i].prob];
  }
  std::vector<double> uniq(tile_cost);
  std::sort(uniq.begin(), uniq.end(), std::greater<double>());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  std::vector<int64_t> start(uniq.size() + 1, 0);
  std::vector<int32_t> bucket(tiles.size());
  for (size_t i = 0; i < tiles.size(); ++i) {
    const auto it = std::lower_bound(uniq.begin(), uniq.end(), tile_cost[i], std::greater<double>());
    bucket[i] = static_cast<int32_t>(it - uniq.begin());
    ++start[bucket[i] + 1];
  }
  for (size_t b = 0; b < uniq.size(); ++b) start[b + 1] += start[b];
  std::vector<Tile> t2(tiles.size());
  std::vector<double> c2(tiles.size());
  for (size_t i = 0; i < tiles.size(); ++i) {
    const int64_t dst = start[bucket[i]]++;
    t2[dst] = tiles[i];
    c2[dst] = by_problem ? own[i] : tile_cost[i];  // the tile's own cost
  }
  tiles.swap(t2);
  tile_cost.swap(c2);
}

int64_t GemmBatch::flops() const {
  int64_t f = 0;
  for (const Prob& p : probs)
    for (int s = p.seg_begin; s < p.seg_end; ++s) f += 2LL * p.m * p.n * segs[s].k;
  return f;
}

int GemmBatch::upload(DeviceBatch* out, cudaStream_t stream) const {
  out->release();
  int rc;
  if (!tiles.empty()) {
    std::vector<TileRec> recs(tiles.size());
    for (size_t i = 0; i < tiles.size(); ++i) {
      const Tile& t = tiles[i];
      const Prob& p = probs[t.prob];
      recs[i] = TileRec{p.c, p.ldc, p.beta, p.seg_begin, p.seg_end, t.row0, t.col0, t.tm, t.tn,
                        t.colw};
    }
    if ((rc = cuda_check(cudaMalloc(&out->tiles, recs.size() * sizeof(TileRec)), "cudaMalloc tiles")))
      return rc;
    if ((rc = cuda_check(cudaMemcpy(out->tiles, recs.data(), recs.size() * sizeof(TileRec),
                                    cudaMemcpyHostToDevice),
                         "upload tiles")))
      return rc;
  }
  if (!segs.empty()) {
    if ((rc = cuda_check(cudaMalloc(&out->segs, segs.size() * sizeof(Seg)), "cudaMalloc segs")))
      return rc;
    if ((rc = cuda_check(cudaMemcpy(out->segs, segs.data(), segs.size() * sizeof(Seg),
                                    cudaMemcpyHostToDevice),
                         "upload segs")))
      return rc;
  }
  out->ntiles = static_cast<int64_t>(tiles.size());
  out->nprobs = static_cast<int64_t>(probs.size());
  out->nsegs = static_cast<int64_t>(segs.size());
  (void)stream;
  return SDMRG_OK;
}

template <bool TA, bool TB>
static void launch_t(bool bulk, bool one, const DeviceBatch& b, const Bases& bases, int* counter,
                     cudaStream_t stream) {
  const int grid = std::min<int64_t>(grid_for<TA, TB>(), std::max<int64_t>(b.ntiles, 1));
  if constexpr (!TA && !TB) {
    if (bulk && one) {
      seg_gemm_kernel<false, false, true, true><<<grid, THREADS, smem_bytes<TA, TB>(), stream>>>(
          b.tiles, static_cast<int>(b.ntiles), b.segs, counter, bases);
      return;
    }
  }
  if (bulk)
    seg_gemm_kernel<TA, TB, true><<<grid, THREADS, smem_bytes<TA, TB>(), stream>>>(
        b.tiles, static_cast<int>(b.ntiles), b.segs, counter, bases);
  else
    seg_gemm_kernel<TA, TB, false><<<grid, THREADS, smem_bytes<TA, TB>(), stream>>>(
        b.tiles, static_cast<int>(b.ntiles), b.segs, counter, bases);
}

int launch_engine(bool ta, bool tb, const DeviceBatch& b, const Bases& bases, int* counter,
                  cudaStream_t stream, bool bulk, bool one_body) {
  if (b.ntiles == 0) return SDMRG_OK;
  if (!ta && !tb) launch_t<false, false>(bulk, one_body, b, bases, counter, stream);
  else if (!ta && tb) launch_t<false, true>(bulk, false, b, bases, counter, stream);
  else if (ta && !tb) launch_t<true, false>(bulk, false, b, bases, counter, stream);
  else launch_t<true, true>(bulk, false, b, bases, counter, stream);
  count_launch();
  return cuda_check(cudaGetLastError(), "seg_gemm_kernel launch");
}

// ------------------------------------------------------------- small kernels
__global__ void axpy_kernel(int64_t n, double alpha, const double* __restrict__ x,
                            double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] += alpha * x[i];
}

// c(i, j) *= s over a column-major m x n matrix (general beta of dgemm).
__global__ void scale_cm_kernel(int m, int n, double s, double* c, int ldc) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)m * n;
       e += (int64_t)gridDim.x * blockDim.x)
    c[(e / m) * ldc + (e % m)] *= s;
}

// One-shot launch of a host-built batch (uploads, launches, frees).
// Every operand of the batch 16-byte aligned with even leading dimensions:
// the engine may use 16-byte cp.async (engine.cuh ALIGNED).
static bool batch_aligned(const GemmBatch& gb, const Bases& bases) {
  for (const Seg& sg : gb.segs) {
    const uint64_t a = reinterpret_cast<uint64_t>(bases.p[sg.a >> kHandleShift] + (sg.a & kHandleMask));
    const uint64_t b = reinterpret_cast<uint64_t>(bases.p[sg.b >> kHandleShift] + (sg.b & kHandleMask));
    if ((a & 15) || (b & 15) || (sg.lda & 1) || (sg.ldb & 1)) return false;
  }
  return true;
}

static int run_batch(GemmBatch& gb, bool ta, bool tb, const Bases& bases, cudaStream_t stream) {
  gb.finalize_tiles();
  const bool aligned = batch_aligned(gb, bases);
  DeviceBatch db;
  int rc = gb.upload(&db, stream);
  int* counter = nullptr;
  if (!rc) rc = cuda_check(cudaMalloc(&counter, sizeof(int)), "cudaMalloc counter");
  if (!rc) rc = cuda_check(cudaMemsetAsync(counter, 0, sizeof(int), stream), "memset counter");
  if (!rc) rc = launch_engine(ta, tb, db, bases, counter, stream, aligned);
  if (!rc) rc = cuda_check(cudaStreamSynchronize(stream), "batch sync");
  if (counter) cudaFree(counter);
  db.release();
  return rc;
}

}  // namespace sdmrg

using namespace sdmrg;

extern "C" {

const char* sdmrg_last_error(void) { return g_err.c_str(); }
int sdmrg_version(void) { return 1; }
int64_t sdmrg_launch_count(void) { return g_launches.load(); }

// Column-major C(m x n) = alpha op(A) op(B) + beta C  ->  row-major engine on
// C^T (n x m) = op(B)^T op(A)^T (see engine.cuh TA/TB conventions).
static int dgemm_impl(int transa, int transb, int m, int n, int k, double alpha, const double* a,
                      int lda, const double* b, int ldb, double beta, double* c, int ldc,
                      cudaStream_t stream) {
  if (m < 0 || n < 0 || k < 0) return fail(SDMRG_EINVAL, "dgemm: negative dimension");
  if (m == 0 || n == 0) return SDMRG_OK;
  if (ldc < m) return fail(SDMRG_EINVAL, "dgemm: ldc < m");
  if (beta != 0.0 && beta != 1.0) {
    // general beta: pre-scale C (c := beta*c); rare on this path — the
    // reference only ever passes 0 and 1.
    const int64_t mn = (int64_t)m * n;
    scale_cm_kernel<<<(int)std::min<int64_t>((mn + 255) / 256, 148 * 8), 256, 0, stream>>>(
        m, n, beta, c, ldc);
    count_launch();
    beta = 1.0;
  }
  Bases bases{};
  bases.p[0] = const_cast<double*>(a);
  bases.p[1] = const_cast<double*>(b);
  bases.p[2] = c;
  GemmBatch gb;
  gb.begin_prob(make_handle(2, 0), ldc, n, m, beta != 0.0 ? 1 : 0);
  if (k > 0 && alpha != 0.0) gb.add_seg(make_handle(1, 0), ldb, make_handle(0, 0), lda, k, alpha);
  gb.end_prob();
  // A' = op(B)^T: M-contig iff transb; B' = op(A)^T: K-contig iff transa
  return run_batch(gb, transb != 0, transa != 0, bases, stream);
}

int sdmrg_dgemm(int transa, int transb, int m, int n, int k, double alpha, const double* a,
                int lda, const double* b, int ldb, double beta, double* c, int ldc,
                void* stream) {
  return dgemm_impl(transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc,
                    static_cast<cudaStream_t>(stream));
}

int sdmrg_dgemm_strided_batched(int transa, int transb, int m, int n, int k, const double* a,
                                int lda, int64_t stride_a, const double* b, int ldb,
                                int64_t stride_b, double* c, int ldc, int64_t stride_c,
                                int batch, void* stream) {
  if (m < 0 || n < 0 || k < 0 || batch < 0)
    return fail(SDMRG_EINVAL, "gemm_strided_batched: negative dimension");
  if (m == 0 || n == 0 || batch == 0) return SDMRG_OK;
  Bases bases{};
  bases.p[0] = const_cast<double*>(a);
  bases.p[1] = const_cast<double*>(b);
  bases.p[2] = c;
  GemmBatch gb;
  for (int i = 0; i < batch; ++i) {
    gb.begin_prob(make_handle(2, i * stride_c), ldc, n, m, 0);
    if (k > 0) gb.add_seg(make_handle(1, i * stride_b), ldb, make_handle(0, i * stride_a), lda, k, 1.0);
    gb.end_prob();
  }
  return run_batch(gb, transb != 0, transa != 0, bases, static_cast<cudaStream_t>(stream));
}

int sdmrg_daxpy(int64_t n, double alpha, const double* x, double* y, void* stream) {
  if (n < 0) return fail(SDMRG_EINVAL, "daxpy: negative length");
  if (n == 0) return SDMRG_OK;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  axpy_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(n, alpha, x, y);
  count_launch();
  return cuda_check(cudaGetLastError(), "axpy launch");
}

// Alg. 2 (sbmm4s.py:127-184).  Step 1: batched GEMM with interleaved output
// temp(member i rows [i*m,(i+1)*m), ld m*p) = A @ R_i^T.  Step 2: one
// concatenated GEMM B += alpha * [L_1 .. L_p] @ temp — as segments of one
// problem, so the members' sum is the shared inner dimension.
static int sbmm4s_impl(int m, int n, int q, int r, int p, double alpha, const double* a, int lda,
                       const double* l, int ldl, int64_t sl, const double* rs, int ldr,
                       int64_t sr, double* b, int ldb, double* ws, int64_t wsd, int* kernels,
                       cudaStream_t stream) {
  if ((int64_t)m * r > wsd)
    return fail(SDMRG_EWORKSPACE, "sbmm4s: workspace cannot hold a single member");
  if ((int64_t)m * p * r > wsd && p > 1) {
    const int lo = p / 2;
    int rc = sbmm4s_impl(m, n, q, r, lo, alpha, a, lda, l, ldl, sl, rs, ldr, sr, b, ldb, ws, wsd,
                         kernels, stream);
    if (rc) return rc;
    return sbmm4s_impl(m, n, q, r, p - lo, alpha, a, lda, l + lo * sl, ldl, sl, rs + lo * sr, ldr,
                       sr, b, ldb, ws, wsd, kernels, stream);
  }
  Bases bases{};
  bases.p[0] = const_cast<double*>(a);
  bases.p[1] = const_cast<double*>(rs);
  bases.p[2] = ws;
  bases.p[3] = const_cast<double*>(l);
  bases.p[4] = b;
  // step 1 (column-major temp_i = A R_i^T, m x r, ld m*p, offset i*m) as
  // row-major temp_i^T (r x m) = R_i (r x n, col-major => M-contig) @ A^T
  // (n x m, A col-major => B'(k,j)=a[k*lda+j] N-contig)
  GemmBatch g1;
  for (int i = 0; i < p; ++i) {
    g1.begin_prob(make_handle(2, (int64_t)i * m), m * p, r, m, 0);
    g1.add_seg(make_handle(1, i * sr), ldr, make_handle(0, 0), lda, n, 1.0);
    g1.end_prob();
  }
  int rc = run_batch(g1, true, false, bases, stream);
  if (rc) return rc;
  // step 2: column-major B (q x r) += alpha L_concat (q x m*p) @ temp (m*p x r)
  // row-major B^T (r x q) += temp^T (r x m*p; temp col-major ld m*p => K-contig)
  //                          @ L_concat^T (m*p x q; L col-major => N-contig)
  GemmBatch g2;
  g2.begin_prob(make_handle(4, 0), ldb, r, q, 1);
  for (int i = 0; i < p; ++i)
    g2.add_seg(make_handle(2, (int64_t)i * m), m * p, make_handle(3, i * sl), ldl, m, alpha);
  g2.end_prob();
  rc = run_batch(g2, false, false, bases, stream);
  if (kernels) *kernels += 2;
  return rc;
}

int sdmrg_sbmm4s(int m, int n, int q, int r, int p, double alpha, const double* a, int lda,
                 const double* l_stack, int ldl, int64_t stride_l, const double* r_stack, int ldr,
                 int64_t stride_r, double* b, int ldb, double* workspace,
                 int64_t workspace_doubles, int* kernels_out, void* stream) {
  if (m <= 0 || n <= 0 || q <= 0 || r <= 0 || p <= 0)
    return fail(SDMRG_EINVAL, "sbmm4s: dimensions must be positive");
  if (lda < m || ldl < q || ldr < r || ldb < q)
    return fail(SDMRG_EINVAL, "sbmm4s: leading dimension smaller than rows");
  if (kernels_out) *kernels_out = 0;
  return sbmm4s_impl(m, n, q, r, p, alpha, a, lda, l_stack, ldl, stride_l, r_stack, ldr, stride_r,
                     b, ldb, workspace, workspace_doubles, kernels_out,
                     static_cast<cudaStream_t>(stream));
}

}  // extern "C"
