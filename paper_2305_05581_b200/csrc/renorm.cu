// renorm.cu — renormalization on the same grouped-GEMM engine (north star
// item (5)): the per-operator rotation W^T O W of dmrg.py:254 _transform_tree
// ("no summation over the position index", paper §IV.D) and the reduced
// density matrix accumulation ρ += S S^T of dmrg.py:221 rdm_eigensystem.
#include <algorithm>
#include <map>
#include <vector>

#include "../../include/sdmrg_b200.h"
#include "runtime.h"

using namespace sdmrg;

namespace {

int run(GemmBatch& gb, bool ta, bool tb, const Bases& bases, cudaStream_t stream) {
  if (gb.probs.empty()) return SDMRG_OK;
  gb.finalize_tiles();
  DeviceBatch db;
  int rc = gb.upload(&db, stream);
  int* counter = nullptr;
  if (!rc) rc = cuda_check(cudaMallocAsync(&counter, sizeof(int), stream), "counter alloc");
  if (!rc) rc = cuda_check(cudaMemsetAsync(counter, 0, sizeof(int), stream), "counter memset");
  if (!rc) rc = launch_engine(ta, tb, db, bases, counter, stream);
  if (counter) cudaFreeAsync(counter, stream);
  if (!rc) rc = cuda_check(cudaStreamSynchronize(stream), "renorm sync");
  db.release();
  return rc;
}

}  // namespace

extern "C" {

int sdmrg_rotate(int64_t ntasks, const int64_t* w_l, const int64_t* w_r, const int64_t* o,
                 const int64_t* dst, const int32_t* rows, const int32_t* cols, const int32_t* kl,
                 const int32_t* kr, const double* base_w, const double* base_o, double* base_dst,
                 double* workspace, int64_t workspace_doubles, void* stream_) {
  if (ntasks < 0) return fail(SDMRG_EINVAL, "rotate: negative task count");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  for (int64_t t = 0; t < ntasks; ++t) {
    if (rows[t] < 0 || cols[t] < 0 || kl[t] < 0 || kr[t] < 0)
      return fail(SDMRG_EINVAL, "rotate: negative dimension");
    if ((int64_t)kl[t] * cols[t] > workspace_doubles)
      return fail(SDMRG_EWORKSPACE, "rotate: workspace cannot hold one intermediate");
  }
  Bases bases{};
  bases.p[0] = const_cast<double*>(base_w);
  bases.p[1] = const_cast<double*>(base_o);
  bases.p[2] = base_dst;
  bases.p[3] = workspace;
  int64_t t0 = 0;
  while (t0 < ntasks) {
    GemmBatch ga, gb;
    int64_t ws = 0, t1 = t0;
    for (; t1 < ntasks; ++t1) {
      const int64_t need = (int64_t)kl[t1] * cols[t1];
      if (ws + need > workspace_doubles) break;
      if (kl[t1] == 0 || kr[t1] == 0) continue;
      // tmp (kl x cols) = W_l^T @ O   [W_l rows x kl row-major -> M-contig]
      ga.begin_prob(make_handle(3, ws), cols[t1], kl[t1], cols[t1], 0);
      ga.add_seg(make_handle(0, w_l[t1]), kl[t1], make_handle(1, o[t1]), cols[t1], rows[t1], 1.0);
      ga.end_prob();
      // dst (kl x kr) = tmp @ W_r     [W_r cols x kr row-major]
      gb.begin_prob(make_handle(2, dst[t1]), kr[t1], kl[t1], kr[t1], 0);
      gb.add_seg(make_handle(3, ws), cols[t1], make_handle(0, w_r[t1]), kr[t1], cols[t1], 1.0);
      gb.end_prob();
      ws += need;
    }
    int rc = run(ga, true, false, bases, stream);
    if (!rc) rc = run(gb, false, false, bases, stream);
    if (rc) return rc;
    t0 = t1;
  }
  return SDMRG_OK;
}

int sdmrg_rdm_accumulate(int64_t ntasks, const int64_t* s_off, const int64_t* rho_off,
                         const int32_t* rows, const int32_t* cols, const double* base_s,
                         double* base_rho, void* stream_) {
  if (ntasks < 0) return fail(SDMRG_EINVAL, "rdm: negative task count");
  Bases bases{};
  bases.p[0] = const_cast<double*>(base_s);
  bases.p[1] = base_rho;
  // tasks sharing one ρ block become one problem with ordered segments
  std::map<int64_t, std::vector<int64_t>> by_rho;
  std::vector<int64_t> order;
  for (int64_t t = 0; t < ntasks; ++t) {
    if (rows[t] < 0 || cols[t] < 0) return fail(SDMRG_EINVAL, "rdm: negative dimension");
    if (!by_rho.count(rho_off[t])) order.push_back(rho_off[t]);
    by_rho[rho_off[t]].push_back(t);
  }
  GemmBatch g;
  for (int64_t ro : order) {
    const auto& ts = by_rho[ro];
    const int m = rows[ts[0]];
    for (int64_t t : ts)
      if (rows[t] != m) return fail(SDMRG_EINVAL, "rdm: tasks of one block disagree on rows");
    if (m == 0) continue;
    g.begin_prob(make_handle(1, ro), m, m, m, 1);
    for (int64_t t : ts)
      if (cols[t] > 0) g.add_seg(make_handle(0, s_off[t]), cols[t], make_handle(0, s_off[t]), cols[t], cols[t], 1.0);
    g.end_prob();
  }
  return run(g, false, true, bases, static_cast<cudaStream_t>(stream_));
}

}  // extern "C"
