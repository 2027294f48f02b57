// plan.cu — task generation and execution of H_eff·ψ (blocks.py:503
// build_plan + dmrg.py:107 apply_plan), the north star's items (1)-(3):
//
//  (1) block-sparse layout: operator blocks packed in one device arena per
//      block side with an (op, column sector) -> offset index table; ψ/σ in
//      the reference's to_vector layout (blocks.py:448).
//  (2) task generation: every operator-table row is matched against every ψ
//      sector (the reference's row x ψ-key double loop, blocks.py:521-565),
//      producing the reference's (ψ key, out key) groups with per-member
//      scales — bit-identical grouping, retained on request for parity.
//  (3) the work list for the FP64 engine, in two phases per workspace chunk:
//        phase 1   T(k, R) = A_k R^T           one GEMM per distinct (ψ key,
//                                              right op) — shared by every
//                                              member that uses it
//        phase 0   Lsum = Σ s_t L_t            per (group, right op) with >1
//                                              member (combine.cuh)
//        phase 2   σ[out] += Σ Lsum T          one problem per out key, its K
//                                              the concatenation of products
//      which is SBMM4S (sbmm4s.py Alg. 2) with the interleaved temp stack
//      replaced by deduplicated T blocks and the member sum carried by the
//      shared inner dimension (no reduction pass, no atomics).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <chrono>
#include <vector>

#include "../../include/sdmrg_b200.h"
#include "combine.cuh"
#include "runtime.h"

using namespace sdmrg;

extern "C" int sdmrg_internal_launch_big(const void* tiles, int ntiles, const void* segs,
                                         int* counter, const void* bases, void* stream,
                                         int one_body, int trans_b);
extern "C" int sdmrg_internal_big_grid();

namespace {

// Phase-2 σ blocks that span more than one 64 x 64 tile go to the 128 x 128
// big-tile engine instance (engine_big.cu), whose CTA loads each shared
// row / column operand panel once for all its quadrants.  SDMRG_BIG: 0 off;
// 1 σ blocks of 65..128 x 65..128; 2 (default) also wider / taller blocks
// (max(q, r) > 64, min(q, r) > 32) in <= 128 x 128 tiles (r2o: L=50 D=4096
// 290 / 297 / 311 ms for 2 / 1 / 0).
int big_tiles_mode() {
  const char* e = getenv("SDMRG_BIG");
  return e ? std::atoi(e) : 2;
}
bool big_tiles_enabled() { return big_tiles_mode() > 0; }
inline bool big_problem(int q, int r) {
  const int mode = big_tiles_mode();
  if (mode == 2) return std::max(q, r) > 64 && std::min(q, r) > 32;
  return q > 64 && q <= 128 && r > 64 && r <= 128;
}

// Engine bases.  The engine's bulk-copy producer needs 16-byte aligned
// operand rows, so the plan keeps padded copies of everything it reads
// (even leading dimensions, even element offsets, zero pads): the operator
// arenas (repacked once at build), ψ (copied per apply) and the workspace.
// σ is only written (epilogue) and keeps the reference layout.
enum { B_PSI = 0, B_SIGMA = 1, B_ARENA_L = 2, B_ARENA_R = 3, B_WS = 4, B_PSIT = 5, B_LSUM = 6 };

// Stage-tiled T (phase 2's B operand): T(i, b) (m x r) is stored as column
// tiles of the σ problems' width w = col_tile_width(r), each a contiguous
// [pad16(m)][NC_LD_B] block, so every 16-deep K stage of phase 2 is one
// contiguous run fetched by a single bulk copy.  Identity right ops read ψ in
// the same form (psi_tiled, refilled per apply).
inline int pad16(int x) { return (x + 15) & ~15; }
inline int64_t tiled_size(int m, int r) {
  const int w = GemmBatch::col_tile_width(r);
  return (int64_t)((r + w - 1) / w) * pad16(m) * NC_LD_B;
}

inline int pad2(int x) { return x + (x & 1); }

struct Member {
  int32_t out;
  int32_t row;
  double scale;
};

// One phase-2 product: (group (ψ key, out key), right op) with the member
// left operators pre-summed (combine.cuh).
struct Pair {
  int32_t out, rop;
  int32_t term_begin, term_end;  // into the key's Term list
};
struct Term {
  int32_t lop;
  double coef;
};

// Block copies into a padded layout (row stride change), one CTA per block.
struct PadTask {
  int64_t src, dst;      // element offsets
  int32_t rows, cols;
  int32_t src_ld, dst_ld;
};
__global__ void pad_kernel(const PadTask* __restrict__ tasks, int64_t n,
                           const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
    const PadTask pt = tasks[t];
    const int64_t count = (int64_t)pt.rows * pt.cols;
    for (int64_t e = threadIdx.x; e < count; e += blockDim.x) {
      const int64_t r = e / pt.cols, c = e - r * pt.cols;
      dst[pt.dst + r * pt.dst_ld + c] = src[pt.src + r * pt.src_ld + c];
    }
  }
}
struct PadList {
  PadTask* d_tasks = nullptr;
  int64_t n = 0;
  void release() {
    if (d_tasks) cudaFree(d_tasks);
    d_tasks = nullptr;
    n = 0;
  }
};

// Diagonal of H_eff (the Davidson preconditioner): for every ψ key i, the
// members of its diagonal group (i -> i) contribute s · L_a[x][x] R_b[y][y]
// to element (x, y) of block i.  One CTA per key, members in table order
// (deterministic).  Handles index the plan's padded arenas.
struct DiagKey {
  int64_t off;          // ψ offset of block i (to_vector layout)
  int32_t m, n;         // block i: m x n
  int32_t ldl, ldr;     // padded row strides of its L (m x m) / R (n x n) blocks
  int32_t mem_begin, mem_end;
};
struct DiagMem {
  int64_t l, r;         // element offsets of the L / R blocks in the padded arenas
  double s;
};
__global__ void diag_kernel(const DiagKey* __restrict__ keys, int nkeys,
                            const DiagMem* __restrict__ mems, const double* __restrict__ al,
                            const double* __restrict__ ar, double* __restrict__ diag) {
  for (int k = blockIdx.x; k < nkeys; k += gridDim.x) {
    const DiagKey dk = keys[k];
    const int64_t cnt = (int64_t)dk.m * dk.n;
    for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) {
      const int x = static_cast<int>(e / dk.n), y = static_cast<int>(e - (int64_t)x * dk.n);
      double acc = 0.0;
      for (int t = dk.mem_begin; t < dk.mem_end; ++t) {
        const DiagMem mm = mems[t];
        acc += mm.s * al[mm.l + (int64_t)x * dk.ldl + x] * ar[mm.r + (int64_t)y * dk.ldr + y];
      }
      diag[dk.off + e] = acc;
    }
  }
}

// Host staging + device copy of one combine launch (combine.cuh).
struct CombList {
  std::vector<CombTask> tasks;
  std::vector<CombOut> outs;
  std::vector<CombTerm> terms;
  CombTask* d_tasks = nullptr;
  CombOut* d_outs = nullptr;
  CombTerm* d_terms = nullptr;
  int64_t ntasks = 0;
  // chunk the elements of outputs [first, outs.size()) of n elements each
  void add_tasks(int32_t first, int n) {
    const int32_t last = static_cast<int32_t>(outs.size());
    if (last > first)
      for (int e0 = 0; e0 < n; e0 += COMB_CHUNK)
        tasks.push_back({first, last, e0, std::min(COMB_CHUNK, n - e0)});
  }
  void release() {
    if (d_tasks) cudaFree(d_tasks);
    if (d_outs) cudaFree(d_outs);
    if (d_terms) cudaFree(d_terms);
    d_tasks = nullptr;
    d_outs = nullptr;
    d_terms = nullptr;
  }
};

struct Chunk {
  GemmBatch host1, host2;  // released after upload
  DeviceBatch p1, p2;
  GemmBatch host2big;      // phase 2, σ blocks of 65..128 x 65..128 (engine_big.cu)
  DeviceBatch p2big;
  GemmBatch host1big;      // phase 1, ψ keys of 65..128 rows (engine_big.cu)
  DeviceBatch p1big;
  bool p2big_one_body = false;
  FusedBatch fused;        // small-sector σ problems on the fused kernel (fused.cuh)
  CombList comb0;          // phase 0: pre-summed left operators
  CombList comb3;          // phase 3: split-K partial sums into σ
  int64_t ws_doubles = 0;
  int64_t flops0 = 0, flops1 = 0, flops2 = 0;
  int64_t bytes0 = 0, bytes3 = 0;
  bool p2_one_body = false;  // phase 2 on the single-body engine instance
  cudaEvent_t ev[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
};

}  // namespace

struct sdmrg_plan {
  int ncomp = 0, nsite = 0, nL = 0, nR = 0;
  std::vector<int32_t> keys;     // psi_keys x 4 (jl, s1, s2, jr)
  std::vector<int64_t> offs;     // psi_keys + 1
  // reference grouping (optional)
  std::vector<int32_t> g_psi, g_out;
  std::vector<int64_t> g_begin;
  std::vector<int32_t> m_row;
  std::vector<double> m_scale;
  std::vector<Chunk> chunks;
  double* workspace = nullptr;
  int* counters = nullptr;
  double* arena_l = nullptr;       // padded device copies (owned)
  double* arena_r = nullptr;
  int64_t arena_size[2] = {0, 0};
  std::vector<int64_t> arena_off[2];  // padded (op, column sector) offsets
  double* psi_pad = nullptr;       // padded ψ, refilled by every apply
  std::vector<int64_t> poffs;      // padded ψ block offsets (psi_keys + 1)
  std::vector<char> mine;          // ψ keys of this rank's shard
  PadList psi_copy;                // ψ -> psi_pad block list (device)
  PadList psit_copy;               // ψ -> psi_tiled (stage-tiled ψ, phase 2 B)
  // Pre-summed left operators (phase 0) depend on the operators and the
  // table only — not on ψ — so they live in their own buffer, computed by
  // the first apply after the arenas are final and reused by every later
  // apply of the plan (a Lanczos / Davidson loop)
  double* lsum = nullptr;
  int64_t lsum_doubles = 0;
  bool lsum_ready = false;
  bool lsum_persistent = true;     // false: pre-sums in the chunk workspace, per apply
  double* psi_tiled = nullptr;
  std::vector<int64_t> ptoffs;     // psi_tiled block offsets
  bool tiled = false;
  bool stack_t = false;  // phase 1 per run of arena-adjacent right operators
  // optional (SDMRG_SIDE_STREAM=1): phase 0 (combine) on a low-priority side
  // stream concurrently with phase 1 (it only needs the L arena).  Measured
  // no gain at L=30 D=2048 (99.0 vs 99.4 ms, same box), and it blurs the
  // per-phase timing, so phases run in order on the caller's stream.
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  sdmrg_plan_stats stats{};
  int64_t fused_outs = 0;          // σ problems on the fused kernel
  std::vector<DiagKey> diag_keys;  // H_eff diagonal work (this rank's ψ keys)
  std::vector<DiagMem> diag_mems;
  double shard_balance = 1.0;      // mean / max rank load (world > 1)
  int timing = 0;
};

namespace {

using QN = std::vector<int32_t>;

QN qn_at(const int32_t* base, int i, int ncomp) { return QN(base + (int64_t)i * ncomp, base + (int64_t)(i + 1) * ncomp); }

int validate(const sdmrg_plan_desc* d) {
  if (!d) return fail(SDMRG_EINVAL, "plan: null descriptor");
  if (d->ncomp <= 0 || d->nsite <= 0 || d->nsec_l <= 0 || d->nsec_r <= 0)
    return fail(SDMRG_EINVAL, "plan: empty basis or bad QN width");
  if (d->nrows < 0 || d->nops_l < 0 || d->nops_r < 0) return fail(SDMRG_EINVAL, "plan: negative count");
  if (d->world < 1 || d->rank < 0 || d->rank >= d->world)
    return fail(SDMRG_EINVAL, "plan: bad rank/world");
  for (int64_t t = 0; t < d->nrows; ++t) {
    if (d->lop[t] < 0 || d->lop[t] >= d->nops_l || d->rop[t] < 0 || d->rop[t] >= d->nops_r)
      return fail(SDMRG_EINVAL, "plan: row references a missing operator");
    for (int s = 0; s < d->nsite; ++s) {
      if (d->site1_dst[t * d->nsite + s] >= d->nsite || d->site2_dst[t * d->nsite + s] >= d->nsite)
        return fail(SDMRG_EINVAL, "plan: site map out of range");
    }
  }
  for (int j = 0; j < d->nsec_l; ++j)
    if (d->dim_l[j] <= 0) return fail(SDMRG_EINVAL, "plan: non-positive left sector dim");
  for (int j = 0; j < d->nsec_r; ++j)
    if (d->dim_r[j] <= 0) return fail(SDMRG_EINVAL, "plan: non-positive right sector dim");
  return SDMRG_OK;
}

// shift[o * nsec + j] = index of qn[j] + delta[o] in the basis, or -1
std::vector<int32_t> shift_table(int nops, const int32_t* delta, int nsec, const int32_t* qn,
                                 int ncomp) {
  std::map<QN, int> index;
  for (int j = 0; j < nsec; ++j) index[qn_at(qn, j, ncomp)] = j;
  std::vector<int32_t> out((size_t)nops * nsec, -1);
  std::map<QN, std::vector<int32_t>> memo;
  for (int o = 0; o < nops; ++o) {
    QN dq = qn_at(delta, o, ncomp);
    auto it = memo.find(dq);
    if (it == memo.end()) {
      std::vector<int32_t> row(nsec, -1);
      for (int j = 0; j < nsec; ++j) {
        QN q = qn_at(qn, j, ncomp);
        for (int c = 0; c < ncomp; ++c) q[c] += dq[c];
        auto f = index.find(q);
        if (f != index.end()) row[j] = f->second;
      }
      it = memo.emplace(dq, row).first;
    }
    std::copy(it->second.begin(), it->second.end(), out.begin() + (size_t)o * nsec);
  }
  return out;
}

template <class T>
int upload_vec(const std::vector<T>& v, T** out) {
  *out = nullptr;
  if (v.empty()) return SDMRG_OK;
  int rc = cuda_check(cudaMalloc(out, v.size() * sizeof(T)), "cudaMalloc combine list");
  if (!rc)
    rc = cuda_check(cudaMemcpy(*out, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice),
                    "upload combine list");
  return rc;
}

// Split-K granule = 1/split_factor of one persistent CTA's share of the
// phase-2 work (SDMRG_SPLIT overrides; experiments).
// Phase-2 engine instance: the single-body one when the work is spread over
// many tile shapes (8-row x 8-column block counts) — a wide shape mix is what
// overflows the instruction cache.  Criterion: the three most common shapes
// carry < 40% of the phase-2 work (L=30 D=2048: 53% -> two bodies, 0.3-1.2 ms
// faster; L=50 D=4096: 31% -> one body, 6 ms faster; profiles/r1_notes.md).
// SDMRG_ONE_BODY=0/1 forces it.
bool use_one_body(const GemmBatch& gb) {
  const char* env = getenv("SDMRG_ONE_BODY");
  if (env) return atoi(env) != 0;
  std::vector<double> by_shape(9 * 9, 0.0);
  double all = 0.0;
  for (size_t t = 0; t < gb.tiles.size(); ++t) {
    const int mb = std::min((gb.tiles[t].tm + 7) / 8, 8), nb = std::min((gb.tiles[t].tn + 7) / 8, 8);
    by_shape[mb * 9 + nb] += gb.tile_cost[t];
    all += gb.tile_cost[t];
  }
  std::sort(by_shape.begin(), by_shape.end(), std::greater<double>());
  return all > 0.0 && by_shape[0] + by_shape[1] + by_shape[2] < 0.4 * all;
}
int p2_octaves() {
  static const int v = getenv("SDMRG_P2_OCTAVES") ? atoi(getenv("SDMRG_P2_OCTAVES")) : 0;
  return v;
}
// Floor of the split-K granule (tile cost units: rows x cols x K): parts
// smaller than this cost more in tile start-up, partial-buffer writes and the
// phase-3 sum (a serial chain over the parts per σ element) than their
// balance gains — small-D plans only (D=2048's granule is ~10 M).
double split_min() {
  const char* e = getenv("SDMRG_SPLIT_MIN");
  return e ? std::max(0.0, atof(e)) : 0.0;
}
double split_factor() {
  const char* e = getenv("SDMRG_SPLIT");
  return e ? std::max(1.0, atof(e)) : 96.0;
}

int launch_combine(const CombList& cl, const Bases& bases, cudaStream_t stream,
                   bool latency_bound = false) {
  if (cl.ntasks == 0) return SDMRG_OK;
  if (latency_bound && !getenv("SDMRG_COMB3_U1"))
    combine_kernel<4><<<static_cast<unsigned>(cl.ntasks), COMB_THREADS, 0, stream>>>(
        cl.d_tasks, cl.d_outs, cl.d_terms, bases);
  else
    combine_kernel<1><<<static_cast<unsigned>(cl.ntasks), COMB_THREADS, 0, stream>>>(
        cl.d_tasks, cl.d_outs, cl.d_terms, bases);
  count_launch();
  return cuda_check(cudaGetLastError(), "combine_kernel launch");
}

}  // namespace

extern "C" {

int sdmrg_plan_build(const sdmrg_plan_desc* d, sdmrg_plan** out) {
  if (!out) return fail(SDMRG_EINVAL, "plan: null output");
  *out = nullptr;
  int rc = validate(d);
  if (rc) return rc;
  const int nc = d->ncomp, ns = d->nsite, nL = d->nsec_l, nR = d->nsec_r;
  auto* plan = new sdmrg_plan();
  plan->ncomp = nc;
  plan->nsite = ns;
  plan->nL = nL;
  plan->nR = nR;

  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  auto ms_since = [](clk::time_point t0) {
    return static_cast<int64_t>(
        std::chrono::duration_cast<std::chrono::microseconds>(clk::now() - t0).count() / 1000);
  };
  // ---- ψ keys (blocks.py:416-429): qR = target - qL - q1 - q2 ∈ right basis
  std::map<QN, int> rindex;
  for (int j = 0; j < nR; ++j) rindex[qn_at(d->qn_r, j, nc)] = j;
  struct Key {
    int32_t jl, s1, s2, jr;
  };
  std::vector<Key> keys;
  for (int jl = 0; jl < nL; ++jl)
    for (int s1 = 0; s1 < ns; ++s1)
      for (int s2 = 0; s2 < ns; ++s2) {
        QN q(nc);
        for (int c = 0; c < nc; ++c)
          q[c] = d->target[c] - d->qn_l[jl * nc + c] - d->site_qn[s1 * nc + c] - d->site_qn[s2 * nc + c];
        auto f = rindex.find(q);
        if (f != rindex.end()) keys.push_back({jl, s1, s2, f->second});
      }
  auto key_qns = [&](const Key& k) {
    QN v;
    v.reserve(4 * nc);
    for (int c = 0; c < nc; ++c) v.push_back(d->qn_l[k.jl * nc + c]);
    for (int c = 0; c < nc; ++c) v.push_back(d->site_qn[k.s1 * nc + c]);
    for (int c = 0; c < nc; ++c) v.push_back(d->site_qn[k.s2 * nc + c]);
    for (int c = 0; c < nc; ++c) v.push_back(d->qn_r[k.jr * nc + c]);
    return v;
  };
  std::stable_sort(keys.begin(), keys.end(),
                   [&](const Key& a, const Key& b) { return key_qns(a) < key_qns(b); });
  const int64_t nk = static_cast<int64_t>(keys.size());
  plan->keys.resize(nk * 4);
  plan->offs.resize(nk + 1);
  std::vector<int32_t> psi_index((size_t)nL * ns * ns, -1);
  int64_t off = 0;
  for (int64_t i = 0; i < nk; ++i) {
    const Key& k = keys[i];
    plan->keys[i * 4 + 0] = k.jl;
    plan->keys[i * 4 + 1] = k.s1;
    plan->keys[i * 4 + 2] = k.s2;
    plan->keys[i * 4 + 3] = k.jr;
    plan->offs[i] = off;
    off += (int64_t)d->dim_l[k.jl] * d->dim_r[k.jr];
    psi_index[((size_t)k.jl * ns + k.s1) * ns + k.s2] = static_cast<int32_t>(i);
  }
  plan->offs[nk] = off;
  plan->poffs.resize(nk + 1);
  {
    int64_t po = 0;
    for (int64_t i = 0; i < nk; ++i) {
      plan->poffs[i] = po;
      po += (int64_t)d->dim_l[keys[i].jl] * pad2(d->dim_r[keys[i].jr]);
    }
    plan->poffs[nk] = po;
  }
  plan->tiled = !d->dry_run && getenv("SDMRG_TILED_T") != nullptr;
  plan->ptoffs.assign(nk + 1, 0);
  for (int64_t i = 0; i < nk; ++i)
    plan->ptoffs[i + 1] =
        plan->ptoffs[i] + tiled_size(d->dim_l[keys[i].jl], d->dim_r[keys[i].jr]);
  // padded arena offsets: block (op, column sector j) has rows dim(j + delta),
  // row stride pad2(dim(j)); right-arena blocks also get an even row count
  // (one pad row when dim(j + delta) is odd) so that a run of adjacent right
  // blocks is one matrix whose T = A R^T columns start at even offsets
  // column-sector-major: all operators' blocks of column sector j are one
  // contiguous run of rows with the same row stride pad2(dim(j)) (the R
  // blocks a ψ key's phase 1 reads sit together; fillers see 2-d runs)
  auto pad_offsets = [](int nops, int nsec, const int64_t* boff, const int32_t* shift,
                        const int32_t* dim, bool even_rows, std::vector<int64_t>& out) {
    out.assign((size_t)nops * nsec, -1);
    int64_t pos = 0;
    for (int j = 0; j < nsec; ++j)
      for (int o = 0; o < nops; ++o) {
        const size_t x = (size_t)o * nsec + j;
        if (boff[x] < 0 || shift[x] < 0) continue;
        out[x] = pos;
        pos += (int64_t)(even_rows ? pad2(dim[shift[x]]) : dim[shift[x]]) * pad2(dim[j]);
      }
    return pos;
  };

  const std::vector<int32_t> shL = shift_table(d->nops_l, d->delta_l, nL, d->qn_l, nc);
  const std::vector<int32_t> shR = shift_table(d->nops_r, d->delta_r, nR, d->qn_r, nc);
  plan->stack_t = !plan->tiled && getenv("SDMRG_NO_STACK_T") == nullptr;

  // ---- task generation: members per ψ key, rows in table order
  std::vector<std::vector<Member>> per_key(nk);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < nk; ++i) {
    const Key& k = keys[i];
    std::vector<Member>& mem = per_key[i];
    for (int64_t t = 0; t < d->nrows; ++t) {
      const int d1 = d->site1_dst[t * ns + k.s1];
      if (d1 < 0) continue;
      const int d2 = d->site2_dst[t * ns + k.s2];
      if (d2 < 0) continue;
      const int lo = d->lop[t], ro = d->rop[t];
      const int jlp = shL[(size_t)lo * nL + k.jl];
      if (jlp < 0 || d->blk_off_l[(int64_t)lo * nL + k.jl] < 0) continue;
      const int jrp = shR[(size_t)ro * nR + k.jr];
      if (jrp < 0 || d->blk_off_r[(int64_t)ro * nR + k.jr] < 0) continue;
      const int o = psi_index[((size_t)jlp * ns + d1) * ns + d2];
      if (o < 0 || keys[o].jr != jrp) continue;
      double scale = d->alpha[t] * d->site1_val[t * ns + k.s1] * d->site2_val[t * ns + k.s2];
      if (d->e_l[t]) scale *= d->left_sign[k.jl];
      if (scale == 0.0) continue;
      mem.push_back({o, static_cast<int32_t>(t), scale});
    }
    std::stable_sort(mem.begin(), mem.end(),
                     [](const Member& a, const Member& b) { return a.out < b.out; });
  }

  // ---- phase-2 products: per group, members with the same right operator
  // share T(i, b); their left operators are pre-summed (combine.cuh).  Terms
  // of one (group, rop) are ordered by left op; duplicate left ops sum their
  // scales in member (table-row) order.
  std::vector<std::vector<Pair>> pairs(nk);
  std::vector<std::vector<Term>> terms(nk);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < nk; ++i) {
    const auto& mem = per_key[i];
    std::vector<Pair>& pv = pairs[i];
    std::vector<Term>& tv = terms[i];
    std::vector<int64_t> idx;
    for (size_t a = 0; a < mem.size();) {
      size_t b = a;
      while (b < mem.size() && mem[b].out == mem[a].out) ++b;
      idx.resize(b - a);
      std::iota(idx.begin(), idx.end(), (int64_t)a);
      std::stable_sort(idx.begin(), idx.end(), [&](int64_t x, int64_t y) {
        const int32_t rx = d->rop[mem[x].row], ry = d->rop[mem[y].row];
        if (rx != ry) return rx < ry;
        return d->lop[mem[x].row] < d->lop[mem[y].row];
      });
      for (size_t u = 0; u < idx.size();) {
        const int32_t ro = d->rop[mem[idx[u]].row];
        Pair p{mem[a].out, ro, static_cast<int32_t>(tv.size()), 0};
        size_t v = u;
        while (v < idx.size() && d->rop[mem[idx[v]].row] == ro) {
          const int32_t lo = d->lop[mem[idx[v]].row];
          double coef = 0.0;
          while (v < idx.size() && d->rop[mem[idx[v]].row] == ro && d->lop[mem[idx[v]].row] == lo)
            coef += mem[idx[v++]].scale;
          if (coef != 0.0) tv.push_back({lo, coef});
        }
        p.term_end = static_cast<int32_t>(tv.size());
        if (p.term_end > p.term_begin) pv.push_back(p);
        u = v;
      }
      a = b;
    }
  }

  // ---- statistics in the reference's FLOP convention (sbmm4s.py:205)
  int64_t groups = 0, members = 0, ref_flops = 0;
  std::vector<double> key_cost(nk, 0.0);
  for (int64_t i = 0; i < nk; ++i) {
    const auto& mem = per_key[i];
    const int64_t m = d->dim_l[keys[i].jl], n = d->dim_r[keys[i].jr];
    members += (int64_t)mem.size();
    for (size_t a = 0; a < mem.size();) {
      size_t b = a;
      while (b < mem.size() && mem[b].out == mem[a].out) ++b;
      const int64_t p = (int64_t)(b - a);
      const int64_t q = d->dim_l[keys[mem[a].out].jl], r = d->dim_r[keys[mem[a].out].jr];
      ref_flops += 2 * m * r * n * p + 2 * q * r * m * p;
      ++groups;
      a = b;
    }
    // sharding cost: the executed FLOPs of this key — phase-2 products plus
    // its distinct non-identity T = A R^T (phase 1)
    std::vector<int32_t> rops;
    for (const Pair& p : pairs[i]) {
      key_cost[i] += 2.0 * d->dim_l[keys[p.out].jl] * d->dim_r[keys[p.out].jr] * m;
      if (d->kind_r[p.rop] != 1) rops.push_back(p.rop);
    }
    std::sort(rops.begin(), rops.end());
    rops.erase(std::unique(rops.begin(), rops.end()), rops.end());
    for (int32_t ro : rops) {
      const int jrp = shR[(size_t)ro * nR + keys[i].jr];
      if (jrp >= 0) key_cost[i] += 2.0 * m * n * d->dim_r[jrp];
    }
  }
  if (d->keep_groups) {
    plan->g_begin.push_back(0);
    for (int64_t i = 0; i < nk; ++i) {
      const auto& mem = per_key[i];
      for (size_t a = 0; a < mem.size();) {
        size_t b = a;
        while (b < mem.size() && mem[b].out == mem[a].out) ++b;
        plan->g_psi.push_back(static_cast<int32_t>(i));
        plan->g_out.push_back(mem[a].out);
        for (size_t c = a; c < b; ++c) {
          plan->m_row.push_back(mem[c].row);
          plan->m_scale.push_back(mem[c].scale);
        }
        plan->g_begin.push_back(static_cast<int64_t>(plan->m_row.size()));
        a = b;
      }
    }
  }

  // ---- shard ψ keys over ranks (greedy LPT on executed cost, deterministic).
  // Default: whole left column sectors (every ψ key with the same left
  // sector) go to one rank, so a rank reads — and holds — only the left
  // operator blocks of its own sectors and the right blocks they pair with:
  // operator memory scales with the rank count.  SDMRG_SHARD=key deals single
  // ψ keys instead (finest balance, every rank touches nearly every block).
  std::vector<char> mine(nk, 1);
  if (d->world > 1) {
    const char* sm = getenv("SDMRG_SHARD");
    const bool by_key = sm && std::strcmp(sm, "key") == 0;
    // units: whole left sectors, except a sector heavier than half a rank's
    // share, whose ψ keys are dealt singly (one central sector can exceed
    // 1/8 of the work at L=30 D=2048)
    std::vector<double> jcost(nL, 0.0);
    double tot = 0.0;
    for (int64_t i = 0; i < nk; ++i) {
      jcost[keys[i].jl] += key_cost[i] + 1.0;
      tot += key_cost[i] + 1.0;
    }
    std::vector<int64_t> unit_of(nk);
    std::vector<double> ucost;
    std::vector<int64_t> jl_unit(nL, -1);
    for (int64_t i = 0; i < nk; ++i) {
      const int jl = keys[i].jl;
      if (by_key || jcost[jl] > tot / (2.0 * d->world)) {
        unit_of[i] = static_cast<int64_t>(ucost.size());
        ucost.push_back(key_cost[i] + 1.0);
      } else {
        if (jl_unit[jl] < 0) {
          jl_unit[jl] = static_cast<int64_t>(ucost.size());
          ucost.push_back(0.0);
        }
        unit_of[i] = jl_unit[jl];
        ucost[jl_unit[jl]] += key_cost[i] + 1.0;
      }
    }
    const int64_t nunit = static_cast<int64_t>(ucost.size());
    std::vector<int64_t> order(nunit);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return ucost[a] > ucost[b]; });
    std::vector<double> load(d->world, 0.0);
    std::vector<int> owner(nunit, 0);
    for (int64_t u : order) {
      int best = 0;
      for (int w = 1; w < d->world; ++w)
        if (load[w] < load[best]) best = w;
      load[best] += ucost[u];
      owner[u] = best;
    }
    for (int64_t i = 0; i < nk; ++i) mine[i] = owner[unit_of[i]] == d->rank;
    double mx = 0.0;
    for (double x : load) mx = std::max(mx, x);
    plan->shard_balance = mx > 0.0 ? tot / (d->world * mx) : 1.0;
  }

  plan->mine = mine;

  // ---- padded arenas: the blocks this rank's ψ keys read (all of them at
  // world 1), column-sector-major
  std::vector<int64_t> poff_l, poff_r;
  int64_t psize_l, psize_r;
  {
    std::vector<int64_t> use_l((size_t)d->nops_l * nL, -1), use_r((size_t)d->nops_r * nR, -1);
    for (int64_t i = 0; i < nk; ++i) {
      if (!mine[i]) continue;
      for (const Pair& p : pairs[i]) {
        const size_t xr = (size_t)p.rop * nR + keys[i].jr;
        use_r[xr] = d->blk_off_r[xr];
        for (int32_t t = p.term_begin; t < p.term_end; ++t) {
          const size_t xl = (size_t)terms[i][t].lop * nL + keys[i].jl;
          use_l[xl] = d->blk_off_l[xl];
        }
      }
    }
    psize_l = pad_offsets(d->nops_l, nL, use_l.data(), shL.data(), d->dim_l, false, poff_l);
    psize_r = pad_offsets(d->nops_r, nR, use_r.data(), shR.data(), d->dim_r, true, poff_r);
  }
  // diagonal-group members of this rank's ψ keys (sdmrg_plan_diagonal)
  for (int64_t i = 0; i < nk; ++i) {
    if (!mine[i]) continue;
    const int m = d->dim_l[keys[i].jl], n = d->dim_r[keys[i].jr];
    DiagKey dk{plan->offs[i], m, n, pad2(m), pad2(n), static_cast<int32_t>(plan->diag_mems.size()), 0};
    for (const Member& mb : per_key[i]) {
      if (mb.out != i) continue;
      const size_t xl = (size_t)d->lop[mb.row] * nL + keys[i].jl;
      const size_t xr = (size_t)d->rop[mb.row] * nR + keys[i].jr;
      if (poff_l[xl] < 0 || poff_r[xr] < 0) continue;
      plan->diag_mems.push_back({poff_l[xl], poff_r[xr], mb.scale});
    }
    dk.mem_end = static_cast<int32_t>(plan->diag_mems.size());
    if (dk.mem_end > dk.mem_begin) plan->diag_keys.push_back(dk);
  }

  // ---- fused small-sector σ problems (fused.cuh): an out key whose rows q
  // and every contributing ψ key's rows m are <= 64 is evaluated by the fused
  // kernel (T = ψ R^T chained in registers, never stored); the others by the
  // two-phase engine.  SDMRG_FUSED=1 turns the fused path on.
  std::vector<char> fuse_out(nk, 0);
  {
    // off by default: on one B200 the fused kernel is still slower than the
    // two-phase engine (L=76 D=4096: 393-400 vs 238-249 ms, profiles/r2_notes.md)
    const char* fe = getenv("SDMRG_FUSED");
    const bool allow = fe && fe[0] == '1';
    if (allow) {
      std::vector<int> maxm(nk, 0);
      for (int64_t i = 0; i < nk; ++i) {
        if (!mine[i]) continue;
        for (const Pair& p : pairs[i])
          maxm[p.out] = std::max(maxm[p.out], (int)d->dim_l[keys[i].jl]);
      }
      for (int64_t o = 0; o < nk; ++o)
        fuse_out[o] = maxm[o] > 0 && maxm[o] <= 8 * F_MB && d->dim_l[keys[o].jl] <= 8 * F_QB;
    }
  }
  plan->fused_outs = 0;
  for (int64_t o = 0; o < nk; ++o) plan->fused_outs += fuse_out[o];

  // ---- execution schedule: chunks of ψ keys bounded by the workspace
  // (distinct non-identity T blocks of two-phase products + pre-summed left
  // operators per key)
  std::vector<int64_t> t_need(nk, 0), l_need(nk, 0);
  for (int64_t i = 0; i < nk; ++i) {
    if (!mine[i]) continue;
    const int64_t m = d->dim_l[keys[i].jl];
    std::vector<int32_t> rops;
    for (const Pair& p : pairs[i]) {
      if (!fuse_out[p.out]) rops.push_back(p.rop);
      if (p.term_end - p.term_begin > 1) l_need[i] += (int64_t)d->dim_l[keys[p.out].jl] * pad2(m);
    }
    std::sort(rops.begin(), rops.end());
    rops.erase(std::unique(rops.begin(), rops.end()), rops.end());
    for (int32_t ro : rops) {
      if (d->kind_r[ro] == 1) continue;
      const int jrp = shR[(size_t)ro * nR + keys[i].jr];
      t_need[i] += plan->tiled ? tiled_size((int)m, d->dim_r[jrp]) : m * pad2(d->dim_r[jrp]);
    }
  }
  // Pre-sums persist across applies (formed once) when they take at most a
  // quarter of free HBM; otherwise they live in the chunk workspace and are
  // re-formed by every apply (large D), as the workspace is reused per chunk.
  int64_t total_l = 0;
  for (int64_t i = 0; i < nk; ++i) total_l += l_need[i];
  size_t free_b = 0, total_b = 0;
  if (!d->dry_run) cudaMemGetInfo(&free_b, &total_b);
  plan->lsum_persistent =
      !d->dry_run && (double)total_l * 8.0 <= 0.25 * (double)free_b && !getenv("SDMRG_LSUM_PER_APPLY");
  if (!plan->lsum_persistent)
    for (int64_t i = 0; i < nk; ++i) t_need[i] += l_need[i];
  int64_t total_t = 0;
  for (int64_t i = 0; i < nk; ++i) total_t += t_need[i];
  int64_t budget = d->workspace_doubles;
  if (budget <= 0 && !d->dry_run) {
    // what the plan allocates besides the workspace: padded arenas (unless
    // the caller already holds them: empty_arenas), padded ψ, pre-sums
    const double own = 8.0 * ((double)psize_l + (double)psize_r + (double)plan->poffs[nk] +
                              (plan->tiled ? (double)plan->ptoffs[nk] : 0.0));
    const double avail = std::max(0.0, (double)free_b - own -
                                  (plan->lsum_persistent ? 8.0 * total_l : 0.0));
    budget = std::max<int64_t>(1 << 20, (int64_t)(avail / 8 * 0.30));
  }
  int64_t max_key = 0;
  for (int64_t i = 0; i < nk; ++i) max_key = std::max(max_key, t_need[i]);
  budget = std::max(budget, max_key);
  budget = std::min(budget, std::max<int64_t>(total_t, 1));

  int64_t exec_flops = 0, local_members = 0, t_problems = 0, tiles = 0, segments = 0;
  int64_t products = 0, comb_outputs = 0, comb_terms = 0;
  double algo_bytes = 16.0 * off;
  {
    // unique operator blocks touched (compulsory reads)
    std::vector<char> seen_l((size_t)d->nops_l * nL, 0), seen_r((size_t)d->nops_r * nR, 0);
    for (int64_t i = 0; i < nk; ++i) {
      if (!mine[i]) continue;
      local_members += (int64_t)per_key[i].size();
      for (const Member& mb : per_key[i]) {
        const int lo = d->lop[mb.row], ro = d->rop[mb.row];
        char& sl = seen_l[(size_t)lo * nL + keys[i].jl];
        if (!sl) {
          sl = 1;
          algo_bytes += 8.0 * d->dim_l[keys[i].jl] * d->dim_l[shL[(size_t)lo * nL + keys[i].jl]];
        }
        char& sr = seen_r[(size_t)ro * nR + keys[i].jr];
        if (!sr) {
          sr = 1;
          algo_bytes += 8.0 * d->dim_r[keys[i].jr] * d->dim_r[shR[(size_t)ro * nR + keys[i].jr]];
        }
      }
    }
  }

  const int64_t taskgen_ms = ms_since(t_start);
  const auto t_emit = clk::now();
  int64_t lsum_pos = 0;  // running offset in the persistent lsum buffer
  int64_t i0 = d->dry_run ? nk : 0;  // dry run: task generation + stats only
  while (i0 < nk) {
    Chunk ch;
    int64_t used = 0, i1 = i0;
    while (i1 < nk && (i1 == i0 || used + t_need[i1] <= budget)) {
      used += t_need[i1];
      ++i1;
    }
    // phase 1: distinct T per (key, right op); tmap[i - i0] holds the key's
    // right ops sorted, with the handle / leading dimension of their T
    struct TEntry {
      int32_t rop;
      int32_t ld;
      uint64_t handle;
      int32_t btile;  // > 0: stage-tiled T (phase 2 B operand)
      int32_t run;    // > 0: first of `run` arena-adjacent right ops (one product)
    };
    std::vector<std::vector<TEntry>> tmap(i1 - i0);
    auto t_lookup = [&](int64_t i, int32_t ro) -> const TEntry& {
      const auto& v = tmap[i - i0];
      return *std::lower_bound(v.begin(), v.end(), ro,
                               [](const TEntry& e, int32_t x) { return e.rop < x; });
    };
    // parallel over keys: per-key T tables and problem lists, workspace
    // offsets from a prefix sum, merged in key order (deterministic)
    const int64_t nkc = i1 - i0;
    std::vector<int64_t> ws_key(nkc + 1, 0);
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t i = i0; i < i1; ++i) {
      if (!mine[i]) continue;
      const Key& k = keys[i];
      const int m = d->dim_l[k.jl], n = d->dim_r[k.jr];
      auto& tm = tmap[i - i0];
      std::vector<int32_t> rops;
      rops.reserve(pairs[i].size());
      for (const Pair& pr : pairs[i])
        if (!fuse_out[pr.out]) rops.push_back(pr.rop);
      std::sort(rops.begin(), rops.end());
      rops.erase(std::unique(rops.begin(), rops.end()), rops.end());
      tm.reserve(rops.size());
      int64_t need = 0;
      for (const int32_t ro : rops) {
        if (d->kind_r[ro] == 1) {  // R = identity: T = A (no product)
          if (plan->tiled)
            tm.push_back({ro, NC_LD_B, make_handle(B_PSIT, plan->ptoffs[i]), pad16(m), 0});
          else
            tm.push_back({ro, pad2(n), make_handle(B_PSI, plan->poffs[i]), 0, 0});
          continue;
        }
        const int r = d->dim_r[shR[(size_t)ro * nR + k.jr]];
        if (plan->tiled) {
          tm.push_back({ro, NC_LD_B, make_handle(B_WS, need), pad16(m), 1});  // rebased below
          need += tiled_size(m, r);
        } else {
          tm.push_back({ro, pad2(r), make_handle(B_WS, need), 0, 1});  // relative; rebased below
          need += (int64_t)m * pad2(r);
        }
      }
      // Right ops whose arena blocks are adjacent (column-sector-major arena,
      // even row counts) form one stacked matrix [R_b1; R_b2; ...] with row
      // stride pad2(n): T for the whole run is ONE m x sum(pad2(r_b)) product
      // with T(i, b) its column block (ld = the run width).  Fewer, fuller
      // 64 x 64 tiles than one product per operator (L=30 D=2048: 2.62 M ->
      // 1.63 M phase-1 tiles, tools/stack_stats.py).  Same workspace size.
      if (plan->stack_t) {
        int64_t pos = 0;  // relative workspace position of the run being formed
        for (size_t u = 0; u < tm.size();) {
          if (d->kind_r[tm[u].rop] == 1) { ++u; continue; }
          size_t v = u + 1;
          int64_t end = poff_r[(size_t)tm[u].rop * nR + k.jr] + (int64_t)tm[u].ld * pad2(n);
          int width = tm[u].ld;
          while (v < tm.size() && d->kind_r[tm[v].rop] != 1 &&
                 poff_r[(size_t)tm[v].rop * nR + k.jr] == end) {
            end += (int64_t)tm[v].ld * pad2(n);
            width += tm[v].ld;
            ++v;
          }
          int col = 0;
          for (size_t x = u; x < v; ++x) {
            const int w = tm[x].ld;
            tm[x].handle = make_handle(B_WS, pos + col);
            tm[x].ld = width;
            tm[x].run = x == u ? static_cast<int32_t>(v - u) : 0;
            col += w;
          }
          pos += (int64_t)m * width;
          u = v;
        }
      }
      ws_key[i - i0 + 1] = need;
    }
    for (int64_t x = 0; x < nkc; ++x) ws_key[x + 1] += ws_key[x];
    std::vector<GemmBatch> p1key(nkc);
    // phase-1 products of ψ keys with 65..128 rows on the big-tile instance
    // (row siblings share the right-operator panel; SDMRG_BIG_P1=0: off)
    // SDMRG_BIG_P1: 0 off, 1 (default) m in 65..128, 2 every m > 64 (rows
    // cut into <= 128-row tiles)
    const char* bp1 = getenv("SDMRG_BIG_P1");
    const int big1 = big_tiles_enabled() ? (bp1 ? std::atoi(bp1) : 1) : 0;
    if (big1 > 0)
      for (int64_t i = i0; i < i1; ++i) {
        const int m = d->dim_l[keys[i].jl];
        if (m > 64 && (m <= 128 || big1 == 2)) p1key[i - i0].cap = 128;
      }
    int64_t f1 = 0, np1 = 0;
#pragma omp parallel for schedule(dynamic, 8) reduction(+ : f1, np1)
    for (int64_t i = i0; i < i1; ++i) {
      if (!mine[i]) continue;
      const Key& k = keys[i];
      const int m = d->dim_l[k.jl], n = d->dim_r[k.jr];
      GemmBatch& gb = p1key[i - i0];
      auto& tv = tmap[i - i0];
      for (size_t x = 0; x < tv.size(); ++x) {
        TEntry& te = tv[x];
        if (d->kind_r[te.rop] == 1) continue;
        const int64_t base = ws_key[i - i0] + (int64_t)(te.handle & kHandleMask);
        te.handle = make_handle(B_WS, base);
        const int r = d->dim_r[shR[(size_t)te.rop * nR + k.jr]];
        const uint64_t rblk = make_handle(B_ARENA_R, poff_r[(size_t)te.rop * nR + k.jr]);
        f1 += 2LL * m * n * r;
        ++np1;
        if (te.run == 0) continue;  // inside a stacked run: formed by its first op
        if (plan->stack_t) {
          // te.ld = run width: T(run) = A [R_b ...]^T, m x width
          gb.begin_prob(te.handle, te.ld, m, te.ld, 0);
          gb.add_seg(make_handle(B_PSI, plan->poffs[i]), pad2(n), rblk, pad2(n), n, 1.0);
          gb.end_prob();
        } else if (te.btile > 0) {
          // one problem per column tile of T, written as its [pad16(m)][NC_LD_B] block
          const int w = GemmBatch::col_tile_width(r);
          for (int c0 = 0, ct = 0; c0 < r; c0 += w, ++ct) {
            gb.begin_prob(make_handle(B_WS, base + (int64_t)ct * te.btile * NC_LD_B), NC_LD_B, m,
                          std::min(w, r - c0), 0);
            gb.add_seg(make_handle(B_PSI, plan->poffs[i]), pad2(n),
                       rblk + (uint64_t)((int64_t)c0 * pad2(n)), pad2(n), n, 1.0);
            gb.end_prob();
          }
        } else {
          gb.begin_prob(te.handle, pad2(r), m, r, 0);
          gb.add_seg(make_handle(B_PSI, plan->poffs[i]), pad2(n), rblk, pad2(n), n, 1.0);
          gb.end_prob();
        }
      }
    }
    ch.host1big.cap = 128;
    for (auto& gb : p1key) {
      if (gb.cap == 128) ch.host1big.append(std::move(gb));
      else ch.host1.append(std::move(gb));
    }
    p1key.clear();
    int64_t ws = ws_key[nkc];
    exec_flops += f1;
    ch.flops1 += f1;
    t_problems += np1;
    // phase 0 + 2: one σ problem per out key; one segment per (ψ key, right
    // op) product, ordered (ψ key, rop); multi-term left sums staged by the
    // combine kernel into the workspace after the T blocks
    std::vector<std::vector<std::pair<int64_t, const Pair*>>> by_out_v(nk);
    for (int64_t i = i0; i < i1; ++i) {
      if (!mine[i]) continue;
      for (const Pair& pr : pairs[i]) by_out_v[pr.out].push_back({i, &pr});
    }
    std::vector<std::pair<int32_t, std::vector<std::pair<int64_t, const Pair*>>*>> by_out;
    for (int64_t o = 0; o < nk; ++o)
      if (!by_out_v[o].empty()) by_out.push_back({static_cast<int32_t>(o), &by_out_v[o]});
    struct OutProb {
      int32_t o;
      int q, r;
      int64_t ksum;
      std::vector<Seg> segs;
      std::vector<FSeg> fsegs;  // fused σ problems: one product per entry
      double fcost = 0.0;       // fused: DMMA work units of the whole problem
    };
    std::vector<OutProb> outs;
    outs.reserve(by_out.size());
    for (auto& kvp : by_out) {
      const int32_t o = kvp.first;
      const bool fz = fuse_out[o] != 0;
      const auto& entries = *kvp.second;
      const int q = d->dim_l[keys[o].jl], r = d->dim_r[keys[o].jr];
      OutProb op{o, q, r, 0, {}, {}, 0.0};
      for (size_t u = 0; u < entries.size();) {
        const int64_t i = entries[u].first;
        const int m = d->dim_l[keys[i].jl];
        const int n = d->dim_r[keys[i].jr];
        const int qm = q * pad2(m);  // a padded q x m block, pads included
        const int32_t out_first = static_cast<int32_t>(ch.comb0.outs.size());
        for (; u < entries.size() && entries[u].first == i; ++u) {
          const Pair& pr = *entries[u].second;
          const Term* tt = terms[i].data();
          uint64_t ahandle;
          double ascale;
          if (pr.term_end - pr.term_begin == 1) {
            const Term& t = tt[pr.term_begin];
            ahandle = make_handle(B_ARENA_L, poff_l[(size_t)t.lop * nL + keys[i].jl]);
            ascale = t.coef;
          } else {
            const uint64_t lh = plan->lsum_persistent ? make_handle(B_LSUM, lsum_pos)
                                                      : make_handle(B_WS, ws);
            CombOut co{lh, static_cast<int32_t>(ch.comb0.terms.size()), 0};
            for (int32_t x = pr.term_begin; x < pr.term_end; ++x)
              ch.comb0.terms.push_back(
                  {make_handle(B_ARENA_L, poff_l[(size_t)tt[x].lop * nL + keys[i].jl]),
                   tt[x].coef});
            co.term_end = static_cast<int32_t>(ch.comb0.terms.size());
            ch.comb0.outs.push_back(co);
            ahandle = lh;
            ascale = 1.0;
            if (plan->lsum_persistent) lsum_pos += qm;
            else ws += qm;
            ch.flops0 += 2LL * (co.term_end - co.term_begin) * qm;
            ch.bytes0 += 8LL * (co.term_end - co.term_begin + 1) * qm;
            ++comb_outputs;
            comb_terms += co.term_end - co.term_begin;
          }
          if (fz) {
            // fused product: T(i, b) = ψ_i R_b^T formed in registers per use
            FSeg fs{};
            fs.psi = make_handle(B_PSI, plan->poffs[i]);
            fs.ident = d->kind_r[pr.rop] == 1;
            fs.rb = fs.ident ? 0 : make_handle(B_ARENA_R, poff_r[(size_t)pr.rop * nR + keys[i].jr]);
            fs.l = ahandle;
            fs.m = m;
            fs.n = n;
            fs.scale = ascale;
            op.fsegs.push_back(fs);
            const int64_t f1 = fs.ident ? 0 : 2LL * m * n * r;
            exec_flops += f1 + 2LL * q * r * m;
            ch.flops2 += f1 + 2LL * q * r * m;
            op.fcost += double((m + 7) / 8 * 8) * r * ((fs.ident ? 0 : (n + 3) / 4 * 4) + 2.0 * q);
            op.ksum += m;
          } else {
            const TEntry& th = t_lookup(i, pr.rop);
            Seg sg{};
            sg.b = th.handle;
            sg.ldb = th.ld;
            sg.btile = th.btile;
            sg.lda = pad2(m);
            sg.k = m;
            sg.a = ahandle;
            sg.scale = ascale;
            op.segs.push_back(sg);
            op.ksum += m;
            exec_flops += 2LL * q * r * m;
            ch.flops2 += 2LL * q * r * m;
          }
          ++products;
        }
        ch.comb0.add_tasks(out_first, qm);
      }
      outs.push_back(std::move(op));
    }
    if (p2_octaves() > 0)  // σ blocks sharing T(i, b) share the right sector
      std::stable_sort(outs.begin(), outs.end(), [&](const OutProb& a, const OutProb& b) {
        return keys[a.o].jr < keys[b.o].jr;
      });
    // split-K for load balance: a σ tile whose K work exceeds the granule
    // (1/96 of one persistent CTA's share: short tiles keep sibling tiles of one
    // σ block in step, so their shared operand panels hit in L2 — 1/6 was 5%
    // slower in phase 2) is cut into contiguous segment
    // ranges written to partial buffers; phase 3 adds them to σ in order
    // (σ first, then parts 0..S-1: deterministic, no atomics).  Fused σ
    // problems use the same rule against the fused kernel's grid.
    auto tiles_of = [](int extent) { return (extent + BM - 1) / BM; };
    const bool big_on = big_tiles_enabled();
    double total_cost = 0.0, total_fcost = 0.0, total_bcost = 0.0;
    for (const OutProb& op : outs) {
      if (!op.fsegs.empty()) total_fcost += op.fcost;
      else if (big_on && big_problem(op.q, op.r)) total_bcost += double(op.q) * op.r * op.ksum;
      else total_cost += double(op.q) * op.r * op.ksum;
    }
    // small-sector plans (every σ block one 64-tile: CAS(113,76) D=4096)
    // balance better with a granule of 1/192 of a CTA's share (r2z: phase 2
    // 137 vs 145 ms there; multi-tile plans keep 1/96)
    bool all_small = true;
    for (const OutProb& op : outs)
      if (op.q > 64 || op.r > 64) {
        all_small = false;
        break;
      }
    const double sf = (all_small && !getenv("SDMRG_SPLIT")) ? 2.0 * split_factor() : split_factor();
    const double granule = std::max(
        total_cost / (double(d->dry_run ? 1 : engine_grid(false, false)) * sf) + 1.0,
        split_min());
    // big tiles: one CTA per SM, a granule per SDMRG_BIG_SPLIT (default as
    // the 64-tile instance) of its share
    const char* bse = getenv("SDMRG_BIG_SPLIT");
    const double bsplit = bse ? std::max(1.0, std::atof(bse)) : split_factor();
    const double bgranule = std::max(
        total_bcost / (double(d->dry_run ? 148 : sdmrg_internal_big_grid()) * bsplit) + 1.0,
        split_min());
    ch.host2big.cap = 128;
    const double fgranule =
        total_fcost / (double(d->dry_run ? 148 : fused_grid_size()) * split_factor()) + 1.0;
    for (const OutProb& op : outs) {
      const bool fz = !op.fsegs.empty();
      const bool bg = !fz && big_on && big_problem(op.q, op.r);
      GemmBatch& h2 = bg ? ch.host2big : ch.host2;
      const size_t nseg = fz ? op.fsegs.size() : op.segs.size();
      double tile_cost;
      if (bg) {
        tile_cost = double(op.q) * op.r * op.ksum;
      } else if (fz) {
        const int rb = (op.r + 7) / 8;
        tile_cost = op.fcost * std::min(rb, F_RT) / rb;  // the widest column tile's share
      } else {
        tile_cost = double(op.q) / tiles_of(op.q) * (double(op.r) / tiles_of(op.r)) * op.ksum;
      }
      int nsplit = static_cast<int>(std::min<double>(
          std::ceil(tile_cost / (fz ? fgranule : (bg ? bgranule : granule))), double(nseg)));
      nsplit = std::max(nsplit, 1);
      const uint64_t sig = make_handle(B_SIGMA, plan->offs[op.o]);
      auto emit = [&](uint64_t c, int beta, size_t s0, size_t s1) {
        if (fz) {
          const int32_t fb = static_cast<int32_t>(ch.fused.segs.size());
          ch.fused.segs.insert(ch.fused.segs.end(), op.fsegs.begin() + s0, op.fsegs.begin() + s1);
          ch.fused.add_problem(c, op.r, op.q, op.r, beta, fb);
        } else {
          h2.begin_prob(c, op.r, op.q, op.r, beta);
          for (size_t x = s0; x < s1; ++x) {
            const Seg& sg = op.segs[x];
            h2.add_seg(sg.a, sg.lda, sg.b, sg.ldb, sg.k, sg.scale, sg.btile);
          }
          h2.end_prob();
        }
      };
      auto seg_k = [&](size_t x) { return fz ? op.fsegs[x].m : op.segs[x].k; };
      if (nsplit == 1) {
        emit(sig, 1, 0, nseg);
        continue;
      }
      const int64_t qr = (int64_t)op.q * op.r;
      const int32_t out_first = static_cast<int32_t>(ch.comb3.outs.size());
      CombOut co{sig, static_cast<int32_t>(ch.comb3.terms.size()), 0};
      ch.comb3.terms.push_back({sig, 1.0});
      size_t u = 0;
      int64_t kdone = 0;
      for (int sp = 0; sp < nsplit && u < nseg; ++sp) {
        const int64_t kcut = op.ksum * (sp + 1) / nsplit;
        const uint64_t part = make_handle(B_WS, ws);
        const size_t u0 = u;
        do {
          kdone += seg_k(u++);
        } while (u < nseg && (kdone < kcut || sp == nsplit - 1));
        emit(part, 0, u0, u);
        ch.comb3.terms.push_back({part, 1.0});
        ws += qr + (qr & 1);
      }
      co.term_end = static_cast<int32_t>(ch.comb3.terms.size());
      ch.comb3.outs.push_back(co);
      ch.comb3.add_tasks(out_first, static_cast<int>(qr));
      ch.bytes3 += 8LL * (co.term_end - co.term_begin + 1) * qr;
    }
    ch.host1.finalize_tiles(0, getenv("SDMRG_P1_BY_PROBLEM") != nullptr);
    ch.host1big.finalize_tiles(0, false);
    tiles += (int64_t)ch.host1big.tiles.size();
    segments += (int64_t)ch.host1big.segs.size();
    ch.host2.finalize_tiles(p2_octaves(), getenv("SDMRG_P2_BY_PROBLEM") != nullptr);
    ch.p2_one_body = use_one_body(ch.host2);
    ch.host2big.finalize_tiles(0, false);
    ch.p2big_one_body = use_one_body(ch.host2big);
    tiles += (int64_t)ch.host2big.tiles.size();
    segments += (int64_t)ch.host2big.segs.size();
    ch.fused.finalize();
    tiles += (int64_t)ch.fused.tiles.size();
    segments += (int64_t)ch.fused.segs.size();
    ch.ws_doubles = ws;
    tiles += (int64_t)(ch.host1.tiles.size() + ch.host2.tiles.size());
    segments += (int64_t)(ch.host1.segs.size() + ch.host2.segs.size());
    plan->chunks.push_back(std::move(ch));
    i0 = i1;
  }

  plan->lsum_doubles = lsum_pos;
  const int64_t emit_ms = ms_since(t_emit);
  const auto t_dev = clk::now();
  int64_t ws_max = 0;
  for (auto& ch : plan->chunks) ws_max = std::max(ws_max, ch.ws_doubles);
  rc = SDMRG_OK;
  plan->arena_size[0] = psize_l;
  plan->arena_size[1] = psize_r;
  plan->arena_off[0] = poff_l;
  plan->arena_off[1] = poff_r;
  if (!d->dry_run) {
    // padded device copies of the arenas and ψ; zeroed so every pad is 0
    auto repack = [&](const double* src, const int64_t* boff, const std::vector<int64_t>& poff,
                      const std::vector<int32_t>& shift, const int32_t* dim, int nops, int nsec,
                      int64_t psize, double** out) {
      int r = cuda_check(cudaMalloc(out, sizeof(double) * std::max<int64_t>(psize, 2)),
                         "cudaMalloc padded arena");
      if (!r) r = cuda_check(cudaMemset(*out, 0, sizeof(double) * std::max<int64_t>(psize, 2)),
                             "memset padded arena");
      std::vector<PadTask> tasks;
      for (int o = 0; o < nops; ++o)
        for (int j = 0; j < nsec; ++j) {
          const size_t x = (size_t)o * nsec + j;
          if (poff[x] < 0) continue;
          tasks.push_back({boff[x], poff[x], dim[shift[x]], dim[j], dim[j], pad2(dim[j])});
        }
      PadList pl;
      if (!r) r = upload_vec(tasks, &pl.d_tasks);
      pl.n = static_cast<int64_t>(tasks.size());
      // no source arena: the plan owns zeroed padded arenas that the caller
      // fills in place (sdmrg_plan_arena) — no dense copy ever coexists
      if (!r && pl.n > 0 && src) {
        {
          pad_kernel<<<static_cast<unsigned>(std::min<int64_t>(pl.n, 148 * 16)), 256>>>(
              pl.d_tasks, pl.n, src, *out);
          count_launch();
          r = cuda_check(cudaDeviceSynchronize(), "repack arena");
        }
      }
      pl.release();
      return r;
    };
    rc = repack(d->arena_l, d->blk_off_l, poff_l, shL, d->dim_l, d->nops_l, nL, psize_l,
                &plan->arena_l);
    if (!rc)
      rc = repack(d->arena_r, d->blk_off_r, poff_r, shR, d->dim_r, d->nops_r, nR, psize_r,
                  &plan->arena_r);
    const int64_t pp = std::max<int64_t>(plan->poffs[nk], 2);
    if (!rc) rc = cuda_check(cudaMalloc(&plan->psi_pad, sizeof(double) * pp), "cudaMalloc psi_pad");
    if (!rc) rc = cuda_check(cudaMemset(plan->psi_pad, 0, sizeof(double) * pp), "memset psi_pad");
    std::vector<PadTask> ptasks;
    for (int64_t i = 0; i < nk; ++i) {
      const int m = d->dim_l[keys[i].jl], n = d->dim_r[keys[i].jr];
      ptasks.push_back({plan->offs[i], plan->poffs[i], m, n, n, pad2(n)});
    }
    if (!rc) rc = upload_vec(ptasks, &plan->psi_copy.d_tasks);
    plan->psi_copy.n = static_cast<int64_t>(ptasks.size());
    if (!rc && plan->tiled) {
      const int64_t pt = std::max<int64_t>(plan->ptoffs[nk], 2);
      rc = cuda_check(cudaMalloc(&plan->psi_tiled, sizeof(double) * pt), "cudaMalloc psi_tiled");
      if (!rc) rc = cuda_check(cudaMemset(plan->psi_tiled, 0, sizeof(double) * pt), "memset");
      std::vector<PadTask> tt;
      for (int64_t i = 0; i < nk; ++i) {
        const int m = d->dim_l[keys[i].jl], n = d->dim_r[keys[i].jr];
        const int w = GemmBatch::col_tile_width(n);
        for (int c0 = 0, ct = 0; c0 < n; c0 += w, ++ct)
          tt.push_back({plan->offs[i] + c0, plan->ptoffs[i] + (int64_t)ct * pad16(m) * NC_LD_B, m,
                        std::min(w, n - c0), n, NC_LD_B});
      }
      if (!rc) rc = upload_vec(tt, &plan->psit_copy.d_tasks);
      plan->psit_copy.n = static_cast<int64_t>(tt.size());
    }
  }
  if (!rc && !d->dry_run && getenv("SDMRG_SIDE_STREAM")) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    rc = cuda_check(cudaStreamCreateWithPriority(&plan->side, cudaStreamNonBlocking, lo),
                    "create side stream");
    if (!rc) rc = cuda_check(cudaEventCreateWithFlags(&plan->fork, cudaEventDisableTiming), "event");
    if (!rc) rc = cuda_check(cudaEventCreateWithFlags(&plan->join, cudaEventDisableTiming), "event");
  }
  if (!rc && plan->lsum_doubles > 0)
    rc = cuda_check(cudaMalloc(&plan->lsum, sizeof(double) * plan->lsum_doubles), "cudaMalloc lsum");
  if (!rc && ws_max > 0) {
    rc = cuda_check(cudaMalloc(&plan->workspace, sizeof(double) * ws_max), "cudaMalloc workspace");
    // T pads are never written by the engine: zero them once
    if (!rc) rc = cuda_check(cudaMemset(plan->workspace, 0, sizeof(double) * ws_max),
                             "memset workspace");
  }
  if (!rc && !plan->chunks.empty())
    rc = cuda_check(cudaMalloc(&plan->counters, sizeof(int) * 5 * plan->chunks.size()),
                    "cudaMalloc counters");
  for (auto& ch : plan->chunks) {
    if (rc) break;
    rc = ch.host1.upload(&ch.p1, 0);
    if (!rc) rc = ch.host2.upload(&ch.p2, 0);
    if (!rc) rc = ch.host2big.upload(&ch.p2big, 0);
    if (!rc) rc = ch.host1big.upload(&ch.p1big, 0);
    if (!rc) rc = ch.fused.upload();
    for (CombList* cl : {&ch.comb0, &ch.comb3}) {
      if (!rc) rc = upload_vec(cl->tasks, &cl->d_tasks);
      if (!rc) rc = upload_vec(cl->outs, &cl->d_outs);
      if (!rc) rc = upload_vec(cl->terms, &cl->d_terms);
      cl->ntasks = static_cast<int64_t>(cl->tasks.size());
      cl->tasks = std::vector<CombTask>();
      cl->outs = std::vector<CombOut>();
      cl->terms = std::vector<CombTerm>();
    }
    ch.host1 = GemmBatch();
    ch.host2 = GemmBatch();
    ch.host2big = GemmBatch();
    ch.host1big = GemmBatch();
  }
  if (rc) {
    sdmrg_plan_destroy(plan);
    return rc;
  }
  sdmrg_plan_stats& st = plan->stats;
  st.build_ms_taskgen = taskgen_ms;
  st.build_ms_emit = emit_ms;
  st.build_ms_device = ms_since(t_dev);
  st.psi_keys = nk;
  st.psi_size = off;
  st.groups = groups;
  st.members = members;
  st.ref_flops = ref_flops;
  st.exec_flops = exec_flops;
  st.local_members = local_members;
  st.t_problems = t_problems;
  st.tiles = tiles;
  st.segments = segments;
  st.chunks = static_cast<int64_t>(plan->chunks.size());
  st.workspace_doubles = ws_max;
  int64_t kernels = 0;
  for (auto& ch : plan->chunks)
    kernels += (ch.comb0.ntasks > 0) + (ch.p1.ntiles > 0) + (ch.p2.ntiles > 0) + (ch.p2big.ntiles > 0) + (ch.p1big.ntiles > 0) + (ch.fused.ntiles > 0) +
               (ch.comb3.ntasks > 0);
  st.kernels_per_apply = kernels;
  st.algo_bytes = static_cast<int64_t>(algo_bytes);
  st.products = products;
  st.combine_outputs = comb_outputs;
  st.combine_terms = comb_terms;
  st.fused_outs = plan->fused_outs;
  st.arena_bytes = 8 * (psize_l + psize_r);
  st.shard_balance_ppm = static_cast<int64_t>(plan->shard_balance * 1e6);
  *out = plan;
  return SDMRG_OK;
}

int sdmrg_plan_stats_get(const sdmrg_plan* plan, sdmrg_plan_stats* out) {
  if (!plan || !out) return fail(SDMRG_EINVAL, "plan_stats: null argument");
  *out = plan->stats;
  return SDMRG_OK;
}

int sdmrg_plan_layout(const sdmrg_plan* plan, int32_t* keys, int64_t* offsets) {
  if (!plan) return fail(SDMRG_EINVAL, "plan_layout: null plan");
  if (keys) std::memcpy(keys, plan->keys.data(), plan->keys.size() * sizeof(int32_t));
  if (offsets) std::memcpy(offsets, plan->offs.data(), plan->offs.size() * sizeof(int64_t));
  return SDMRG_OK;
}

int sdmrg_plan_arena(const sdmrg_plan* plan, int side, double** base, int64_t* size,
                     int64_t* offsets) {
  if (!plan || (side != 0 && side != 1)) return fail(SDMRG_EINVAL, "plan_arena: bad argument");
  if (base) *base = side == 0 ? plan->arena_l : plan->arena_r;
  if (size) *size = plan->arena_size[side];
  if (offsets)
    std::copy(plan->arena_off[side].begin(), plan->arena_off[side].end(), offsets);
  return SDMRG_OK;
}

int sdmrg_plan_diagonal(sdmrg_plan* plan, double* diag, void* stream_) {
  if (!plan || !diag) return fail(SDMRG_EINVAL, "plan_diagonal: null argument");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  int rc = cuda_check(cudaMemsetAsync(diag, 0, sizeof(double) * std::max<int64_t>(plan->stats.psi_size, 1),
                                      stream), "memset diagonal");
  if (rc || plan->diag_keys.empty()) return rc;
  DiagKey* dk = nullptr;
  DiagMem* dm = nullptr;
  rc = cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&dk), plan->diag_keys.size() * sizeof(DiagKey),
                                  stream), "diag keys");
  if (!rc) rc = cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&dm),
                                           std::max<size_t>(plan->diag_mems.size(), 1) * sizeof(DiagMem),
                                           stream), "diag members");
  if (!rc) rc = cuda_check(cudaMemcpyAsync(dk, plan->diag_keys.data(), plan->diag_keys.size() * sizeof(DiagKey),
                                           cudaMemcpyHostToDevice, stream), "diag keys upload");
  if (!rc && !plan->diag_mems.empty())
    rc = cuda_check(cudaMemcpyAsync(dm, plan->diag_mems.data(), plan->diag_mems.size() * sizeof(DiagMem),
                                    cudaMemcpyHostToDevice, stream), "diag members upload");
  if (!rc) {
    const int nkeys = static_cast<int>(plan->diag_keys.size());
    diag_kernel<<<std::min(nkeys, 148 * 8), 256, 0, stream>>>(dk, nkeys, dm, plan->arena_l,
                                                              plan->arena_r, diag);
    count_launch();
    rc = cuda_check(cudaGetLastError(), "diag launch");
  }
  if (dk) cudaFreeAsync(dk, stream);
  if (dm) cudaFreeAsync(dm, stream);
  return rc;
}

int sdmrg_plan_shard(const sdmrg_plan* plan, int32_t* mine) {
  if (!plan || !mine) return fail(SDMRG_EINVAL, "plan_shard: null argument");
  for (size_t i = 0; i < plan->mine.size(); ++i) mine[i] = plan->mine[i] ? 1 : 0;
  return SDMRG_OK;
}

int sdmrg_plan_groups(const sdmrg_plan* plan, int32_t* group_psi, int32_t* group_out,
                      int64_t* group_begin, int64_t* member_row, double* member_scale) {
  if (!plan) return fail(SDMRG_EINVAL, "plan_groups: null plan");
  if (plan->g_begin.empty()) return fail(SDMRG_EINVAL, "plan_groups: built without keep_groups");
  std::copy(plan->g_psi.begin(), plan->g_psi.end(), group_psi);
  std::copy(plan->g_out.begin(), plan->g_out.end(), group_out);
  std::copy(plan->g_begin.begin(), plan->g_begin.end(), group_begin);
  for (size_t i = 0; i < plan->m_row.size(); ++i) member_row[i] = plan->m_row[i];
  std::copy(plan->m_scale.begin(), plan->m_scale.end(), member_scale);
  return SDMRG_OK;
}

int sdmrg_plan_apply(sdmrg_plan* plan, const double* psi, double* sigma, int accumulate,
                     void* stream_) {
  if (!plan || !psi || !sigma) return fail(SDMRG_EINVAL, "plan_apply: null argument");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  int rc;
  if (!accumulate && plan->stats.psi_size > 0) {
    rc = cuda_check(cudaMemsetAsync(sigma, 0, sizeof(double) * plan->stats.psi_size, stream),
                    "memset sigma");
    if (rc) return rc;
  }
  if (plan->chunks.empty()) return SDMRG_OK;
  rc = cuda_check(cudaMemsetAsync(plan->counters, 0, sizeof(int) * 5 * plan->chunks.size(), stream),
                  "memset counters");
  if (rc) return rc;
  if (plan->psi_copy.n > 0) {
    pad_kernel<<<static_cast<unsigned>(std::min<int64_t>(plan->psi_copy.n, 148 * 8)), 256, 0,
                 stream>>>(plan->psi_copy.d_tasks, plan->psi_copy.n, psi, plan->psi_pad);
    count_launch();
    rc = cuda_check(cudaGetLastError(), "psi pad launch");
    if (rc) return rc;
  }
  if (plan->psit_copy.n > 0) {
    pad_kernel<<<static_cast<unsigned>(std::min<int64_t>(plan->psit_copy.n, 148 * 8)), 256, 0,
                 stream>>>(plan->psit_copy.d_tasks, plan->psit_copy.n, psi, plan->psi_tiled);
    count_launch();
    rc = cuda_check(cudaGetLastError(), "psi tiled launch");
    if (rc) return rc;
  }
  Bases bases{};
  bases.p[B_LSUM] = plan->lsum;
  bases.p[B_PSIT] = plan->psi_tiled;
  bases.p[B_PSI] = plan->psi_pad;
  bases.p[B_SIGMA] = sigma;
  bases.p[B_ARENA_L] = const_cast<double*>(plan->arena_l);
  bases.p[B_ARENA_R] = const_cast<double*>(plan->arena_r);
  bases.p[B_WS] = plan->workspace;
  for (size_t c = 0; c < plan->chunks.size(); ++c) {
    Chunk& ch = plan->chunks[c];
    // phase 0 on the side stream, ordered after everything queued so far
    // (the previous chunk / apply still reads the workspace it rewrites)
    const bool fork = ch.comb0.ntasks > 0 && plan->side != nullptr;
    cudaStream_t s0 = fork ? plan->side : stream;
    if (fork) {
      cudaEventRecord(plan->fork, stream);
      cudaStreamWaitEvent(plan->side, plan->fork, 0);
    }
    if (plan->timing) cudaEventRecord(ch.ev[0], s0);
    if (!plan->lsum_ready || !plan->lsum_persistent) {
      rc = launch_combine(ch.comb0, bases, s0);
      if (rc) return rc;
    }
    if (plan->timing) cudaEventRecord(ch.ev[1], s0);
    if (fork) cudaEventRecord(plan->join, plan->side);
    if (plan->timing) cudaEventRecord(ch.ev[2], stream);
    rc = launch_engine(false, true, ch.p1, bases, plan->counters + 5 * c, stream, true);
    if (rc) return rc;
    if (ch.p1big.ntiles > 0) {
      rc = cuda_check(static_cast<cudaError_t>(sdmrg_internal_launch_big(
                          ch.p1big.tiles, static_cast<int>(ch.p1big.ntiles), ch.p1big.segs,
                          plan->counters + 5 * c + 4, &bases, stream, 0, 1)),
                      "big-tile phase-1 launch");
      count_launch();
      if (rc) return rc;
    }
    if (plan->timing) cudaEventRecord(ch.ev[3], stream);
    if (fork) cudaStreamWaitEvent(stream, plan->join, 0);
    if (plan->timing) cudaEventRecord(ch.ev[4], stream);
    rc = launch_engine(false, false, ch.p2, bases, plan->counters + 5 * c + 1, stream, true,
                       ch.p2_one_body);
    if (rc) return rc;
    rc = launch_fused(ch.fused, bases, plan->counters + 5 * c + 2, stream);
    if (rc) return rc;
    if (ch.p2big.ntiles > 0) {
      rc = cuda_check(static_cast<cudaError_t>(sdmrg_internal_launch_big(
                          ch.p2big.tiles, static_cast<int>(ch.p2big.ntiles), ch.p2big.segs,
                          plan->counters + 5 * c + 3, &bases, stream, ch.p2big_one_body, 0)),
                      "big-tile engine launch");
      count_launch();
    }
    if (rc) return rc;
    if (plan->timing) {
      cudaEventRecord(ch.ev[5], stream);
      cudaEventRecord(ch.ev[6], stream);
    }
    rc = launch_combine(ch.comb3, bases, stream, true);
    if (rc) return rc;
    if (plan->timing) cudaEventRecord(ch.ev[7], stream);
  }
  plan->lsum_ready = true;
  return SDMRG_OK;
}

int sdmrg_plan_invalidate(sdmrg_plan* plan) {
  if (!plan) return fail(SDMRG_EINVAL, "plan_invalidate: null plan");
  plan->lsum_ready = false;
  return SDMRG_OK;
}

int sdmrg_plan_set_timing(sdmrg_plan* plan, int enable) {
  if (!plan) return fail(SDMRG_EINVAL, "plan_set_timing: null plan");
  if (enable && !plan->timing) {
    for (auto& ch : plan->chunks)
      for (auto& e : ch.ev) {
        int rc = cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        if (rc) return rc;
      }
  }
  plan->timing = enable ? 1 : 0;
  return SDMRG_OK;
}

int sdmrg_plan_timing(sdmrg_plan* plan, double* ms, int64_t* flops, int64_t* bytes) {
  if (!plan || !plan->timing) return fail(SDMRG_EINVAL, "plan_timing: timing not enabled");
  double t[4] = {0.0, 0.0, 0.0, 0.0};
  int64_t f[4] = {0, 0, 0, 0}, by[4] = {0, 0, 0, 0};
  for (auto& ch : plan->chunks) {
    int rc = cuda_check(cudaEventSynchronize(ch.ev[7]), "timing sync");
    if (rc) return rc;
    for (int p = 0; p < 4; ++p) {
      float x = 0.f;
      cudaEventElapsedTime(&x, ch.ev[2 * p], ch.ev[2 * p + 1]);
      t[p] += x;
    }
    f[0] += ch.flops0;
    f[1] += ch.flops1;
    f[2] += ch.flops2;
    by[0] += ch.bytes0;
    by[3] += ch.bytes3;
  }
  for (int p = 0; p < 4; ++p) {
    if (ms) ms[p] = t[p];
    if (flops) flops[p] = f[p];
    if (bytes) bytes[p] = by[p];
  }
  return SDMRG_OK;
}

int sdmrg_plan_destroy(sdmrg_plan* plan) {
  if (!plan) return SDMRG_OK;
  for (auto& ch : plan->chunks) {
    ch.p1.release();
    ch.p2.release();
    ch.p2big.release();
    ch.p1big.release();
    ch.fused.release();
    ch.comb0.release();
    ch.comb3.release();
    for (auto& e : ch.ev)
      if (e) cudaEventDestroy(e);
  }
  if (plan->workspace) cudaFree(plan->workspace);
  if (plan->lsum) cudaFree(plan->lsum);
  if (plan->arena_l) cudaFree(plan->arena_l);
  if (plan->arena_r) cudaFree(plan->arena_r);
  if (plan->psi_pad) cudaFree(plan->psi_pad);
  plan->psi_copy.release();
  plan->psit_copy.release();
  if (plan->psi_tiled) cudaFree(plan->psi_tiled);
  if (plan->fork) cudaEventDestroy(plan->fork);
  if (plan->join) cudaEventDestroy(plan->join);
  if (plan->side) cudaStreamDestroy(plan->side);
  if (plan->counters) cudaFree(plan->counters);
  delete plan;
  return SDMRG_OK;
}

}  // extern "C"
