// engine.cuh — persistent segmented grouped GEMM in FP64 for sm_100a.
//
// One kernel family executes every dense contraction of the H_eff·ψ /
// renormalization path:
//
//     C_p  =  beta_p * C_p  +  sum_{s in segs(p)}  scale_s * opA_s @ opB_s
//
// over a flat list of output tiles (64 x 64) drawn from many problems p of
// arbitrary size.  The K dimension of a problem is a *list of segments*: this
// is SBMM4S's concatenated GEMM (sbmm4s.py:150 concat_gemm_accumulate — the
// horizontally concatenated L stack times the vertically concatenated temp)
// without requiring the members to be contiguous, so the "sum over members"
// is carried by the shared inner dimension and no reduction pass exists
// (sbmm4s.py:1-12, paper §II.C).  Each tile is owned by exactly one CTA, so
// accumulation order is fixed and results are deterministic.
//
// Math: DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).  tcgen05 has no f64
// kind; on B200 the FP64 tensor pipe is reached through DMMA (measured 37.1
// TFLOP/s issue ceiling, profiles/).  Staging: 3-stage cp.async (LDGSTS.64)
// ring in shared memory, padded so fragment loads are conflict-free; sector
// blocks have odd leading dimensions, hence 8-byte async copies.
//
// Instruction diet (profiles/r1_phase*.txt showed ~11 instructions per DMMA
// in the first version): per-thread load pointers are set up once per
// segment and advanced by a constant per stage; stage metadata rotates in
// registers; the next segment's descriptor is prefetched one segment ahead;
// fragment loads use [base + immediate] addressing; the warp's active 8x8
// block count selects a branch-free DMMA body (no predicated mma.sync, so
// no WARPSYNC per DMMA).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sdmrg {

// Encoded device address: bits 60..63 select a base pointer (kernel
// parameter), bits 0..59 are an element offset.  Lets one descriptor list
// serve every apply while ψ/σ buffers change (Lanczos vectors).
constexpr int kHandleShift = 60;
constexpr uint64_t kHandleMask = (uint64_t(1) << kHandleShift) - 1;
__host__ __device__ inline uint64_t make_handle(int base, int64_t off) {
  return (uint64_t(base) << kHandleShift) | (uint64_t(off) & kHandleMask);
}
constexpr int kMaxBases = 8;
struct Bases {
  double* p[kMaxBases];
};

struct Prob {        // 32 B
  uint64_t c;        // handle of C(0,0); C row-major, ldc
  int32_t ldc;
  int32_t m, n;      // problem extents
  int32_t seg_begin, seg_end;
  int32_t beta;      // 1: accumulate into C, 0: overwrite
};
struct Tile {        // 16 B
  int32_t prob;
  int32_t row0, col0;
  int32_t pad;
};
struct Seg {         // 40 B
  uint64_t a;        // handle of opA(0,0)
  uint64_t b;        // handle of opB(0,0)
  int32_t lda, ldb;
  int32_t k;         // > 0 (empty segments are never emitted)
  int32_t pad;
  double scale;
};

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, THREADS = 128;
constexpr int PAD = 4;
constexpr int SA_ELEMS = BM * (BK + PAD);  // >= BK * (BM + PAD)
constexpr int SB_ELEMS = BN * (BK + PAD);
constexpr int STAGE_ELEMS = SA_ELEMS + SB_ELEMS;
constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * 8;
static_assert(BK * (BM + PAD) <= SA_ELEMS, "A stage too small");

__device__ __forceinline__ const double* resolve(const Bases& bases, uint64_t h) {
  return bases.p[h >> kHandleShift] + (h & kHandleMask);
}

__device__ __forceinline__ void cp_async8(uint32_t saddr, const double* gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// Per-thread load geometry (see load mapping in issue_stage):
//   A K-contig : kk = tid % 16, rows tid/16 + 8i      smem [BM][BK+PAD]
//   A M-contig : row = tid % 64, kk = tid/64 + 2i     smem [BK][BM+PAD]
//   B N-contig : col = tid % 64, kk = tid/64 + 2i     smem [BK][BN+PAD]
//   B K-contig : kk = tid % 16, cols tid/16 + 8i      smem [BN][BK+PAD]
// TA: opA stored M-contiguous (A(i,k) = a[k*lda + i]); else K-contiguous.
// TB: opB stored K-contiguous (B(k,j) = b[j*ldb + k]); else N-contiguous.
struct SegState {
  const double* a;   // thread's A base for k = 0 of this segment
  const double* b;
  int64_t a_kstep;   // element step of the A base per +1 in k
  int64_t b_kstep;
  int64_t a_istep;   // element step between the thread's 8 A elements
  int64_t b_istep;
  int k;
  double scale;
};

template <bool TA, bool TB>
__device__ __forceinline__ void setup_seg(SegState& st, const Seg& s, const Bases& bases,
                                          int row0, int col0, int tid) {
  const double* a = resolve(bases, s.a);
  const double* b = resolve(bases, s.b);
  if (!TA) {  // A(i,k) = a[i*lda + k]; thread: kk = tid%16, row = tid/16 + 8i
    st.a = a + (int64_t)(row0 + tid / BK) * s.lda + (tid % BK);
    st.a_kstep = 1;
    st.a_istep = (int64_t)8 * s.lda;
  } else {    // A(i,k) = a[k*lda + i]; thread: row = tid%64, kk = tid/64 + 2i
    st.a = a + (int64_t)(tid / BM) * s.lda + row0 + (tid % BM);
    st.a_kstep = s.lda;
    st.a_istep = (int64_t)2 * s.lda;
  }
  if (TB) {   // B(k,j) = b[j*ldb + k]; thread: kk = tid%16, col = tid/16 + 8i
    st.b = b + (int64_t)(col0 + tid / BK) * s.ldb + (tid % BK);
    st.b_kstep = 1;
    st.b_istep = (int64_t)8 * s.ldb;
  } else {    // B(k,j) = b[k*ldb + j]; thread: col = tid%64, kk = tid/64 + 2i
    st.b = b + (int64_t)(tid / BN) * s.ldb + col0 + (tid % BN);
    st.b_kstep = s.ldb;
    st.b_istep = (int64_t)2 * s.ldb;
  }
  st.k = s.k;
  st.scale = s.scale;
}

// Branch-free DMMA body over one stage for a warp owning MB x NB active
// 8x8 blocks.  aoff/boff: per-thread byte addresses of fragment (0,0).
template <bool TA, bool TB, int MB, int NB>
__device__ __forceinline__ void mma_stage(double (&acc)[4][4][2], uint32_t a_base, uint32_t b_base,
                                          int nks, double scale, bool scaled) {
  // byte strides inside a stage (compile-time)
  constexpr int A_I = TA ? 8 * 8 : 8 * (BK + PAD) * 8;   // next 8-row block
  constexpr int A_K = TA ? 4 * (BM + PAD) * 8 : 4 * 8;   // next k4 step
  constexpr int B_J = TB ? 8 * (BK + PAD) * 8 : 8 * 8;   // next 8-col block
  constexpr int B_K = TB ? 4 * 8 : 4 * (BN + PAD) * 8;
#pragma unroll
  for (int ks = 0; ks < BK / 4; ++ks) {
    if (ks < nks) {
      double af[MB], bf[NB];
#pragma unroll
      for (int i = 0; i < MB; ++i) af[i] = lds64(a_base + i * A_I + ks * A_K);
#pragma unroll
      for (int j = 0; j < NB; ++j) bf[j] = lds64(b_base + j * B_J + ks * B_K);
      if (scaled) {
#pragma unroll
        for (int i = 0; i < MB; ++i) af[i] *= scale;
      }
#pragma unroll
      for (int i = 0; i < MB; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
}

template <bool TA, bool TB, int MB>
__device__ __forceinline__ void mma_stage_nb(double (&acc)[4][4][2], uint32_t a, uint32_t b,
                                             int nblk, int nks, double scale, bool scaled) {
  switch (nblk) {
    case 4: mma_stage<TA, TB, MB, 4>(acc, a, b, nks, scale, scaled); break;
    case 3: mma_stage<TA, TB, MB, 3>(acc, a, b, nks, scale, scaled); break;
    case 2: mma_stage<TA, TB, MB, 2>(acc, a, b, nks, scale, scaled); break;
    case 1: mma_stage<TA, TB, MB, 1>(acc, a, b, nks, scale, scaled); break;
    default: break;
  }
}

template <bool TA, bool TB>
__device__ __forceinline__ void mma_dispatch(double (&acc)[4][4][2], uint32_t a, uint32_t b,
                                             int mblk, int nblk, int nks, double scale) {
  const bool scaled = scale != 1.0;
  if (mblk == 4 && nblk == 4) {
    mma_stage<TA, TB, 4, 4>(acc, a, b, nks, scale, scaled);
    return;
  }
  switch (mblk) {
    case 4: mma_stage_nb<TA, TB, 4>(acc, a, b, nblk, nks, scale, scaled); break;
    case 3: mma_stage_nb<TA, TB, 3>(acc, a, b, nblk, nks, scale, scaled); break;
    case 2: mma_stage_nb<TA, TB, 2>(acc, a, b, nblk, nks, scale, scaled); break;
    case 1: mma_stage_nb<TA, TB, 1>(acc, a, b, nblk, nks, scale, scaled); break;
    default: break;
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS, 3)
seg_gemm_kernel(const Tile* __restrict__ tiles, int ntiles, const Prob* __restrict__ probs,
                const Seg* __restrict__ segs, int* __restrict__ counter, Bases bases) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_tile[2];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wr0 = (warp >> 1) * 32, wc0 = (warp & 1) * 32;  // 2 x 2 warps, 32 x 32 each
  const int lr = lane >> 2, lc = lane & 3;
  const uint32_t smem_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));

  // per-thread smem store offsets (bytes, within a stage) of load element i=0
  const uint32_t sa_st = TA ? ((tid / BM) * (BM + PAD) + (tid % BM)) * 8
                            : ((tid / BK) * (BK + PAD) + (tid % BK)) * 8;
  const uint32_t sa_step = TA ? 2 * (BM + PAD) * 8 : 8 * (BK + PAD) * 8;
  const uint32_t sb_st = TB ? ((tid / BK) * (BK + PAD) + (tid % BK)) * 8
                            : ((tid / BN) * (BN + PAD) + (tid % BN)) * 8;
  const uint32_t sb_step = TB ? 8 * (BK + PAD) * 8 : 2 * (BN + PAD) * 8;
  // per-thread fragment base (bytes, within a stage)
  const uint32_t fa = TA ? (lc * (BM + PAD) + wr0 + lr) * 8 : ((wr0 + lr) * (BK + PAD) + lc) * 8;
  const uint32_t fb = SA_ELEMS * 8 +
                      (TB ? ((wc0 + lr) * (BK + PAD) + lc) * 8 : (lc * (BN + PAD) + wc0 + lr) * 8);
  // k index of this thread's load elements (for k-tail masking)
  const int a_k0 = TA ? tid / BM : tid % BK;   // + 2i when TA
  const int b_k0 = TB ? tid % BK : tid / BN;   // + 2i when !TB

  if (tid == 0) s_tile[0] = atomicAdd(counter, 1);
  __syncthreads();
  int t = s_tile[0];
  int flip = 0;

  while (t < ntiles) {
    // prefetch the next tile index while this one runs
    if (tid == 0) s_tile[flip ^ 1] = atomicAdd(counter, 1);
    const Tile tile = tiles[t];
    const Prob prob = probs[tile.prob];
    const int mrem = prob.m - tile.row0;
    const int nrem = prob.n - tile.col0;
    const int mblk = min(4, max(0, (mrem - wr0 + 7) >> 3));
    const int nblk = min(4, max(0, (nrem - wc0 + 7) >> 3));
    // row / col validity masks of this thread's 8 load elements
    uint32_t amask = 0, bmask = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int ar = TA ? (tid % BM) : (tid / BK + 8 * i);
      const int bc = TB ? (tid / BK + 8 * i) : (tid % BN);
      amask |= (ar < mrem ? 1u : 0u) << i;
      bmask |= (bc < nrem ? 1u : 0u) << i;
    }

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // loader cursor
    int seg = prob.seg_begin;
    int koff = 0;
    SegState cur;
    Seg nxt;  // raw descriptor of seg+1, loaded one segment ahead
    if (seg < prob.seg_end) setup_seg<TA, TB>(cur, segs[seg], bases, tile.row0, tile.col0, tid);
    if (seg + 1 < prob.seg_end) nxt = segs[seg + 1];
    // stage metadata ring (registers): nks (0 = end) and scale
    int nks0 = 0, nks1 = 0, nks2 = 0;
    double sc0 = 0.0, sc1 = 0.0, sc2 = 0.0;

    auto issue = [&](int stage, int& nks_out, double& sc_out) {
      if (seg < prob.seg_end) {
        const int krem = min(BK, cur.k - koff);
        const uint32_t sbase = smem_base + stage * (STAGE_ELEMS * 8);
        const double* pa = cur.a + (int64_t)koff * cur.a_kstep;
        const double* pb = cur.b + (int64_t)koff * cur.b_kstep;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int ak = TA ? a_k0 + 2 * i : a_k0;
          const bool v = ((amask >> i) & 1u) && ak < krem;
          cp_async8(sbase + sa_st + i * sa_step, v ? pa + i * cur.a_istep : cur.a, v);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int bk = TB ? b_k0 : b_k0 + 2 * i;
          const bool v = ((bmask >> i) & 1u) && bk < krem;
          cp_async8(sbase + SA_ELEMS * 8 + sb_st + i * sb_step, v ? pb + i * cur.b_istep : cur.b, v);
        }
        nks_out = (krem + 3) >> 2;
        sc_out = cur.scale;
        koff += BK;
        if (koff >= cur.k) {
          koff = 0;
          ++seg;
          if (seg < prob.seg_end) setup_seg<TA, TB>(cur, nxt, bases, tile.row0, tile.col0, tid);
          if (seg + 1 < prob.seg_end) nxt = segs[seg + 1];
        }
      } else {
        nks_out = 0;
        sc_out = 0.0;
      }
      cp_async_commit();
    };

    issue(0, nks0, sc0);
    issue(1, nks1, sc1);
    int stage = 0;
    for (;;) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (nks0 == 0) break;
      const int nks = nks0;
      const double sc = sc0;
      int ns = stage + 2;
      if (ns >= STAGES) ns -= STAGES;
      issue(ns, nks2, sc2);
      const uint32_t st_base = smem_base + stage * (STAGE_ELEMS * 8);
      mma_dispatch<TA, TB>(acc, st_base + fa, st_base + fb, mblk, nblk, nks, sc);
      // rotate the metadata ring
      nks0 = nks1;
      sc0 = sc1;
      nks1 = nks2;
      sc1 = sc2;
      stage = stage + 1 == STAGES ? 0 : stage + 1;
    }
    cp_async_wait<0>();

    // ---- epilogue: masked store (optionally accumulating)
    double* c = const_cast<double*>(resolve(bases, prob.c));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = wr0 + i * 8 + lr;
      if (i < mblk && row < mrem) {
        double* crow = c + (int64_t)(tile.row0 + row) * prob.ldc + tile.col0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = wc0 + j * 8 + lc * 2;
          if (j < nblk) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (col + h < nrem) {
                double v = acc[i][j][h];
                if (prob.beta) v += crow[col + h];
                crow[col + h] = v;
              }
            }
          }
        }
      }
    }
    __syncthreads();  // s_tile[flip^1] visible; smem ring free for the next tile
    t = s_tile[flip ^ 1];
    flip ^= 1;
  }
}

}  // namespace sdmrg
