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
// is done by the shared inner dimension and no reduction pass exists
// (sbmm4s.py:1-12, paper §II.C).  Each tile is owned by exactly one CTA, so
// accumulation order is fixed and results are deterministic.
//
// Math: DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).  tcgen05 has no f64
// kind; on B200 the FP64 tensor pipe is reached through DMMA (measured 37.1
// TFLOP/s issue ceiling, profiles/fp64_peaks.txt).  Staging: 3-stage
// cp.async (LDGSTS.64) ring in shared memory, padded so every fragment load is
// two conflict-free wavefronts.  Block pointers are arbitrary (sector blocks
// have odd leading dimensions), hence 8-byte async copies.
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
  int32_t k;
  int32_t pad;
  double scale;
};

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, THREADS = 128;
constexpr int PAD = 4;
// stage footprint (doubles): the larger of the two layouts per operand
constexpr int SA_ELEMS = (BM * (BK + PAD) > BK * (BM + PAD)) ? BM * (BK + PAD) : BK * (BM + PAD);
constexpr int SB_ELEMS = (BN * (BK + PAD) > BK * (BN + PAD)) ? BN * (BK + PAD) : BK * (BN + PAD);
constexpr int SMEM_BYTES = STAGES * (SA_ELEMS + SB_ELEMS) * 8 + 64;

__device__ __forceinline__ const double* resolve(const Bases& bases, uint64_t h) {
  return bases.p[h >> kHandleShift] + (h & kHandleMask);
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int src_size = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// TA: opA stored M-contiguous (A(i,k) = a[k*lda + i]); else K-contiguous
// (A(i,k) = a[i*lda + k]).  TB: opB stored K-contiguous (B(k,j) = b[j*ldb+k]);
// else N-contiguous (B(k,j) = b[k*ldb + j]).
template <bool TA, bool TB>
__device__ __forceinline__ void load_stage(double* sA, double* sB, const double* a, int lda,
                                           const double* b, int ldb, int mrem, int nrem,
                                           int krem, int tid) {
  const double* dummy = a;
#pragma unroll
  for (int i = 0; i < (BM * BK) / THREADS; ++i) {
    int e = tid + i * THREADS;
    if (!TA) {
      int row = e / BK, kk = e % BK;
      bool v = (row < mrem) && (kk < krem);
      cp_async8(sA + row * (BK + PAD) + kk, v ? a + (int64_t)row * lda + kk : dummy, v);
    } else {
      int kk = e / BM, row = e % BM;
      bool v = (row < mrem) && (kk < krem);
      cp_async8(sA + kk * (BM + PAD) + row, v ? a + (int64_t)kk * lda + row : dummy, v);
    }
  }
#pragma unroll
  for (int i = 0; i < (BN * BK) / THREADS; ++i) {
    int e = tid + i * THREADS;
    if (TB) {
      int col = e / BK, kk = e % BK;
      bool v = (col < nrem) && (kk < krem);
      cp_async8(sB + col * (BK + PAD) + kk, v ? b + (int64_t)col * ldb + kk : dummy, v);
    } else {
      int kk = e / BN, col = e % BN;
      bool v = (col < nrem) && (kk < krem);
      cp_async8(sB + kk * (BN + PAD) + col, v ? b + (int64_t)kk * ldb + col : dummy, v);
    }
  }
}

struct Cursor {
  int seg;
  int k0;
};

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS, 3)
seg_gemm_kernel(const Tile* __restrict__ tiles, int ntiles, const Prob* __restrict__ probs,
                const Seg* __restrict__ segs, int* __restrict__ counter, Bases bases) {
  extern __shared__ __align__(16) double smem[];
  double* sA0 = smem;
  double* sB0 = smem + STAGES * SA_ELEMS;
  __shared__ int s_tile;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // 2 x 2 warps, 32 x 32 each
  const int lr = lane >> 2, lc = lane & 3;

  for (;;) {
    if (tid == 0) s_tile = atomicAdd(counter, 1);
    __syncthreads();
    const int t = s_tile;
    __syncthreads();
    if (t >= ntiles) break;
    const Tile tile = tiles[t];
    const Prob prob = probs[tile.prob];
    const int mrem = prob.m - tile.row0;
    const int nrem = prob.n - tile.col0;
    // active 8x8 blocks of this warp's 32x32 sub-tile
    const int wr0 = wm * 32, wc0 = wn * 32;
    const int mblk = min(4, max(0, (mrem - wr0 + 7) >> 3));
    const int nblk = min(4, max(0, (nrem - wc0 + 7) >> 3));

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // ---- pipelined walk over (segment, k-chunk) pairs
    Cursor cur{prob.seg_begin, 0};
    // skip empty segments
    while (cur.seg < prob.seg_end && __ldg(&segs[cur.seg].k) <= 0) ++cur.seg;
    int meta_nks[STAGES];
    double meta_scale[STAGES];

    auto issue = [&](int stage) -> void {
      if (cur.seg < prob.seg_end) {
        const Seg& s = segs[cur.seg];
        const int k = s.k;
        const int krem = min(BK, k - cur.k0);
        const double* a = resolve(bases, s.a);
        const double* b = resolve(bases, s.b);
        const double* ap = TA ? a + (int64_t)cur.k0 * s.lda + tile.row0
                              : a + (int64_t)tile.row0 * s.lda + cur.k0;
        const double* bp = TB ? b + (int64_t)tile.col0 * s.ldb + cur.k0
                              : b + (int64_t)cur.k0 * s.ldb + tile.col0;
        load_stage<TA, TB>(sA0 + stage * SA_ELEMS, sB0 + stage * SB_ELEMS, ap, s.lda, bp, s.ldb,
                           mrem, nrem, krem, tid);
        meta_nks[stage] = (krem + 3) >> 2;
        meta_scale[stage] = s.scale;
        cur.k0 += BK;
        if (cur.k0 >= k) {
          cur.k0 = 0;
          ++cur.seg;
          while (cur.seg < prob.seg_end && __ldg(&segs[cur.seg].k) <= 0) ++cur.seg;
        }
      } else {
        meta_nks[stage] = 0;
        meta_scale[stage] = 0.0;
      }
      cp_async_commit();
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) issue(s);

    int stage = 0;
    for (;;) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int nks = meta_nks[stage];
      if (nks == 0) break;
      const double scale = meta_scale[stage];
      issue((stage + STAGES - 1) % STAGES);

      const double* sA = sA0 + stage * SA_ELEMS;
      const double* sB = sB0 + stage * SB_ELEMS;
      if (mblk > 0 && nblk > 0) {
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
          if (ks < nks) {
            const int kk = ks * 4 + lc;
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int row = wr0 + i * 8 + lr;
              af[i] = TA ? sA[kk * (BM + PAD) + row] : sA[row * (BK + PAD) + kk];
              af[i] *= scale;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int col = wc0 + j * 8 + lr;
              bf[j] = TB ? sB[col * (BK + PAD) + kk] : sB[kk * (BN + PAD) + col];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (i < mblk && j < nblk) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
          }
        }
      }
      stage = (stage + 1) % STAGES;
    }
    cp_async_wait<0>();
    __syncthreads();

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
  }
}

}  // namespace sdmrg
