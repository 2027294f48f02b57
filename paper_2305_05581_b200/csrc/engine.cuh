// engine.cuh — persistent segmented grouped GEMM in FP64 for sm_100a.
//
// One kernel family executes every dense contraction of the H_eff·ψ /
// renormalization path:
//
//     C_p  =  beta_p * C_p  +  sum_{s in segs(p)}  scale_s * opA_s @ opB_s
//
// over a flat list of output tiles (<= 64 x 64) drawn from many problems p of
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
// ring in shared memory; sector blocks have odd leading dimensions, hence
// 8-byte async copies.
//
// Shape handling: the host cuts every problem into *balanced* tiles (a
// 138-row sector becomes 48+48+42, not 64+64+10) and each CTA splits its
// tile's 8x8 blocks evenly over a 2x2 warp grid, so the four warps issue the
// same number of DMMAs per stage.  A warp's (rows, cols) block count selects a
// branch-free DMMA body (no predicated mma.sync).
//
// Shared-memory layouts per stage (doubles):
//   K-contiguous operand tile [64][16], XOR-swizzled on 4-wide k groups:
//       (r, k) -> r*16 + (((k>>2) ^ (r&3))<<2 | (k&3))
//   M/N-contiguous operand tile [16][64+4] (padding): (k, r) -> k*68 + r
// Both give conflict-free DMMA fragment loads (2 wavefronts per LDS.64).
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
  int16_t tm, tn;    // tile extents (<= 64)
};
struct Seg {         // 40 B
  uint64_t a;        // handle of opA(0,0)
  uint64_t b;        // handle of opB(0,0)
  int32_t lda, ldb;
  int32_t k;         // > 0 (empty segments are never emitted)
  int32_t pad;
  double scale;
};

#ifndef SDMRG_STAGES
#define SDMRG_STAGES 3
#endif
#ifndef SDMRG_MINB
#define SDMRG_MINB 3
#endif
constexpr int BM = 64, BN = 64, BK = 16, STAGES = SDMRG_STAGES, THREADS = 128;
constexpr int PADN = 4;                        // padding of M/N-contiguous tiles
constexpr int KC_ELEMS = 64 * BK;              // K-contiguous tile
constexpr int NC_ELEMS = BK * (64 + PADN);     // M/N-contiguous tile
template <bool TA>
__host__ __device__ constexpr int a_elems() { return TA ? NC_ELEMS : KC_ELEMS; }
template <bool TB>
__host__ __device__ constexpr int b_elems() { return TB ? KC_ELEMS : NC_ELEMS; }
template <bool TA, bool TB>
__host__ __device__ constexpr int stage_elems() { return a_elems<TA>() + b_elems<TB>(); }
template <bool TA, bool TB>
__host__ __device__ constexpr int smem_bytes() { return STAGES * stage_elems<TA, TB>() * 8; }

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

// Volatile on purpose: letting ptxas reorder fragment loads and DMMAs freely
// measured 7% slower (more live registers, profiles/r1_notes.md).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// swizzled position (in doubles) of element (r, k) in a K-contiguous tile
__host__ __device__ constexpr int kc_pos(int r, int k) {
  return r * BK + ((((k >> 2) ^ (r & 3)) << 2) | (k & 3));
}

// Per-thread load geometry.  TA: opA stored M-contiguous (A(i,k) =
// a[k*lda + i]); else K-contiguous (A(i,k) = a[i*lda + k]).  TB: opB stored
// K-contiguous (B(k,j) = b[j*ldb + k]); else N-contiguous (b[k*ldb + j]).
//   K-contig operand : kk = tid % 16, rows tid/16 + 8i      (i < 8)
//   M/N-contig       : row = tid % 64, kk = tid/64 + 2i     (i < 8)
struct SegState {
  const double* a;   // this thread's A element 0 at the current k offset
  const double* b;
  int32_t a_k16, b_k16;      // element step of the bases per stage (+16 in k)
  int32_t a_istep, b_istep;  // element step between the thread's 8 elements
  int32_t kleft;             // k remaining in this segment from the offset
  double scale;
};

template <bool TA, bool TB>
__device__ __forceinline__ void setup_seg(SegState& st, const Seg& s, const Bases& bases,
                                          int row0, int col0, int tid) {
  const double* a = resolve(bases, s.a);
  const double* b = resolve(bases, s.b);
  if (!TA) {
    st.a = a + (int64_t)(row0 + tid / BK) * s.lda + (tid % BK);
    st.a_k16 = BK;
    st.a_istep = 8 * s.lda;
  } else {
    st.a = a + (int64_t)(tid / 64) * s.lda + row0 + (tid % 64);
    st.a_k16 = BK * s.lda;
    st.a_istep = 2 * s.lda;
  }
  if (TB) {
    st.b = b + (int64_t)(col0 + tid / BK) * s.ldb + (tid % BK);
    st.b_k16 = BK;
    st.b_istep = 8 * s.ldb;
  } else {
    st.b = b + (int64_t)(tid / 64) * s.ldb + col0 + (tid % 64);
    st.b_k16 = BK * s.ldb;
    st.b_istep = 2 * s.ldb;
  }
  st.kleft = s.k;
  st.scale = s.scale;
}

__device__ __forceinline__ void cp_async8_full(uint32_t saddr, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem));
}

// Branch-free DMMA body over one stage for a warp owning MB x NB 8x8 blocks.
// a_ks[ks] / b_ks[ks]: per-thread byte address of fragment (block 0, k4 ks).
template <bool TA, bool TB, int MB, int NB>
__device__ __forceinline__ void mma_stage(double (&acc)[4][4][2], const uint32_t (&a_ks)[4],
                                          const uint32_t (&b_ks)[4], int nks, double scale) {
  constexpr int A_I = TA ? 8 * 8 : 8 * BK * 8;           // next 8-row block (bytes)
  constexpr int B_J = TB ? 8 * BK * 8 : 8 * 8;           // next 8-col block
  const bool scaled = scale != 1.0;
#pragma unroll
  for (int ks = 0; ks < BK / 4; ++ks) {
    if (ks < nks) {
      double af[MB], bf[NB];
#pragma unroll
      for (int i = 0; i < MB; ++i) af[i] = lds64(a_ks[ks] + i * A_I);
#pragma unroll
      for (int j = 0; j < NB; ++j) bf[j] = lds64(b_ks[ks] + j * B_J);
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
__device__ __forceinline__ void mma_stage_nb(double (&acc)[4][4][2], const uint32_t (&a)[4],
                                             const uint32_t (&b)[4], int nblk, int nks,
                                             double scale) {
  switch (nblk) {
    case 4: mma_stage<TA, TB, MB, 4>(acc, a, b, nks, scale); break;
    case 3: mma_stage<TA, TB, MB, 3>(acc, a, b, nks, scale); break;
    case 2: mma_stage<TA, TB, MB, 2>(acc, a, b, nks, scale); break;
    case 1: mma_stage<TA, TB, MB, 1>(acc, a, b, nks, scale); break;
    default: break;
  }
}

template <bool TA, bool TB>
__device__ __forceinline__ void mma_dispatch(double (&acc)[4][4][2], const uint32_t (&a)[4],
                                             const uint32_t (&b)[4], int mblk, int nblk, int nks,
                                             double scale) {
  if (mblk == 4 && nblk == 4) {
    mma_stage<TA, TB, 4, 4>(acc, a, b, nks, scale);
    return;
  }
  switch (mblk) {
    case 4: mma_stage_nb<TA, TB, 4>(acc, a, b, nblk, nks, scale); break;
    case 3: mma_stage_nb<TA, TB, 3>(acc, a, b, nblk, nks, scale); break;
    case 2: mma_stage_nb<TA, TB, 2>(acc, a, b, nblk, nks, scale); break;
    case 1: mma_stage_nb<TA, TB, 1>(acc, a, b, nblk, nks, scale); break;
    default: break;
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS, SDMRG_MINB)
seg_gemm_kernel(const Tile* __restrict__ tiles, int ntiles, const Prob* __restrict__ probs,
                const Seg* __restrict__ segs, int* __restrict__ counter, Bases bases) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_tile[2];
  constexpr int A_EL = a_elems<TA>();
  constexpr uint32_t STAGE_B = stage_elems<TA, TB>() * 8;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1;
  const int lr = lane >> 2, lc = lane & 3;
  const uint32_t smem_base = static_cast<uint32_t>(__cvta_generic_to_shared(smem));

  // per-thread cp.async destinations (bytes within a stage) of element 0 and step
  const uint32_t sa_st = TA ? ((tid / 64) * (64 + PADN) + (tid % 64)) * 8
                            : kc_pos(tid / BK, tid % BK) * 8;
  const uint32_t sa_step = TA ? 2 * (64 + PADN) * 8 : 8 * BK * 8;
  const uint32_t sb_st = A_EL * 8 + (TB ? kc_pos(tid / BK, tid % BK) * 8
                                        : ((tid / 64) * (64 + PADN) + (tid % 64)) * 8);
  const uint32_t sb_step = TB ? 8 * BK * 8 : 2 * (64 + PADN) * 8;
  // k index of this thread's load element 0 (+2i for M/N-contig operands)
  const int a_k0 = TA ? tid / 64 : tid % BK;
  const int b_k0 = TB ? tid % BK : tid / 64;

  if (tid == 0) s_tile[0] = atomicAdd(counter, 1);
  __syncthreads();
  int t = s_tile[0];
  int flip = 0;

  while (t < ntiles) {
    if (tid == 0) s_tile[flip ^ 1] = atomicAdd(counter, 1);  // prefetch next tile index
    const Tile tile = tiles[t];
    const Prob prob = probs[tile.prob];
    const int tm = tile.tm, tn = tile.tn;
    // balanced 2x2 warp split of the tile's 8x8 blocks
    const int mb = (tm + 7) >> 3, nb = (tn + 7) >> 3;
    const int mb0 = (mb + 1) >> 1, nb0 = (nb + 1) >> 1;
    const int mblk = wr == 0 ? mb0 : mb - mb0;
    const int nblk = wc == 0 ? nb0 : nb - nb0;
    const int wr0 = wr == 0 ? 0 : mb0 * 8;
    const int wc0 = wc == 0 ? 0 : nb0 * 8;
    // fragment addresses per k4 step (bytes within a stage)
    uint32_t fa[4], fb[4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      fa[ks] = TA ? ((4 * ks + lc) * (64 + PADN) + wr0 + lr) * 8
                  : kc_pos(wr0 + lr, 4 * ks + lc) * 8;
      fb[ks] = A_EL * 8 + (TB ? kc_pos(wc0 + lr, 4 * ks + lc) * 8
                              : ((4 * ks + lc) * (64 + PADN) + wc0 + lr) * 8);
    }
    // row / col validity of this thread's 8 load elements
    uint32_t amask = 0, bmask = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int ar = TA ? (tid % 64) : (tid / BK + 8 * i);
      const int bc = TB ? (tid / BK + 8 * i) : (tid % 64);
      amask |= (ar < tm ? 1u : 0u) << i;
      bmask |= (bc < tn ? 1u : 0u) << i;
    }

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const bool rows_full = amask == 0xffu && bmask == 0xffu;
    int seg = prob.seg_begin;
    SegState cur;
    Seg nxt;  // raw descriptor of seg+1, loaded one segment ahead
    if (seg < prob.seg_end) setup_seg<TA, TB>(cur, segs[seg], bases, tile.row0, tile.col0, tid);
    if (seg + 1 < prob.seg_end) nxt = segs[seg + 1];
    int nks0 = 0, nks1 = 0, nks2 = 0;
    double sc0 = 0.0, sc1 = 0.0, sc2 = 0.0;

    auto issue = [&](uint32_t sbase, int& nks_out, double& sc_out) {
      if (seg < prob.seg_end) {
        const int krem = min(BK, cur.kleft);
        const uint32_t sa = sbase + sa_st, sb = sbase + sb_st;
        if (krem == BK && rows_full) {
          // full stage: no predicates, pointer-increment addressing
#pragma unroll
          for (int i = 0; i < 8; ++i) cp_async8_full(sa + i * sa_step, cur.a + i * cur.a_istep);
#pragma unroll
          for (int i = 0; i < 8; ++i) cp_async8_full(sb + i * sb_step, cur.b + i * cur.b_istep);
        } else {
          // edge stage: skip rows outside the tile, zero-fill the k tail
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool kv = (TA ? a_k0 + 2 * i : a_k0) < krem;
            if ((amask >> i) & 1u)
              cp_async8(sa + i * sa_step, kv ? cur.a + i * cur.a_istep : cur.a, kv);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const bool kv = (TB ? b_k0 : b_k0 + 2 * i) < krem;
            if ((bmask >> i) & 1u)
              cp_async8(sb + i * sb_step, kv ? cur.b + i * cur.b_istep : cur.b, kv);
          }
        }
        nks_out = (krem + 3) >> 2;
        sc_out = cur.scale;
        cur.a += cur.a_k16;
        cur.b += cur.b_k16;
        cur.kleft -= BK;
        if (cur.kleft <= 0) {
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

    issue(smem_base, nks0, sc0);
    issue(smem_base + STAGE_B, nks1, sc1);
    uint32_t st_cur = smem_base;                 // stage being computed
    uint32_t st_nxt = smem_base + 2 * STAGE_B;   // stage being filled
    for (;;) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      if (nks0 == 0) break;
      const int nks = nks0;
      const double sc = sc0;
      issue(st_nxt, nks2, sc2);
      uint32_t a_ks[4], b_ks[4];
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        a_ks[ks] = st_cur + fa[ks];
        b_ks[ks] = st_cur + fb[ks];
      }
      mma_dispatch<TA, TB>(acc, a_ks, b_ks, mblk, nblk, nks, sc);
      nks0 = nks1;
      sc0 = sc1;
      nks1 = nks2;
      sc1 = sc2;
      st_cur = st_cur + STAGE_B == smem_base + STAGES * STAGE_B ? smem_base : st_cur + STAGE_B;
      st_nxt = st_nxt + STAGE_B == smem_base + STAGES * STAGE_B ? smem_base : st_nxt + STAGE_B;
    }
    cp_async_wait<0>();

    // ---- epilogue: masked store (optionally accumulating)
    double* c = const_cast<double*>(resolve(bases, prob.c));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = wr0 + i * 8 + lr;
      if (i < mblk && row < tm) {
        double* crow = c + (int64_t)(tile.row0 + row) * prob.ldc + tile.col0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int col = wc0 + j * 8 + lc * 2;
          if (j < nblk) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (col + h < tn) {
                double v = acc[i][j][h];
                if (prob.beta) v += crow[col + h];
                crow[col + h] = v;
              }
            }
          }
        }
      }
    }
    __syncthreads();  // s_tile visible; smem ring free for the next tile
    t = s_tile[flip ^ 1];
    flip ^= 1;
  }
}

}  // namespace sdmrg
