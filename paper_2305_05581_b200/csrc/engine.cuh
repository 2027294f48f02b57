// engine.cuh — persistent, warp-specialized segmented grouped GEMM in FP64
// for sm_100a.
//
// One kernel family executes every dense contraction of the H_eff·ψ /
// renormalization path:
//
//     C_p  =  beta_p * C_p  +  sum_{s in segs(p)}  scale_s * opA_s @ opB_s
//
// over a flat list of output tiles (<= 64 x 64) drawn from many problems p of
// arbitrary size.  The K dimension of a problem is a *list of segments*:
// SBMM4S's concatenated GEMM (sbmm4s.py:155 concat_gemm_accumulate — the
// horizontally concatenated L stack times the vertically concatenated temp)
// without requiring the members to be contiguous, so the sum over members is
// carried by the shared inner dimension and no reduction pass exists
// (sbmm4s.py:1-12, paper §II.C).  Each tile has exactly one owner CTA, so
// the accumulation order is fixed and results are bitwise deterministic.
//
// Math: DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).  tcgen05 has no f64
// kind; on B200 the FP64 pipe is shared by DMMA and DFMA (37.1 / 36.7
// TFLOP/s measured, tools/fp64_probe.cu) and cuBLAS's own DGEMM is a DMMA
// kernel (cutlass_80_tensorop_d884gemm, profiles/r1a_launches.txt).
//
// CTA = 1 producer warp + 4 consumer warps, 4 CTAs per SM (persistent; 3-stage
// rings, 96 registers — 4 CTAs x 3 stages measured 1-2% faster than 3 x 4):
//   producer  pulls tiles from a global counter (one tile of lookahead, the
//             next tile's descriptor and first segment prefetched), walks
//             their segments and streams 16-deep K stages of both operands
//             into a STAGES-deep shared-memory ring, across tile boundaries.
//             The H_eff plan keeps every operand block in a padded layout
//             (even leading dimension, 16-byte aligned rows) so its loads are
//             16-byte cp.async (LDGSTS.128); arbitrary user pointers
//             (sdmrg_dgemm, sbmm4s, ...) take 8-byte cp.async.  Completion is
//             tracked by mbarriers (cp.async.mbarrier.arrive.noinc), so
//             descriptor and global-memory latency never stalls the math
//             warps.  (One TMA-unit bulk copy per 128-byte operand row was
//             measured 1.7x slower: profiles/r1_notes.md.)
//   consumers a 2 x 2 warp grid over the tile's 8x8 blocks, balanced (a warp
//             owns up to 4 x 4 blocks, 32 accumulators).  The (row blocks,
//             col blocks) shape is dispatched once per tile into a
//             branch-free DMMA body that loops over the tile's stages and
//             ends in the epilogue (stores straight from registers).
// Why 64 x 64 and 4 math warps per tile: the sector problems are small
// (L=30, D=2048: flop-weighted 124 x 119 x 129 in phase 1, output sectors
// <= 183 in phase 2); a 128 x 128 CTA tile with 8 warps left each warp 8
// DMMAs per k4 step on typical tiles and ran at 12-16 TFLOP/s (profiles/n4a).
//
// Shared-memory layouts per stage (doubles), rows 16-byte aligned for bulk
// copies and conflict-free for DMMA fragment loads (2 wavefronts per LDS.64):
//   K-contiguous operand tile [64][16] with row stride 18: (r, k) -> r*18 + k
//   M/N-contiguous operand tile [16][64+4]:                (k, r) -> k*68 + r
#pragma once
#include <cstdint>
#include <type_traits>
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

__device__ __forceinline__ const double* resolve(const Bases& bases, uint64_t h) {
  return bases.p[h >> kHandleShift] + (h & kHandleMask);
}

struct Prob {        // 32 B
  uint64_t c;        // handle of C(0,0); C row-major, ldc
  int32_t ldc;
  int32_t m, n;      // problem extents
  int32_t seg_begin, seg_end;
  int32_t beta;      // 1: accumulate into C, 0: overwrite
};
struct Tile {        // host only
  int32_t prob;
  int32_t row0, col0;
  int16_t tm, tn;    // tile extents (<= 128)
  int32_t colw;      // the problem's column-tile width (stage-tiled B operands)
};
// Device form of a tile: the problem fields folded in, so the producer needs
// one dependent load (tile -> segment) instead of two.
struct TileRec {     // 40 B
  uint64_t c;        // handle of C(0,0) of the problem
  int32_t ldc, beta;
  int32_t seg_begin, seg_end;
  int32_t row0, col0;
  int16_t tm, tn;
  int32_t colw;      // column-tile width of the problem (stage-tiled B)
};
struct Seg {         // 40 B
  uint64_t a;        // handle of opA(0,0)
  uint64_t b;        // handle of opB(0,0)
  int32_t lda, ldb;
  int32_t k;         // > 0 (empty segments are never emitted)
  // > 0: B is stage-tiled (M/N-contiguous B only): column tile ct of the
  // problem is a contiguous [btile rows = K rounded up to 16][NC_LD_B] block
  // at b + ct * btile * NC_LD_B, so one K stage is ONE contiguous run (a TMA
  // bulk copy); rows >= K are zero.  ldb must be NC_LD_B.
  int32_t btile;
  double scale;
};

// SDMRG_BIG: 128 x 128 tiles, 16 DMMA warps (4 x 4 grid of <= 32 x 32 warp
// tiles) and 2 producer warps, one CTA per SM — the phase-2 instance for σ
// blocks of 65..128 rows and columns, whose four 64 x 64 tiles would each
// stream their own copy of the shared row / column operand panels
// (compiled as a second instance in engine_big.cu, namespace sdmrg_big)
#ifndef SDMRG_BIG
#define SDMRG_BIG 0
#endif
#ifndef SDMRG_STAGES
#define SDMRG_STAGES (SDMRG_BIG ? 5 : 3)
#endif
#ifndef SDMRG_TILE
#define SDMRG_TILE 64
#endif
#ifndef SDMRG_STCS
#define SDMRG_STCS 0
#endif
// per-tile warp grid: 1 x 4 or 4 x 1 instead of 2 x 2 when a tile has an odd
// number of 8-row (8-column) blocks, so the four DMMA warps stay balanced
#ifndef SDMRG_ROTATE
#define SDMRG_ROTATE 1
#endif
#ifndef SDMRG_GRID_ADAPT
#define SDMRG_GRID_ADAPT 1
#endif
__host__ __device__ constexpr int cw_index(int wr, int wc) { return wr * 2 + wc; }
// only for the T = A R^T instances (phase 1): in the phase-2 instance the extra
// bodies push the consumer past its 96-register budget (spills; measured
// slower at L=50 D=4096, profiles/r1_notes.md)
// Phase 2 alternates scaled single-operator segments with unit-scale
// pre-summed ones inside one tile, so both consumer bodies of a tile shape are
// hot.  With many distinct tile shapes (small sectors) that overflows the
// instruction cache (ncu, L=50 D=4096: 24% of phase-2 stall samples were
// no_instruction); the ONE instance runs a single always-scaling body instead
// (a DMUL per fragment, a few % of the FP64 pipe).  The plan picks it per
// launch from its tile-shape mix (plan.cu).
template <bool TB>
__host__ __device__ constexpr bool grid_adapt() {
  return SDMRG_GRID_ADAPT && SDMRG_TILE == 64 && TB;
}
#ifndef SDMRG_MINB
#define SDMRG_MINB (SDMRG_BIG ? 1 : 4)
#endif
constexpr int BM = SDMRG_TILE, BN = SDMRG_TILE, BK = 16;
constexpr int STAGES = SDMRG_STAGES;
static_assert(BM == 64 || (SDMRG_BIG && BM == 128), "tile edge 64 (128: the big instance)");
constexpr int WGRID_R = SDMRG_BIG ? 4 : 2, WGRID_C = SDMRG_BIG ? 4 : 2,
              CONSUMERS = WGRID_R * WGRID_C;
// SDMRG_PRODUCERS=2: one producer warp per operand (A loader leads the tile
// queue, the B loader follows through shared memory and a named barrier)
#ifndef SDMRG_PRODUCERS
#define SDMRG_PRODUCERS (SDMRG_BIG ? 2 : 1)
#endif
constexpr int PRODUCERS = SDMRG_PRODUCERS;
static_assert(PRODUCERS == 1 || PRODUCERS == 2, "one or two producer warps");
constexpr int THREADS = 32 * (CONSUMERS + PRODUCERS);
// SDMRG_SWZ: K-contiguous tiles unpadded ([64][16], 128-byte rows) with the
// k4 groups of row r XOR-swizzled by (r & 3): element (r, k) at
// r * 16 + (k ^ 4 (r & 3)).  A DMMA fragment load (rows lr, k lc of one k4
// step) then hits 16 distinct bank pairs per half-warp; the padded stride 18
// maps rows lr and lr + 1 two bank pairs apart (2-way conflicts for lc >= 2).
#ifndef SDMRG_SWZ
#define SDMRG_SWZ 1
#endif
constexpr int KC_LD = SDMRG_SWZ ? BK : BK + 2;   // K-contiguous row stride
constexpr int NC_LD_A = BM + 4;                  // M-contiguous A row stride
constexpr int NC_LD_B = BN + 4;                  // N-contiguous B row stride
template <bool TA>
__host__ __device__ constexpr int a_elems() { return TA ? BK * NC_LD_A : BM * KC_LD; }
template <bool TB>
__host__ __device__ constexpr int b_elems() { return TB ? BN * KC_LD : BK * NC_LD_B; }
template <bool TA, bool TB>
__host__ __device__ constexpr int stage_elems() { return a_elems<TA>() + b_elems<TB>(); }

// Per-stage metadata written by the producer's lane 0.
struct StageMeta {
  double* c;         // tile origin in C (first stage of a tile)
  double scale;      // != 1: the stage's segment is scaled
  int32_t nks;       // k4 steps in this stage (0: no K, or kEnd)
  int32_t flags;
  int32_t ldc, beta;
  int16_t tm, tn;
  int32_t pad;
};
constexpr int kFirst = 1, kLast = 2, kEnd = 4;
template <bool TA, bool TB>
__host__ __device__ constexpr int smem_bytes() {
  return STAGES * stage_elems<TA, TB>() * 8 + STAGES * (int)sizeof(StageMeta) + 2 * STAGES * 8 +
         kMaxBases * 8 + 16;
}

__device__ __forceinline__ void cp_async8(uint32_t saddr, const double* gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async8_full(uint32_t saddr, const double* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem));
}
// TMA-unit bulk copy global -> shared, completion counted in bytes on an mbarrier
__device__ __forceinline__ void bulk_copy(uint32_t saddr, const double* gmem, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(saddr),
      "l"(gmem), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void sts64_zero(uint32_t saddr) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(saddr), "d"(0.0) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Volatile on purpose: the issue order written here is the schedule.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// k4 steps needed to cover stage k < krem (every stage k >= krem is zero in
// both operands: the loaders zero-fill the tail of every stage).
__host__ __device__ constexpr int steps_for(int krem) { return (krem + 3) >> 2; }

__device__ __forceinline__ void lds128(uint32_t addr, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(addr));
}

// Shared state of one CTA's pipeline.
struct Ring {
  uint32_t smem;     // shared address of stage 0
  uint32_t full0;    // full barriers (STAGES x 8 bytes), then empty barriers
  uint32_t empty0;
  StageMeta* meta;
};

// ------------------------------------------------------------------ consumer
// A warp owning MB x NB 8x8 blocks of a tile: runs every stage of the tile
// (the first one already waited for), then the epilogue.  a_off/b_off: byte
// offset of fragment (block 0, k4 step 0) within a stage.
template <bool TA, bool TB, int MB, int NB, bool ONE>
__device__ __forceinline__ void consume_tile(const Ring& ring, int& stage, uint32_t& phase,
                                             uint32_t a_off, uint32_t b_off, double* c, int ldc,
                                             int beta, int row_lim, int col_lim, int lane) {
  constexpr uint32_t STAGE_B = stage_elems<TA, TB>() * 8;
  constexpr int A_I = TA ? 8 * 8 : 8 * KC_LD * 8;         // next 8-row block (bytes)
  constexpr int B_J = TB ? 8 * KC_LD * 8 : 8 * 8;         // next 8-col block
  constexpr int A_KS = TA ? 4 * NC_LD_A * 8 : 4 * 8;      // next k4 step
  constexpr int B_KS = TB ? 4 * 8 : 4 * NC_LD_B * 8;
  // swizzled K-contiguous operands: k4 step ks of row block sits at k4 group
  // ks ^ (lr & 3) (a0 / b0 then point at k = lc of group 0)
  const uint32_t sw = SDMRG_SWZ ? static_cast<uint32_t>((lane >> 2) & 3) : 0u;
  auto koff_a = [&](int ks) -> uint32_t {
    return (SDMRG_SWZ && !TA) ? ((static_cast<uint32_t>(ks) ^ sw) << 5) : uint32_t(ks * A_KS);
  };
  auto koff_b = [&](int ks) -> uint32_t {
    return (SDMRG_SWZ && TB) ? ((static_cast<uint32_t>(ks) ^ sw) << 5) : uint32_t(ks * B_KS);
  };
  double acc[MB > 0 ? MB : 1][NB > 0 ? NB : 1][2];
#pragma unroll
  for (int i = 0; i < MB; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  while (true) {
    const StageMeta& m = ring.meta[stage];
    const int flags = m.flags;
    const int nks = m.nks;
    const double scale = m.scale;
    const uint32_t a0 = ring.smem + stage * STAGE_B + a_off;
    const uint32_t b0 = ring.smem + stage * STAGE_B + b_off;
    if (MB > 0 && NB > 0) {
#ifdef SDMRG_EXP_NOSCALE
      const bool scaled = false;
#else
      // integer test of the bit pattern: a DSETP would queue on the FP64 pipe
      // behind the DMMAs (ncu: 5% of the consumer stall samples)
      const bool scaled = __double_as_longlong(scale) != 0x3FF0000000000000LL;
#endif
      // the scale branch is warp-uniform per stage; two bodies keep ptxas
      // from if-converting the DMULs into unscaled stages (phase 1 never
      // scales, and a DMUL takes FP64-pipe slots from the DMMAs)
      auto body = [&](auto scaled_t) {
        constexpr bool SCALED = decltype(scaled_t)::value;
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
          if (ks < nks) {
            double af[MB > 0 ? MB : 1], bf[NB > 0 ? NB : 1];
#pragma unroll
            for (int i = 0; i < MB; ++i) af[i] = lds64(a0 + koff_a(ks) + i * A_I);
#pragma unroll
            for (int j = 0; j < NB; ++j) bf[j] = lds64(b0 + koff_b(ks) + j * B_J);
            if (SCALED) {
              const double sk = scale;
              if (NB <= MB) {
#pragma unroll
                for (int j = 0; j < NB; ++j) bf[j] *= sk;
              } else {
#pragma unroll
                for (int i = 0; i < MB; ++i) af[i] *= sk;
              }
            }
#ifndef SDMRG_EXP_NOMMA
#pragma unroll
            for (int i = 0; i < MB; ++i)
#pragma unroll
              for (int j = 0; j < NB; ++j) dmma(acc[i][j], af[i], bf[j]);
#endif
          }
        }
      };
      if constexpr (ONE) {
        body(std::true_type{});  // unit scales multiply too: half the code
      } else {
        if (scaled) body(std::true_type{});
        else body(std::false_type{});
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(ring.empty0 + 8 * stage);
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1;
    }
    if (flags & kLast) break;
    mbar_wait(ring.full0 + 8 * stage, phase);
  }
  // epilogue: masked store (optionally accumulating); row_lim/col_lim are the
  // tile extents relative to this thread's first row / column.  A thread's
  // two accumulators per block are adjacent columns: one 16-byte store when
  // C is 16-byte aligned with an even leading dimension (the plan's T blocks)
  const bool vec2 = ((reinterpret_cast<uintptr_t>(c) | (uintptr_t(ldc) << 3)) & 15) == 0;
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    if (8 * i < row_lim) {
      double* crow = c + (int64_t)(8 * i) * ldc;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (vec2 && 8 * j + 1 < col_lim) {
          double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
          double2* p = reinterpret_cast<double2*>(crow + 8 * j);
          if (beta) {
            const double2 o = *p;
            v.x += o.x;
            v.y += o.y;
            *p = v;
          } else {
#if SDMRG_STCS
            // overwrite-only outputs (the T blocks: 32 GB per apply, read
            // back much later) are streamed: evict-first in L2, so they do
            // not push out the operand panels the running tiles re-read
            __stcs(p, v);
#else
            *p = v;
#endif
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (8 * j + h < col_lim) {
              double v = acc[i][j][h];
              if (beta) v += crow[8 * j + h];
              crow[8 * j + h] = v;
            }
          }
        }
      }
    }
  }
}

#define SDMRG_TILE_CASE(MB, NB)                                                                   \
  case (MB) * 8 + (NB):                                                                           \
    consume_tile<TA, TB, MB, NB, ONE>(ring, stage, phase, a_off, b_off, c, ldc, beta, row_lim,      \
                                      col_lim,                                                \
                                      lane);                                                  \
    break;

template <bool TA, bool TB, bool ONE>
__device__ __forceinline__ void consume_dispatch(int mblk, int nblk, const Ring& ring, int& stage,
                                                 uint32_t& phase, uint32_t a_off, uint32_t b_off,
                                                 double* c, int ldc, int beta, int row_lim,
                                                 int col_lim, int lane) {
  if constexpr (grid_adapt<TB>()) {
    if (mblk > 4 || nblk > 4) {  // 1 x 4 / 4 x 1 warp grids of odd-block tiles
      switch (mblk * 8 + nblk) {
        SDMRG_TILE_CASE(7, 2) SDMRG_TILE_CASE(7, 1) SDMRG_TILE_CASE(5, 2) SDMRG_TILE_CASE(5, 1)
        SDMRG_TILE_CASE(2, 7) SDMRG_TILE_CASE(1, 7) SDMRG_TILE_CASE(2, 5) SDMRG_TILE_CASE(1, 5)
        default: break;
      }
      return;
    }
  }
  switch (mblk * 8 + nblk) {
    SDMRG_TILE_CASE(4, 4) SDMRG_TILE_CASE(4, 3) SDMRG_TILE_CASE(4, 2) SDMRG_TILE_CASE(4, 1)
    SDMRG_TILE_CASE(3, 4) SDMRG_TILE_CASE(3, 3) SDMRG_TILE_CASE(3, 2) SDMRG_TILE_CASE(3, 1)
    SDMRG_TILE_CASE(2, 4) SDMRG_TILE_CASE(2, 3) SDMRG_TILE_CASE(2, 2) SDMRG_TILE_CASE(2, 1)
    SDMRG_TILE_CASE(1, 4) SDMRG_TILE_CASE(1, 3) SDMRG_TILE_CASE(1, 2) SDMRG_TILE_CASE(1, 1)
    default:  // no blocks for this warp: walk the tile's stages
      consume_tile<TA, TB, 0, 0, ONE>(ring, stage, phase, a_off, b_off, c, ldc, beta, row_lim, col_lim,
                                 lane);
      break;
  }
}
#undef SDMRG_TILE_CASE

// ------------------------------------------------------------------ producer
// 8-byte cp.async geometry of one operand within a stage (one producer warp).
//   K-contiguous (A when !TA, B when TB): lane -> k = lane & 15, rows
//     (lane >> 4) + 2i, i < 32; element (r, k) at src + r*ld + k.
//   M/N-contiguous: lane -> columns lane, lane + 32; k = 0..15; element
//     (k, c) at src + k*ld + c.
// The k tail beyond krem is zero-filled (stale shared memory may hold
// non-finite data at kernel start).
template <bool KCONTIG, int NC_LD, int CAP>
__device__ __forceinline__ void load_operand_async(uint32_t sbase, const double* src, int ld,
                                                   int extent, int krem, int lane) {
  if (KCONTIG) {
    const int kk = lane & 15, r0 = lane >> 4;
    const double* p = src + (int64_t)r0 * ld + kk;
    // swizzle: rows r0 + 2i alternate (r & 3) between r0 and r0 + 2
    const int ke = SDMRG_SWZ ? kk ^ (4 * r0) : kk, ko = SDMRG_SWZ ? kk ^ (4 * (r0 + 2)) : kk;
    const uint32_t se = sbase + (r0 * KC_LD + ke) * 8, so = sbase + (r0 * KC_LD + ko) * 8;
    const int nrow = (extent - r0 + 1) >> 1;
    if (kk < krem) {
#pragma unroll 8
      for (int i = 0; i < nrow; ++i)
        cp_async8_full((i & 1 ? so : se) + i * (2 * KC_LD * 8), p + (int64_t)(2 * i) * ld);
    } else {
#pragma unroll 8
      for (int i = 0; i < nrow; ++i) cp_async8((i & 1 ? so : se) + i * (2 * KC_LD * 8), src, false);
    }
  } else {
#pragma unroll
    for (int j = 0; j < CAP / 32; ++j) {
      const int c = lane + 32 * j;
      if (c < extent) {
        const double* p = src + c;
        const uint32_t s0 = sbase + c * 8;
        if (krem >= BK) {
#pragma unroll
          for (int k = 0; k < BK; ++k) cp_async8_full(s0 + k * (NC_LD * 8), p + (int64_t)k * ld);
        } else {
#pragma unroll
          for (int k = 0; k < BK; ++k)
            cp_async8(s0 + k * (NC_LD * 8), k < krem ? p + (int64_t)k * ld : src, k < krem);
        }
      }
    }
  }
}

// 16-byte cp.async geometry (padded layouts: even leading dimensions, even
// element offsets, so every element pair (k, k+1) / (c, c+1) is 16-byte
// aligned in global and shared memory):
//   K-contiguous: lane -> k pair kp = lane & 7 (k = 2kp, 2kp+1), rows
//     (lane >> 3) + 4i, i < 16;
//   M/N-contiguous: lane -> column pairs (2 lane + 64 j, +1), k = 0..15.
// A pair straddling the k tail copies its first element and zero-fills the
// second (src-size 8); pairs past the tail are zero-filled (src-size 0).
__device__ __forceinline__ void cp_async16(uint32_t saddr, const double* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16_full(uint32_t saddr, const double* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
template <bool KCONTIG, int NC_LD, int CAP>
__device__ __forceinline__ void load_operand_aligned(uint32_t sbase, const double* src, int ld,
                                                     int extent, int krem, int lane) {
  if (KCONTIG) {
    const int k = 2 * (lane & 7), r0 = lane >> 3;
    const double* p = src + (int64_t)r0 * ld + k;
    // rows r0 + 4i share (r & 3) = r0 & 3: one swizzled column per lane
    const uint32_t s0 = sbase + (r0 * KC_LD + (SDMRG_SWZ ? k ^ (4 * (r0 & 3)) : k)) * 8;
    const int nrow = (extent - r0 + 3) >> 2;
    if (k + 1 < krem) {
#pragma unroll 4
      for (int i = 0; i < nrow; ++i) cp_async16_full(s0 + i * (4 * KC_LD * 8), p + (int64_t)(4 * i) * ld);
    } else {
      const int bytes = k < krem ? 8 : 0;
      const double* q = k < krem ? p : src;
      const int64_t step = k < krem ? 4 * (int64_t)ld : 0;
#pragma unroll 4
      for (int i = 0; i < nrow; ++i) cp_async16(s0 + i * (4 * KC_LD * 8), q + i * step, bytes);
    }
  } else {
#pragma unroll
    for (int j = 0; j < (CAP + 63) / 64; ++j) {
      const int c = 2 * lane + 64 * j;
      if (c < extent) {
        const double* p = src + c;
        const uint32_t s0 = sbase + c * 8;
        if (krem >= BK) {
#pragma unroll
          for (int k = 0; k < BK; ++k) cp_async16_full(s0 + k * (NC_LD * 8), p + (int64_t)k * ld);
        } else {
#pragma unroll
          for (int k = 0; k < BK; ++k)
            cp_async16(s0 + k * (NC_LD * 8), k < krem ? p + (int64_t)k * ld : src,
                       k < krem ? 16 : 0);
        }
      }
    }
  }
}

template <bool TA, bool TB, bool BULK>
__device__ __forceinline__ void produce(const Ring& ring, const TileRec* __restrict__ tiles,
                                        int ntiles, const Seg* __restrict__ segs,
                                        int* __restrict__ counter, double* const* sbases,
                                        int lane, int role, volatile int* s_next) {
  // role 0: the only producer; 1: A loader + tile-queue leader; 2: B loader
  const bool load_a = role != 2, load_b = role != 1, leader = role != 2;
  constexpr int A_EL = a_elems<TA>();
  constexpr uint32_t STAGE_B = stage_elems<TA, TB>() * 8;
  // lane 0 writes the stage metadata; the arrive publishes it (release)
  auto meta_write = [&](int stage, int nks, double scale, int flags, const TileRec& tr,
                        double* cptr) {
    if (lane == 0 && leader) {
      StageMeta& m = ring.meta[stage];
      m.nks = nks;
      m.scale = scale;
      m.flags = flags;
      if (flags & kFirst) {
        m.c = cptr;
        m.ldc = tr.ldc;
        m.beta = tr.beta;
        m.tm = tr.tm;
        m.tn = tr.tn;
      }
    }
  };
  auto publish_empty = [&](int stage) {  // a stage without operand data
    __syncwarp();
    mbar_arrive_cp_async(ring.full0 + 8 * stage);
    if (lane == 0 && leader) mbar_arrive(ring.full0 + 8 * stage);
  };
  // tile indices: the leader claims, a follower reads them from s_next
  auto share = [&](int& v, int slot) {
    if (PRODUCERS == 1) return;
    if (role == 1 && lane == 0) s_next[slot] = v;
    asm volatile("bar.sync 1, 64;\n" ::: "memory");
    if (role == 2) v = s_next[slot];
    asm volatile("bar.sync 1, 64;\n" ::: "memory");
  };
  int stage = 0;
  uint32_t phase = 0;
  // Tile queue with two tiles of lookahead: the index of tile i+2 is claimed
  // while tile i streams and its descriptor is loaded at the end of tile i, so
  // neither the atomic nor the dependent descriptor load sits on the path
  // between two tiles (consumers measured waiting at tile starts otherwise).
  int t = 0, t1 = 0;
  if (lane == 0 && leader) {
    t = atomicAdd(counter, 1);
    t1 = atomicAdd(counter, 1);
  }
  t = __shfl_sync(0xffffffffu, t, 0);
  t1 = __shfl_sync(0xffffffffu, t1, 0);
  share(t, 0);
  share(t1, 1);
  TileRec cur{}, nrec{};
  Seg sn{};                       // prefetched next segment descriptor
  if (t < ntiles) {
    cur = tiles[t];
    if (cur.seg_begin < cur.seg_end) sn = segs[cur.seg_begin];
  }
  if (t1 < ntiles) nrec = tiles[t1];
  while (t < ntiles) {
    int t2 = 0;
    if (lane == 0 && leader) t2 = atomicAdd(counter, 1);  // resolved by the tile's end
    const int next = t1;
    double* cptr = sbases[cur.c >> kHandleShift] + (cur.c & kHandleMask) +
                   (int64_t)cur.row0 * cur.ldc + cur.col0;
    if (cur.seg_begin == cur.seg_end) {
      // no K at all: C = beta * C (one empty stage carries the epilogue)
      mbar_wait(ring.empty0 + 8 * stage, phase ^ 1);
      meta_write(stage, 0, 1.0, kFirst | kLast, cur, cptr);
      publish_empty(stage);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
      if (next < ntiles && nrec.seg_begin < nrec.seg_end) sn = segs[nrec.seg_begin];
    }
    bool first = true;
    for (int s = cur.seg_begin; s < cur.seg_end; ++s) {
      const Seg sg = sn;
      if (s + 1 < cur.seg_end) sn = segs[s + 1];
      else if (next < ntiles && nrec.seg_begin < nrec.seg_end) sn = segs[nrec.seg_begin];
      const double* a = sbases[sg.a >> kHandleShift] + (sg.a & kHandleMask);
      const double* b = sbases[sg.b >> kHandleShift] + (sg.b & kHandleMask);
      // operand origins at this tile: A rows row0.., B cols col0..
      a += TA ? cur.row0 : (int64_t)cur.row0 * sg.lda;
      const bool btiled = !TB && BULK && sg.btile > 0;
      if (btiled) b += (int64_t)(cur.col0 / cur.colw) * sg.btile * NC_LD_B;
      else b += TB ? (int64_t)cur.col0 * sg.ldb : cur.col0;
      for (int k0 = 0; k0 < sg.k; k0 += BK) {
        const int krem = min(BK, sg.k - k0);
        mbar_wait(ring.empty0 + 8 * stage, phase ^ 1);
        const uint32_t sa = ring.smem + stage * STAGE_B;
        const uint32_t sb = sa + A_EL * 8;
        const uint32_t full = ring.full0 + 8 * stage;
        const bool last = (s + 1 == cur.seg_end) && (k0 + BK >= sg.k);
        meta_write(stage, steps_for(krem), sg.scale, (first ? kFirst : 0) | (last ? kLast : 0),
                   cur, cptr);
        // A: K-contig iff !TA (element (r,k) at a + r*lda + k); B: K-contig iff TB
        const double* asrc = TA ? a + (int64_t)k0 * sg.lda : a + k0;
        const double* bsrc = TB ? b + k0 : b + (int64_t)k0 * sg.ldb;
#ifndef SDMRG_EXP_NOLOAD
        if (btiled) {
          // the whole B stage is one contiguous [16][NC_LD_B] run: lane 0
          // registers its bytes and issues one TMA-unit bulk copy (its
          // expect_tx arrive stands in for the meta arrive)
          __syncwarp();
          if (lane == 0 && load_b) {
            mbar_arrive_expect_tx(full, BK * NC_LD_B * 8);
            bulk_copy(sb, bsrc, BK * NC_LD_B * 8, full);
          }
          if (load_a) load_operand_aligned<!TA, NC_LD_A, BM>(sa, asrc, sg.lda, cur.tm, krem, lane);
        } else if (BULK) {
          if (load_a) load_operand_aligned<!TA, NC_LD_A, BM>(sa, asrc, sg.lda, cur.tm, krem, lane);
          if (load_b) load_operand_aligned<TB, NC_LD_B, BN>(sb, bsrc, sg.ldb, cur.tn, krem, lane);
        } else {
          if (load_a) load_operand_async<!TA, NC_LD_A, BM>(sa, asrc, sg.lda, cur.tm, krem, lane);
          if (load_b) load_operand_async<TB, NC_LD_B, BN>(sb, bsrc, sg.ldb, cur.tn, krem, lane);
        }
#endif
        __syncwarp();
        mbar_arrive_cp_async(full);
        if (lane == 0 && leader && !btiled) mbar_arrive(full);
        first = false;
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    t2 = __shfl_sync(0xffffffffu, t2, 0);
    share(t2, 0);
    TileRec n2{};
    if (t2 < ntiles) n2 = tiles[t2];
    t = next;
    cur = nrec;
    nrec = n2;
    t1 = t2;
  }
  mbar_wait(ring.empty0 + 8 * stage, phase ^ 1);
  meta_write(stage, 0, 1.0, kEnd, cur, nullptr);
  publish_empty(stage);
}

// BULK ("aligned"): every operand block 16-byte aligned with even leading
// dimensions (the H_eff plan's padded layouts) -> 16-byte cp.async; the
// launcher selects it per batch.
#if SDMRG_BIG
#define SDMRG_KERNEL_BOUNDS __launch_bounds__(THREADS, 1)
#else
#define SDMRG_KERNEL_BOUNDS __launch_bounds__(THREADS, SDMRG_MINB)
#endif
// ONE: single always-scaling consumer body (see one_body_default)
template <bool TA, bool TB, bool BULK, bool ONE = false>
__global__ void SDMRG_KERNEL_BOUNDS
seg_gemm_kernel(const TileRec* __restrict__ tiles, int ntiles, const Seg* __restrict__ segs,
                int* __restrict__ counter, Bases bases) {
  extern __shared__ __align__(128) double smem[];
  constexpr int A_EL = a_elems<TA>();
  StageMeta* meta = reinterpret_cast<StageMeta*>(smem + STAGES * stage_elems<TA, TB>());
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta + STAGES);   // full[STAGES], empty[STAGES]
  double** sbases = reinterpret_cast<double**>(bars + 2 * STAGES);
  volatile int* s_next = reinterpret_cast<volatile int*>(sbases + kMaxBases);
  Ring ring;
  ring.smem = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  ring.full0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
  ring.empty0 = ring.full0 + STAGES * 8;
  ring.meta = meta;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < kMaxBases; ++k) sbases[k] = bases.p[k];
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(ring.full0 + 8 * s, 32 * PRODUCERS + 1);  // cp.async arrivals + meta arrive
      mbar_init(ring.empty0 + 8 * s, CONSUMERS);  // one arrive per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= CONSUMERS) {
    const int role = PRODUCERS == 1 ? 0 : (warp == CONSUMERS ? 1 : 2);
    produce<TA, TB, BULK>(ring, tiles, ntiles, segs, counter, sbases, lane, role, s_next);
    return;
  }

  // ================================================================ consumers
  const int lr = lane >> 2, lc = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  // Warp roles rotate per tile (SDMRG_ROTATE): the balanced split of an odd
  // block count gives role 0 the most blocks, and warp w of every CTA tends
  // to sit on the same SM sub-partition (one FP64 pipe each) — rotating the
  // roles spreads the heavy share over the four pipes.
  int rot = SDMRG_ROTATE ? static_cast<int>(blockIdx.x) : 0;
  while (true) {
    mbar_wait(ring.full0 + 8 * stage, phase);
    const StageMeta& m = meta[stage];
    if (m.flags & kEnd) break;
    const int vw = SDMRG_ROTATE ? (warp + rot) % CONSUMERS : warp;
    rot += 1;
    const int wr = vw / WGRID_C, wc = vw % WGRID_C;
    // first stage of a tile: balanced 2 x 2 warp split of its 8x8 blocks
    const int tm = m.tm, tn = m.tn;
    const int mb = (tm + 7) >> 3, nb = (tn + 7) >> 3;
    int mblk, nblk, wr0, wc0;
    if (grid_adapt<TB>() && CONSUMERS == 4 && (mb & 1) && (nb & 3) == 0 && mb <= 8 && nb <= 8) {
      // odd block rows: a 2 x 2 split would give 4:3 row blocks; four warps
      // side by side over all rows balance exactly (1 x 4 grid)
      mblk = mb;
      wr0 = 0;
      nblk = nb >> 2;
      wc0 = 8 * nblk * cw_index(wr, wc);
    } else if (grid_adapt<TB>() && CONSUMERS == 4 && (nb & 1) && (mb & 3) == 0 && nb <= 8 && mb <= 8) {
      nblk = nb;  // odd block columns: 4 x 1 grid
      wc0 = 0;
      mblk = mb >> 2;
      wr0 = 8 * mblk * cw_index(wr, wc);
    } else if (WGRID_R == 2) {
      const int mb0 = (mb + 1) >> 1;
      mblk = wr == 0 ? mb0 : mb - mb0;
      wr0 = wr == 0 ? 0 : mb0 * 8;
      // columns: balanced over WGRID_C warps
      const int nbase = nb / WGRID_C, nextra = nb - nbase * WGRID_C;
      nblk = nbase + (wc < nextra ? 1 : 0);
      wc0 = 8 * (wc * nbase + min(wc, nextra));
    } else {
      // rows and columns balanced over the WGRID_R x WGRID_C grid
      const int mbase = mb / WGRID_R, mextra = mb - mbase * WGRID_R;
      mblk = mbase + (wr < mextra ? 1 : 0);
      wr0 = 8 * (wr * mbase + min(wr, mextra));
      // columns: balanced over WGRID_C warps
      const int nbase = nb / WGRID_C, nextra = nb - nbase * WGRID_C;
      nblk = nbase + (wc < nextra ? 1 : 0);
      wc0 = 8 * (wc * nbase + min(wc, nextra));
    }
    // fragment origin: stage k = lc (natural order) or 2 lc (kperm)
    const int kf = lc;
    const uint32_t a_off = TA ? (kf * NC_LD_A + wr0 + lr) * 8 : ((wr0 + lr) * KC_LD + kf) * 8;
    const uint32_t b_off =
        A_EL * 8 + (TB ? ((wc0 + lr) * KC_LD + kf) * 8 : (kf * NC_LD_B + wc0 + lr) * 8);
    double* c = m.c + (int64_t)(wr0 + lr) * m.ldc + wc0 + 2 * lc;
    consume_dispatch<TA, TB, ONE>(mblk, nblk, ring, stage, phase, a_off, b_off, c, m.ldc,
                                  m.beta, tm - wr0 - lr, tn - wc0 - 2 * lc, lane);
  }
}

}  // namespace sdmrg
