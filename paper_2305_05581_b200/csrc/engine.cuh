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
struct TileRec {     // 48 B
  uint64_t c;        // handle of C(0,0) of the problem
  int32_t ldc, beta;
  int32_t seg_begin, seg_end;
  int32_t row0, col0;
  int16_t tm, tn;
  int32_t colw;      // column-tile width of the problem (stage-tiled B)
  int32_t sib_slot;  // SDMRG_LOCKSTEP: first progress slot of the problem's tiles
  int16_t nsib, sib; // tiles of the problem, this tile's index among them
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
#define SDMRG_STAGES (SDMRG_BIG ? 5 : (SDMRG_WIDE ? 4 : 3))
#endif
#ifndef SDMRG_TILE
#define SDMRG_TILE 64
#endif
#ifndef SDMRG_DB
#define SDMRG_DB 0
#endif
#ifndef SDMRG_STCS
#define SDMRG_STCS 0
#endif
// per-tile warp grid: 1 x 4 or 4 x 1 instead of 2 x 2 when a tile has an odd
// number of 8-row (8-column) blocks, so the four DMMA warps stay balanced
#ifndef SDMRG_ROTATE
#define SDMRG_ROTATE 1
#endif
#ifndef SDMRG_LOCKSTEP
#define SDMRG_LOCKSTEP 0
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
// K order inside a stage (same for both operands, so any bijection is
// exact): DMMA k4 step ks, thread column lc reads stage k
//   kperm(ks, lc) = 8 (ks >> 1) + 2 lc + (ks & 1)
// so a thread's k pairs (2lc, 2lc+1) and (8+2lc, 9+2lc) feed steps (0,1) and
// (2,3): one LDS.128 per K-contiguous fragment pair instead of two LDS.64.
// Off by default: parity-exact but measured 2% slower (96.1 vs 94.2 ms).
#ifndef SDMRG_LDS128
#define SDMRG_LDS128 0
#endif
#ifndef SDMRG_MINB
#define SDMRG_MINB (SDMRG_BIG ? 1 : ((SDMRG_TILE > 64 || SDMRG_WIDE) ? 2 : 4))
#endif
// SDMRG_WIDE: 64 x 128 tiles, 8 DMMA warps (2 x 4 grid of <= 32 x 32 warp
// tiles) per CTA, 2 CTAs per SM — the same 16 DMMA warps per SM as the
// default, with half the A-panel re-reads between column tiles.
#ifndef SDMRG_WIDE
#define SDMRG_WIDE 0
#endif
constexpr int BM = SDMRG_TILE, BN = SDMRG_WIDE ? 2 * SDMRG_TILE : SDMRG_TILE, BK = 16;
constexpr int STAGES = SDMRG_STAGES;
constexpr int MAXB = BM / 16;                    // 8x8 blocks per warp and dimension
static_assert(BM == 64 || BM == 96 || (SDMRG_BIG && BM == 128), "tile edge 64, 96 (or 128 big)");
constexpr int WGRID_R = SDMRG_BIG ? 4 : 2, WGRID_C = (SDMRG_WIDE || SDMRG_BIG) ? 4 : 2,
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
  double scale;      // != 1: some k4 step of the stage is scaled
  double kscale[4];  // scale of each k4 step (packed stages: one per segment piece)
  int32_t nks;       // k4 steps in this stage (0: no K, or kEnd)
  int32_t flags;
  int32_t ldc, beta;
  int16_t tm, tn;
  int32_t pad;
};
constexpr int kFirst = 1, kLast = 2, kEnd = 4, kPacked = 8;
// Segment packing (aligned path): a stage's 16 k rows are filled from as many
// consecutive segments of the tile as fit, each starting on a k4 boundary
// with its own scale per k4 step — short segments (small sectors: K = a few
// states) no longer cost one ring stage each (L=30 D=512: 1.5x fewer phase-2
// stages, D=2048: 1.09x).
#ifndef SDMRG_PACK
#define SDMRG_PACK 0
#endif
#ifndef SDMRG_ROUND
#define SDMRG_ROUND 0
#endif
#ifndef SDMRG_PACK_P2
#define SDMRG_PACK_P2 0
#endif
// Measured (profiles/r1_notes.md): packing made phase 2 13-17% slower (and
// 1.8x slower at D=512) even with uniform-scale stages only (SDMRG_PACK=2),
// and phase 1 (one segment per tile) neutral — off by default; build
// variants SDMRG_PACK=1/2 (+ SDMRG_PACK_P2=1 for the phase-2 instance) are
// parity-tested.
template <bool TB>
__host__ __device__ constexpr bool pack_path() {
  return SDMRG_PACK && (TB || SDMRG_PACK_P2);
}
static_assert(!(SDMRG_PACK && (SDMRG_LDS128 || SDMRG_DB)), "packing needs the natural k order");
static_assert(!(SDMRG_SWZ && (SDMRG_PACK || SDMRG_LDS128 || SDMRG_DB)), "swizzle: natural-order bodies only");

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
__host__ __device__ constexpr int steps_for(int krem) {
#if SDMRG_LDS128
  return krem <= 1 ? 1 : krem <= 8 ? 2 : krem <= 9 ? 3 : 4;
#else
  return (krem + 3) >> 2;
#endif
}

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
    // per-k4-step scale (packed stages; an LDS issued with the step's
    // fragment loads); the whole-stage scale otherwise
    const uint32_t ksc_addr = static_cast<uint32_t>(__cvta_generic_to_shared(&m.kscale[0]));
    auto ksc = [&](int ks) { return pack_path<TB>() && SDMRG_PACK == 1 ? lds64(ksc_addr + 8 * ks) : scale; };
    const uint32_t a0 = ring.smem + stage * STAGE_B + a_off;
    const uint32_t b0 = ring.smem + stage * STAGE_B + b_off;
#if SDMRG_DB
static_assert(!SDMRG_LDS128, "double buffering assumes the natural k order");
    if (MB > 0 && NB > 0 && nks > 0) {
      // fragments of k4 step ks+1 loaded (and scaled) around the DMMAs of ks
      const bool scaled = __double_as_longlong(scale) != 0x3FF0000000000000LL;
      double af[2][MB > 0 ? MB : 1], bf[2][NB > 0 ? NB : 1];
      auto load = [&](int ks, int buf) {
#pragma unroll
        for (int i = 0; i < MB; ++i) af[buf][i] = lds64(a0 + ks * A_KS + i * A_I);
#pragma unroll
        for (int j = 0; j < NB; ++j) bf[buf][j] = lds64(b0 + ks * B_KS + j * B_J);
      };
      auto rescale = [&](int buf) {
        if (NB <= MB) {
#pragma unroll
          for (int j = 0; j < NB; ++j) bf[buf][j] *= scale;
        } else {
#pragma unroll
          for (int i = 0; i < MB; ++i) af[buf][i] *= scale;
        }
      };
      load(0, 0);
      if (scaled) rescale(0);
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        if (ks < nks) {
          const int cur = ks & 1, nxt = cur ^ 1;
          const bool more = ks + 1 < BK / 4 && ks + 1 < nks;
          if (more) load(ks + 1, nxt);
#pragma unroll
          for (int i = 0; i < MB; ++i)
#pragma unroll
            for (int j = 0; j < NB; ++j) dmma(acc[i][j], af[cur][i], bf[cur][j]);
          if (more && scaled) rescale(nxt);
        }
      }
    }
#else
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
#if SDMRG_LDS128
        // K-contiguous operands: fragments of steps (2h, 2h+1) in one LDS.128
        // at stage k = 8h + 2lc (a0/b0 point at k = 2lc); M/N-contiguous
        // operands: one LDS.64 per step at stage row kperm(ks, lc)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (2 * h < nks) {
            double ap[MB > 0 ? MB : 1][2], bp[NB > 0 ? NB : 1][2];
#pragma unroll
            for (int i = 0; i < MB; ++i) {
              if (!TA) lds128(a0 + h * 64 + i * A_I, ap[i][0], ap[i][1]);
              else {
                ap[i][0] = lds64(a0 + (8 * h) * NC_LD_A * 8 + i * A_I);
                ap[i][1] = lds64(a0 + (8 * h + 1) * NC_LD_A * 8 + i * A_I);
              }
            }
#pragma unroll
            for (int j = 0; j < NB; ++j) {
              if (TB) lds128(b0 + h * 64 + j * B_J, bp[j][0], bp[j][1]);
              else {
                bp[j][0] = lds64(b0 + (8 * h) * NC_LD_B * 8 + j * B_J);
                bp[j][1] = lds64(b0 + (8 * h + 1) * NC_LD_B * 8 + j * B_J);
              }
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              if (2 * h + e < nks) {
                if (SCALED) {
                  if (NB <= MB) {
#pragma unroll
                    for (int j = 0; j < NB; ++j) bp[j][e] *= scale;
                  } else {
#pragma unroll
                    for (int i = 0; i < MB; ++i) ap[i][e] *= scale;
                  }
                }
#ifndef SDMRG_EXP_NOMMA
#pragma unroll
                for (int i = 0; i < MB; ++i)
#pragma unroll
                  for (int j = 0; j < NB; ++j) dmma(acc[i][j], ap[i][e], bp[j][e]);
#endif
              }
            }
          }
        }
#else
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
          if (ks < nks) {
            double af[MB > 0 ? MB : 1], bf[NB > 0 ? NB : 1];
#pragma unroll
            for (int i = 0; i < MB; ++i) af[i] = lds64(a0 + koff_a(ks) + i * A_I);
#pragma unroll
            for (int j = 0; j < NB; ++j) bf[j] = lds64(b0 + koff_b(ks) + j * B_J);
            if (SCALED) {
              const double sk = ksc(ks);
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
#endif
      };
      if constexpr (ONE) {
        body(std::true_type{});  // unit scales multiply too: half the code
      } else {
        if (scaled) body(std::true_type{});
        else body(std::false_type{});
      }
    }
#endif
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
  if constexpr (ONE && SDMRG_ROUND) {
    switch (mblk * 8 + nblk) {
      SDMRG_TILE_CASE(4, 4) SDMRG_TILE_CASE(4, 2) SDMRG_TILE_CASE(4, 1)
      SDMRG_TILE_CASE(2, 4) SDMRG_TILE_CASE(2, 2) SDMRG_TILE_CASE(2, 1)
      SDMRG_TILE_CASE(1, 4) SDMRG_TILE_CASE(1, 2) SDMRG_TILE_CASE(1, 1)
      default:
        consume_tile<TA, TB, 0, 0, ONE>(ring, stage, phase, a_off, b_off, c, ldc, beta, row_lim,
                                        col_lim, lane);
        break;
    }
    return;
  }
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
#if SDMRG_TILE > 64 && !SDMRG_BIG
    SDMRG_TILE_CASE(6, 6) SDMRG_TILE_CASE(6, 5) SDMRG_TILE_CASE(5, 6) SDMRG_TILE_CASE(5, 5)
    SDMRG_TILE_CASE(6, 4) SDMRG_TILE_CASE(6, 3) SDMRG_TILE_CASE(6, 2) SDMRG_TILE_CASE(6, 1)
    SDMRG_TILE_CASE(5, 4) SDMRG_TILE_CASE(5, 3) SDMRG_TILE_CASE(5, 2) SDMRG_TILE_CASE(5, 1)
    SDMRG_TILE_CASE(4, 6) SDMRG_TILE_CASE(4, 5) SDMRG_TILE_CASE(3, 6) SDMRG_TILE_CASE(3, 5)
    SDMRG_TILE_CASE(2, 6) SDMRG_TILE_CASE(2, 5) SDMRG_TILE_CASE(1, 6) SDMRG_TILE_CASE(1, 5)
#endif
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
// SDMRG_L2HINT: L2 eviction priority per operand (createpolicy +
// cp.async ...L2::cache_hint): the streamed-once operand (phase 2: T,
// written by phase 1 and read by ~1.1 groups) evict-first, the re-used one
// (the operator blocks, each read by many products) evict-last.
#ifndef SDMRG_L2HINT
#define SDMRG_L2HINT 0
#endif
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t p;
  if (keep) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void cp_async16_hint(uint32_t saddr, const double* gmem, int src_bytes,
                                                uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(saddr),
               "l"(gmem), "r"(src_bytes), "l"(pol));
}
template <bool HINT>
__device__ __forceinline__ void cp16(uint32_t saddr, const double* gmem, int src_bytes, uint64_t pol) {
  if (HINT) cp_async16_hint(saddr, gmem, src_bytes, pol);
  else cp_async16(saddr, gmem, src_bytes);
}
template <bool HINT>
__device__ __forceinline__ void cp16_full(uint32_t saddr, const double* gmem, uint64_t pol) {
  if (HINT) cp_async16_hint(saddr, gmem, 16, pol);
  else cp_async16_full(saddr, gmem);
}

template <bool KCONTIG, int NC_LD, int CAP, bool HINT = false>
__device__ __forceinline__ void load_operand_aligned(uint32_t sbase, const double* src, int ld,
                                                     int extent, int krem, int lane,
                                                     uint64_t pol = 0) {
  if (KCONTIG) {
    const int k = 2 * (lane & 7), r0 = lane >> 3;
    const double* p = src + (int64_t)r0 * ld + k;
    // rows r0 + 4i share (r & 3) = r0 & 3: one swizzled column per lane
    const uint32_t s0 = sbase + (r0 * KC_LD + (SDMRG_SWZ ? k ^ (4 * (r0 & 3)) : k)) * 8;
    const int nrow = (extent - r0 + 3) >> 2;
    if (k + 1 < krem) {
#pragma unroll 4
      for (int i = 0; i < nrow; ++i) cp16_full<HINT>(s0 + i * (4 * KC_LD * 8), p + (int64_t)(4 * i) * ld, pol);
    } else {
      const int bytes = k < krem ? 8 : 0;
      const double* q = k < krem ? p : src;
      const int64_t step = k < krem ? 4 * (int64_t)ld : 0;
#pragma unroll 4
      for (int i = 0; i < nrow; ++i) cp16<HINT>(s0 + i * (4 * KC_LD * 8), q + i * step, bytes, pol);
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
          for (int k = 0; k < BK; ++k) cp16_full<HINT>(s0 + k * (NC_LD * 8), p + (int64_t)k * ld, pol);
        } else {
#pragma unroll
          for (int k = 0; k < BK; ++k)
            cp16<HINT>(s0 + k * (NC_LD * 8), k < krem ? p + (int64_t)k * ld : src,
                       k < krem ? 16 : 0, pol);
        }
      }
    }
  }
}

// Packed-stage variant: stage k rows [kb, kb + len) (kb, len multiples of 4)
// from source k rows [0, len), rows >= valid zero-filled; the stage's other
// rows belong to other segments and are not touched.
template <bool KCONTIG, int NC_LD, int CAP>
__device__ __forceinline__ void load_operand_range(uint32_t sbase, const double* src, int ld,
                                                   int extent, int kb, int len, int valid,
                                                   int lane) {
  if (KCONTIG) {
    const int k = 2 * (lane & 7), r0 = lane >> 3;
    if (k < kb || k >= kb + len) return;
    const int kk = k - kb;
    const int bytes = kk + 1 < valid ? 16 : (kk < valid ? 8 : 0);
    const double* p = bytes ? src + (int64_t)r0 * ld + kk : src;
    const int64_t step = bytes ? 4 * (int64_t)ld : 0;
    const uint32_t s0 = sbase + (r0 * KC_LD + k) * 8;
    const int nrow = (extent - r0 + 3) >> 2;
#pragma unroll 4
    for (int i = 0; i < nrow; ++i) cp_async16(s0 + i * (4 * KC_LD * 8), p + i * step, bytes);
  } else {
#pragma unroll
    for (int j = 0; j < (CAP + 63) / 64; ++j) {
      const int c = 2 * lane + 64 * j;
      if (c < extent) {
        const double* p = src + c;
        const uint32_t s0 = sbase + c * 8;
#pragma unroll
        for (int k = 0; k < BK; ++k) {
          const int kk = k - kb;
          if (kk >= 0 && kk < len)
            cp_async16(s0 + k * (NC_LD * 8), kk < valid ? p + (int64_t)kk * ld : src,
                       kk < valid ? 16 : 0);
        }
      }
    }
  }
}

// L2 prefetch of one contiguous element range with a single bulk (TMA-unit)
// prefetch: the range is widened to 16-byte alignment.
__device__ __forceinline__ void bulk_prefetch_l2(const double* first, const double* last) {
  const uint64_t lo = reinterpret_cast<uint64_t>(first) & ~uint64_t(15);
  const uint64_t hi = (reinterpret_cast<uint64_t>(last) + 8 + 15) & ~uint64_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(lo), "r"((uint32_t)(hi - lo))
               : "memory");
}

// Prefetch both operand panels of segment sg for the tile (row0, col0, tm,
// tn) into L2: each panel of a row-major sector block is one address range.
template <bool TA, bool TB>
__device__ __forceinline__ void prefetch_segment(const Seg& sg, const TileRec& tr,
                                                 double* const* sbases) {
  const double* a = sbases[sg.a >> kHandleShift] + (sg.a & kHandleMask);
  const double* b = sbases[sg.b >> kHandleShift] + (sg.b & kHandleMask);
  if (TA) {
    const double* p = a + tr.row0;
    bulk_prefetch_l2(p, p + (int64_t)(sg.k - 1) * sg.lda + tr.tm - 1);
  } else {
    const double* p = a + (int64_t)tr.row0 * sg.lda;
    bulk_prefetch_l2(p, p + (int64_t)(tr.tm - 1) * sg.lda + sg.k - 1);
  }
  if (TB) {
    const double* p = b + (int64_t)tr.col0 * sg.ldb;
    bulk_prefetch_l2(p, p + (int64_t)(tr.tn - 1) * sg.ldb + sg.k - 1);
  } else {
    const double* p = b + tr.col0;
    bulk_prefetch_l2(p, p + (int64_t)(sg.k - 1) * sg.ldb + tr.tn - 1);
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
      if (!(flags & kPacked))
        m.kscale[0] = m.kscale[1] = m.kscale[2] = m.kscale[3] = scale;
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
  // phase 1 (TB): A = ψ (small, L2-resident), B = right operator blocks
  // (re-used by every ψ key of their sector); phase 2: A = operator blocks /
  // pre-sums (re-used), B = T (streamed)
  uint64_t pol_a = 0, pol_b = 0;
  if (SDMRG_L2HINT) {
    pol_a = l2_policy(true);
    pol_b = l2_policy(TB);
  }
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
    // SDMRG_LOCKSTEP: the tiles of one σ problem read the same operand
    // panels (row siblings the same A rows, column siblings the same B
    // columns); a producer more than SDMRG_LOCKSTEP segments ahead of a
    // started, unfinished sibling waits for it, so the shared panels are
    // read while still in L2.  The slowest sibling never waits: no deadlock,
    // and the data flow is untouched (timing only).
    volatile int* prog = reinterpret_cast<volatile int*>(sbases[kMaxBases - 1]);
    const bool lock = SDMRG_LOCKSTEP > 0 && prog != nullptr && cur.nsib > 1;
    if (lock && lane == 0) prog[cur.sib_slot + cur.sib] = 1;
    bool first = true;
    int kfill = 0;           // packed rows in the open stage (multiple of 4)
    double open_scale = 1.0; // SDMRG_PACK == 2: the open stage's (uniform) scale
    bool unit = true;        // every k4 step of the open stage unscaled
    for (int s = cur.seg_begin; s < cur.seg_end; ++s) {
      if (lock) {
        const int k = s - cur.seg_begin;
        if (lane == 0) {
          prog[cur.sib_slot + cur.sib] = k + 1;
          for (int j = 0; j < cur.nsib; ++j) {
            if (j == cur.sib) continue;
            int v = prog[cur.sib_slot + j];
            while (v >= 1 && v < (1 << 30) && v - 1 < k - SDMRG_LOCKSTEP) {
              __nanosleep(256);
              v = prog[cur.sib_slot + j];
            }
          }
        }
        __syncwarp();
      }
      const Seg sg = sn;
      if (s + 1 < cur.seg_end) {
        sn = segs[s + 1];
#ifdef SDMRG_L2_PREFETCH
        if (lane == 0) prefetch_segment<TA, TB>(sn, cur, sbases);
#endif
      } else if (next < ntiles && nrec.seg_begin < nrec.seg_end) {
        sn = segs[nrec.seg_begin];
#ifdef SDMRG_L2_PREFETCH
        if (lane == 0) prefetch_segment<TA, TB>(sn, nrec, sbases);
#endif
      }
      const double* a = sbases[sg.a >> kHandleShift] + (sg.a & kHandleMask);
      const double* b = sbases[sg.b >> kHandleShift] + (sg.b & kHandleMask);
      // operand origins at this tile: A rows row0.., B cols col0..
      a += TA ? cur.row0 : (int64_t)cur.row0 * sg.lda;
      const bool btiled = !TB && BULK && sg.btile > 0;
      if (btiled) b += (int64_t)(cur.col0 / cur.colw) * sg.btile * NC_LD_B;
      else b += TB ? (int64_t)cur.col0 * sg.ldb : cur.col0;
      if (pack_path<TB>() && BULK && !btiled) {
        if (SDMRG_PACK == 2 && kfill > 0 &&
            __double_as_longlong(sg.scale) != __double_as_longlong(open_scale)) {
          // uniform-scale stages: close the open one before a new scale
          meta_write(stage, kfill >> 2, open_scale, (first ? kFirst : 0), cur, cptr);
          __syncwarp();
          mbar_arrive_cp_async(ring.full0 + 8 * stage);
          if (lane == 0 && leader) mbar_arrive(ring.full0 + 8 * stage);
          first = false;
          kfill = 0;
          unit = true;
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        open_scale = sg.scale;
        for (int k0 = 0; k0 < sg.k;) {
          if (kfill == 0) mbar_wait(ring.empty0 + 8 * stage, phase ^ 1);
          const uint32_t sa = ring.smem + stage * STAGE_B;
          const uint32_t sb = sa + A_EL * 8;
          const int valid = min(BK - kfill, sg.k - k0);
          const int len = min(BK - kfill, (sg.k - k0 + 3) & ~3);
          const double* asrc = TA ? a + (int64_t)k0 * sg.lda : a + k0;
          const double* bsrc = TB ? b + k0 : b + (int64_t)k0 * sg.ldb;
#ifndef SDMRG_EXP_NOLOAD
          if (kfill == 0 && len == BK) {
            if (load_a) load_operand_aligned<!TA, NC_LD_A, BM>(sa, asrc, sg.lda, cur.tm, valid, lane);
            if (load_b) load_operand_aligned<TB, NC_LD_B, BN>(sb, bsrc, sg.ldb, cur.tn, valid, lane);
          } else {
            if (load_a)
              load_operand_range<!TA, NC_LD_A, BM>(sa, asrc, sg.lda, cur.tm, kfill, len, valid, lane);
            if (load_b)
              load_operand_range<TB, NC_LD_B, BN>(sb, bsrc, sg.ldb, cur.tn, kfill, len, valid, lane);
          }
#endif
          if (lane == 0 && leader) {
            StageMeta& m = ring.meta[stage];
            for (int q = kfill >> 2; q < (kfill + len) >> 2; ++q) m.kscale[q] = sg.scale;
          }
          unit = unit && __double_as_longlong(sg.scale) == 0x3FF0000000000000LL;
          kfill += len;
          k0 += len;
          const bool last = (s + 1 == cur.seg_end) && k0 >= sg.k;
          if (kfill == BK || last) {
            meta_write(stage, kfill >> 2, SDMRG_PACK == 2 ? open_scale : (unit ? 1.0 : 2.0),
                       (SDMRG_PACK == 2 ? 0 : kPacked) | (first ? kFirst : 0) | (last ? kLast : 0),
                       cur, cptr);
            __syncwarp();
            const uint32_t full = ring.full0 + 8 * stage;
            mbar_arrive_cp_async(full);
            if (lane == 0 && leader) mbar_arrive(full);
            first = false;
            kfill = 0;
            unit = true;
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        continue;
      }
      if (kfill > 0) {
        // a stage-tiled segment after packed ones: close the open stage
        meta_write(stage, kfill >> 2, SDMRG_PACK == 2 ? open_scale : (unit ? 1.0 : 2.0),
                   (SDMRG_PACK == 2 ? 0 : kPacked) | (first ? kFirst : 0), cur, cptr);
        __syncwarp();
        mbar_arrive_cp_async(ring.full0 + 8 * stage);
        if (lane == 0 && leader) mbar_arrive(ring.full0 + 8 * stage);
        first = false;
        kfill = 0;
        unit = true;
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
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
          constexpr bool H = SDMRG_L2HINT != 0;
          if (load_a)
            load_operand_aligned<!TA, NC_LD_A, BM, H>(sa, asrc, sg.lda, cur.tm, krem, lane, pol_a);
          if (load_b)
            load_operand_aligned<TB, NC_LD_B, BN, H>(sb, bsrc, sg.ldb, cur.tn, krem, lane, pol_b);
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
    if (lock && lane == 0) prog[cur.sib_slot + cur.sib] = 1 << 30;  // finished
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
#elif SDMRG_TILE > 64
#define SDMRG_KERNEL_BOUNDS __maxnreg__(200)
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
    const int kf = SDMRG_LDS128 ? 2 * lc : lc;
    const uint32_t a_off = TA ? (kf * NC_LD_A + wr0 + lr) * 8 : ((wr0 + lr) * KC_LD + kf) * 8;
    const uint32_t b_off =
        A_EL * 8 + (TB ? ((wc0 + lr) * KC_LD + kf) * 8 : (kf * NC_LD_B + wc0 + lr) * 8);
    double* c = m.c + (int64_t)(wr0 + lr) * m.ldc + wc0 + 2 * lc;
    if constexpr (ONE && SDMRG_ROUND) {
      // 3 -> 4 blocks (the extra block's DMMAs are discarded: its stores are
      // cut at the warp's own extent): 9 shape bodies instead of 16
      const int re = min(tm - wr0, 8 * mblk) - lr, ce = min(tn - wc0, 8 * nblk) - 2 * lc;
      consume_dispatch<TA, TB, ONE>(mblk == 3 ? 4 : mblk, nblk == 3 ? 4 : nblk, ring, stage, phase,
                                    a_off, b_off, c, m.ldc, m.beta, re, ce, lane);
    } else {
      consume_dispatch<TA, TB, ONE>(mblk, nblk, ring, stage, phase, a_off, b_off, c, m.ldc,
                                    m.beta, tm - wr0 - lr, tn - wc0 - 2 * lc, lane);
    }
  }
}

}  // namespace sdmrg
