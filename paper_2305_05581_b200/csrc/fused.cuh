// fused.cuh — the fused small-sector H_eff·ψ kernel: both engine phases of
// one σ tile in one CTA, the intermediate T never leaving the registers.
//
// For a σ block o (q x r) the two-phase plan computes
//     T(i, b)  = ψ_i R_b^T                      (phase 1, m x r, to HBM)
//     σ_o     += Σ_(i, b) s · L(g, b) T(i, b)    (phase 2, reads T back)
// and T is written and re-read once per use: at L=76 D=4096 that is 150 GB
// of T per H_eff·ψ against 1.4 TFLOP of phase-2 math (each T block is used
// by ~1.1 groups), so the two-phase path streams ~500 GB on small sectors.
// This kernel evaluates the same sum per σ tile in the transposed form
//     σ_o^T[r-tile, :] += Σ  (R_b[r-tile, :] ψ_i^T) · (s L^T)
// chained in registers: a warp computes T^T = R_b ψ_i^T for its 8 rows of
// the r-tile (8 σ columns) and the 8-column blocks j of m it owns into DMMA
// accumulators, and those accumulators ARE the A fragments of the second
// product (DMMA C layout: lane holds T^T[row lr][cols 2lc, 2lc+1]; taking the
// k order of a k4 step as the column pair (8j + 2lc + e, e = 0/1) makes
// element e of every accumulator the A fragment of step e).  The B fragments
// of the second product are L[q][8j + 2lc + e] — one 16-byte shared load
// gives both steps.
//
// Work split (CTA = 4 DMMA warps + 2 producer warps, 2 CTAs per SM): a tile
// is one σ problem's q rows x R = 4, 2 or 1 column blocks (r is cut
// 4 + 4 + ... + 2 + 1).  Warp w owns column block w / S of the tile, S = 4 / R,
// and of each product the m blocks j with (j + g) mod S == w mod S (g: the
// tile's running block count, so the deal rotates across products).  R = 4:
// every warp owns all of m and its own σ^T rows — no reduction; R = 2 / 1:
// the S warps of a column block sum their partial σ^T in a fixed order at
// the tile's end (deterministic, no atomics).  Accumulators per thread:
// σ^T QB x 2 and T^T (8 / S) x 2 doubles — small enough for 2 CTAs (8 DMMA
// warps) per SM: one DMMA warp per sub-partition cannot keep its FP64 pipe
// busy (ncu r2f of the one-CTA variant: 29% DMMA-pipe activity, the stall
// on the NOP that follows each DMMA).
//
// Pipeline: the warp-specialized ring of engine.cuh (16-byte cp.async with
// mbarrier completion), stage kinds:
//   STEP1  R_b[8R rows][32 n-cols] + ψ_i[8 mb rows][32 n-cols]
//   COPY   ψ_i[8 mb rows][r-tile cols]            (identity R: T = ψ_i)
//   LHALF  L[q rows][32 m-cols]  (one per 32 columns of m)
// Zero fill: every k (n) tail, the ψ rows [m, 8 mb) and the L columns
// [m, 32) of a half are zero-filled by the copies (so the padded T^T columns
// are exactly zero); rows of R beyond the tile and of L beyond q only feed
// accumulator rows / columns the epilogue never stores.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "engine.cuh"

namespace sdmrg {

struct FTileRec {     // 32 B
  uint64_t c;         // handle of C(0, r0) — the tile's first σ column
  int32_t ldc, beta;
  int32_t seg_begin, seg_end;
  int16_t q, rt;      // rows (all of the σ block), columns of this tile
  int32_t r0;         // column offset of the tile inside its σ block
};
struct FSeg {         // 48 B: one (ψ key, right op) product of a σ problem
  uint64_t psi;       // ψ_i(0, 0), padded: m x n, ld pad2(n)
  uint64_t rb;        // R_b(0, 0) in the padded right arena: r x n, ld pad2(n)
  uint64_t l;         // L / Lsum (0, 0): q x m, ld pad2(m)
  int32_t m, n;
  int32_t ident;      // 1: R_b is the identity (T = ψ_i, r = n)
  int32_t pad;
  double scale;
};

constexpr int FKC = 32;             // n columns per STEP1 stage
constexpr int FKLD = FKC + 4;       // K-contiguous row stride (≡ 4 mod 16: the 16 lanes of an
                                    // LDS.64 phase (rows lr, k lc) hit 16 distinct bank pairs)
constexpr int F_RT = 4;             // <= 4 column blocks per tile (32 σ columns)
constexpr int F_QB = 8;             // q <= 64
constexpr int F_MB = 8;             // m <= 64
constexpr int FLLD = 32 + 8;        // L half row stride (≡ 8 mod 16: conflict-free LDS.128)
constexpr int FCLD = 8 * F_RT + 2;  // COPY row stride (≡ 2 mod 16)
constexpr int F_A_EL = 8 * F_RT * FKLD;
constexpr int F_STAGE_EL = F_A_EL + 8 * F_MB * FKLD;
static_assert(8 * F_QB * FLLD <= F_STAGE_EL, "L half fits a stage");
static_assert(8 * F_MB * FCLD <= F_STAGE_EL, "COPY stage fits a stage");
#ifndef SDMRG_FMINB
#define SDMRG_FMINB 2
#endif
#ifndef SDMRG_FSTAGES
#define SDMRG_FSTAGES 3
#endif
constexpr int FSTAGES = SDMRG_FSTAGES;
constexpr int F_SLD = 8 * F_QB + 8;                   // reduction scratch row stride (≡ 8 mod 16)
constexpr int F_SCRATCH_EL = 4 * 8 * F_SLD;           // one 8 x 64 σ^T slab per column block
#ifndef SDMRG_FPRODUCERS
#define SDMRG_FPRODUCERS 2
#endif
constexpr int F_PRODUCERS = SDMRG_FPRODUCERS;
constexpr int F_THREADS = 32 * (4 + F_PRODUCERS);

struct FMeta {
  double* c;
  double scale;
  int32_t type;      // 1 STEP1, 2 LHALF, 3 COPY
  int32_t nks;       // STEP1: k4 steps in the stage
  int32_t mb;        // m blocks of the stage's product
  int32_t half;      // LHALF: which 32 columns of m
  int32_t flags;     // kFirst / kLast / kEnd / kSegEnd
  int32_t ldc, beta;
  int16_t q, rt;
};
constexpr int kSegEnd = 16;

__host__ __device__ constexpr int fused_smem_bytes() {
  return FSTAGES * F_STAGE_EL * 8 + F_SCRATCH_EL * 8 + FSTAGES * (int)sizeof(FMeta) +
         2 * FSTAGES * 8 + kMaxBases * 8 + 16;
}

__host__ __device__ inline int pad2d(int x) { return x + (x & 1); }

// Column blocks per tile: 4, then 2 and 1 for the remainder (each tile keeps
// all four DMMA warps busy: R = 2 / 1 split m between 2 / 4 warps).
__host__ __device__ inline int fused_tile_blocks(int remaining_blocks) {
  return remaining_blocks >= 4 ? 4 : (remaining_blocks >= 2 ? 2 : 1);
}

// The kernel itself is compiled in fused.cu only (runtime.h includes the
// descriptor types above).
#ifdef SDMRG_FUSED_KERNEL
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// ------------------------------------------------------------------ consumer
// One warp's part of one σ tile: column block a = w / S of the tile, m
// blocks dealt S-ways; QB row blocks of σ.  Runs the tile's stages, then the
// ordered S-way reduction and the (transposing) epilogue.
template <int S>
__device__ __forceinline__ void fused_tile(const Ring& ring, int& stage, uint32_t& phase, int w,
                                           int lane, double* scratch) {
  // one body per m-split S (three in all): the σ row-block count qb and the
  // owned m-block count are warp-uniform runtime guards around unrolled
  // loops, not template parameters — 24 shape bodies (r2g) spent 30% of the
  // stall samples on instruction-cache misses
  constexpr int QB = F_QB;
  constexpr int J = 8 / S;            // max m blocks this warp owns per product
  const int lr = lane >> 2, lc = lane & 3;
  const int a = w / S, p = w % S;
  double sacc[QB][2];
  double tt[J][2];
#pragma unroll
  for (int c = 0; c < QB; ++c) sacc[c][0] = sacc[c][1] = 0.0;
#pragma unroll
  for (int j = 0; j < J; ++j) tt[j][0] = tt[j][1] = 0.0;
  const FMeta& first = reinterpret_cast<const FMeta*>(ring.meta)[stage];
  double* const cbase = first.c;
  const int ldc = first.ldc, beta = first.beta, q = first.q, rt = first.rt;
  const int qb = (q + 7) >> 3;
  int g = 0;  // m blocks dealt so far in this tile (per-tile: bitwise determinism)
  constexpr uint32_t STAGE_B = F_STAGE_EL * 8;
  while (true) {
    const FMeta& m = reinterpret_cast<const FMeta*>(ring.meta)[stage];
    const int type = m.type, flags = m.flags, mb = m.mb;
    const uint32_t sa = ring.smem + stage * STAGE_B;
    // owned blocks of this product: j = j0 + S x, x < nj
    const int j0 = (p - g) & (S - 1);
    const int nj = j0 < mb ? (mb - j0 + S - 1) / S : 0;
    if (type == 1) {
      // T^T[8a + lr][8j + ·] += R[8a + lr][k] ψ[8j + ·][k], k4 steps of 32 n
      const int nks = m.nks;
      const uint32_t pa = sa + ((8 * a + lr) * FKLD + lc) * 8;
      const uint32_t pb = sa + F_A_EL * 8 + ((8 * j0 + lr) * FKLD + lc) * 8;
#pragma unroll 2
      for (int ks = 0; ks < nks; ++ks) {
        const double af = lds64(pa + 4 * ks * 8);
#pragma unroll
        for (int x = 0; x < J; ++x)
          if (x < nj) dmma(tt[x], af, lds64(pb + (8 * S * x * FKLD + 4 * ks) * 8));
      }
    } else if (type == 3) {
      // identity R: T^T[8a + lr][8j + 2lc + e] = ψ[8j + 2lc + e][8a + lr]
#pragma unroll
      for (int x = 0; x < J; ++x) {
        if (x < nj) {
          const uint32_t pc = sa + ((8 * (j0 + S * x) + 2 * lc) * FCLD + 8 * a + lr) * 8;
          tt[x][0] = lds64(pc);
          tt[x][1] = lds64(pc + FCLD * 8);
        }
      }
    } else {
      // σ^T[8a + lr][8c + ·] += s T^T[8a + lr][8j + 2lc + e] L[8c + ·][8j + 2lc + e]
      // for the owned blocks j inside this 32-column half of m
      const int h = m.half;
      const double s = m.scale;
      const bool scaled = __double_as_longlong(s) != 0x3FF0000000000000LL;
#pragma unroll
      for (int x = 0; x < J; ++x) {
        const int j = j0 + S * x;
        if (x < nj && j >= 4 * h && j < 4 * h + 4) {
          if (scaled) {
            tt[x][0] *= s;
            tt[x][1] *= s;
          }
          const uint32_t pl = sa + (lr * FLLD + 8 * (j - 4 * h) + 2 * lc) * 8;
#pragma unroll
          for (int c = 0; c < QB; ++c) {
            if (c < qb) {
              double b0, b1;
              lds128(pl + 8 * c * FLLD * 8, b0, b1);
              dmma(sacc[c], tt[x][0], b0);
              dmma(sacc[c], tt[x][1], b1);
            }
          }
        }
      }
      if (flags & kSegEnd) {
#pragma unroll
        for (int x = 0; x < J; ++x) tt[x][0] = tt[x][1] = 0.0;
        g += mb;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(ring.empty0 + 8 * stage);
    if (++stage == FSTAGES) {
      stage = 0;
      phase ^= 1;
    }
    if (flags & kLast) break;
    mbar_wait(ring.full0 + 8 * stage, phase);
  }
  // epilogue: the S warps of column block a sum their partial σ^T rows in
  // order p = 0 .. S-1 through a scratch slab; the last writes σ (transposed)
  const int col = 8 * a + lr;
  auto store = [&]() {
    if (col < rt) {
#pragma unroll
      for (int c = 0; c < QB; ++c) {
        const int row = 8 * c + 2 * lc;
        double* p0 = cbase + (int64_t)row * ldc + col;
        if (row < q) *p0 = beta ? *p0 + sacc[c][0] : sacc[c][0];
        if (row + 1 < q) p0[ldc] = beta ? p0[ldc] + sacc[c][1] : sacc[c][1];
      }
    }
  };
  if constexpr (S == 1) {
    store();
  } else {
    const uint32_t sp = static_cast<uint32_t>(__cvta_generic_to_shared(scratch)) +
                        ((a * 8 + lr) * F_SLD + 2 * lc) * 8;
#pragma unroll 1
    for (int step = 0; step < S; ++step) {
      if (p == step) {
        if (step > 0) {
#pragma unroll
          for (int c = 0; c < QB; ++c) {
            double u, v;
            lds128(sp + 8 * c * 8, u, v);
            sacc[c][0] += u;
            sacc[c][1] += v;
          }
        }
        if (step + 1 < S) {
#pragma unroll
          for (int c = 0; c < QB; ++c)
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(sp + 8 * c * 8),
                         "d"(sacc[c][0]), "d"(sacc[c][1])
                         : "memory");
        } else {
          store();
        }
      }
      named_bar(1, 128);
    }
  }
}

// ------------------------------------------------------------------ producer
// F_PRODUCERS warps share every stage's copies (row r -> warp (r / 2) mod
// F_PRODUCERS).  16-byte copies of `rows` rows x 32 K-columns of a
// row-major source (ld even, column offset even), zero-filling columns >=
// kvalid and rows >= rvalid; destination row stride LD.
template <int LD>
__device__ __forceinline__ void f_load_rows32(uint32_t sdst, const double* src, int ld, int rows,
                                              int rvalid, int kvalid, int lane, int pw) {
  const int kp = lane & 15, k = 2 * kp;
  const int bytes = k + 1 < kvalid ? 16 : (k < kvalid ? 8 : 0);
  for (int r = (lane >> 4) + 2 * pw; r < rows; r += 2 * F_PRODUCERS) {
    const bool ok = r < rvalid && bytes > 0;
    cp_async16(sdst + (r * LD + k) * 8, ok ? src + (int64_t)r * ld + k : src, ok ? bytes : 0);
  }
}

__device__ __forceinline__ void fused_produce(const Ring& ring, const FTileRec* __restrict__ tiles,
                                              int ntiles, const FSeg* __restrict__ segs,
                                              int* __restrict__ counter, double* const* sbases,
                                              int lane, int pw, volatile int* s_tile) {
  FMeta* meta = reinterpret_cast<FMeta*>(ring.meta);
  const bool lead = pw == 0 && lane == 0;
  int stage = 0;
  uint32_t phase = 0;
  auto open = [&]() { mbar_wait(ring.empty0 + 8 * stage, phase ^ 1); };
  auto close = [&]() {
    __syncwarp();
    mbar_arrive_cp_async(ring.full0 + 8 * stage);
    if (lead) mbar_arrive(ring.full0 + 8 * stage);
    if (++stage == FSTAGES) {
      stage = 0;
      phase ^= 1;
    }
  };
  auto res = [&](uint64_t h) { return sbases[h >> kHandleShift] + (h & kHandleMask); };
  // tile queue: the lead claims, the producer warps read it after a named
  // barrier (slots alternate, so a slot is rewritten only after every warp
  // has passed the next barrier)
  int par = 0;
  auto next_tile = [&]() {
    if (lead) s_tile[par] = atomicAdd(counter, 1);
    named_bar(2, 32 * F_PRODUCERS);
    const int v = s_tile[par];
    par ^= 1;
    return v;
  };
  int t = next_tile();
  while (t < ntiles) {
    const FTileRec tr = tiles[t];
    double* cptr = res(tr.c);
    bool first = true;
    FSeg sn = segs[tr.seg_begin];
    for (int s = tr.seg_begin; s < tr.seg_end; ++s) {
      const FSeg sg = sn;
      if (s + 1 < tr.seg_end) sn = segs[s + 1];
      const int m = sg.m, n = sg.n, mb = (m + 7) >> 3;
      const bool last_seg = s + 1 == tr.seg_end;
      const double* psi = res(sg.psi);
      auto meta_write = [&](int type, int nks, int half, int flags) {
        if (lead) {
          FMeta& mt = meta[stage];
          mt.type = type;
          mt.nks = nks;
          mt.mb = mb;
          mt.half = half;
          mt.scale = sg.scale;
          mt.flags = flags | (first ? kFirst : 0);
          if (first) {
            mt.c = cptr;
            mt.ldc = tr.ldc;
            mt.beta = tr.beta;
            mt.q = tr.q;
            mt.rt = tr.rt;
          }
        }
        first = false;
      };
      if (!sg.ident) {
        const double* rb = res(sg.rb) + (int64_t)tr.r0 * pad2d(n);
        for (int c0 = 0; c0 < n; c0 += FKC) {
          open();
          const uint32_t st = ring.smem + stage * (F_STAGE_EL * 8);
          const int kv = n - c0;
          meta_write(1, (min(FKC, kv) + 3) >> 2, 0, 0);
          f_load_rows32<FKLD>(st, rb + c0, pad2d(n), tr.rt, tr.rt, kv, lane, pw);
          f_load_rows32<FKLD>(st + F_A_EL * 8, psi + c0, pad2d(n), 8 * mb, m, kv, lane, pw);
          close();
        }
      } else {
        open();
        const uint32_t st = ring.smem + stage * (F_STAGE_EL * 8);
        meta_write(3, 0, 0, 0);
        // ψ rows [0, 8 mb) x columns [r0, r0 + rt) (pairs; ψ's pad column
        // keeps an odd last pair in bounds), rows >= m zero
        const int npair = (tr.rt + 1) >> 1;
        const double* p0 = psi + tr.r0;
        for (int x = lane + 32 * pw; x < 8 * mb * npair; x += 32 * F_PRODUCERS) {
          const int r = x / npair, cp = x - r * npair;
          const bool ok = r < m;
          cp_async16(st + (r * FCLD + 2 * cp) * 8, ok ? p0 + (int64_t)r * pad2d(n) + 2 * cp : p0,
                     ok ? 16 : 0);
        }
        close();
      }
      const double* l = res(sg.l);
      for (int h = 0; 32 * h < m; ++h) {
        open();
        const uint32_t st = ring.smem + stage * (F_STAGE_EL * 8);
        const bool seg_end = 32 * (h + 1) >= m;
        meta_write(2, 0, h, (seg_end ? kSegEnd : 0) | (seg_end && last_seg ? kLast : 0));
        f_load_rows32<FLLD>(st, l + 32 * h, pad2d(m), tr.q, tr.q, m - 32 * h, lane, pw);
        close();
      }
    }
    t = next_tile();
  }
  open();
  if (lead) meta[stage].flags = kEnd;
  close();
}

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(F_THREADS, SDMRG_FMINB)
fused_heff_kernel(const FTileRec* __restrict__ tiles, int ntiles, const FSeg* __restrict__ segs,
                  int* __restrict__ counter, Bases bases) {
  extern __shared__ __align__(128) double smem[];
  double* scratch = smem + FSTAGES * F_STAGE_EL;
  FMeta* meta = reinterpret_cast<FMeta*>(scratch + F_SCRATCH_EL);
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta + FSTAGES);
  double** sbases = reinterpret_cast<double**>(bars + 2 * FSTAGES);
  volatile int* s_tile = reinterpret_cast<volatile int*>(sbases + kMaxBases);
  Ring ring;
  ring.smem = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  ring.full0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
  ring.empty0 = ring.full0 + FSTAGES * 8;
  ring.meta = reinterpret_cast<StageMeta*>(meta);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < kMaxBases; ++k) sbases[k] = bases.p[k];
    for (int s = 0; s < FSTAGES; ++s) {
      mbar_init(ring.full0 + 8 * s, 32 * F_PRODUCERS + 1);
      mbar_init(ring.empty0 + 8 * s, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp >= 4) {
    fused_produce(ring, tiles, ntiles, segs, counter, sbases, lane, warp - 4, s_tile);
    return;
  }
  const int w = warp;
  int stage = 0;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(ring.full0 + 8 * stage, phase);
    const FMeta& m = meta[stage];
    if (m.flags & kEnd) break;
    const int rtb = (m.rt + 7) >> 3;
    switch (4 / fused_tile_blocks(rtb)) {   // m-split factor S
      case 1: fused_tile<1>(ring, stage, phase, w, lane, scratch); break;
      case 2: fused_tile<2>(ring, stage, phase, w, lane, scratch); break;
      default: fused_tile<4>(ring, stage, phase, w, lane, scratch); break;
    }
  }
}
#endif  // SDMRG_FUSED_KERNEL

}  // namespace sdmrg
