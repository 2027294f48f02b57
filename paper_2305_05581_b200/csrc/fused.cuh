// fused.cuh — the fused small-sector H_eff·ψ kernel: both engine phases of
// one σ tile in one CTA, the intermediate T never leaving the registers.
//
// For a σ block o (q x r) the two-phase plan computes
//     T(i, b)  = ψ_i R_b^T                      (phase 1, m x r, to HBM)
//     σ_o     += Σ_(i, b) s · L(g, b) T(i, b)    (phase 2, reads T back)
// and T is written and re-read once per use: at L=76 D=4096 that is 150 GB
// of T per H_eff·ψ against 1.4 TFLOP of phase-2 math (tools: each T block is
// used by ~1.1 groups), so the two-phase path is HBM-bound on small sectors.
// This kernel evaluates the same sum per σ tile in the transposed form
//     σ_o^T[r-tile, :] += Σ  (R_b[r-tile, :] ψ_i^T) · (s L^T)
// chained in registers: a warp computes T^T = R_b ψ_i^T for an 8-column block
// j of T^T (8 ψ rows) into DMMA accumulators, and those accumulators ARE the
// A fragments of the second product (DMMA C layout: lane holds
// T^T[row lr][cols 2lc, 2lc+1]; taking the k order of a k4 step as the
// column pair (8j + 2lc + e, e = 0/1) makes element e of every accumulator
// the A fragment of step e), so T exists only as 2 x RT registers per block.
// The B fragments of the second product are L[q][8j + 2lc + e] — one
// 16-byte shared load gives both steps.
//
// Work split: a CTA owns one σ tile (all q rows, an r-range of <= 40
// columns = RT 8-blocks) and walks its products (the concatenated K of
// SBMM4S, sbmm4s.py:132-165).  The 8-row blocks j of each product's m
// dimension are dealt round-robin to the 4 DMMA warps, continuing across
// products, so the warps stay balanced whatever the sector sizes; each warp
// accumulates a full σ^T tile (RT x QB blocks) and the four partial tiles
// are summed in a fixed order at the tile's end (deterministic, no atomics).
// Identity right operators (T = ψ_i) skip the first product: the A
// fragments are read straight from a staged ψ block.
//
// Pipeline: the same warp-specialized ring as engine.cuh (1 producer warp,
// 16-byte cp.async with mbarrier completion), stage kinds:
//   STEP1  R_b[r-tile rows][64 n-cols] + ψ_i[8 mb rows][64 n-cols]
//   COPY   ψ_i[8 mb rows][r-tile cols]            (identity R)
//   LSTAGE L[q rows][m cols]  (m <= 64: one stage per product)
// Zero fill: every k (n) tail, the ψ rows [m, 8 mb) and the L columns
// [m, 64) are zero-filled by the copies (so the padded T^T columns
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

constexpr int FKC = 64;             // n columns per STEP1 stage
constexpr int FKLD = FKC + 2;       // K-contiguous row stride (≡ 2 mod 16: conflict-free LDS.64)
constexpr int F_RT = 5;             // <= 5 column blocks per tile (40 σ columns)
constexpr int F_QB = 8;             // q <= 64
constexpr int F_MB = 8;             // m <= 64
constexpr int FLLD = 64 + 8;        // L stage row stride (≡ 8 mod 16: conflict-free LDS.128)
constexpr int FCLD = 8 * F_RT + 10; // COPY row stride (≡ 2 mod 16)
constexpr int F_A_EL = 8 * F_RT * FKLD;
constexpr int F_STAGE_EL = F_A_EL + 8 * F_MB * FKLD;
static_assert(8 * F_QB * FLLD <= F_STAGE_EL, "L stage fits a stage");
static_assert(8 * F_MB * FCLD <= F_STAGE_EL, "COPY stage fits a stage");
#ifndef SDMRG_FMINB
#define SDMRG_FMINB 1
#endif
#ifndef SDMRG_FSTAGES
#define SDMRG_FSTAGES 3
#endif
constexpr int FSTAGES = SDMRG_FSTAGES;
constexpr int F_SLD = 8 * F_QB + 2;                   // reduction scratch row stride
constexpr int F_SCRATCH_EL = 8 * F_RT * F_SLD;
#ifndef SDMRG_FPRODUCERS
#define SDMRG_FPRODUCERS 4
#endif
constexpr int F_PRODUCERS = SDMRG_FPRODUCERS;
constexpr int F_THREADS = 32 * (4 + F_PRODUCERS);

struct FMeta {
  double* c;
  double scale;
  int32_t type;      // 1 STEP1, 2 LSTAGE, 3 COPY
  int32_t nks;       // STEP1: k4 steps in the stage
  int32_t mb;        // m blocks of the stage's product
  int32_t half;      // unused
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

// The kernel itself is compiled in fused.cu only (runtime.h includes the
// descriptor types above).
#ifdef SDMRG_FUSED_KERNEL
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}

// ------------------------------------------------------------------ consumer
// One warp's part of one σ tile (RT column blocks, QB row blocks of σ):
// stages until the tile's last, then the ordered 4-warp reduction.
template <int RT, int QB>
__device__ __forceinline__ void fused_tile(const Ring& ring, int& stage, uint32_t& phase, int& g,
                                           int w, int lane, double* scratch) {
  const int lr = lane >> 2, lc = lane & 3;
  double sacc[RT][QB][2];
  double tt[RT][2][2];
#pragma unroll
  for (int a = 0; a < RT; ++a) {
#pragma unroll
    for (int c = 0; c < QB; ++c) sacc[a][c][0] = sacc[a][c][1] = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) tt[a][h][0] = tt[a][h][1] = 0.0;
  }
  const FMeta& first = reinterpret_cast<const FMeta*>(ring.meta)[stage];
  double* const cbase = first.c;
  const int ldc = first.ldc, beta = first.beta, q = first.q, rt = first.rt;
  g = 0;  // per-tile deal: the result depends on the tile only (bitwise determinism)
  int j0 = (w - g) & 3;
  constexpr uint32_t STAGE_B = F_STAGE_EL * 8;
  while (true) {
    const FMeta& m = reinterpret_cast<const FMeta*>(ring.meta)[stage];
    const int type = m.type, flags = m.flags, mb = m.mb;
    const uint32_t sa = ring.smem + stage * STAGE_B;
    const bool v0 = j0 < mb, v1 = j0 + 4 < mb;
    if (type == 1) {
      // T^T[8a + lr][8j + ·] += R[8a + lr][k] ψ[8j + ·][k], k4 steps of 32 n
      const int nks = m.nks;
      const uint32_t pa = sa + (lr * FKLD + lc) * 8;
      const uint32_t pb = sa + F_A_EL * 8 + ((8 * j0 + lr) * FKLD + lc) * 8;
      auto body = [&](auto two_t) {
        constexpr bool TWO = decltype(two_t)::value;
#pragma unroll
        for (int ks = 0; ks < FKC / 4; ++ks) {
          if (ks < nks) {
            double af[RT];
#pragma unroll
            for (int a = 0; a < RT; ++a) af[a] = lds64(pa + (8 * a * FKLD + 4 * ks) * 8);
            const double b0 = lds64(pb + 4 * ks * 8);
            double b1 = 0.0;
            if (TWO) b1 = lds64(pb + (32 * FKLD + 4 * ks) * 8);
#pragma unroll
            for (int a = 0; a < RT; ++a) dmma(tt[a][0], af[a], b0);
            if (TWO) {
#pragma unroll
              for (int a = 0; a < RT; ++a) dmma(tt[a][1], af[a], b1);
            }
          }
        }
      };
#ifndef FX_NOSTEP1
      if (v1) body(std::true_type{});
      else if (v0) body(std::false_type{});
#endif
    } else if (type == 3) {
      // identity R: T^T[8a + lr][8j + 2lc + e] = ψ[8j + 2lc + e][8a + lr]
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 0 ? v0 : v1) {
          const uint32_t p = sa + ((8 * (j0 + 4 * h) + 2 * lc) * FCLD + lr) * 8;
#pragma unroll
          for (int a = 0; a < RT; ++a) {
            tt[a][h][0] = lds64(p + 8 * a * 8);
            tt[a][h][1] = lds64(p + (FCLD + 8 * a) * 8);
          }
        }
      }
    } else {
      // σ^T[8a + lr][8c + ·] += s T^T[8a + lr][8j + 2lc + e] L[8c + ·][8j + 2lc + e]
      const double s = m.scale;
      auto step2 = [&](auto h_t) {
        constexpr int H = decltype(h_t)::value;
        const uint32_t pl = sa + (lr * FLLD + 8 * (j0 + 4 * H) + 2 * lc) * 8;
#ifndef FX_NOSCALE
        if (__double_as_longlong(s) != 0x3FF0000000000000LL) {
#pragma unroll
          for (int a = 0; a < RT; ++a) {
            tt[a][H][0] *= s;
            tt[a][H][1] *= s;
          }
        }
#endif
#pragma unroll
        for (int c = 0; c < QB; ++c) {
          double b0, b1;
          lds128(pl + 8 * c * FLLD * 8, b0, b1);
#pragma unroll
          for (int a = 0; a < RT; ++a) {
            dmma(sacc[a][c], tt[a][H][0], b0);
            dmma(sacc[a][c], tt[a][H][1], b1);
          }
        }
      };
#ifndef FX_NOSTEP2
      if (v0) step2(std::integral_constant<int, 0>{});
      if (v1) step2(std::integral_constant<int, 1>{});
#endif
      if (flags & kSegEnd) {
#pragma unroll
        for (int a = 0; a < RT; ++a)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) tt[a][hh][0] = tt[a][hh][1] = 0.0;
        g += mb;
        j0 = (w - g) & 3;
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
  // ordered reduction of the four partial σ^T tiles: warp 0 stores, warps 1
  // and 2 add, warp 3 adds and writes σ (transposed back); the last barrier
  // frees the scratch for the next tile
  const uint32_t sp = static_cast<uint32_t>(__cvta_generic_to_shared(scratch)) +
                      (lr * F_SLD + 2 * lc) * 8;
#pragma unroll 1
  for (int s = 0; s < 4; ++s) {
    if (w == s) {
#pragma unroll
      for (int a = 0; a < RT; ++a)
#pragma unroll
        for (int c = 0; c < QB; ++c) {
          const uint32_t p = sp + (8 * a * F_SLD + 8 * c) * 8;
          double x = sacc[a][c][0], y = sacc[a][c][1];
          if (s > 0) {
            double u, v;
            lds128(p, u, v);
            x += u;
            y += v;
          }
          if (s < 3) {
            asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(p), "d"(x), "d"(y) : "memory");
          } else {
            // σ[8c + 2lc + e][8a + lr] (tile-relative), rows < q, cols < rt
            const int col = 8 * a + lr;
            if (col < rt) {
              const int row = 8 * c + 2 * lc;
              double* p0 = cbase + (int64_t)row * ldc + col;
              if (row < q) *p0 = beta ? *p0 + x : x;
              if (row + 1 < q) p0[ldc] = beta ? p0[ldc] + y : y;
            }
          }
        }
    }
    named_bar(1, 128);
  }
}

#define SDMRG_FCASE(RT, QB) \
  case (RT) * 16 + (QB):    \
    fused_tile<RT, QB>(ring, stage, phase, g, w, lane, scratch); \
    break;
#define SDMRG_FROW(RT)                                                                  \
  SDMRG_FCASE(RT, 1) SDMRG_FCASE(RT, 2) SDMRG_FCASE(RT, 3) SDMRG_FCASE(RT, 4)           \
  SDMRG_FCASE(RT, 5) SDMRG_FCASE(RT, 6) SDMRG_FCASE(RT, 7) SDMRG_FCASE(RT, 8)

// ------------------------------------------------------------------ producer
// F_PRODUCERS warps share every stage's copies (row r -> warp r mod
// F_PRODUCERS): one warp issuing ~50 cp.async per lane and stage could not
// keep four DMMA warps fed (ncu r2d: 14% DMMA-pipe activity with a single
// producer, consumers spinning on the full barriers).
//
// 16-byte copies of `rows` rows x 64 K-columns of a row-major source (ld
// even, column offset even), zero-filling columns >= kvalid and rows >=
// rvalid; destination row stride LD.
template <int LD>
__device__ __forceinline__ void f_load_rows64(uint32_t sdst, const double* src, int ld, int rows,
                                              int rvalid, int kvalid, int lane, int pw) {
  const int k = 2 * lane;
  const int bytes = k + 1 < kvalid ? 16 : (k < kvalid ? 8 : 0);
  for (int r = pw; r < rows; r += F_PRODUCERS) {
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
          f_load_rows64<FKLD>(st, rb + c0, pad2d(n), tr.rt, tr.rt, kv, lane, pw);
          f_load_rows64<FKLD>(st + F_A_EL * 8, psi + c0, pad2d(n), 8 * mb, m, kv, lane, pw);
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
      open();
      const uint32_t st = ring.smem + stage * (F_STAGE_EL * 8);
      meta_write(2, 0, 0, kSegEnd | (last_seg ? kLast : 0));
      f_load_rows64<FLLD>(st, l, pad2d(m), tr.q, tr.q, m, lane, pw);
      close();
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
  int stage = 0, g = 0;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(ring.full0 + 8 * stage, phase);
    const FMeta& m = meta[stage];
    if (m.flags & kEnd) break;
    const int rtb = (m.rt + 7) >> 3, qb = (m.q + 7) >> 3;
    switch (rtb * 16 + qb) {
#ifdef SDMRG_FONE
      SDMRG_FCASE(5, 8)
#else
      SDMRG_FROW(1) SDMRG_FROW(2) SDMRG_FROW(3) SDMRG_FROW(4) SDMRG_FROW(5)
#endif
      default: __trap();
    }
  }
}
#undef SDMRG_FCASE
#undef SDMRG_FROW
#endif  // SDMRG_FUSED_KERNEL

}  // namespace sdmrg
