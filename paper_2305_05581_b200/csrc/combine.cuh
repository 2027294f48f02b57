// combine.cuh — operator pre-summation for H_eff·ψ phase 2.
//
// Inside one reference group (ψ key i -> out key o, blocks.py:563) the
// members (row t: left op a_t, right op b_t, scale s_t) form a bipartite set:
// the table keeps bilinear terms Σ_ab C_ab L_a ⊗ (site ops) ⊗ R_b whose
// coefficients depend on both sides (e.g. two-body integrals straddling the
// two free sites), so one right operator b meets many left operators.  With
// T(i, b) = A_i R_b^T shared per (ψ key, right op),
//
//     Σ_t s_t L_{a_t} A_i R_{b_t}^T  =  Σ_b ( Σ_{t: b_t = b} s_t L_{a_t} ) T(i, b)
//
// so phase 2 runs one q x m x r product per distinct (group, right op)
// instead of one per member (L=30, D=2048: 5.10 M -> 1.78 M products, 3.33 ->
// 1.10 TFLOP).  The inner sums  Lsum_b = Σ_t s_t L_{a_t}  are formed here:
// HBM-bound elementwise work, one CTA per (group, element chunk) producing
// every Lsum of that group, so each L_a chunk comes from HBM/L2 once and its
// re-reads for the group's other outputs hit L1.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "engine.cuh"

namespace sdmrg {

struct CombTask {     // 16 B: elements [e0, e0 + ne) of outputs [ob, oe)
  int32_t out_begin, out_end;
  int32_t e0, ne;
};
struct CombOut {      // 16 B: dst[e] = Σ_{terms} coef * src[e]
  uint64_t dst;
  int32_t term_begin, term_end;
};
struct CombTerm {     // 16 B
  uint64_t src;
  double coef;
};

constexpr int COMB_THREADS = 256;
constexpr int COMB_PER_THREAD = 4;
constexpr int COMB_CHUNK = COMB_THREADS * COMB_PER_THREAD;

// U > 1: the loads of U terms are issued before their FMAs (same summation
// order, bitwise the same result) — for the split-K partial sums (phase 3),
// whose long per-element term chains are latency-bound at small D.  Phase 0
// (HBM-bound, many outputs) measured slower that way and keeps U = 1.
template <int U>
__global__ void __launch_bounds__(COMB_THREADS)
combine_kernel(const CombTask* __restrict__ tasks, const CombOut* __restrict__ outs,
               const CombTerm* __restrict__ terms, Bases bases) {
  const CombTask t = tasks[blockIdx.x];
  for (int o = t.out_begin; o < t.out_end; ++o) {
    const CombOut out = outs[o];
    double acc[COMB_PER_THREAD];
#pragma unroll
    for (int u = 0; u < COMB_PER_THREAD; ++u) acc[u] = 0.0;
    int k = out.term_begin;
    if (U > 1) {
      for (; k + U <= out.term_end; k += U) {
        double v[U][COMB_PER_THREAD], cf[U];
#pragma unroll
        for (int x = 0; x < U; ++x) {
          const CombTerm term = terms[k + x];
          const double* src = resolve(bases, term.src) + t.e0;
          cf[x] = term.coef;
#pragma unroll
          for (int u = 0; u < COMB_PER_THREAD; ++u) {
            const int e = threadIdx.x + u * COMB_THREADS;
            v[x][u] = e < t.ne ? __ldg(src + e) : 0.0;
          }
        }
#pragma unroll
        for (int x = 0; x < U; ++x)
#pragma unroll
          for (int u = 0; u < COMB_PER_THREAD; ++u) acc[u] = fma(cf[x], v[x][u], acc[u]);
      }
    }
    for (; k < out.term_end; ++k) {
      const CombTerm term = terms[k];
      const double* src = resolve(bases, term.src) + t.e0;
#pragma unroll
      for (int u = 0; u < COMB_PER_THREAD; ++u) {
        const int e = threadIdx.x + u * COMB_THREADS;
        if (e < t.ne) acc[u] = fma(term.coef, __ldg(src + e), acc[u]);
      }
    }
    double* dst = const_cast<double*>(resolve(bases, out.dst)) + t.e0;
#pragma unroll
    for (int u = 0; u < COMB_PER_THREAD; ++u) {
      const int e = threadIdx.x + u * COMB_THREADS;
      if (e < t.ne) dst[e] = acc[u];
    }
  }
}

}  // namespace sdmrg
