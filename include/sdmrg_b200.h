/*
 * sdmrg_b200.h — C ABI of the B200-native H_eff·ψ / renormalization path.
 *
 * Drop-in boundary for the hot path of the reference package `sector_dmrg`
 * (arxiv 2305.05581 artifact, /root/reference/pkg/src/sector_dmrg).  Every
 * entry point takes plain pointers and sizes; device pointers are CUDA global
 * memory on the current device, host pointers are ordinary process memory.
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Entry point                     replaces (reference file:line)
 * ------------------------------  -------------------------------------------
 * sdmrg_dgemm                     gemm.py:61   NumpyGemm.gemm
 * sdmrg_dgemm_strided_batched     gemm.py:76   NumpyGemm.gemm_strided_batched
 * sdmrg_daxpy                     gemm.py:86   NumpyGemm.add_inplace
 * sdmrg_sbmm4s                    sbmm4s.py:167 sbmm4s (Alg. 2: two kernels,
 *                                 no reduction pass; chunked fallback :176)
 * sdmrg_plan_build                blocks.py:503 build_plan (task generation:
 *                                 operator-table rows x ψ sectors -> work list)
 * sdmrg_plan_groups               blocks.py:563 the per-(ψ key, out key) groups
 * sdmrg_plan_shard                (multi-GPU) ψ-sector ownership of a rank
 * sdmrg_plan_arena                the plan's padded operator arenas (fill in
 *                                 place: large synthetic workloads)
 * sdmrg_plan_apply                dmrg.py:107  apply_plan (out += H_eff ψ)
 * sdmrg_dot / sdmrg_nrm2 /
 * sdmrg_gemv_t / sdmrg_gemv_n /
 * sdmrg_scal_dev / sdmrg_axpby    dmrg.py:43   lanczos_ground vector algebra
 *                                 (dot, axpy, full reorthogonalisation, norms)
 * sdmrg_rotate                    dmrg.py:254  _transform_tree (W^T O W for
 *                                 every maintained operator block)
 * sdmrg_rdm_accumulate            dmrg.py:221  rdm_eigensystem (ρ += S S^T)
 * sdmrg_grouped_gemm              the block algebra of a sweep step on the same
 *                                 engine: blocks.py:331 materialize_aux,
 *                                 blocks.py:190 enlarge_block (+ :262 the
 *                                 enlarged H) fused with dmrg.py:254
 *                                 _transform_tree, driver.py:200/228 White's
 *                                 prediction (paper_2305_05581_b200/blockops.py)
 *
 * Errors: every function returns SDMRG_OK (0) or a nonzero code and records a
 * message retrievable with sdmrg_last_error() (thread-local).  Argument errors
 * mirror the reference's ValueError/WorkspaceError cases.
 */
#ifndef SDMRG_B200_H
#define SDMRG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDMRG_OK 0
#define SDMRG_EINVAL 1      /* dimension/argument mismatch (ValueError)        */
#define SDMRG_ECUDA 2       /* CUDA runtime failure                            */
#define SDMRG_EWORKSPACE 3  /* workspace cannot hold one member (WorkspaceError)*/
#define SDMRG_ENOMEM 4      /* device allocation failed                        */

const char* sdmrg_last_error(void);
int sdmrg_version(void);
/* Number of kernels this library has launched since load (all entry points). */
int64_t sdmrg_launch_count(void);

/* ------------------------------------------------------------------ GEMM --
 * Column-major (BLAS) convention, as sbmm4s.py's DenseMatrix (sbmm4s.py:29).
 * c := alpha * op(a) @ op(b) + beta * c ; op = transpose when trans != 0.    */
int sdmrg_dgemm(int transa, int transb, int m, int n, int k, double alpha,
                const double* a, int lda, const double* b, int ldb,
                double beta, double* c, int ldc, void* stream);

/* c_i := op(a_i) @ op(b_i) for i < batch (one kernel; gemm.py:76 semantics:
 * beta = 0, the members' outputs may interleave, e.g. ld = m*p, stride = m). */
int sdmrg_dgemm_strided_batched(int transa, int transb, int m, int n, int k,
                                const double* a, int lda, int64_t stride_a,
                                const double* b, int ldb, int64_t stride_b,
                                double* c, int ldc, int64_t stride_c,
                                int batch, void* stream);

/* y += alpha * x (the lone standalone reduction kernel, gemm.py:86). */
int sdmrg_daxpy(int64_t n, double alpha, const double* x, double* y,
                void* stream);

/* ---------------------------------------------------------------- SBMM4S --
 * B := B + alpha * sum_{i<p} L_i A R_i^T      (sbmm4s.py:167, Alg. 2)
 * A: m x n (lda), B: q x r (ldb), L_i: q x m at l + i*stride_l (ldl),
 * R_i: r x n at r_stack + i*stride_r (ldr); all column-major device memory.
 * workspace: >= m*r doubles; with < m*p*r the batch is split in halves
 * recursively (sbmm4s.py:176).  Two kernels per (sub)batch, zero reduction
 * kernels.  *kernels_out (nullable) receives the kernel count.                */
int sdmrg_sbmm4s(int m, int n, int q, int r, int p, double alpha,
                 const double* a, int lda,
                 const double* l_stack, int ldl, int64_t stride_l,
                 const double* r_stack, int ldr, int64_t stride_r,
                 double* b, int ldb,
                 double* workspace, int64_t workspace_doubles,
                 int* kernels_out, void* stream);

/* ------------------------------------------------------------ H_eff plan --
 * Compact operator-table form of blocks.py:503 build_plan.
 *
 * Quantum numbers are int32 tuples of `ncomp` components, compared
 * lexicographically (sectors.py:53 SectorBasis sorts them).  A block basis is
 * `nsec` sorted QNs + dims.  The two free sites share one local basis of
 * `nsite` one-dimensional states (model.py:54 LocalSpace).
 *
 * Operators of the left (right) block live in one device arena of doubles;
 * op `o` with shift delta_o stores block (q+delta_o, q) — rows dim(q+delta),
 * cols dim(q), row-major (numpy C order) — at arena offset
 * blk_off[o*nsec + j] (j = index of column sector q), or -1 when absent.
 * op_kind[o]: 0 general, 1 identity (KEY_I; multiplication may be skipped).
 *
 * Row t of the operator table (model.py:341 TableRow, resolved as in
 * blocks.py:521-565): left op lop[t], right op rop[t], coefficient alpha[t],
 * left-parity dressing e_l[t] (scale *= left_sign[j] of the input left
 * sector), and the two site operators as column maps over local states:
 * site1_dst[t*nsite + s] = output state of input state s or -1, with value
 * site1_val[...] (site parity dressings e_1/e_2 already folded in).
 *
 * ψ layout (blocks.py:416 SuperblockWavefunction): keys (qL,q1,q2,qR) with
 * qL+q1+q2+qR = target, sorted lexicographically; block dims(qL) x dims(qR)
 * row-major, concatenated in key order (blocks.py:448 to_vector).
 *
 * Sharding (multi-GPU): rank/world select a balanced subset of ψ input keys;
 * the partial σ of all ranks sums to H_eff ψ (allreduce on the host side).   */
typedef struct sdmrg_plan_desc {
  int ncomp;
  int nsite;
  const int32_t* site_qn;          /* nsite * ncomp                           */
  const int32_t* target;           /* ncomp                                   */
  int nsec_l;
  const int32_t* qn_l;             /* nsec_l * ncomp, sorted                  */
  const int32_t* dim_l;            /* nsec_l                                  */
  const double* left_sign;         /* nsec_l: parity sign of each left sector */
  int nsec_r;
  const int32_t* qn_r;
  const int32_t* dim_r;
  int nops_l;
  const int32_t* delta_l;          /* nops_l * ncomp                          */
  const int64_t* blk_off_l;        /* nops_l * nsec_l                         */
  const int32_t* kind_l;           /* nops_l                                  */
  int nops_r;
  const int32_t* delta_r;
  const int64_t* blk_off_r;        /* nops_r * nsec_r                         */
  const int32_t* kind_r;
  int64_t nrows;
  const int32_t* lop;
  const int32_t* rop;
  const double* alpha;
  const int32_t* e_l;
  const int32_t* site1_dst;        /* nrows * nsite                           */
  const double* site1_val;
  const int32_t* site2_dst;
  const double* site2_val;
  const double* arena_l;           /* device; repacked into plan-owned padded */
  const double* arena_r;           /* memory at build (may be freed after);
                                      NULL: zeroed, fill via sdmrg_plan_arena */
  int64_t workspace_doubles;       /* budget for the T = A R^T staging (0 = auto) */
  int rank;
  int world;
  int keep_groups;                 /* 1: retain the reference grouping (parity) */
  int dry_run;                     /* 1: task generation only, no device work  */
} sdmrg_plan_desc;

typedef struct sdmrg_plan sdmrg_plan;

typedef struct sdmrg_plan_stats {
  int64_t psi_keys;
  int64_t psi_size;                /* doubles in ψ (to_vector length)         */
  int64_t groups;                  /* (ψ key, out key) groups, all ranks      */
  int64_t members;                 /* (row, ψ key) tasks, all ranks           */
  int64_t ref_flops;               /* reference plan.flops (flops_fused)      */
  int64_t exec_flops;              /* FLOPs this rank's kernels execute       */
  int64_t local_members;
  int64_t t_problems;              /* A R^T products staged (this rank)       */
  int64_t tiles;                   /* output tiles launched per apply         */
  int64_t segments;
  int64_t chunks;                  /* workspace chunks per apply              */
  int64_t workspace_doubles;
  int64_t kernels_per_apply;
  int64_t algo_bytes;              /* algorithmic HBM bytes per apply         */
  int64_t products;                /* phase-2 products (group, right op)      */
  int64_t combine_outputs;         /* pre-summed left operators per apply     */
  int64_t combine_terms;           /* their summands                          */
  int64_t build_ms_taskgen;        /* host: ψ keys, matching, pre-summation   */
  int64_t build_ms_emit;           /* host: work lists                        */
  int64_t build_ms_device;         /* repack, allocations, uploads            */
  int64_t fused_outs;              /* σ problems on the fused small-sector    */
                                   /* kernel (T chained in registers)         */
  int64_t arena_bytes;             /* padded operator arenas held by the plan */
  int64_t shard_balance_ppm;       /* mean / max rank cost x 1e6 (world > 1)  */
} sdmrg_plan_stats;

int sdmrg_plan_build(const sdmrg_plan_desc* desc, sdmrg_plan** out);
int sdmrg_plan_stats_get(const sdmrg_plan* plan, sdmrg_plan_stats* out);
/* ψ layout: keys (psi_keys * 4 sector indices: l, s1, s2, r) and offsets.   */
int sdmrg_plan_layout(const sdmrg_plan* plan, int32_t* keys, int64_t* offsets);
/* Reference grouping, for parity: per group (psi key index, out key index,
 * member begin); per member (row, left block col-sector j, scale).  Arrays
 * sized from stats (groups, members); group_begin has groups+1 entries.     */
int sdmrg_plan_groups(const sdmrg_plan* plan, int32_t* group_psi,
                      int32_t* group_out, int64_t* group_begin,
                      int64_t* member_row, double* member_scale);
/* The plan-owned padded operator arena of one side (0 left, 1 right): device
 * base pointer, size in doubles, and per (op, column sector) element offsets
 * (nops * nsec, -1 = absent).  Block (q+δ, q) is dim(q+δ) x dim(q) row-major
 * with row stride dim(q) rounded up to even; pad columns are zero.  A plan
 * built with arena_l/arena_r == NULL has zeroed arenas the caller fills in
 * place through this view (keeping the pads zero) before the first apply.  */
int sdmrg_plan_arena(const sdmrg_plan* plan, int side, double** base, int64_t* size,
                     int64_t* offsets);
/* Shard ownership: mine[i] = 1 when ψ key i is this rank's input sector
 * (psi_keys entries).  Every key belongs to exactly one rank of `world`.    */
int sdmrg_plan_shard(const sdmrg_plan* plan, int32_t* mine);
/* diag (device, psi_size doubles) := the diagonal of H_eff over this rank's
 * ψ sectors (zero elsewhere; sum over ranks for the full diagonal) — the
 * Davidson preconditioner of lanczos.py davidson_ground.  Stream-ordered. */
int sdmrg_plan_diagonal(sdmrg_plan* plan, double* diag, void* stream);
/* sigma (+)= H_eff psi over this rank's shard; device vectors of psi_size.
 * The operator pre-sums (phase 0: ψ-independent) are formed by the first
 * apply and reused by later ones; after changing the arenas in place call
 * sdmrg_plan_invalidate so the next apply forms them again.                 */
int sdmrg_plan_apply(sdmrg_plan* plan, const double* psi, double* sigma,
                     int accumulate, void* stream);
int sdmrg_plan_invalidate(sdmrg_plan* plan);
/* Per-launch CUDA-event timing of subsequent applies (bench instrumentation).
 * sdmrg_plan_timing syncs the last apply's events and writes, per phase
 * (0: left-operator pre-summation, 1: T = A R^T, 2: σ += Lsum T, 3: split-K
 * partial sums into σ), the summed device milliseconds ms[4], the executed
 * tensor FLOPs flops[4] and the algorithmic bytes of the elementwise phases
 * bytes[4].  Any pointer may be NULL.                                        */
int sdmrg_plan_set_timing(sdmrg_plan* plan, int enable);
int sdmrg_plan_timing(sdmrg_plan* plan, double* ms, int64_t* flops, int64_t* bytes);
int sdmrg_plan_destroy(sdmrg_plan* plan);

/* ------------------------------------------------------- vector algebra --
 * Deterministic (fixed-order) reductions; results land in DEVICE memory so a
 * Krylov step needs no host round-trip until the caller reads the scalars.  */
int sdmrg_dot(int64_t n, const double* x, const double* y, double* out_dev,
              void* stream);
int sdmrg_nrm2(int64_t n, const double* x, double* out_dev, void* stream);
/* coef[i] = <V_i, w> for i < k; V row-major k x n (ldv).                     */
int sdmrg_gemv_t(int k, int64_t n, const double* v, int64_t ldv,
                 const double* w, double* coef_dev, void* stream);
/* w += sign * sum_i coef[i] V_i (coef on device).                           */
int sdmrg_gemv_n(int k, int64_t n, const double* v, int64_t ldv,
                 const double* coef_dev, double sign, double* w, void* stream);
/* x *= s where s = num/den read from device scalars (den NULL -> 1).        */
/* One classical Gram-Schmidt pass of the device Lanczos (dmrg.py:67-71
 * reorthogonalisation) over a Krylov basis held as nslabs (<= 16) slabs of
 * slab_rows contiguous length-n vectors (k vectors in all):
 *   coef = V^T w;  w -= V coef;  and, if norm_dev, *norm_dev = ||w|| after.
 * Four launches whatever k is; fixed-order reductions (bitwise repeatable). */
int sdmrg_krylov_project(int nslabs, const double* const* slabs, int slab_rows, int k, int64_t n,
                         double* w, double* coef_dev, double* norm_dev, void* stream);
/* Davidson correction vector with the diagonal preconditioner of H_eff
 * (sdmrg_plan_diagonal): t = r / (theta - diag), |theta - diag| >= 1e-3. */
int sdmrg_davidson_precond(int64_t n, const double* r, const double* diag, double theta,
                           double* t, void* stream);
int sdmrg_scal_dev(int64_t n, const double* num_dev, const double* den_dev,
                   int invert_den, double* x, void* stream);
/* y = a*x + b*y with host scalars.                                          */
int sdmrg_axpby(int64_t n, double a, const double* x, double b, double* y,
                void* stream);

/* --------------------------------------------------- renormalization ------
 * Grouped W^T O W (dmrg.py:254 _transform_tree).  For task t:
 *   tmp = W_l^T (rows x kl)^T @ O (rows x cols)   -> kl x cols
 *   dst = tmp @ W_r (cols x kr)                   -> kl x kr
 * All matrices row-major device memory at the given pointers.  Tasks run as
 * two grouped kernels; tmp lives in `workspace` (sum kl*cols doubles).      */
int sdmrg_rotate(int64_t ntasks, const int64_t* w_l, const int64_t* w_r,
                 const int64_t* o, const int64_t* dst, const int32_t* rows,
                 const int32_t* cols, const int32_t* kl, const int32_t* kr,
                 const double* base_w, const double* base_o, double* base_dst,
                 double* workspace, int64_t workspace_doubles, void* stream);

/* ρ_blocks: for task t, rho[t] (+)= S_t S_t^T  (dmrg.py:245). S row-major
 * rows_t x cols_t at base_s + s_off[t]; rho at base_rho + rho_off[t]
 * (rows_t x rows_t).  Tasks sharing one rho offset are summed in order.     */
int sdmrg_rdm_accumulate(int64_t ntasks, const int64_t* s_off,
                         const int64_t* rho_off, const int32_t* rows,
                         const int32_t* cols, const double* base_s,
                         double* base_rho, void* stream);

/* ------------------------------------------------- generic grouped GEMM --
 * Row-major, stream-ordered (no host synchronisation).  For problem p:
 *   C_p (m[p] x n[p], ldc[p]) = beta[p] * C_p
 *        + sum_{s = seg_begin[p]}^{seg_begin[p+1]-1} scale[s] * op(A_s) op(B_s)
 * op(A_s) is m x k[s]: A stored m x k (lda) or, trans_a, stored k x m (lda);
 * op(B_s) is k[s] x n: B stored k x n (ldb) or, trans_b, stored n x k (ldb).
 * Operands are handles: (base index << 60) | element offset, the base index
 * selecting one of `nbases` (<= 8) device pointers in the HOST array `bases`.
 * beta is 0 (overwrite; a problem without segments writes zeros) or 1.
 * Segments of one problem are summed in order (deterministic).              */
int sdmrg_grouped_gemm(int trans_a, int trans_b, int64_t nprob, const int64_t* c_h,
                       const int32_t* ldc, const int32_t* m, const int32_t* n,
                       const int32_t* beta, const int64_t* seg_begin, const int64_t* a_h,
                       const int32_t* lda, const int64_t* b_h, const int32_t* ldb,
                       const int32_t* k, const double* scale, double* const* bases,
                       int nbases, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SDMRG_B200_H */
