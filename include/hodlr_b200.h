/*
 * hodlr_b200.h -- C ABI of the B200-native HODLR factorize/solve engine.
 *
 * Plain pointers, sizes and a cudaStream_t (passed as void*); no torch types.
 * Every entry point is stream-ordered, allocates nothing (workspace is passed
 * in) and returns a hodlr_status.  Device pointers are column-major buffers in
 * the reference's layout (Fig. 3):
 *   D   leaf a at a*m*m (m x m, ld m)
 *   U/Y N x rL slab, ld N, level l' in 1..L at columns [(l'-1) r, l' r)
 *   V   same as U
 *   K   level l (0..L-1) at ((2^l)-1)*(2r)^2, parent p at +p*(2r)^2 (2r x 2r)
 * (uniform rank r; with per-level ranks (hodlr_desc.ranks) the slabs have
 * sum(ranks) columns and the per-level blocks follow each other, see below).
 *
 * Each entry point replaces a reference interface (file:line under
 * /root/reference); see INTEGRATION.md for the Python/ctypes binding.
 */
#ifndef HODLR_B200_H
#define HODLR_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HODLR_OK = 0,
  HODLR_ERR_ARG = 1,      /* bad argument (shape, size, layout)             */
  HODLR_ERR_SHAPE = 2,    /* operand shapes disagree                        */
  HODLR_ERR_SINGULAR = 3, /* a block was flagged singular (see info arrays) */
  HODLR_ERR_CUDA = 4,     /* CUDA launch / runtime error                    */
  HODLR_ERR_NCCL = 5      /* collective failure (distributed entry points)  */
} hodlr_status;

/* dtype tags */
#define HODLR_F64 0
#define HODLR_F32 1

/* Library version + last CUDA error string (thread-local, for diagnostics). */
const char* hodlr_version(void);
const char* hodlr_last_error(void);

/* Scalars per s x s block of the factorization-internal solve aids (the Dinv /
 * Kinv buffers of hodlr_factors): 8 s for s in {32, 64, 128} (8x8
 * diagonal-block inverses), s^2 for s = 16 (packed inverses), 0 otherwise. */
size_t hodlr_inv_elems(int s);

/* Instrumentation (no reference counterpart; the reference only returns flop
 * counts, backend.py:18-20).  hodlr_launch_count: kernels launched by this
 * library since load.  hodlr_profile_enable(1) brackets every factorize /
 * solve phase with CUDA events on the caller's stream; hodlr_profile_read
 * synchronises, writes the accumulated milliseconds per phase class
 * (HODLR_PHASE_*) into ms[0..n) and resets.  Returns the number of classes. */
#define HODLR_PHASE_LEAF_GETRF 0
#define HODLR_PHASE_LEAF_APPLY 1
#define HODLR_PHASE_K_GETRF 2
#define HODLR_PHASE_K_APPLY 3
#define HODLR_PHASE_LEVEL 4
#define HODLR_PHASE_GEMM 5
#define HODLR_PHASE_SOLVE_LEAF 6
#define HODLR_PHASE_SOLVE_K 7
#define HODLR_PHASE_SOLVE_LEVEL 8
#define HODLR_NUM_PHASES 9
long long hodlr_launch_count(void);
void hodlr_profile_enable(int on);
int hodlr_profile_read(double* ms, int n);

/* ------------------------------------------------------------------------
 * Batched kernels (reference batched-kernel layer, backend.py)
 * --------------------------------------------------------------------- */

/* Batched right-looking partial-pivot LU, in place, bit-identical to the
 * reference (first-max pivot, true division, separately rounded multiply and
 * subtract, singular guard |piv| <= eps*s*max|orig col|).
 * Replaces backend.py:481 batched_lu_factor_inplace / :444 _lu_factor_stack.
 * A: batch blocks of s x s at A + b*strideA (ld lda).
 * swaps/perm: int32 [batch*s] (0-based, LAPACK-style swaps; P A = A[perm]).
 * info: int32 [batch], 1 = flagged singular.
 * Ainv (optional, may be NULL; s in {16,32,64,128}): packed triangular inverses
 * strict_lower(L^-1) + upper(U^-1) written at Ainv + b*strideInv (ld ldinv);
 * X = U^-1 (L^-1 (P B)) is then two masked DMMA GEMMs (the solves of the
 * factor and solve phases). */
hodlr_status hodlr_getrf_batched(int dtype, int s, int batch, void* A, int64_t lda, int64_t strideA,
                                 int32_t* swaps, int32_t* perm, int32_t* info, void* Ainv,
                                 int64_t ldinv, int64_t strideInv, void* stream);

/* Batched LU solve from stored factors: rhs <- A^-1 rhs (gather by perm,
 * unit-L forward, U backward with true division).
 * Replaces backend.py:570 batched_lu_solve_inplace / :532 lu_solve_stacks. */
hodlr_status hodlr_getrs_batched(int dtype, int s, int nrhs, int batch, const void* LU, int64_t lda,
                                 int64_t strideA, const int32_t* perm, void* B, int64_t ldb,
                                 int64_t strideB, void* stream);

/* Batched GEMM  C_b <- alpha op(A_b) B_b + beta C_b,  op in {N, T}.
 * Operand b lives at X + (b / bdiv) * strideX_hi + (b % bdiv) * strideX_lo,
 * which covers the reference's constant-stride fast path (bdiv = 1) and the
 * paired-child layouts of the level GEMMs (bdiv = 2).  The product is formed
 * first and combined afterwards (tmp = op(A)B; C = beta C + alpha tmp),
 * as in backend.py:282-303.  C may alias B when the whole of C's rows fit
 * one tile (M <= 64) -- used for in-place inverse applications.
 * Replaces backend.py:320 batched_gemm, :266 gemm_stacks, :367
 * grouped_gemm_large (split-K with a fixed reduction order for huge K). */
hodlr_status hodlr_gemm_batched(int dtype, int transA, int M, int N, int K, double alpha,
                                const void* A, int64_t lda, int64_t sA_hi, int64_t sA_lo,
                                const void* B, int64_t ldb, int64_t sB_hi, int64_t sB_lo, double beta,
                                void* C, int64_t ldc, int64_t sC_hi, int64_t sC_lo, int batch, int bdiv,
                                void* work, size_t work_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Whole-phase entry points (SPEC factorization / solver modules)
 * --------------------------------------------------------------------- */

typedef struct {
  int64_t n;     /* matrix dimension N = m * 2^L                   */
  int32_t m;     /* leaf size                                      */
  int32_t r;     /* uniform rank, or the max of ranks[]            */
  int32_t L;     /* tree depth                                     */
  int32_t dtype; /* HODLR_F64 / HODLR_F32                          */
  const int32_t* ranks; /* NULL: rank r at every level.  Else ranks[l'-1] =
                     rank of level l' (1..L), each node of a level zero-
                     padded to its level's rank (SPEC.md:147-160 ragged
                     panels).  Level l' then owns slab columns
                     [c_l', c_l' + ranks[l'-1]) with c_l' = sum of the ranks
                     above; parent level l's K blocks are 2 ranks[l] square,
                     stored level after level.  fp64 factorize / solve /
                     matvec; the builders and the row-sharded entry points
                     take uniform ranks only. */
} hodlr_desc;

/* Device buffers of a factorization (all owned by the caller). */
typedef struct {
  void* D;        /* in: leaf blocks; out: leaf LU                       */
  void* Dinv;     /* out: leaf solve aids, 2^L * hodlr_inv_elems(m) scalars
                     (fp64; unused by fp32): for m in {32,64,128} the 8x8
                     diagonal-block inverses P_q = strict_lower(L_qq^-1) +
                     upper(U_qq^-1), row-major at block + 64 q (blocked DMMA
                     substitutions); m = 16: packed L^-1 / U^-1             */
  void* Y;        /* in: U slab; out: Y slab                             */
  void* V;        /* in: V slab                                          */
  void* K;        /* out: K LU per level ((2^L - 1) (2r)^2)              */
  void* Kinv;     /* out: the same for the K blocks: (2^L - 1) *
                     hodlr_inv_elems(2r), level l at (2^l - 1) * that      */
  int32_t* dswaps; /* out: 2^L m                                          */
  int32_t* dperm;  /* out: 2^L m                                          */
  int32_t* dinfo;  /* out: 2^L                                            */
  int32_t* kswaps; /* out: (2^L - 1) 2r                                   */
  int32_t* kperm;  /* out: (2^L - 1) 2r                                   */
  int32_t* kinfo;  /* out: 2^L - 1                                        */
} hodlr_factors;

/* Workspace bytes for factorize / solve with nrhs columns. */
size_t hodlr_factorize_workspace(const hodlr_desc* d);
size_t hodlr_solve_workspace(const hodlr_desc* d, int nrhs);

/* Alg. 3.  Singularity is reported in the
 * info arrays (the host wrapper raises naming level and node). */
hodlr_status hodlr_factorize(const hodlr_desc* d, const hodlr_factors* f, void* work,
                             size_t work_bytes, void* stream);

/* Alg. 3 from host memory: D / U / V (host buffers in the reference layout)
 * are uploaded on copy_stream in the order the factorization consumes them (D,
 * U, V^(L), then V^(L-1) .. V^(1)) while the factorization runs on `stream`,
 * each level waiting only for its own V panel.  f->D / f->Y / f->V are the
 * device destinations (f->Y receives U).  fp64.  Pinned buffers are copied
 * directly (keep them alive until `stream` has passed the call); pageable ones
 * stream through a library-owned pinned ring (host copy threads, the
 * factorization enqueued by a second host thread as the panels land) and are
 * no longer read once the call returns.  Calls are serialised per process. */
hodlr_status hodlr_factorize_from_host(const hodlr_desc* d, const hodlr_factors* f, const void* D_host,
                                       const void* U_host, const void* V_host, void* work, size_t work_bytes,
                                       void* stream, void* copy_stream);

/* Alg. 4: X (N x nrhs, ld ldx) is
 * overwritten with A^-1 X. */
hodlr_status hodlr_solve(const hodlr_desc* d, const hodlr_factors* f, void* X, int64_t ldx, int nrhs,
                         void* work, size_t work_bytes, void* stream);

/* HODLR matvec Y = A X on the unfactored representation (SPEC.md:183-191
 * [OP] matvec): D / U / V in the layout above (U, not the
 * factored Y), X and Y N x nrhs (ld ldx / ldy, Y must not alias X).  Two HBM
 * streams: w = V^T X for every child of every level, then Y = D X + U w_sib.
 * Vector loads when m % 4 == 0 and V / U / D are 4 / 2 / 2-scalar aligned,
 * scalar loads otherwise.  Per-column results do not depend on nrhs. */
size_t hodlr_matvec_workspace(const hodlr_desc* d, int nrhs);
hodlr_status hodlr_matvec(const hodlr_desc* d, const void* D, const void* U, const void* V, const void* X,
                          int64_t ldx, void* Y, int64_t ldy, int nrhs, void* work, size_t work_bytes,
                          void* stream);

/* Layout helper of the solve API: X[c * ldx + i] = B[i * ldb + c] for i < n,
 * c < k (a row-major n x k block to column-major, or back with the roles of
 * n / k swapped), fp64, asynchronous on `stream`. */
hodlr_status hodlr_transpose_f64(const void* B, int64_t n, int64_t k, int64_t ldb, void* X, int64_t ldx,
                                 void* stream);

/* HODLR assembly on the device (SPEC.md:163-171 [OP] assemble): leaf blocks
 * D materialized exactly; every sibling off-diagonal block A(I_a, I_b)
 * compressed to U_a V_b^T by ACA with rook pivoting at rank cap r (replaces
 * compress.py:87-200 compress(..., CompressionConfig(tol=0, max_rank=r,
 * method="aca_rook_pivot")) called per block; same operation order, so the
 * crosses are bit-identical for bit-identical entries).  Blocks of exact rank
 * < r keep zero columns.  Synchronous with respect to `stream` (the ACA
 * control loop reads per-level flags back).  ERR_ARG also flags a non-finite
 * oracle entry (the reference raises ValueError).
 * hodlr_build_laplace_dl: geom = 7 x N doubles (x, y, nx, ny, weights,
 *   -log|x - z| / 2pi, -curvature / 4pi) of the contour (problems.py:133-217).
 * hodlr_build_gaussian: exp(-|p_i - p_j|^2 / h^2) + lambda delta_ij on dim-major
 *   point coordinates pts (dim in 1..3, p_k at pts + k N), already in cluster
 *   (kd) order -- BASELINE cfg1 (2-D) / cfg3 (3-D) operators.
 * hodlr_build_dense: entries of a dense column-major N x N device matrix. */
size_t hodlr_build_workspace(const hodlr_desc* d);
/* The xorshift64* uniform stream of problems.py:26-48 (XorShift64Star(seed).uniform(count))
 * written to out[0..count) on the device, bit-identical (point sets of the cfg1/cfg3 operators). */
hodlr_status hodlr_xorshift_uniform(uint64_t seed, int64_t count, double* out, void* stream);
hodlr_status hodlr_build_laplace_dl(const hodlr_desc* d, const double* geom, void* D, void* U, void* V, void* work,
                                    size_t work_bytes, void* stream);
hodlr_status hodlr_build_gaussian(const hodlr_desc* d, const double* pts, int dim, double h, double lambda, void* D,
                                  void* U, void* V, void* work, size_t work_bytes, void* stream);
hodlr_status hodlr_build_dense(const hodlr_desc* d, const double* A, int64_t lda, void* D, void* U, void* V,
                               void* work, size_t work_bytes, void* stream);
/* Schur-complement surrogate of BASELINE cfg4 (no reference counterpart): the
 * hypersingular kernel -1 / (pi r^3) of a planar separator's half-space
 * Dirichlet-to-Neumann map on 2-D grid points pts (dim-major, cluster order),
 * diagonal 2.8755 (lattice row sum) + sigma. */
hodlr_status hodlr_build_schur_plane(const hodlr_desc* d, const double* pts, double sigma, void* D, void* U,
                                     void* V, void* work, size_t work_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Row-sharded (multi-GPU) schedule, SURVEY.md §8e.  The caller holds the rows
 * [row0, row0 + n_loc) of one level-p node (n_loc = N / 2^p): its leaves' D
 * (local arrays), its rows of the Y / V slabs (ld n_loc) and the full K /
 * K-pivot arrays in the global level layout.  Levels >= p are local
 * (hodlr_factorize_local); each level lv < p is one sum all-reduce of the
 * packed [W|T] of the 2^(lv+1) children (paired per parent: 2r x r(lv+1), ld
 * 2r, parent stride 2r*r(lv+1)) followed by hodlr_factorize_top.  Outputs
 * tw_out / w_out are the caller's contribution for its own node, r x ncols,
 * ld r.  The solve mirrors it with w (2r x nrhs per parent).  With n_loc = N
 * these reduce to hodlr_factorize / hodlr_solve.
 * --------------------------------------------------------------------- */
size_t hodlr_factorize_local_workspace(const hodlr_desc* d, int64_t n_loc);
hodlr_status hodlr_factorize_local(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0,
                                   int lv_stop, double* tw_out, void* work, size_t work_bytes, void* stream);
hodlr_status hodlr_factorize_top(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0, int lv,
                                 const double* tw_all, double* tw_out, void* work, size_t work_bytes,
                                 void* stream);
hodlr_status hodlr_solve_local(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0,
                               int lv_stop, void* X, int64_t ldx, int nrhs, double* w_out, void* work,
                               size_t work_bytes, void* stream);
hodlr_status hodlr_solve_top(const hodlr_desc* d, const hodlr_factors* f, int64_t n_loc, int64_t row0, int lv,
                             const double* w_all, double* w_out, void* X, int64_t ldx, int nrhs, void* work,
                             size_t work_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HODLR_B200_H */
