/*
 * biluk.h -- C ABI of the B200-native block ILU(k) hot path.
 *
 * Every entry point replaces one stage of the reference Python package
 * `blockiluk` (/root/reference/pkg/src/blockiluk); the replaced interface is
 * cited next to each declaration.  Conventions:
 *
 *   - plain pointers and sizes only, no torch / C++ types;
 *   - "dev_" pointers are CUDA device pointers (the Python host passes
 *     torch.Tensor.data_ptr()), everything else is host memory;
 *   - `stream` is a cudaStream_t passed as void* (0 = legacy default stream);
 *   - every function returns a status code (BILUK_*), the message of the last
 *     failure on the calling thread is available from biluk_last_error();
 *   - block values are FP64, each bs x bs block flattened COLUMN-MAJOR, exactly
 *     the reference BcsrMatrix.values layout (sparse.py:92-99, :126-130);
 *   - indices on the boundary are int64 like the reference (sparse.py:16-20).
 *
 * Error codes map 1:1 onto the reference exception taxonomy (errors.py:4-31):
 *   BILUK_ESTRUCT    -> StructuralError        (pattern / shape problems)
 *   BILUK_ESINGULAR  -> SingularBlockError     (.row = *err_row)
 *   BILUK_EZEROPIVOT -> FactorizationError     (.row = *err_row, bs == 1 path)
 *   BILUK_EARG       -> ValueError             (bad k, bad lengths, config)
 */
#ifndef BILUK_H
#define BILUK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    BILUK_OK = 0,
    BILUK_ESTRUCT = 1,
    BILUK_ESINGULAR = 2,
    BILUK_EZEROPIVOT = 3,
    BILUK_ECUDA = 4,
    BILUK_ETIMEOUT = 5,     /* device-side dependency wait exceeded its budget */
    BILUK_EARG = 6,
    BILUK_ENOMEM = 7,
    BILUK_EUNSUPPORTED = 8
};

typedef struct biluk_plan biluk_plan_t;
typedef struct biluk_pattern biluk_pattern_t;
typedef struct biluk_op biluk_op_t;

/* Message of the last failing call on this thread ("" if none). */
const char *biluk_last_error(void);
/* Library version string. */
const char *biluk_version(void);
/* Make `device` current for this thread's subsequent calls (the Python host
 * passes torch.cuda.current_device()). */
int biluk_set_device(int32_t device);

/* ------------------------------------------------------------------------
 * Dense-block and scatter stages (device buffers, float64)
 * ---------------------------------------------------------------------- */

/* block_invert (factor.py:38-70), batched: n row-major bs x bs blocks
 * (the reference's (n, bs, bs) layout) -> their inverses, LU with partial
 * pivoting and the reference's singularity rules (all-zero block; |pivot| <
 * 1e-13 max|B|).  BILUK_ESINGULAR with *err_idx = the first singular block.
 * Synchronises the stream. */
int biluk_block_invert(int32_t bs, int64_t n, const double *dev_in, double *dev_out, int64_t *err_idx,
                       void *stream);

/* apply_block_diagonal (trisolve.py:148-166): z_I = dinv[I] y_I, dinv row-major
 * (n, bs, bs).  Asynchronous. */
int biluk_block_diag_apply(int32_t bs, int64_t n, const double *dev_dinv, const double *dev_y, double *dev_z,
                           void *stream);

/* materialize (factor.py:83-121), value side: dst[map[s]] = src[s] for nsrc
 * blocks of bs2 doubles (dst pre-zeroed by the caller; the slot map is
 * integer host work).  Asynchronous. */
int biluk_scatter_blocks(int32_t bs2, int64_t nsrc, const int64_t *dev_map, const double *dev_src, double *dev_dst,
                         void *stream);

/* ------------------------------------------------------------------------
 * Host-side symbolic helpers (integer, bit-exact with the reference)
 * ---------------------------------------------------------------------- */

/* symbolic_phase(pattern, k) -- symbolic.py:27-72.
 * Grows the square pattern (row_ptr[n+1], col_idx[nnz], strictly increasing
 * columns per row) to its ILU(k) level-of-fill pattern.  Missing diagonal ->
 * BILUK_ESTRUCT with *err_row = row; k < 0 -> BILUK_EARG. */
int biluk_symbolic(int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int32_t k,
                   biluk_pattern_t **out, int64_t *err_row);
int64_t biluk_pattern_nnz(const biluk_pattern_t *p);
/* copies row_ptr[n+1] and col_idx[nnz] (int64) out of the pattern */
int biluk_pattern_copy(const biluk_pattern_t *p, int64_t *row_ptr, int64_t *col_idx);
void biluk_pattern_free(biluk_pattern_t *p);

/* build_level_schedule(t) -- trisolve.py:98-118 (Eq. 4).
 * Levels of a strictly lower (upper = 0) or strictly upper (upper = 1)
 * CSR operand of dimension m: level_of_row[m] (1-based), *num_levels.
 * Lower rows are scanned forward, upper rows in reverse. */
int biluk_level_schedule(int64_t m, const int64_t *row_ptr, const int64_t *col_idx, int32_t upper,
                         int64_t *level_of_row, int64_t *num_levels);

/* ------------------------------------------------------------------------
 * Preconditioner plan: build_preconditioner (factor.py:302-323) split into
 * a host analysis step, a device binding step and a device numeric step.
 * ---------------------------------------------------------------------- */

/* Stages extract-pattern + symbolic-phase + schedules (factor.py:314-317,
 * trisolve.py:98-118): analyses the block pattern of the n x n block matrix,
 * builds the ILU(k) pattern, the block level sets of L and U' and the
 * level-ordered tile layout of both sweeps.  Host only, no device memory. */
int biluk_plan_create(int32_t bs, int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                      int32_t k, biluk_plan_t **out, int64_t *err_row);
void biluk_plan_destroy(biluk_plan_t *plan);
/* The same with flags: BILUK_PLAN_FACTOR_ONLY skips the sweep planning (the
 * plan then serves biluk_plan_factor_lu only -- the reference's
 * block_ilu0_factorize / point_ilu0_factorize, factor.py:151-205). */
#define BILUK_PLAN_FACTOR_ONLY 1
int biluk_plan_create_ex(int32_t bs, int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int32_t k,
                         int32_t flags, biluk_plan_t **out, int64_t *err_row);

/* Device workspace the plan needs (bytes, 256-byte aligned pointer expected). */
uint64_t biluk_plan_workspace_bytes(const biluk_plan_t *plan);

/* Upload the plan's index structures into the caller-owned device workspace. */
int biluk_plan_bind(biluk_plan_t *plan, void *dev_workspace, uint64_t bytes, void *stream);

/* Stages materialize + factorize + split (factor.py:83-121, :165-205,
 * :230-289) on the device.  dev_a_vals: the ORIGINAL matrix values
 * (nnzb * bs * bs, column-major blocks, same pattern as plan_create).
 * Synchronises the stream; on a singular block returns BILUK_ESINGULAR
 * (bs > 1) or BILUK_EZEROPIVOT (bs == 1) with *err_row = the first failing
 * block row, as the reference would report it (factor.py:202-203, :144-145). */
int biluk_plan_factor(biluk_plan_t *plan, const double *dev_a_vals, void *stream, int64_t *err_row);

/* block_ilu0_factorize / point_ilu0_factorize (factor.py:151-205): stages
 * materialize + factorize only.  dev_out_vals receives the in-place factored
 * L\U values on the plan's ILU(k) pattern (nnz(P') * bs * bs, column-major
 * blocks; unit-lower multipliers strictly below the diagonal, U unscaled).
 * Errors as biluk_plan_factor.  Synchronises the stream. */
int biluk_plan_factor_lu(biluk_plan_t *plan, const double *dev_a_vals, double *dev_out_vals, void *stream,
                         int64_t *err_row);

/* split_ldu (factor.py:230-289) of an already factored matrix: dev_lu_vals
 * holds L\U on the plan's pattern (plan created with k = 0 on that pattern);
 * D_i^-1 = block_invert(U_ii) (BILUK_ESINGULAR, *err_row = i), U' = D^-1 U,
 * then the sweep records -- the plan is ready for biluk_plan_apply.  With
 * D = I and T as L or U' this is also solve_unit_triangular
 * (trisolve.py:121-145).  Synchronises the stream. */
int biluk_plan_load_factored(biluk_plan_t *plan, const double *dev_lu_vals, void *stream, int64_t *err_row);

/* apply_preconditioner(f, b) -- trisolve.py:169-182 (Alg. 7):
 * x = U'^{-1} D^{-1} L^{-1} b, one persistent sync-free kernel for both
 * sweeps.  dev_b and dev_x hold n*bs doubles; dev_x may not alias dev_b.
 * Asynchronous; a dependency-wait timeout is reported by biluk_plan_status.
 * Applies of one plan share its device workspace, so they run one at a time:
 * an apply issued on a different stream than the previous one first waits
 * (cudaStreamWaitEvent) for that previous apply.  Plans are independent. */
int biluk_plan_apply(biluk_plan_t *plan, const double *dev_b, double *dev_x, void *stream);

/* Diagnostics: CUDA events around the sweep launch of every subsequent apply
 * (on = 1; 0 removes them).  biluk_plan_sweep_ms waits for the last apply's
 * sweep and returns its duration -- the sweep kernel alone, without the
 * right-hand-side permutation launched before it. */
int biluk_plan_set_timing(biluk_plan_t *plan, int32_t on);
int biluk_plan_sweep_ms(biluk_plan_t *plan, float *ms);

/* Runtime knobs of the sweep kernel (no effect on results):
 *   "gap"             fine-grained dependency polling starts when every level
 *                     <= (tile level - gap) is complete (default 2)
 *   "coarse_sleep_ns" back-off of the per-warp progress poll (default 64)
 *   "fine_sleep_ns"   back-off of the per-value dependency poll (default 0) */
int biluk_plan_tune(biluk_plan_t *plan, const char *key, int64_t value);

/* Diagnostics: when dev_trace != NULL every later apply writes, per tile
 * (L tiles then U' tiles), 4 uint64 {record ready, released to poll, done,
 * SM id} (globaltimer ns) into dev_trace.  NULL disables tracing. */
int biluk_plan_set_trace(biluk_plan_t *plan, void *dev_trace);

/* Combined dependency level of every tile (L tiles 1..levels_L, then U'
 * tiles levels_L+1..), host array of info[9]+info[10] entries. */
int biluk_plan_tile_levels(const biluk_plan_t *plan, int32_t *levels);

/* Diagnostics: copies up to max_records sweep-record descriptors (64 bytes
 * each, layout PRecInfo in csrc/biluk_internal.h) to `out` (may be NULL) and
 * returns the number of records of the plan's partitioned sweep. */
int biluk_plan_records(const biluk_plan_t *plan, void *out, int64_t max_records);

/* Synchronises the stream and returns the sticky device status of the plan
 * (BILUK_OK or BILUK_ETIMEOUT), clearing it. */
int biluk_plan_status(biluk_plan_t *plan, void *stream);

/* Plan facts: sizes of the factors and of the schedules.
 * info[0]=n  info[1]=bs  info[2]=k  info[3]=nnzb(A)  info[4]=nnzb(P')
 * info[5]=nL  info[6]=nU  info[7]=block levels of L  info[8]=block levels of U'
 * info[9]=L tiles  info[10]=U tiles  info[11]=rows per tile
 * info[12]=workspace bytes  info[13]=apply algorithmic bytes
 * info[14]=spmv algorithmic bytes  info[15]=sweep grid CTAs
 * info[16]=warps per CTA  info[17]=pipeline stages  info[18]=max tile record bytes
 * info[19]=max slots per tile */
int biluk_plan_info(const biluk_plan_t *plan, int64_t *info, int32_t ninfo);

/* Copy the factors to the host in the reference layout (factor.py:279-289):
 * L  : L_row_ptr[n+1], L_col_idx[nL], L_vals[nL*bs*bs]   (column-major blocks)
 * dinv: dinv[n*bs*bs] ROW-MAJOR (n, bs, bs) like the reference ndarray
 * U' : U_row_ptr[n+1], U_col_idx[nU], U_vals[nU*bs*bs]
 * Any pointer may be NULL to skip that array.  Synchronous. */
int biluk_plan_copy_factors(biluk_plan_t *plan, int64_t *L_row_ptr, int64_t *L_col_idx, double *L_vals,
                            double *dinv, int64_t *U_row_ptr, int64_t *U_col_idx, double *U_vals,
                            void *stream);

/* ------------------------------------------------------------------------
 * Block sparse operator for y = A x -- spmv(a, x), sparse.py:278-301, on
 * the block matrix directly (the reference expands to point CSR first,
 * gmres.py:99 / sparse.py:337-374; the products are the same).
 * ---------------------------------------------------------------------- */
int biluk_op_create(int32_t bs, int64_t n_block_rows, int64_t n_block_cols, const int64_t *row_ptr,
                    const int64_t *col_idx, biluk_op_t **out);
void biluk_op_destroy(biluk_op_t *op);
uint64_t biluk_op_workspace_bytes(const biluk_op_t *op);
int biluk_op_bind(biluk_op_t *op, void *dev_workspace, uint64_t bytes, void *stream);
/* (re)load the block values (nnzb*bs*bs, column-major blocks); asynchronous */
int biluk_op_set_values(biluk_op_t *op, const double *dev_vals, void *stream);
/* y = A x; x has n_block_cols*bs entries, y n_block_rows*bs; asynchronous */
int biluk_op_spmv(biluk_op_t *op, const double *dev_x, double *dev_y, void *stream);

/* ------------------------------------------------------------------------
 * Krylov drivers (gmres.py:76-186; BiCGSTAB is new, see oracle/iluk_oracle.py)
 * The iteration runs on the device; the host only reads the scalars its
 * stopping tests need.  The preconditioner is, in order of precedence, the
 * plan `M` (device apply), the callback `cb` (the reference's opaque `M`
 * callable, gmres.py:85-87, given device pointers), or the identity.
 * ---------------------------------------------------------------------- */
typedef int (*biluk_precond_fn)(void *user, const double *dev_in, double *dev_out, void *stream);

/* Scratch bytes for the solvers (caller-owned device memory), len = n*bs. */
uint64_t biluk_krylov_workspace_bytes(int64_t len, int32_t restart);

/* stats[0]=iterations stats[1]=converged(0/1) stats[2]=final true relative
 * residual  stats[3]=number of history entries produced (history: host array
 * of capacity hist_cap, may be NULL).  dev_x receives the solution (x0 = 0). */
int biluk_bicgstab(biluk_op_t *A, biluk_plan_t *M, biluk_precond_fn cb, void *user, const double *dev_b,
                   double *dev_x, void *dev_work, int64_t max_iters, double rel_tol,
                   double *stats, double *history, int64_t hist_cap, void *stream);

int biluk_gmres(biluk_op_t *A, biluk_plan_t *M, biluk_precond_fn cb, void *user, const double *dev_b,
                double *dev_x, void *dev_work, int32_t restart, int64_t max_iters, double rel_tol,
                double abs_tol, double *stats, double *history, int64_t hist_cap, void *stream);

/* Batched BiCGSTAB over nsys independent systems packed as ONE block-diagonal
 * operator A (and one preconditioner M factored over it, e.g. from
 * biluk_bind of the block-diagonal pattern): system s owns block rows
 * [seg[s], seg[s+1]) (host array, seg[0] = 0, seg[nsys] = n; the caller
 * guarantees A has no entries coupling two segments).  Each system runs the
 * iteration of biluk_bicgstab with its own scalars and stopping tests (the
 * single solve's result up to the preconditioner's rounding); SpMV and
 * preconditioner sweeps run once per step over all systems.  stats: 4 doubles per system, as biluk_bicgstab. */
uint64_t biluk_krylov_batched_workspace_bytes(int64_t len, int32_t nsys);
int biluk_bicgstab_batched(biluk_op_t *A, biluk_plan_t *M, biluk_precond_fn cb, void *user, int32_t nsys,
                           const int64_t *seg, const double *dev_b, double *dev_x, void *dev_work,
                           int64_t max_iters, double rel_tol, double *stats, void *stream);

/* Deterministic FP64 dot product of two device vectors (fixed reduction tree). */
int biluk_dot(const double *dev_a, const double *dev_b, int64_t len, double *result, void *dev_work,
              void *stream);

#ifdef __cplusplus
}
#endif
#endif /* BILUK_H */
