/*
 * pgmres.h -- C-ABI of libpgmres.so, the B200 (sm_100a) hot path of
 * polynomial-preconditioned restarted GMRES(m) (Loe, Thornquist & Boman,
 * arxiv 1907.00072; reference package `polygmres` v0.1.0).
 *
 * Plain C types only: pointers, sizes, doubles.  No torch types cross this
 * boundary.  Device pointers (`const double* d_*`) are caller-owned device
 * allocations; `stream` is a cudaStream_t passed as void*.  Every call is
 * asynchronous on `stream` unless stated; results written to device memory.
 *
 * Status: every function returns int, PG_OK (0) or a negative PG_ERR_* code;
 * pg_last_error() returns the message of the calling thread's last failure.
 * The Python host layer maps the codes onto the reference's exception types
 * (errors.py:4-70): PG_ERR_DIMENSION -> DimensionMismatchError,
 * PG_ERR_PARAMETER -> ParameterError, PG_ERR_CUDA/PG_ERR_ALLOC -> DeviceError.
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/pkg/src/polygmres).  INTEGRATION.md shows the ctypes
 * binding a maintainer adds to the reference to route through this library.
 */
#ifndef PGMRES_H
#define PGMRES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_API __attribute__((visibility("default")))

#define PG_OK 0
#define PG_ERR_DIMENSION (-1)
#define PG_ERR_PARAMETER (-2)
#define PG_ERR_CUDA (-3)
#define PG_ERR_ALLOC (-4)

/* SELL-C-sigma slice height (one warp of rows). */
#define PG_SLICE 32
/* Largest basis / power-sequence width one tall-skinny kernel call accepts;
 * wider bases (restart lengths up to PG_MMAX) are orthogonalized in column
 * tiles of PG_KMAX (pg_cgs2_wide, the native step). */
#define PG_KMAX 64
#define PG_MMAX 256

/* pg_poly_pass flags */
#define PG_PASS_FIRST 1   /* acc = y0*x[row] + yk*(A x)[row]; acc_in unused   */
#define PG_PASS_WRITE_W 2 /* also store w = A x (the next pass's operand)     */

typedef struct pg_matrix pg_matrix;
typedef struct pg_workspace pg_workspace;
typedef struct pg_dist pg_dist;

/* ---- library / errors -------------------------------------------------- */
PG_API int pg_version(void); /* ABI version, currently 1 */
/* 1 when this build carries the device-side invariant checks (PG_CHECKS:
 * ring-slot tags and shared-memory bounds of the asynchronous kernels,
 * libpgmres_checked.so), else 0 */
PG_API int pg_build_checks(void);
PG_API int pg_last_error(char* buf, size_t len);
PG_API int pg_device_count(int* count);
/* Make `device` current for the calling thread (kernels launch on it). */
PG_API int pg_set_device(int device);

/* ---- host-side SELL-C-sigma plan (no GPU needed; used by tests) ----------
 * Replaces the CSR layout of CsrMatrix (sparse.py:42-148) with SELL-C-sigma:
 * rows (optionally length-sorted inside windows of `sigma` rows) are grouped
 * in slices of 32; slice s stores entry j of its lane t at
 * slice_ptr[s] + j*32 + t.  Entry order inside a row is the CSR order, so the
 * device SpMV sums each row in exactly the reference's order.
 * pg_sell_size: padded entry count and slice count for (row_ptr, sigma).
 * pg_sell_fill: fills caller arrays: slice_ptr[n_slices+1], slice_w[n_slices],
 * row_len[n_slices*32], perm[n_slices*32] (-1 = padding lane),
 * col[padded], val[padded]. */
PG_API int pg_sell_size(int64_t nrows, const int64_t* row_ptr, int sigma,
                        int64_t* n_slices, int64_t* padded_nnz);
PG_API int pg_sell_fill(int64_t nrows, int64_t ncols, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* values, int sigma,
                        int64_t* slice_ptr, int32_t* slice_w, int32_t* row_len,
                        int32_t* perm, int32_t* col, double* val);

/* ---- host-side row-pattern plan (no GPU needed; used by tests) ------------
 * The grouping behind the row-pattern and offset-pattern formats, on CSR rows
 * in natural order: rows with identical (column offset[, value bits])
 * sequences share an id (first-seen order); the most frequent sequence is the
 * master; masks[p] = bit set of master positions pattern p uses in order when
 * it is an ordered subsequence of the master (bit 31 set otherwise; all bit
 * 31 when the master is longer than 31).  *npat = -1 (no plan) when there are
 * more than 256 distinct rows.  ids[nrows], masks[256] may be NULL. */
PG_API int pg_row_patterns(int64_t nrows, const int64_t* row_ptr, const int64_t* col_idx,
                           const double* values, int with_values, uint8_t* ids, int* npat,
                           int* master, int* master_len, uint32_t* masks);

/* ---- device operator ------------------------------------------------------
 * Replaces MatrixOperator(matrix) (gmres.py:46-60) / CsrMatrix storage.
 * Host CSR in (int64 row_ptr[nrows+1], int64 col_idx[nnz] in
 * [0, ncols), float64 values[nnz]); the library keeps a device SELL copy.
 * For a row-block shard, ncols = owned rows + ghost columns (local numbering,
 * owned columns first).  `device` is the CUDA ordinal to allocate on. */
PG_API int pg_matrix_create(int device, int64_t nrows, int64_t ncols,
                            const int64_t* row_ptr, const int64_t* col_idx,
                            const double* values, int sigma, pg_matrix** out);
PG_API int pg_matrix_destroy(pg_matrix* mat);
/* stats[12] = {nrows, ncols, nnz, padded_nnz, n_slices, device_bytes,
 *              max_width, sigma, bytes per column entry (1 = dictionary-
 *              compressed offsets, 4 = int32), bytes per value (1 or 8),
 *              matrix-stream bytes per entry of the kernel pg_spmv runs
 *              (1 = pair dictionary, 2 = two dictionary streams, 12 = plain),
 *              that kernel (0 plain SELL, 1 two-stream dictionary, 2 pair
 *              dictionary with global gathers, 3 windowed pair TMA ring,
 *              4 pair dictionary, short uniform rows, 5 row-pattern
 *              dictionary (1 B per row), 6 windowed row patterns, 7 offset
 *              patterns (1 B per row + f64 values), 8 plane marching,
 *              9 plane ring (TMA-staged plane windows))} */
PG_API int pg_matrix_stats(const pg_matrix* mat, int64_t* stats);
/* Launch plan of the plane-ring kernel (stats kernel 9), fixed at creation:
 * plan[10] = {stencil kind (27, 7, 9, 5; 0 = not a plane stencil), tile width
 *            Q, planes per chunk, ring stages, blocks, in-plane halo H,
 *            box level (0: pattern ids read on every plane, 1: none on
 *            interior planes, 2: none at all -- end planes verified too),
 *            stage bytes, shared outer-group products (1: the dz = -1 and
 *            dz = +1 coefficients are equal at every in-plane offset but the
 *            center, each such product is computed once for both rows),
 *            aligned row pairs (1: a row thread's two adjacent rows read
 *            their operands and write their results as 16-byte pairs)}. */
PG_API int pg_plane_plan(const pg_matrix* mat, int64_t* plan);

/* ---- reduction workspace (one per stream) --------------------------------
 * Block partials + a completion counter for the deterministic fixed-order
 * "last block reduces" pattern.  Not shareable between concurrent streams. */
PG_API int pg_workspace_create(int device, pg_workspace** out);
PG_API int pg_workspace_destroy(pg_workspace* ws);

/* ---- SpMV and the fused polynomial pass ------------------------------------
 * pg_spmv: y = A x.  Replaces spmv() (sparse.py:151-168), bitwise: per row
 * a sequential sum in stored column order of separately rounded products.
 * x has ncols entries, y nrows. */
PG_API int pg_spmv(const pg_matrix* mat, const double* d_x, double* d_y, void* stream);

/* One pass of apply_poly's running-power recurrence (polyprec.py:205-211),
 * fused into the SpMV epilogue:
 *   w   = A x
 *   acc = (FIRST ? y0*x[row] : acc_in[row]) + yk*w      (mul, then add)
 *   out = base ? base[row] + acc : acc                  (x + p(A)u, gmres.py:330)
 *   if WRITE_W: w_out[row] = w
 * acc_out may alias acc_in; base may alias acc_out. */
PG_API int pg_poly_pass(const pg_matrix* mat, const double* d_x, const double* d_acc_in,
                        const double* d_base, double* d_acc_out, double* d_w_out,
                        double y0, double yk, int flags, void* stream);

/* One pass of the ROOT-PRODUCT form of the same polynomial (SURVEY row f1,
 * BASELINE north_star "root-product terms, complex-conjugate root pairs in
 * real arithmetic, running sum"): with pi(z) = 1 - z p(z) = prod (1 - z/theta_i)
 * and the invariant prod = v - A y (Loe & Morgan's running sum):
 *   PG_ROOT_REAL   (c1 = 1/theta):  ax = A x; v_out = x - c1*ax; y_out = y_in + c1*x
 *                  [+ c3*v_out: a trailing real root folded in]
 *   PG_ROOT_PAIR_A (c1 = 1/|theta|^2, c2 = 2 Re theta):  ax = A x;
 *                  t2 = c2*x - ax -> v_out; y_out = y_in + c1*t2
 *   PG_ROOT_PAIR_B (c1 = 1/|theta|^2):  ax = A x (x = t2); v_out = p - c1*ax
 *                  [+ y_out = y_in + c3*v_out when c3 != 0]
 * d_y_in may be NULL (running sum starts at zero); v_out may be NULL when the
 * product is not needed again (the final pass); y_out may be NULL when only the
 * product is wanted.
 *   | PG_ROOT_RESID (with REAL or PAIR_B; y_in = v, y_out = NULL):
 *                  v_out = v - (p - c1*ax) -- the last factor of pi(A) v, giving
 *                  A p(A) v = v - pi(A) v directly (the Arnoldi step's
 *                  d+1 passes then never read or write a running sum).
 * d SpMV passes for a degree-d polynomial, like the monomial form; not
 * bit-identical to apply_poly (different evaluation order), parity within the
 * north_star's 1e-10 relative bound at the usable degrees. */
#define PG_ROOT_REAL 0
#define PG_ROOT_PAIR_A 1
#define PG_ROOT_PAIR_B 2
#define PG_ROOT_RESID 4
PG_API int pg_root_pass(const pg_matrix* mat, const double* d_x, const double* d_p,
                        const double* d_y_in, double* d_y_out, double* d_v_out, double c1,
                        double c2, double c3, int mode, void* stream);

/* ---- ILU(0) left preconditioning ---------------------------
 * pg_ilu0_factor: host (no GPU).  Replaces ilu0_factor (ilu.py:38-95): IKJ
 * elimination restricted to the pattern of (row_ptr, col_idx, values) after
 * adding diag_shift to the diagonal, in the reference's operation order (the
 * factors are bit-identical).  out_values[nnz] = combined L\U, out_diag_ptr[n]
 * = position of each diagonal.  On a missing structural diagonal
 * (*fail_kind = 1) or a pivot |u_kk| <= eps*max|diag| (*fail_kind = 2) the
 * failing 0-based row is in *fail_row (PivotError(row)); status stays PG_OK.
 * pg_ilu_create: device copy of the factors (split L / U / diagonal).
 * pg_ilu_apply: z = U^{-1} L^{-1} v (ilu0_apply, ilu.py:98-114) as two
 * sync-free triangular sweeps; d_y is an n-vector scratch (must not alias). */
typedef struct pg_ilu pg_ilu;
PG_API int pg_ilu0_factor(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                          const double* values, double diag_shift, double* out_values,
                          int64_t* out_diag_ptr, int64_t* fail_row, int* fail_kind);
PG_API int pg_ilu_create(int device, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                         const double* values, const int64_t* diag_ptr, pg_ilu** out);
PG_API int pg_ilu_destroy(pg_ilu* ilu);
PG_API int pg_ilu_apply(pg_ilu* ilu, const double* d_v, double* d_y, double* d_z, void* stream);

/* ---- whole steps as single calls (host-overhead reduction) ------------------
 * pg_event_*: a CUDA event owned by the library (record / wait / elapsed ms).
 * pg_poly_chain: out = (base +) p(A) x with the d fused passes of
 *   pg_poly_pass (apply_poly, polyprec.py:193-212; x + p(A)u, gmres.py:330);
 *   d = 0: out = base + y0 x.  Optional ev_start / ev_end bracket the chain.
 * pg_arnoldi_step: one Arnoldi step of solve (gmres.py:282-316) on a
 *   single-shard operator: z = A p(A) v_j (d fused passes + the wrapper SpMV;
 *   d = -1: z = A v_j), CGS2 of z against V[:,0..j] (ortho.py:53-70) with
 *   w2/|w2| into V[:,j+1], the scalars [c1 (PG_KMAX) | c2 (PG_KMAX) | |w2|^2]
 *   into d_ring and copied to the pinned h_ring, then ev_done recorded.  V is
 *   column-major with leading dimension ld.  Bit-identical to issuing the
 *   same entry points one by one.  nroot > 0: z is computed in root-product
 *   form instead (y, d unused): nroot pg_root_pass passes with modes rmode[q]
 *   and constants (c1, c2, c3) = rc[3q .. 3q+2], the last one PG_ROOT_RESID
 *   (RootPlan.resid_steps), with scratch acc (pair temporary), w0, w1.
 *   On matrices pg_chain_fused reports, the step's d+1 passes (or nroot root
 *   passes) run as ONE dependency-driven kernel (temporal blocking across the
 *   passes): bit-identical results, and ev_chain1 is then
 *   recorded after the wrapper SpMV instead of before it.
 * pg_chain_fused: *fused = 1 when pg_arnoldi_step runs its passes as one
 *   kernel on this matrix (natural-order square short-row pair format,
 *   narrow dependency pattern, PG_CHAIN != 0). */
typedef struct pg_event pg_event;
PG_API int pg_chain_fused(const pg_matrix* mat, int* fused);
/* pg_power_sequence: P[:, k] = A P[:, k-1] for k = 1 .. ncols-1 (the power
 * sequence of _power_sequence, polyprec.py:96-112; column 0 holds the unit
 * seed), columns ld apart; one native call, the pg_spmv kernels back to back.
 * Single-shard operators (no halo between the products). */
PG_API int pg_power_sequence(const pg_matrix* mat, double* d_P, int64_t ld, int ncols,
                             void* stream);
/* pg_wrapped_apply: z = A p(A) x, t = p(A) x (PolynomialWrappedOperator.apply,
 * gmres.py:98-113) for d >= 1: the d monomial passes + the wrapper SpMV, as
 * one chain kernel when pg_chain_fused, else pass by pass; acc, w0, w1 are
 * scratch n-vectors.  Bit-identical either way. */
PG_API int pg_wrapped_apply(const pg_matrix* mat, const double* y, int d, const double* d_x,
                            double* d_t, double* d_z, double* d_acc, double* d_w0, double* d_w1,
                            pg_workspace* ws, void* stream);
PG_API int pg_event_create(int device, pg_event** out);
PG_API int pg_event_destroy(pg_event* ev);
PG_API int pg_event_record(pg_event* ev, void* stream);
PG_API int pg_event_wait(pg_event* ev);
PG_API int pg_event_elapsed(pg_event* start, pg_event* end, float* ms);
PG_API int pg_poly_chain(const pg_matrix* mat, const double* y, int d, const double* d_x,
                         const double* d_base, double* d_out, double* d_acc, double* d_w0,
                         double* d_w1, pg_event* ev_start, pg_event* ev_end, void* stream);
PG_API int pg_arnoldi_step(const pg_matrix* mat, const double* y, int d, double* d_V, int64_t ld,
                           int j, double* d_z, double* d_t, double* d_acc, double* d_w0,
                           double* d_w1, double* d_ring, double* h_ring, pg_workspace* ws,
                           pg_event* ev_done, pg_event* ev_chain0, pg_event* ev_chain1,
                           int nroot, const int* rmode, const double* rc, void* stream);
/* The same step recorded once as a CUDA graph (launched later with
 * pg_graph_launch on any stream): for solves repeated with the same operator,
 * polynomial and buffers.  The coefficients and pointers are baked in; the
 * recorded launches carry plain edges (no programmatic serialization). */
typedef struct pg_graph pg_graph;
PG_API int pg_step_graph_create(const pg_matrix* mat, const double* y, int d, double* d_V,
                                int64_t ld, int j, double* d_z, double* d_t, double* d_acc,
                                double* d_w0, double* d_w1, double* d_ring, double* h_ring,
                                pg_workspace* ws, pg_event* ev_done, pg_event* ev_chain0,
                                pg_event* ev_chain1, int nroot, const int* rmode,
                                const double* rc, pg_graph** out);
PG_API int pg_graph_launch(pg_graph* graph, void* stream);
PG_API int pg_graph_destroy(pg_graph* graph);

/* ---- row-block shards over NCCL (csrc/dist.cu; SURVEY §8 row e) ------------
 * One process per GPU.  The halo exchange before every SpMV pass and the
 * batched CGS2 reductions run as NCCL operations issued from C on the solve's
 * stream (libnccl dlopen'ed at run time), so an Arnoldi step stays one native
 * call or one recorded graph per device.  Reductions all-gather every rank's
 * partials and sum them in rank order: identical on every rank and bitwise
 * the in-process multi-shard result.  The reference is single-process
 * (SPEC.md:13); this replaces no reference call but `solve`'s inner loop
 * (gmres.py:282-316) across shards.
 * pg_nccl_unique_id: 128-byte ncclUniqueId (rank 0; broadcast it yourself).
 * pg_dist_create: communicator of `nranks` ranks on `device`.
 * pg_dist_set_halo: this shard's plan -- sends: peer, count and the local
 *   rows to pack (concatenated in send order); receives: peer, ghost offset
 *   (a contiguous range of every vector) and count.
 * pg_dist_halo: fill d_x's ghost slots.  pg_dist_allreduce: rank-order sum of
 *   count (<= 2*PG_KMAX + 8) doubles in place.
 * pg_arnoldi_step_dist / pg_step_graph_create_dist / pg_poly_chain_dist /
 * pg_power_sequence_dist: pg_arnoldi_step & co. with those exchanges between
 * the kernels (the operand's ghosts are filled by the call itself). */
PG_API int pg_nccl_unique_id(void* out, size_t len);
PG_API int pg_dist_create(const void* uid, int nranks, int rank, int device, pg_dist** out);
PG_API int pg_dist_set_halo(pg_dist* dist, int nsend, const int* send_peer,
                            const int64_t* send_count, const int32_t* send_idx, int nrecv,
                            const int* recv_peer, const int64_t* recv_off,
                            const int64_t* recv_count);
PG_API int pg_dist_destroy(pg_dist* dist);
PG_API int pg_dist_halo(pg_dist* dist, double* d_x, void* stream);
PG_API int pg_dist_allreduce(pg_dist* dist, double* d_buf, int count, void* stream);
PG_API int pg_arnoldi_step_dist(const pg_matrix* mat, const double* y, int d, double* d_V,
                                int64_t ld, int j, double* d_z, double* d_t, double* d_acc,
                                double* d_w0, double* d_w1, double* d_ring, double* h_ring,
                                pg_workspace* ws, pg_event* ev_done, pg_event* ev_chain0,
                                pg_event* ev_chain1, int nroot, const int* rmode, const double* rc,
                                pg_dist* dist, void* stream);
PG_API int pg_step_graph_create_dist(const pg_matrix* mat, const double* y, int d, double* d_V,
                                     int64_t ld, int j, double* d_z, double* d_t, double* d_acc,
                                     double* d_w0, double* d_w1, double* d_ring, double* h_ring,
                                     pg_workspace* ws, pg_event* ev_done, pg_event* ev_chain0,
                                     pg_event* ev_chain1, int nroot, const int* rmode,
                                     const double* rc, pg_dist* dist, pg_graph** out);
PG_API int pg_poly_chain_dist(const pg_matrix* mat, const double* y, int d, double* d_x,
                              const double* d_base, double* d_out, double* d_acc, double* d_w0,
                              double* d_w1, pg_event* ev_start, pg_event* ev_end, pg_dist* dist,
                              void* stream);
PG_API int pg_power_sequence_dist(const pg_matrix* mat, double* d_P, int64_t ld, int ncols,
                                  pg_dist* dist, void* stream);

/* r = b - A x and the partial sum of r^2 into d_nsq[0] (gmres.py:334-335). */
PG_API int pg_residual(const pg_matrix* mat, const double* d_x, const double* d_b,
                       double* d_r, double* d_nsq, pg_workspace* ws, void* stream);

/* ---- two-pass classical Gram-Schmidt (ortho.py:33-70) ----------------------
 * V is column-major with leading dimension ld (even); columns 0..k-1 are the
 * basis, 1 <= k <= PG_KMAX; z, w2 have n entries.  Coefficient vectors are
 * device arrays of k doubles (sum over THIS shard's rows; a multi-GPU caller
 * all-reduces them between phases).
 *   phase 1: c1 = V^T z                                      (ortho.py:53)
 *   phase 2: w1 = z - V c1 (on the fly);  c2 = V^T w1         (ortho.py:54-55)
 *   phase 3: w2 = (z - V c1) - V c2;  nsq = sum w2^2          (ortho.py:56,59)
 * then pg_normalize: out = w2 / sqrt(nsq)                    (ortho.py:70) */
PG_API int pg_cgs2_phase1(const double* d_V, int64_t ld, int k, const double* d_z,
                          int64_t n, double* d_c1, pg_workspace* ws, void* stream);
PG_API int pg_cgs2_phase2(const double* d_V, int64_t ld, int k, const double* d_z,
                          int64_t n, const double* d_c1, double* d_c2, pg_workspace* ws,
                          void* stream);
PG_API int pg_cgs2_phase3(const double* d_V, int64_t ld, int k, const double* d_z,
                          int64_t n, const double* d_c1, const double* d_c2, double* d_w2,
                          double* d_nsq, pg_workspace* ws, void* stream);
PG_API int pg_normalize(const double* d_x, const double* d_nsq, int64_t n, double* d_out,
                        void* stream);

/* ---- polynomial construction / recovery helpers ---------------------------
 * pg_gram: G = P^T P for the ncols columns of P -- the Gram blocks of
 * _normal_equations (polyprec.py:115-122) -- accumulated in double-double;
 * d_G receives 2*ncols^2 doubles: G rounded (full symmetric, row-major) then
 * the rounding remainder, so shards can be combined in double-double.
 * pg_gemv: out = V[:, :k] y (gmres.py:326), y a device array of k doubles.
 * pg_dot: d_out[0] = sum x*y (np.linalg.norm's squared sum, gmres.py:241).
 * pg_scale_add: out = (base ? base + a*v : a*v) (polyprec.py:205, gmres.py:330).
 * pg_gather: out[i] = x[idx[i]] (halo packing for row-block shards). */
PG_API int pg_gram(const double* d_P, int64_t ld, int ncols, int64_t n, double* d_G,
                   pg_workspace* ws, void* stream);
PG_API int pg_gemv(const double* d_V, int64_t ld, int k, const double* d_y, int64_t n,
                   double* d_out, void* stream);
/* out = base + sgn * (V[:, :k] y) (base may be NULL: out = sgn * V y); the
 * column tiles of a basis wider than PG_KMAX (gmres.py:326, ortho.py:54-56). */
PG_API int pg_gemv_acc(const double* d_V, int64_t ld, int k, const double* d_y, int64_t n,
                       const double* d_base, double sgn, double* d_out, void* stream);
/* CGS2 of z against a basis of k <= PG_MMAX columns in PG_KMAX-column tiles
 * (k > PG_KMAX; ortho.py:53-59 with the reference's four passes): c1 = V^T z,
 * w1 = z - V c1 (into d_w1, n entries), c2 = V^T w1, w2 = w1 - V c2 into d_w2,
 * nsq = |w2|^2.  d_c1, d_c2 hold k doubles each. */
PG_API int pg_cgs2_wide(const double* d_V, int64_t ld, int k, const double* d_z, int64_t n,
                        double* d_c1, double* d_c2, double* d_nsq, double* d_w1, double* d_w2,
                        pg_workspace* ws, void* stream);
PG_API int pg_dot(const double* d_x, const double* d_y, int64_t n, double* d_out,
                  pg_workspace* ws, void* stream);
PG_API int pg_scale_add(const double* d_base, double a, const double* d_v, int64_t n,
                        double* d_out, void* stream);
PG_API int pg_gather(const double* d_x, const int32_t* d_idx, int64_t m, double* d_out,
                     void* stream);

/* ---- reference-order reductions for the degree decision ---------------------
 * The reference's Cholesky pass/fail and auto_degree choice (polyprec.py:60-93,
 * 150-190) are decided by the rounding of the seed norm and of the Gram matrix,
 * i.e. by the summation order of the BLAS numpy calls (np.linalg.norm -> ddot,
 * polyprec.py:46-51; AV.T @ AV -> syrk, polyprec.py:115-122).  These evaluate
 * both in OpenBLAS 0.3.30's x86-64 order (csrc/blasorder.cu):
 * pg_dot_blas: d_out[0] = x.y as OpenBLAS ddot with `nthreads` (1..32) chunks
 *   (one chunk when n <= 10000) -- bit-identical to numpy's x.dot(y) on a host
 *   whose OpenBLAS runs `nthreads` threads with the SkylakeX/Haswell kernel.
 * pg_gram_blas: upper triangle (packed row-major, (i,j) i<=j) of P^T P over
 *   the ncols columns of P, rows in syrk K-blocks of 384 (halving rule for the
 *   last two), one FMA chain per entry and block, blocks added in order.  For
 *   a row-block shard [g0, g0+n) of N rows: d_state_in (NULL for the first
 *   shard) and d_state_out hold 2*npairs doubles, [open block chains | sum of
 *   completed blocks]; the last shard's sum is the Gram.  d_scratch holds
 *   pg_gram_blas_scratch() doubles.  in and out must not alias. */
PG_API int pg_dot_blas(const double* d_x, const double* d_y, int64_t n, int nthreads,
                       double* d_out, void* stream);
PG_API int pg_gram_blas_scratch(int64_t n, int64_t g0, int64_t N, int ncols, int64_t* doubles);
PG_API int pg_gram_blas(const double* d_P, int64_t ld, int ncols, int64_t n, int64_t g0,
                        int64_t N, const double* d_state_in, double* d_state_out,
                        double* d_scratch, void* stream);

/* ---- host routines (CPU, synchronous) --------------------------------------
 * The small dense steps the reference keeps on the host, natively:
 * pg_host_cholesky_solve: dense_cholesky (polyprec.py:60-93) of the leading
 *   order x order block of row-major G (leading dimension ldg); *failed_pivot
 *   = 0 and y filled on success, else the 1-based pivot failing
 *   pivot <= order*eps*G[k,k].
 * pg_host_degree_select: auto_degree's choice (polyprec.py:171-182): largest
 *   d <= cap whose order-(d+1) system factors with finite y; *degree = -1 if
 *   none.  G, rhs are the cap+1 normal-equation blocks.
 * pg_host_backsolve: y = R[:j,:j]^{-1} g (gmres.py:319-325), R row-major with
 *   leading dimension ldr; *zero_col = index of a zero diagonal (-1 if none;
 *   the caller raises SingularHessenbergError). */
PG_API int pg_host_cholesky_solve(int order, const double* G, int ldg, const double* rhs,
                                  double* y, int* failed_pivot);
PG_API int pg_host_degree_select(int cap, const double* G, int ldg, const double* rhs,
                                 double* y, int* degree);
PG_API int pg_host_backsolve(int j, const double* R, int ldr, const double* g, double* y,
                             int* zero_col);

#ifdef __cplusplus
}
#endif
#endif /* PGMRES_H */
