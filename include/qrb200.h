/*
 * qrb200 -- C ABI of the B200-native (sm_100a) FP64 blocked Householder QR and
 * multi-slice least-squares solve.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `oocqr` (Python).  The reference exposes the path as two Python functions
 * re-exported from pkg/src/oocqr/__init__.py:9-23:
 *
 *   factorize(a, config, factors_dir, geometry_hash="")   task_engine.py:606-641
 *   solve(factors, b_mat, config, out_dir)                task_engine.py:644-685
 *
 * whose work is dispatched per tile by `_run_kernel` (task_engine.py:287-317)
 * to six numpy/numba kernels (kernels.py:296-455).  The Python mirror in
 * paper_1907_01891_b200/task_engine.py keeps those two signatures and calls
 * this library through ctypes; each entry point below names the reference
 * interface it replaces.
 *
 * Conventions
 *   - all matrices are column-major float64 with an explicit leading dimension
 *     (the reference's on-disk tile order, tile_store.py:25-30);
 *   - return value: 0 = ok; > 0 = singular triangular factor, the value is
 *     1 + the global column the reference would report (kernels.py:423-426
 *     visited bottom-up in tiles of `report_block`, task_engine.py:246-253);
 *     < 0 = error code (QRB_E*), message via qrb_last_error();
 *   - host buffers are borrowed for the duration of a call; device memory owned
 *     by a handle is freed by qrb_destroy; `stream` arguments are cudaStream_t
 *     passed as void* (0 = legacy default stream);
 *   - a handle is single-caller; calls return after the device work finished
 *     unless documented as stream-ordered ("_op_" entry points).
 */
#ifndef QRB200_H
#define QRB200_H

#include <stdint.h>

#if defined(__GNUC__)
#define QRB_API __attribute__((visibility("default")))
#else
#define QRB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define QRB_OK 0
#define QRB_EARG (-1)
#define QRB_ECUDA (-2)
#define QRB_ENOMEM (-3)
#define QRB_ENONFINITE (-4)
#define QRB_ESTATE (-5)
#define QRB_EUNSUPPORTED (-6)

typedef struct qrb_handle qrb_handle;

/* Timing/accounting of one call; mirrors the reference RunReport
 * (task_engine.py:136-181) with device-side (CUDA event) times. */
/* Per-kernel-family accounting, filled when profiling is on (qrb_set_profiling):
 * device time from CUDA events on the launching stream around each launch,
 * algorithmic flops / bytes of those launches. */
typedef struct qrb_kernel_stat {
  double ms;
  double flops;
  double bytes;
  int64_t launches;
} qrb_kernel_stat;

#define QRB_K_PANEL 0   /* panel geqr2 + larft (incl. its inner block updates) */
#define QRB_K_GEMM_TN 1 /* W = V^T C (DMMA, split-K + reduce)                  */
#define QRB_K_GEMM_TT 2 /* W2 = T^T W                                          */
#define QRB_K_GEMM_NN 3 /* C -= V W2 (DMMA)                                    */
#define QRB_K_TRSM 4    /* back substitution                                    */
#define QRB_K_GEMM_NN_CAP 5 /* C -= V W2 on a capped grid beside the look-ahead panel */
#define QRB_K_COUNT 8

typedef struct qrb_report {
  double total_ms;     /* whole call, CUDA events on the handle stream        */
  double panel_ms;     /* panel factorization (geqr2 + larft) share           */
  double update_ms;    /* trailing / Q^T block-reflector updates             */
  double trsm_ms;      /* back substitution                                   */
  double h2d_ms;       /* host -> device copies inside the call               */
  double d2h_ms;       /* device -> host copies inside the call               */
  double flops;        /* algorithmic flops (2mn^2 - 2n^3/3, or 4mn - n^2 per slice) */
  int64_t kernel_launches; /* kernels this library launched for the call     */
  int64_t h2d_bytes;
  int64_t d2h_bytes;
  qrb_kernel_stat kernels[QRB_K_COUNT];
} qrb_report;

/* library */
QRB_API int qrb_version(void);
QRB_API const char* qrb_last_error(void);
QRB_API int qrb_device_count(int* count);
QRB_API int qrb_set_device(int device);

/* ---- handle API (drop-in for factorize / solve) ------------------------ */

/* Allocate an m x n (m >= n) matrix on `device` with panel width nb
 * (reference EngineConfig.inner_block, task_engine.py:77-121).
 * Replaces: factorize's store setup (task_engine.py:614-628). */
QRB_API int qrb_create(int device, int64_t m, int64_t n, int nb, qrb_handle** out);

/* As qrb_create, but over the caller's device matrix A (column-major, ld even
 * and >= m, 16-byte aligned), factored in place; A is not freed by
 * qrb_destroy.  The in-core step of the host-staged (out-of-HBM) engine
 * (ooc.py; replaces the reference's in-cache execution of a tile column's
 * tasks, task_engine.py:330-474). */
QRB_API int qrb_create_view(int device, int64_t m, int64_t n, int nb, double* A, int64_t lda,
                            qrb_handle** out);
QRB_API int qrb_destroy(qrb_handle* h);

/* Copy columns [col0, col0+ncols) of A in/out (column-major, leading dim ld).
 * After qrb_factorize, qrb_get_matrix returns the factored storage: R on and
 * above the diagonal, Householder vectors (implicit unit diagonal) below --
 * the reference `factored` store convention (kernels.py:6-14).
 * Replaces: TiledMatrix load_tile/store_tile staging (tile_store.py:181-209). */
QRB_API int qrb_set_matrix(qrb_handle* h, int64_t col0, int64_t ncols, const double* src, int64_t ld,
                   int src_on_device);
QRB_API int qrb_get_matrix(qrb_handle* h, int64_t col0, int64_t ncols, double* dst, int64_t ld,
                   int dst_on_device);

/* Enqueue the handle's work on `stream` (cudaStream_t as void*; NULL restores the
 * handle's own stream, a blocking stream ordered with the legacy default stream).
 * Use it to order device-pointer calls with a caller's non-default stream. */
QRB_API int qrb_set_stream(qrb_handle* h, void* stream);

/* Enable (1) / disable (0) per-kernel CUDA-event accounting in qrb_report.kernels. */
QRB_API int qrb_set_profiling(qrb_handle* h, int on);

/* In-place blocked Householder QR of the handle's matrix.
 * Replaces: factorize -> execute(gen_factorization_tasks) (task_engine.py:606-641,
 * 187-217) and kernels comp_dense_qr / comp_td_qr / apply_left_qt_* (kernels.py:296-405).
 * Returns QRB_ENONFINITE if A holds NaN/Inf (KernelInputError, kernels.py:305-306). */
QRB_API int qrb_factorize(qrb_handle* h, qrb_report* rep);

/* qrb_set_matrix(host) + qrb_factorize with the PCIe copy overlapped: A (host,
 * column-major, leading dim ld; pinned memory for overlap) is copied in column
 * chunks of `chunk_cols` (0 = automatic) on a copy stream, and each chunk is
 * factored left-looking as soon as it lands -- all earlier panels applied to
 * it, then its own panels -- the reference's left-looking order
 * (task_engine.py:187-217) applied to host->HBM staging.  Same factors and
 * flop count as qrb_factorize; rep->h2d_ms / h2d_bytes report the copy, and
 * rep->total_ms runs from the first copy to the last panel.
 * Replaces: factorize's stage-and-execute sequence (task_engine.py:606-641). */
QRB_API int qrb_factorize_host(qrb_handle* h, const double* src, int64_t ld, int64_t chunk_cols,
                               qrb_report* rep);

/* qrb_factorize_host while the caller is still filling src: the column chunk c
 * (columns [c*chunk_cols, (c+1)*chunk_cols), chunk_cols a multiple of nb) is
 * copied only once ready[c] > 0 (a host int32 per chunk, set by the caller's
 * reader threads after the chunk's columns are in src; ready[c] < 0 aborts the
 * call with QRB_EARG -- the caller could not read the chunk).  progress (optional,
 * page-locked mapped host int64): the library keeps storing there, in stream
 * order, how many leading columns are final, so the caller can stream finished
 * columns out (qrb_get_matrix_async) while the factorization runs.  The first chunks are
 * factored left-looking while later ones are still being read; input_gbps is the
 * arrival rate assumed for switching to the right-looking order (0 = PCIe).
 * Replaces the reference's overlapped mode (one prefetching I/O agent feeding
 * the tile tasks, task_engine.py:330-474) for the in-HBM drop-in factorize. */
QRB_API int qrb_factorize_host_gated(qrb_handle* h, const double* src, int64_t ld,
                                     int64_t chunk_cols, const int32_t* ready, double input_gbps,
                                     int64_t* progress, qrb_report* rep);

/* Columns [col0, col0+ncols) of the handle's matrix to dst on the caller's
 * stream, without waiting (the caller orders it -- e.g. after *progress of
 * qrb_factorize_host_gated covers the columns).  Replaces the reference's
 * eager write-back of finished tiles by its I/O agent (task_engine.py:330-474). */
QRB_API int qrb_get_matrix_async(qrb_handle* h, int64_t col0, int64_t ncols, double* dst,
                                 int64_t ld, void* stream);

/* Persisted-factor interop: tau (n) and the per-panel T factors
 * (nb x nb each, panel k at T + k*nb*ldt... stored as an nb x (npanels*nb) matrix). */
QRB_API int qrb_get_factors(qrb_handle* h, double* tau, double* T, int64_t ldt);
QRB_API int qrb_set_factors(qrb_handle* h, const double* tau, const double* T, int64_t ldt);

/* Merged 2nb x 2nb block reflectors of the panel pairs (2p, 2p+1) of a factored
 * handle, pair p at columns [2nb p, 2nb (p+1)) of a 2nb x (npanels/2 * 2nb)
 * matrix with leading dim ldt2 (zeros where a pair does not exist).  Host or
 * device destination.  Lets later column blocks apply Q^T two panels at a
 * time (K = 2nb GEMMs; kernels.py:324-341 applies one inner panel at a time). */
QRB_API int qrb_get_pair_factors(qrb_handle* h, double* T2, int64_t ldt2);

/* The inverse of qrb_get_pair_factors (after qrb_set_factors): merged pair
 * reflectors someone already formed -- e.g. the multi-GPU factorization, which
 * broadcasts one per column block -- so the solve does not merge them again. */
QRB_API int qrb_set_pair_factors(qrb_handle* h, const double* T2, int64_t ldt2);

/* X = R^-1 (Q^T B)[0:n] for nrhs right-hand sides; resid[j] = ||(Q^T B)[n:m, j]||_2
 * (= ||A x_j - b_j||_2; may be NULL).  B is m x nrhs (ldb), X is n x nrhs (ldx).
 * `on_device` = 1 when B/X/resid are device pointers.  report_block = the tile
 * size whose bottom-up order decides which singular column is reported.
 * Replaces: solve -> execute(gen_solve_tasks) (task_engine.py:644-685, 220-254)
 * with apply_left_qt_* / gemm_nn_mo / trsm_lunn (kernels.py:324-455). */
QRB_API int qrb_solve(qrb_handle* h, const double* B, int64_t ldb, int64_t nrhs, double* X, int64_t ldx,
              double* resid, int on_device, int64_t report_block, qrb_report* rep);

/* Diagonal of R (n values, host).  Used for the singularity rule. */
QRB_API int qrb_get_rdiag(qrb_handle* h, double* diag);

/* ---- stream-ordered device-pointer operators ----------------------------
 * Used by the multi-GPU driver (one process per GPU, NCCL broadcast of each
 * panel between calls) and by the parity tests.  All pointers are device
 * pointers; work is enqueued on `stream` and not synchronized. */

/* Householder QR of an m x w panel (w <= 128) in place + its T factor (w x w,
 * upper).  Replaces comp_dense_qr's panel loop + T builder (kernels.py:80-169). */
QRB_API int qrb_op_panel(double* panel, int64_t ldp, int64_t m, int64_t w, double* tau, double* T,
                 int64_t ldt, void* stream);

/* C <- Q^T C with Q = I - V T V^T, V (m x w, unit lower, stored in place under
 * R) and T (w x w).  Replaces apply_left_qt_dense (kernels.py:324-341). */
QRB_API int qrb_op_apply_qt(const double* V, int64_t ldv, int64_t m, int64_t w, const double* T,
                    int64_t ldt, double* C, int64_t ldc, int64_t nc, void* stream);

/* Householder QR of an m x w block (w <= 2 nb) in place, as two panels: the
 * first nb columns, Q_a^T applied to the rest, the remaining w - nb columns;
 * per-panel T factors in T (two nb x nb column-major blocks, ld nb) and the
 * merged w x w block reflector T2 = [[T_a, -T_a V_a^T V_b T_b], [0, T_b]]
 * (ld ldt2).  side != 0 uses a second library workspace, so the call may run
 * on another stream concurrently with qrb_op_apply_qt_*.  One step of the
 * multi-GPU factorization (dist.py; comp_dense_qr, kernels.py:296-321, for a
 * 2nb-wide tile column). */
QRB_API int qrb_op_panel_block(double* A, int64_t lda, int64_t m, int64_t w, int nb, double* tau,
                               double* T, double* T2, int64_t ldt2, void* stream, int side);

/* qrb_op_apply_qt in two phases: _begin forms W2 = T^T V^T C for all nc
 * columns (kept in the library workspace), _cols then applies C -= V W2 to
 * columns [c_from, c_from + ncols) -- so a look-ahead panel can start after the
 * first columns while the rest is updated (on a capped grid, "grid_cap").
 * The workspace is per device: _begin and its _cols calls must come from one
 * host thread, on one stream, with the same V / m / w, and no other W2-forming
 * call (qrb_solve, qrb_op_apply_qt, qrb_factorize ...) on that device in
 * between -- _cols checks this and returns QRB_ESTATE otherwise. */
QRB_API int qrb_op_apply_qt_begin(const double* V, int64_t ldv, int64_t m, int64_t w,
                                  const double* T, int64_t ldt, const double* C, int64_t ldc,
                                  int64_t nc, void* stream);
QRB_API int qrb_op_apply_qt_cols(const double* V, int64_t ldv, int64_t m, int64_t w, double* C,
                                 int64_t ldc, int64_t c_from, int64_t ncols, void* stream);

/* Reference-format interop: [F; G] <- Q^T [F; G] for a triangle-on-dense tile
 * factorization produced by the reference (D = b x b reflector tile, S = its
 * packed T tile with inner width w, F / G = b x nc blocks).  Replaces
 * apply_left_qt_td (kernels.py:385-405) so the GPU can solve against factors
 * the CPU reference computed (apply_left_qt_dense maps onto qrb_op_apply_qt). */
QRB_API int qrb_op_apply_qt_td(const double* D, int64_t ldd, int64_t b, int64_t w, const double* S,
                               int64_t lds, double* F, int64_t ldf, double* G, int64_t ldg,
                               int64_t nc, void* stream);

/* C <- C - A B (A m x k, B k x n).  Replaces gemm_nn_mo (kernels.py:442-455). */
QRB_API int qrb_op_gemm_nn_sub(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                       int64_t ldc, int64_t m, int64_t n, int64_t k, void* stream);

/* C (M x N) = A^T B with A (K x M), B (K x N); K split into `splits` ranges
 * summed in a fixed order.  mask_a / mask_b: treat that operand as a unit-lower
 * Householder block (upper triangle 0, diagonal 1).  Building block of the
 * W = V^T C step of apply_left_qt_* (kernels.py:337, 400). */
QRB_API int qrb_op_gemm_tn(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                           int64_t ldc, int64_t m, int64_t n, int64_t k, int splits, int mask_a,
                           int mask_b, void* stream);

/* B <- upper(R)^-1 B for an n x n upper-triangular R (block size nb).
 * Replaces trsm_lunn (kernels.py:408-439) for a whole triangular factor. */
QRB_API int qrb_op_trsm_upper(const double* R, int64_t ldr, int64_t n, int nb, double* B, int64_t ldb,
                      int64_t nrhs, void* stream);

/* GPU Siddon densifier (the producer of A; reference analogue: Joseph
 * assemble_system_matrix, ct_model.py:515-547).  `ends` = device array of
 * 4 x n_rays doubles (sx[], sy[], px[], py[]) for global rows [row0, row0+n_rays);
 * writes exact intersection lengths (pixel units) of a W x W image (column
 * index r*W + c, row 0 at +y) into the zeroed column-major A.  Columns are
 * distributed 1D block-cyclically by panels of nb over `world` ranks; this rank
 * holds n_local of them (world = 1: A holds all W*W columns).  Stream-ordered. */
QRB_API int qrb_siddon_densify(const double* ends, int64_t n_rays, int64_t row0, int image_pixels,
                               double* A, int64_t lda, int nb, int world, int rank,
                               int64_t n_local, void* stream);

/* Stream-ordered strided copy of a rows x cols column-major block (pitched);
 * kind: 0 = host->device, 1 = device->host, 2 = device->device, 3 = host->host.
 * The host-staged (out-of-HBM) path streams reflector panels with it
 * (reference analogue: TileCache staging, tile_store.py:225-415). */
QRB_API int qrb_copy_2d(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                        int64_t cols, int kind, void* stream);

/* Kernels launched by this library since load (gpu_launches accounting). */
QRB_API int64_t qrb_launch_count(void);

/* Release all library workspaces of the current device. */
QRB_API int qrb_release_workspace(void);

/* Process-wide tuning knobs and counters (no reference counterpart: the
 * reference's only backend switch is kernels.use_path, kernels.py:265-283).
 *   "panel_algo"       0 auto | 1 Householder columns | 2 CholeskyQR2 when the shape allows
 *   "cholqr_min_rows"  auto mode uses CholeskyQR2 for panels with at least this many rows
 *   "outer_panels"     4 (default): while "outer4_min_cols" (24576) trailing columns remain,
 *                      two panel pairs are merged into one 4nb-wide block reflector
 *                      (K = 4nb trailing-update GEMMs), then pairs (K = 2nb); 2: pairs only;
 *                      1: one panel at a time (qrb_factorize / qrb_factorize_host)
 *   "tn_tail"          1 (default): the W = V^T C product's last partial wave split along K
 *   "nn_dynamic"       1: the persistent trailing-update GEMM hands out tiles dynamically
 *                      (for multi-GPU runs, where NCCL kernels may hold SMs); 0: static
 *   "lookahead"        1 (default): while the trailing update of panel pair s runs on
 *                      capped GEMM grids, pair s+1 is factored on a second (high-priority)
 *                      stream on the remaining SMs; 0: serial; 3: only when the update
 *                      outlasts the modelled panel time.  Results are bitwise identical.
 *   "la_sms"           SMs left to the look-ahead panel (default 16; "la_sms_tall", also 16
 *                      by default, in steps with at least "la_tall_rows" = 32768 rows)
 *   "la_sms_max"       in chain-bound steps (the whole remaining update shorter than the
 *                      modelled chain) the chain is left more SMs, up to this many (72),
 *                      until the two balance
 *   "la_lat_us", "la_margin_pct"  panel-time model sizing the capped part of the update
 *                      (450 us per pair + its GEMM flops on the chain's SMs; +10%)
 *   "few_tiles_bn32"   2 (default): NN products and split TN products with few 128 x 64
 *                      tiles run 128 x 32 tiles (twice the CTAs); 1: NN only; 0: off
 *   "early_singles"    1 (default): factorizations of single panels narrower than 2048
 *                      columns apply each update in two pieces (the next panel's columns
 *                      first) and start the next panel beside the second, which leaves it
 *                      "early_sms" (8) SMs; same arithmetic with and without look-ahead
 *   "la_steps"         (read only) steps that ran with look-ahead
 *   "grid_cap"         CTAs of the GEMMs launched by the calling host thread (0 = no cap)
 *   "sf_diag"          bit mask, 63 by default: the 32-wide diagonal steps of the 128 x 128
 *                      Cholesky (1) / modified LU (2) / triangular inverses (4) of the
 *                      CholeskyQR2 panel run barrier-free in one warp; Cholesky (8) / LU
 *                      (16) with four warps sharing the rows (win over 1 / 2); 32: the
 *                      batched 128^3 products on 16 CTAs each; 0: the 8-warp
 *                      one-barrier-per-column versions (initial value from QRB_SF_DIAG)
 *   "gram_min_rows"    rows of K per CTA when a product has few output tiles (a panel's
 *                      Gram matrices): 32 by default
 *   "sm_count"         (read only) SMs of the current device
 *   "cholqr_panels"    (read only) panels that tried the CholeskyQR2 route
 *   "cholqr_fallbacks" (read only) of those, panels that fell back to Householder columns
 * qrb_set_tuning returns QRB_ERR_ARG for an unknown or read-only key. */
QRB_API int qrb_set_tuning(const char* key, int64_t value);
QRB_API int qrb_get_tuning(const char* key, int64_t* value);

#ifdef __cplusplus
}
#endif

#endif /* QRB200_H */
