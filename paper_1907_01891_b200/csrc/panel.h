// Internal C++ interface of the panel factorization and helper kernels.
#pragma once
#include "common.cuh"

namespace qrb {

struct PanelPlan {
  int P;   // cooperative CTAs
  int R;   // rows per CTA
  int ib;  // panel width held in shared memory
};

PanelPlan panel_plan(int m, int w_max);
size_t panel_smem_bytes(int R, int ib);
size_t panel_part_doubles(int P, int ib);
int panel_max_ctas();

// Householder QR of an m x w panel in place (R on/above the diagonal, unit-lower
// reflectors below), writes tau[w] and the strict upper Gram entries
// G[c + j*ldg] = v_c . v_j (c < j).
int panel_factor(const MatView& panel, int P, int R, double* tau, double* G, int ldg,
                 double* part, unsigned int* bar, cudaStream_t stream);

// T (w x w upper) from the Gram matrix G and tau (larft forward recurrence).
int build_t(const double* G, int ldg, const double* tau, int w, double* T, int ldt,
            cudaStream_t stream);

int reduce_splits(const double* parts, int64_t split_stride, int splits, int rows, int cols,
                  int64_t ldp, double* out, int64_t ldo, cudaStream_t stream);

// inverses of the 2nb x 2nb diagonal blocks of R (pairs p of nb blocks) from the
// packed nb-block inverses, one launch; out: npairs blocks of 2nb x 2nb (ld 2nb)
int rinv2_pairs(const double* R, int64_t ldr, const double* Rinv, int nb, int npairs, double* out,
                cudaStream_t stream);

int trtri_blocks(const double* A, int64_t lda, int n, int bs, double* Rinv, cudaStream_t stream);

int axpy_block(double alpha, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t rows,
               int64_t cols, cudaStream_t stream);

int column_sumsq(const double* B, int64_t ldb, int r0, int r1, int ncols, double* out,
                 cudaStream_t stream);

}  // namespace qrb
