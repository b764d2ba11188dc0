// Internal C++ interface of the CholeskyQR2 panel pieces (see cholqr.cu).
#pragma once
#include "common.cuh"

namespace qrb {

// R = chol(G) (upper), Rinv = R^-1; b <= 128, outputs b x b with leading dim ldo.
// Raises `bit` in *flag on a non-positive pivot, a non-finite inverse, or (when
// check_identity) ||G - I||_F > 1/2.
int chol_inv(const double* G, int ldg, int b, double* R, double* Rinv, int ldo, int* flag, int bit,
             int check_identity, cudaStream_t stream);

// LU without pivoting of Qt - diag(s), s_k = -sign(current pivot):
// Uc, NUcS = -Uc diag(s), L1 (strict lower), Ucinv, L1invT = L1^-T, s.
int modified_lu(const double* Qt, int ldq, int b, double* Uc, double* NUcS, double* L1,
                double* Ucinv, double* L1invT, double* s, int ldo, int* flag, int bit,
                cudaStream_t stream);

// blocked shared-memory versions of the two above (smallfact.cu); chol_inv /
// modified_lu dispatch to them unless QRB_SWEEP_LEGACY is set
int chol_inv_blk(const double* G, int ldg, int b, double* R, double* Rinv, int ldo, int* flag,
                 int bit, int check_identity, cudaStream_t stream);
int modified_lu_blk(const double* Qt, int ldq, int b, double* Uc, double* NUcS, double* L1,
                    double* Ucinv, double* L1invT, double* s, int ldo, int* flag, int bit,
                    cudaStream_t stream);

// which diagonal steps run barrier-free in one warp (bit 0 Cholesky, 1 LU, 2
// triangular inverse; 7 by default, 0 = the 8-warp barrier versions)
void smallfact_set_diag(int mask);
int smallfact_diag();

// C_p = A_p B_p for up to kMax independent products with M, N, K <= 128
// (column-major, any leading dimensions), one launch
struct SmallMm {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int M, N, K;
};
struct SmallMmBatch {
  static constexpr int kMax = 4;
  SmallMm p[kMax];
  // inside a stream capture: the launch also sets the graph conditional `cond`
  // to (*cond_flag != 0) (saves the one-thread kernel that would do it)
  cudaGraphConditionalHandle cond;
  const int* cond_flag;  // nullptr: no conditional to set
};
int small_mm_batch(const SmallMmBatch& batch, int count, cudaStream_t stream);

// P[0:b,0:b] <- diag(s) R on/above the diagonal, L1 below; tau_k = T_kk; Tout <- T
// (ld ldto) -- only when *flag == 0; otherwise the launch counts one fallback
// panel on the device (cholqr_fallback_count) and writes nothing.
int cholqr_write_top(double* P, int64_t ldp, int b, const double* R, const double* s,
                     const double* L1, const double* T, int64_t ldt, double* tau, int ldo,
                     double* Tout, int64_t ldto, const int* flag, cudaStream_t stream);

// inside a stream capture: sets the graph conditional h to (*flag != 0)
int set_conditional_from_flag(cudaGraphConditionalHandle h, const int* flag, cudaStream_t stream);

// panels (on the current device) whose CholeskyQR2 route fell back to the
// Householder kernels; reads a device counter (synchronous)
int64_t cholqr_fallback_count();

}  // namespace qrb
