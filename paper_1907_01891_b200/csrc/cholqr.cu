// Small dense kernels of the CholeskyQR2 + Householder-reconstruction panel.
//
// The reference factors a panel column by column (dlarfg convention,
// kernels.py:74-131): one norm reduction over all m rows per column.  On a
// B200 that is a grid-wide reduction per column (panel.cu), ~7 us each.  For a
// tall panel P (m x b) the same Householder factors can instead be produced
// from BLAS-3 work on the DMMA pipe:
//
//   CholeskyQR2:    G1 = P^T P,  R1 = chol(G1),  Q1 = P R1^-1
//                   G2 = Q1^T Q1, R2 = chol(G2), Q = Q1 R2^-1,  R = R2 R1
//   reconstruction (Ballard et al., "Reconstructing Householder vectors from
//   TSQR"): LU without pivoting of Q - [S; 0], S = diag(s) chosen on the fly
//   as s_k = -sign(w_kk) of the current pivot entry, gives
//                   Q - [S; 0] = L Uc,   V = L (unit lower), U = Uc S,
//                   T = -Uc S L1^-T,    R_householder = S R,  tau_k = T_kk,
//   which are the factors the dlarfg recurrence produces in exact arithmetic
//   (|pivot| = |w_kk| + 1 >= 1, so the LU needs no pivoting).
//
// The kernels here are the b x b (b <= 128) single-CTA pieces: Cholesky +
// triangular inverse, and the modified LU + the two inverses T needs.  The
// m x b products run on the DMMA GEMMs.  Every kernel raises a bit in *flag
// when the factorization is not trustworthy (non-positive Cholesky pivot,
// ||Q1^T Q1 - I||_F > 1/2, non-finite values) so the host can fall back to the
// column-by-column Householder panel before the panel storage is overwritten.
#include "cholqr.h"
#include "common.cuh"

namespace qrb {

namespace {

constexpr int SD_THREADS = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

// In-place inverse of the upper triangle of a (ld L): X = U^-1 with X[r][c]
// (r < c) stored transposed at a[c + r*L] (strictly lower part) and X[c][c] in
// xd[c].  Row-oriented back substitution, 8 threads per column, one barrier
// per row.
__device__ void inv_upper_into_lower(double* a, int L, int b, double* xd) {
  const int tid = threadIdx.x;
  const int jj = tid >> 3, part = tid & 7;
  for (int i = b - 1; i >= 0; --i) {
    const int j = i + 1 + jj;
    double s = 0.0;
    if (j < b) {
      for (int l = i + 1 + part; l <= j; l += 8)
        s += a[i + l * L] * (l == j ? xd[j] : a[j + l * L]);
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    const double xii = 1.0 / a[i + i * L];
    if (part == 0 && j < b) a[j + i * L] = -xii * s;
    if (tid == 0) xd[i] = xii;
    __syncthreads();
  }
}

// In-place inverse of the unit lower triangle of a: Y = L^-1 (unit lower) with
// Y[r][c] (r > c) stored transposed at a[c + r*L] (strictly upper part), i.e.
// the strict upper part then holds L^-T.  Forward, one barrier per row.
__device__ void inv_unit_lower_into_upper(double* a, int L, int b) {
  const int tid = threadIdx.x;
  const int jj = tid >> 3, part = tid & 7;
  for (int i = 1; i < b; ++i) {
    const int j = jj;  // Y[i][j], j < i
    double s = 0.0;
    if (j < i) {
      // Y[i][j] = -sum_{l=j}^{i-1} L[i][l] Y[l][j],  Y[j][j] = 1
      for (int l = j + part; l < i; l += 8) s += a[i + l * L] * (l == j ? 1.0 : a[j + l * L]);
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (part == 0 && j < i) a[j + i * L] = -s;
    __syncthreads();
  }
}

// R = chol(G) (upper, G = R^T R) and R^-1, both written b x b with zero lower part.
__global__ void __launch_bounds__(SD_THREADS, 1)
    chol_inv_kernel(const double* G, int ldg, int b, double* R, double* Rinv, int ldo, int* flag,
                    int bit, int check_identity) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  __shared__ int bad;
  const int L = b + 1;
  double* a = sm;
  double* xd = a + (size_t)b * L;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  double fro = 0.0;
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    if (r <= c) {
      const double v = G[r + (int64_t)c * ldg];
      a[r + c * L] = v;
      const double d = v - (r == c ? 1.0 : 0.0);
      fro += (r == c ? 1.0 : 2.0) * d * d;
    }
  }
  fro = block_sum(fro, red);  // includes a barrier
  if (tid == 0 && (check_identity && !(fro <= 0.25))) bad = 1;
  // right-looking Cholesky on the upper triangle; column j = tid % 128, rows i = g (mod 8)
  const int j = tid & 127, g = tid >> 7;
  for (int k = 0; k < b; ++k) {
    double d = a[k + k * L];
    if (!(d > 0.0 && d < INFINITY)) {
      d = 1.0;
      if (tid == 0) bad = 1;
    }
    if (j > k && j < b) {
      const double akj = a[k + j * L] / d;
      const int i0 = k + 1 + ((g - (k + 1)) & 7);
      for (int i = i0; i <= j; i += 8) a[i + j * L] -= a[k + i * L] * akj;
    }
    __syncthreads();
  }
  // scale rows: R[k][c] = S[k][c] / sqrt(S[k][k])
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    if (r < c) {
      double d = a[r + r * L];
      if (!(d > 0.0 && d < INFINITY)) d = 1.0;
      a[r + c * L] = a[r + c * L] / sqrt(d);
    }
  }
  __syncthreads();
  for (int r = tid; r < b; r += SD_THREADS) {
    double d = a[r + r * L];
    if (!(d > 0.0 && d < INFINITY)) d = 1.0;
    a[r + r * L] = sqrt(d);
  }
  __syncthreads();
  inv_upper_into_lower(a, L, b, xd);
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    const double rv = r <= c ? a[r + c * L] : 0.0;
    const double xv = r < c ? a[c + r * L] : (r == c ? xd[c] : 0.0);
    R[r + (int64_t)c * ldo] = rv;
    Rinv[r + (int64_t)c * ldo] = xv;
    if (!(fabs(xv) < INFINITY)) bad = 1;  // benign race: any writer sets 1
  }
  __syncthreads();
  if (tid == 0 && bad) atomicOr(flag, bit);
}

// Modified LU of Qt - S (Qt b x b, s chosen on the fly), then
//   Uc (upper), NUcS = -Uc S, L1 (strict lower), Ucinv = Uc^-1, L1invT = L1^-T (unit upper), s.
__global__ void __launch_bounds__(SD_THREADS, 1)
    mlu_kernel(const double* Qt, int ldq, int b, double* Uc, double* NUcS, double* L1,
               double* Ucinv, double* L1invT, double* s_out, int ldo, int* flag, int bit) {
  extern __shared__ double sm[];
  __shared__ int bad;
  const int L = b + 1;
  double* a = sm;
  double* xd = a + (size_t)b * L;
  double* piv = xd + b;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    a[r + c * L] = Qt[r + (int64_t)c * ldq];
  }
  __syncthreads();
  const int j = tid & 127, g = tid >> 7;
  for (int k = 0; k < b; ++k) {
    const double w = a[k + k * L];
    const double p = w + (w >= 0.0 ? 1.0 : -1.0);  // w - s_k, s_k = -sign(w)
    if (j > k && j < b) {
      const double ukj = a[k + j * L] / p;
      const int i0 = k + 1 + ((g - (k + 1)) & 7);
      for (int i = i0; i < b; i += 8) a[i + j * L] -= a[i + k * L] * ukj;
    }
    __syncthreads();
  }
  for (int k = tid; k < b; k += SD_THREADS) {
    const double w = a[k + k * L];
    const double sg = w >= 0.0 ? 1.0 : -1.0;
    piv[k] = w + sg;
    s_out[k] = -sg;
    if (!(fabs(w) < INFINITY)) bad = 1;
  }
  __syncthreads();
  // L1[i][k] = a[i][k] / piv_k ; Uc[k][c] = a[k][c] (c > k), Uc[k][k] = piv_k
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    double u = 0.0, l = 0.0;
    if (r > c) {
      l = a[r + c * L] / piv[c];
      a[r + c * L] = l;
    } else if (r == c) {
      u = piv[c];
      a[r + c * L] = u;
    } else {
      u = a[r + c * L];
    }
    Uc[r + (int64_t)c * ldo] = u;
    L1[r + (int64_t)c * ldo] = l;
  }
  __syncthreads();
  // NUcS = -Uc diag(s): column c scaled by -s_c
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    NUcS[r + (int64_t)c * ldo] = r <= c ? -a[r + c * L] * s_out[c] : 0.0;
  }
  __syncthreads();
  // Uc^-1 into the strict lower part (L1 saved to global above)
  inv_upper_into_lower(a, L, b, xd);
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    const double xv = r < c ? a[c + r * L] : (r == c ? xd[c] : 0.0);
    Ucinv[r + (int64_t)c * ldo] = xv;
    if (!(fabs(xv) < INFINITY)) bad = 1;
  }
  __syncthreads();
  // reload L1 into the strict lower part, invert into the strict upper part
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    if (r > c) a[r + c * L] = L1[r + (int64_t)c * ldo];
  }
  __syncthreads();
  inv_unit_lower_into_upper(a, L, b);
  for (int idx = tid; idx < b * b; idx += SD_THREADS) {
    const int c = idx / b, r = idx - c * b;
    const double v = r < c ? a[r + c * L] : (r == c ? 1.0 : 0.0);
    L1invT[r + (int64_t)c * ldo] = v;
    if (!(fabs(v) < INFINITY)) bad = 1;
  }
  __syncthreads();
  if (tid == 0 && bad) atomicOr(flag, bit);
}

// P[0:b, 0:b] <- S R (on/above the diagonal) and L1 (below); tau_k = T_kk
__global__ void cholqr_write_top_kernel(double* P, int64_t ldp, int b, const double* R,
                                        const double* s, const double* L1, const double* T,
                                        int64_t ldt, double* tau, int ldo) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= b * b) return;
  const int c = idx / b, r = idx - c * b;
  P[r + c * ldp] = r <= c ? s[r] * R[r + (int64_t)c * ldo] : L1[r + (int64_t)c * ldo];
  if (r == c) tau[c] = T[c + c * ldt];
}

size_t sd_smem(int b) { return ((size_t)b * (b + 1) + 2 * (size_t)b + 8) * sizeof(double); }

}  // namespace

int chol_inv(const double* G, int ldg, int b, double* R, double* Rinv, int ldo, int* flag, int bit,
             int check_identity, cudaStream_t stream) {
  if (b < 1 || b > 128) {
    set_last_error("chol_inv: b must be in [1, 128]");
    return QRB_ERR_ARG;
  }
  static bool configured = false;
  if (!configured) {
    QRB_CUDA_TRY(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sd_smem(128)));
    configured = true;
  }
  chol_inv_kernel<<<1, SD_THREADS, sd_smem(b), stream>>>(G, ldg, b, R, Rinv, ldo, flag, bit,
                                                          check_identity);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int modified_lu(const double* Qt, int ldq, int b, double* Uc, double* NUcS, double* L1,
                double* Ucinv, double* L1invT, double* s, int ldo, int* flag, int bit,
                cudaStream_t stream) {
  if (b < 1 || b > 128) {
    set_last_error("modified_lu: b must be in [1, 128]");
    return QRB_ERR_ARG;
  }
  static bool configured = false;
  if (!configured) {
    QRB_CUDA_TRY(cudaFuncSetAttribute(mlu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sd_smem(128)));
    configured = true;
  }
  mlu_kernel<<<1, SD_THREADS, sd_smem(b), stream>>>(Qt, ldq, b, Uc, NUcS, L1, Ucinv, L1invT, s,
                                                     ldo, flag, bit);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int cholqr_write_top(double* P, int64_t ldp, int b, const double* R, const double* s,
                     const double* L1, const double* T, int64_t ldt, double* tau, int ldo,
                     cudaStream_t stream) {
  const int total = b * b;
  cholqr_write_top_kernel<<<(total + 255) / 256, 256, 0, stream>>>(P, ldp, b, R, s, L1, T, ldt,
                                                                   tau, ldo);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

}  // namespace qrb
