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

#include <cstdlib>

namespace qrb {

namespace {

// One CTA of 512 threads per b x b (b <= 128) problem, always padded to 128
// (identity / zero padding that factors trivially), so no thread tests b inside
// a sweep.  Thread t owns column c = t % 128, rows i = g + 4q (g = t / 128,
// q = 0..31) of the working matrix in REGISTERS for a whole sweep.  Each step
// is one barrier: the row the next step needs (and for the LU the column) is
// published to double-buffered shared vectors by the threads that finish it;
// the multiplier vector is published already masked (zero for rows that must
// not change), so the update is the same predicate-free
//     x[q] -= m[g + 4q] * f_c
// for every thread, 8 rows per chunk, chunks skipped warp-uniformly once all
// their rows are finished.
constexpr int SD_THREADS = 512;
constexpr int NP = 128;

struct SdBuf {
  int series;          // G = I + F with ||F|| <= 1e-8: first-order closed form
  double row[2][NP];   // row k of the working matrix (f operands)
  double mul[2][NP];   // masked multipliers
  double piv[NP];
  double rec[NP];
  double sg[NP];
  double red[SD_THREADS / 32];
  int bad;
};

// reciprocal: hardware approximation + two Newton steps (off the IEEE
// division's slow path; within an ulp, which the tolerances allow)
__device__ __forceinline__ double frcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = __fma_rn(-d, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-d, r, 1.0);
  return __fma_rn(r, e, r);
}

// X = U^-1 (x[q] = X(g + 4q, c)) for U upper: strictly upper part in shared
// memory u (ld lu, diagonal and lower part stored as zero), reciprocals of the
// diagonal in sb.rec.  Bottom-up Gauss-Jordan: the unscaled row k of X
// eliminates U(i, k) for i < k; its owners then scale it.  Row k-1 (needed by
// the next step) is published by its owners as soon as their chunk is done.
__device__ void inv_upper_sweep(double (&x)[32], const double* u, int lu, SdBuf& sb) {
  const int t = threadIdx.x, c = t & 127, g = t >> 7;
#pragma unroll
  for (int q = 0; q < 32; ++q) x[q] = (g + 4 * q == c) ? 1.0 : 0.0;
  sb.row[(NP - 1) & 1][c] = (c == NP - 1) ? 1.0 : 0.0;
  __syncthreads();
  for (int k = NP - 1; k >= 0; --k) {
    const double rk = sb.rec[k];
    const double f = sb.row[k & 1][c] * rk;  // X(k, c) = 0 for c < k
    double* rown = sb.row[(k - 1) & 1];
    const double* uk = u + (size_t)k * lu;   // U(i, k), zero for i >= k
    const bool own_k = g == (k & 3), own_k1 = k >= 1 && g == ((k - 1) & 3);
#pragma unroll
    for (int qc = 0; qc < 32; qc += 8) {
      if (g + 4 * qc <= k) {
        double mv[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) mv[v] = uk[g + 4 * (qc + v)];
#pragma unroll
        for (int v = 0; v < 8; ++v) x[qc + v] = __fma_rn(-mv[v], f, x[qc + v]);
        if (own_k && (k >> 2) >= qc && (k >> 2) < qc + 8) {
#pragma unroll
          for (int v = 0; v < 8; ++v)
            if (qc + v == (k >> 2)) x[qc + v] *= rk;
        }
        if (own_k1 && ((k - 1) >> 2) >= qc && ((k - 1) >> 2) < qc + 8) {
#pragma unroll
          for (int v = 0; v < 8; ++v)
            if (qc + v == ((k - 1) >> 2)) rown[c] = x[qc + v];
        }
      }
    }
    __syncthreads();
  }
}

// R = chol(G) (upper, G = R^T R) and R^-1, both written b x b with zero lower part.
// One sweep of symmetric elimination on the upper triangle S of G; the same
// row operations applied to B = I (strictly lower part of the same columns)
// give B = L^-1 of G = L D L^T, so R = D^-1/2 S and R^-T = D^-1/2 L^-1.
// Column c > k updates rows k < i <= c (S), column c <= k rows i > k (B).
__global__ void __launch_bounds__(SD_THREADS, 1)
    chol_inv_kernel(const double* G, int ldg, int b, double* R, double* Rinv, int ldo, int* flag,
                    int bit, int check_identity) {
  __shared__ SdBuf sb;
  const int t = threadIdx.x, c = t & 127, g = t >> 7, lane = t & 31, warp = t >> 5;
  double x[32];
  if (t == 0) sb.bad = 0;
  double fro = 0.0;
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const int i = g + 4 * q;
    double v = (i == c) ? 1.0 : 0.0;
    if (i <= c && c < b) {
      v = G[i + (int64_t)c * ldg];
      const double e = v - (i == c ? 1.0 : 0.0);
      fro += (i == c ? 1.0 : 2.0) * e * e;
    }
    x[q] = v;  // upper: G (identity padding); strictly lower: B = 0
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  if (lane == 0) sb.red[warp] = fro;
  if (g == 0) {
    sb.row[0][c] = x[0];
    sb.mul[0][c] = c > 0 ? x[0] : 0.0;
  }
  __syncthreads();
  if (t == 0) {
    double tot = 0.0;
    for (int w = 0; w < SD_THREADS / 32; ++w) tot += sb.red[w];
    if (check_identity && !(tot <= 0.25)) sb.bad = 1;
    // second CholeskyQR pass on a well-conditioned panel: G = I + F with tiny F.
    // chol(I + F) = I + U + O(||F||^2), (I + U)^-1 = I - U + O(||F||^2) with
    // U = strict_upper(F) + diag(F)/2, so below 1e-8 both are exact to rounding
    // and the 128-step sweep is skipped.
    sb.series = check_identity && tot <= 1e-16;
    double d = sb.row[0][0];
    if (!(d > 0.0 && d < INFINITY)) {
      sb.bad = 1;
      d = 1.0;
    }
    sb.piv[0] = d;
    sb.rec[0] = frcp(d);
  }
  __syncthreads();
  if (sb.series) {
    if (c < b) {
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int i = g + 4 * q;
        if (i < b) {
          const double u = i < c ? x[q] : (i == c ? 0.5 * (x[q] - 1.0) : 0.0);
          R[i + (int64_t)c * ldo] = (i == c ? 1.0 : 0.0) + u;
          Rinv[i + (int64_t)c * ldo] = (i == c ? 1.0 : 0.0) - u;
        }
      }
    }
    return;  // bad is 0 here (the identity check passed)
  }
  for (int k = 0; k < NP; ++k) {
    const double rk = sb.rec[k];
    const double* mul = sb.mul[k & 1];       // S(k, i) for i > k, else 0
    double* rown = sb.row[(k + 1) & 1];
    double* muln = sb.mul[(k + 1) & 1];
    const double f = (c == k ? 1.0 : sb.row[k & 1][c]) * rk;
    const int lim = c > k ? c : NP;          // S rows stop at the diagonal
    const int k1 = k + 1, q1 = k1 >> 2;
    const bool pub = k1 < NP && g == (k1 & 3);
#pragma unroll
    for (int qc = 0; qc < 32; qc += 8) {
      if (g + 4 * (qc + 7) > k) {
        double mv[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) mv[v] = mul[g + 4 * (qc + v)];
#pragma unroll
        for (int v = 0; v < 8; ++v)
          if (g + 4 * (qc + v) <= lim) x[qc + v] = __fma_rn(-mv[v], f, x[qc + v]);
        if (pub && q1 >= qc && q1 < qc + 8) {
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            if (qc + v == q1) {
              const double y = x[qc + v];
              rown[c] = y;
              muln[c] = c > k1 ? y : 0.0;
              if (c == k1) {
                double d = y;
                if (!(d > 0.0 && d < INFINITY)) {
                  sb.bad = 1;
                  d = 1.0;
                }
                sb.piv[c] = d;
                sb.rec[c] = frcp(d);
              }
            }
          }
        }
      }
    }
    __syncthreads();
  }
  for (int r = t; r < NP; r += SD_THREADS) sb.rec[r] = 1.0 / sqrt(sb.piv[r]);
  __syncthreads();
  if (c < b) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int i = g + 4 * q;
      if (i < b) {
        if (i <= c) {
          const double rv = x[q] * sb.rec[i];                  // R(i, c)
          R[i + (int64_t)c * ldo] = rv;
          if (i == c) Rinv[i + (int64_t)c * ldo] = sb.rec[c];  // (i < c) comes from column i
          if (!(fabs(rv) < INFINITY)) sb.bad = 1;
        } else {
          const double xt = x[q] * sb.rec[i];                  // R^-1(c, i) = B(i, c)/sqrt(d_i)
          R[i + (int64_t)c * ldo] = 0.0;
          Rinv[i + (int64_t)c * ldo] = 0.0;
          Rinv[c + (int64_t)i * ldo] = xt;
          if (!(fabs(xt) < INFINITY)) sb.bad = 1;
        }
      }
    }
  }
  __syncthreads();
  if (t == 0 && sb.bad) atomicOr(flag, bit);
}

// Modified LU of Qt - diag(s) (s_k = -sign of the current pivot entry):
//   Uc (upper), NUcS = -Uc diag(s), L1 (strict lower), s.
__global__ void __launch_bounds__(SD_THREADS, 1)
    mlu_kernel(const double* Qt, int ldq, int b, double* Uc, double* NUcS, double* L1,
               double* s_out, int ldo, int* flag, int bit) {
  __shared__ SdBuf sb;
  const int t = threadIdx.x, c = t & 127, g = t >> 7;
  double x[32];
  if (t == 0) sb.bad = 0;
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const int i = g + 4 * q;
    x[q] = (c < b && i < b) ? Qt[i + (int64_t)c * ldq] : 0.0;
  }
  auto pivot = [&](int k, double w) {
    const double sgn = w >= 0.0 ? 1.0 : -1.0;
    const double p = w + sgn;
    sb.sg[k] = -sgn;
    sb.piv[k] = p;
    sb.rec[k] = 1.0 / p;
    if (!(fabs(w) < INFINITY)) sb.bad = 1;
  };
  // row 0 (f operands), column 0 (masked multipliers), pivot 0
  if (g == 0) sb.row[0][c] = x[0];
  if (c == 0) {
#pragma unroll
    for (int q = 0; q < 32; ++q) sb.mul[0][g + 4 * q] = (g + 4 * q > 0) ? x[q] : 0.0;
    if (g == 0) pivot(0, x[0]);
  }
  __syncthreads();
  for (int k = 0; k < NP; ++k) {
    const double rk = sb.rec[k], pk = sb.piv[k];
    const double* mul = sb.mul[k & 1];       // A(i, k) for i > k, else 0
    double* rown = sb.row[(k + 1) & 1];
    double* muln = sb.mul[(k + 1) & 1];
    const double f = c > k ? sb.row[k & 1][c] * rk : 0.0;
    const int k1 = k + 1, q1 = k1 >> 2;
    const bool pub_row = k1 < NP && g == (k1 & 3) && c > k;
    const bool pub_col = c == k1;
#pragma unroll
    for (int qc = 0; qc < 32; qc += 8) {
      if (g + 4 * (qc + 7) >= k) {
        double mv[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) mv[v] = mul[g + 4 * (qc + v)];
        if (c > k) {
#pragma unroll
          for (int v = 0; v < 8; ++v) x[qc + v] = __fma_rn(-mv[v], f, x[qc + v]);
        } else if (c == k) {
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const int i = g + 4 * (qc + v);
            if (i > k) x[qc + v] *= rk;      // column k becomes L(:, k)
            if (i == k) x[qc + v] = pk;      // U(k, k)
          }
        }
        if (pub_col) {
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const int i = g + 4 * (qc + v);
            muln[i] = i > k1 ? x[qc + v] : 0.0;
          }
        }
        if (pub_row && q1 >= qc && q1 < qc + 8) {
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            if (qc + v == q1) {
              rown[c] = x[qc + v];
              if (c == k1) {
                const double w = x[qc + v];
                const double sgn = w >= 0.0 ? 1.0 : -1.0;
                const double p = w + sgn;
                sb.sg[k1] = -sgn;
                sb.piv[k1] = p;
                sb.rec[k1] = frcp(p);
                if (!(fabs(w) < INFINITY)) sb.bad = 1;
              }
            }
          }
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const int i = g + 4 * q;
    const double v = x[q];
    if (c < b && i < b) {
      Uc[i + (int64_t)c * ldo] = i <= c ? v : 0.0;
      NUcS[i + (int64_t)c * ldo] = i <= c ? -v * sb.sg[c] : 0.0;
      L1[i + (int64_t)c * ldo] = i > c ? v : 0.0;
      if (!(fabs(v) < INFINITY)) sb.bad = 1;
    }
  }
  if (t < b) s_out[t] = sb.sg[t];
  __syncthreads();
  if (t == 0 && sb.bad) atomicOr(flag, bit);
}

// CTA 0: Ucinv = Uc^-1;  CTA 1: L1invT = (L1^T)^-1 (unit upper).  Padded to NP
// with the identity.
__global__ void __launch_bounds__(SD_THREADS, 1)
    tri_inv_kernel(const double* Uc, const double* L1, int b, double* Ucinv, double* L1invT,
                   int ldo, int* flag, int bit) {
  extern __shared__ double um[];  // strict upper part, ld NP + 1
  __shared__ SdBuf sb;
  constexpr int LU = NP + 1;
  const int t = threadIdx.x, c = t & 127, g = t >> 7;
  const bool lower = blockIdx.x == 1;
  if (t == 0) sb.bad = 0;
  for (int idx = t; idx < NP * NP; idx += SD_THREADS) {
    const int cc = idx / NP, r = idx - cc * NP;
    double v = 0.0;
    if (r < cc && cc < b) v = lower ? L1[cc + (int64_t)r * ldo] : Uc[r + (int64_t)cc * ldo];
    um[r + (size_t)cc * LU] = v;
  }
  if (t < NP) sb.rec[t] = (lower || t >= b) ? 1.0 : 1.0 / Uc[t + (int64_t)t * ldo];
  __syncthreads();
  double x[32];
  inv_upper_sweep(x, um, LU, sb);
  double* out = lower ? L1invT : Ucinv;
  if (c < b) {
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int i = g + 4 * q;
      if (i < b) {
        out[i + (int64_t)c * ldo] = i <= c ? x[q] : 0.0;
        if (!(fabs(x[q]) < INFINITY)) sb.bad = 1;
      }
    }
  }
  __syncthreads();
  if (t == 0 && sb.bad) atomicOr(flag, bit);
}

// P[0:b, 0:b] <- S R (on/above the diagonal) and L1 (below); tau_k = T_kk;
// Tout <- T.  Runs only when the chain's flag is clear; otherwise it counts the
// panel as a Householder fallback (the predicated fallback kernels follow).
__device__ unsigned long long g_cholqr_fallback_count = 0;

__global__ void cholqr_write_top_kernel(double* P, int64_t ldp, int b, const double* R,
                                        const double* s, const double* L1, const double* T,
                                        int64_t ldt, double* tau, int ldo, double* Tout,
                                        int64_t ldto, const int* flag) {
  if (*reinterpret_cast<const volatile int*>(flag) != 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_cholqr_fallback_count, 1ull);
    return;
  }
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= b * b) return;
  const int c = idx / b, r = idx - c * b;
  P[r + c * ldp] = r <= c ? s[r] * R[r + (int64_t)c * ldo] : L1[r + (int64_t)c * ldo];
  const double tv = T[r + c * ldt];
  Tout[r + c * ldto] = tv;
  if (r == c) tau[c] = tv;
}

// graph capture: the CholeskyQR2 panel's IF node takes the Householder branch
// when the chain raised its flag
__global__ void set_conditional_kernel(cudaGraphConditionalHandle h, const int* flag) {
  cudaGraphSetConditional(h, *reinterpret_cast<const volatile int*>(flag) != 0 ? 1u : 0u);
}

size_t sd_smem(int) { return (size_t)NP * (NP + 1) * sizeof(double); }

}  // namespace

static const bool g_sweep_legacy = std::getenv("QRB_SWEEP_LEGACY") != nullptr;

int chol_inv(const double* G, int ldg, int b, double* R, double* Rinv, int ldo, int* flag, int bit,
             int check_identity, cudaStream_t stream) {
  if (b < 1 || b > 128) {
    set_last_error("chol_inv: b must be in [1, 128]");
    return QRB_ERR_ARG;
  }
  if (!g_sweep_legacy) return chol_inv_blk(G, ldg, b, R, Rinv, ldo, flag, bit, check_identity, stream);
  chol_inv_kernel<<<1, SD_THREADS, 0, stream>>>(G, ldg, b, R, Rinv, ldo, flag, bit,
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
  if (!g_sweep_legacy)
    return modified_lu_blk(Qt, ldq, b, Uc, NUcS, L1, Ucinv, L1invT, s, ldo, flag, bit, stream);
  QRB_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(tri_inv_kernel), sd_smem(128)));
  mlu_kernel<<<1, SD_THREADS, 0, stream>>>(Qt, ldq, b, Uc, NUcS, L1, s, ldo, flag, bit);
  QRB_CUDA_TRY(cudaGetLastError());
  tri_inv_kernel<<<2, SD_THREADS, sd_smem(b), stream>>>(Uc, L1, b, Ucinv, L1invT, ldo, flag, bit);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int cholqr_write_top(double* P, int64_t ldp, int b, const double* R, const double* s,
                     const double* L1, const double* T, int64_t ldt, double* tau, int ldo,
                     double* Tout, int64_t ldto, const int* flag, cudaStream_t stream) {
  const int total = b * b;
  cholqr_write_top_kernel<<<(total + 255) / 256, 256, 0, stream>>>(P, ldp, b, R, s, L1, T, ldt,
                                                                   tau, ldo, Tout, ldto, flag);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int set_conditional_from_flag(cudaGraphConditionalHandle h, const int* flag,
                              cudaStream_t stream) {
  set_conditional_kernel<<<1, 1, 0, stream>>>(h, flag);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int64_t cholqr_fallback_count() {
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_cholqr_fallback_count, sizeof(v)) != cudaSuccess) return -1;
  return static_cast<int64_t>(v);
}

}  // namespace qrb
