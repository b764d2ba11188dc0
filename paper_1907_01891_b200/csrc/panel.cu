// Householder panel factorization (geqr2 + the Gram data for larft) as one
// cooperative sm_100a kernel, plus the small kernels around it.
//
// Reference algorithm (per column, dlarfg convention): kernels.py:74-101
//   sigma = ||x2||^2 ; sigma == 0 -> tau = 0, column untouched
//   beta = -copysign(sqrt(alpha^2 + sigma), alpha) ; tau = (beta - alpha) / beta
//   v = x2 / (alpha - beta) ; a[col, col] = beta
//   srow = tau * (a[col, j] + v . a[col+1:, j]) ; a[col, j] -= srow ; a[col+1:, j] -= v * srow
// and the T factor recurrence (kernels.py:134-147):
//   T[k,k] = tau_k ; T[:k, k] = -tau_k * T[:k,:k] @ (V[:, :k]^T v_k)
//
// B200 mapping: the m x ib panel is split into row slabs, one CTA per SM, and
// each slab is held in shared memory for the whole panel (so the BLAS-2 column
// sweep never touches HBM).  Per column there are two grid-wide reductions:
// (1) the column norm, (2) the dot products of v_j with every other panel
// column.  (2) yields both the rank-1 update row (columns > j) and the Gram
// entries V[:, :j]^T v_j needed for T (columns < j) in a single pass.  Partial
// sums go to a global scratch array and are re-summed by every CTA in the same
// fixed order, so every CTA sees bit-identical scalars and the result is
// run-to-run deterministic.
#include "common.cuh"
#include "panel.h"

#include <cmath>

namespace qrb {

namespace {

constexpr int PANEL_THREADS = 512;
constexpr int PANEL_WARPS = PANEL_THREADS / 32;

struct PanelArgs {
  double* A;
  int64_t lda;
  int m;
  int ib;
  int R;  // rows per CTA
  double* tau;
  double* G;  // ib x ib, ld = ib
  int ldg;
  double* part;  // [P][ib + 2] partial sums, then scalar slots
  unsigned int* bar;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block sum; result valid in all threads
__device__ double block_sum(double v, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (warp == 0) {
    s = lane < PANEL_WARPS ? red[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) red[PANEL_WARPS] = s;
  }
  __syncthreads();
  return red[PANEL_WARPS];
}

__global__ void __launch_bounds__(PANEL_THREADS, 1) panel_qr_kernel(PanelArgs p) {
  extern __shared__ double smem_d[];
  const int R = p.R;
  const int ib = p.ib;
  double* slab = smem_d;                 // ib columns x R rows, column-major
  double* dsum = slab + (size_t)ib * R;  // ib reduced dot products
  double* red = dsum + ib;               // PANEL_WARPS + 1
  double* scal = red + PANEL_WARPS + 2;  // tau, scale, beta, skip

  const int P = gridDim.x;
  const int cta = blockIdx.x;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int r0 = cta * R;
  const int nrows = max(0, min(R, p.m - r0));
  const int stride = ib + 2;
  double* my_part = p.part + (size_t)cta * stride;
  double* alpha_slot = p.part + (size_t)P * stride;
  unsigned int nbar = 0;

  for (int idx = tid; idx < ib * R; idx += PANEL_THREADS) {
    const int c = idx / R, lr = idx - c * R;
    slab[idx] = lr < nrows ? p.A[(int64_t)(r0 + lr) + (int64_t)c * p.lda] : 0.0;
  }
  __syncthreads();

  // partial norm of column 0 below the diagonal
  double nrm = 0.0;
  for (int lr = tid; lr < nrows; lr += PANEL_THREADS) {
    if (r0 + lr > 0) {
      const double x = slab[lr];
      nrm += x * x;
    }
  }
  nrm = block_sum(nrm, red);

  const int tpc = PANEL_THREADS / ib;  // threads per column in the dot reduction

  for (int j = 0; j < ib; ++j) {
    const int lj = j - r0;  // local index of the diagonal row (may be out of slab)
    if (tid == 0) {
      my_part[0] = nrm;
      if (lj >= 0 && lj < nrows) *alpha_slot = slab[(size_t)j * R + lj];
    }
    grid_barrier(p.bar, (++nbar) * P);

    if (warp == 0) {
      double s = 0.0;
      for (int c = lane; c < P; c += 32) s += __ldcg(p.part + (size_t)c * stride);
      s = warp_sum(s);
      if (lane == 0) {
        const double alpha = __ldcg(alpha_slot);
        if (s == 0.0) {
          scal[0] = 0.0;
          scal[3] = 1.0;
        } else {
          const double beta = -copysign(sqrt(alpha * alpha + s), alpha);
          scal[0] = (beta - alpha) / beta;
          scal[1] = 1.0 / (alpha - beta);
          scal[2] = beta;
          scal[3] = 0.0;
        }
      }
    }
    __syncthreads();
    const bool skip = scal[3] != 0.0;
    double* vcol = slab + (size_t)j * R;
    const int lstart = max(0, lj);  // first local row with global row >= j

    if (!skip) {
      const double sc = scal[1];
      for (int lr = max(0, lj + 1) + tid; lr < nrows; lr += PANEL_THREADS) vcol[lr] *= sc;
      __syncthreads();
      // partial dots of v_j (unit at row j) with every other panel column
      for (int c = warp; c < ib; c += PANEL_WARPS) {
        if (c == j) continue;
        const double* col = slab + (size_t)c * R;
        double s = 0.0;
        for (int lr = lstart + lane; lr < nrows; lr += 32) {
          const double v = (lr == lj) ? 1.0 : vcol[lr];
          s += col[lr] * v;
        }
        s = warp_sum(s);
        if (lane == 0) my_part[1 + c] = s;
      }
      grid_barrier(p.bar, (++nbar) * P);
      // every CTA re-sums the partial dots in a fixed order
      {
        const int c = tid % ib;
        const int sub = tid / ib;
        double s = 0.0;
        if (sub < tpc)
          for (int b = sub; b < P; b += tpc) s += __ldcg(p.part + (size_t)b * stride + 1 + c);
        // combine the tpc sub-sums through shared memory in fixed order
        double* tmp = slab + (size_t)ib * R + ib + PANEL_WARPS + 8;  // scratch after scal
        if (sub < tpc) tmp[sub * ib + c] = s;
        __syncthreads();
        if (tid < ib) {
          double t = 0.0;
          for (int u = 0; u < tpc; ++u) t += tmp[u * ib + tid];
          dsum[tid] = t;
        }
        __syncthreads();
      }
      const double tau = scal[0];
      if (cta == 0) {
        if (tid < j) p.G[tid + (int64_t)j * p.ldg] = dsum[tid];
        if (tid == 0) p.tau[j] = tau;
      }
      // rank-1 update of the columns right of j (rows >= j in this slab)
      const int ncol = ib - j - 1;
      const int nr = nrows - lstart;
      if (ncol > 0 && nr > 0) {
        for (int idx = tid; idx < ncol * nr; idx += PANEL_THREADS) {
          const int cc = idx / nr;
          const int lr = lstart + (idx - cc * nr);
          const int c = j + 1 + cc;
          const double srow = tau * dsum[c];
          const double v = (lr == lj) ? 1.0 : vcol[lr];
          slab[(size_t)c * R + lr] -= v * srow;
        }
      }
      if (tid == 0 && lj >= 0 && lj < nrows) vcol[lj] = scal[2];
    } else {
      if (cta == 0) {
        if (tid < j) p.G[tid + (int64_t)j * p.ldg] = 0.0;
        if (tid == 0) p.tau[j] = 0.0;
      }
    }
    __syncthreads();
    if (j + 1 < ib) {
      const double* col = slab + (size_t)(j + 1) * R;
      double s = 0.0;
      for (int lr = tid; lr < nrows; lr += PANEL_THREADS)
        if (r0 + lr > j + 1) s += col[lr] * col[lr];
      nrm = block_sum(s, red);
    }
  }

  for (int idx = tid; idx < ib * R; idx += PANEL_THREADS) {
    const int c = idx / R, lr = idx - c * R;
    if (lr < nrows) p.A[(int64_t)(r0 + lr) + (int64_t)c * p.lda] = slab[idx];
  }
}

// T from the Gram matrix: T[k,k] = tau_k, T[:k,k] = -tau_k * T[:k,:k] G[:k,k]
constexpr int BT_THREADS = 512;
__global__ void __launch_bounds__(BT_THREADS) build_t_kernel(const double* G, int ldg,
                                                             const double* tau, int w, double* T,
                                                             int ldt) {
  extern __shared__ double ts[];  // w*w column-major + w (g column)
  double* gcol = ts + (size_t)w * w;
  for (int i = threadIdx.x; i < w * w; i += BT_THREADS) ts[i] = 0.0;
  const int sub_n = BT_THREADS / w >= 4 ? 4 : (BT_THREADS / w >= 2 ? 2 : 1);
  __syncthreads();
  for (int j = 0; j < w; ++j) {
    const double tj = tau[j];
    for (int i = threadIdx.x; i < j; i += BT_THREADS) gcol[i] = G[i + (int64_t)j * ldg];
    __syncthreads();
    if (tj != 0.0 && j > 0) {
      // rows i < j, sub_n threads per row (consecutive lanes)
      const int i = threadIdx.x / sub_n;
      const int sub = threadIdx.x % sub_n;
      double s = 0.0;
      if (i < j)
        for (int l = i + sub; l < j; l += sub_n) s += ts[i + (size_t)l * w] * gcol[l];
      for (int o = sub_n / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, sub_n);
      if (i < j && sub == 0) ts[i + (size_t)j * w] = -tj * s;
    }
    if (threadIdx.x == 0) ts[j + (size_t)j * w] = tj;
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < w * w; idx += BT_THREADS) {
    const int c = idx / w, r = idx - c * w;
    T[r + (int64_t)c * ldt] = ts[idx];
  }
}

// W = sum_s parts[s]   (fixed order, deterministic)
__global__ void reduce_splits_kernel(const double* parts, int64_t split_stride, int splits,
                                     int rows, int cols, int64_t ldp, double* out, int64_t ldo) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / rows, r = idx - c * rows;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += parts[z * split_stride + r + c * ldp];
    out[r + c * ldo] = s;
  }
}

// inverse of each upper-triangular diagonal block of R (block size bs); one CTA
// per block, R_kk staged in shared memory, one thread per inverse column
__global__ void trtri_blocks_kernel(const double* A, int64_t lda, int n, int bs, double* Rinv) {
  extern __shared__ double sm[];
  const int k = blockIdx.x;
  const int i0 = k * bs;
  const int w = min(bs, n - i0);
  double* r = sm;  // w x w
  double* out = Rinv + (int64_t)k * bs * bs;
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
    const int c = idx / w, rr = idx - c * w;
    r[rr + c * w] = rr <= c ? A[(int64_t)(i0 + rr) + (int64_t)(i0 + c) * lda] : 0.0;
  }
  for (int idx = threadIdx.x; idx < bs * bs; idx += blockDim.x) out[idx] = 0.0;
  __syncthreads();
  for (int j = threadIdx.x; j < w; j += blockDim.x) {
    // solve R x = e_j by back substitution -> column j of the inverse
    double* x = out + (int64_t)j * bs;
    x[j] = 1.0 / r[j + j * w];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int l = i + 1; l <= j; ++l) s += r[i + l * w] * x[l];
      x[i] = -s / r[i + i * w];
    }
  }
}

// per-column sum of squares of rows [r0, r1) of a column-major matrix
__global__ void column_sumsq_kernel(const double* B, int64_t ldb, int r0, int r1, double* out) {
  const int col = blockIdx.x;
  const double* c = B + (int64_t)col * ldb;
  double s = 0.0;
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) s += c[r] * c[r];
  __shared__ double red[33];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) out[col] = s;
  }
}

}  // namespace

int panel_max_ctas() {
  static int cap = -1;
  if (cap < 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = sms > 0 ? sms : 148;
  }
  return cap;
}

PanelPlan panel_plan(int m, int w_max) {
  PanelPlan pl;
  const int cap = panel_max_ctas();
  int P = (m + 63) / 64;
  if (P > cap) P = cap;
  if (P < 1) P = 1;
  int R = (m + P - 1) / P;
  R = (R + 1) & ~1;
  P = (m + R - 1) / R;
  const size_t budget = 200 * 1024;
  int ib = 128;
  while (ib > 8 && (size_t)ib * R * 8 + (size_t)ib * 8 * (PANEL_THREADS / ib + 1) > budget) ib >>= 1;
  if (ib > w_max) ib = w_max;
  pl.P = P;
  pl.R = R;
  pl.ib = ib;
  return pl;
}

size_t panel_smem_bytes(int R, int ib) {
  const int tpc = PANEL_THREADS / ib;
  return ((size_t)ib * R + ib + PANEL_WARPS + 8 + (size_t)tpc * ib + 8) * sizeof(double);
}

int panel_factor(const MatView& panel, int P, int R, double* tau, double* G, int ldg,
                 double* part, unsigned int* bar, cudaStream_t stream) {
  const int m = static_cast<int>(panel.rows);
  const int ib = static_cast<int>(panel.cols);
  if (ib < 1 || ib > 128 || m < ib) {
    set_last_error("panel_factor: need 1 <= width <= 128 and rows >= width");
    return QRB_ERR_ARG;
  }
  if ((int64_t)P * R < m || P < 1 || P > panel_max_ctas()) {
    set_last_error("panel_factor: bad row partition");
    return QRB_ERR_ARG;
  }
  const size_t smem = panel_smem_bytes(R, ib);
  static size_t configured = 0;
  if (smem > configured) {
    QRB_CUDA_TRY(cudaFuncSetAttribute(panel_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    configured = smem;
  }
  QRB_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned int), stream));
  PanelArgs a;
  a.A = panel.ptr;
  a.lda = panel.ld;
  a.m = m;
  a.ib = ib;
  a.R = R;
  a.tau = tau;
  a.G = G;
  a.ldg = ldg;
  a.part = part;
  a.bar = bar;
  void* args[] = {&a};
  QRB_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(panel_qr_kernel), dim3(P),
                                           dim3(PANEL_THREADS), args, smem, stream));
  return QRB_OK;
}

int build_t(const double* G, int ldg, const double* tau, int w, double* T, int ldt,
            cudaStream_t stream) {
  const size_t smem = ((size_t)w * w + w) * sizeof(double);
  static size_t configured = 0;
  if (smem > configured) {
    QRB_CUDA_TRY(cudaFuncSetAttribute(build_t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    configured = smem;
  }
  build_t_kernel<<<1, BT_THREADS, smem, stream>>>(G, ldg, tau, w, T, ldt);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int reduce_splits(const double* parts, int64_t split_stride, int splits, int rows, int cols,
                  int64_t ldp, double* out, int64_t ldo, cudaStream_t stream) {
  const int64_t total = (int64_t)rows * cols;
  if (total == 0) return QRB_OK;
  int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 4 * 148));
  reduce_splits_kernel<<<blocks, 256, 0, stream>>>(parts, split_stride, splits, rows, cols, ldp,
                                                   out, ldo);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int trtri_blocks(const double* A, int64_t lda, int n, int bs, double* Rinv, cudaStream_t stream) {
  const int nblk = (n + bs - 1) / bs;
  const size_t smem = (size_t)bs * bs * sizeof(double);
  static size_t configured = 0;
  if (smem > configured) {
    QRB_CUDA_TRY(cudaFuncSetAttribute(trtri_blocks_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    configured = smem;
  }
  trtri_blocks_kernel<<<nblk, 128, smem, stream>>>(A, lda, n, bs, Rinv);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int column_sumsq(const double* B, int64_t ldb, int r0, int r1, int ncols, double* out,
                 cudaStream_t stream) {
  if (ncols <= 0) return QRB_OK;
  column_sumsq_kernel<<<ncols, 256, 0, stream>>>(B, ldb, r0, r1, out);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

}  // namespace qrb
