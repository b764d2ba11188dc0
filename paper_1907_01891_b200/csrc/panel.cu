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
#include <cstdio>
#include <cstdlib>

namespace qrb {

namespace {

constexpr int PANEL_THREADS = 512;
constexpr int PART_REPL = 1;  // >1 tried: no gain (loads are MLP-bound, not line-bound)
constexpr int PANEL_WARPS = PANEL_THREADS / 32;

struct PanelArgs {
  double* A;
  int64_t lda;
  int m;
  int ib;
  int R;  // rows per CTA
  double* tau;
  double* G;  // ib x ib, ld = ldg
  int ldg;
  double* part;  // 2 x [(ib + 1) * P + ib] partial sums / pivot-row slots
  unsigned int* bar;
  unsigned long long* trace;  // optional per-phase timing (QRB_PANEL_TRACE)
  LaunchPred pred;
};

// loads of data published by other CTAs before the last grid barrier; the
// barrier's acquire already invalidated L1, so plain loads are coherent here
#ifdef QRB_PANEL_LDCG
#define PART_LD(p) __ldcg(p)
#else
#define PART_LD(p) (*(p))
#endif

__device__ __forceinline__ unsigned long long gtimer() {
  return clock64();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One grid-wide reduction per column.  For column j with x = a[j+1:, j]
// (not yet scaled) every CTA publishes, over its own rows r > j,
//     sigma_p = sum x_r^2          d'_p[c] = sum x_r a[r][c]   (all c != j)
// and the CTA owning row j publishes that row.  After one grid barrier all
// CTAs derive beta, tau, scale = 1/(alpha - beta) and
//     d[c] = a[j][c] + scale * sum_p d'_p[c]  = v_j^T a[:, c]
// which is the rank-1 update row for c > j (kernels.py:97-100) and the Gram
// entry V[:, c]^T v_j of the T recurrence for c < j (kernels.py:143-146).
// Partial buffers alternate by column parity, so a CTA that races ahead into
// column j+1 never overwrites partials another CTA is still summing.
template <int OWN>  // columns owned per warp: ceil(ib / 16)
__global__ void __launch_bounds__(PANEL_THREADS, 1) panel_qr_kernel(PanelArgs p) {
  if (pred_off(p.pred)) return;  // uniform over the grid: no CTA reaches a grid barrier
  extern __shared__ double smem_d[];
  const int R = p.R;
  const int ib = p.ib;
  double* slab = smem_d;                 // ib columns x R rows, column-major
  double* red = slab + (size_t)ib * R;   // ib reduced sums
  double* rowj = red + ib;               // ib pivot-row values
  double* scal = rowj + ib;              // tau, scale, beta, skip

  const int P = gridDim.x;
  const int cta = blockIdx.x;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int r0 = cta * R;
  const int nrows = max(0, min(R, p.m - r0));
  // the partial-sum vectors are written PART_REPL times and each CTA reads the
  // copy cta % PART_REPL, so every L2 line is hit by P / PART_REPL readers
  // instead of all P (the all-to-all re-sum is L2 line-contention bound)
  const size_t repl_stride = (size_t)(ib + 1) * P;
  const size_t buf_stride = repl_stride * PART_REPL + ib + 8;
  unsigned int nbar = 0;

  for (int idx = tid; idx < ib * R; idx += PANEL_THREADS) {
    const int c = idx / R, lr = idx - c * R;
    slab[idx] = lr < nrows ? p.A[(int64_t)(r0 + lr) + (int64_t)c * p.lda] : 0.0;
  }
  __syncthreads();

  unsigned long long tph[5] = {0, 0, 0, 0, 0};
  const bool tracing = p.trace != nullptr && tid == 0;
  // column c is owned by warp c % PANEL_WARPS: that warp computes its partial
  // sums, reduces its w_c after the barrier and applies its rank-1 update, so
  // the only intra-CTA synchronisation per column is one __syncthreads.
  constexpr int MAXB = 5;  // partial loads per lane (P <= 160)
  for (int j = 0; j < ib; ++j) {
    unsigned long long ta = tracing ? gtimer() : 0, tb = 0;
    double* part_w = p.part + (size_t)(j & 1) * buf_stride;      // replica 0
    double* part = part_w + (size_t)(cta % PART_REPL) * repl_stride;  // my read replica
    double* prow = part_w + repl_stride * PART_REPL;                // pivot row j
    const int lj = j - r0;
    const bool owner = lj >= 0 && lj < nrows;
    double* x = slab + (size_t)j * R;
    const int lstart = max(0, lj + 1);

    // ---- local partial sums over this slab's rows r > j ----
    {
      double acc[OWN];
#pragma unroll
      for (int i = 0; i < OWN; ++i) acc[i] = 0.0;
      for (int lr = lstart + lane; lr < nrows; lr += 32) {
        const double xv = x[lr];
#pragma unroll
        for (int i = 0; i < OWN; ++i) {
          const int c = warp + i * PANEL_WARPS;
          if (c < ib) acc[i] += xv * slab[(size_t)c * R + lr];
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < OWN; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
      if (lane < OWN) {
        double v = acc[0];
#pragma unroll
        for (int i = 1; i < OWN; ++i)
          if (lane == i) v = acc[i];
        const int c = warp + lane * PANEL_WARPS;
        if (c < ib)  // c == j holds sigma
#pragma unroll
          for (int r = 0; r < PART_REPL; ++r) part_w[r * repl_stride + (size_t)c * P + cta] = v;
      }
    }
    if (owner)
      for (int c = tid; c < ib; c += PANEL_THREADS) prow[c] = slab[(size_t)c * R + lj];
    if (tracing) {
      tb = gtimer();
      tph[0] += tb - ta;
      ta = tb;
    }
    grid_barrier(p.bar, (++nbar) * P);
    if (tracing) {
      tb = gtimer();
      tph[1] += tb - ta;
      ta = tb;
    }

    // ---- every warp re-sums sigma and its own columns' partials (fixed order) ----
    double red_i[OWN], row_i[OWN];
    double sigma, alpha;
    {
      // warp 0 alone fetches sigma / alpha (one reader per CTA for the hot line)
      if (warp == 0) {
        const double* src = part + (size_t)j * P;
        double t = 0.0;
        for (int b = lane; b < P; b += 32) t += PART_LD(src + b);
        t = warp_sum(t);
        if (lane == 0) {
          scal[0] = t;
          scal[1] = PART_LD(prow + j);
        }
      }
      double v[OWN][MAXB];
      double rv[OWN];
#pragma unroll
      for (int i = 0; i < OWN; ++i) {
        const int c = warp + i * PANEL_WARPS;
        const bool need = c < ib && (c > j || (cta == 0 && c < j));
        const double* src = part + (size_t)c * P;
#pragma unroll
        for (int k = 0; k < MAXB; ++k) {
          const int b = lane + 32 * k;
          v[i][k] = (need && b < P) ? PART_LD(src + b) : 0.0;
        }
        rv[i] = (need && lane == i) ? PART_LD(prow + c) : 0.0;
      }
      double sm[OWN];
#pragma unroll
      for (int i = 0; i < OWN; ++i) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < MAXB; ++k) t += v[i][k];
        sm[i] = t;
      }
      if (tracing) {
        double guard = 0.0;
#pragma unroll
        for (int i = 0; i < OWN; ++i) guard += sm[i] + rv[i];
        tb = gtimer() + (guard == 12345.678 ? 1 : 0);
        tph[4] += tb - ta;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < OWN; ++i) sm[i] += __shfl_xor_sync(0xffffffffu, sm[i], o);
#pragma unroll
      for (int i = 0; i < OWN; ++i) {
        red_i[i] = sm[i];
        row_i[i] = __shfl_sync(0xffffffffu, rv[i], i);
      }
      __syncthreads();
      sigma = scal[0];
      alpha = scal[1];
    }
    const bool skip = sigma == 0.0;
    double tau = 0.0, sc = 0.0, beta = 0.0;
    if (!skip) {
      beta = -copysign(sqrt(alpha * alpha + sigma), alpha);
      tau = (beta - alpha) / beta;
      sc = 1.0 / (alpha - beta);
    }
    if (tracing) {
      tb = gtimer();
      tph[2] += tb - ta;
      ta = tb;
    }
    if (cta == 0) {
#pragma unroll
      for (int i = 0; i < OWN; ++i) {
        const int c = warp + i * PANEL_WARPS;
        if (c < j && lane == i) p.G[c + (int64_t)j * p.ldg] = skip ? 0.0 : row_i[i] + sc * red_i[i];
      }
      if (tid == 0) p.tau[j] = tau;
    }
    if (!skip) {
      // rank-1 update of the owned columns c > j on rows >= j of this slab
      const int lfirst = max(0, lj);
#pragma unroll
      for (int i = 0; i < OWN; ++i) {
        const int c = warp + i * PANEL_WARPS;
        if (c > j && c < ib) {
          const double srow = tau * (row_i[i] + sc * red_i[i]);
          double* col = slab + (size_t)c * R;
          for (int lr = lfirst + lane; lr < nrows; lr += 32) {
            const double vv = (lr == lj) ? 1.0 : x[lr] * sc;
            col[lr] -= vv * srow;
          }
        }
      }
    }
    __syncthreads();
    if (!skip && warp == (j % PANEL_WARPS)) {
      // the owner warp turns column j into the reflector (and beta on the diagonal)
      for (int lr = lstart + lane; lr < nrows; lr += 32) x[lr] *= sc;
      if (owner && lane == 0) x[lj] = beta;
      __syncwarp();
    }
    if (tracing) tph[3] += gtimer() - ta;
  }
  __syncthreads();
  if (tracing && (cta == 0 || cta == P - 1)) {
    unsigned long long* t = p.trace + (cta == 0 ? 0 : 4);
    for (int i = 0; i < 4; ++i) atomicAdd(t + i, tph[i]);
    if (cta == 0) atomicAdd(p.trace + 8, tph[4]);
  }

  for (int idx = tid; idx < ib * R; idx += PANEL_THREADS) {
    const int c = idx / R, lr = idx - c * R;
    if (lr < nrows) p.A[(int64_t)(r0 + lr) + (int64_t)c * p.lda] = slab[idx];
  }
}

// T from the Gram matrix: T[k,k] = tau_k, T[:k,k] = -tau_k * T[:k,:k] G[:k,k]
// (kernels.py:134-147).  Blocked by 32: the diagonal 32 x 32 blocks follow the
// column recurrence inside one warp each (warp-synchronous, no block barriers),
// then the off-diagonal blocks are filled block column by block column with
// T[I,J] = -T[I,I..J-1] G[I..J-1, J] T[J,J]-style products that need only one
// __syncthreads per block column:  for the block column J,
//   Z = G[0:j0, J] T[J,J]     (j0 x 32)
//   T[0:j0, J] = -T[0:j0, 0:j0] Z
// which is the recurrence applied 32 columns at a time.
constexpr int BT_THREADS = 512;
__global__ void __launch_bounds__(BT_THREADS) build_t_kernel(const double* G, int ldg,
                                                             const double* tau, int w, double* T,
                                                             int ldt, const LaunchPred pred) {
  if (pred_off(pred)) return;
  extern __shared__ double ts[];  // T: w*w column-major, then Z: w*32
  double* z = ts + (size_t)w * w;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < w * w; i += BT_THREADS) ts[i] = 0.0;
  __syncthreads();
  // strict upper Gram entries, read through the read-only path (tiny, cached)
  auto gs_at = [&](int r, int c) { return __ldg(G + r + (int64_t)c * ldg); };
  const int nblk = (w + 31) / 32;
  // diagonal blocks: warp b handles block b with the plain recurrence
  for (int b = warp; b < nblk; b += BT_THREADS / 32) {
    const int o = b * 32, bw = min(32, w - o);
    for (int j = 0; j < bw; ++j) {
      const double tj = tau[o + j];
      // lane i < j: s_i = sum_{l=i}^{j-1} T[o+i][o+l] G[o+l][o+j]
      double sacc = 0.0;
      if (lane < j)
        for (int l = lane; l < j; ++l) sacc += ts[(o + lane) + (size_t)(o + l) * w] * gs_at(o + l, o + j);
      __syncwarp();
      if (lane < j) ts[(o + lane) + (size_t)(o + j) * w] = (tj != 0.0) ? -tj * sacc : 0.0;
      if (lane == j) ts[(o + j) + (size_t)(o + j) * w] = tj;
      __syncwarp();
    }
  }
  __syncthreads();
  // off-diagonal block columns J = 1..nblk-1
  for (int J = 1; J < nblk; ++J) {
    const int j0 = J * 32, bw = min(32, w - j0);
    // Z[0:j0, 0:bw] = G[0:j0, J] * T[J,J]
    for (int idx = tid; idx < j0 * bw; idx += BT_THREADS) {
      const int c = idx / j0, r = idx - c * j0;
      double sacc = 0.0;
      for (int l = 0; l <= c; ++l) sacc += gs_at(r, j0 + l) * ts[(j0 + l) + (size_t)(j0 + c) * w];
      z[r + (size_t)c * w] = sacc;
    }
    __syncthreads();
    // T[0:j0, J] = -T[0:j0, 0:j0] Z
    for (int idx = tid; idx < j0 * bw; idx += BT_THREADS) {
      const int c = idx / j0, r = idx - c * j0;
      double sacc = 0.0;
      for (int l = r; l < j0; ++l) sacc += ts[r + (size_t)l * w] * z[l + (size_t)c * w];
      ts[r + (size_t)(j0 + c) * w] = -sacc;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < w * w; idx += BT_THREADS) {
    const int c = idx / w, r = idx - c * w;
    T[r + (int64_t)c * ldt] = ts[idx];
  }
}

// W = sum_s parts[s]   (fixed order, deterministic)
// out = sum over z of parts_z.  TPE threads per element (consecutive lanes)
// each sum every TPE-th split in two chains, then combine by xor shuffles: a
// fixed order, so the result is deterministic; more loads in flight than one
// thread per element (the Gram partials are read right after they are written,
// from L2: latency-bound with few elements and many splits)
template <int TPE>
__global__ void reduce_splits_kernel(const double* parts, int64_t split_stride, int splits,
                                     int rows, int cols, int64_t ldp, double* out, int64_t ldo,
                                     const LaunchPred pred) {
  if (pred_off(pred)) return;
  const int64_t total = (int64_t)rows * cols;
  const int sub = threadIdx.x % TPE, lane = threadIdx.x & 31;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / TPE;;
       base += (int64_t)gridDim.x * blockDim.x / TPE) {
    if (base - lane / TPE >= total) break;  // warp-uniform: the shuffles need every lane
    const bool valid = base < total;
    double s0 = 0.0, s1 = 0.0;
    int64_t r = 0, c = 0;
    if (valid) {
      c = base / rows;
      r = base - c * rows;
      const double* src = parts + r + c * ldp;
      int z = sub;
      for (; z + TPE < splits; z += 2 * TPE) {
        s0 += src[(int64_t)z * split_stride];
        s1 += src[(int64_t)(z + TPE) * split_stride];
      }
      if (z < splits) s0 += src[(int64_t)z * split_stride];
    }
    double v = s0 + s1;
#pragma unroll
    for (int o = 1; o < TPE; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (valid && sub == 0) out[r + c * ldo] = v;
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

// Inverses of the 2nb x 2nb diagonal blocks of R for the panel pairs, one CTA
// per pair, from the nb-block inverses:
//   [[A, B], [0, C]]^-1 = [[A^-1, -A^-1 B C^-1], [0, C^-1]]
// (one launch for all pairs instead of two small GEMM launches per pair).
// Block p covers rows/cols [p*2nb, (p+1)*2nb) of R; Rinv holds the nb-block
// inverses (nb x nb each, packed); out gets 2nb x 2nb blocks (ld 2nb).
constexpr int RI2_THREADS = 512;
__global__ void __launch_bounds__(RI2_THREADS) rinv2_kernel(const double* R, int64_t ldr,
                                                            const double* Rinv, int nb,
                                                            double* out) {
  extern __shared__ double zs[];  // Z = A^-1 B, nb x nb, ld nb + 1
  const int p = blockIdx.x;
  const int64_t j0 = (int64_t)p * 2 * nb;
  const double* Ai = Rinv + (int64_t)(2 * p) * nb * nb;
  const double* Ci = Ai + (int64_t)nb * nb;
  const double* Bb = R + j0 + (j0 + nb) * ldr;  // R[j0:j0+nb, j0+nb:j0+2nb]
  const int w2 = 2 * nb, L = nb + 1;
  double* D = out + (int64_t)p * w2 * w2;
  const int t = threadIdx.x;
  const int cg = t / nb, r = t - cg * nb;      // row r, column group cg
  const int ngroups = RI2_THREADS / nb;        // 4 for nb = 128
  // phase 1: Z[r][c] = sum_{l >= r} A^-1[r][l] B[l][c]
  if (cg < ngroups) {
    for (int c0 = cg; c0 < nb; c0 += ngroups * 8) {
      double z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int l = r; l < nb; ++l) {
        const double a = Ai[r + (int64_t)l * nb];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + u * ngroups;
          if (c < nb) z[u] += a * __ldg(Bb + l + (int64_t)c * ldr);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * ngroups;
        if (c < nb) zs[r + c * L] = z[u];
      }
    }
  }
  __syncthreads();
  // phase 2: D12[r][c] = -sum_{l <= c} Z[r][l] C^-1[l][c]; the diagonal blocks copied
  if (cg < ngroups) {
    for (int c = cg; c < nb; c += ngroups) {
      double acc = 0.0;
      for (int l = 0; l <= c; ++l) acc += zs[r + l * L] * __ldg(Ci + l + (int64_t)c * nb);
      D[r + (int64_t)(nb + c) * w2] = -acc;
      D[r + (int64_t)c * w2] = Ai[r + (int64_t)c * nb];
      D[nb + r + (int64_t)(nb + c) * w2] = Ci[r + (int64_t)c * nb];
      D[nb + r + (int64_t)c * w2] = 0.0;
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

// Y += alpha * X on a rows x cols column-major block
__global__ void axpy_block_kernel(double alpha, const double* X, int64_t ldx, double* Y,
                                  int64_t ldy, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / rows, r = idx - c * rows;
    Y[r + c * ldy] += alpha * X[r + c * ldx];
  }
}

}  // namespace

int axpy_block(double alpha, const double* X, int64_t ldx, double* Y, int64_t ldy, int64_t rows,
               int64_t cols, cudaStream_t stream) {
  const int64_t total = rows * cols;
  if (total <= 0) return QRB_OK;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * 148));
  axpy_block_kernel<<<blocks, 256, 0, stream>>>(alpha, X, ldx, Y, ldy, rows, cols);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int panel_max_ctas() {
  static int cap = -1;
  if (cap < 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cap = sms > 0 ? (sms < 160 ? sms : 160) : 148;  // reduce loop handles P <= 160
  }
  return cap;
}

PanelPlan panel_plan(int m, int w_max) {
  PanelPlan pl;
  const int cap = panel_max_ctas();
  static int min_rows = [] {
    const char* e = std::getenv("QRB_PANEL_MINROWS");
    return e ? std::max(16, std::atoi(e)) : 64;
  }();
  int P = (m + min_rows - 1) / min_rows;
  if (P > cap) P = cap;
  if (P < 1) P = 1;
  int R = (m + P - 1) / P;
  R = (R + 1) & ~1;
  P = (m + R - 1) / R;
  const size_t budget = 200 * 1024;
  int ib = 128;
  while (ib > 8 && panel_smem_bytes(R, ib) > budget) ib >>= 1;
  static int ib_cap = [] {
    const char* e = std::getenv("QRB_PANEL_IB");
    return e ? std::atoi(e) : 64;  // measured best cap (r01 sweep, m = 2160 .. 69120)
  }();
  if (ib > ib_cap) ib = ib_cap;
  if (ib > w_max) ib = w_max;
  pl.P = P;
  pl.R = R;
  pl.ib = ib;
  return pl;
}

size_t panel_smem_bytes(int R, int ib) {
  return ((size_t)ib * R + 2 * (size_t)ib + 8) * sizeof(double);
}

size_t panel_part_doubles(int P, int ib) {
  return 2 * ((size_t)(ib + 1) * P * PART_REPL + ib + 8);
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
  void* fn;
  const int own = (ib + PANEL_WARPS - 1) / PANEL_WARPS;
  if (own <= 1)
    fn = reinterpret_cast<void*>(panel_qr_kernel<1>);
  else if (own <= 2)
    fn = reinterpret_cast<void*>(panel_qr_kernel<2>);
  else if (own <= 4)
    fn = reinterpret_cast<void*>(panel_qr_kernel<4>);
  else
    fn = reinterpret_cast<void*>(panel_qr_kernel<8>);
  QRB_TRY(set_max_dynamic_smem(fn, smem));
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
  a.trace = nullptr;
  a.pred = launch_pred();
  static unsigned long long* trace_buf = nullptr;
  static bool trace_on = std::getenv("QRB_PANEL_TRACE") != nullptr;
  if (trace_on) {
    if (!trace_buf) {
      QRB_CUDA_TRY(cudaMallocManaged(&trace_buf, 16 * sizeof(unsigned long long)));
      for (int i = 0; i < 16; ++i) trace_buf[i] = 0;
    }
    a.trace = trace_buf;
  }
  // cooperative launch through cudaLaunchKernelEx (capturable into a graph).
  // Under a launch predicate (the CholeskyQR2 fallback, normally skipped) the
  // launch is NOT cooperative: a cooperative launch waits until all P CTAs fit
  // at once, i.e. behind the look-ahead's capped update on the other SMs, even
  // when every CTA would return at entry (r02: config-2 panel chain 69 -> 123
  // ms).  P <= one CTA per SM and nothing waits on the panel while it runs, so
  // CTAs of a taken fallback that start late only delay the barrier.
  const bool coop = a.pred.flag == nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(PANEL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 1 : 0;
  void* args[] = {&a};
  QRB_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, args));
  if (trace_on) {
    static int calls = 0;
    static double cols_total = 0;
    QRB_CUDA_TRY(cudaStreamSynchronize(stream));
    cols_total += ib;
    if (++calls % 64 == 0)
      std::fprintf(stderr,
                   "[panel trace] %d calls, %.0f cols: per column (kcycles) cta0 local %.2f barrier "
                   "%.2f reduce %.2f (loads %.2f) update %.2f | last cta local %.2f barrier %.2f "
                   "reduce %.2f update %.2f\n",
                   calls, cols_total, trace_buf[0] / cols_total / 1e3,
                   trace_buf[1] / cols_total / 1e3, trace_buf[2] / cols_total / 1e3,
                   trace_buf[8] / cols_total / 1e3,
                   trace_buf[3] / cols_total / 1e3, trace_buf[4] / cols_total / 1e3,
                   trace_buf[5] / cols_total / 1e3, trace_buf[6] / cols_total / 1e3,
                   trace_buf[7] / cols_total / 1e3);
  }
  return QRB_OK;
}

int build_t(const double* G, int ldg, const double* tau, int w, double* T, int ldt,
            cudaStream_t stream) {
  const size_t smem = ((size_t)w * w + (size_t)w * 32) * sizeof(double);
  QRB_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(build_t_kernel), smem));
  build_t_kernel<<<1, BT_THREADS, smem, stream>>>(G, ldg, tau, w, T, ldt, launch_pred());
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int reduce_splits(const double* parts, int64_t split_stride, int splits, int rows, int cols,
                  int64_t ldp, double* out, int64_t ldo, cudaStream_t stream) {
  const int64_t total = (int64_t)rows * cols;
  if (total == 0) return QRB_OK;
  const int tpe = splits <= 8 ? 1 : splits <= 16 ? 2 : splits <= 32 ? 4 : 8;
  // whole warps per grid-stride round, so the shuffles see full groups
  const int64_t threads = ((total * tpe + 127) / 128) * 128;
  const int blocks = static_cast<int>(std::min<int64_t>(threads / 128, 16 * 148));
  switch (tpe) {
    case 1:
      reduce_splits_kernel<1><<<blocks, 128, 0, stream>>>(parts, split_stride, splits, rows, cols,
                                                          ldp, out, ldo, launch_pred());
      break;
    case 2:
      reduce_splits_kernel<2><<<blocks, 128, 0, stream>>>(parts, split_stride, splits, rows, cols,
                                                          ldp, out, ldo, launch_pred());
      break;
    case 4:
      reduce_splits_kernel<4><<<blocks, 128, 0, stream>>>(parts, split_stride, splits, rows, cols,
                                                          ldp, out, ldo, launch_pred());
      break;
    default:
      reduce_splits_kernel<8><<<blocks, 128, 0, stream>>>(parts, split_stride, splits, rows, cols,
                                                          ldp, out, ldo, launch_pred());
  }
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int rinv2_pairs(const double* R, int64_t ldr, const double* Rinv, int nb, int npairs, double* out,
                cudaStream_t stream) {
  if (npairs <= 0) return QRB_OK;
  if (nb < 1 || nb > 128 || RI2_THREADS % nb) {
    set_last_error("rinv2_pairs: nb must divide 512 and be <= 128");
    return QRB_ERR_ARG;
  }
  const size_t smem = (size_t)nb * (nb + 1) * sizeof(double);
  QRB_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(rinv2_kernel), smem));
  rinv2_kernel<<<npairs, RI2_THREADS, smem, stream>>>(R, ldr, Rinv, nb, out);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

int trtri_blocks(const double* A, int64_t lda, int n, int bs, double* Rinv, cudaStream_t stream) {
  const int nblk = (n + bs - 1) / bs;
  const size_t smem = (size_t)bs * bs * sizeof(double);
  QRB_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(trtri_blocks_kernel), smem));
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
