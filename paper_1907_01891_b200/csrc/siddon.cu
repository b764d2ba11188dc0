// GPU Siddon densifier: exact ray / pixel intersection lengths of a fan-beam
// system matrix written straight into the (column-major, optionally
// block-cyclic) device matrix.
//
// This is the step before the hot path: the reference builds
// its system matrix on the host, ray by ray, with Joseph's method and scatters
// it into tiles (ct_model.py:515-547, _trace_ray_loops :223-275).  The benchmark
// configurations specify Siddon weights; the host restatement is
// paper_1907_01891_b200/ct_system.py::_siddon_block.  This kernel follows the
// same arithmetic (plane crossings alpha = (plane - s) / d, merged in increasing
// order, zero-length segments skipped, pixel = floor of the segment midpoint,
// weight = segment * |P - S|, no FMA contraction) so its output is bit-identical
// to the host version, while never materialising the matrix on the host (the
// 566 GB config-4 matrix cannot be).
//
// One thread per ray.  Endpoints (sx, sy, px, py) come from the host so the
// trigonometry is the same double-precision numpy evaluation.
#include "common.cuh"
#include "siddon.h"

namespace qrb {

namespace {

struct SiddonArgs {
  const double* ends;  // 4 x n_rays: sx[], sy[], px[], py[]
  int64_t n_rays;
  int W;
  double* A;
  int64_t lda;
  int64_t row0;  // global row of this call's first ray
  int nb, world, rank;  // block-cyclic column ownership (world = 1: plain)
  int64_t n_local;      // local columns held by this rank
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

__global__ void siddon_kernel(SiddonArgs a) {
  const int64_t ray = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (ray >= a.n_rays) return;
  const double sx = a.ends[ray], sy = a.ends[a.n_rays + ray];
  const double px = a.ends[2 * a.n_rays + ray], py = a.ends[3 * a.n_rays + ray];
  const int W = a.W;
  const double half = W / 2.0;
  const double dx = dsub(px, sx), dy = dsub(py, sy);
  const double length = sqrt(dadd(dmul(dx, dx), dmul(dy, dy)));
  const double lo_plane = 0.0 - half, hi_plane = static_cast<double>(W) - half;

  double amin = 0.0, amax = 1.0;
  bool hit = true;
  if (dx != 0.0) {
    const double a0 = __ddiv_rn(dsub(lo_plane, sx), dx), a1 = __ddiv_rn(dsub(hi_plane, sx), dx);
    amin = fmax(amin, fmin(a0, a1));
    amax = fmin(amax, fmax(a0, a1));
  } else if (!(sx > -half && sx < half)) {
    hit = false;
  }
  if (dy != 0.0) {
    const double a0 = __ddiv_rn(dsub(lo_plane, sy), dy), a1 = __ddiv_rn(dsub(hi_plane, sy), dy);
    amin = fmax(amin, fmin(a0, a1));
    amax = fmin(amax, fmax(a0, a1));
  } else if (!(sy > -half && sy < half)) {
    hit = false;
  }
  if (!hit || !(amax > amin)) return;

  // iterate the x- and y-plane crossings in increasing alpha
  int ix = dx > 0.0 ? 0 : W, stepx = dx > 0.0 ? 1 : -1;
  int iy = dy > 0.0 ? 0 : W, stepy = dy > 0.0 ? 1 : -1;
  auto ax_at = [&](int i) {
    return dx != 0.0 ? __ddiv_rn(dsub(static_cast<double>(i) - half, sx), dx) : 2.0;
  };
  auto ay_at = [&](int i) {
    return dy != 0.0 ? __ddiv_rn(dsub(static_cast<double>(i) - half, sy), dy) : 2.0;
  };
  // skip crossings below the entry point (the host keeps alpha >= amin)
  double axn = ax_at(ix), ayn = ay_at(iy);
  while (dx != 0.0 && ix >= 0 && ix <= W && axn < amin) {
    ix += stepx;
    axn = (ix >= 0 && ix <= W) ? ax_at(ix) : 2.0;
  }
  if (dx == 0.0 || ix < 0 || ix > W) axn = 2.0;
  while (dy != 0.0 && iy >= 0 && iy <= W && ayn < amin) {
    iy += stepy;
    ayn = (iy >= 0 && iy <= W) ? ay_at(iy) : 2.0;
  }
  if (dy == 0.0 || iy < 0 || iy > W) ayn = 2.0;

  const int64_t grow = a.row0 + ray;
  double acur = amin;
  while (true) {
    double anext = fmin(fmin(axn, ayn), amax);
    if (anext > acur) {
      const double seg = dsub(anext, acur);
      const double mid = dadd(acur, dmul(0.5, seg));
      const double xm = dadd(sx, dmul(mid, dx));
      const double ym = dadd(sy, dmul(mid, dy));
      const int c = static_cast<int>(floor(dadd(xm, half)));
      const int r = static_cast<int>(floor(dsub(half, ym)));
      if (c >= 0 && c < W && r >= 0 && r < W) {
        const int64_t col = static_cast<int64_t>(r) * W + c;
        int64_t lcol = col;
        bool mine = true;
        if (a.world > 1) {
          const int64_t k = col / a.nb;
          mine = (k % a.world) == a.rank;
          lcol = (k / a.world) * a.nb + (col - k * a.nb);
        }
        if (mine && lcol < a.n_local) a.A[grow + lcol * a.lda] = dmul(seg, length);
      }
      acur = anext;
    }
    if (anext >= amax) break;
    if (axn <= ayn) {
      ix += stepx;
      axn = (ix >= 0 && ix <= W) ? ax_at(ix) : 2.0;
    } else {
      iy += stepy;
      ayn = (iy >= 0 && iy <= W) ? ay_at(iy) : 2.0;
    }
    if (axn > 1.5 && ayn > 1.5 && acur >= amax) break;
  }
}

}  // namespace

int siddon_densify(const double* ends, int64_t n_rays, int W, double* A, int64_t lda,
                   int64_t row0, int nb, int world, int rank, int64_t n_local,
                   cudaStream_t stream) {
  if (n_rays <= 0) return QRB_OK;
  SiddonArgs a{ends, n_rays, W, A, lda, row0, nb, world, rank, n_local};
  const int threads = 128;
  const int64_t blocks = (n_rays + threads - 1) / threads;
  siddon_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(a);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

}  // namespace qrb
