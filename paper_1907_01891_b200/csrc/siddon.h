// Internal interface of the GPU Siddon densifier (siddon.cu).
#pragma once
#include "common.cuh"

namespace qrb {

// Write the Siddon intersection lengths of rays [row0, row0 + n_rays) into the
// column-major matrix A (lda); columns are distributed block-cyclically by
// panels of nb over `world` ranks (world = 1: all columns local).  A must be
// zeroed beforehand (absent intersections stay 0).
int siddon_densify(const double* ends, int64_t n_rays, int W, double* A, int64_t lda,
                   int64_t row0, int nb, int world, int rank, int64_t n_local,
                   cudaStream_t stream);

}  // namespace qrb
