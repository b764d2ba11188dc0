// Internal C++ interface of the DMMA GEMM family (see gemm_dmma.cu).
#pragma once
#include "common.cuh"

namespace qrb {

enum { GEMM_EPI_STORE = 0, GEMM_EPI_SUB = 1 };

// out(M x N) [+ split z * split_stride] = Aview^T * Bview, Aview K x M, Bview K x N.
// K is split into `splits` contiguous ranges, each written to its own slice.
int gemm_tn(const MatView& a_km, const MatView& b, double* out, int64_t ldo, int64_t split_stride,
            int M, int N, int K, int splits, int mask_a, int mask_b, cudaStream_t stream);

// as gemm_tn; *used = number of K slices actually written (<= splits)
int gemm_tn_split(const MatView& a_km, const MatView& b, double* out, int64_t ldo,
                  int64_t split_stride, int M, int N, int K, int splits, int mask_a, int mask_b,
                  cudaStream_t stream, int* used);

// out(M x N) (=|-=) Aview * Bview, Aview M x K, Bview K x N.
int gemm_nn(const MatView& a_mm, const MatView& b, double* out, int64_t ldo, int M, int N, int K,
            int epi, int mask_a, cudaStream_t stream);

// out_z (M x N, z < splits) = Aview[:, K range z] * Bview[K range z, :] (partial products)
int gemm_nn_split(const MatView& a_mm, const MatView& b, double* out, int64_t ldo,
                  int64_t split_stride, int M, int N, int K, int splits, int mask_a,
                  cudaStream_t stream, int* used);

int gemm_pick_splits(int M, int N, int K, int max_splits);
int gemm_tn_split_tiles(int M, int N, int K);
void gemm_set_few_tiles_bn32(int on);
int gemm_few_tiles_bn32();
void gemm_set_few_tiles_min_rows(int rows);
int gemm_few_tiles_min_rows();

// dynamic tile tickets for the persistent NN update (multi-GPU runs, where an
// NCCL kernel can hold SMs while the update starts); static otherwise
void gemm_set_nn_dynamic(bool on);
bool gemm_nn_dynamic();
int gemm_sm_count();

// Upper bound on the CTAs of the GEMMs launched by this host thread (0 = no
// cap): a capped launch runs persistent on that many SMs, leaving the rest to
// work on another stream (the look-ahead panel of qrb_factorize).
void gemm_set_grid_cap(int cap);
int gemm_grid_cap();
struct GemmGridCap {
  int old;
  explicit GemmGridCap(int cap) : old(gemm_grid_cap()) { gemm_set_grid_cap(cap); }
  ~GemmGridCap() { gemm_set_grid_cap(old); }
};

}  // namespace qrb
