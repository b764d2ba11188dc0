// Standalone timing / correctness probe of the CholeskyQR2 small kernels
// (compiled together with csrc/cholqr.cu; no Python).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1907_01891_b200/csrc/cholqr.h"

namespace qrb {
void set_last_error(const std::string&) {}
}

int main() {
  const int b = 128, ld = 128;
  std::vector<double> G(ld * b), A(ld * b);
  srand(1);
  for (int i = 0; i < b * b; ++i) A[i] = (rand() / (double)RAND_MAX) - 0.5 + (i % (b + 1) == 0 ? 8 : 0);
  // G = A^T A (SPD)
  for (int c = 0; c < b; ++c)
    for (int r = 0; r < b; ++r) {
      double s = 0;
      for (int k = 0; k < b; ++k) s += A[k + r * ld] * A[k + c * ld];
      G[r + c * ld] = s;
    }
  double *dG, *dR, *dRi, *dQ, *dU, *dN, *dL, *dUi, *dLi, *ds;
  int* flag;
  cudaMalloc(&dG, 8 * ld * b); cudaMalloc(&dR, 8 * ld * b); cudaMalloc(&dRi, 8 * ld * b);
  cudaMalloc(&dQ, 8 * ld * b); cudaMalloc(&dU, 8 * ld * b); cudaMalloc(&dN, 8 * ld * b);
  cudaMalloc(&dL, 8 * ld * b); cudaMalloc(&dUi, 8 * ld * b); cudaMalloc(&dLi, 8 * ld * b);
  cudaMalloc(&ds, 8 * b); cudaMalloc(&flag, 4);
  cudaMemcpy(dG, G.data(), 8 * ld * b, cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, A.data(), 8 * ld * b, cudaMemcpyHostToDevice);
  cudaMemset(flag, 0, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) qrb::chol_inv(dG, ld, b, dR, dRi, ld, flag, 1, 0, 0);
  cudaEventRecord(e0);
  for (int w = 0; w < 20; ++w) qrb::chol_inv(dG, ld, b, dR, dRi, ld, flag, 1, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("chol_inv: %.1f us\n", ms * 1e3 / 20);
  for (int w = 0; w < 3; ++w) qrb::modified_lu(dQ, ld, b, dU, dN, dL, dUi, dLi, ds, ld, flag, 4, 0);
  cudaEventRecord(e0);
  for (int w = 0; w < 20; ++w) qrb::modified_lu(dQ, ld, b, dU, dN, dL, dUi, dLi, ds, ld, flag, 4, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("modified_lu (+2 inverses): %.1f us\n", ms * 1e3 / 20);
  // check R^T R = G, R Rinv = I
  std::vector<double> R(ld * b), Ri(ld * b);
  cudaMemcpy(R.data(), dR, 8 * ld * b, cudaMemcpyDeviceToHost);
  cudaMemcpy(Ri.data(), dRi, 8 * ld * b, cudaMemcpyDeviceToHost);
  double e1m = 0, e2m = 0, gm = 0;
  for (int c = 0; c < b; ++c)
    for (int r = 0; r < b; ++r) {
      double s = 0, t = 0;
      for (int k = 0; k < b; ++k) {
        s += R[k + r * ld] * R[k + c * ld];
        t += R[r + k * ld] * Ri[k + c * ld];
      }
      e1m = fmax(e1m, fabs(s - G[r + c * ld]));
      gm = fmax(gm, fabs(G[r + c * ld]));
      e2m = fmax(e2m, fabs(t - (r == c)));
    }
  int hf;
  cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost);
  printf("|R^T R - G|/|G| = %.2e  |R Rinv - I| = %.2e  flag %d  %s\n", e1m / gm, e2m, hf,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
