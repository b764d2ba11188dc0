// Standalone correctness / timing probe of the blocked small factorizations
// (csrc/smallfact.cu) against their definitions and against the sweep kernels
// (csrc/cholqr.cu).  Build (here; -DSF_TRACE adds per-phase cycle counts) and
// run on the GPU box:
//   nvcc -DSF_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     -o tools/probe/smallfact_probe tools/probe/smallfact_probe.cu \
//     paper_1907_01891_b200/csrc/cholqr.cu paper_1907_01891_b200/csrc/smallfact.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "../../paper_1907_01891_b200/csrc/cholqr.h"

namespace qrb {
void set_last_error(const std::string& m) { fprintf(stderr, "err: %s\n", m.c_str()); }
int set_max_dynamic_smem(const void* f, size_t bytes) {  // once per kernel, like the library
  static std::map<const void*, size_t> done;
  if (done[f] >= bytes) return 0;
  done[f] = bytes;
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) ==
                 cudaSuccess
             ? 0
             : -1;
}
#ifdef SF_TRACE
void smallfact_trace(long long* out);
#endif
}  // namespace qrb

static const int LD = 128;
using Mat = std::vector<double>;

static double maxabs(const Mat& a) {
  double m = 0;
  for (double v : a) m = std::fmax(m, std::fabs(v));
  return m;
}
static Mat mul(const Mat& a, const Mat& b, int n) {  // column-major n x n, ld LD
  Mat c(LD * LD, 0.0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const double bk = b[k + j * LD];
      if (bk == 0.0) continue;
      for (int i = 0; i < n; ++i) c[i + j * LD] += a[i + k * LD] * bk;
    }
  return c;
}
static double err_identity(const Mat& a, int n) {
  double e = 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) e = std::fmax(e, std::fabs(a[i + j * LD] - (i == j)));
  return e;
}

struct Dev {
  double* p;
  explicit Dev(size_t n) { cudaMalloc(&p, n * 8); cudaMemset(p, 0, n * 8); }
  ~Dev() { cudaFree(p); }
  Mat get(size_t n = LD * LD) const {
    Mat h(n);
    cudaMemcpy(h.data(), p, n * 8, cudaMemcpyDeviceToHost);
    return h;
  }
  void put(const Mat& h) { cudaMemcpy(p, h.data(), h.size() * 8, cudaMemcpyHostToDevice); }
};

template <class F>
static float time_us(F f, int reps = 50) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

int main() {
  int fails = 0;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  for (int b : {128, 96, 34}) {
    // ---- Cholesky + inverse of G = A^T A
    Mat A(LD * LD, 0.0), G(LD * LD, 0.0);
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) A[i + j * LD] = nd(rng) + (i == j ? 6.0 : 0.0);
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) {
        double s = 0;
        for (int k = 0; k < b; ++k) s += A[k + i * LD] * A[k + j * LD];
        G[i + j * LD] = s;
      }
    Dev dG(LD * LD), dR(LD * LD), dRi(LD * LD), dR0(LD * LD), dRi0(LD * LD);
    int* flag;
    cudaMalloc(&flag, 4);
    cudaMemset(flag, 0, 4);
    dG.put(G);
    qrb::chol_inv_blk(dG.p, LD, b, dR.p, dRi.p, LD, flag, 1, 0, 0);
    cudaDeviceSynchronize();
    Mat R = dR.get(), Ri = dRi.get();
    Mat RtR(LD * LD, 0.0);
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) {
        double s = 0;
        for (int k = 0; k < b; ++k) s += R[k + i * LD] * R[k + j * LD];
        RtR[i + j * LD] = s - G[i + j * LD];
      }
    const double e1 = maxabs(RtR) / maxabs(G), e2 = err_identity(mul(R, Ri, b), b);
    bool lowz = true;
    for (int j = 0; j < b; ++j)
      for (int i = j + 1; i < b; ++i) lowz &= R[i + j * LD] == 0.0 && Ri[i + j * LD] == 0.0;
    int hf;
    cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost);
    const bool ok1 = e1 < 1e-14 && e2 < 1e-12 && lowz && hf == 0;
    fails += !ok1;
    const float tb = time_us([&] { qrb::chol_inv_blk(dG.p, LD, b, dR.p, dRi.p, LD, flag, 1, 0, 0); });
    const float tl = time_us([&] { qrb::chol_inv(dG.p, LD, b, dR0.p, dRi0.p, LD, flag, 1, 0, 0); });
    {
      Mat Gi(LD * LD, 0.0);
      for (int j = 0; j < b; ++j)
        for (int i = 0; i <= j; ++i) Gi[i + j * LD] = (i == j) + 1e-12 * nd(rng);
      Dev dGi(LD * LD);
      dGi.put(Gi);
      const float ts = time_us([&] { qrb::chol_inv_blk(dGi.p, LD, b, dR0.p, dRi0.p, LD, flag, 2, 1, 0); });
      printf("b=%3d chol closed form (second pass): %.1f us\n", b, ts);
    }
    printf("b=%3d chol_blk: |RtR-G|/|G| %.2e |R Rinv - I| %.2e lower0 %d flag %d  %s  %.1f us "
           "(chol_inv default path %.1f us)\n",
           b, e1, e2, (int)lowz, hf, ok1 ? "OK" : "FAIL", tb, tl);

    // ---- modified LU of the top block of an orthonormal Q
    Mat Q(LD * LD, 0.0);
    {
      const int m = 3 * b;
      std::vector<double> P((size_t)m * b);
      for (auto& v : P) v = nd(rng);
      for (int j = 0; j < b; ++j) {  // modified Gram-Schmidt, twice
        for (int pass = 0; pass < 2; ++pass)
          for (int k = 0; k < j; ++k) {
            double s = 0;
            for (int i = 0; i < m; ++i) s += P[i + (size_t)k * m] * P[i + (size_t)j * m];
            for (int i = 0; i < m; ++i) P[i + (size_t)j * m] -= s * P[i + (size_t)k * m];
          }
        double nn = 0;
        for (int i = 0; i < m; ++i) nn += P[i + (size_t)j * m] * P[i + (size_t)j * m];
        nn = std::sqrt(nn);
        for (int i = 0; i < m; ++i) P[i + (size_t)j * m] /= nn;
      }
      for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) Q[i + j * LD] = P[i + (size_t)j * m];
    }
    Dev dQ(LD * LD), dU(LD * LD), dN(LD * LD), dL(LD * LD), dUi(LD * LD), dLi(LD * LD), ds(LD);
    dQ.put(Q);
    cudaMemset(flag, 0, 4);
    qrb::modified_lu_blk(dQ.p, LD, b, dU.p, dN.p, dL.p, dUi.p, dLi.p, ds.p, LD, flag, 4, 0);
    cudaDeviceSynchronize();
    Mat U = dU.get(), N = dN.get(), L = dL.get(), Ui = dUi.get(), Li = dLi.get(), s = ds.get(LD);
    // (I + L1) Uc = Q - diag(s)
    Mat Lu(LD * LD, 0.0);
    for (int j = 0; j < b; ++j) Lu[j + j * LD] = 1.0;
    for (int j = 0; j < b; ++j)
      for (int i = j + 1; i < b; ++i) Lu[i + j * LD] = L[i + j * LD];
    Mat LU = mul(Lu, U, b);
    double e3 = 0, e6 = 0;
    bool sgn = true;
    for (int j = 0; j < b; ++j) {
      sgn &= std::fabs(s[j]) == 1.0;
      for (int i = 0; i < b; ++i) {
        e3 = std::fmax(e3, std::fabs(LU[i + j * LD] - (Q[i + j * LD] - (i == j ? s[j] : 0.0))));
        e6 = std::fmax(e6, std::fabs(N[i + j * LD] + U[i + j * LD] * s[j]));
      }
    }
    const double e4 = err_identity(mul(Ui, U, b), b);
    Mat LuT(LD * LD, 0.0);  // L1^T + I (unit upper)
    for (int j = 0; j < b; ++j)
      for (int i = 0; i < b; ++i) LuT[i + j * LD] = Lu[j + i * LD];
    const double e5 = err_identity(mul(Li, LuT, b), b);
    cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost);
    const bool ok2 = e3 < 1e-13 && e4 < 1e-12 && e5 < 1e-12 && e6 == 0.0 && sgn && hf == 0;
    fails += !ok2;
    // compare with the sweep kernels' s (sign choices must agree)
    Dev dU0(LD * LD), dN0(LD * LD), dL0(LD * LD), dUi0(LD * LD), dLi0(LD * LD), ds0(LD);
    const float tb2 = time_us([&] {
      qrb::modified_lu_blk(dQ.p, LD, b, dU.p, dN.p, dL.p, dUi.p, dLi.p, ds.p, LD, flag, 4, 0);
    });
    const float tl2 = time_us([&] {
      qrb::modified_lu(dQ.p, LD, b, dU0.p, dN0.p, dL0.p, dUi0.p, dLi0.p, ds0.p, LD, flag, 4, 0);
    });
    printf("b=%3d mlu_blk: |LU-(Q-S)| %.2e |Uinv U - I| %.2e |L1invT (I+L1)^T - I| %.2e "
           "NUcS %.1e signs %d flag %d  %s  %.1f us (modified_lu default path %.1f us)\n",
           b, e3, e4, e5, e6, (int)sgn, hf, ok2 ? "OK" : "FAIL", tb2, tl2);
    cudaFree(flag);
  }
#ifdef SF_TRACE
  long long tr[3][32];
  qrb::smallfact_trace(&tr[0][0]);
  const char* names[3] = {"chol", "mlu", "triinv"};
  for (int k = 0; k < 3; ++k) {
    printf("%s phase cycles:", names[k]);
    for (int i = 1; i < 13; ++i) printf(" %lld", tr[k][i] - tr[k][i - 1]);
    printf("\n");
  }
  printf("mlu diag (last block) steps 0-8-16-24-end: %lld %lld %lld %lld; l21 row %lld, u12 column %lld\n",
         tr[1][14] - tr[1][13], tr[1][15] - tr[1][14], tr[1][16] - tr[1][15], tr[1][17] - tr[1][16],
         tr[1][19] - tr[1][18], tr[1][21] - tr[1][20]);
  printf("chol load %lld  output %lld\n", tr[0][0] - tr[0][31], tr[0][29] - tr[0][30]);
#endif
  printf("%s (%s)\n", fails ? "FAILURES" : "ALL OK", cudaGetErrorString(cudaGetLastError()));
  return fails ? 1 : 0;
}
