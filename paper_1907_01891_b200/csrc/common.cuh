// Shared device helpers for the sm_100a FP64 QR library: error plumbing,
// mbarrier / TMA (cp.async.bulk.tensor) PTX wrappers and the FP64 tensor-core
// (DMMA, mma.sync m8n8k4 .f64) primitive.
//
// Everything here is written for sm_100a only (compiled with
// -gencode arch=compute_100a,code=sm_100a). tcgen05/UMMA has no FP64 kind, so
// the FP64 tensor path on Blackwell is the warp-level DMMA.8x8x4 instruction.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

namespace qrb {

// ---------------------------------------------------------------------------
// status codes shared with include/qrb200.h
// ---------------------------------------------------------------------------
enum : int {
  QRB_OK = 0,
  QRB_ERR_ARG = -1,
  QRB_ERR_CUDA = -2,
  QRB_ERR_NOMEM = -3,
  QRB_ERR_NONFINITE = -4,
  QRB_ERR_STATE = -5,
  QRB_ERR_UNSUPPORTED = -6,
};

void set_last_error(const std::string& msg);

#define QRB_CUDA_TRY(expr)                                                     \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::qrb::set_last_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
      return ::qrb::QRB_ERR_CUDA;                                              \
    }                                                                          \
  } while (0)

#define QRB_TRY(expr)          \
  do {                         \
    int _s = (expr);           \
    if (_s != 0) return _s;    \
  } while (0)

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting: raise
// it once per (kernel, device), growing only.
int set_max_dynamic_smem(const void* func, size_t bytes);


// ---------------------------------------------------------------------------
// column-major matrix view (device memory); ld in elements
// ---------------------------------------------------------------------------
struct MatView {
  double* ptr;
  int64_t rows;
  int64_t cols;
  int64_t ld;
  MatView sub(int64_t r0, int64_t c0, int64_t nr, int64_t nc) const {
    return MatView{ptr + r0 + c0 * ld, nr, nc, ld};
  }
};

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 2-D tiled TMA load global -> shared, completion signalled on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// 3-D tiled TMA load global -> shared
__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// 2-D tiled TMA store shared -> global (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem_src,
                                             int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
      : "memory");
}
// bulk reduce-add of `bytes` (multiple of 16) doubles from shared to global (in L2)
__device__ __forceinline__ void bulk_reduce_add_f64(double* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(
                   gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}

// bulk copy of `bytes` (multiple of 16) from shared to global memory
__device__ __forceinline__ void bulk_store_f64(double* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// producer side of a split barrier: counts this warp in without waiting
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col).
// Fragment ownership for lane = 4*g + q:  A[g][q], B[q][g], D[g][2q], D[g][2q+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

// ---------------------------------------------------------------------------
// launch predicate: a kernel launched under a PredScope reads one device int at
// entry and returns at once unless (*flag != 0) == want.  The CholeskyQR2 panel
// uses it to choose its Householder fallback on the device, so the panel chain
// never waits on a device->host flag read (and can be captured in a graph).
// ---------------------------------------------------------------------------
struct LaunchPred {
  const int* flag;
  int want;
};
__device__ __forceinline__ bool pred_off(const LaunchPred& p) {
  if (p.flag == nullptr) return false;
  const int v = *reinterpret_cast<const volatile int*>(p.flag);
  return (v != 0) != (p.want != 0);
}
LaunchPred launch_pred();  // this host thread's current predicate ({nullptr, 0}: none)
void set_launch_pred(LaunchPred p);
struct PredScope {
  LaunchPred old;
  PredScope(const int* flag, int want) : old(launch_pred()) { set_launch_pred({flag, want}); }
  ~PredScope() { set_launch_pred(old); }
};

// grid-wide barrier for cooperatively launched kernels. `counter` is zeroed
// before the launch; `target` = (#barriers passed so far + 1) * gridDim.x.
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

}  // namespace qrb
