// FP64 tensor-core GEMM family for the blocked Householder QR (sm_100a).
//
// The compact-WY trailing update of a panel (reference: kernels.py:315-319,
// 332-340, 375-380, 396-404 -- W = V^T C ; Z = T^T W ; C -= V Z) and the
// off-diagonal back-substitution update (reference gemm_nn_mo, kernels.py:442-455)
// are all dense FP64 contractions.  They run here on the FP64 tensor pipe
// (DMMA.8x8x4 via mma.sync.m8n8k4.f64) fed by TMA:
//
//   * one producer warp streams 16-deep K slices of both operands with
//     cp.async.bulk.tensor (128-byte swizzle) into a 4-stage shared-memory ring
//     guarded by mbarriers (full: TMA transaction count, empty: consumer warps);
//   * eight consumer warps load conflict-free 16-byte fragments
//     (ld.shared.v2.f64) and issue DMMA with register accumulators (tcgen05 /
//     TMEM have no FP64 kind on Blackwell, so this is the FP64 tensor path);
//   * the epilogue either stores the tile or subtracts it from C in place.
//
// Operand conventions (all matrices column-major, views are MatView):
//   A_KMAJOR = true  : op(A) = Aview^T, Aview is K x M (rows = K)   [W = V^T C]
//   A_KMAJOR = false : op(A) = Aview,   Aview is M x K (rows = M)   [C -= V W]
//   B is always a K x N view (rows = K).
// A view flagged "unit lower" (a Householder block V stored in place under R)
// is read with its upper triangle as zeros and its diagonal as ones -- the
// same implicit-unit-diagonal convention as the reference's _unit_lower
// (kernels.py:286-290).  TMA zero-fills everything outside a view, so ragged
// M/N/K edges need no padding.
#include "common.cuh"
#include "gemm.h"

#include <atomic>

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace qrb {

namespace {

constexpr int BM = 128;
constexpr int BK = 16;
constexpr int STAGES = 4;
constexpr int CONSUMER_WARPS = 8;
constexpr int THREADS = (CONSUMER_WARPS + 1) * 32;

struct GemmArgs {
  int M, N, K;
  int k_per_split, nsplit;
  double* out;
  int64_t ldo;
  int64_t split_stride;
  int mask_a, mask_b;
  int group_m;
  LaunchPred pred;
};

__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return static_cast<uint32_t>(row * 128 + (((chunk ^ (row & 7)) & 7) << 4));
}

// Fragment row permutation for K-major operands.  An LDS.128 is served per
// quarter-warp (8 lanes = fragment rows g in {2k, 2k+1}); mapping fragment row g
// to tile row RP(g) = [0,5,2,7,4,1,6,3][g] makes those two rows differ in bit 2,
// so the 128B-swizzled chunks of the 8 lanes are distinct (no bank conflicts),
// and even / odd output columns land on even / odd swizzle rows, which keeps
// the swizzled C-tile epilogue conflict-free as well.
__device__ __forceinline__ int rp(int g) { return (g & 6) ^ ((g & 1) * 5); }

// unit-lower-trapezoid masking of a pair of consecutive view rows (r, r+1) at view column c
__device__ __forceinline__ void mask_pair(double2& v, int r, int c) {
  if (r <= c) v.x = (r == c) ? 1.0 : 0.0;
  if (r + 1 <= c) v.y = (r + 1 == c) ? 1.0 : 0.0;
}

template <bool A_KMAJOR, int BN, bool MASK_A, bool MASK_B>
__device__ __forceinline__ void consume_stage(double (&acc)[4][BN / 16][2], const uint8_t* sA,
                                              const uint8_t* sB, int m0, int n0, int g, int q,
                                              int kg0, int mg0, int ng0) {
  constexpr int NT = BN / 16;
#pragma unroll
  for (int kc = 0; kc < BK; kc += 8) {
    double2 b[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int row = n0 + nt * 8 + rp(g);
      b[nt] = *reinterpret_cast<const double2*>(sB + swz(row, (kc >> 1) + q));
      if constexpr (MASK_B) mask_pair(b[nt], kg0 + kc + 2 * q, ng0 + row);
    }
    if constexpr (A_KMAJOR) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int row = m0 + mt * 8 + rp(g);
        double2 a = *reinterpret_cast<const double2*>(sA + swz(row, (kc >> 1) + q));
        if constexpr (MASK_A) mask_pair(a, kg0 + kc + 2 * q, mg0 + row);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a.x, b[nt].x);
          dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a.y, b[nt].y);
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int k = kc + 2 * q + p;
#pragma unroll
        for (int mp = 0; mp < 2; ++mp) {
          const int m = m0 + mp * 16 + 2 * g;  // even row; pair (m, m+1)
          double2 a = *reinterpret_cast<const double2*>(sA + (m >> 4) * 2048 + swz(k, (m & 15) >> 1));
          if constexpr (MASK_A) mask_pair(a, mg0 + m, kg0 + k);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const double bv = p ? b[nt].y : b[nt].x;
            dmma_8x8x4(acc[mp * 2 + 0][nt][0], acc[mp * 2 + 0][nt][1], a.x, bv);
            dmma_8x8x4(acc[mp * 2 + 1][nt][0], acc[mp * 2 + 1][nt][1], a.y, bv);
          }
        }
      }
    }
  }
}

template <bool A_KMAJOR, int BN, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_dmma_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, const GemmArgs args) {
  if (pred_off(args.pred)) return;
  constexpr int NT = BN / 16;
  constexpr uint32_t A_BYTES = BM * BK * 8;
  constexpr uint32_t B_BYTES = BN * BK * 8;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;

  extern __shared__ uint8_t smem_raw[];
  // keep the pointer derived from the __shared__ array so loads compile to LDS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // work units = (output tile, K split); CTAs stride over them (a capped grid
  // makes the kernel persistent, e.g. to leave SMs to a concurrent panel)
  const int num_m = (args.M + BM - 1) / BM;
  const int num_n = (args.N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int units = tiles * args.nsplit;
  auto decode = [&](int u, int& m_tile, int& n_tile, int& split) {
    split = u / tiles;
    const int tile = u - split * tiles;
    const int per_group = args.group_m * num_n;
    const int first_m = (tile / per_group) * args.group_m;
    const int gsize = min(num_m - first_m, args.group_m);
    const int local = tile % per_group;
    m_tile = first_m + local % gsize;
    n_tile = local / gsize;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CONSUMER_WARPS) {
    // ---------------- producer warp: TMA ----------------
    if (lane == 0) {
      prefetch_tmap(&mapA);
      prefetch_tmap(&mapB);
      int kit = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int m_tile, n_tile, split;
        decode(u, m_tile, n_tile, split);
        const int k_begin = split * args.k_per_split;
        const int k_end = min(args.K, k_begin + args.k_per_split);
        const int num_k = (k_end - k_begin + BK - 1) / BK;
        for (int kt = 0; kt < num_k; ++kt, ++kit) {
          const int s = kit % STAGES;
          if (kit >= STAGES) mbar_wait(&empty[s], ((kit / STAGES) & 1) ^ 1);
          uint8_t* sA = smem + s * STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          const int k = k_begin + kt * BK;
          if constexpr (A_KMAJOR) {
            tma_load_2d(sA, &mapA, k, m_tile * BM, &full[s]);
          } else {
#pragma unroll
            for (int mb = 0; mb < BM / 16; ++mb)
              tma_load_2d(sA + mb * 2048, &mapA, m_tile * BM + mb * 16, k, &full[s]);
          }
          tma_load_2d(sB, &mapB, k, n_tile * BN, &full[s]);
        }
      }
    }
    return;
  }

  // ---------------- consumer warps: DMMA ----------------
  const int g = lane >> 2;
  const int q = lane & 3;
  const int m0 = (warp & 3) * 32;
  const int n0 = (warp >> 2) * (BN / 2);
  int s = 0;  // ring position carried across work units
  uint32_t ph = 0;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    int m_tile, n_tile, split;
    decode(u, m_tile, n_tile, split);
    const int k_begin = split * args.k_per_split;
    const int k_end = min(args.K, k_begin + args.k_per_split);
    const int num_k = (k_end - k_begin + BK - 1) / BK;
    const int mg0 = m_tile * BM;
    const int ng0 = n_tile * BN;
    // K-slice ranges that touch a unit-lower (masked) block, as per-unit bounds:
    // K-major A / B are masked while kg0 <= (first row of the tile) + rows - 1,
    // an M-major A from kg0 >= mg0 - BK + 1 on
    auto last_masked = [&](int lim) { return lim < k_begin ? 0 : (lim - k_begin) / BK + 1; };
    const int ka_lo = A_KMAJOR ? 0 : (mg0 - BK + 1 <= k_begin ? 0 : (mg0 - k_begin) / BK);
    const int ka_hi = !args.mask_a ? 0 : A_KMAJOR ? last_masked(mg0 + BM - 1) : num_k;
    const int kb_hi = args.mask_b ? last_masked(ng0 + BN - 1) : 0;

    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < num_k; ++kt) {
      mbar_wait(&full[s], ph);
      const uint8_t* sA = smem + s * STAGE_BYTES;
      const uint8_t* sB = sA + A_BYTES;
      const int kg0 = k_begin + kt * BK;
      const bool ma = kt >= ka_lo && kt < ka_hi;
      const bool mb = kt < kb_hi;
      if (ma || mb) {
        if (ma && mb)
          consume_stage<A_KMAJOR, BN, true, true>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
        else if (ma)
          consume_stage<A_KMAJOR, BN, true, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
        else
          consume_stage<A_KMAJOR, BN, false, true>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      } else {
        consume_stage<A_KMAJOR, BN, false, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) {
        s = 0;
        ph ^= 1u;
      }
    }

    // ---------------- epilogue ----------------
    double* out = args.out + static_cast<int64_t>(split) * args.split_stride;
    const int64_t ldo = args.ldo;
    if constexpr (A_KMAJOR) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int m = mg0 + m0 + mt * 8 + rp(g);
        if (m >= args.M) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = ng0 + n0 + nt * 8 + rp(2 * q + e);
            if (n < args.N) {
              double* p = out + m + static_cast<int64_t>(n) * ldo;
              if constexpr (EPI == GEMM_EPI_SUB)
                *p -= acc[mt][nt][e];
              else
                *p = acc[mt][nt][e];
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int mp = 0; mp < 2; ++mp) {
        const int m = mg0 + m0 + mp * 16 + 2 * g;
        if (m >= args.M) continue;
        const bool pair = (m + 1 < args.M);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = ng0 + n0 + nt * 8 + rp(2 * q + e);
            if (n >= args.N) continue;
            double* p = out + m + static_cast<int64_t>(n) * ldo;
            const double v0 = acc[mp * 2 + 0][nt][e];
            const double v1 = acc[mp * 2 + 1][nt][e];
            if (pair) {
              double2* p2 = reinterpret_cast<double2*>(p);
              if constexpr (EPI == GEMM_EPI_SUB) {
                double2 c = *p2;
                c.x -= v0;
                c.y -= v1;
                *p2 = c;
              } else {
                *p2 = make_double2(v0, v1);
              }
            } else {
              if constexpr (EPI == GEMM_EPI_SUB)
                *p -= v0;
              else
                *p = v0;
            }
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// persistent C -= A B with TMA-staged C tiles (the trailing-update GEMM)
//
// One CTA per SM walks its share of the 128 x 64 output tiles.  The producer
// warp streams A/B K-slices through the same 4-stage ring as above and, ahead
// of every tile, TMA-loads the C tile into one of two 64 KB shared buffers.
// The consumer warps subtract their register accumulators from the staged C
// tile in shared memory and one thread TMA-stores it back, so the read-modify-
// write of C (the HBM-bound part of a K = 128 update) overlaps the next tile's
// DMMA main loop instead of stalling it.
// ---------------------------------------------------------------------------
constexpr int NN_BN = 64;
constexpr uint32_t NN_A_BYTES = BM * BK * 8;
constexpr uint32_t NN_B_BYTES = NN_BN * BK * 8;
constexpr uint32_t NN_STAGE_BYTES = NN_A_BYTES + NN_B_BYTES;
constexpr uint32_t NN_C_BYTES = BM * NN_BN * 8;
constexpr int NN_SMEM = STAGES * NN_STAGE_BYTES + 2 * NN_C_BYTES + 1024 + 256;

struct NnArgs {
  int M, N, K;
  int mask_a;
  int group_m;
  int num_tiles;
  int* counter;  // dynamic tile scheduler (async-epilogue kernel); nullptr = static
  LaunchPred pred;
};

__device__ __forceinline__ double neg_bits(double x) {
  return __hiloint2double(__double2hiint(x) ^ static_cast<int>(0x80000000u), __double2loint(x));
}

__device__ __forceinline__ void decode_tile(int tile, int num_m, int num_n, int group_m,
                                            int& m_tile, int& n_tile) {
  const int per_group = group_m * num_n;
  const int first_m = (tile / per_group) * group_m;
  const int gsize = min(num_m - first_m, group_m);
  const int local = tile % per_group;
  m_tile = first_m + local % gsize;
  n_tile = local / gsize;
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_nn_sub_persistent(const __grid_constant__ CUtensorMap mapA,
                           const __grid_constant__ CUtensorMap mapB,
                           const __grid_constant__ CUtensorMap mapC, const NnArgs args) {
  if (pred_off(args.pred)) return;
  constexpr int NT = NN_BN / 16;
  extern __shared__ uint8_t smem_raw[];
  // keep the pointer derived from the __shared__ array so loads compile to LDS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* cbuf0 = smem + STAGES * NN_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(cbuf0 + 2 * NN_C_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* cfull = empty + STAGES;
  uint64_t* cempty = cfull + 2;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (args.M + BM - 1) / BM;
  const int num_n = (args.N + NN_BN - 1) / NN_BN;
  const int num_k = (args.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&cfull[b], 1);
      mbar_init(&cempty[b], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CONSUMER_WARPS) {
    if (lane == 0) {
      prefetch_tmap(&mapA);
      prefetch_tmap(&mapB);
      prefetch_tmap(&mapC);
      int kit = 0, it = 0;
      for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x, ++it) {
        int m_tile, n_tile;
        decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
        const int cb = it & 1;
        if (it >= 2) mbar_wait(&cempty[cb], ((it >> 1) - 1) & 1);
        mbar_arrive_expect_tx(&cfull[cb], NN_C_BYTES);
#pragma unroll
        for (int mb = 0; mb < BM / 16; ++mb)
          tma_load_2d(cbuf0 + cb * NN_C_BYTES + mb * (NN_BN * 128), &mapC, m_tile * BM + mb * 16,
                      n_tile * NN_BN, &cfull[cb]);
        for (int kt = 0; kt < num_k; ++kt, ++kit) {
          const int s = kit % STAGES;
          if (kit >= STAGES) mbar_wait(&empty[s], ((kit / STAGES) & 1) ^ 1);
          uint8_t* sA = smem + s * NN_STAGE_BYTES;
          uint8_t* sB = sA + NN_A_BYTES;
          mbar_arrive_expect_tx(&full[s], NN_STAGE_BYTES);
          const int k = kt * BK;
#pragma unroll
          for (int mb = 0; mb < BM / 16; ++mb)
            tma_load_2d(sA + mb * 2048, &mapA, m_tile * BM + mb * 16, k, &full[s]);
          tma_load_2d(sB, &mapB, k, n_tile * NN_BN, &full[s]);
        }
      }
    }
    return;
  }

  const int g = lane >> 2;
  const int q = lane & 3;
  const int m0 = (warp & 3) * 32;
  const int n0 = (warp >> 2) * (NN_BN / 2);
  int kit = 0, it = 0;
  for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x, ++it) {
    int m_tile, n_tile;
    decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
    const int cb = it & 1;
    const int mg0 = m_tile * BM;
    const int ng0 = n_tile * NN_BN;
    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < num_k; ++kt, ++kit) {
      const int s = kit % STAGES;
      mbar_wait(&full[s], (kit / STAGES) & 1);
      const uint8_t* sA = smem + s * NN_STAGE_BYTES;
      const uint8_t* sB = sA + NN_A_BYTES;
      const int kg0 = kt * BK;
      if (args.mask_a && mg0 <= kg0 + BK - 1)
        consume_stage<false, NN_BN, true, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      else
        consume_stage<false, NN_BN, false, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // epilogue: C_smem -= acc, then one TMA store of the tile
    mbar_wait(&cfull[cb], (it >> 1) & 1);
    uint8_t* cbuf = cbuf0 + cb * NN_C_BYTES;
#pragma unroll
    for (int mp = 0; mp < 2; ++mp) {
      const int m = m0 + mp * 16 + 2 * g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + nt * 8 + rp(2 * q + e);
          // swizzled [16-row block][64 cols][16 rows] staging (TMA SWIZZLE_128B)
          double2* p = reinterpret_cast<double2*>(cbuf + (m >> 4) * (NN_BN * 128) +
                                                  swz(n, (m & 15) >> 1));
          double2 c = *p;
          c.x -= acc[mp * 2 + 0][nt][e];
          c.y -= acc[mp * 2 + 1][nt][e];
          *p = c;
        }
      }
    }
    fence_proxy_async();
    named_bar_sync(1, CONSUMER_WARPS * 32);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int mb = 0; mb < BM / 16; ++mb)
        tma_store_2d(&mapC, cbuf + mb * (NN_BN * 128), mg0 + mb * 16, ng0);
      bulk_commit();
      bulk_wait_read0();
      mbar_arrive(&cempty[cb]);
    }
  }
  if (threadIdx.x == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------
// persistent C -= A B with an L2 reduce-add epilogue: the consumers stage -acc
// column by column in shared memory (padded 1040-byte columns, conflict-free)
// and 64 threads each issue one cp.reduce.async.bulk .add.f64 of their column
// into C, which the L2 applies in place.  No C tile is loaded into the SM at
// all, so the epilogue is a handful of STS per thread plus one barrier.
// ---------------------------------------------------------------------------
constexpr int RA_STAGES = 6;
constexpr int RA_COL_BYTES = BM * 8 + 16;
constexpr uint32_t RA_STAGING = NN_BN * RA_COL_BYTES;
constexpr int RA_SMEM = RA_STAGES * NN_STAGE_BYTES + RA_STAGING + 1024 + 256;

__global__ void __launch_bounds__(THREADS, 1)
    gemm_nn_sub_redadd(const __grid_constant__ CUtensorMap mapA,
                       const __grid_constant__ CUtensorMap mapB, double* __restrict__ C,
                       const int64_t ldc, const NnArgs args) {
  if (pred_off(args.pred)) return;
  constexpr int NT = NN_BN / 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage = smem + RA_STAGES * NN_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage + RA_STAGING);
  uint64_t* empty = full + RA_STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (args.M + BM - 1) / BM;
  const int num_n = (args.N + NN_BN - 1) / NN_BN;
  const int num_k = (args.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RA_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CONSUMER_WARPS) {
    if (lane == 0) {
      prefetch_tmap(&mapA);
      prefetch_tmap(&mapB);
      int kit = 0;
      for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x) {
        int m_tile, n_tile;
        decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
        for (int kt = 0; kt < num_k; ++kt, ++kit) {
          const int s = kit % RA_STAGES;
          if (kit >= RA_STAGES) mbar_wait(&empty[s], ((kit / RA_STAGES) & 1) ^ 1);
          uint8_t* sA = smem + s * NN_STAGE_BYTES;
          uint8_t* sB = sA + NN_A_BYTES;
          mbar_arrive_expect_tx(&full[s], NN_STAGE_BYTES);
          const int k = kt * BK;
#pragma unroll
          for (int mb = 0; mb < BM / 16; ++mb)
            tma_load_2d(sA + mb * 2048, &mapA, m_tile * BM + mb * 16, k, &full[s]);
          tma_load_2d(sB, &mapB, k, n_tile * NN_BN, &full[s]);
        }
      }
    }
    return;
  }

  const int g = lane >> 2;
  const int q = lane & 3;
  const int m0 = (warp & 3) * 32;
  const int n0 = (warp >> 2) * (NN_BN / 2);
  int kit = 0;
  for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x) {
    int m_tile, n_tile;
    decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
    const int mg0 = m_tile * BM;
    const int ng0 = n_tile * NN_BN;
    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < num_k; ++kt, ++kit) {
      const int s = kit % RA_STAGES;
      mbar_wait(&full[s], (kit / RA_STAGES) & 1);
      const uint8_t* sA = smem + s * NN_STAGE_BYTES;
      const uint8_t* sB = sA + NN_A_BYTES;
      const int kg0 = kt * BK;
      if (args.mask_a && mg0 <= kg0 + BK - 1)
        consume_stage<false, NN_BN, true, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      else
        consume_stage<false, NN_BN, false, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // the previous tile's bulk reduces must have finished reading the staging
    // (waited for here, one tile later, so the issuing warps never stall)
    if (threadIdx.x < NN_BN) bulk_wait_read0();
    named_bar_sync(1, CONSUMER_WARPS * 32);
#pragma unroll
    for (int mp = 0; mp < 2; ++mp) {
      const int m = m0 + mp * 16 + 2 * g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + nt * 8 + rp(2 * q + e);
          *reinterpret_cast<double2*>(stage + n * RA_COL_BYTES + m * 8) =
              make_double2(-acc[mp * 2 + 0][nt][e], -acc[mp * 2 + 1][nt][e]);
        }
      }
    }
    fence_proxy_async();
    named_bar_sync(1, CONSUMER_WARPS * 32);
    if (threadIdx.x < NN_BN) {
      const int n = threadIdx.x;
      const int rows = min(BM, args.M - mg0);
      if (ng0 + n < args.N && rows > 0) {
        double* dst = C + mg0 + static_cast<int64_t>(ng0 + n) * ldc;
        const int even = rows & ~1;
        if (even) bulk_reduce_add_f64(dst, stage + n * RA_COL_BYTES, even * 8);
        if (rows & 1)
          atomicAdd(dst + even,
                    *reinterpret_cast<const double*>(stage + n * RA_COL_BYTES + even * 8));
        bulk_commit();
      }
    }
  }
  if (threadIdx.x < NN_BN) bulk_wait0();
}


// ---------------------------------------------------------------------------
// persistent C -= A B with an ASYNCHRONOUS L2 reduce-add epilogue: the eight
// consumer warps stage -acc into one of two padded shared-memory buffers and
// only *arrive* on an mbarrier; a dedicated epilogue warp waits for the staged
// tile and issues the 64 per-column cp.reduce.async.bulk .add.f64 reductions,
// releasing the buffer when the bulk reads are done.  The consumers go straight
// back to the DMMA main loop of the next tile (no named barrier in their path).
// ---------------------------------------------------------------------------
#ifndef QRB_NN_STAGES
#define QRB_NN_STAGES 6
#endif
constexpr int AE_STAGES = QRB_NN_STAGES;
#ifndef QRB_NN_STAGGER_NS
#define QRB_NN_STAGGER_NS 0
#endif
constexpr int AE_SBUF = 1;  // staging buffers (the bulk read of one finishes long before the next tile)
constexpr int AE_THREADS = (CONSUMER_WARPS + 2) * 32;  // + producer warp + epilogue warp
constexpr int AE_SMEM = AE_STAGES * NN_STAGE_BYTES + AE_SBUF * RA_STAGING + 1024 + 256;

// STORE = false: C -= A B (bulk L2 reduce-add of -acc);
// STORE = true:  C = A B   (bulk copy of +acc: the panel chain's K = nb products
// Q1 = P R1^-1 and V = Q1 M, where the one-tile-per-CTA kernel spent ~30% of
// every tile in its prologue and epilogue)
template <bool STORE>
__device__ __forceinline__ void nn_asyncepi_body(const CUtensorMap& mapA, const CUtensorMap& mapB,
                                                 double* __restrict__ C, const int64_t ldc,
                                                 const NnArgs& args) {
  if (pred_off(args.pred)) return;
  constexpr int NT = NN_BN / 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage0 = smem + AE_STAGES * NN_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + AE_SBUF * RA_STAGING);
  uint64_t* empty = full + AE_STAGES;
  uint64_t* sfull = empty + AE_STAGES;
  uint64_t* sempty = sfull + 2;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (args.M + BM - 1) / BM;
  const int num_n = (args.N + NN_BN - 1) / NN_BN;
  const int num_k = (args.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < AE_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], CONSUMER_WARPS);
      mbar_init(&sempty[b], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CONSUMER_WARPS) {  // ---- TMA producer ----
    if (lane == 0) {
      prefetch_tmap(&mapA);
      prefetch_tmap(&mapB);
      int kit = 0;
      for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x) {
        int m_tile, n_tile;
        decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
        for (int kt = 0; kt < num_k; ++kt, ++kit) {
          const int s = kit % AE_STAGES;
          if (kit >= AE_STAGES) mbar_wait(&empty[s], ((kit / AE_STAGES) & 1) ^ 1);
          uint8_t* sA = smem + s * NN_STAGE_BYTES;
          uint8_t* sB = sA + NN_A_BYTES;
          mbar_arrive_expect_tx(&full[s], NN_STAGE_BYTES);
          const int k = kt * BK;
#pragma unroll
          for (int mb = 0; mb < BM / 16; ++mb)
            tma_load_2d(sA + mb * 2048, &mapA, m_tile * BM + mb * 16, k, &full[s]);
          tma_load_2d(sB, &mapB, k, n_tile * NN_BN, &full[s]);
        }
      }
    }
    return;
  }
  if (warp == CONSUMER_WARPS + 1) {  // ---- epilogue warp: bulk L2 reductions ----
    int it = 0;
    for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x, ++it) {
      int m_tile, n_tile;
      decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
      const int sb = it % AE_SBUF;
      const int mg0 = m_tile * BM, ng0 = n_tile * NN_BN;
      mbar_wait(&sfull[sb], (it / AE_SBUF) & 1);
      const uint8_t* stage = stage0 + sb * RA_STAGING;
      const int rows = min(BM, args.M - mg0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = lane + 32 * h;
        if (ng0 + n < args.N && rows > 0) {
          double* dst = C + mg0 + static_cast<int64_t>(ng0 + n) * ldc;
          const int even = rows & ~1;
          const double* src = reinterpret_cast<const double*>(stage + n * RA_COL_BYTES);
          if (STORE) {
            if (even) bulk_store_f64(dst, src, even * 8);
            if (rows & 1) dst[even] = src[even];
          } else {
            if (even) bulk_reduce_add_f64(dst, src, even * 8);
            if (rows & 1) atomicAdd(dst + even, src[even]);
          }
        }
      }
      bulk_commit();
      bulk_wait_read0();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[sb]);
    }
    bulk_wait0();
    return;
  }

  // ---- consumer warps: DMMA main loop, stage -acc, arrive ----
  // Loop bookkeeping is kept off the DMMA warps' issue path: the ring position
  // (stage, parity) is carried across tiles instead of kit % 6 / kit / 6, the
  // V-mask test is one compare against a per-tile bound, and -acc is formed by
  // flipping sign bits on the integer pipe (a DADD shares the FP64 pipe with
  // DMMA).  r02 (tools/nn_variants.py, 69120 x 32768): K = 256 34.87 -> 35.84,
  // K = 512 35.37 -> 36.04 TFLOP/s.  With that, the r01 stagger of warps 4-7
  // (QRB_NN_STAGGER_NS, which made them hold ring stages the leading warps were
  // waiting for) no longer pays: 0 / 2 / 4 / 8 us = 35.84 / 35.79 / 35.37 / 35.37
  // at K = 256, so it is off by default.
  const int g = lane >> 2;
  const int q = lane & 3;
  const int m0 = (warp & 3) * 32;
  const int n0 = (warp >> 2) * (NN_BN / 2);
  int it = 0;
  // ring position (stage, parity) carried across tiles: no divisions in the loop
  int s = 0;
  uint32_t ph = 0;
  if (QRB_NN_STAGGER_NS > 0 && warp >= CONSUMER_WARPS / 2) __nanosleep(QRB_NN_STAGGER_NS);
  for (int tile = blockIdx.x; tile < args.num_tiles; tile += gridDim.x, ++it) {
    int m_tile, n_tile;
    decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
    const int mg0 = m_tile * BM;
    const int ng0 = n_tile * NN_BN;
    // K slices from kt_mask on touch the unit-lower block of V (rows mg0.. <= k)
    const int kt_mask = args.mask_a ? mg0 / BK : num_k;
    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < num_k; ++kt) {
      mbar_wait(&full[s], ph);
      const uint8_t* sA = smem + s * NN_STAGE_BYTES;
      const uint8_t* sB = sA + NN_A_BYTES;
      const int kg0 = kt * BK;
      if (kt >= kt_mask)
        consume_stage<false, NN_BN, true, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      else
        consume_stage<false, NN_BN, false, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == AE_STAGES) {
        s = 0;
        ph ^= 1u;
      }
    }
    const int sb = it % AE_SBUF;
    if (it >= AE_SBUF) mbar_wait(&sempty[sb], ((it / AE_SBUF) - 1) & 1);
    uint8_t* stage = stage0 + sb * RA_STAGING;
#pragma unroll
    for (int mp = 0; mp < 2; ++mp) {
      const int m = m0 + mp * 16 + 2 * g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + nt * 8 + rp(2 * q + e);
          // -acc by flipping the sign bits on the integer pipe (a DADD would
          // occupy the FP64 pipe the DMMAs share)
          *reinterpret_cast<double2*>(stage + n * RA_COL_BYTES + m * 8) =
              STORE ? make_double2(acc[mp * 2 + 0][nt][e], acc[mp * 2 + 1][nt][e])
                    : make_double2(neg_bits(acc[mp * 2 + 0][nt][e]),
                                   neg_bits(acc[mp * 2 + 1][nt][e]));
        }
      }
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sfull[sb]);
  }
}

__global__ void __launch_bounds__(AE_THREADS, 1)
    gemm_nn_sub_asyncepi(const __grid_constant__ CUtensorMap mapA,
                         const __grid_constant__ CUtensorMap mapB, double* __restrict__ C,
                         const int64_t ldc, const NnArgs args) {
  nn_asyncepi_body<false>(mapA, mapB, C, ldc, args);
}

__global__ void __launch_bounds__(AE_THREADS, 1)
    gemm_nn_store_asyncepi(const __grid_constant__ CUtensorMap mapA,
                           const __grid_constant__ CUtensorMap mapB, double* __restrict__ C,
                           const int64_t ldc, const NnArgs args) {
  nn_asyncepi_body<true>(mapA, mapB, C, ldc, args);
}

// Same kernel with dynamic tile tickets (first tile static, then a per-launch
// global counter; the tile id travels through the smem ring).  CTAs that start
// late -- e.g. behind an NCCL kernel holding a few SMs on a multi-GPU run --
// take fewer tiles instead of stretching the launch.  Selected with
// qrb_set_tuning("nn_dynamic", 1) (dist.py does so on more than one GPU); on
// an idle GPU the static schedule above is ~1% faster (r01 A/B in bench.py).
__global__ void __launch_bounds__(AE_THREADS, 1)
    gemm_nn_sub_asyncepi_dyn(const __grid_constant__ CUtensorMap mapA,
                         const __grid_constant__ CUtensorMap mapB, double* __restrict__ C,
                         const int64_t ldc, const NnArgs args) {
  if (pred_off(args.pred)) return;
  constexpr int NT = NN_BN / 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage0 = smem + AE_STAGES * NN_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + AE_SBUF * RA_STAGING);
  uint64_t* empty = full + AE_STAGES;
  uint64_t* sfull = empty + AE_STAGES;
  uint64_t* sempty = sfull + 2;
  // tile id travelling with every ring stage (producer -> consumers) and with
  // every staged result (consumers -> epilogue warp); -1 = no more tiles
  volatile int* stage_tile = reinterpret_cast<volatile int*>(sempty + 2);
  volatile int* sbuf_tile = stage_tile + AE_STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (args.M + BM - 1) / BM;
  const int num_n = (args.N + NN_BN - 1) / NN_BN;
  const int num_k = (args.K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < AE_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMER_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sfull[b], CONSUMER_WARPS);
      mbar_init(&sempty[b], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == CONSUMER_WARPS) {  // ---- TMA producer ----
    if (lane == 0) {
      prefetch_tmap(&mapA);
      prefetch_tmap(&mapB);
      // Tiles: the first one static, then one ticket per tile from a global
      // counter (fetched a tile ahead).  CTAs that start late -- e.g. behind a
      // NCCL kernel holding a few SMs -- simply take fewer tiles.
      auto next_tile = [&](int cur) {
        if (cur >= args.num_tiles) return args.num_tiles;
        return args.counter ? (int)gridDim.x + atomicAdd(args.counter, 1) : cur + (int)gridDim.x;
      };
      int kit = 0;
      int tile = blockIdx.x;
      int nxt = next_tile(tile);
      for (;;) {
        if (tile >= args.num_tiles) {  // sentinel stage: consumers stop
          const int s = kit % AE_STAGES;
          if (kit >= AE_STAGES) mbar_wait(&empty[s], ((kit / AE_STAGES) & 1) ^ 1);
          stage_tile[s] = -1;
          mbar_arrive(&full[s]);
          break;
        }
        int m_tile, n_tile;
        decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
        for (int kt = 0; kt < num_k; ++kt, ++kit) {
          const int s = kit % AE_STAGES;
          if (kit >= AE_STAGES) mbar_wait(&empty[s], ((kit / AE_STAGES) & 1) ^ 1);
          stage_tile[s] = tile;
          uint8_t* sA = smem + s * NN_STAGE_BYTES;
          uint8_t* sB = sA + NN_A_BYTES;
          mbar_arrive_expect_tx(&full[s], NN_STAGE_BYTES);
          const int k = kt * BK;
#pragma unroll
          for (int mb = 0; mb < BM / 16; ++mb)
            tma_load_2d(sA + mb * 2048, &mapA, m_tile * BM + mb * 16, k, &full[s]);
          tma_load_2d(sB, &mapB, k, n_tile * NN_BN, &full[s]);
        }
        tile = nxt;
        nxt = next_tile(tile);
      }
    }
    return;
  }
  if (warp == CONSUMER_WARPS + 1) {  // ---- epilogue warp: bulk L2 reductions ----
    for (int it = 0;; ++it) {
      const int sb = it % AE_SBUF;
      mbar_wait(&sfull[sb], (it / AE_SBUF) & 1);
      const int tile = sbuf_tile[sb];
      if (tile < 0) break;
      int m_tile, n_tile;
      decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
      const int mg0 = m_tile * BM, ng0 = n_tile * NN_BN;
      const uint8_t* stage = stage0 + sb * RA_STAGING;
      const int rows = min(BM, args.M - mg0);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = lane + 32 * h;
        if (ng0 + n < args.N && rows > 0) {
          double* dst = C + mg0 + static_cast<int64_t>(ng0 + n) * ldc;
          const int even = rows & ~1;
          if (even) bulk_reduce_add_f64(dst, stage + n * RA_COL_BYTES, even * 8);
          if (rows & 1)
            atomicAdd(dst + even,
                      *reinterpret_cast<const double*>(stage + n * RA_COL_BYTES + even * 8));
        }
      }
      bulk_commit();
      bulk_wait_read0();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[sb]);
    }
    bulk_wait0();
    return;
  }

  // ---- consumer warps: DMMA main loop, stage -acc, arrive ----
  const int g = lane >> 2;
  const int q = lane & 3;
  const int m0 = (warp & 3) * 32;
  const int n0 = (warp >> 2) * (NN_BN / 2);
  int s = 0;  // ring position carried across tiles (no divisions in the loop)
  uint32_t ph = 0;
  for (int it = 0;; ++it) {
    // the tile id arrives with the first ring stage of the tile
    mbar_wait(&full[s], ph);
    const int tile = stage_tile[s];
    if (tile < 0) {
      // pass the end marker on to the epilogue warp (after its last staging)
      const int sb = it % AE_SBUF;
      if (it >= AE_SBUF) mbar_wait(&sempty[sb], ((it / AE_SBUF) - 1) & 1);
      if (lane == 0 && warp == 0) sbuf_tile[sb] = -1;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[sb]);
      break;
    }
    int m_tile, n_tile;
    decode_tile(tile, num_m, num_n, args.group_m, m_tile, n_tile);
    const int mg0 = m_tile * BM;
    const int ng0 = n_tile * NN_BN;
    const int kt_mask = args.mask_a ? mg0 / BK : num_k;
    double acc[4][NT][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < num_k; ++kt) {
      if (kt > 0) mbar_wait(&full[s], ph);  // (the first stage was waited for above)
      const uint8_t* sA = smem + s * NN_STAGE_BYTES;
      const uint8_t* sB = sA + NN_A_BYTES;
      const int kg0 = kt * BK;
      if (kt >= kt_mask)
        consume_stage<false, NN_BN, true, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      else
        consume_stage<false, NN_BN, false, false>(acc, sA, sB, m0, n0, g, q, kg0, mg0, ng0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == AE_STAGES) {
        s = 0;
        ph ^= 1u;
      }
    }
    const int sb = it % AE_SBUF;
    if (it >= AE_SBUF) mbar_wait(&sempty[sb], ((it / AE_SBUF) - 1) & 1);
    uint8_t* stage = stage0 + sb * RA_STAGING;
#pragma unroll
    for (int mp = 0; mp < 2; ++mp) {
      const int m = m0 + mp * 16 + 2 * g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + nt * 8 + rp(2 * q + e);
          *reinterpret_cast<double2*>(stage + n * RA_COL_BYTES + m * 8) =
              make_double2(neg_bits(acc[mp * 2 + 0][nt][e]), neg_bits(acc[mp * 2 + 1][nt][e]));
        }
      }
    }
    if (lane == 0 && warp == 0) sbuf_tile[sb] = tile;
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&sfull[sb]);
  }
}


// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

int get_encoder() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult qres;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres) ==
            cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return QRB_ERR_CUDA;
  }
  return QRB_OK;
}

int make_map(CUtensorMap* map, const MatView& v, uint32_t box_rows, uint32_t box_cols,
             bool swizzle = true) {
  QRB_TRY(get_encoder());
  if (v.rows < 1 || v.cols < 1) {
    set_last_error("make_map: empty view");
    return QRB_ERR_ARG;
  }
  if ((reinterpret_cast<uintptr_t>(v.ptr) & 15) != 0 || (v.ld & 1) != 0) {
    set_last_error("make_map: view base must be 16-byte aligned and ld even");
    return QRB_ERR_ARG;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(v.rows), static_cast<cuuint64_t>(v.cols)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(v.ld) * 8};
  cuuint32_t box[2] = {box_rows, box_cols};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, v.ptr, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return QRB_ERR_CUDA;
  }
  return QRB_OK;
}

template <bool A_KMAJOR, int BN, int EPI>
int launch(const MatView& a, const MatView& b, double* out, int64_t ldo, int64_t split_stride,
           int M, int N, int K, int splits, int mask_a, int mask_b, cudaStream_t stream,
           int* used = nullptr) {
  constexpr int SMEM = STAGES * (BM * BK * 8 + BN * BK * 8) + 2 * STAGES * 8 + 1024;
  QRB_TRY(set_max_dynamic_smem(
      reinterpret_cast<const void*>(gemm_dmma_kernel<A_KMAJOR, BN, EPI>), SMEM));
  CUtensorMap ma, mb;
  if (A_KMAJOR)
    QRB_TRY(make_map(&ma, a, BK, BM));
  else
    QRB_TRY(make_map(&ma, a, 16, BK));
  QRB_TRY(make_map(&mb, b, BK, BN));
  GemmArgs args;
  args.M = M;
  args.N = N;
  args.K = K;
  int kps = (K + splits - 1) / splits;
  kps = ((kps + BK - 1) / BK) * BK;
  args.k_per_split = kps;
  args.out = out;
  args.ldo = ldo;
  args.split_stride = split_stride;
  args.mask_a = mask_a;
  args.mask_b = mask_b;
  args.group_m = 16;
  args.pred = launch_pred();
  const int num_m = (M + BM - 1) / BM;
  const int num_n = (N + BN - 1) / BN;
  const int nsplit = (K + kps - 1) / kps;
  if (used) *used = nsplit;
  args.nsplit = nsplit;
  const int units = num_m * num_n * nsplit;
  const int cap = gemm_grid_cap();
  const int grid = cap > 0 ? std::min(units, cap) : units;
  gemm_dmma_kernel<A_KMAJOR, BN, EPI><<<grid, THREADS, SMEM, stream>>>(ma, mb, args);
  QRB_CUDA_TRY(cudaGetLastError());
  return QRB_OK;
}

}  // namespace

static thread_local int t_grid_cap = 0;
static thread_local LaunchPred t_pred = {nullptr, 0};
LaunchPred launch_pred() { return t_pred; }
void set_launch_pred(LaunchPred p) { t_pred = p; }
void gemm_set_grid_cap(int cap) { t_grid_cap = cap; }
int gemm_grid_cap() { return t_grid_cap; }

int gemm_sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// number of K splits for a long-K (TN) product so that the tile grid fills
// the machine with little wave quantization
// 128 x 32 tiles for NN products with few 128 x 64 tiles ("few_tiles_bn32")
static std::atomic<int> g_few_tiles_bn32{2};
void gemm_set_few_tiles_bn32(int on) { g_few_tiles_bn32 = on; }  // 1: NN products, 2: + split TN
int gemm_few_tiles_bn32() { return g_few_tiles_bn32.load(); }

// rows of K per split when the product has few output tiles ("gram_min_rows")
static std::atomic<int> g_few_tiles_min_rows{32};  // r02 sweep at config 1: 128 -> 1.96 ms, 64 -> 1.90, 32 -> 1.88
void gemm_set_few_tiles_min_rows(int rows) { g_few_tiles_min_rows = std::max(16, rows); }
int gemm_few_tiles_min_rows() { return g_few_tiles_min_rows.load(); }

// ... and a short K per CTA (<= 256 rows with 128 x 64 tiles): in a long main
// loop the 128 x 64 tile's operand reuse matters more than the epilogue (the
// 256-slice solve's W = V^T B, K = m_k / 9, lost 5% with 128 x 32 tiles)
static bool few_tiles_tn32(int M, int N, int K) {
  const int tiles = ((M + BM - 1) / BM) * ((N + 63) / 64);
  return g_few_tiles_bn32.load() > 1 && N > 32 && tiles * 2 <= gemm_sm_count() &&
         static_cast<int64_t>(K) * tiles <= 256 * static_cast<int64_t>(gemm_sm_count());
}

// output tiles of a split TN launch of this shape (128 x 32 tiles when the
// few-tile rule applies, 128 x 64 otherwise)
int gemm_tn_split_tiles(int M, int N, int K) {
  return ((M + BM - 1) / BM) * (few_tiles_tn32(M, N, K) ? (N + 31) / 32 : (N + 63) / 64);
}

int gemm_pick_splits(int M, int N, int K, int max_splits) {
  const int tiles = ((M + BM - 1) / BM) * ((N + 63) / 64);
  const int slots = gemm_sm_count();  // one 288-thread CTA per SM (168 regs)
  // few output tiles (the panel's Gram matrices, late trailing updates): one
  // wave whatever the split, so split as far as gram_min_rows (32) rows of K per
  // split allow (r02 trace: the 2160-row Gram ran 7 splits, 21 us; 17 splits of
  // 128 rows 12 us, each CTA 8 us of DMMA work on 34 of the 148 SMs)
  if (tiles * 2 <= slots) {
    // the TN launch then runs 128 x 32 tiles (few_tiles_tn32): half the partial
    // output per CTA to store and to reduce, twice the K per split
    const int t = few_tiles_tn32(M, N, K) ? ((M + BM - 1) / BM) * ((N + 31) / 32) : tiles;
    return std::max(1, std::min(std::min(max_splits, K / g_few_tiles_min_rows.load()), slots / t));
  }
  const int kmax = std::max(1, K / 256);  // keep >= 256 rows of K per split
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= std::min(max_splits, kmax); ++s) {
    const long units = static_cast<long>(tiles) * s;
    const long waves = (units + slots - 1) / slots;
    const double eff = static_cast<double>(units) / static_cast<double>(waves * slots);
    // prefer fewer splits unless a split count is clearly better
    if (eff > best_eff + 0.03) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

int gemm_tn(const MatView& a_km, const MatView& b, double* out, int64_t ldo, int64_t split_stride,
            int M, int N, int K, int splits, int mask_a, int mask_b, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0) return QRB_OK;
  return launch<true, 64, GEMM_EPI_STORE>(a_km, b, out, ldo, split_stride, M, N, K, splits,
                                          mask_a, mask_b, stream);
}

int gemm_tn_split(const MatView& a_km, const MatView& b, double* out, int64_t ldo,
                  int64_t split_stride, int M, int N, int K, int splits, int mask_a, int mask_b,
                  cudaStream_t stream, int* used) {
  *used = 0;
  if (M <= 0 || N <= 0 || K <= 0) return QRB_OK;
  if (splits > 1 && gemm_grid_cap() == 0 && few_tiles_tn32(M, N, K))
    return launch<true, 32, GEMM_EPI_STORE>(a_km, b, out, ldo, split_stride, M, N, K, splits,
                                            mask_a, mask_b, stream, used);
  return launch<true, 64, GEMM_EPI_STORE>(a_km, b, out, ldo, split_stride, M, N, K, splits,
                                          mask_a, mask_b, stream, used);
}

int gemm_nn_split(const MatView& a_mm, const MatView& b, double* out, int64_t ldo,
                  int64_t split_stride, int M, int N, int K, int splits, int mask_a,
                  cudaStream_t stream, int* used) {
  *used = 0;
  if (M <= 0 || N <= 0 || K <= 0) return QRB_OK;
  return launch<false, 64, GEMM_EPI_STORE>(a_mm, b, out, ldo, split_stride, M, N, K, splits,
                                           mask_a, 0, stream, used);
}

static std::atomic<bool> g_nn_dynamic{false};
void gemm_set_nn_dynamic(bool on) { g_nn_dynamic.store(on); }
bool gemm_nn_dynamic() { return g_nn_dynamic.load(); }

int gemm_nn(const MatView& a_mm, const MatView& b, double* out, int64_t ldo, int M, int N, int K,
            int epi, int mask_a, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0) return QRB_OK;
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0 || (ldo & 1) != 0) {
    set_last_error("gemm_nn: output must be 16-byte aligned with even ld");
    return QRB_ERR_ARG;
  }
  // few tiles and a short K (the trailing update of a small matrix: 16 x 4 tiles
  // of 8 us at m = 2160): 128 x 32 tiles, one per CTA, put twice as many SMs to
  // work; C - acc is rounded once either way, so the result is bitwise the
  // persistent kernel's (uncapped launches only: a capped launch must stay on
  // its SMs)
  if (epi == GEMM_EPI_SUB && g_few_tiles_bn32.load() && gemm_grid_cap() == 0 && N > 32 &&
      K <= 512 && ((M + BM - 1) / BM) * ((N + 63) / 64) * 2 <= gemm_sm_count())
    return launch<false, 32, GEMM_EPI_SUB>(a_mm, b, out, ldo, 0, M, N, K, 1, mask_a, 0, stream);
  static const bool asyncepi = std::getenv("QRB_NN_SYNC_EPI") == nullptr;
  if (epi == GEMM_EPI_SUB && asyncepi && !(std::getenv("QRB_NN_STAGED_C")) &&
      !(std::getenv("QRB_NN_CLASSIC"))) {
    const bool dyn = g_nn_dynamic.load();
    QRB_TRY(set_max_dynamic_smem(dyn ? reinterpret_cast<const void*>(gemm_nn_sub_asyncepi_dyn)
                                     : reinterpret_cast<const void*>(gemm_nn_sub_asyncepi),
                                 AE_SMEM));
    CUtensorMap ma, mb;
    QRB_TRY(make_map(&ma, a_mm, 16, BK));
    QRB_TRY(make_map(&mb, b, BK, NN_BN));
    NnArgs args{};
    args.pred = launch_pred();
    args.M = M;
    args.N = N;
    args.K = K;
    args.mask_a = mask_a;
    args.group_m = 16;
    const int num_m = (M + BM - 1) / BM;
    const int num_n = (N + NN_BN - 1) / NN_BN;
    args.num_tiles = num_m * num_n;
    const int cap = gemm_grid_cap();
    const int grid = std::min(args.num_tiles, cap > 0 ? std::min(cap, gemm_sm_count()) : gemm_sm_count());
    if (!dyn) {
      gemm_nn_sub_asyncepi<<<grid, AE_THREADS, AE_SMEM, stream>>>(ma, mb, out, ldo, args);
      QRB_CUDA_TRY(cudaGetLastError());
      return QRB_OK;
    }
    // tile tickets: one zeroed counter per launch from a ring (launches on
    // different streams never share one while in flight)
    args.counter = nullptr;
    if (args.num_tiles > grid) {
      constexpr int RING = 4096;
      static int* rings[64] = {nullptr};  // per device
      static std::mutex ring_mu;
      static std::atomic<unsigned> slot{0};
      int dev = 0;
      QRB_CUDA_TRY(cudaGetDevice(&dev));
      int* ring;
      {
        std::lock_guard<std::mutex> lk(ring_mu);
        if (!rings[dev & 63]) QRB_CUDA_TRY(cudaMalloc(&rings[dev & 63], RING * 32 * sizeof(int)));
        ring = rings[dev & 63];
      }
      args.counter = ring + 32 * (slot.fetch_add(1) % RING);  // one 128-byte line each
      QRB_CUDA_TRY(cudaMemsetAsync(args.counter, 0, sizeof(int), stream));
    }
    gemm_nn_sub_asyncepi_dyn<<<grid, AE_THREADS, AE_SMEM, stream>>>(ma, mb, out, ldo, args);
    QRB_CUDA_TRY(cudaGetLastError());
    return QRB_OK;
  }
  static const bool redadd = std::getenv("QRB_NN_STAGED_C") == nullptr;
  if (epi == GEMM_EPI_SUB && redadd && !(std::getenv("QRB_NN_CLASSIC"))) {
    QRB_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(gemm_nn_sub_redadd), RA_SMEM));
    CUtensorMap ma, mb;
    QRB_TRY(make_map(&ma, a_mm, 16, BK));
    QRB_TRY(make_map(&mb, b, BK, NN_BN));
    NnArgs args{};
    args.pred = launch_pred();
    args.M = M;
    args.N = N;
    args.K = K;
    args.mask_a = mask_a;
    args.group_m = 16;
    const int num_m = (M + BM - 1) / BM;
    const int num_n = (N + NN_BN - 1) / NN_BN;
    args.num_tiles = num_m * num_n;
    const int grid = std::min(args.num_tiles, gemm_sm_count());
    gemm_nn_sub_redadd<<<grid, THREADS, RA_SMEM, stream>>>(ma, mb, out, ldo, args);
    QRB_CUDA_TRY(cudaGetLastError());
    return QRB_OK;
  }
  if (epi == GEMM_EPI_SUB && !(std::getenv("QRB_NN_CLASSIC"))) {
    QRB_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(gemm_nn_sub_persistent), NN_SMEM));
    CUtensorMap ma, mb, mc;
    QRB_TRY(make_map(&ma, a_mm, 16, BK));
    QRB_TRY(make_map(&mb, b, BK, NN_BN));
    QRB_TRY(make_map(&mc, MatView{out, M, N, ldo}, 16, NN_BN));
    NnArgs args{};
    args.pred = launch_pred();
    args.M = M;
    args.N = N;
    args.K = K;
    args.mask_a = mask_a;
    args.group_m = 16;
    const int num_m = (M + BM - 1) / BM;
    const int num_n = (N + NN_BN - 1) / NN_BN;
    args.num_tiles = num_m * num_n;
    const int grid = std::min(args.num_tiles, gemm_sm_count());
    gemm_nn_sub_persistent<<<grid, THREADS, NN_SMEM, stream>>>(ma, mb, mc, args);
    QRB_CUDA_TRY(cudaGetLastError());
    return QRB_OK;
  }
  if (epi == GEMM_EPI_SUB)
    return launch<false, 64, GEMM_EPI_SUB>(a_mm, b, out, ldo, 0, M, N, K, 1, mask_a, 0, stream);
  {
    // C = A B with more tiles than SMs: persistent, async bulk-store epilogue
    const int num_m = (M + BM - 1) / BM;
    const int num_n = (N + NN_BN - 1) / NN_BN;
    static const bool store_persistent = std::getenv("QRB_NN_STORE_CLASSIC") == nullptr;
    if (store_persistent && num_m * num_n > gemm_sm_count()) {
      QRB_TRY(set_max_dynamic_smem(reinterpret_cast<const void*>(gemm_nn_store_asyncepi), AE_SMEM));
      CUtensorMap ma, mb;
      QRB_TRY(make_map(&ma, a_mm, 16, BK));
      QRB_TRY(make_map(&mb, b, BK, NN_BN));
      NnArgs args{};
      args.pred = launch_pred();
      args.M = M;
      args.N = N;
      args.K = K;
      args.mask_a = mask_a;
      args.group_m = 16;
      args.num_tiles = num_m * num_n;
      const int cap = gemm_grid_cap();
      const int grid =
          std::min(args.num_tiles, cap > 0 ? std::min(cap, gemm_sm_count()) : gemm_sm_count());
      gemm_nn_store_asyncepi<<<grid, AE_THREADS, AE_SMEM, stream>>>(ma, mb, out, ldo, args);
      QRB_CUDA_TRY(cudaGetLastError());
      return QRB_OK;
    }
  }
  {
    // few tiles (a short panel's Q1 = P R1^-1: 17 x 2 tiles of 8 us at m = 2160):
    // 128 x 32 tiles put twice as many SMs to work; same K order per element, so
    // the result is bitwise the 128 x 64 kernel's
    const int num_m = (M + BM - 1) / BM;
    if (g_few_tiles_bn32.load() && N > 32 && num_m * ((N + 63) / 64) * 2 <= gemm_sm_count())
      return launch<false, 32, GEMM_EPI_STORE>(a_mm, b, out, ldo, 0, M, N, K, 1, mask_a, 0,
                                               stream);
  }
  return launch<false, 64, GEMM_EPI_STORE>(a_mm, b, out, ldo, 0, M, N, K, 1, mask_a, 0, stream);
}

}  // namespace qrb
