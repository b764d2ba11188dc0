// C ABI of the B200 FP64 QR library (include/qrb200.h): device handle,
// right-looking blocked Householder QR driver, block-reflector application
// and the multi-slice least-squares solve.
//
// Reference path being replaced (pkg/src/oocqr):
//   factorize  task_engine.py:606-641  -> qrb_factorize
//   solve      task_engine.py:644-685  -> qrb_solve
//   kernels    kernels.py:296-455      -> panel_factor / apply_qt / trsm below
// The reference orders the work as a left-looking tile DAG to minimise disk
// writes (task_engine.py:187-254); with the matrix resident in HBM the
// B200-native order is right-looking by panels of nb columns, every trailing
// update being two large DMMA GEMMs.
#include "cholqr.h"
#include "common.cuh"
#include "gemm.h"
#include "panel.h"
#include "siddon.h"

#include "../../include/qrb200.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace qrb {

static thread_local std::string t_last_error;
void set_last_error(const std::string& msg) { t_last_error = msg; }

int set_max_dynamic_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  QRB_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[std::make_pair(func, dev)];
  if (bytes <= have) return QRB_OK;
  QRB_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(bytes)));
  have = bytes;
  return QRB_OK;
}

// ---------------------------------------------------------------------------
// grow-only device buffers
// ---------------------------------------------------------------------------
// bumped whenever a device buffer is (re)allocated or a tuning knob changes: a
// captured factorization graph (qrb_factorize) is valid only for the epoch it
// was captured in
static std::atomic<uint64_t> g_graph_epoch{1};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t need, cudaStream_t st) {
    if (need <= bytes) return QRB_OK;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      set_last_error("device buffer growth during graph capture");
      return QRB_ERR_STATE;  // the caller abandons the capture and runs eagerly
    }
    ++g_graph_epoch;
    if (p) {
      QRB_CUDA_TRY(cudaStreamSynchronize(st));
      QRB_CUDA_TRY(cudaFree(p));
      p = nullptr;
      bytes = 0;
    }
    if (cudaMalloc(&p, need) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      set_last_error("cudaMalloc of " + std::to_string(need) + " bytes failed");
      return QRB_ERR_NOMEM;
    }
    bytes = need;
    return QRB_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  double* d() const { return static_cast<double*>(p); }
};

struct Workspace {
  DevBuf part, bar, G, Ti, W, W2, Wparts;
  DevBuf Wq, small, flag;  // CholeskyQR2 panel: Q1 (m x b), 12 b x b blocks, status word
  DevBuf T2;               // merged block reflector of a panel pair (2nb x 2nb) + scratch
  DevBuf T4;               // scratch of the 4-panel merge (outer_panels = 4)
  int64_t w2_cols = 0;     // columns / width of the W2 the last apply_qt_w2 formed
  int64_t w2_w = 0;
  uint64_t w2_gen = 0;     // bumped by every apply_qt_w2 (qrb_op_apply_qt_cols checks it)
  // serialisation of calls that share this workspace (WsUse): one host thread
  // at a time, and a call on another stream waits for the last call's work
  std::recursive_mutex mu;
  cudaEvent_t last_ev = nullptr;
  cudaStream_t last_st = nullptr;
  void release() {
    Wq.release();
    small.release();
    T2.release();
    T4.release();
    flag.release();
    part.release();
    bar.release();
    G.release();
    Ti.release();
    W.release();
    W2.release();
    Wparts.release();
  }
};

static std::atomic<int64_t> g_launches{0};

// ---------------------------------------------------------------------------
// optional per-kernel-family CUDA-event accounting (qrb_set_profiling)
// ---------------------------------------------------------------------------
struct Profiler {
  struct Rec {
    int kind;
    cudaEvent_t a, b;
    double flops, bytes;
  };
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<Rec> recs;
  int depth = 0;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void reset() {
    used = 0;
    recs.clear();
    depth = 0;
  }
  ~Profiler() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};
static thread_local Profiler* g_prof = nullptr;

struct ProfScope {
  Profiler* p;
  cudaStream_t st;
  Profiler::Rec rec;
  bool active;
  ProfScope(int kind, double flops, double bytes, cudaStream_t s)
      : p(g_prof), st(s), active(false) {
    if (p && p->depth == 0) {
      rec.kind = kind;
      rec.flops = flops;
      rec.bytes = bytes;
      rec.a = p->get();
      rec.b = p->get();
      cudaEventRecord(rec.a, st);
      active = true;
    }
    if (p) p->depth++;
  }
  ~ProfScope() {
    if (p) p->depth--;
    if (active) {
      cudaEventRecord(rec.b, st);
      p->recs.push_back(rec);
    }
  }
};

static Workspace& device_workspace() {
  static Workspace ws[64];
  int dev = 0;
  cudaGetDevice(&dev);
  return ws[dev & 63];
}

// buffers of the look-ahead panel, which runs on a second stream concurrently
// with the trailing update that uses device_workspace()
static Workspace& side_workspace() {
  static Workspace ws[64];
  int dev = 0;
  cudaGetDevice(&dev);
  return ws[dev & 63];
}

// Entry points of the library share one workspace per device (and a second one
// for the look-ahead panel).  WsUse makes that safe for several handles and
// streams: the calling thread holds the workspace for the call, and a call on a
// different stream than the previous user first waits (on the device) for the
// previous call's work.  Inside a graph capture no events are used (the
// captured schedule is replayed on one handle's streams).
struct WsUse {
  Workspace& ws;
  cudaStream_t st;
  std::lock_guard<std::recursive_mutex> lk;
  bool active;
  WsUse(Workspace& w, cudaStream_t s) : ws(w), st(s), lk(w.mu), active(true) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      active = false;
      return;
    }
    if (ws.last_ev && ws.last_st != st) cudaStreamWaitEvent(st, ws.last_ev, 0);
  }
  ~WsUse() {
    if (!active) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();  // joined a capture meanwhile: its work is ordered by the graph
      return;
    }
    if (!ws.last_ev) cudaEventCreateWithFlags(&ws.last_ev, cudaEventDisableTiming);
    if (ws.last_ev) cudaEventRecord(ws.last_ev, st);
    ws.last_st = st;
  }
};

static inline int64_t even(int64_t x) { return (x + 1) & ~int64_t(1); }

// K splits for a product whose output has only a few 128 x 64 tiles (the solve's
// T^T W and R_kk^-1 Y_k with 256 right-hand sides: 8 tiles on 148 SMs); a
// function of the shape only, so results are deterministic
static int small_splits(int M, int N, int K, bool tn = false) {
  const int tiles = tn ? gemm_tn_split_tiles(M, N, K) : ((M + 127) / 128) * ((N + 63) / 64);
  int s = 1;
  while (tiles * s * 2 <= gemm_sm_count() && K / (s * 2) >= 32 && s < 16) s *= 2;
  return s;
}

// out (M x N) = op(A) B with few output tiles: K split over the SMs, partial
// products summed in a fixed order by reduce_splits (out may alias B: the
// partial GEMM reads B before the reduction writes out)
static int small_product(bool a_kmajor, const MatView& a, const MatView& b, double* out,
                         int64_t ldo, int M, int N, int K, int splits, Workspace& ws,
                         cudaStream_t st) {
  const int64_t ldp = even(M), per = ldp * N;
  QRB_TRY(ws.Wparts.ensure(sizeof(double) * per * splits, st));
  int used = 0;
  if (a_kmajor)
    QRB_TRY(gemm_tn_split(a, b, ws.Wparts.d(), ldp, per, M, N, K, splits, 0, 0, st, &used));
  else
    QRB_TRY(gemm_nn_split(a, b, ws.Wparts.d(), ldp, per, M, N, K, splits, 0, st, &used));
  QRB_TRY(reduce_splits(ws.Wparts.d(), per, used, M, N, ldp, out, ldo, st));
  g_launches += 2;
  return QRB_OK;
}

// Wave-quantisation fix for the long-K TN product W = V^T C (one 128 x 64 tile
// over all m_k rows per CTA, 4.4 ms at m_k = 69120): the column tiles that fill
// whole waves of the SMs run as usual, the tail's tiles are split along K into
// s parts (s minimising ceil(units * s / sms) / s) and reduced in a fixed order.
// A function of the shape only (deterministic).  Returns false when not worth it.
static int g_tn_tail = 1;
static bool tn_tail_split(const MatView& V, const MatView& C, int w, int nc, int m, int64_t ldw,
                          Workspace& ws, cudaStream_t st) {
  if (!g_tn_tail) return false;
  const int G = gemm_sm_count();
  const int tm = (w + 127) / 128, tn = (nc + 63) / 64;
  const int units = tm * tn;
  if (units <= G || units % G == 0 || m < 16 * 256) return false;
  const int nt1 = (units / G) * G / tm;  // column tiles of the full waves
  const int rt = tn - nt1, ru = rt * tm;
  if (nt1 <= 0 || rt <= 0) return false;
  int best_s = 1;
  double best = 1.0;  // tail time in units of one full-K tile
  for (int s = 2; s <= 32 && m / s >= 256; ++s) {
    const double t = static_cast<double>((ru * s + G - 1) / G) / s;
    if (t < best - 1e-9) {
      best = t;
      best_s = s;
    }
  }
  if (best_s == 1 || best > 0.9) return false;
  const int64_t n1 = int64_t(nt1) * 64;
  const int n2 = nc - static_cast<int>(n1);
  if (gemm_tn(V, C.sub(0, 0, C.rows, n1), ws.W.d(), ldw, 0, w, static_cast<int>(n1), m, 1, 1, 0,
              st) != QRB_OK)
    return false;
  const int64_t per = ldw * n2;
  int used = 0;
  if (ws.Wparts.ensure(sizeof(double) * per * best_s, st) != QRB_OK ||
      gemm_tn_split(V, C.sub(0, n1, C.rows, n2), ws.Wparts.d(), ldw, per, w, n2, m, best_s, 1, 0,
                    st, &used) != QRB_OK ||
      reduce_splits(ws.Wparts.d(), per, used, w, n2, ldw, ws.W.d() + n1 * ldw, ldw, st) != QRB_OK)
    return false;
  g_launches += 3;
  return true;
}

// W2 = T^T (V^T C) into ws.W2 (w x nc, ld even(w)); V m x w unit lower (in place under R)
static int apply_qt_w2(const MatView& V, const double* T, int64_t ldt, const MatView& C,
                       Workspace& ws, cudaStream_t st) {
  const int m = static_cast<int>(V.rows);
  const int w = static_cast<int>(V.cols);
  const int nc = static_cast<int>(C.cols);
  const int64_t ldw = even(w);
  QRB_TRY(ws.W.ensure(sizeof(double) * ldw * nc, st));
  QRB_TRY(ws.W2.ensure(sizeof(double) * ldw * nc, st));
  ws.w2_cols = nc;
  ws.w2_w = w;
  ++ws.w2_gen;
  const int64_t per_split = ldw * nc;
  const int max_splits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, (int64_t(32) << 20) / per_split)));
  const int splits = gemm_pick_splits(w, nc, m, max_splits);
  const double fl = 2.0 * m * static_cast<double>(nc) * w;
  {
    ProfScope ps(QRB_K_GEMM_TN, fl, 8.0 * ((double)m * w + (double)m * nc + (double)w * nc), st);
    if (splits > 1) {
      QRB_TRY(ws.Wparts.ensure(sizeof(double) * per_split * splits, st));
      int used = 0;
      QRB_TRY(gemm_tn_split(V, C, ws.Wparts.d(), ldw, per_split, w, nc, m, splits, 1, 0, st,
                            &used));
      QRB_TRY(reduce_splits(ws.Wparts.d(), per_split, used, w, nc, ldw, ws.W.d(), ldw, st));
      g_launches += 2;
    } else if (!tn_tail_split(V, C, w, nc, m, ldw, ws, st)) {
      QRB_TRY(gemm_tn(V, C, ws.W.d(), ldw, 0, w, nc, m, 1, 1, 0, st));
      g_launches += 1;
    }
  }
  // W2 = T^T W
  MatView Tv{const_cast<double*>(T), w, w, ldt};
  MatView Wv{ws.W.d(), w, nc, ldw};
  {
    ProfScope ps(QRB_K_GEMM_TT, 2.0 * w * static_cast<double>(w) * nc,
                 8.0 * (2.0 * w * nc + (double)w * w), st);
    const int s2 = small_splits(w, nc, w, true);
    if (s2 > 1) {
      QRB_TRY(small_product(true, Tv, Wv, ws.W2.d(), ldw, w, nc, w, s2, ws, st));
    } else {
      QRB_TRY(gemm_tn(Tv, Wv, ws.W2.d(), ldw, 0, w, nc, w, 1, 0, 0, st));
      g_launches += 1;
    }
  }
  return QRB_OK;
}

// C[:, c_from : c_from + cols] -= V W2[:, c_from : ...]   (W2 from apply_qt_w2 over C)
static int apply_qt_nn(const MatView& V, const MatView& C, int64_t c_from, int64_t cols,
                       Workspace& ws, cudaStream_t st, int kind = QRB_K_GEMM_NN) {
  if (cols <= 0) return QRB_OK;
  const int m = static_cast<int>(V.rows);
  const int w = static_cast<int>(V.cols);
  const int64_t ldw = even(w);
  const double fl = 2.0 * m * static_cast<double>(cols) * w;
  MatView W2v{ws.W2.d() + c_from * ldw, w, cols, ldw};
  ProfScope ps(kind, fl, 8.0 * (2.0 * m * cols + (double)m * w + (double)w * cols), st);
  QRB_TRY(gemm_nn(V, W2v, C.ptr + c_from * C.ld, C.ld, m, static_cast<int>(cols), w,
                  GEMM_EPI_SUB, 1, st));
  g_launches += 1;
  return QRB_OK;
}

// C <- (I - V T^T V^T) C   i.e. C <- Q^T C,  V m x w unit lower (in place under R)
static int apply_qt(const MatView& V, const double* T, int64_t ldt, const MatView& C,
                    Workspace& ws, cudaStream_t st) {
  if (C.cols <= 0 || V.cols <= 0 || V.rows <= 0) return QRB_OK;
  QRB_TRY(apply_qt_w2(V, T, ldt, C, ws, st));
  return apply_qt_nn(V, C, 0, C.cols, ws, st);
}

// Householder QR of an m x w panel (w <= 128) in place, tau[w], T (w x w, ldt)
static int factor_panel_impl(const MatView& panel, double* tau, double* T, int64_t ldt,
                             Workspace& ws, cudaStream_t st);

static int factor_panel(const MatView& panel, double* tau, double* T, int64_t ldt, Workspace& ws,
                        cudaStream_t st) {
  const double m = static_cast<double>(panel.rows), w = static_cast<double>(panel.cols);
  ProfScope ps(QRB_K_PANEL, 2.0 * m * w * w - 2.0 * w * w * w / 3.0, 16.0 * m * w, st);
  return factor_panel_impl(panel, tau, T, ldt, ws, st);
}

// Panel algorithm selection (qrb_set_tuning): 0 = auto (CholeskyQR2 +
// reconstruction for tall panels, Householder columns otherwise),
// 1 = Householder columns always, 2 = CholeskyQR2 whenever the shape allows.
static int g_panel_algo = [] {
  const char* e = std::getenv("QRB_PANEL_ALGO");
  return e ? std::atoi(e) : 0;
}();
static int64_t g_cholqr_min_rows = 1024;  // CholeskyQR2 wins from ~2k rows up (r01 sweep)
static std::atomic<int64_t> g_cholqr_panels{0};

// a non-blocking stream per device for capturing conditional-node bodies
static cudaStream_t capture_helper_stream(int which = 0) {
  static cudaStream_t hs[2][64] = {{nullptr}};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  cudaStream_t& s = hs[which & 1][dev & 63];
  if (!s && cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) s = nullptr;
  return s;
}
static int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return QRB_OK;
  set_last_error(std::string("CUDA: ") + cudaGetErrorString(e));
  return QRB_ERR_CUDA;
}
// fork / join events for two independent kernels inside a captured IF body
static cudaEvent_t capture_helper_event(int which) {
  static cudaEvent_t ev[2][64] = {{nullptr}};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  cudaEvent_t& e = ev[which & 1][dev & 63];
  if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) e = nullptr;
  return e;
}

// Householder QR of the panel column by column (the path for short panels and
// the CholeskyQR2 route's fallback)
static int factor_panel_householder(const MatView& panel, double* tau, double* T, int64_t ldt,
                                    Workspace& ws, cudaStream_t st);

// CholeskyQR2 + Householder reconstruction of an m x b panel (cholqr.cu header
// for the algebra).  The small factorizations raise bits in a device flag when
// the Cholesky route is not trustworthy for this panel; the completion kernels
// run only when the flag is clear and the Householder kernels (launched right
// after, predicated on the same flag) only when it is set -- the choice is made
// on the device, so the panel chain never stops for a device->host flag read.
static int factor_panel_cholqr2(const MatView& panel, double* tau, double* T, int64_t ldt,
                                Workspace& ws, cudaStream_t st) {
  const int m = static_cast<int>(panel.rows);
  const int b = static_cast<int>(panel.cols);
  const int64_t mw = (static_cast<int64_t>(m) + 1) & ~int64_t(1);
  constexpr int LD = 128;
  constexpr int64_t BLK = int64_t(LD) * LD;
  QRB_TRY(ws.Wq.ensure(sizeof(double) * mw * b, st));
  QRB_TRY(ws.small.ensure(sizeof(double) * (BLK * 13 + LD), st));
  QRB_TRY(ws.flag.ensure(64, st));
  QRB_TRY(ws.G.ensure(sizeof(double) * LD * 128, st));
  double* sb = ws.small.d();
  double *R1 = sb, *R1i = sb + BLK, *R2 = sb + 2 * BLK, *R2i = sb + 3 * BLK, *Qt = sb + 4 * BLK;
  double *Uc = sb + 5 * BLK, *NUcS = sb + 6 * BLK, *L1 = sb + 7 * BLK, *Uci = sb + 8 * BLK;
  double *L1iT = sb + 9 * BLK, *M = sb + 10 * BLK, *R = sb + 11 * BLK, *Tt = sb + 12 * BLK;
  double* s = sb + 13 * BLK;
  int* flag = static_cast<int*>(ws.flag.p);
  double* Wq = ws.Wq.d();
  QRB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
  auto gram = [&](const MatView& X) -> int {
    const int64_t per = int64_t(LD) * b;
    const int splits = gemm_pick_splits(b, b, m, 256);  // one tile pair: use every SM
    if (splits > 1) {
      QRB_TRY(ws.Wparts.ensure(sizeof(double) * per * splits, st));
      int used = 0;
      QRB_TRY(gemm_tn_split(X, X, ws.Wparts.d(), LD, per, b, b, m, splits, 0, 0, st, &used));
      QRB_TRY(reduce_splits(ws.Wparts.d(), per, used, b, b, LD, ws.G.d(), LD, st));
      g_launches += 2;
    } else {
      QRB_TRY(gemm_tn(X, X, ws.G.d(), LD, 0, b, b, m, 1, 0, 0, st));
      g_launches += 1;
    }
    return QRB_OK;
  };
  const MatView Q1{Wq, m, b, mw};
  // pass 1: G1 = P^T P, R1 = chol(G1), Q1 = P R1^-1
  QRB_TRY(gram(panel));
  QRB_TRY(chol_inv(ws.G.d(), LD, b, R1, R1i, LD, flag, 1, 0, st));
  QRB_TRY(gemm_nn(panel, MatView{R1i, b, b, LD}, Wq, mw, m, b, b, GEMM_EPI_STORE, 0, st));
  // pass 2: G2 = Q1^T Q1 (must be close to I), R2 = chol(G2)
  QRB_TRY(gram(Q1));
  QRB_TRY(chol_inv(ws.G.d(), LD, b, R2, R2i, LD, flag, 2, 1, st));
  // top block of Q = Q1 R2^-1 and R = R2 R1 (one batched launch), modified LU,
  // then M = R2^-1 Uc^-1 and T^T = -Uc S L1^-T (one batched launch)
  {
    SmallMmBatch bt{};
    bt.p[0] = SmallMm{Wq, R2i, Qt, mw, LD, LD, b, b, b};
    bt.p[1] = SmallMm{R2, R1, R, LD, LD, LD, b, b, b};
    QRB_TRY(small_mm_batch(bt, 2, st));
  }
  QRB_TRY(modified_lu(Qt, LD, b, Uc, NUcS, L1, Uci, L1iT, s, LD, flag, 4, st));
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  cudaGraph_t cg = nullptr;
  QRB_CUDA_TRY(cudaStreamGetCaptureInfo(st, &cst, nullptr, &cg, nullptr, nullptr));
  cudaGraphConditionalHandle hc{};
  {
    SmallMmBatch bt{};
    bt.p[0] = SmallMm{R2i, Uci, M, LD, LD, LD, b, b, b};
    bt.p[1] = SmallMm{NUcS, L1iT, Tt, LD, LD, LD, b, b, b};
    if (cst == cudaStreamCaptureStatusActive) {
      // captured: the flag is final here (every kernel that raises it precedes
      // this launch), so this launch also sets the IF node's condition
      QRB_CUDA_TRY(cudaGraphConditionalHandleCreate(&hc, cg, 0, 0));
      bt.cond = hc;
      bt.cond_flag = flag;
    }
    QRB_TRY(small_mm_batch(bt, 2, st));
  }
  g_launches += 8;
  ++g_cholqr_panels;
  auto finish = [&](cudaStream_t s2) -> int {
    // V below the top block: L2 = Q1[b:] R2^-1 Uc^-1 = Q1[b:] M, written over P[b:]
    if (m > b)
      QRB_TRY(gemm_nn(MatView{Wq + b, m - b, b, mw}, MatView{M, b, b, LD}, panel.ptr + b,
                      panel.ld, m - b, b, b, GEMM_EPI_STORE, 0, s2));
    QRB_TRY(cholqr_write_top(panel.ptr, panel.ld, b, R, s, L1, Tt, LD, tau, LD, T, ldt, flag, s2));
    g_launches += 2;
    return QRB_OK;
  };
  if (cst == cudaStreamCaptureStatusActive) {
    // captured (qrb_factorize graph): an IF/ELSE node on the flag -- the
    // branch not taken costs nothing at replay
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    QRB_CUDA_TRY(cudaStreamGetCaptureInfo(st, &cst, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hc;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 2;
    cudaGraphNode_t node;
    QRB_CUDA_TRY(cudaGraphAddNode(&node, cg, deps, ndeps, &cp));
    QRB_CUDA_TRY(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    cudaStream_t hs = capture_helper_stream();
    if (!hs) {
      set_last_error("no capture helper stream");
      return QRB_ERR_STATE;
    }
    for (int br = 0; br < 2; ++br) {
      QRB_CUDA_TRY(cudaStreamBeginCaptureToGraph(hs, cp.conditional.phGraph_out[br], nullptr,
                                                 nullptr, 0, cudaStreamCaptureModeThreadLocal));
      int rc = QRB_OK;
      if (br == 0) {  // flag set: count the fallback, then the Householder kernels
        rc = cholqr_write_top(panel.ptr, panel.ld, b, R, s, L1, Tt, LD, tau, LD, T, ldt, flag, hs);
        if (rc == QRB_OK) rc = factor_panel_householder(panel, tau, T, ldt, ws, hs);
      } else {
        // V below the top block and the top block / tau / T are independent:
        // two parallel nodes of the body (fork and join by events)
        cudaStream_t hs2 = capture_helper_stream(1);
        cudaEvent_t ef = capture_helper_event(0), ej = capture_helper_event(1);
        if (m > b && hs2 && ef && ej) {
          rc = cuda_status(cudaEventRecord(ef, hs));
          if (rc == QRB_OK) rc = cuda_status(cudaStreamWaitEvent(hs2, ef, 0));
          if (rc == QRB_OK)
            rc = cholqr_write_top(panel.ptr, panel.ld, b, R, s, L1, Tt, LD, tau, LD, T, ldt, flag,
                                  hs2);
          if (rc == QRB_OK) rc = cuda_status(cudaEventRecord(ej, hs2));
          if (rc == QRB_OK)
            rc = gemm_nn(MatView{Wq + b, m - b, b, mw}, MatView{M, b, b, LD}, panel.ptr + b,
                         panel.ld, m - b, b, b, GEMM_EPI_STORE, 0, hs);
          if (rc == QRB_OK) rc = cuda_status(cudaStreamWaitEvent(hs, ej, 0));
          g_launches += 2;
        } else {
          rc = finish(hs);
        }
      }
      cudaGraph_t body = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(hs, &body);
      QRB_TRY(rc);
      QRB_CUDA_TRY(ce);
    }
    return QRB_OK;
  }
  {
    PredScope ok(flag, 0);
    QRB_TRY(finish(st));
  }
  // fallback: the panel is still untouched when the flag is set
  PredScope fb(flag, 1);
  return factor_panel_householder(panel, tau, T, ldt, ws, st);
}

static bool cholqr_eligible(const MatView& panel) {
  if (g_panel_algo == 1) return false;
  const int64_t m = panel.rows, b = panel.cols;
  if (b < 2 || b > 128 || (b & 1) || m < b) return false;
  if ((panel.ld & 1) || (reinterpret_cast<uintptr_t>(panel.ptr) & 15)) return false;
  if (g_panel_algo == 2) return true;
  return m >= g_cholqr_min_rows;
}

static int factor_panel_impl(const MatView& panel, double* tau, double* T, int64_t ldt,
                             Workspace& ws, cudaStream_t st) {
  const int m = static_cast<int>(panel.rows);
  const int pw = static_cast<int>(panel.cols);
  if (pw <= 0) return QRB_OK;
  if (m < pw) {
    set_last_error("panel rows < width");
    return QRB_ERR_ARG;
  }
  if (cholqr_eligible(panel)) return factor_panel_cholqr2(panel, tau, T, ldt, ws, st);
  return factor_panel_householder(panel, tau, T, ldt, ws, st);
}

static int factor_panel_householder(const MatView& panel, double* tau, double* T, int64_t ldt,
                                    Workspace& ws, cudaStream_t st) {
  const int m = static_cast<int>(panel.rows);
  const int pw = static_cast<int>(panel.cols);
  const int ldg = 128;
  QRB_TRY(ws.G.ensure(sizeof(double) * ldg * 128, st));
  QRB_TRY(ws.Ti.ensure(sizeof(double) * 128 * 128, st));
  QRB_TRY(ws.bar.ensure(64, st));
  PanelPlan pl = panel_plan(m, pw);
  QRB_TRY(ws.part.ensure(sizeof(double) * panel_part_doubles(panel_max_ctas(), 128), st));
  unsigned int* bar = static_cast<unsigned int*>(ws.bar.p);
  if (pl.ib >= pw) {
    QRB_TRY(panel_factor(panel, pl.P, pl.R, tau, ws.G.d(), ldg, ws.part.d(), bar, st));
    QRB_TRY(build_t(ws.G.d(), ldg, tau, pw, T, static_cast<int>(ldt), st));
    g_launches += 3;  // memset + panel + build_t
    return QRB_OK;
  }
  const int ib = pl.ib;
  for (int i0 = 0; i0 < pw; i0 += ib) {
    const int w = std::min(ib, pw - i0);
    const int mi = m - i0;
    PanelPlan pi = panel_plan(mi, w);
    MatView sub = panel.sub(i0, i0, mi, w);
    QRB_TRY(panel_factor(sub, pi.P, pi.R, tau + i0, ws.G.d(), ldg, ws.part.d(), bar, st));
    g_launches += 2;
    if (i0 + w < pw) {
      QRB_TRY(build_t(ws.G.d(), ldg, tau + i0, w, ws.Ti.d(), 128, st));
      g_launches += 1;
      QRB_TRY(apply_qt(sub, ws.Ti.d(), 128, panel.sub(i0, i0 + w, mi, pw - i0 - w), ws, st));
    }
  }
  // Gram matrix of the whole panel, then T
  const int64_t per = int64_t(ldg) * pw;
  const int splits = gemm_pick_splits(pw, pw, m, 256);
  if (splits > 1) {
    QRB_TRY(ws.Wparts.ensure(sizeof(double) * per * splits, st));
    int used = 0;
    QRB_TRY(gemm_tn_split(panel, panel, ws.Wparts.d(), ldg, per, pw, pw, m, splits, 1, 1, st,
                          &used));
    QRB_TRY(reduce_splits(ws.Wparts.d(), per, used, pw, pw, ldg, ws.G.d(), ldg, st));
    g_launches += 2;
  } else {
    QRB_TRY(gemm_tn(panel, panel, ws.G.d(), ldg, 0, pw, pw, m, 1, 1, 1, st));
    g_launches += 1;
  }
  QRB_TRY(build_t(ws.G.d(), ldg, tau, pw, T, static_cast<int>(ldt), st));
  g_launches += 1;
  return QRB_OK;
}

// Two nb-wide panels merged into one 2nb-wide block reflector for the trailing
// update: the GEMMs then run with K = 2nb, halving the NN kernel's per-tile
// switches (NN 33.6 -> 34.7 TFLOP/s at K = 256, r01 tools/gemm_k.py).
//   factor panel a; apply Q_a^T to panel b's columns; factor panel b;
//   T = [[T_a, -T_a (V_a^T V_b) T_b], [0, T_b]]   (larft merge)
// T_a / T_b are also stored per panel (the solve applies nb-wide panels).
// Panels per outer step (qrb_set_tuning "outer_panels": 0 = auto, or forced 1, 2
// or 4).  Auto: single panels for factorizations narrower than "pairs_min_cols"
// (r02 sweep: config 1, 2160 x 1024, 2.38 -> 2.17 ms; 4230 x 4096 14.85 -> 14.45
// ms -- the pair's Q_a^T apply and T merge lengthen a chain nothing hides there;
// config 2, 16384 columns: pairs 209.3 vs singles 207.7 ms with their look-ahead,
// but the 64-slice solve after it 7.1 vs 9.6 ms -- pairs keep their merged
// reflectors for the solve), pairs / 4-panel blocks otherwise.  The solve
// applies merged pairs / quads where they exist unless forced to 1.
static int g_outer_panels = [] {
  const char* e = std::getenv("QRB_OUTER_PANELS");
  if (!e) return 0;
  const int v = std::atoi(e);
  return v >= 4 ? 4 : std::max(0, std::min(2, v));
}();
static int64_t g_pairs_min_cols = 8192;
static int g_tail_singles = 0;  // auto mode: single panels instead of pairs after the 4-panel blocks
static int outer_panels_for(int64_t n) {
  if (g_outer_panels > 0) return g_outer_panels;
  return n < g_pairs_min_cols ? 1 : 4;
}
static int outer_panels_solve() { return g_outer_panels > 0 ? g_outer_panels : 4; }

static int factor_panel(const MatView& panel, double* tau, double* T, int64_t ldt, Workspace& ws,
                        cudaStream_t st);

// T2 (2nb x 2nb, leading dim ldt2) = [[Ta, -Ta (V_a[nb:]^T V_b) Tb], [0, Tb]] for the
// factored panels a = A[j0:, j0:j0+nb] and b = A[j0+nb:, j0+nb:j0+2nb] (larft merge);
// scratch: 2 nb x nb blocks
static int merge_pair_t(const MatView& A, int64_t j0, int nb, const double* Ta, const double* Tb,
                        double* T2, int64_t ldt2, double* scratch, Workspace& ws,
                        cudaStream_t st, int wb = 0) {
  if (wb <= 0) wb = nb;  // width of the second panel (the last block may be narrower)
  const int64_t mk = A.rows - j0;
  double* Y = scratch;
  double* Z = Y + int64_t(nb) * nb;
  const MatView Va_lo = A.sub(j0 + nb, j0, mk - nb, nb);      // plain rows of V_a
  const MatView Vb = A.sub(j0 + nb, j0 + nb, mk - nb, wb);    // unit lower V_b
  const int64_t per = int64_t(nb) * nb;
  const int splits = gemm_pick_splits(nb, wb, static_cast<int>(mk - nb), 256);
  if (splits > 1) {
    QRB_TRY(ws.Wparts.ensure(sizeof(double) * per * splits, st));
    int used = 0;
    QRB_TRY(gemm_tn_split(Va_lo, Vb, ws.Wparts.d(), nb, per, nb, wb, static_cast<int>(mk - nb),
                          splits, 0, 1, st, &used));
    QRB_TRY(reduce_splits(ws.Wparts.d(), per, used, nb, wb, nb, Y, nb, st));
    g_launches += 2;
  } else {
    QRB_TRY(gemm_tn(Va_lo, Vb, Y, nb, 0, nb, wb, static_cast<int>(mk - nb), 1, 0, 1, st));
    g_launches += 1;
  }
  const int w2 = nb + wb;
  QRB_CUDA_TRY(cudaMemset2DAsync(T2, sizeof(double) * ldt2, 0, sizeof(double) * w2, w2, st));
  QRB_CUDA_TRY(cudaMemcpy2DAsync(T2, sizeof(double) * ldt2, Ta, sizeof(double) * nb,
                                 sizeof(double) * nb, nb, cudaMemcpyDeviceToDevice, st));
  QRB_CUDA_TRY(cudaMemcpy2DAsync(T2 + nb + ldt2 * nb, sizeof(double) * ldt2, Tb,
                                 sizeof(double) * nb, sizeof(double) * wb, wb,
                                 cudaMemcpyDeviceToDevice, st));
  QRB_TRY(gemm_nn(MatView{const_cast<double*>(Ta), nb, nb, nb}, MatView{Y, nb, wb, nb}, Z, nb, nb,
                  wb, nb, GEMM_EPI_STORE, 0, st));
  QRB_TRY(gemm_nn(MatView{Z, nb, wb, nb}, MatView{const_cast<double*>(Tb), wb, wb, nb},
                  T2 + ldt2 * nb, ldt2, nb, wb, wb, GEMM_EPI_SUB, 0, st));
  g_launches += 2;
  return QRB_OK;
}

static int factor_panel_pair(const MatView& A, int64_t j0, int nb, double* Ta, double* Tb,
                             double* tau, double** T2out, Workspace& ws, cudaStream_t st,
                             double* T2dst = nullptr) {
  const int64_t mk = A.rows - j0;
  const int w2 = 2 * nb;
  const MatView Va = A.sub(j0, j0, mk, nb);
  QRB_TRY(factor_panel(Va, tau + j0, Ta, nb, ws, st));
  QRB_TRY(apply_qt(Va, Ta, nb, A.sub(j0, j0 + nb, mk, nb), ws, st));
  const MatView Vb = A.sub(j0 + nb, j0 + nb, mk - nb, nb);
  QRB_TRY(factor_panel(Vb, tau + j0 + nb, Tb, nb, ws, st));
  QRB_TRY(ws.T2.ensure(sizeof(double) * (int64_t(w2) * w2 + 3 * int64_t(nb) * nb), st));
  double* dst = T2dst ? T2dst : ws.T2.d();
  QRB_TRY(merge_pair_t(A, j0, nb, Ta, Tb, dst, w2, ws.T2.d() + int64_t(w2) * w2, ws, st));
  *T2out = dst;
  return QRB_OK;
}

// B (n x nrhs) <- upper(R)^-1 B using precomputed inverses of the nb x nb diagonal blocks
static int trsm_upper(const MatView& R, const double* Rinv, int nb, const MatView& B,
                      cudaStream_t st) {
  const int n = static_cast<int>(R.rows);
  const int nrhs = static_cast<int>(B.cols);
  if (n <= 0 || nrhs <= 0) return QRB_OK;
  ProfScope ps(QRB_K_TRSM, static_cast<double>(n) * n * nrhs,
               8.0 * (0.5 * n * (double)n + 2.0 * n * (double)nrhs), st);
  const int nblk = (n + nb - 1) / nb;
  for (int k = nblk - 1; k >= 0; --k) {
    const int i0 = k * nb;
    const int bs = std::min(nb, n - i0);
    MatView Ri{const_cast<double*>(Rinv) + (int64_t)k * nb * nb, bs, bs, nb};
    MatView Yk = B.sub(i0, 0, bs, nrhs);
    QRB_TRY(gemm_nn(Ri, Yk, Yk.ptr, Yk.ld, bs, nrhs, bs, GEMM_EPI_STORE, 0, st));
    g_launches += 1;
    if (i0 > 0) {
      MatView Rk = R.sub(0, i0, i0, bs);
      QRB_TRY(gemm_nn(Rk, Yk, B.ptr, B.ld, i0, nrhs, bs, GEMM_EPI_SUB, 0, st));
      g_launches += 1;
    }
  }
  return QRB_OK;
}

// the factorization's progress for a caller streaming finished columns out
// (qrb_factorize_host_gated): one thread stores into page-locked host memory
__global__ void progress_kernel(volatile int64_t* p, int64_t v) { *p = v; }

__global__ void nonfinite_kernel(const double* A, int64_t lda, int64_t m, int64_t n, int* flag) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / m, r = idx - c * m;
    if (!isfinite(A[r + c * lda])) {
      *flag = 1;
      return;
    }
  }
}

// first singular column in the reference's bottom-up tile order (kernels.py:423-426,
// task_engine.py:246-253): diagonal tiles visited from the last one up, first
// |d| < 1e-300 (or NaN) inside the first bad tile met.
static int64_t singular_column(const std::vector<double>& diag, int64_t block) {
  const int64_t n = static_cast<int64_t>(diag.size());
  if (block <= 0) block = n > 0 ? n : 1;
  const int64_t ntiles = (n + block - 1) / block;
  for (int64_t t = ntiles - 1; t >= 0; --t) {
    const int64_t e = std::min(n, (t + 1) * block);
    for (int64_t i = t * block; i < e; ++i) {
      if (!(std::fabs(diag[i]) >= 1e-300)) return i;
    }
  }
  return -1;
}

}  // namespace qrb

using namespace qrb;

struct qrb_handle {
  int device = 0;
  int64_t m = 0, n = 0, lda = 0;
  int nb = 128;
  int npanels = 0;
  double* A = nullptr;
  double* tau = nullptr;
  double* T = nullptr;     // nb x (npanels * nb), ld = nb
  double* Rinv = nullptr;  // npanels blocks of nb x nb
  bool factored = false;
  bool owns_a = true;      // false for qrb_create_view (A is the caller's memory)
  bool rinv_ready = false;
  double* T2 = nullptr;    // merged 2nb x 2nb reflectors of panel pairs (kept from the
  bool t2_ready = false;   //   factorization's pair steps, the rest filled at the first solve)
  std::vector<char> t2_valid;
  double* T4 = nullptr;    // merged 4nb x 4nb reflectors of panel quads (4q .. 4q+3): kept
  std::vector<char> t4_valid;  //   from the factorization's 4-panel blocks, the rest at the
  bool t4_ready = false;       //   first solve (Q^T B with K = 4nb GEMMs)
  double* Rinv2 = nullptr; // inverses of the 2nb x 2nb diagonal blocks of R (pairs), lazily
  bool rinv2_ready = false;
  DevBuf Ytmp;             // copy of a 2nb-row block of the right-hand sides
  cudaStream_t stream = nullptr;      // stream all work of the handle is enqueued on
  cudaStream_t own_stream = nullptr;  // the handle's own stream
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  DevBuf Bw;  // solve work buffer
  DevBuf resid;
  bool profiling = false;
  Profiler prof;
  cudaStream_t side = nullptr;                // look-ahead panel stream (high priority)
  cudaEvent_t ev_upd = nullptr, ev_pan = nullptr;
  DevBuf T2scratch;                           // merged reflectors of pairs not kept in T2
  DevBuf T4scratch;                           // merged 4nb x 4nb reflectors (outer_panels = 4)
  // the whole right-looking factorization captured as one CUDA graph (small
  // shapes, where the panel chain is launch-latency bound), replayed while the
  // buffer / tuning epoch it was captured in holds
  cudaGraphExec_t fgraph = nullptr;
  uint64_t fgraph_epoch = 0;
  int64_t fgraph_launches = 0;
  std::vector<char> fgraph_t2;  // t2_valid as the captured run leaves it
  std::vector<char> fgraph_t4;
  bool fgraph_warm = false;     // one eager run first (sizes every buffer)
  int64_t* progress = nullptr;  // device alias of a caller's page-locked counter: number of
                                //   leading columns whose factored values are final
};

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

void clear_report(qrb_report* rep) {
  if (rep) std::memset(rep, 0, sizeof(*rep));
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// activate the handle's profiler for one call; fold its records into rep at the end
struct ProfSession {
  qrb_handle* h;
  explicit ProfSession(qrb_handle* hh) : h(hh) {
    if (h->profiling) {
      h->prof.reset();
      g_prof = &h->prof;
    }
  }
  void finish(qrb_report* rep) {
    if (!h->profiling) return;
    g_prof = nullptr;
    if (!rep) return;
    static const bool dump = std::getenv("QRB_PROF_DUMP") != nullptr;
    for (auto& r : h->prof.recs) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, r.a, r.b);
      if (dump)
        std::fprintf(stderr, "[qrb prof] kind %d ms %.4f gflop %.3f tflops %.2f\n", r.kind, ms,
                     r.flops * 1e-9, r.flops / (ms > 0 ? ms : 1e-9) * 1e-9);
      qrb_kernel_stat& k = rep->kernels[r.kind];
      k.ms += ms;
      k.flops += r.flops;
      k.bytes += r.bytes;
      k.launches += 1;
    }
  }
  ~ProfSession() {
    if (g_prof == &h->prof) g_prof = nullptr;
  }
};

// everything derived from the factors (R^-1 blocks, merged pair reflectors)
// must be rebuilt after the matrix or the factors were replaced
void invalidate_derived(qrb_handle* h) {
  h->rinv_ready = false;
  h->t2_ready = false;
  h->rinv2_ready = false;
  h->t4_ready = false;
  std::fill(h->t2_valid.begin(), h->t2_valid.end(), 0);
  std::fill(h->t4_valid.begin(), h->t4_valid.end(), 0);
}

// merged 2nb-wide reflectors of panel pairs (2p, 2p+1), for the solve's Q^T B
bool pair_ok(const qrb_handle* h, int k) {
  const int64_t j0 = int64_t(k) * h->nb;
  return outer_panels_solve() >= 2 && (k & 1) == 0 && j0 + 2 * int64_t(h->nb) <= h->n &&
         h->m - j0 >= 2 * int64_t(h->nb);
}

// right-hand-side batches from this width on merge the quad reflectors the
// factorization did not keep (qrb_set_tuning "t4_min_rhs")
static int64_t g_t4_min_rhs = 1024;

// merged 4nb-wide reflectors of panel quads (4q .. 4q+3)
bool quad_ok(const qrb_handle* h, int k) {
  const int64_t j0 = int64_t(k) * h->nb, w4 = 4 * int64_t(h->nb);
  return outer_panels_solve() >= 4 && (k & 3) == 0 && j0 + w4 <= h->n && h->m - j0 >= w4;
}

// storage of the merged pair reflectors (npairs blocks of 2nb x 2nb + scratch)
// and of the quad reflectors (nquads blocks of 4nb x 4nb)
int t2_storage(qrb_handle* h) {
  const int64_t w2 = 2 * int64_t(h->nb), blk = w2 * w2, blk4 = 4 * blk;
  const int npairs = h->npanels / 2, nquads = h->npanels / 4;
  if (!h->T2 && npairs > 0) {
    if (cudaMalloc(&h->T2, sizeof(double) * (npairs * blk + 2 * int64_t(h->nb) * h->nb)) !=
        cudaSuccess) {
      cudaGetLastError();
      h->T2 = nullptr;
      set_last_error("T2 alloc failed");
      return QRB_ENOMEM;
    }
    ++g_graph_epoch;
  }
  if (!h->T4 && nquads > 0) {
    if (cudaMalloc(&h->T4, sizeof(double) * nquads * blk4) != cudaSuccess) {
      cudaGetLastError();
      h->T4 = nullptr;
      set_last_error("T4 alloc failed");
      return QRB_ENOMEM;
    }
    ++g_graph_epoch;
  }
  h->t2_valid.assign(npairs, 0);
  h->t4_valid.assign(nquads, 0);
  return QRB_OK;
}

int ensure_t2(qrb_handle* h, Workspace& ws) {
  if (h->t2_ready) return QRB_OK;
  const int nb = h->nb;
  const int64_t w2 = 2 * int64_t(nb), blk = w2 * w2;
  const int npairs = h->npanels / 2;
  if (npairs == 0) {
    h->t2_ready = true;
    return QRB_OK;
  }
  if (!h->T2 || static_cast<int>(h->t2_valid.size()) != npairs) QRB_TRY(t2_storage(h));
  MatView A{h->A, h->m, h->n, h->lda};
  double* scratch = h->T2 + npairs * blk;
  for (int p = 0; p < npairs; ++p) {
    if (!pair_ok(h, 2 * p) || h->t2_valid[p]) continue;
    const double* Ta = h->T + int64_t(2 * p) * nb * nb;
    QRB_TRY(merge_pair_t(A, int64_t(2 * p) * nb, nb, Ta, Ta + int64_t(nb) * nb, h->T2 + p * blk,
                         w2, scratch, ws, h->stream));
    h->t2_valid[p] = 1;
  }
  h->t2_ready = true;
  return QRB_OK;
}

// quad reflectors the factorization did not keep (its pair steps), merged from
// the pair reflectors: T4 = [[T2a, -T2a (V_a^T V_b) T2b], [0, T2b]]
int ensure_t4(qrb_handle* h, Workspace& ws) {
  if (h->t4_ready) return QRB_OK;
  QRB_TRY(ensure_t2(h, ws));
  const int nb = h->nb;
  const int64_t w2 = 2 * int64_t(nb), blk2 = w2 * w2, w4 = 2 * w2, blk4 = w4 * w4;
  const int nquads = h->npanels / 4;
  MatView A{h->A, h->m, h->n, h->lda};
  for (int q = 0; q < nquads; ++q) {
    if (!quad_ok(h, 4 * q) || h->t4_valid[q]) continue;
    QRB_TRY(ws.T4.ensure(sizeof(double) * 2 * blk2, h->stream));
    QRB_TRY(merge_pair_t(A, int64_t(4 * q) * nb, static_cast<int>(w2),
                         h->T2 + int64_t(2 * q) * blk2, h->T2 + int64_t(2 * q + 1) * blk2,
                         h->T4 + q * blk4, w4, ws.T4.d(), ws, h->stream));
    h->t4_valid[q] = 1;
  }
  h->t4_ready = true;
  return QRB_OK;
}

int ensure_rinv(qrb_handle* h) {
  if (h->rinv_ready) return QRB_OK;
  QRB_TRY(trtri_blocks(h->A, h->lda, static_cast<int>(h->n), h->nb, h->Rinv, h->stream));
  g_launches += 1;
  h->rinv_ready = true;
  return QRB_OK;
}

// inverses of the 2nb x 2nb diagonal blocks of R for the panel pairs:
// [[A, B], [0, C]]^-1 = [[A^-1, -A^-1 B C^-1], [0, C^-1]] from the nb-block inverses
int ensure_rinv2(qrb_handle* h) {
  if (h->rinv2_ready) return QRB_OK;
  QRB_TRY(ensure_rinv(h));
  const int nb = h->nb;
  const int64_t w2 = 2 * int64_t(nb), blk = w2 * w2, nb2 = int64_t(nb) * nb;
  const int npairs = h->npanels / 2;
  if (npairs == 0) {
    h->rinv2_ready = true;
    return QRB_OK;
  }
  if (!h->Rinv2) {
    if (cudaMalloc(&h->Rinv2, sizeof(double) * (npairs * blk + nb2)) != cudaSuccess) {
      cudaGetLastError();
      h->Rinv2 = nullptr;
      set_last_error("qrb_solve: Rinv2 alloc failed");
      return QRB_ENOMEM;
    }
  }
  // every pair's diagonal block is inverted (pairs that the solve does not use --
  // a partial last panel -- are simply never read)
  const int full_pairs = static_cast<int>(std::min<int64_t>(npairs, h->n / w2));
  QRB_TRY(rinv2_pairs(h->A, h->lda, h->Rinv, nb, full_pairs, h->Rinv2, h->stream));
  g_launches += 1;
  h->rinv2_ready = true;
  return QRB_OK;
}

// B (n x nrhs) <- R^-1 B, bottom-up: panel pairs as 2nb blocks (inverse block +
// rank-2nb update, K = 2nb GEMMs), single nb blocks where no full pair exists.
// (4nb blocks -- the two pair inverses with the coupling block between them,
// then one K = 4nb update -- measured 38.1 -> 40.0 ms for 256 slices at config 3:
// the unsplit 256 x 256 coupling product costs more than the wider update saves)
int trsm_upper_h(qrb_handle* h, const MatView& B, cudaStream_t st) {
  const int nb = h->nb;
  const int64_t n = h->n, nrhs = B.cols;
  if (n <= 0 || nrhs <= 0) return QRB_OK;
  ProfScope ps(QRB_K_TRSM, static_cast<double>(n) * n * nrhs,
               8.0 * (0.5 * n * (double)n + 2.0 * n * (double)nrhs), st);
  MatView R{h->A, n, n, h->lda};
  const int64_t w2 = 2 * int64_t(nb);
  // Y_kb <- D Y_kb for the pair starting at panel kb (D = its 2nb x 2nb inverse)
  auto pair_diag = [&](int kb) -> int {
    const int64_t i0 = int64_t(kb) * nb;
    const int64_t bs = w2;
    MatView Yk = B.sub(i0, 0, bs, nrhs);
    const MatView D{h->Rinv2 + int64_t(kb / 2) * w2 * w2, bs, bs, w2};
    const int s2 = small_splits(static_cast<int>(bs), static_cast<int>(nrhs), static_cast<int>(bs));
    if (s2 > 1) {
      // Y_k <- D Y_k as split-K partial products reduced into Y_k (few output tiles)
      QRB_TRY(small_product(false, D, Yk, Yk.ptr, Yk.ld, static_cast<int>(bs),
                            static_cast<int>(nrhs), static_cast<int>(bs), s2, device_workspace(),
                            st));
      return QRB_OK;
    }
    // Y_k <- D Y_k through a copy (M = 2nb spans two row tiles: no in-place GEMM)
    const int64_t ldt = w2;
    QRB_TRY(h->Ytmp.ensure(sizeof(double) * ldt * nrhs, st));
    QRB_CUDA_TRY(cudaMemcpy2DAsync(h->Ytmp.d(), sizeof(double) * ldt, Yk.ptr,
                                   sizeof(double) * Yk.ld, sizeof(double) * bs, nrhs,
                                   cudaMemcpyDeviceToDevice, st));
    QRB_TRY(gemm_nn(D, MatView{h->Ytmp.d(), bs, nrhs, ldt}, Yk.ptr, Yk.ld, bs, nrhs, bs,
                    GEMM_EPI_STORE, 0, st));
    g_launches += 1;
    return QRB_OK;
  };
  for (int k = h->npanels - 1; k >= 0;) {
    const bool pair = (k & 1) && pair_ok(h, k - 1);
    const int kb = pair ? k - 1 : k;
    const int64_t i0 = int64_t(kb) * nb;
    const int64_t bs = pair ? w2 : std::min<int64_t>(nb, n - i0);
    MatView Yk = B.sub(i0, 0, bs, nrhs);
    if (pair) {
      QRB_TRY(pair_diag(kb));
    } else {
      MatView Ri{h->Rinv + int64_t(kb) * nb * nb, bs, bs, nb};
      QRB_TRY(gemm_nn(Ri, Yk, Yk.ptr, Yk.ld, bs, nrhs, bs, GEMM_EPI_STORE, 0, st));
      g_launches += 1;
    }
    if (i0 > 0) {
      MatView Rk = R.sub(0, i0, i0, bs);
      QRB_TRY(gemm_nn(Rk, Yk, B.ptr, B.ld, i0, nrhs, bs, GEMM_EPI_SUB, 0, st));
      g_launches += 1;
    }
    k = kb - 1;
  }
  return QRB_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// right-looking steps from column col0 to the end, panel pairs with look-ahead
//
// Step s (pair at j0, merged reflector V, T2; trailing columns c0 = j0 + 2nb ..):
//   main stream:  C[:, c0 : c0+2nb] <- Q^T C   (the next pair's columns, all SMs)
//                 C[:, c0+2nb : c_cap] <- Q^T C  (GEMM grids capped to sms - R)
//                 C[:, c_cap : n]  <- Q^T C      (all SMs)
//   side stream:  (after the first update) factor the next pair on the R free
//                 SMs -- the panel's latency-bound chain (small factorizations,
//                 launch gaps, host flag check) runs under the big update.
// c_cap is a deterministic function of the shape (a model of the panel time on
// R SMs), so the rounding of every column is the same run to run.  With too
// little trailing work left the step runs serially (panel, then update).
// ---------------------------------------------------------------------------
static int g_lookahead = [] {
  const char* e = std::getenv("QRB_LOOKAHEAD");
  return e ? std::atoi(e) : 1;
}();
static int g_la_sms = 16;              // SMs left to the look-ahead panel (r01 sweep: 8..48)
static int64_t g_la_lat_us = 450;      // latency part of a pair's panel chain (r01 sweep)
static int64_t g_la_margin_pct = 10;   // capped window = (1 + margin) x modelled panel time
static int64_t g_la_sms_max = 72;      // chain-bound steps may leave the chain up to this many SMs
static int g_early_singles = 1;        // "early_singles": two-piece update of narrow single-panel factorizations
static int64_t g_early_sms = 8;        // SMs its second piece leaves to the chain (0: none reserved; sweep 0..32: 1.492, 1.482 at 4-16)
static int64_t g_la_sms_tall = 16;     // SMs left to the chain in steps with >= g_la_tall_rows rows (24: cleaner overlap, -0.15% at config 3)
static int64_t g_la_tall_rows = 32768;
static std::atomic<int64_t> g_la_steps{0};
// outer_panels = 4 (default): 4-panel blocks while >= 24576 trailing columns
// remain, pairs after (r01 sweep at config 3: pairs only 34.49, 4-panel blocks
// to 16384 / 32768 / 49152 remaining columns 34.75 / 34.75 / 34.63 TFLOP/s;
// config 2 (16384 columns) never takes them)
static int64_t g_outer4_min_cols = 24576;
// factorizations with at most this many columns run as a captured CUDA graph
// (qrb_set_tuning "graph_max_cols"; 0 = never)
static int64_t g_graph_max_cols = [] {
  const char* e = std::getenv("QRB_GRAPH_MAX_COLS");
  return e ? std::atoll(e) : int64_t(16384);
}();

static int report_progress(qrb_handle* h, int64_t cols, cudaStream_t st) {
  if (!h->progress) return QRB_OK;
  progress_kernel<<<1, 1, 0, st>>>(h->progress, cols);
  QRB_CUDA_TRY(cudaGetLastError());
  g_launches += 1;
  return QRB_OK;
}

static int right_looking(qrb_handle* h, int64_t col0, Workspace& ws, cudaStream_t st) {
  const int nb = h->nb;
  const int64_t m = h->m, n = h->n, w2 = 2 * int64_t(nb), blk2 = w2 * w2;
  // outer block = q panels (2: a pair, 4: two pairs merged -> K = 4nb updates)
  const int op = outer_panels_for(n);
  const int q = op >= 4 ? 4 : 2;
  const int64_t wq = q * int64_t(nb), blkq = wq * wq;
  MatView A{h->A, m, n, h->lda};
  auto block_here = [&](int64_t j0, int64_t w) {
    // 4-panel blocks only while at least g_outer4_min_cols trailing columns
    // remain (their K = 4nb update pays where the update is long; late steps
    // take pairs, whose shorter panel chain hides better)
    if (w > w2 && n - j0 - w < g_outer4_min_cols) return false;
    return op >= 2 && j0 + w < n && m - j0 >= w;
  };
  // width of the block at j0: 4nb / 2nb blocks, or with single panels (op = 1)
  // nb-wide blocks that still take the look-ahead (the last panel runs serially)
  auto block_at = [&](int64_t j0) -> int64_t {
    const bool single = op == 1 || (g_outer_panels == 0 && g_tail_singles && !block_here(j0, wq));
    if (single) return (j0 + nb < n && m - j0 >= nb) ? nb : 0;
    return block_here(j0, wq) ? wq : block_here(j0, w2) ? w2 : 0;
  };
  // merged reflector storage: pairs starting at an even panel are kept for the
  // solve (h->T2); others alternate between two scratch slots
  auto t2dst = [&](int64_t j0) -> double* {
    const int64_t kp = j0 / nb;
    if ((kp & 1) == 0) return h->T2 + (kp / 2) * blk2;
    return h->T2scratch.d() + ((j0 / w2) & 1) * blk2;
  };
  auto t2mark = [&](int64_t j0) {
    const int64_t kp = j0 / nb;
    if ((kp & 1) == 0) h->t2_valid[kp / 2] = 1;
  };
  QRB_TRY(h->T2scratch.ensure(sizeof(double) * 2 * blk2, st));
  if (q == 4) QRB_TRY(h->T4scratch.ensure(sizeof(double) * 2 * blkq, st));
  // a q-panel block at j0: pairs factored in sequence (Q_pair^T on the next
  // pair's columns in between), merged reflector in *Tout
  auto factor_block = [&](int64_t j0, int w, Workspace& wsb, cudaStream_t sb,
                          double** Tout) -> int {
    const int64_t mk = m - j0;
    double* Tk = h->T + (j0 / nb) * nb * int64_t(nb);
    if (w == nb) {  // single panel (T of ld nb)
      QRB_TRY(factor_panel(A.sub(j0, j0, mk, nb), h->tau + j0, Tk, nb, wsb, sb));
      *Tout = Tk;
      return QRB_OK;
    }
    double* T2a = nullptr;
    QRB_TRY(factor_panel_pair(A, j0, nb, Tk, Tk + int64_t(nb) * nb, h->tau, &T2a, wsb, sb,
                              t2dst(j0)));
    t2mark(j0);
    if (w == w2) {
      *Tout = T2a;
      return QRB_OK;
    }
    QRB_TRY(apply_qt(A.sub(j0, j0, mk, w2), T2a, w2, A.sub(j0, j0 + w2, mk, w2), wsb, sb));
    double* Tb = Tk + 2 * int64_t(nb) * nb;
    double* T2b = nullptr;
    QRB_TRY(factor_panel_pair(A, j0 + w2, nb, Tb, Tb + int64_t(nb) * nb, h->tau, &T2b, wsb, sb,
                              t2dst(j0 + w2)));
    t2mark(j0 + w2);
    QRB_TRY(wsb.T4.ensure(sizeof(double) * 2 * blk2, sb));
    // quad-aligned blocks keep their merged reflector for the solve
    const bool keep = h->T4 && j0 % wq == 0 && quad_ok(h, static_cast<int>(j0 / nb));
    double* T4 = keep ? h->T4 + (j0 / wq) * blkq : h->T4scratch.d() + ((j0 / wq) & 1) * blkq;
    QRB_TRY(merge_pair_t(A, j0, static_cast<int>(w2), T2a, T2b, T4, wq, wsb.T4.d(), wsb, sb));
    if (keep) h->t4_valid[j0 / wq] = 1;
    *Tout = T4;
    return QRB_OK;
  };
  const int sms = gemm_sm_count();
  const int R = std::min(g_la_sms, sms / 2);
  if (g_lookahead && !h->side) {
    int lo = 0, hi = 0;
    QRB_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    QRB_CUDA_TRY(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi));
    QRB_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_upd, cudaEventDisableTiming));
    QRB_CUDA_TRY(cudaEventCreateWithFlags(&h->ev_pan, cudaEventDisableTiming));
  }
  // the look-ahead's panel workspace is shared with qrb_op_panel_block(side = 1)
  std::unique_ptr<WsUse> side_use;
  if (h->side) side_use.reset(new WsUse(side_workspace(), h->side));
  const double rate = 34.0e9;  // flop per ms of the DMMA update on all SMs (r01 bench)
  double* TB = nullptr;
  int64_t have = 0;  // width of the block at j0 factored by the previous step's look-ahead
  int64_t j0 = col0;
  while (j0 < n) {
    const int64_t mk = m - j0;
    double* Tk = h->T + (j0 / nb) * nb * int64_t(nb);
    const int64_t w = have ? have : block_at(j0);
    if (w == 0) {
      const int64_t pw = std::min<int64_t>(nb, n - j0);
      QRB_TRY(factor_panel(A.sub(j0, j0, mk, pw), h->tau + j0, Tk, nb, ws, st));
      QRB_TRY(report_progress(h, j0 + pw, st));
      if (j0 + pw < n)
        QRB_TRY(apply_qt(A.sub(j0, j0, mk, pw), Tk, nb, A.sub(j0, j0 + pw, mk, n - j0 - pw), ws,
                         st));
      j0 += pw;
      have = 0;
      continue;
    }
    if (!have) QRB_TRY(factor_block(j0, static_cast<int>(w), ws, st, &TB));
    QRB_TRY(report_progress(h, j0 + w, st));  // (a look-ahead block: st waited for it)
    have = 0;
    const int64_t c0 = j0 + w, rest = n - c0;
    const MatView V = A.sub(j0, j0, mk, w);
    const int64_t wn = block_at(c0);
    bool la = g_lookahead && h->side && wn > 0;
    int64_t ncap = 0;
    int Rs = R;  // SMs left to the chain in this step
    if (la) {
      // modelled chain time of the next block on R SMs: latency part + its GEMM
      // flops (per pair: 2 Gram + 2 NN per panel, Q_a^T on panel b, the T merge
      // ~ 26 m nb^2; a 4-panel block ~2.3 pairs)
      const double mk1 = static_cast<double>(m - c0);
      const double pairs = wn == nb ? 0.45 : wn == w2 ? 1.0 : 2.3;
      const double per_col = 2.0 * static_cast<double>(mk) * w;  // NN flops per column
      auto chain_ms = [&](int r) {
        return pairs * (g_la_lat_us * 1e-3 + 26.0 * mk1 * nb * nb / (rate * r / sms));
      };
      // chain-bound steps (the whole capped update is shorter than the chain on
      // R SMs: the second half of a config-2-sized factorization): leave the
      // chain more SMs, up to "la_sms_max", until the two balance
      // tall steps: the chain's GEMM part grows with the rows (7.4 ms per pair on
      // 16 SMs at m = 69120, 13.9 ms on 8), and a chain that outlasts its capped
      // window contends with the full-grid launches that follow; from
      // "la_tall_rows" rows on it gets "la_sms_tall" SMs
      Rs = mk1 >= static_cast<double>(g_la_tall_rows)
               ? std::max<int>(R, static_cast<int>(std::min<int64_t>(g_la_sms_tall, sms / 2)))
               : R;
      if (g_la_sms_max > Rs)
        while (Rs + 8 <= std::min<int64_t>(g_la_sms_max, sms / 2 + 22) &&
               chain_ms(Rs) > (rest - wn) * per_col / (rate * (sms - Rs) / sms))
          Rs += 8;
      const double tp = chain_ms(Rs);
      const double capped_rate = rate * (sms - Rs) / sms;
      const double want = (1.0 + g_la_margin_pct / 100.0) * tp * capped_rate / per_col;
      ncap = std::min<int64_t>(rest - wn, (static_cast<int64_t>(want) + 63) / 64 * 64);
      // lookahead = 1: always (even a short update hides part of the panel:
      // r01 sweep, config 2 27.5 -> 28.8 TFLOP/s against skipping short steps);
      // lookahead = 3: only when the remaining NN update outlasts the panel chain
      if (g_lookahead == 3) la = (rest - wn) * per_col / capped_rate > tp;
      // single panels overlap only on wider matrices (r02: 4230 x 4096 14.46 ->
      // 13.92 ms with look-ahead; config 1, 2160 x 1024, 2.17 -> 2.20 ms)
      if (wn == nb && g_lookahead == 1 && n < 2048) la = false;
    }
    // Narrow factorizations of single panels (config 1: 2160 x 1024): the update
    // is too short to hide anything behind its NN part alone, so it is applied in
    // two complete pieces -- the next panel's columns first (TN + T^T + NN on nb
    // columns), then the rest -- and the next panel's chain starts after the
    // first piece, beside the second.  The two-piece arithmetic is used with and
    // without look-ahead (the split-K of a piece depends on its width), so the
    // factors stay bitwise identical between the two.
    if (g_early_singles && wn == nb && w == nb && n < 2048 && rest > wn) {
      const MatView C = A.sub(j0, c0, mk, rest);
      QRB_TRY(apply_qt(V, TB, w, C.sub(0, 0, mk, wn), ws, st));
      const bool ov = g_lookahead && h->side;
      if (ov) QRB_CUDA_TRY(cudaEventRecord(h->ev_upd, st));
      {
        // (beside the chain the second piece leaves it "early_sms" SMs)
        GemmGridCap cap(ov && g_early_sms > 0 ? sms - static_cast<int>(g_early_sms) : gemm_grid_cap());
        QRB_TRY(apply_qt(V, TB, w, C.sub(0, wn, mk, rest - wn), ws, st));
      }
      if (ov) {
        ++g_la_steps;
        QRB_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_upd, 0));
        QRB_TRY(factor_block(c0, static_cast<int>(wn), side_workspace(), h->side, &TB));
        QRB_CUDA_TRY(cudaEventRecord(h->ev_pan, h->side));
        QRB_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_pan, 0));
        have = wn;
      }
      j0 = c0;
      continue;
    }
    if (!la) {
      QRB_TRY(apply_qt(V, TB, w, A.sub(j0, c0, mk, rest), ws, st));
      j0 = c0;
      continue;
    }
    ++g_la_steps;
    // W2 for every trailing column in one TN pass (same split-K as the serial
    // schedule: bitwise-identical results), then the NN update in three parts
    const MatView C = A.sub(j0, c0, mk, rest);
    QRB_TRY(apply_qt_w2(V, TB, w, C, ws, st));
    QRB_TRY(apply_qt_nn(V, C, 0, wn, ws, st));
    QRB_CUDA_TRY(cudaEventRecord(h->ev_upd, st));
    {
      GemmGridCap cap(sms - Rs);
      QRB_TRY(apply_qt_nn(V, C, wn, ncap, ws, st, QRB_K_GEMM_NN_CAP));
    }
    QRB_TRY(apply_qt_nn(V, C, wn + ncap, rest - wn - ncap, ws, st));
    // the next block on the side stream (its host-side flag check blocks this
    // thread only while the update above is already queued on the GPU)
    QRB_CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev_upd, 0));
    QRB_TRY(factor_block(c0, static_cast<int>(wn), side_workspace(), h->side, &TB));
    QRB_CUDA_TRY(cudaEventRecord(h->ev_pan, h->side));
    QRB_CUDA_TRY(cudaStreamWaitEvent(st, h->ev_pan, 0));
    have = wn;
    j0 = c0;
  }
  return QRB_OK;
}

// ---------------------------------------------------------------------------
// graph-captured factorization (qrb_factorize, n <= graph_max_cols)
//
// Configs 1-2 are bound by the panel chain's launch latency (r02 trace of
// config 1: 183 gaps, 0.6 of 3.3 ms idle).  With the CholeskyQR2 fallback
// chosen on the device the whole right-looking schedule -- both streams of the
// look-ahead included -- has no host decision left, so it is captured once per
// handle and replayed as one graph.  The first factorization of a handle runs
// eagerly (it sizes every buffer and creates the look-ahead stream); any buffer
// growth or tuning change afterwards bumps g_graph_epoch and forces a fresh
// capture.  A capture that fails for any reason runs the schedule eagerly.
// Same kernels, same order, same shapes: the factors are bitwise those of the
// eager run.
// ---------------------------------------------------------------------------
static std::atomic<int64_t> g_graph_captures{0}, g_graph_replays{0};

static int factorize_graphed(qrb_handle* h, Workspace& ws, cudaStream_t st) {
  const uint64_t epoch = g_graph_epoch.load();
  if (h->fgraph && h->fgraph_epoch == epoch) {
    ++g_graph_replays;
    WsUse side_use(side_workspace(), st);  // the graph's look-ahead panels use it
    QRB_CUDA_TRY(cudaGraphLaunch(h->fgraph, st));
    g_launches += h->fgraph_launches;
    h->t2_valid = h->fgraph_t2;
    h->t4_valid = h->fgraph_t4;
    return QRB_OK;
  }
  if (h->fgraph) {
    cudaGraphExecDestroy(h->fgraph);
    h->fgraph = nullptr;
  }
  if (!h->fgraph_warm) {
    h->fgraph_warm = true;
    return right_looking(h, 0, ws, st);
  }
  const int64_t l0 = g_launches.load();
  if (!capture_helper_stream()) return right_looking(h, 0, ws, st);
  QRB_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const int rc = right_looking(h, 0, ws, st);
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(st, &graph);
  cudaGraphExec_t exec = nullptr;
  bool ok = rc == QRB_OK && ce == cudaSuccess && graph != nullptr;
  if (ok)
    ok = cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority) ==
         cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  if (!ok) {
    static const bool dbg = std::getenv("QRB_GRAPH_DEBUG") != nullptr;
    if (dbg)
      std::fprintf(stderr, "[qrb] factorization capture failed: rc %d, %s, last error: %s\n", rc,
                   cudaGetErrorString(ce), t_last_error.c_str());
    cudaGetLastError();  // nothing ran during the capture: do it eagerly
    g_launches = l0;
    h->fgraph_epoch = 0;
    return right_looking(h, 0, ws, st);
  }
  h->fgraph = exec;
  h->fgraph_epoch = g_graph_epoch.load() == epoch ? epoch : 0;
  h->fgraph_launches = g_launches.load() - l0;
  h->fgraph_t2 = h->t2_valid;
  h->fgraph_t4 = h->t4_valid;
  ++g_graph_captures;
  QRB_CUDA_TRY(cudaGraphLaunch(exec, st));
  return QRB_OK;
}

static bool graph_eligible(const qrb_handle* h) {
  return g_graph_max_cols > 0 && h->n <= g_graph_max_cols && !h->profiling && !g_prof &&
         !gemm_nn_dynamic();
}

// what this host thread's last qrb_op_apply_qt_begin formed (checked by _cols)
struct BeginRecord {
  uint64_t gen = 0;
  const void* V = nullptr;
  int64_t m = 0, w = 0;
  void* stream = nullptr;
};
static thread_local BeginRecord t_begin;

extern "C" {

int qrb_version(void) { return 100; }

const char* qrb_last_error(void) { return t_last_error.c_str(); }

int qrb_device_count(int* count) {
  if (!count) return QRB_EARG;
  QRB_CUDA_TRY(cudaGetDeviceCount(count));
  return QRB_OK;
}

int qrb_set_device(int device) {
  QRB_CUDA_TRY(cudaSetDevice(device));
  return QRB_OK;
}

static int create_handle(int device, int64_t m, int64_t n, int nb, double* view, int64_t ld,
                         qrb_handle** out) {
  if (!out || m < 1 || n < 1 || m < n || nb < 16 || nb > 128 || (nb % 16) != 0) {
    set_last_error("qrb_create: need m >= n >= 1 and nb in {16, 32, ..., 128}");
    return QRB_EARG;
  }
  if (m > (int64_t(1) << 31) - 1024 || n > (int64_t(1) << 31) - 1024) {
    set_last_error("qrb_create: dimensions exceed int32 TMA coordinates");
    return QRB_EARG;
  }
  if (view && (ld < m || (ld & 1) || (reinterpret_cast<uintptr_t>(view) & 15))) {
    set_last_error("qrb_create_view: need ld >= m, ld even and a 16-byte aligned matrix");
    return QRB_EARG;
  }
  *out = nullptr;
  QRB_CUDA_TRY(cudaSetDevice(device));
  qrb_handle* h = new qrb_handle();
  h->device = device;
  h->m = m;
  h->n = n;
  h->lda = view ? ld : (m + 31) & ~int64_t(31);
  h->nb = nb;
  h->npanels = static_cast<int>((n + nb - 1) / nb);
  h->owns_a = view == nullptr;
  auto fail = [&](const char* what) {
    set_last_error(std::string("qrb_create: ") + what);
    qrb_destroy(h);
    return QRB_ENOMEM;
  };
  if (view)
    h->A = view;
  else if (cudaMalloc(&h->A, sizeof(double) * h->lda * n) != cudaSuccess)
    return fail("matrix alloc");
  if (cudaMalloc(&h->tau, sizeof(double) * n) != cudaSuccess) return fail("tau alloc");
  if (cudaMalloc(&h->T, sizeof(double) * nb * nb * h->npanels) != cudaSuccess)
    return fail("T alloc");
  if (cudaMalloc(&h->Rinv, sizeof(double) * nb * nb * h->npanels) != cudaSuccess)
    return fail("Rinv alloc");
  cudaGetLastError();
  // a blocking stream: it orders implicitly with the legacy default stream,
  // so device buffers produced there (e.g. by torch) are complete before use
  QRB_CUDA_TRY(cudaStreamCreate(&h->own_stream));
  h->stream = h->own_stream;
  QRB_CUDA_TRY(cudaEventCreate(&h->ev0));
  QRB_CUDA_TRY(cudaEventCreate(&h->ev1));
  QRB_CUDA_TRY(cudaEventCreate(&h->ev2));
  if (!view) QRB_CUDA_TRY(cudaMemsetAsync(h->A, 0, sizeof(double) * h->lda * n, h->stream));
  QRB_CUDA_TRY(cudaMemsetAsync(h->T, 0, sizeof(double) * nb * nb * h->npanels, h->stream));
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  *out = h;
  return QRB_OK;
}

int qrb_create(int device, int64_t m, int64_t n, int nb, qrb_handle** out) {
  return create_handle(device, m, n, nb, nullptr, 0, out);
}

int qrb_create_view(int device, int64_t m, int64_t n, int nb, double* A, int64_t lda,
                    qrb_handle** out) {
  if (!A) {
    set_last_error("qrb_create_view: null matrix");
    return QRB_EARG;
  }
  return create_handle(device, m, n, nb, A, lda, out);
}

int qrb_destroy(qrb_handle* h) {
  if (!h) return QRB_OK;
  DeviceGuard g(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->own_stream && h->own_stream != h->stream) cudaStreamSynchronize(h->own_stream);
  if (h->A && h->owns_a) cudaFree(h->A);
  if (h->tau) cudaFree(h->tau);
  if (h->T) cudaFree(h->T);
  if (h->Rinv) cudaFree(h->Rinv);
  if (h->T2) cudaFree(h->T2);
  if (h->T4) cudaFree(h->T4);
  if (h->Rinv2) cudaFree(h->Rinv2);
  h->Ytmp.release();
  h->Bw.release();
  h->resid.release();
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->ev2) cudaEventDestroy(h->ev2);
  if (h->side) {
    cudaStreamSynchronize(h->side);
    cudaStreamDestroy(h->side);
  }
  if (h->ev_upd) cudaEventDestroy(h->ev_upd);
  if (h->ev_pan) cudaEventDestroy(h->ev_pan);
  h->T2scratch.release();
  h->T4scratch.release();
  if (h->fgraph) cudaGraphExecDestroy(h->fgraph);
  if (h->own_stream) cudaStreamDestroy(h->own_stream);
  delete h;
  return QRB_OK;
}

int qrb_set_stream(qrb_handle* h, void* stream) {
  if (!h) return QRB_EARG;
  DeviceGuard g(h->device);
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
  return QRB_OK;
}

int qrb_set_profiling(qrb_handle* h, int on) {
  if (!h) return QRB_EARG;
  h->profiling = on != 0;
  return QRB_OK;
}

int qrb_set_matrix(qrb_handle* h, int64_t col0, int64_t ncols, const double* src, int64_t ld,
                   int src_on_device) {
  if (!h || !src || col0 < 0 || ncols < 0 || col0 + ncols > h->n || ld < h->m) {
    set_last_error("qrb_set_matrix: bad arguments");
    return QRB_EARG;
  }
  DeviceGuard g(h->device);
  if (ncols == 0) return QRB_OK;
  QRB_CUDA_TRY(cudaMemcpy2DAsync(h->A + col0 * h->lda, h->lda * sizeof(double), src,
                                 ld * sizeof(double), h->m * sizeof(double), ncols,
                                 src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 h->stream));
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->factored = false;
  invalidate_derived(h);
  return QRB_OK;
}

int qrb_get_matrix_async(qrb_handle* h, int64_t col0, int64_t ncols, double* dst, int64_t ld,
                         void* stream) {
  if (!h || !dst || col0 < 0 || ncols < 0 || col0 + ncols > h->n || ld < h->m) {
    set_last_error("qrb_get_matrix_async: bad arguments");
    return QRB_EARG;
  }
  DeviceGuard g(h->device);
  if (ncols == 0) return QRB_OK;
  QRB_CUDA_TRY(cudaMemcpy2DAsync(dst, ld * sizeof(double), h->A + col0 * h->lda,
                                 h->lda * sizeof(double), h->m * sizeof(double), ncols,
                                 cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  return QRB_OK;
}

int qrb_get_matrix(qrb_handle* h, int64_t col0, int64_t ncols, double* dst, int64_t ld,
                   int dst_on_device) {
  if (!h || !dst || col0 < 0 || ncols < 0 || col0 + ncols > h->n || ld < h->m) {
    set_last_error("qrb_get_matrix: bad arguments");
    return QRB_EARG;
  }
  DeviceGuard g(h->device);
  if (ncols == 0) return QRB_OK;
  QRB_CUDA_TRY(cudaMemcpy2DAsync(dst, ld * sizeof(double), h->A + col0 * h->lda,
                                 h->lda * sizeof(double), h->m * sizeof(double), ncols,
                                 dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 h->stream));
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return QRB_OK;
}

int qrb_factorize(qrb_handle* h, qrb_report* rep) {
  clear_report(rep);
  if (!h) return QRB_EARG;
  DeviceGuard g(h->device);
  h->factored = false;  // until this factorization completes
  invalidate_derived(h);
  Workspace& ws = device_workspace();
  WsUse use(ws, h->stream);
  const int64_t launches0 = g_launches.load();
  cudaStream_t st = h->stream;
  // non-finite input -> KernelInputError (kernels.py:305-306)
  {
    QRB_TRY(ws.bar.ensure(64, st));
    int* flag = static_cast<int*>(ws.bar.p) + 4;
    QRB_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int), st));
    nonfinite_kernel<<<4 * 148, 256, 0, st>>>(h->A, h->lda, h->m, h->n, flag);
    QRB_CUDA_TRY(cudaGetLastError());
    int hflag = 0;
    QRB_CUDA_TRY(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    QRB_CUDA_TRY(cudaStreamSynchronize(st));
    g_launches += 2;
    if (hflag) {
      set_last_error("factorize: input matrix has non-finite entries");
      return QRB_ENONFINITE;
    }
  }
  const bool timing = std::getenv("QRB_TIMING") != nullptr;
  double panel_ms = 0.0, update_ms = 0.0;
  ProfSession session(h);
  cudaEvent_t ep0 = nullptr, ep1 = nullptr, ep2 = nullptr;
  if (timing) {
    cudaEventCreate(&ep0);
    cudaEventCreate(&ep1);
    cudaEventCreate(&ep2);
  }
  QRB_TRY(t2_storage(h));
  QRB_CUDA_TRY(cudaEventRecord(h->ev0, st));
  MatView A{h->A, h->m, h->n, h->lda};
  if (!timing) {
    if (graph_eligible(h))
      QRB_TRY(factorize_graphed(h, ws, st));
    else
      QRB_TRY(right_looking(h, 0, ws, st));
  } else {
    for (int k = 0; k < h->npanels; ++k) {  // serial, single panels, per-phase events
      const int64_t j0 = int64_t(k) * h->nb;
      const int64_t pw = std::min<int64_t>(h->nb, h->n - j0);
      const int64_t mk = h->m - j0;
      double* Tk = h->T + int64_t(k) * h->nb * h->nb;
      cudaEventRecord(ep0, st);
      QRB_TRY(factor_panel(A.sub(j0, j0, mk, pw), h->tau + j0, Tk, h->nb, ws, st));
      cudaEventRecord(ep1, st);
      if (j0 + pw < h->n)
        QRB_TRY(apply_qt(A.sub(j0, j0, mk, pw), Tk, h->nb,
                         A.sub(j0, j0 + pw, mk, h->n - j0 - pw), ws, st));
      cudaEventRecord(ep2, st);
      cudaEventSynchronize(ep2);
      panel_ms += elapsed(ep0, ep1);
      update_ms += elapsed(ep1, ep2);
    }
  }
  QRB_CUDA_TRY(cudaEventRecord(h->ev1, st));
  QRB_CUDA_TRY(cudaEventSynchronize(h->ev1));
  QRB_CUDA_TRY(cudaGetLastError());
  if (timing) {
    cudaEventDestroy(ep0);
    cudaEventDestroy(ep1);
    cudaEventDestroy(ep2);
  }
  h->factored = true;
  h->rinv_ready = false;
  h->t2_ready = false;
  h->rinv2_ready = false;
  session.finish(rep);
  if (rep) {
    const double m = static_cast<double>(h->m), n = static_cast<double>(h->n);
    rep->total_ms = elapsed(h->ev0, h->ev1);
    rep->panel_ms = panel_ms;
    rep->update_ms = update_ms;
    rep->flops = 2.0 * m * n * n - 2.0 * n * n * n / 3.0;
    rep->kernel_launches = g_launches.load() - launches0;
  }
  return QRB_OK;
}

// Deterministic left-looking -> right-looking switch of qrb_factorize_host: the
// chunk index at which the modelled compute of the left-looking chunks before it
// covers the modelled H2D time of the whole matrix (PCIe ~45 GB/s, update
// ~34 TFLOP/s).  A function of the shape only, so the factors (and their
// rounding) are the same every run; QRB_E2E_NO_SWITCH keeps the left-looking
// order to the end.
static int64_t host_switch_chunk(int64_t m, int64_t n, int64_t W, int64_t nchunks,
                                 double input_gbps = 45.0) {
  static const bool no_switch = std::getenv("QRB_E2E_NO_SWITCH") != nullptr;
  if (no_switch) return nchunks;
  const double copy_s = 8.0 * static_cast<double>(m) * n / (input_gbps * 1e9);
  double work_s = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) {
    if (c > 0 && work_s >= copy_s) return c;
    const double c0 = static_cast<double>(c * W), w = static_cast<double>(std::min(W, n - c * W));
    // Q^T of the c0 earlier columns on this chunk + the chunk's own QR
    work_s += (4.0 * m * c0 * w + 2.0 * (m - c0) * w * w) / 34e12;
  }
  return nchunks;
}

// ready != nullptr: chunk c of src (columns [c W, c W + W)) may be read only once
// ready[c] != 0 -- the caller is still filling src (e.g. from disk) while the
// factorization runs; input_gbps is the rate the model of the left-looking ->
// right-looking switch assumes for the arrival of the whole matrix.
static int factorize_host_impl(qrb_handle* h, const double* src, int64_t ld, int64_t chunk_cols,
                               const volatile int32_t* ready, double input_gbps,
                               int64_t* progress_host, qrb_report* rep) {
  clear_report(rep);
  if (!h || !src || ld < h->m || chunk_cols < 0) {
    set_last_error("qrb_factorize_host: bad arguments");
    return QRB_EARG;
  }
  DeviceGuard g(h->device);
  h->factored = false;  // A is overwritten from here on
  invalidate_derived(h);
  Workspace& ws = device_workspace();
  WsUse use(ws, h->stream);
  const int64_t launches0 = g_launches.load();
  cudaStream_t st = h->stream;
  const int nb = h->nb;
  int64_t W = chunk_cols;
  if (W == 0) W = 4096;  // measured best at config 3 (2048..32768 swept)
  W = std::max<int64_t>(nb, (W + nb - 1) / nb * nb);
  const int64_t nchunks = (h->n + W - 1) / W;
  const int64_t c_switch =
      host_switch_chunk(h->m, h->n, W, nchunks, input_gbps > 0 ? input_gbps : 45.0);
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> landed(nchunks, nullptr);
  cudaEvent_t c0ev = nullptr, c1ev = nullptr;
  ProfSession session(h);
  // the whole call; every failure returns through here so the copy stream is
  // drained and its events released (the caller's src may still be read by it)
  auto body = [&]() -> int {
    QRB_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    QRB_CUDA_TRY(cudaEventCreate(&c0ev));
    QRB_CUDA_TRY(cudaEventCreate(&c1ev));
    // the copy stream starts after everything already queued on the handle's stream
    QRB_CUDA_TRY(cudaEventRecord(h->ev0, st));
    QRB_CUDA_TRY(cudaStreamWaitEvent(cs, h->ev0, 0));
    QRB_CUDA_TRY(cudaEventRecord(c0ev, cs));
    // copies are enqueued in chunk order; gated chunks only once the caller has
    // filled them (this thread waits, the GPU keeps working on queued chunks)
    int64_t enq = 0;
    auto copy_upto = [&](int64_t last) -> int {
      for (; enq <= last && enq < nchunks; ++enq) {
        const int64_t col0 = enq * W, nc = std::min(W, h->n - col0);
        if (ready) {
          while (ready[enq] == 0) std::this_thread::sleep_for(std::chrono::microseconds(50));
          if (ready[enq] < 0) {  // the caller could not produce this chunk
            set_last_error("qrb_factorize_host_gated: input chunk " + std::to_string(enq) +
                           " reported unavailable");
            return QRB_EARG;
          }
        }
        QRB_CUDA_TRY(cudaEventCreateWithFlags(&landed[enq], cudaEventDisableTiming));
        QRB_CUDA_TRY(cudaMemcpy2DAsync(h->A + col0 * h->lda, h->lda * sizeof(double),
                                       src + col0 * ld, ld * sizeof(double),
                                       h->m * sizeof(double), nc, cudaMemcpyHostToDevice, cs));
        QRB_CUDA_TRY(cudaEventRecord(landed[enq], cs));
        if (enq == nchunks - 1) QRB_CUDA_TRY(cudaEventRecord(c1ev, cs));
      }
      return QRB_OK;
    };
    if (!ready) QRB_TRY(copy_upto(nchunks - 1));
    MatView A{h->A, h->m, h->n, h->lda};
    QRB_TRY(t2_storage(h));
    // non-finite input check per landed chunk (flag read once at the end)
    QRB_TRY(ws.bar.ensure(64, st));
    int* nf = static_cast<int*>(ws.bar.p) + 8;
    QRB_CUDA_TRY(cudaMemsetAsync(nf, 0, sizeof(int), st));
    const int64_t w2 = 2 * int64_t(nb), blk2 = w2 * w2;
    // Q_k^T for every factored panel k < kc0 on the columns C (left-looking):
    // pairs with their merged reflector (K = 2nb GEMMs; the TN runs 35.7 instead
    // of 31.2 TFLOP/s at M = 2nb), single panels otherwise
    auto apply_prev = [&](int kc0, int64_t c0, int64_t ncols) -> int {
      for (int k = 0; k < kc0;) {
        const int64_t j0 = int64_t(k) * nb, mk = h->m - j0;
        if ((k & 1) == 0 && k + 1 < kc0 && h->t2_valid[k / 2]) {
          QRB_TRY(apply_qt(A.sub(j0, j0, mk, w2), h->T2 + int64_t(k / 2) * blk2, w2,
                           A.sub(j0, c0, mk, ncols), ws, st));
          k += 2;
          continue;
        }
        QRB_TRY(apply_qt(A.sub(j0, j0, mk, nb), h->T + int64_t(k) * nb * nb, nb,
                         A.sub(j0, c0, mk, ncols), ws, st));
        ++k;
      }
      return QRB_OK;
    };
    for (int64_t c = 0; c < nchunks; ++c) {
      const int64_t col0 = c * W, nc = std::min(W, h->n - col0);
      if (c > 0 && c >= c_switch) {
        // the rest of the matrix is (modelled to be) on the device: finish in the
        // right-looking order (the remaining columns catch up on every earlier
        // panel with wide GEMMs, then the usual panel + trailing-update steps)
        const int64_t rem = h->n - col0;
        QRB_TRY(copy_upto(nchunks - 1));
        QRB_CUDA_TRY(cudaStreamWaitEvent(st, landed[nchunks - 1], 0));
        nonfinite_kernel<<<4 * 148, 256, 0, st>>>(h->A + col0 * h->lda, h->lda, h->m, rem, nf);
        QRB_CUDA_TRY(cudaGetLastError());
        g_launches += 1;
        QRB_TRY(apply_prev(static_cast<int>(col0 / nb), col0, rem));
        QRB_TRY(right_looking(h, col0, ws, st));
        break;
      }
      QRB_TRY(copy_upto(c));
      QRB_CUDA_TRY(cudaStreamWaitEvent(st, landed[c], 0));
      nonfinite_kernel<<<4 * 148, 256, 0, st>>>(h->A + col0 * h->lda, h->lda, h->m, nc, nf);
      QRB_CUDA_TRY(cudaGetLastError());
      g_launches += 1;
      // left-looking: every earlier panel applied to this chunk, in order
      QRB_TRY(apply_prev(static_cast<int>(col0 / nb), col0, nc));
      // then the chunk's own panels, right-looking inside the chunk (in pairs)
      for (int64_t j0 = col0; j0 < col0 + nc; j0 += nb) {
        const int64_t pw = std::min<int64_t>(nb, h->n - j0), mk = h->m - j0;
        const int k = static_cast<int>(j0 / nb);
        double* Tk = h->T + int64_t(k) * nb * nb;
        if (outer_panels_for(h->n) >= 2 && (k & 1) == 0 && j0 + w2 <= col0 + nc && mk >= w2) {
          double* T2 = nullptr;
          QRB_TRY(factor_panel_pair(A, j0, nb, Tk, Tk + int64_t(nb) * nb, h->tau, &T2, ws, st,
                                    h->T2 + int64_t(k / 2) * blk2));
          h->t2_valid[k / 2] = 1;
          const int64_t rest2 = col0 + nc - (j0 + w2);
          if (rest2 > 0)
            QRB_TRY(apply_qt(A.sub(j0, j0, mk, w2), T2, w2, A.sub(j0, j0 + w2, mk, rest2), ws, st));
          j0 += nb;
          continue;
        }
        QRB_TRY(factor_panel(A.sub(j0, j0, mk, pw), h->tau + j0, Tk, nb, ws, st));
        const int64_t rest = col0 + nc - (j0 + pw);
        if (rest > 0)
          QRB_TRY(apply_qt(A.sub(j0, j0, mk, pw), Tk, nb, A.sub(j0, j0 + pw, mk, rest), ws, st));
      }
      QRB_TRY(report_progress(h, col0 + nc, st));
    }
    QRB_CUDA_TRY(cudaEventRecord(h->ev1, st));
    QRB_CUDA_TRY(cudaEventSynchronize(h->ev1));
    QRB_CUDA_TRY(cudaGetLastError());
    int hflag = 0;
    QRB_CUDA_TRY(cudaMemcpy(&hflag, nf, sizeof(int), cudaMemcpyDeviceToHost));
    if (hflag) {
      set_last_error("factorize: input matrix has non-finite entries");
      return QRB_ENONFINITE;
    }
    return QRB_OK;
  };
  h->progress = nullptr;
  int status = QRB_OK;
  if (progress_host) {
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, progress_host, 0) != cudaSuccess) {
      cudaGetLastError();
      set_last_error("qrb_factorize_host_gated: progress must be page-locked, mapped host memory");
      status = QRB_EARG;
    }
    h->progress = static_cast<int64_t*>(dp);
  }
  if (status == QRB_OK) status = body();
  if (status == QRB_OK && h->progress) status = report_progress(h, h->n, st);
  h->progress = nullptr;
  if (cs) cudaStreamSynchronize(cs);  // no copy from src may outlive the call
  if (status == QRB_OK) {
    h->factored = true;
    session.finish(rep);
    if (rep) {
      const double m = static_cast<double>(h->m), n = static_cast<double>(h->n);
      rep->total_ms = elapsed(h->ev0, h->ev1);
      rep->h2d_ms = elapsed(c0ev, c1ev);
      rep->h2d_bytes = static_cast<int64_t>(8.0 * m * n);
      rep->flops = 2.0 * m * n * n - 2.0 * n * n * n / 3.0;
      rep->kernel_launches = g_launches.load() - launches0;
    }
  } else {
    cudaStreamSynchronize(st);
    cudaGetLastError();
  }
  for (auto& e : landed)
    if (e) cudaEventDestroy(e);
  if (c0ev) cudaEventDestroy(c0ev);
  if (c1ev) cudaEventDestroy(c1ev);
  if (cs) cudaStreamDestroy(cs);
  return status;
}

int qrb_factorize_host(qrb_handle* h, const double* src, int64_t ld, int64_t chunk_cols,
                       qrb_report* rep) {
  return factorize_host_impl(h, src, ld, chunk_cols, nullptr, 0.0, nullptr, rep);
}

int qrb_factorize_host_gated(qrb_handle* h, const double* src, int64_t ld, int64_t chunk_cols,
                             const int32_t* ready, double input_gbps, int64_t* progress,
                             qrb_report* rep) {
  if (!h || !ready || chunk_cols <= 0 || chunk_cols % h->nb != 0) {
    clear_report(rep);
    set_last_error("qrb_factorize_host_gated: need ready flags and chunk_cols a multiple of nb");
    return QRB_EARG;
  }
  return factorize_host_impl(h, src, ld, chunk_cols, ready, input_gbps, progress, rep);
}

int qrb_get_factors(qrb_handle* h, double* tau, double* T, int64_t ldt) {
  if (!h || (T && ldt < h->nb)) return QRB_EARG;
  DeviceGuard g(h->device);
  if (tau)
    QRB_CUDA_TRY(cudaMemcpyAsync(tau, h->tau, sizeof(double) * h->n, cudaMemcpyDefault,
                                 h->stream));
  if (T)
    QRB_CUDA_TRY(cudaMemcpy2DAsync(T, ldt * sizeof(double), h->T, h->nb * sizeof(double),
                                   h->nb * sizeof(double), int64_t(h->npanels) * h->nb,
                                   cudaMemcpyDefault, h->stream));
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return QRB_OK;
}

int qrb_get_pair_factors(qrb_handle* h, double* T2, int64_t ldt2) {
  const int64_t w2 = 2 * int64_t(h ? h->nb : 0);
  if (!h || !T2 || ldt2 < w2) {
    set_last_error("qrb_get_pair_factors: bad arguments");
    return QRB_EARG;
  }
  if (!h->factored) {
    set_last_error("qrb_get_pair_factors: handle is not factored");
    return QRB_ESTATE;
  }
  DeviceGuard g(h->device);
  WsUse use(device_workspace(), h->stream);
  QRB_TRY(ensure_t2(h, device_workspace()));
  const int npairs = h->npanels / 2;
  for (int p = 0; p < npairs; ++p) {
    double* dst = T2 + int64_t(p) * w2 * ldt2;
    if (pair_ok(h, 2 * p))
      QRB_CUDA_TRY(cudaMemcpy2DAsync(dst, ldt2 * sizeof(double), h->T2 + p * w2 * w2,
                                     w2 * sizeof(double), w2 * sizeof(double), w2,
                                     cudaMemcpyDefault, h->stream));
    else
      QRB_CUDA_TRY(cudaMemset2DAsync(dst, ldt2 * sizeof(double), 0, w2 * sizeof(double), w2,
                                     h->stream));
  }
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return QRB_OK;
}

int qrb_set_pair_factors(qrb_handle* h, const double* T2, int64_t ldt2) {
  const int64_t w2 = 2 * int64_t(h ? h->nb : 0);
  if (!h || !T2 || ldt2 < w2) {
    set_last_error("qrb_set_pair_factors: bad arguments");
    return QRB_EARG;
  }
  if (!h->factored) {
    set_last_error("qrb_set_pair_factors: set the factors (qrb_set_factors) first");
    return QRB_ESTATE;
  }
  DeviceGuard g(h->device);
  const int npairs = h->npanels / 2;
  if (npairs == 0) return QRB_OK;
  if (!h->T2 || static_cast<int>(h->t2_valid.size()) != npairs) QRB_TRY(t2_storage(h));
  for (int p = 0; p < npairs; ++p) {
    if (!pair_ok(h, 2 * p)) continue;
    QRB_CUDA_TRY(cudaMemcpy2DAsync(h->T2 + p * w2 * w2, w2 * sizeof(double),
                                   T2 + int64_t(p) * w2 * ldt2, ldt2 * sizeof(double),
                                   w2 * sizeof(double), w2, cudaMemcpyDefault, h->stream));
    h->t2_valid[p] = 1;
  }
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return QRB_OK;
}

int qrb_set_factors(qrb_handle* h, const double* tau, const double* T, int64_t ldt) {
  if (!h || !tau || !T || ldt < h->nb) return QRB_EARG;
  DeviceGuard g(h->device);
  QRB_CUDA_TRY(cudaMemcpyAsync(h->tau, tau, sizeof(double) * h->n, cudaMemcpyHostToDevice,
                               h->stream));
  QRB_CUDA_TRY(cudaMemcpy2DAsync(h->T, h->nb * sizeof(double), T, ldt * sizeof(double),
                                 h->nb * sizeof(double), int64_t(h->npanels) * h->nb,
                                 cudaMemcpyHostToDevice, h->stream));
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->factored = true;
  invalidate_derived(h);  // merged pair reflectors of earlier factors are stale
  return QRB_OK;
}

int qrb_get_rdiag(qrb_handle* h, double* diag) {
  if (!h || !diag) return QRB_EARG;
  DeviceGuard g(h->device);
  QRB_CUDA_TRY(cudaMemcpy2DAsync(diag, sizeof(double), h->A, (h->lda + 1) * sizeof(double),
                                 sizeof(double), h->n, cudaMemcpyDeviceToHost, h->stream));
  QRB_CUDA_TRY(cudaStreamSynchronize(h->stream));
  return QRB_OK;
}

int qrb_solve(qrb_handle* h, const double* B, int64_t ldb, int64_t nrhs, double* X, int64_t ldx,
              double* resid, int on_device, int64_t report_block, qrb_report* rep) {
  clear_report(rep);
  if (!h || !B || !X || nrhs < 0 || ldb < h->m || ldx < h->n) {
    set_last_error("qrb_solve: bad arguments");
    return QRB_EARG;
  }
  if (!h->factored) {
    set_last_error("qrb_solve: matrix not factorized");
    return QRB_ESTATE;
  }
  DeviceGuard g(h->device);
  if (nrhs == 0) return QRB_OK;
  const int64_t launches0 = g_launches.load();
  // singularity rule first (the reference raises before touching B's result)
  std::vector<double> diag(h->n);
  QRB_TRY(qrb_get_rdiag(h, diag.data()));
  const int64_t bad = singular_column(diag, report_block);
  if (bad >= 0) {
    set_last_error("singular upper-triangular factor: zero pivot at global column " +
                   std::to_string(bad));
    return static_cast<int>(1 + bad);
  }
  Workspace& ws = device_workspace();
  WsUse use(ws, h->stream);
  cudaStream_t st = h->stream;
  ProfSession session(h);
  const int64_t ldw = (h->m + 31) & ~int64_t(31);
  QRB_TRY(h->Bw.ensure(sizeof(double) * ldw * nrhs, st));
  double* Bw = h->Bw.d();
  QRB_CUDA_TRY(cudaEventRecord(h->ev0, st));
  QRB_CUDA_TRY(cudaMemcpy2DAsync(Bw, ldw * sizeof(double), B, ldb * sizeof(double),
                                 h->m * sizeof(double), nrhs,
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  QRB_CUDA_TRY(cudaEventRecord(h->ev1, st));
  QRB_TRY(ensure_rinv(h));
  // pair reflectors: those the factorization (or qrb_set_pair_factors) kept are
  // free; merging the rest pays only for wide right-hand-side batches -- with a
  // single-panel factorization (config 2) a 64-slice solve applies panels
  if (static_cast<int>(h->t2_valid.size()) != h->npanels / 2 ||
      static_cast<int>(h->t4_valid.size()) != h->npanels / 4)
    QRB_TRY(t2_storage(h));  // factors set without a factorization on this handle
  if (nrhs >= g_t4_min_rhs) QRB_TRY(ensure_t2(h, ws));
  // quad reflectors: the ones the factorization kept are free; merging the rest
  // (one m_k x 2nb x 2nb product each) pays only for wide right-hand-side
  // batches (config 2, 64 slices: 7.7 -> 9.3 ms with every quad merged per solve)
  if (nrhs >= g_t4_min_rhs) QRB_TRY(ensure_t4(h, ws));
  MatView A{h->A, h->m, h->n, h->lda};
  MatView Bv{Bw, h->m, nrhs, ldw};
  for (int k = 0; k < h->npanels;) {
    const int64_t j0 = int64_t(k) * h->nb;
    const int64_t pw = std::min<int64_t>(h->nb, h->n - j0);
    const int64_t mk = h->m - j0;
    if (quad_ok(h, k) && h->t4_valid[k / 4]) {  // four panels at once (K = 4nb)
      const int64_t w4 = 4 * int64_t(h->nb);
      QRB_TRY(apply_qt(A.sub(j0, j0, mk, w4), h->T4 + int64_t(k / 4) * w4 * w4, w4,
                       Bv.sub(j0, 0, mk, nrhs), ws, st));
      k += 4;
      continue;
    }
    if (pair_ok(h, k) && h->t2_valid[k / 2]) {  // two panels at once (K = 2nb)
      const int64_t w2 = 2 * int64_t(h->nb);
      QRB_TRY(apply_qt(A.sub(j0, j0, mk, w2), h->T2 + int64_t(k / 2) * w2 * w2, w2,
                       Bv.sub(j0, 0, mk, nrhs), ws, st));
      k += 2;
      continue;
    }
    QRB_TRY(apply_qt(A.sub(j0, j0, mk, pw), h->T + int64_t(k) * h->nb * h->nb, h->nb,
                     Bv.sub(j0, 0, mk, nrhs), ws, st));
    ++k;
  }
  if (resid) {
    QRB_TRY(h->resid.ensure(sizeof(double) * nrhs, st));
    QRB_TRY(column_sumsq(Bw, ldw, static_cast<int>(h->n), static_cast<int>(h->m),
                         static_cast<int>(nrhs), h->resid.d(), st));
    g_launches += 1;
  }
  if (outer_panels_solve() >= 2) {
    QRB_TRY(ensure_rinv2(h));
    QRB_TRY(trsm_upper_h(h, Bv.sub(0, 0, h->n, nrhs), st));
  } else {
    QRB_TRY(trsm_upper(A.sub(0, 0, h->n, h->n), h->Rinv, h->nb, Bv.sub(0, 0, h->n, nrhs), st));
  }
  QRB_CUDA_TRY(cudaEventRecord(h->ev2, st));
  QRB_CUDA_TRY(cudaMemcpy2DAsync(X, ldx * sizeof(double), Bw, ldw * sizeof(double),
                                 h->n * sizeof(double), nrhs,
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  std::vector<double> rs;
  if (resid) {
    rs.resize(nrhs);
    QRB_CUDA_TRY(cudaMemcpyAsync(rs.data(), h->resid.d(), sizeof(double) * nrhs,
                                 cudaMemcpyDeviceToHost, st));
  }
  QRB_CUDA_TRY(cudaStreamSynchronize(st));
  QRB_CUDA_TRY(cudaGetLastError());
  session.finish(rep);
  if (resid) {
    if (on_device) {
      for (auto& v : rs) v = std::sqrt(v);
      QRB_CUDA_TRY(cudaMemcpy(resid, rs.data(), sizeof(double) * nrhs, cudaMemcpyHostToDevice));
    } else {
      for (int64_t j = 0; j < nrhs; ++j) resid[j] = std::sqrt(rs[j]);
    }
  }
  if (rep) {
    cudaEvent_t e3;
    cudaEventCreate(&e3);
    cudaEventRecord(e3, st);
    cudaEventSynchronize(e3);
    rep->h2d_ms = on_device ? 0.0 : elapsed(h->ev0, h->ev1);
    rep->update_ms = elapsed(h->ev1, h->ev2);
    rep->d2h_ms = on_device ? 0.0 : elapsed(h->ev2, e3);
    rep->total_ms = elapsed(h->ev0, e3);
    cudaEventDestroy(e3);
    const double m = static_cast<double>(h->m), n = static_cast<double>(h->n);
    rep->flops = (4.0 * m * n - n * n) * static_cast<double>(nrhs);
    rep->kernel_launches = g_launches.load() - launches0;
    rep->h2d_bytes = on_device ? 0 : h->m * nrhs * 8;
    rep->d2h_bytes = on_device ? 0 : h->n * nrhs * 8;
  }
  return QRB_OK;
}

int qrb_op_panel(double* panel, int64_t ldp, int64_t m, int64_t w, double* tau, double* T,
                 int64_t ldt, void* stream) {
  if (!panel || !tau || !T || w < 1 || w > 128 || m < w || (ldp & 1) || ldt < w) {
    set_last_error("qrb_op_panel: bad arguments");
    return QRB_EARG;
  }
  MatView pv{panel, m, w, ldp};
  Workspace& ws = device_workspace();
  WsUse use(ws, static_cast<cudaStream_t>(stream));
  return factor_panel(pv, tau, T, ldt, ws, static_cast<cudaStream_t>(stream));
}

int qrb_op_apply_qt(const double* V, int64_t ldv, int64_t m, int64_t w, const double* T,
                    int64_t ldt, double* C, int64_t ldc, int64_t nc, void* stream) {
  if (!V || !T || !C || w < 1 || m < w || (ldv & 1) || (ldc & 1) || (ldt & 1) || ldt < w) {
    set_last_error("qrb_op_apply_qt: bad arguments (leading dimensions must be even)");
    return QRB_EARG;
  }
  MatView Vv{const_cast<double*>(V), m, w, ldv};
  MatView Cv{C, m, nc, ldc};
  Workspace& ws = device_workspace();
  WsUse use(ws, static_cast<cudaStream_t>(stream));
  return apply_qt(Vv, T, ldt, Cv, ws, static_cast<cudaStream_t>(stream));
}

int qrb_op_gemm_nn_sub(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                       int64_t ldc, int64_t m, int64_t n, int64_t k, void* stream) {
  if (!A || !B || !C || m < 0 || n < 0 || k < 0 || (lda & 1) || (ldb & 1) || (ldc & 1)) {
    set_last_error("qrb_op_gemm_nn_sub: bad arguments (leading dimensions must be even)");
    return QRB_EARG;
  }
  if (m == 0 || n == 0 || k == 0) return QRB_OK;
  MatView Av{const_cast<double*>(A), m, k, lda};
  MatView Bv{const_cast<double*>(B), k, n, ldb};
  g_launches += 1;
  return gemm_nn(Av, Bv, C, ldc, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                 GEMM_EPI_SUB, 0, static_cast<cudaStream_t>(stream));
}

int qrb_op_gemm_tn(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                   int64_t ldc, int64_t m, int64_t n, int64_t k, int splits, int mask_a,
                   int mask_b, void* stream) {
  if (!A || !B || !C || m < 0 || n < 0 || k < 0 || splits < 1 || (lda & 1) || (ldb & 1)) {
    set_last_error("qrb_op_gemm_tn: bad arguments (leading dimensions must be even)");
    return QRB_EARG;
  }
  if (m == 0 || n == 0) return QRB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  MatView Av{const_cast<double*>(A), k, m, lda};
  MatView Bv{const_cast<double*>(B), k, n, ldb};
  if (splits == 1) {
    g_launches += 1;
    return gemm_tn(Av, Bv, C, ldc, 0, static_cast<int>(m), static_cast<int>(n),
                   static_cast<int>(k), 1, mask_a, mask_b, st);
  }
  Workspace& ws = device_workspace();
  WsUse use(ws, st);
  const int64_t per = ldc * n;
  int used = 0;
  QRB_TRY(ws.Wparts.ensure(sizeof(double) * per * splits, st));
  QRB_TRY(gemm_tn_split(Av, Bv, ws.Wparts.d(), ldc, per, static_cast<int>(m), static_cast<int>(n),
                        static_cast<int>(k), splits, mask_a, mask_b, st, &used));
  QRB_TRY(reduce_splits(ws.Wparts.d(), per, used, static_cast<int>(m), static_cast<int>(n), ldc, C,
                        ldc, st));
  g_launches += 2;
  return QRB_OK;
}

int qrb_op_trsm_upper(const double* R, int64_t ldr, int64_t n, int nb, double* B, int64_t ldb,
                      int64_t nrhs, void* stream) {
  if (!R || !B || n < 0 || nrhs < 0 || nb < 16 || nb > 128 || (nb % 16) || (ldr & 1) ||
      (ldb & 1)) {
    set_last_error("qrb_op_trsm_upper: bad arguments");
    return QRB_EARG;
  }
  if (n == 0 || nrhs == 0) return QRB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Workspace& ws = device_workspace();
  WsUse use(ws, st);
  const int nblk = static_cast<int>((n + nb - 1) / nb);
  QRB_TRY(ws.Wparts.ensure(sizeof(double) * nb * nb * nblk, st));
  QRB_TRY(trtri_blocks(R, ldr, static_cast<int>(n), nb, ws.Wparts.d(), st));
  g_launches += 1;
  MatView Rv{const_cast<double*>(R), n, n, ldr};
  MatView Bv{B, n, nrhs, ldb};
  return trsm_upper(Rv, ws.Wparts.d(), nb, Bv, st);
}

int qrb_siddon_densify(const double* ends, int64_t n_rays, int64_t row0, int image_pixels,
                       double* A, int64_t lda, int nb, int world, int rank, int64_t n_local,
                       void* stream) {
  if (!ends || !A || n_rays < 0 || image_pixels < 1 || lda < 1 || world < 1 || rank < 0 ||
      rank >= world || (world > 1 && nb < 1)) {
    set_last_error("qrb_siddon_densify: bad arguments");
    return QRB_EARG;
  }
  g_launches += 1;
  return siddon_densify(ends, n_rays, image_pixels, A, lda, row0, nb, world, rank, n_local,
                        static_cast<cudaStream_t>(stream));
}

int qrb_op_panel_block(double* A, int64_t lda, int64_t m, int64_t w, int nb, double* tau,
                       double* T, double* T2, int64_t ldt2, void* stream, int side) {
  if (!A || !tau || !T || !T2 || nb < 2 || nb > 128 || (nb & 1) || w < 1 || w > 2 * nb ||
      m < w || (lda & 1) || (ldt2 & 1) || ldt2 < w) {
    set_last_error("qrb_op_panel_block: bad arguments");
    return QRB_EARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Workspace& ws = side ? side_workspace() : device_workspace();
  WsUse use(ws, st);
  const MatView Av{A, m, w, lda};
  const int64_t wa = std::min<int64_t>(w, nb), wb = w - wa;
  QRB_TRY(factor_panel(Av.sub(0, 0, m, wa), tau, T, nb, ws, st));
  if (wb == 0) {
    QRB_CUDA_TRY(cudaMemset2DAsync(T2, sizeof(double) * ldt2, 0, sizeof(double) * w, w, st));
    QRB_CUDA_TRY(cudaMemcpy2DAsync(T2, sizeof(double) * ldt2, T, sizeof(double) * nb,
                                   sizeof(double) * w, w, cudaMemcpyDeviceToDevice, st));
    return QRB_OK;
  }
  double* Tb = T + int64_t(nb) * nb;
  QRB_TRY(apply_qt(Av.sub(0, 0, m, nb), T, nb, Av.sub(0, nb, m, wb), ws, st));
  QRB_TRY(factor_panel(Av.sub(nb, nb, m - nb, wb), tau + nb, Tb, nb, ws, st));
  QRB_TRY(ws.T2.ensure(sizeof(double) * 2 * int64_t(nb) * nb, st));
  return merge_pair_t(Av, 0, nb, T, Tb, T2, ldt2, ws.T2.d(), ws, st, static_cast<int>(wb));
}

int qrb_op_apply_qt_begin(const double* V, int64_t ldv, int64_t m, int64_t w, const double* T,
                          int64_t ldt, const double* C, int64_t ldc, int64_t nc, void* stream) {
  if (!V || !T || !C || w < 1 || m < w || nc < 0 || (ldv & 1) || (ldc & 1) || (ldt & 1) ||
      ldt < w) {
    set_last_error("qrb_op_apply_qt_begin: bad arguments (leading dimensions must be even)");
    return QRB_EARG;
  }
  if (nc == 0) return QRB_OK;
  Workspace& ws = device_workspace();
  WsUse use(ws, static_cast<cudaStream_t>(stream));
  QRB_TRY(apply_qt_w2(MatView{const_cast<double*>(V), m, w, ldv}, T, ldt,
                      MatView{const_cast<double*>(C), m, nc, ldc}, ws,
                      static_cast<cudaStream_t>(stream)));
  t_begin = BeginRecord{ws.w2_gen, V, m, w, stream};
  return QRB_OK;
}

int qrb_op_apply_qt_cols(const double* V, int64_t ldv, int64_t m, int64_t w, double* C,
                         int64_t ldc, int64_t c_from, int64_t ncols, void* stream) {
  if (!V || !C || w < 1 || m < w || c_from < 0 || ncols < 0 || (ldv & 1) || (ldc & 1)) {
    set_last_error("qrb_op_apply_qt_cols: bad arguments");
    return QRB_EARG;
  }
  Workspace& ws = device_workspace();
  WsUse use(ws, static_cast<cudaStream_t>(stream));
  if (c_from + ncols > ws.w2_cols || w != ws.w2_w) {
    set_last_error("qrb_op_apply_qt_cols: columns or width beyond the last qrb_op_apply_qt_begin");
    return QRB_EARG;
  }
  // the W2 in the (per-device) workspace must still be the one this thread's
  // last _begin formed, for the same reflector block and stream: any other
  // W2-forming call in between (a solve, qrb_op_apply_qt, another thread)
  // replaced it
  if (t_begin.gen != ws.w2_gen || t_begin.V != V || t_begin.m != m || t_begin.w != w ||
      t_begin.stream != stream) {
    set_last_error("qrb_op_apply_qt_cols: the workspace W2 is not the one the last "
                   "qrb_op_apply_qt_begin formed (another W2-forming call ran in between, or "
                   "a different V / m / stream)");
    return QRB_ESTATE;
  }
  return apply_qt_nn(MatView{const_cast<double*>(V), m, w, ldv}, MatView{C, m, c_from + ncols, ldc},
                     c_from, ncols, ws, static_cast<cudaStream_t>(stream),
                     gemm_grid_cap() > 0 ? QRB_K_GEMM_NN_CAP : QRB_K_GEMM_NN);
}

int qrb_op_apply_qt_td(const double* D, int64_t ldd, int64_t b, int64_t w, const double* S,
                       int64_t lds, double* F, int64_t ldf, double* G, int64_t ldg, int64_t nc,
                       void* stream) {
  if (!D || !S || !F || !G || b < 1 || w < 1 || w > 128 || nc < 0 || (ldd & 1) || (lds & 1) ||
      (ldf & 1) || (ldg & 1)) {
    set_last_error("qrb_op_apply_qt_td: bad arguments (leading dimensions must be even)");
    return QRB_EARG;
  }
  if (nc == 0) return QRB_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Workspace& ws = device_workspace();
  WsUse use(ws, st);
  const int64_t ldw = even(w);
  QRB_TRY(ws.W.ensure(sizeof(double) * ldw * nc, st));
  QRB_TRY(ws.W2.ensure(sizeof(double) * ldw * nc, st));
  // reference apply_left_qt_td (kernels.py:385-405): per inner panel j0 of width pw
  //   W = F[j0:j0+pw] + Vd^T G ;  Z = S_p^T W ;  F[j0:j0+pw] -= Z ;  G -= Vd Z
  for (int64_t j0 = 0; j0 < b; j0 += w) {
    const int pw = static_cast<int>(std::min<int64_t>(w, b - j0));
    MatView Vd{const_cast<double*>(D) + j0 * ldd, b, pw, ldd};
    MatView Gv{G, b, nc, ldg};
    QRB_TRY(gemm_tn(Vd, Gv, ws.W.d(), ldw, 0, pw, static_cast<int>(nc), static_cast<int>(b), 1,
                    0, 0, st));
    QRB_TRY(axpy_block(1.0, F + j0, ldf, ws.W.d(), ldw, pw, nc, st));
    MatView Tv{const_cast<double*>(S) + j0, pw, pw, lds};
    MatView Wv{ws.W.d(), pw, nc, ldw};
    QRB_TRY(gemm_tn(Tv, Wv, ws.W2.d(), ldw, 0, pw, static_cast<int>(nc), pw, 1, 0, 0, st));
    QRB_TRY(axpy_block(-1.0, ws.W2.d(), ldw, F + j0, ldf, pw, nc, st));
    MatView W2v{ws.W2.d(), pw, nc, ldw};
    QRB_TRY(gemm_nn(Vd, W2v, G, ldg, static_cast<int>(b), static_cast<int>(nc), pw, GEMM_EPI_SUB,
                    0, st));
    g_launches += 5;
  }
  return QRB_OK;
}

int qrb_copy_2d(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                int64_t cols, int kind, void* stream) {
  if (!dst || !src || rows < 0 || cols < 0 || ldd < rows || lds < rows || kind < 0 || kind > 3) {
    set_last_error("qrb_copy_2d: bad arguments");
    return QRB_EARG;
  }
  if (rows == 0 || cols == 0) return QRB_OK;
  static const cudaMemcpyKind kinds[4] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost,
                                          cudaMemcpyDeviceToDevice, cudaMemcpyHostToHost};
  QRB_CUDA_TRY(cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double),
                                 rows * sizeof(double), cols, kinds[kind],
                                 static_cast<cudaStream_t>(stream)));
  return QRB_OK;
}

int qrb_release_workspace(void) {
  cudaDeviceSynchronize();
  device_workspace().release();
  side_workspace().release();
  return QRB_OK;
}

int64_t qrb_launch_count(void) { return g_launches.load(); }

int qrb_set_tuning(const char* key, int64_t value) {
  const std::string k = key ? key : "";
  ++g_graph_epoch;  // captured factorization graphs bake the knobs in
  if (k == "t4_min_rhs" && value >= 0) {
    g_t4_min_rhs = value;
    return QRB_OK;
  }
  if (k == "graph_max_cols" && value >= 0) {
    g_graph_max_cols = value;
    return QRB_OK;
  }
  if (k == "panel_algo" && value >= 0 && value <= 2) {
    g_panel_algo = static_cast<int>(value);
    return QRB_OK;
  }
  if (k == "cholqr_min_rows" && value >= 0) {
    g_cholqr_min_rows = value;
    return QRB_OK;
  }
  if (k == "outer_panels" && (value == 0 || value == 1 || value == 2 || value == 4)) {
    g_outer_panels = static_cast<int>(value);
    return QRB_OK;
  }
  if (k == "tail_singles" && (value == 0 || value == 1)) {
    g_tail_singles = static_cast<int>(value);
    return QRB_OK;
  }
  if (k == "pairs_min_cols" && value >= 0) {
    g_pairs_min_cols = value;
    return QRB_OK;
  }
  if (k == "nn_dynamic" && (value == 0 || value == 1)) {
    gemm_set_nn_dynamic(value == 1);
    return QRB_OK;
  }
  if (k == "outer4_min_cols" && value >= 0) {
    g_outer4_min_cols = value;
    return QRB_OK;
  }
  if (k == "tn_tail" && (value == 0 || value == 1)) {
    g_tn_tail = static_cast<int>(value);
    return QRB_OK;
  }
  if (k == "grid_cap" && value >= 0) {  // this host thread's GEMM grid cap (0 = none)
    gemm_set_grid_cap(static_cast<int>(value));
    return QRB_OK;
  }
  if (k == "lookahead" && value >= 0 && value <= 3) {
    g_lookahead = static_cast<int>(value);
    return QRB_OK;
  }
  if (k == "la_sms" && value >= 1 && value <= 100) {
    g_la_sms = static_cast<int>(value);
    return QRB_OK;
  }
  if (k == "la_lat_us" && value >= 0) {
    g_la_lat_us = value;
    return QRB_OK;
  }
  if (k == "early_sms" && value >= 0 && value <= 64) {
    g_early_sms = value;
    return QRB_OK;
  }
  if (k == "early_singles" && value >= 0 && value <= 1) {
    g_early_singles = static_cast<int>(value);
    return QRB_OK;
  }
  if (k == "la_sms_tall" && value >= 0 && value <= 100) {
    g_la_sms_tall = value;
    return QRB_OK;
  }
  if (k == "la_tall_rows" && value >= 0) {
    g_la_tall_rows = value;
    return QRB_OK;
  }
  if (k == "la_sms_max" && value >= 0 && value <= 120) {
    g_la_sms_max = value;
    return QRB_OK;
  }
  if (k == "la_margin_pct" && value >= 0 && value <= 1000) {
    g_la_margin_pct = value;
    return QRB_OK;
  }
  if (k == "sf_diag" && value >= 0 && value <= 63) {
    smallfact_set_diag(static_cast<int>(value));
    return QRB_OK;
  }
  if (k == "few_tiles_bn32" && value >= 0 && value <= 2) {
    gemm_set_few_tiles_bn32(static_cast<int>(value));
    return QRB_OK;
  }
  if (k == "gram_min_rows" && value >= 16 && value <= 4096) {
    gemm_set_few_tiles_min_rows(static_cast<int>(value));
    return QRB_OK;
  }
  set_last_error("qrb_set_tuning: unknown key or bad value: " + k);
  return QRB_ERR_ARG;
}

int qrb_get_tuning(const char* key, int64_t* value) {
  const std::string k = key ? key : "";
  if (!value) {
    set_last_error("qrb_get_tuning: null value");
    return QRB_ERR_ARG;
  }
  if (k == "panel_algo") *value = g_panel_algo;
  else if (k == "cholqr_min_rows") *value = g_cholqr_min_rows;
  else if (k == "nn_dynamic") *value = gemm_nn_dynamic() ? 1 : 0;
  else if (k == "outer_panels") *value = g_outer_panels;
  else if (k == "pairs_min_cols") *value = g_pairs_min_cols;
  else if (k == "tail_singles") *value = g_tail_singles;
  else if (k == "lookahead") *value = g_lookahead;
  else if (k == "grid_cap") *value = gemm_grid_cap();
  else if (k == "tn_tail") *value = g_tn_tail;
  else if (k == "outer4_min_cols") *value = g_outer4_min_cols;
  else if (k == "sm_count") *value = gemm_sm_count();
  else if (k == "la_sms") *value = g_la_sms;
  else if (k == "la_lat_us") *value = g_la_lat_us;
  else if (k == "la_margin_pct") *value = g_la_margin_pct;
  else if (k == "la_sms_max") *value = g_la_sms_max;
  else if (k == "la_sms_tall") *value = g_la_sms_tall;
  else if (k == "early_singles") *value = g_early_singles;
  else if (k == "early_sms") *value = g_early_sms;
  else if (k == "la_tall_rows") *value = g_la_tall_rows;
  else if (k == "gram_min_rows") *value = gemm_few_tiles_min_rows();
  else if (k == "few_tiles_bn32") *value = gemm_few_tiles_bn32();
  else if (k == "sf_diag") *value = smallfact_diag();
  else if (k == "la_steps") *value = g_la_steps.load();
  else if (k == "cholqr_panels") *value = g_cholqr_panels.load();
  else if (k == "cholqr_fallbacks") *value = cholqr_fallback_count();
  else if (k == "graph_max_cols") *value = g_graph_max_cols;
  else if (k == "t4_min_rhs") *value = g_t4_min_rhs;
  else if (k == "graph_captures") *value = g_graph_captures.load();
  else if (k == "graph_replays") *value = g_graph_replays.load();
  else {
    set_last_error("qrb_get_tuning: unknown key: " + k);
    return QRB_ERR_ARG;
  }
  return QRB_OK;
}

}  // extern "C"
