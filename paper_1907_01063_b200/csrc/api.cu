// api.cu -- the C ABI of libstancl (include/stan_cl.h) and the host-side
// schedulers of the blocked forward and adjoint
// algorithms.
//
// Layout: every call works on an N x N row-major working matrix, N = n rounded
// up to NB = 128.  When n is already a multiple of NB and the buffers are
// 16-byte aligned, the output buffer itself is the working matrix (no extra
// HBM traffic).  Otherwise the inputs are copied into a padded workspace:
//   forward  A_pad = [[A, 0], [0, I]]      -> L_pad = [[L, 0], [0, I]]
//   adjoint  L_pad = [[L, 0], [0, I]], L_bar_pad = [[L_bar, 0], [0, 0]]
//                                          -> A_bar_pad = [[A_bar, 0], [0, 0]]
// (the padded problems decouple), so no kernel needs ragged-edge
// code.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <numeric>
#include <tuple>
#include <mutex>
#include <thread>
#include <chrono>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/stan_cl.h"
#include "common.cuh"
#include "kernels.h"

using namespace stancl;

namespace {

struct State {
  cudaStream_t stream = nullptr;  // nullptr = legacy default stream
  cudaStream_t side = nullptr;    // library-owned high-priority stream (panel lookahead)
  cudaStream_t aux = nullptr;     // library-owned stream: the lookahead rows below the diagonal tile
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the *_host entry points
  std::vector<cudaEvent_t> events;
  std::vector<cudaEvent_t> xev;  // per-block events of the streamed host transfers
  // cached working buffers: 0, 1 = N x N matrices of the padded / host paths;
  // 2, 3 = K/L and L_bar/A_bar of the GP gradient; 4 = O(n) GP / solve scratch
  void* mat[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaStream_t cap = nullptr;         // capture stream for the CUDA-graph cache
  size_t mat_cap[5] = {0, 0, 0, 0, 0};
  int nb = 0;      // forward outer block: 0 = auto, 128 or 256
  int adj_nb = 0;  // adjoint block: 0 = auto, 128 or 256
  void* ws = nullptr;  // library-owned persistent workspace
  size_t ws_cap = 0;
  int* h_status = nullptr;  // pinned host word for the synchronous calls
  char last_err[256] = {0};
  // caller-provided workspace (stan_cl_set_workspace): every device buffer the
  // library needs is carved from it, per call, by a bump pointer
  char* user_ws = nullptr;
  size_t user_cap = 0;
  size_t user_next = 0;  // next free byte of this call
  int depth = 0;         // nesting of public calls (the GP gradient calls the others)
  // bumped whenever a workspace buffer moves: cached CUDA graphs captured with an
  // older generation point at freed memory and are re-captured
  unsigned long long gen = 1;
};
State g;

int cuda_fail(cudaError_t e, const char* where) {
  snprintf(g.last_err, sizeof(g.last_err), "%s: %s", where, cudaGetErrorString(e));
  return STAN_CL_ECUDA;
}

#define CK(x)                                              \
  do {                                                     \
    cudaError_t e_ = (x);                                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x);       \
  } while (0)

inline int64_t round_up(int64_t n, int64_t b) { return (n + b - 1) / b * b; }

// no programmatic dependent launch inside the host-streamed entry points
// (kernels.h pdl_allow: measured 185 -> 202 ms per e2e step with it on)
struct PdlOff {
  PdlOff() { pdl_allow(false); }
  ~PdlOff() { pdl_allow(true); }
};
inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

bool ranges_overlap(const void* a, const void* b, size_t bytes) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + bytes && y < x + bytes;
}
// [a, a + abytes) and [b, b + bbytes) intersect
bool ranges_overlap2(const void* a, size_t abytes, const void* b, size_t bbytes) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return x < y + bbytes && y < x + abytes;
}

// ---------------------------------------------------------------- workspace
constexpr size_t kAlign = 256;
inline size_t al(size_t b) { return (b + kAlign - 1) / kAlign * kAlign; }

struct AdjPlan {
  int64_t N;    // padded order (multiple of B)
  int64_t B;    // adjoint block size: 128 or 256
  size_t dinv, part, tmp, ctmp, hscr, cs, total;
};
constexpr int kNumSms = 148;  // B200 (the persistent GEMMs size their grids from the device)

// split-K factor for W = C_bar^T L[k:N, 0:k] (M = B rows; persistent TMA GEMM,
// 128 x 64 output tiles, 32-deep slabs): minimise rounds-of-148 x per-item K
// (+ a fixed per-item cost) plus the reduction's extra reads
void splitk_choice(int64_t m, int64_t k, int64_t B, int* splits_out, int* kps_out, int nsm = kNumSms) {
  const int ntiles = (int)((B / 128) * (k / 64));
  const int kmax = (int)(m / 32);
  double best = 1e300;
  int bs = 1;
  for (int s = 1; s <= 64 && s <= kmax; ++s) {
    const int64_t kps = round_up((m + s - 1) / s, 32);
    const int eff_s = (int)((m + kps - 1) / kps);
    const int64_t items = (int64_t)ntiles * eff_s;
    const int64_t rounds = (items + nsm - 1) / nsm;
    const double t = (double)rounds * (double)(kps + 96) + 3.0 * eff_s * 64 * (double)k * (B / 128) / (nsm * 64.0);
    if (t < best - 1e-9) {
      best = t;
      bs = s;
    }
  }
  const int64_t kps = round_up((m + bs - 1) / bs, 32);
  *kps_out = (int)kps;
  *splits_out = (int)((m + kps - 1) / kps);
}

// adjoint block: 256 (fewer, longer-K steps; measured faster at every size
// from n = 1024: 0.47 vs 0.61 ms, 2048: 1.00 vs 1.25 ms, 8192: 14.7 vs 16.0 ms,
// tools/nb_sweep.py), 128 for the smallest problems (less padding)
int64_t adj_block(int64_t n) {
  if (g.adj_nb) return g.adj_nb;
  return n >= 768 ? 2 * NB : NB;
}

// SMs given to the pipelined adjoint's dependency chain at step k (the rest
// goes to the previous step's bulk update running beside it): proportional to
// the two sides' DMMA work, at least 64 (the fused diagonal step's 64 CTAs
// meet at grid barriers and must all be resident), at most 140 while the
// bulk side has work
int adj_chain_sms(int64_t N, int64_t B, int64_t k) {
  const int64_t m = N - k;
  // DMMA work (FMAs) of the chain of this step (C_bar D^-1, split-K, lookahead
  // column) and of the previous step's bulk update beside it (rows j_prev.. =
  // k.. of B + m - B rows, columns [0, k - B))
  const double wc = (double)m * k * B + (double)m * B * B + (double)(B + m) * B * B;
  const double wm = (double)std::max<int64_t>(m, 0) * (double)std::max<int64_t>(k - B, 0) * B;
  if (wm <= 0) return kNumSms;
  static const int fixed = [] {
    const char* e = getenv("STAN_CL_PIPE_CHAIN_SMS");  // tuning aid: fixed chain share
    return e ? atoi(e) : 0;
  }();
  if (fixed > 0) return std::min(fixed, kNumSms);
  // the chain also carries latency-bound kernels (R0 + reduce, write-back,
  // fused diagonal step: ~L0 us per step whatever its SM share): balance
  //   wc / (R rho) + L0  against  wm / ((148 - R) rho),  rho = FMAs per us per SM
  static const double L0 = [] {
    const char* e = getenv("STAN_CL_PIPE_L0_US");
    return e ? atof(e) : 60.0;
  }();
  const double rho = 33e12 / 2.0 / kNumSms / 1e6;
  int best = 64;
  double bt = 1e300;
  for (int r = 64; r <= kNumSms - 8; ++r) {
    const double t = std::max(wc / (r * rho) + L0, wm / ((kNumSms - r) * rho));
    if (t < bt) {
      bt = t;
      best = r;
    }
  }
  return best;
}

AdjPlan adj_plan(int64_t n) {
  AdjPlan p{};
  p.B = adj_block(n);
  p.N = round_up(n, p.B);
  p.dinv = al((size_t)p.N * p.B * sizeof(double));  // N/B blocks of B x B
  size_t part = 0;
  for (int64_t k = p.N; k > 0; k -= p.B) {
    const int64_t m = p.N - k;
    if (m == 0) continue;
    int s, kps;
    splitk_choice(m, k, p.B, &s, &kps);
    const size_t b = (size_t)s * p.B * (size_t)k * sizeof(double);
    if (b > part) part = b;
  }
  p.part = al(part);
  p.tmp = al(4 * (size_t)p.B * p.B * sizeof(double));
  p.ctmp = al((size_t)p.N * p.B * sizeof(double));
  // (formerly the copy stream's D^-1 scratch; the streamed host path now
  // computes D^-1 in stream order with the sweep, from the Pbuf region)
  p.hscr = 0;
  // pipelined sweep: three rotating [S; C_bar D^-1] buffers of (B + N) x B
  p.cs = 3 * al((size_t)(p.B + p.N) * p.B * sizeof(double));
  p.total = al(sizeof(int) * 64) + p.dinv + p.part + p.tmp + p.ctmp + p.hscr + p.cs;
  return p;
}

constexpr size_t kHdr = 256;  // int header: status word + grid-barrier counters

int user_enomem(size_t need) {
  snprintf(g.last_err, sizeof(g.last_err), "caller workspace too small: need >= %zu bytes, have %zu", need,
           g.user_cap);
  return STAN_CL_ENOMEM;
}

// Caller workspace: [header + shared workspace of this call][matrix slots ...].
// The shared workspace sits at offset 0 and may only grow before the first
// slot of the call is carved (every entry point sizes it first).
int user_ws(size_t bytes) {
  bytes = al(std::max(bytes, kHdr));
  if (bytes <= g.ws_cap) return STAN_CL_OK;
  if (g.user_next > g.ws_cap) {
    snprintf(g.last_err, sizeof(g.last_err), "internal: workspace grown after a slot was carved");
    return STAN_CL_EINVAL;
  }
  if (bytes > g.user_cap) return user_enomem(bytes);
  g.ws_cap = bytes;
  g.user_next = bytes;
  return STAN_CL_OK;
}

int ensure_ws(size_t bytes) {
  if (g.user_ws) return user_ws(bytes);
  if (g.ws_cap >= bytes && g.ws) return STAN_CL_OK;
  ++g.gen;
  if (g.ws) {
    CK(cudaStreamSynchronize(g.stream));
    CK(cudaFree(g.ws));
    g.ws = nullptr;
    g.ws_cap = 0;
  }
  cudaError_t e = cudaMalloc(&g.ws, bytes);
  if (e != cudaSuccess) {
    g.ws = nullptr;
    snprintf(g.last_err, sizeof(g.last_err), "workspace cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    cudaGetLastError();
    return STAN_CL_ENOMEM;
  }
  g.ws_cap = bytes;
  // the int header (status word, grid-barrier counters of the fused diagonal
  // step) starts at zero; the kernels leave the counters at zero
  CK(cudaMemset(g.ws, 0, sizeof(int) * 64));
  return STAN_CL_OK;
}

int ensure_host_status() {
  if (!g.h_status) CK(cudaMallocHost(&g.h_status, sizeof(int)));
  return STAN_CL_OK;
}

// cached working matrix `slot` of at least `bytes` (grown with a sync, kept across
// calls: re-mapping GBs of device memory per call costs 10-1000 ms)
int ensure_mat(int slot, size_t bytes, double** p) {
  if (g.user_ws) {
    if (g.mat[slot] && g.mat_cap[slot] >= bytes) {
      *p = (double*)g.mat[slot];
      return STAN_CL_OK;
    }
    if (g.user_next < g.ws_cap) g.user_next = g.ws_cap;
    const size_t need = g.user_next + al(bytes);
    if (need > g.user_cap) return user_enomem(need);
    g.mat[slot] = g.user_ws + g.user_next;
    g.mat_cap[slot] = al(bytes);
    g.user_next = need;
    *p = (double*)g.mat[slot];
    return STAN_CL_OK;
  }
  if (g.mat_cap[slot] < bytes || !g.mat[slot]) {
    ++g.gen;
    if (g.mat[slot]) {
      CK(cudaDeviceSynchronize());
      CK(cudaFree(g.mat[slot]));
      g.mat[slot] = nullptr;
      g.mat_cap[slot] = 0;
    }
    cudaError_t e = cudaMalloc(&g.mat[slot], bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      g.mat[slot] = nullptr;
      snprintf(g.last_err, sizeof(g.last_err), "matrix workspace cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
      return STAN_CL_ENOMEM;
    }
    g.mat_cap[slot] = bytes;
  }
  *p = (double*)g.mat[slot];
  return STAN_CL_OK;
}


// Scope of one public call: with a caller workspace, the outermost call lays
// its buffers out afresh from the start of that workspace.
// Also an NVTX range named after the entry point (visible in nsys / ncu
// --nvtx; header-only NVTX v3, a no-op unless a tool is attached).
struct CallScope {
  explicit CallScope(const char* name) {
    nvtxRangePushA(name);
    if (g.depth++ == 0 && g.user_ws) {
      g.ws = g.user_ws;
      g.ws_cap = kHdr;
      g.user_next = kHdr;
      for (int i = 0; i < 5; ++i) {
        g.mat[i] = nullptr;
        g.mat_cap[i] = 0;
      }
    }
  }
  ~CallScope() {
    --g.depth;
    nvtxRangePop();
  }
};

// ------------------------------------------------------------------ forward
int ensure_side(size_t nevents) {
  if (!g.side) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&g.side, cudaStreamNonBlocking, hi));
  }
  while (g.events.size() < nevents) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g.events.push_back(e);
  }
  return STAN_CL_OK;
}

int ensure_copy(size_t nevents) {
  if (!g.h2d) CK(cudaStreamCreateWithFlags(&g.h2d, cudaStreamNonBlocking));
  if (!g.d2h) CK(cudaStreamCreateWithFlags(&g.d2h, cudaStreamNonBlocking));
  while (g.xev.size() < nevents) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g.xev.push_back(e);
  }
  return STAN_CL_OK;
}

// host destination of a streamed result: the leading n x n block (row-major,
// leading dimension n) receives the lower triangle (+0.0 above the diagonal
// inside the 128 x 128 diagonal tiles; the rest of the strict upper untouched)
struct HostOut {
  double* host;
  int64_t n;
};

// rows [r0, r1) x columns [c0, c1) of W (ld) -> host (ld n), on stream st
int copy_rect_d2h(const HostOut& o, const double* W, int64_t ld, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                  cudaStream_t st) {
  r1 = std::min(r1, o.n);
  c1 = std::min(c1, o.n);
  if (r1 <= r0 || c1 <= c0) return STAN_CL_OK;
  CK(cudaMemcpy2DAsync(o.host + r0 * o.n + c0, o.n * sizeof(double), W + r0 * ld + c0, ld * sizeof(double),
                       (c1 - c0) * sizeof(double), r1 - r0, cudaMemcpyDeviceToHost, st));
  return STAN_CL_OK;
}

// forward outer block (stan_cl_set_block_size(0) = auto): 256 (two-level: the
// trailing update runs with K = 256) from n = 6144 on, when it divides n or n is
// padded anyway; 128 below, where the panel chain dominates and a 128-wide step
// is shorter (measured: n = 4096 2.85 vs 2.96 ms, 2048 1.28 vs 1.33 ms; 8192
// 9.35 ms with 256 vs 9.79 ms with 128; tools/nb_sweep.py)
int64_t fwd_outer_block(int64_t n) {
  if (n >= 6144) return (n % (2 * NB) == 0 || n % NB != 0) ? 2 * NB : NB;
  return NB;
}

// The factored panel of outer block [c0, c0+OB): L11 = chol(A11) and
// L21 = A21 L11^-T.  OB = 128: one POTRF tile + one TRSM.
// OB = 256 (two-level blocking): two 128 sub-steps with the second half of the
// panel updated in between (GEMM, K = 128), so the trailing update outside
// the panel runs with K = 256.
int panel(double* W, int64_t ld, int64_t c0, int64_t N, int64_t OB, int* status, cudaStream_t st) {
  CK(potrf_tile(W, ld, c0, status, st));
  if (c0 + NB < N) CK(trsm_panel(W, ld, c0, c0 + NB, N, status, st));
  if (OB == 2 * NB) {
    const int64_t h = c0 + NB;
    const double* L21 = W + h * ld + c0;
    CK(gemm_full(true, true, (int)(N - h), NB, NB, -1.0, 1, L21, ld, L21, ld, W + h * ld + h, ld, status, st,
                 /*lower_only=*/1, PROF_LOOKAHEAD, /*allow_persistent=*/false));
    CK(potrf_tile(W, ld, h, status, st));
    if (h + NB < N) CK(trsm_panel(W, ld, h, h + NB, N, status, st));
  }
  return STAN_CL_OK;
}

// Right-looking blocked Cholesky on the N x N working matrix W (lower part),
// PAPER.md:264-285 with a fixed outer block OB (N % OB == 0), and one step of
// lookahead: the panel of step k+1 (the latency-bound critical path) runs on
// the high-priority side stream while the main stream applies the rest of step
// k's trailing update.  Per step k:
//   main: wait panel k; A[col block k+1] -= L21 L21(k+1)^T     (lookahead column)
//   side: panel(k+1)                                          (L11 = chol(A11); L21 = A21 L11^-T)
//   main: A22[k+2.., k+2..] -= L21 L21^T (lower tiles)         (multiply_transpose)
int factor_inplace(double* W, int64_t N, int64_t ld, int64_t OB, int* status, const HostOut* out = nullptr,
                   bool zero_upper_main = false) {
  cudaStream_t main = g.stream;
  const int64_t T = N / OB;
  int rc = ensure_side(2 * T + 2);
  if (rc) return rc;
  static const bool no_lookahead = getenv("STAN_CL_NO_LOOKAHEAD") != nullptr;  // debugging aid
  cudaStream_t side = no_lookahead ? main : g.side;
  cudaEvent_t* ev = g.events.data();  // ev[0]: start; ev[1 + 2k]: panel k done; ev[2 + 2k]: column k+1 ready
  CK(cudaEventRecord(ev[0], main));
  CK(cudaStreamWaitEvent(side, ev[0], 0));
  rc = panel(W, ld, 0, N, OB, status, side);
  if (rc) return rc;
  // in place: the strict upper triangle of A becomes +0.0 (F4).  Nothing in the
  // factorisation reads it, and the POTRF tiles write their own upper parts,
  // so the main stream clears the rest while the first panel runs on the side
  if (zero_upper_main) CK(zero_upper_offdiag(W, N, ld, main));
  CK(cudaEventRecord(ev[1], side));
  // streamed D2H: the rows of panel k are final once panel k is done
  auto ship = [&](int64_t k) -> int {
    if (!out) return STAN_CL_OK;
    CK(cudaStreamWaitEvent(g.d2h, ev[1 + 2 * k], 0));
    for (int64_t r0 = k * OB; r0 < (k + 1) * OB; r0 += NB) {  // lower rows + their diagonal tile
      int rc2 = copy_rect_d2h(*out, W, ld, r0, r0 + NB, 0, r0 + NB, g.d2h);
      if (rc2) return rc2;
    }
    return STAN_CL_OK;
  };
  if ((rc = ship(0))) return rc;
  // Lookahead on the side stream: the lookahead column update runs there too, so the chain
  // LA(k) -> POTRF(k+1) -> TRSM(k+1) -> LA(k+1) is one stream with PDL
  // boundaries instead of two cross-stream event hops per step.  LA(k+1)
  // waits for SYRK(k) (main), which applied panel k to column block k+2.
  //   side: [wait SYRK(k-1)] LA(k); panel(k+1)     main: [wait panel k] SYRK(k)
  // Depth 2 (STAN_CL_LA_SIDE=2): SYRK(k) also leaves column block k+2 alone
  // and LA(k+1) applies panels k and k+1 to it in one K = 2 OB product, so the
  // side chain only waits for SYRK(k-1), a step further back.
  static const int la_mode = [] {
    const char* e = getenv("STAN_CL_LA_SIDE");  // 1 / 2 = depth, 0 = never, unset = auto
    return e ? atoi(e) : -1;
  }();
  // auto (tools/quick_time.py): 128-wide steps (n < 6144) the split schedule below
  // (forward -10..12% at n = 1024 ... 4096 against LA on either stream); 256-wide
  // steps the split schedule below 12288 (6144: 4.95 -> 4.47 ms, 8192: 8.56 -> 8.00)
  // and depth 2 above (n = 16384: 49.5 -> 48.6 ms against LA on the main stream;
  // split: 49.4 -- its third-stream GEMMs are big there and take SMs from the SYRK)
  int la_depth = side == main ? 0 : (la_mode >= 0 ? la_mode : (OB == NB ? 3 : (N < 12288 ? 4 : 2)));
  if (la_depth == 3 && OB != NB) la_depth = 4;  // the split schedules: 3 for 128-wide steps, 4 for 256
  if (la_depth == 4 && OB != 2 * NB) la_depth = 3;
  // Split lookahead (la_depth 3, 128-wide steps): POTRF(k+1) needs only the
  // diagonal tile of column block k+1, so the side stream updates that tile
  // alone on ten CTAs (diag_tile_update) and goes straight on to POTRF; the rows
  // below it (needed by TRSM(k+1) only) are updated on a third stream beside
  // the POTRF and joined before the TRSM.
  //   side: [wait SYRK(k-1)] LAdiag(k); POTRF(k+1); [wait LArest(k)] TRSM(k+1)
  //   aux:  [wait panel k, SYRK(k-1)] LArest(k)       main: [wait panel k] SYRK(k)
  if (la_depth == 3 && OB == NB) {
    if (!g.aux) CK(cudaStreamCreateWithFlags(&g.aux, cudaStreamNonBlocking));
    rc = ensure_side(3 * T + 2);
    if (rc) return rc;
    ev = g.events.data();
    cudaEvent_t* ev_rest = ev + 2 * T + 2;
    for (int64_t k = 0; k < T; ++k) {
      CK(cudaStreamWaitEvent(main, ev[1 + 2 * k], 0));
      if (k == T - 1) break;
      const int64_t c0 = k * OB, r1 = (k + 1) * OB, r2 = r1 + OB;
      const double* L21 = W + r1 * ld + c0;
      if (k > 0) CK(cudaStreamWaitEvent(side, ev[2 + 2 * (k - 1)], 0));
      CK(diag_tile_update(L21, ld, W + r1 * ld + r1, ld, (int)OB, status, side));
      if (r2 < N) {
        CK(cudaStreamWaitEvent(g.aux, ev[1 + 2 * k], 0));
        if (k > 0) CK(cudaStreamWaitEvent(g.aux, ev[2 + 2 * (k - 1)], 0));
        const double* L31 = W + r2 * ld + c0;
        CK(gemm_full(true, true, (int)(N - r2), (int)OB, (int)OB, -1.0, 1, L31, ld, L21, ld, W + r2 * ld + r1, ld,
                     status, g.aux, /*lower_only=*/0, PROF_LOOKAHEAD));
        CK(cudaEventRecord(ev_rest[k], g.aux));
      }
      CK(potrf_tile(W, ld, r1, status, side));
      if (r2 < N) {
        CK(cudaStreamWaitEvent(side, ev_rest[k], 0));
        CK(trsm_panel(W, ld, r1, r2, N, status, side));
      }
      CK(cudaEventRecord(ev[1 + 2 * (k + 1)], side));
      if ((rc = ship(k + 1))) return rc;
      if (r2 < N) {
        const double* L31 = W + r2 * ld + c0;
        CK(gemm_lower_nt((int)(N - r2), (int)OB, L31, ld, L31, ld, W + r2 * ld + r2, ld, status, main));
      }
      CK(cudaEventRecord(ev[2 + 2 * k], main));
    }
    return STAN_CL_OK;
  }
  // Split lookahead for 256-wide steps (la_depth 4; depth-2 dependencies):
  // the next panel's first POTRF needs only its 128 x 128 diagonal tile, the
  // second POTRF only the in-panel update of ITS diagonal tile, so both are
  // updated alone on ten CTAs on the side stream and the remaining rows on the
  // third stream, joined before each TRSM:
  //   side: [wait SYRK(k-2)] LAdiag; POTRF(h0); [wait A] TRSM(h0); [wait B] INdiag; POTRF(h1); [wait C] TRSM(h1)
  //   aux:  [wait panel k, SYRK(k-2)] A = LA rows >= h1 of cols [h0, h1);  B = LA rows >= h1 of cols [h1, r2)
  //         [wait TRSM(h0)] C = in-panel update rows >= h1 + 128 of cols [h1, r2)
  if (la_depth == 4 && OB == 2 * NB) {
    if (!g.aux) CK(cudaStreamCreateWithFlags(&g.aux, cudaStreamNonBlocking));
    rc = ensure_side(6 * T + 2);
    if (rc) return rc;
    ev = g.events.data();
    cudaEvent_t* evx = ev + 2 * T + 2;  // per step: A, B, TRSM(h0), C
    for (int64_t k = 0; k < T; ++k) {
      CK(cudaStreamWaitEvent(main, ev[1 + 2 * k], 0));
      if (k == T - 1) break;
      const int64_t c0 = k * OB, r1 = (k + 1) * OB, h1 = r1 + NB, r2 = r1 + OB;
      const int64_t ka = k > 0 ? 2 * OB : OB, ca = c0 + OB - ka;  // LA(k) applies panels k-1, k
      cudaEvent_t* e4 = evx + 4 * k;
      if (k >= 2) CK(cudaStreamWaitEvent(side, ev[2 + 2 * (k - 2)], 0));
      CK(diag_tile_update(W + r1 * ld + ca, ld, W + r1 * ld + r1, ld, (int)ka, status, side));
      // aux: the rest of LA(k) (rows >= h1), first and second half columns
      CK(cudaStreamWaitEvent(g.aux, ev[1 + 2 * k], 0));
      if (k >= 2) CK(cudaStreamWaitEvent(g.aux, ev[2 + 2 * (k - 2)], 0));
      const double* Ar = W + h1 * ld + ca;
      CK(gemm_full(true, true, (int)(N - h1), (int)NB, (int)ka, -1.0, 1, Ar, ld, W + r1 * ld + ca, ld,
                   W + h1 * ld + r1, ld, status, g.aux, /*lower_only=*/0, PROF_LOOKAHEAD));
      CK(cudaEventRecord(e4[0], g.aux));
      CK(gemm_full(true, true, (int)(N - h1), (int)NB, (int)ka, -1.0, 1, Ar, ld, Ar, ld, W + h1 * ld + h1, ld,
                   status, g.aux, /*lower_only=*/1, PROF_LOOKAHEAD));
      CK(cudaEventRecord(e4[1], g.aux));
      // side: first half of panel k+1
      CK(potrf_tile(W, ld, r1, status, side));
      CK(cudaStreamWaitEvent(side, e4[0], 0));
      CK(trsm_panel(W, ld, r1, h1, N, status, side));
      CK(cudaEventRecord(e4[2], side));
      // in-panel update of the second half: its diagonal tile on the side stream,
      // the rows below on aux
      CK(cudaStreamWaitEvent(side, e4[1], 0));
      const double* Lh = W + h1 * ld + r1;  // L(rows >= h1, first-half columns)
      CK(diag_tile_update(Lh, ld, W + h1 * ld + h1, ld, (int)NB, status, side));
      if (h1 + NB < N) {
        CK(cudaStreamWaitEvent(g.aux, e4[2], 0));
        CK(gemm_full(true, true, (int)(N - h1 - NB), (int)NB, (int)NB, -1.0, 1, Lh + NB * ld, ld, Lh, ld,
                     W + (h1 + NB) * ld + h1, ld, status, g.aux, /*lower_only=*/0, PROF_LOOKAHEAD));
        CK(cudaEventRecord(e4[3], g.aux));
      }
      CK(potrf_tile(W, ld, h1, status, side));
      if (h1 + NB < N) {
        CK(cudaStreamWaitEvent(side, e4[3], 0));
        CK(trsm_panel(W, ld, h1, h1 + NB, N, status, side));
      }
      CK(cudaEventRecord(ev[1 + 2 * (k + 1)], side));
      if ((rc = ship(k + 1))) return rc;
      const int64_t rs = r2 + OB;  // depth 2: SYRK(k) covers rows / columns >= r2 + OB
      if (rs < N) {
        const double* L31 = W + rs * ld + c0;
        CK(gemm_lower_nt((int)(N - rs), (int)OB, L31, ld, L31, ld, W + rs * ld + rs, ld, status, main));
      }
      CK(cudaEventRecord(ev[2 + 2 * k], main));
    }
    return STAN_CL_OK;
  }
  if (la_depth > 0) {
    for (int64_t k = 0; k < T; ++k) {
      CK(cudaStreamWaitEvent(main, ev[1 + 2 * k], 0));
      if (k == T - 1) break;
      const int64_t c0 = k * OB, r1 = (k + 1) * OB, r2 = r1 + OB;
      // LA(k): column block k+1 -= the panels not yet applied to it
      const int64_t ka = (la_depth == 2 && k > 0) ? 2 * OB : OB, ca = c0 + OB - ka;
      if (k >= la_depth) CK(cudaStreamWaitEvent(side, ev[2 + 2 * (k - la_depth)], 0));
      const double* L21 = W + r1 * ld + ca;
      CK(gemm_full(true, true, (int)(N - r1), (int)OB, (int)ka, -1.0, 1, L21, ld, L21, ld, W + r1 * ld + r1, ld,
                   status, side, /*lower_only=*/1, PROF_LOOKAHEAD));
      rc = panel(W, ld, r1, N, OB, status, side);
      if (rc) return rc;
      CK(cudaEventRecord(ev[1 + 2 * (k + 1)], side));
      if ((rc = ship(k + 1))) return rc;
      const int64_t rs = r2 + (la_depth == 2 ? OB : 0);  // SYRK(k) covers rows / columns >= rs
      if (rs < N) {
        const double* L31 = W + rs * ld + c0;
        CK(gemm_lower_nt((int)(N - rs), (int)OB, L31, ld, L31, ld, W + rs * ld + rs, ld, status, main));
      }
      CK(cudaEventRecord(ev[2 + 2 * k], main));
    }
    return STAN_CL_OK;
  }
  for (int64_t k = 0; k < T; ++k) {
    CK(cudaStreamWaitEvent(main, ev[1 + 2 * k], 0));
    if (k == T - 1) break;
    const int64_t c0 = k * OB, r1 = (k + 1) * OB, r2 = r1 + OB;
    const double* L21 = W + r1 * ld + c0;
    CK(gemm_full(true, true, (int)(N - r1), (int)OB, (int)OB, -1.0, 1, L21, ld, L21, ld, W + r1 * ld + r1, ld,
                 status, main, /*lower_only=*/1, PROF_LOOKAHEAD));
    CK(cudaEventRecord(ev[2 + 2 * k], main));
    CK(cudaStreamWaitEvent(side, ev[2 + 2 * k], 0));
    rc = panel(W, ld, r1, N, OB, status, side);
    if (rc) return rc;
    CK(cudaEventRecord(ev[1 + 2 * (k + 1)], side));
    if ((rc = ship(k + 1))) return rc;
    if (r2 < N) {
      const double* L31 = W + r2 * ld + c0;
      CK(gemm_lower_nt((int)(N - r2), (int)OB, L31, ld, L31, ld, W + r2 * ld + r2, ld, status, main));
    }
  }
  return STAN_CL_OK;
}

int cholesky_enqueue(int64_t n, const double* A, double* L, int* d_info) {
  if (n < 0) return STAN_CL_EINVAL;
  if (n == 0) {
    if (d_info) CK(cudaMemsetAsync(d_info, 0, sizeof(int), g.stream));
    return STAN_CL_OK;
  }
  if (!A || !L) return STAN_CL_EINVAL;
  const size_t bytes = (size_t)n * (size_t)n * sizeof(double);
  if (A != L && ranges_overlap(A, L, bytes)) return STAN_CL_EINVAL;
  int rc = ensure_ws(al(sizeof(int) * 64));
  if (rc) return rc;
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  if (n <= 64) {
    // one small matrix: the batched register kernels with batch 1 (one launch,
    // no padded copies; the same arithmetic as the 128-tile kernel, so L is
    // bit-identical to the blocked path); the kernel writes the info word
    if (n <= 32) CK(potrf_batched_w32(A, L, (int)n, 1, status, st));
    else CK(potrf_batched_w64(A, L, (int)n, 1, status, st));
    if (d_info) CK(cudaMemcpyAsync(d_info, status, sizeof(int), cudaMemcpyDeviceToDevice, st));
    return STAN_CL_OK;
  }
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  // outer block: 256 (two-level) when it divides n, else 128 (set_block_size overrides)
  int64_t OB = g.nb;
  if (!OB) OB = fwd_outer_block(n);
  const int64_t N = round_up(n, OB);
  const bool fast = (N == n) && aligned16(A) && aligned16(L);
  if (fast) {
    if (A != L) CK(copy_lower_pad(A, n, n, L, n, n, 1.0, st));
    rc = factor_inplace(L, n, n, OB, status, nullptr, /*zero_upper_main=*/A == L);
    if (rc) return rc;
  } else {
    double* W = nullptr;
    rc = ensure_mat(0, (size_t)N * N * sizeof(double), &W);
    if (rc) return rc;
    CK(copy_lower_pad(A, n, n, W, N, N, 1.0, st));
    rc = factor_inplace(W, N, N, OB, status);
    if (rc) return rc;
    CK(copy_lower_out(W, N, L, n, n, st));
  }
  if (d_info) CK(cudaMemcpyAsync(d_info, status, sizeof(int), cudaMemcpyDeviceToDevice, st));
  return STAN_CL_OK;
}

// ------------------------------------------------------------------ adjoint
// Blocked reverse sweep on the working matrix Wm (initially
// tril(L_bar)) with factor Lw, both N x N with leading dimension ld.
// D^-1 of the B x B diagonal blocks of Lw (B = 128 or 256): the 128 x 128
// inverses by substitution (tri_inverse_batched); for B = 256 the off-diagonal
// block of [[D11, 0], [D21, D22]]^-1 is -D22^-1 D21 D11^-1 (two batched 128^3
// products).  Blocks [b0, b0 + nb) of size B; Dinv holds N/B blocks of B x B.
// tile_stride (optional): element distance between consecutive blocks (default
// the next diagonal block, B ld + B; the distributed adjoint passes the stride
// between a rank's owned diagonal tiles), results contiguous from Dinv + b0 B^2.
int block_inverses(const double* Lw, int64_t ld, int64_t B, int64_t b0, int64_t nb, double* Dinv, double* scratch,
                   int* status, cudaStream_t st, int64_t tile_stride = 0) {
  const double* Lb = Lw + b0 * B * ld + b0 * B;
  double* Db = Dinv + b0 * B * B;
  if (B == NB) {
    CK(tri_inverse_batched(Lb, ld, (int)nb, Db, status, st, 0, 0, 1, tile_stride));
    return STAN_CL_OK;
  }
  // B = 256: the 2*nb diagonal 128-inverses straight into the 256 layout, then
  // T = D21 X11 and X21 = -X22 T, both batched over the nb blocks
  CK(cudaMemsetAsync(Db, 0, (size_t)nb * B * B * sizeof(double), st));
  CK(tri_inverse_batched(Lb, ld, (int)(2 * nb), Db, status, st, B, B * B, 2, tile_stride));
  const double* D21 = Lb + NB * ld;  // rows 128.., cols 0..128 of the first block
  CK(gemm_small(NB, false, false, false, D21, ld, Db, B, scratch, NB, status, st, 1.0, (int)nb,
                tile_stride ? tile_stride : B * ld + B, B * B, (int64_t)NB * NB));
  CK(gemm_small(NB, false, false, false, Db + NB * B + NB, B, scratch, NB, Db + NB * B, B, status, st, -1.0,
                (int)nb, B * B, (int64_t)NB * NB, B * B));
  return STAN_CL_OK;
}

// Blocked reverse sweep with block B = plan.B on the working
// matrix Wm (initially tril(L_bar)) with factor Lw, both N x N with leading
// dimension ld.
// rows_ready (optional): event per 128-row block, recorded when the rows of that
// block of Lw / Wm have arrived and the D^-1 covering it is in the workspace
// (streamed H2D); out (optional): column block j of the result is shipped to the
// host as soon as it is final (after the step that Phi-s D_bar(j)).
// src (optional): L_bar itself (ld lds).  Wm is then NOT pre-initialised: the
// rows of block [j, k) get tril(L_bar) when they enter the sweep, fused with the
// split-K reduction that first writes them (adj_rows_init; R0 costs no pass).
int adjoint_inplace(const double* Lw, double* Wm, int64_t N, int64_t ld, int* status,
                    const AdjPlan& plan, const cudaEvent_t* rows_ready = nullptr,
                    const HostOut* out = nullptr, const cudaEvent_t* col_done = nullptr,
                    const double* src = nullptr, int64_t lds = 0, int64_t host_n = 0) {
  cudaStream_t st = g.stream;
  const int64_t B = plan.B;
  char* base = (char*)g.ws + al(sizeof(int) * 64);
  double* Dinv = (double*)base;
  double* Pbuf = (double*)(base + plan.dinv);
  double* T1 = (double*)(base + plan.dinv + plan.part);
  double* T2 = T1 + B * B;
  double* T3 = T2 + B * B;
  double* T4 = T3 + B * B;
  double* Ctmp = (double*)(base + plan.dinv + plan.part + plan.tmp);  // C_bar D^-1, m x B
  const int64_t nblk = N / B;
  // D^-1 of every diagonal block depends only on L: computed up front, off the
  // critical path (lower_triangular_inverse(D)); the streamed
  // host path computes it per block as the rows arrive.  Pbuf is free here.
  if (!rows_ready) {
    int rc = block_inverses(Lw, ld, B, 0, nblk, Dinv, Pbuf, status, st);
    if (rc) return rc;
  }
  for (int64_t k = N; k > 0; k -= B) {
    const int64_t j = k - B, m = N - k;
    if (rows_ready)
      for (int64_t r = j; r < k; r += NB) CK(cudaStreamWaitEvent(st, rows_ready[r / NB], 0));
    if (rows_ready) {
      // streamed host path: the rows of this block have arrived (the copy stream
      // only copies); the upper triangle of the new L_bar tiles, the diagonal
      // check and D^-1 of the block run here, in stream order with the sweep
      // (as kernels on the copy stream beside the sweep they produced wrong
      // A_bar in ~1 of 12 calls at n = 16384)
      const int64_t nn = host_n;
      for (int64_t r0 = j; r0 < k && r0 < nn; r0 += NB) {
        const int64_t r1 = std::min(r0 + NB, nn);
        CK(zero_tile_upper(Wm, ld, r0, (int)(r1 - r0), st));
        CK(check_diag(Lw + r0 * ld + r0, r1 - r0, ld, status, st, r0));
      }
      int rc2 = block_inverses(Lw, ld, B, j / B, 1, Dinv, Pbuf, status, st);
      if (rc2) return rc2;
    }
    const double* D = Lw + j * ld + j;
    const double* Db = Dinv + (j / B) * B * B;
    const double* R = Lw + j * ld;       // L(j:k, 0:j)
    double* Cb = Wm + k * ld + j;        // C_adj = L_adj(k:N, j:k)
    double* Dbar = Wm + j * ld + j;      // D_adj
    if (m > 0) {
      // C_adj = C_adj * lower_triangular_inverse(D)
      // computed out of place (persistent TMA GEMM) into Ctmp, consumed from there
      // by the two big products, and written back to A_bar afterwards
      CK(gemm_full(true, false, (int)m, (int)B, (int)B, 1.0, 0, Cb, ld, Db, B, Ctmp, B, status, st, 0, PROF_TRMM, true, 0,
                   TRI_B_LOWER));
      // B_adj = B_adj - C_adj * R
      if (j > 0)
        CK(gemm_full(true, false, (int)m, (int)j, (int)B, -1.0, 1, Ctmp, B, R, ld, Wm + k * ld, ld, status, st));
      // [R_adj D_adj] -= C_adj^T [B C]   (PAPER.md:311 and the C_adj^T B term of 319),
      // split-K over the m rows with a fixed-order reduction
      int splits, kps;
      splitk_choice(m, k, B, &splits, &kps);
      CK(gemm_splitk_tn((int)B, (int)k, (int)m, splits, kps, Ctmp, B, Lw + k * ld, ld, Pbuf, status, st));
      if (src) {  // R0 + reduce + C_bar write-back in one launch
        CK(adj_rows_init(Pbuf, splits, (int)B, k, src, lds, Wm, ld, j, N, status, st, Ctmp, B, Cb, ld, m));
      } else {
        CK(splitk_reduce_sub(Pbuf, splits, (int)B, (int)k, Wm + j * ld, ld, status, st));
        CK(copy_block(Ctmp, B, Cb, ld, m, B, st));
      }
    } else if (src) {
      CK(adj_rows_init(nullptr, 0, (int)B, 0, src, lds, Wm, ld, j, N, status, st));  // rows [j, N): tril(L_bar)
    }
    // D_adj = transpose(D) * D_adj; copy_lower_tri_to_upper_tri
    // (only the lower tiles of P = D^T D_adj are formed, stored mirrored)
    // D = transpose(lower_triangular_inverse(D)); D_adj = D * transpose(D * D_adj)
    // computed as S = D^-T sym(P) D^-1
    // copy_lower_tri_to_upper_tri; diagonal * 0.5; set_zeros_in_upper_tri
    // -- all in one launch (three DMMA products separated by grid barriers)
    CK(adj_diag_fused((int)B, D, ld, Dbar, ld, Db, T1, T2, T3, T4, (unsigned*)status + 16, status, st));
    // R_adj = R_adj - D_adj * R
    if (j > 0)
      CK(gemm_full(true, false, (int)B, (int)j, (int)B, -1.0, 1, T4, B, R, ld, Wm + j * ld, ld, status, st));
    if (out) {  // column block j is final: ship rows j.. of it
      CK(cudaEventRecord(col_done[j / B], st));
      CK(cudaStreamWaitEvent(g.d2h, col_done[j / B], 0));
      // the diagonal block per 128-row slab (the strict upper outside the 128 x 128
      // diagonal tiles is left untouched, include/stan_cl.h), then the rows below
      for (int64_t r0 = j; r0 < k; r0 += NB) {
        int rc = copy_rect_d2h(*out, Wm, ld, r0, r0 + NB, j, r0 + NB, g.d2h);
        if (rc) return rc;
      }
      int rc = copy_rect_d2h(*out, Wm, ld, k, N, j, k, g.d2h);
      if (rc) return rc;
    }
  }
  return STAN_CL_OK;
}

// The blocked reverse sweep as a two-stream pipeline (device entry points).
// Per step s (block [j, k), m = N - k) the dependency chain runs on the
// high-priority side stream:
//   C_bar D^-1 -> split-K C_bar^T [B C] -> R0 + reduce -> write-back C_bar ->
//   fused diagonal step S -> the LOOKAHEAD column of the rank-B update
//   ([S; C_bar D^-1] R on columns [j - B, j): the next step's C_bar)
// and the rest of step s's rank-B update (columns [0, j - B), one GEMM for
// both B_bar -= C_bar R and R_bar -= S R since they share R) runs on the main
// stream BESIDE the chain of step s + 1, the SMs split between the two
// persistent kernels in proportion to their DMMA work (adj_chain_sms).  The
// columns [j - 2B, j - B) are updated first on the main stream and signalled:
// they are the lookahead column of step s + 1.  Each element of A_bar receives
// the same updates in the same order as in adjoint_inplace, from the same
// kernels, so the result is bit-identical to the sequential sweep.
int adjoint_pipelined(const double* Lw, double* Wm, int64_t N, int64_t ld, int* status, const AdjPlan& plan,
                      const double* src, int64_t lds, bool two_streams = true) {
  cudaStream_t main = g.stream;
  const int64_t B = plan.B, nblk = N / B;
  int rc = ensure_side((size_t)(3 * nblk + 4));
  if (rc) return rc;
  // no programmatic dependent launch here: a dependent kernel's CTAs would sit
  // resident on SMs the other stream's persistent GEMM is sized to use
  static const bool pdl_on = getenv("STAN_CL_PIPE_PDL") && atoi(getenv("STAN_CL_PIPE_PDL")) != 0;
  struct PdlGuard {
    bool on;
    explicit PdlGuard(bool o) : on(o) { if (!on) pdl_allow(false); }
    ~PdlGuard() { if (!on) pdl_allow(true); }
  } pdl_guard_(pdl_on);
  static const bool serial = getenv("STAN_CL_NO_LOOKAHEAD") != nullptr;  // debugging aid
  cudaStream_t chain = (serial || !two_streams) ? main : g.side;
  char* base = (char*)g.ws + al(sizeof(int) * 64);
  double* Dinv = (double*)base;
  double* Pbuf = (double*)(base + plan.dinv);
  double* T1 = (double*)(base + plan.dinv + plan.part);
  double* T2 = T1 + B * B;
  double* T3 = T2 + B * B;
  char* csb = base + plan.dinv + plan.part + plan.tmp + plan.ctmp + plan.hscr;
  const size_t csz = al((size_t)(B + N) * B * sizeof(double));
  rc = block_inverses(Lw, ld, B, 0, nblk, Dinv, Pbuf, status, main);
  if (rc) return rc;
  cudaEvent_t* ev = g.events.data();  // ev[0] start; step s: ev[1+3s] chain done, ev[2+3s] first cols, ev[3+3s] rest
  if (two_streams) {
    CK(cudaEventRecord(ev[0], main));
    CK(cudaStreamWaitEvent(chain, ev[0], 0));
  }
  // one stream: the merged update of step s and C_bar D^-1 of step s+1 share a
  // persistent launch (the update's column block [j - B, j) -- the next C_bar --
  // goes first and is counted; adj_update_fused_trmm).
  // Default: fused below n = 12288 (adjoint -8% at 4096, -4% at 8192); at
  // 16384 the gain is 0.5 ms of a 144 ms step (noise level) while the fused
  // class would mix the latency-bound panel product into the trailing
  // update's roofline (0.88 instead of 0.91 of the DMMA peak), so the update
  // keeps its own launch there.  STAN_CL_ADJ_FUSE=1 / 0 forces either.
  static const int fuse_env = getenv("STAN_CL_ADJ_FUSE") ? atoi(getenv("STAN_CL_ADJ_FUSE")) : -1;
  const bool fuse = !two_streams && (fuse_env >= 0 ? fuse_env != 0 : N < 12288);
  int* dep_cnt = status + 32;
  int cnt_base = 0;
  bool cdinv_ready = false;  // C_bar D^-1 of this step already computed by the previous launch
  if (fuse) CK(cudaMemsetAsync(dep_cnt, 0, sizeof(int), main));
  int64_t s = 0;
  for (int64_t k = N; k > 0; k -= B, ++s) {
    const int64_t j = k - B, m = N - k;
    const double* D = Lw + j * ld + j;
    const double* Db = Dinv + (j / B) * B * B;
    const double* R = Lw + j * ld;  // L(j:k, 0:j)
    double* Cb = Wm + k * ld + j;   // C_adj = L_adj(k:N, j:k)
    double* Dbar = Wm + j * ld + j;
    double* cs = (double*)(csb + (size_t)(s % 3) * csz);  // [S (B x B); C_bar D^-1 (m x B)]
    const int chain_res = two_streams ? kNumSms - adj_chain_sms(N, B, k) : 0;
    // the buffer's last reader (two streams only: with one stream the order is
    // implied, and the events may last have been recorded inside a captured graph)
    if (two_streams && s >= 3) CK(cudaStreamWaitEvent(chain, ev[3 + 3 * (s - 3)], 0));
    if (m > 0) {
      // C_adj = C_adj * lower_triangular_inverse(D)
      if (!cdinv_ready)
        CK(gemm_full(true, false, (int)m, (int)B, (int)B, 1.0, 0, Cb, ld, Db, B, cs + B * B, B, status, chain, 0,
                     PROF_TRMM, true, chain_res, TRI_B_LOWER));
      // [R_adj D_adj] -= C_adj^T [B C], split-K
      // the split is the sequential sweep's (a function of m, k only), so the
      // partial sums -- and every bit of the result -- match adjoint_inplace
      int splits, kps;
      splitk_choice(m, k, B, &splits, &kps);
      CK(gemm_splitk_tn((int)B, (int)k, (int)m, splits, kps, cs + B * B, B, Lw + k * ld, ld, Pbuf, status, chain,
                        chain_res));
      if (src) {  // R0 + reduce + C_bar write-back in one launch
        CK(adj_rows_init(Pbuf, splits, (int)B, k, src, lds, Wm, ld, j, N, status, chain, cs + B * B, B, Cb, ld, m));
      } else {
        CK(splitk_reduce_sub(Pbuf, splits, (int)B, (int)k, Wm + j * ld, ld, status, chain));
        CK(copy_block(cs + B * B, B, Cb, ld, m, B, chain));
      }
    } else if (src) {
      CK(adj_rows_init(nullptr, 0, (int)B, 0, src, lds, Wm, ld, j, N, status, chain));
    }
    // S = D^-T sym(D^T D_adj) D^-1, D_adj = Phi(S)
    CK(adj_diag_fused((int)B, D, ld, Dbar, ld, Db, T1, T2, T3, cs, (unsigned*)status + 16, status, chain));
    if (!two_streams) {
      // one stream: [R_adj; B_adj] -= [S; C_adj] R over all of [0, j) in one launch
      cdinv_ready = false;
      if (j > 0 && fuse) {
        // + C_bar' D'^-1 of step s+1 (C_bar' = rows [j, N) of column block [j - B, j))
        double* cs1 = (double*)(csb + (size_t)((s + 1) % 3) * csz);
        int dep = 0;
        CK(adj_update_fused_trmm((int)(B + m), (int)j, (int)B, cs, B, R, ld, Wm + j * ld, ld, (int)(m + B),
                                 Wm + j * ld + (j - B), ld, Dinv + ((j - B) / B) * B * B, B, cs1 + B * B, B,
                                 (int)(B / 64), dep_cnt, cnt_base, &dep, status, main));
        cnt_base += dep;
        cdinv_ready = true;
      } else if (j > 0) {
        CK(gemm_full(true, false, (int)(B + m), (int)j, (int)B, -1.0, 1, cs, B, R, ld, Wm + j * ld, ld, status, main, 0,
                     PROF_GEMM));
      }
      continue;
    }
    // [R_adj; B_adj] -= [S; C_adj] R on the lookahead column [j - B, j)
    if (s >= 1) CK(cudaStreamWaitEvent(chain, ev[2 + 3 * (s - 1)], 0));
    if (j >= B)
      CK(gemm_full(true, false, (int)(B + m), (int)B, (int)B, -1.0, 1, cs, B, R + (j - B), ld, Wm + j * ld + (j - B),
                   ld, status, chain, 0, PROF_GEMM, true, chain_res));
    CK(cudaEventRecord(ev[1 + 3 * s], chain));
    // main: the rest of the rank-B update beside the next chain step
    CK(cudaStreamWaitEvent(main, ev[1 + 3 * s], 0));
    const int main_res = (k - B > 0) ? adj_chain_sms(N, B, k - B) : 0;
    if (j >= 2 * B)
      CK(gemm_full(true, false, (int)(B + m), (int)B, (int)B, -1.0, 1, cs, B, R + (j - 2 * B), ld,
                   Wm + j * ld + (j - 2 * B), ld, status, main, 0, PROF_GEMM, true, main_res));
    CK(cudaEventRecord(ev[2 + 3 * s], main));
    if (j > 2 * B)
      CK(gemm_full(true, false, (int)(B + m), (int)(j - 2 * B), (int)B, -1.0, 1, cs, B, R, ld, Wm + j * ld, ld, status,
                   main, 0, PROF_GEMM, true, main_res));
    CK(cudaEventRecord(ev[3 + 3 * s], main));
  }
  if (two_streams) CK(cudaStreamWaitEvent(main, ev[1 + 3 * (s - 1)], 0));
  return STAN_CL_OK;
}

// adjoint sweep variant (all three give bit-identical results):
//   0 = adjoint_inplace (separate B_bar / R_bar updates, one stream),
//   1 = two-stream pipeline, 2 = one stream with the merged [S; C_bar] R update.
// Default 2: with the round-2 chain kernels (blocked D^-1, fused R0 + reduce)
// the merged sweep is as fast or faster at every size (n = 1024: 0.328 vs
// 0.338 ms, 2048: 0.733 vs 0.869 ms, 16384: 94.7 vs 96.7 ms;
// profiles/r02_adjoint_variants.txt): the pipeline's SM split between two
// persistent GEMMs costs more than the chain latency it hides.
int adj_pipe_mode(int64_t N = 0) {
  (void)N;
  static const int m = [] {
    const char* e = getenv("STAN_CL_ADJ_PIPE");
    return e ? atoi(e) : 2;
  }();
  return m;
}
bool adj_pipe_enabled(int64_t N) { return adj_pipe_mode(N) != 0; }

int adjoint_enqueue(int64_t n, const double* L, const double* Lbar, double* Abar, int* d_info) {
  if (n < 0) return STAN_CL_EINVAL;
  if (n == 0) {
    if (d_info) CK(cudaMemsetAsync(d_info, 0, sizeof(int), g.stream));
    return STAN_CL_OK;
  }
  if (!L || !Lbar || !Abar) return STAN_CL_EINVAL;
  const size_t bytes = (size_t)n * (size_t)n * sizeof(double);
  if (ranges_overlap(L, Abar, bytes)) return STAN_CL_EINVAL;
  if (Lbar != Abar && ranges_overlap(Lbar, Abar, bytes)) return STAN_CL_EINVAL;
  const AdjPlan plan = adj_plan(n);
  int rc = ensure_ws(plan.total);
  if (rc) return rc;
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  if (n <= 64) {
    // one small matrix: the batched kernel (the diagonal-block step of
    // PAPER.md:313-321 on the whole matrix, in registers / shared memory);
    // it reads everything before writing, so any aliasing is fine
    if (n <= 32) CK(adjoint_batched_w32(L, Lbar, Abar, (int)n, 1, status, st));
    else CK(adjoint_batched_w64(L, Lbar, Abar, (int)n, 1, status, st));
    if (d_info) CK(cudaMemcpyAsync(d_info, status, sizeof(int), cudaMemcpyDeviceToDevice, st));
    return STAN_CL_OK;
  }
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  CK(check_diag(L, n, n, status, st));
  const int64_t N = plan.N;
  const bool fast = (N == n) && aligned16(L) && aligned16(Lbar) && aligned16(Abar);
  if (fast) {
    // A_bar starts as tril(L_bar) row block by row block inside the sweep
    rc = adj_pipe_enabled(n) ? adjoint_pipelined(L, Abar, n, n, status, plan, Lbar, n, adj_pipe_mode(n) == 1)
                            : adjoint_inplace(L, Abar, n, n, status, plan, nullptr, nullptr, nullptr, Lbar, n);
    if (rc) return rc;
  } else {
    double *Lw = nullptr, *Wm = nullptr;
    rc = ensure_mat(0, (size_t)N * N * sizeof(double), &Lw);
    if (rc) return rc;
    rc = ensure_mat(1, (size_t)N * N * sizeof(double), &Wm);
    if (rc) return rc;
    CK(copy_lower_pad(L, n, n, Lw, N, N, 1.0, st));
    CK(copy_lower_pad(Lbar, n, n, Wm, N, N, 0.0, st));
    rc = adj_pipe_enabled(N) ? adjoint_pipelined(Lw, Wm, N, N, status, plan, nullptr, 0, adj_pipe_mode(N) == 1)
                            : adjoint_inplace(Lw, Wm, N, N, status, plan);
    if (rc) return rc;
    CK(copy_lower_out(Wm, N, Abar, n, n, st));
  }
  if (d_info) CK(cudaMemcpyAsync(d_info, status, sizeof(int), cudaMemcpyDeviceToDevice, st));
  return STAN_CL_OK;
}

// ---- NEXT-2: triangular solve; NEXT-1: GP log density + gradient ----------
// O(n) scratch (slot 4): z, a (n each), hyper partial sums, then the solve's
// ready flags + ticket (ints)
struct VecScratch {
  double* z;
  double* a;
  double* partial;
  double* out;
  int* flags;
};
int vec_scratch(int64_t n, VecScratch* v) {
  const size_t nd = 2 * (size_t)n + gp_hyper_scratch_doubles() + 8;
  const size_t bytes = nd * sizeof(double) + sizeof(int) * ((size_t)n / 64 + 4);
  double* p = nullptr;
  int rc = ensure_mat(4, bytes, &p);
  if (rc) return rc;
  v->z = p;
  v->a = p + n;
  v->partial = p + 2 * n;
  v->out = v->partial + gp_hyper_scratch_doubles();
  v->flags = (int*)(p + nd);
  return STAN_CL_OK;
}

// ---- NEXT-2: lower triangular inverse, multi-RHS solve and its reverse mode ----
// Largest doubling level b = 128 * 2^s with a pair [[C1, 0], [A3, C2]] at order N.
int64_t trinv_top_level(int64_t N) {
  int64_t b = NB;
  while (2 * b < N) b *= 2;
  return b;
}
size_t trinv_scratch_doubles(int64_t N) {
  const int64_t bt = trinv_top_level(N);
  return std::max<size_t>((size_t)N * 128, (size_t)bt * (size_t)bt);
}

// X = L^-1 on N x N (N % 128 == 0) working matrices: the
// diagonal 128-blocks by substitution (tri_inverse_batched, the paper's
// diag_inv over a batch), then doubling: at level b every pair of adjacent
// b-blocks [[C1, 0], [A3, C2]] gets C3 = -C2 (A3 C1) (the paper's T = C2 A3,
// C3 = -T C1 with the association flipped: same product).  Levels 128 and 256
// run all full pairs as one batched launch per product; larger levels one
// persistent TMA GEMM per product; a ragged last pair (N not a power-of-two
// multiple of 128) is a rectangular product.  Xw must be zero on entry.
int tri_inverse_blocked(const double* Lw, int64_t ldl, double* Xw, int64_t ldx, int64_t N, double* T, int* status,
                        cudaStream_t st) {
  CK(tri_inverse_batched(Lw, ldl, (int)(N / NB), Xw, status, st, ldx, NB * ldx + NB, 1, NB * ldl + NB));
  for (int64_t b = NB; b < N; b *= 2) {
    const int64_t nf = N / (2 * b), R = N - nf * 2 * b;
    if (nf > 0 && b <= 2 * NB) {
      const int64_t sL = 2 * b * ldl + 2 * b, sX = 2 * b * ldx + 2 * b;
      CK(gemm_small((int)b, false, false, false, Lw + b * ldl, ldl, Xw, ldx, T, b, status, st, 1.0, (int)nf, sL, sX,
                    b * b));
      CK(gemm_small((int)b, false, false, false, Xw + b * ldx + b, ldx, T, b, Xw + b * ldx, ldx, status, st, -1.0,
                    (int)nf, sX, b * b, sX));
    } else {
      for (int64_t p = 0; p < nf; ++p) {
        const int64_t c0 = 2 * b * p, r0 = c0 + b;
        CK(gemm_full(true, false, (int)b, (int)b, (int)b, 1.0, 0, Lw + r0 * ldl + c0, ldl, Xw + c0 * ldx + c0, ldx,
                     T, b, status, st, 0, PROF_GP, true, 0, TRI_B_LOWER));
        CK(gemm_full(true, false, (int)b, (int)b, (int)b, -1.0, 0, Xw + r0 * ldx + r0, ldx, T, b,
                     Xw + r0 * ldx + c0, ldx, status, st, 0, PROF_GP, true, 0, TRI_A_LOWER));
      }
    }
    if (R > b) {  // ragged pair: C1 is b x b, C2 is rb x rb
      const int64_t c0 = nf * 2 * b, r0 = c0 + b, rb = R - b;
      CK(gemm_full(true, false, (int)rb, (int)b, (int)b, 1.0, 0, Lw + r0 * ldl + c0, ldl, Xw + c0 * ldx + c0, ldx,
                   T, b, status, st, 0, PROF_GP, true, 0, TRI_B_LOWER));
      CK(gemm_full(true, false, (int)rb, (int)b, (int)rb, -1.0, 0, Xw + r0 * ldx + r0, ldx, T, b,
                   Xw + r0 * ldx + c0, ldx, status, st, 0, PROF_GP, true, 0, TRI_A_LOWER));
    }
  }
  return STAN_CL_OK;
}

// block of the multi-RHS solve: 256 from n = 768 (as the adjoint), else 128
int64_t trsm_block(int64_t n) { return n >= 768 ? 2 * NB : NB; }
size_t trsm_ws_bytes(int64_t n, int64_t m) {
  const int64_t Bk = trsm_block(n), N = round_up(n, Bk), Mp = round_up(std::max<int64_t>(m, 1), 64);
  return kHdr + al((size_t)N * Bk * sizeof(double)) + al((size_t)Bk * Mp * sizeof(double)) +
         al((size_t)(N / Bk + 1) * NB * NB * sizeof(double));
}

// Wx <- L^-1 Wx (trans = false) or L^-T Wx (trans = true), in place on the
// N x Mp working matrix (ld ldw), L's working copy Lw (ld ldl), N % Bk == 0:
// right-looking blocked substitution with explicit diagonal-block inverses
// (the paper's "general solver ... adds a multiplication of the inverse",
// PAPER.md:207, applied per block so the inverses stay Bk x Bk):
//   forward, block i ascending:   S = D_i^-1 X_i;   X_{>i} -= L_{>i,i} S;   X_i = S
//   trans, block i descending:    S = D_i^-T X_i;   X_{<i} -= L_{i,<i}^T S; X_i = S
int trsm_blocked(const double* Lw, int64_t ldl, double* Wx, int64_t ldw, int64_t N, int64_t Mp, int64_t Bk,
                 bool trans, int* status, cudaStream_t st) {
  char* base = (char*)g.ws + kHdr;
  double* Dinv = (double*)base;
  double* S = (double*)(base + al((size_t)N * Bk * sizeof(double)));
  double* bscr = (double*)((char*)S + al((size_t)Bk * Mp * sizeof(double)));
  const int64_t nblk = N / Bk;
  int rc = block_inverses(Lw, ldl, Bk, 0, nblk, Dinv, bscr, status, st);
  if (rc) return rc;
  for (int64_t t = 0; t < nblk; ++t) {
    const int64_t i = trans ? nblk - 1 - t : t, r0 = i * Bk;
    const double* Di = Dinv + i * Bk * Bk;
    double* Xi = Wx + r0 * ldw;
    CK(gemm_full(!trans, false, (int)Bk, (int)Mp, (int)Bk, 1.0, 0, Di, Bk, Xi, ldw, S, Mp, status, st, 0, PROF_GP, true, 0,
                 trans ? TRI_A_UPPER : TRI_A_LOWER));
    if (!trans && r0 + Bk < N)
      CK(gemm_full(true, false, (int)(N - r0 - Bk), (int)Mp, (int)Bk, -1.0, 1, Lw + (r0 + Bk) * ldl + r0, ldl, S, Mp,
                   Xi + Bk * ldw, ldw, status, st, 0, PROF_GP));
    if (trans && r0 > 0)
      CK(gemm_full(false, false, (int)r0, (int)Mp, (int)Bk, -1.0, 1, Lw + r0 * ldl, ldl, S, Mp, Wx, ldw, status, st, 0,
                   PROF_GP));
    CK(copy_block(S, Mp, Xi, ldw, Bk, Mp, st));
  }
  return STAN_CL_OK;
}

// the working copies of a multi-RHS solve: L (N x N, padded with I) and the
// right-hand sides (N x Mp, zero padded), or the caller's buffers when aligned
struct TrsmWork {
  const double* Lw;
  int64_t ldl;
  double* Wx;
  int64_t ldw, N, Mp, Bk;
  bool direct;  // Wx is the caller's output
};
int trsm_prepare(int64_t n, int64_t m, const double* L, const double* B, double* X, TrsmWork* w, int* status,
                 cudaStream_t st) {
  w->Bk = trsm_block(n);
  w->N = round_up(n, w->Bk);
  w->Mp = round_up(m, 64);
  int rc = ensure_ws(trsm_ws_bytes(n, m));
  if (rc) return rc;
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  CK(check_diag(L, n, n, status, st));
  if (w->N == n && aligned16(L)) {
    w->Lw = L;
    w->ldl = n;
  } else {
    double* Lp = nullptr;
    if ((rc = ensure_mat(0, (size_t)w->N * w->N * sizeof(double), &Lp))) return rc;
    CK(copy_lower_pad(L, n, n, Lp, w->N, w->N, 1.0, st));
    w->Lw = Lp;
    w->ldl = w->N;
  }
  w->direct = (w->N == n && w->Mp == m && aligned16(X) && aligned16(B));
  if (w->direct) {
    w->Wx = X;
    w->ldw = m;
    if (X != B) CK(cudaMemcpyAsync(X, B, (size_t)n * m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    double* Wp = nullptr;
    if ((rc = ensure_mat(1, (size_t)w->N * w->Mp * sizeof(double), &Wp))) return rc;
    CK(cudaMemsetAsync(Wp, 0, (size_t)w->N * w->Mp * sizeof(double), st));
    CK(cudaMemcpy2DAsync(Wp, w->Mp * sizeof(double), B, m * sizeof(double), m * sizeof(double), n,
                         cudaMemcpyDeviceToDevice, st));
    w->Wx = Wp;
    w->ldw = w->Mp;
  }
  return STAN_CL_OK;
}

int read_status() {
  int rc = ensure_host_status();
  if (rc) return rc;
  CK(cudaMemcpyAsync(g.h_status, g.ws, sizeof(int), cudaMemcpyDeviceToHost, g.stream));
  CK(cudaStreamSynchronize(g.stream));
  return *g.h_status;
}

}  // namespace

// ------------------------------------------------------------- graph cache
// The first call with a given (operation, order, buffers, block sizes) runs
// eagerly (it sizes every workspace); the second captures the same enqueue
// sequence -- including the lookahead side stream and the copy streams, joined
// by events -- into a CUDA graph, and later calls replay it.  This removes the
// per-launch CPU cost of ~1000 launches per call (latency-bound small n).
// Used for the device entry points when n <= 4096 (the latency-bound regime,
// where it saves ~10%); at large n the captured graph loses the stream priority
// that lets the lookahead panel overtake the trailing update, so eager launches
// are faster there (measured: n=16384 +2%, host path +35%).  STAN_CL_GRAPH=0
// disables, =2 forces it for every size.  Off while per-launch profiling is on.
struct GraphKey {
  int op;
  int64_t n;
  const void* p[4];
  int64_t a, b;
  bool operator<(const GraphKey& o) const {
    return std::tie(op, n, p[0], p[1], p[2], p[3], a, b) < std::tie(o.op, o.n, o.p[0], o.p[1], o.p[2], o.p[3], o.a, o.b);
  }
};
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  long long launches = 0;
  int seen = 0;
  bool broken = false;
  unsigned long long gen = 0;  // workspace generation the graph was captured with
};
std::map<GraphKey, GraphEntry> g_graphs;

int graph_mode() {
  static const int m = [] {
    const char* e = getenv("STAN_CL_GRAPH");
    return e ? atoi(e) : 1;
  }();
  return m;
}
bool graphs_enabled(int64_t n) {
  const int m = graph_mode();
  return m != 0 && !prof_active() && (m == 2 || n <= 4096);
}

void clear_graphs() {
  for (auto& kv : g_graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  g_graphs.clear();
}

template <class F>
int run_cached(const GraphKey& key, F&& enqueue) {
  if (!graphs_enabled(key.op >= 2 ? 1 << 30 : key.n)) return enqueue();  // host paths: eager
  auto it = g_graphs.find(key);
  if (it == g_graphs.end()) {
    if (g_graphs.size() >= 16) clear_graphs();
    it = g_graphs.emplace(key, GraphEntry{}).first;
  }
  GraphEntry& e = it->second;
  if (e.exec && e.gen != g.gen) {
    // a workspace buffer the graph writes through was freed / moved since the
    // capture: drop it and run eagerly (this also re-sizes the workspace); the
    // next call re-captures
    cudaGraphExecDestroy(e.exec);
    e.exec = nullptr;
    e.seen = 0;
  }
  if (e.broken || e.seen++ == 0) return enqueue();
  if (!e.exec) {
    if (!g.cap) CK(cudaStreamCreateWithFlags(&g.cap, cudaStreamNonBlocking));
    cudaStream_t user = g.stream;
    g.stream = g.cap;
    const long long l0 = launches();
    cudaError_t ce = cudaStreamBeginCapture(g.cap, cudaStreamCaptureModeThreadLocal);
    int rc = ce == cudaSuccess ? enqueue() : STAN_CL_ECUDA;
    cudaGraph_t graph = nullptr;
    cudaError_t ee = cudaStreamEndCapture(g.cap, &graph);
    g.stream = user;
    const long long captured = launches() - l0;
    count_launch((int)-captured);  // nothing ran yet: replays count
    if (rc != STAN_CL_OK || ce != cudaSuccess || ee != cudaSuccess || !graph) {
      cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      e.broken = true;  // fall back to eager launches for this key
      return enqueue();
    }
    cudaError_t ie = cudaGraphInstantiate(&e.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      cudaGetLastError();
      e.exec = nullptr;
      e.broken = true;
      return enqueue();
    }
    e.launches = captured;
    e.gen = g.gen;
  }
  CK(cudaGraphLaunch(e.exec, g.stream));
  count_launch((int)e.launches);
  return STAN_CL_OK;
}

// ===================================================================== C ABI
extern "C" {

int stan_cl_cholesky_async(int64_t n, const double* A, double* L, int* d_info) {
  CallScope call_("stan_cl_cholesky_async");
  if (n <= 0) return cholesky_enqueue(n, A, L, d_info);
  return run_cached(GraphKey{0, n, {A, L, d_info, nullptr}, g.nb, 0},
                    [&] { return cholesky_enqueue(n, A, L, d_info); });
}

int stan_cl_cholesky(int64_t n, const double* A, double* L) {
  CallScope call_("stan_cl_cholesky");
  int rc = stan_cl_cholesky_async(n, A, L, nullptr);
  if (rc || n == 0) return rc;
  return read_status();
}

int stan_cl_cholesky_adjoint_async(int64_t n, const double* L, const double* L_bar, double* A_bar,
                                   int* d_info) {
  CallScope call_("stan_cl_cholesky_adjoint_async");
  if (n <= 0) return adjoint_enqueue(n, L, L_bar, A_bar, d_info);
  return run_cached(GraphKey{1, n, {L, L_bar, A_bar, d_info}, g.adj_nb, 0},
                    [&] { return adjoint_enqueue(n, L, L_bar, A_bar, d_info); });
}

int stan_cl_cholesky_adjoint(int64_t n, const double* L, const double* L_bar, double* A_bar) {
  CallScope call_("stan_cl_cholesky_adjoint");
  int rc = stan_cl_cholesky_adjoint_async(n, L, L_bar, A_bar, nullptr);
  if (rc || n == 0) return rc;
  return read_status();
}

int stan_cl_lower_triangular_inverse(int64_t n, const double* L, double* X) {
  CallScope call_("stan_cl_lower_triangular_inverse");
  if (n < 0) return STAN_CL_EINVAL;
  if (n == 0) return STAN_CL_OK;
  if (!L || !X) return STAN_CL_EINVAL;
  const size_t bytes = (size_t)n * (size_t)n * sizeof(double);
  if (ranges_overlap(L, X, bytes)) return STAN_CL_EINVAL;
  const int64_t N = round_up(n, NB);
  int rc = ensure_ws(kHdr);
  if (rc) return rc;
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  const bool fast = (N == n) && aligned16(L) && aligned16(X);
  const double* Lw = L;
  double* Xw = X;
  if (!fast) {
    double *Lp = nullptr, *Xp = nullptr;
    if ((rc = ensure_mat(0, (size_t)N * N * sizeof(double), &Lp))) return rc;
    if ((rc = ensure_mat(1, (size_t)N * N * sizeof(double), &Xp))) return rc;
    CK(copy_lower_pad(L, n, n, Lp, N, N, 1.0, st));
    Lw = Lp;
    Xw = Xp;
  }
  double* T = nullptr;
  if ((rc = ensure_mat(2, trinv_scratch_doubles(N) * sizeof(double), &T))) return rc;
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  CK(check_diag(L, n, n, status, st));
  CK(cudaMemsetAsync(Xw, 0, (size_t)N * N * sizeof(double), st));
  if ((rc = tri_inverse_blocked(Lw, N, Xw, N, N, T, status, st))) return rc;
  if (!fast) CK(copy_lower_out(Xw, N, X, n, n, st));
  return read_status();
}

int stan_cl_trsm(int64_t n, int64_t m, const double* L, const double* B, double* X, int trans) {
  CallScope call_("stan_cl_trsm");
  if (n < 0 || m < 0) return STAN_CL_EINVAL;
  if (n == 0 || m == 0) return STAN_CL_OK;
  if (!L || !B || !X) return STAN_CL_EINVAL;
  const size_t xb = (size_t)n * (size_t)m * sizeof(double);
  if (X != B && ranges_overlap(X, B, xb)) return STAN_CL_EINVAL;
  if (ranges_overlap2(X, xb, L, (size_t)n * n * sizeof(double))) return STAN_CL_EINVAL;
  int* status = nullptr;
  TrsmWork w;
  int rc = ensure_ws(trsm_ws_bytes(n, m));
  if (rc) return rc;
  status = (int*)g.ws;
  cudaStream_t st = g.stream;
  if ((rc = trsm_prepare(n, m, L, B, X, &w, status, st))) return rc;
  if ((rc = trsm_blocked(w.Lw, w.ldl, w.Wx, w.ldw, w.N, w.Mp, w.Bk, trans != 0, status, st))) return rc;
  if (!w.direct)
    CK(cudaMemcpy2DAsync(X, m * sizeof(double), w.Wx, w.ldw * sizeof(double), m * sizeof(double), n,
                         cudaMemcpyDeviceToDevice, st));
  return read_status();
}

int stan_cl_trsm_adjoint(int64_t n, int64_t m, const double* L, const double* C, const double* C_bar,
                         double* L_bar, double* B_bar) {
  CallScope call_("stan_cl_trsm_adjoint");
  if (n < 0 || m < 0) return STAN_CL_EINVAL;
  if (n == 0) return STAN_CL_OK;
  if (!L || !L_bar || (m > 0 && (!C || !C_bar || !B_bar))) return STAN_CL_EINVAL;
  const size_t xb = (size_t)n * (size_t)m * sizeof(double), lb = (size_t)n * n * sizeof(double);
  if (m > 0) {
    if (B_bar != C_bar && ranges_overlap(B_bar, C_bar, xb)) return STAN_CL_EINVAL;
    if (ranges_overlap2(B_bar, xb, L, lb) || ranges_overlap2(B_bar, xb, C, xb) ||
        ranges_overlap2(B_bar, xb, L_bar, lb))
      return STAN_CL_EINVAL;
    if (ranges_overlap2(L_bar, lb, L, lb) || ranges_overlap2(L_bar, lb, C, xb) || ranges_overlap2(L_bar, lb, C_bar, xb))
      return STAN_CL_EINVAL;
  } else if (ranges_overlap(L_bar, L, lb)) {
    return STAN_CL_EINVAL;
  }
  int rc = ensure_ws(trsm_ws_bytes(n, std::max<int64_t>(m, 1)));
  if (rc) return rc;
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  if (m == 0) {
    CK(cudaMemsetAsync(status, 0, sizeof(int), st));
    CK(check_diag(L, n, n, status, st));
    CK(cudaMemsetAsync(L_bar, 0, lb, st));
    return read_status();
  }
  // B_bar = L^-T C_bar (the solve of the primitive, transposed)
  TrsmWork w;
  if ((rc = trsm_prepare(n, m, L, C_bar, B_bar, &w, status, st))) return rc;
  if ((rc = trsm_blocked(w.Lw, w.ldl, w.Wx, w.ldw, w.N, w.Mp, w.Bk, true, status, st))) return rc;
  // L_bar = tril(-B_bar C^T): lower tiles only (PAPER.md:236 adjA = -adjB C^T),
  // into an N x N working matrix when padded; C is staged zero-padded to N x Mp
  const double* Cw = C;
  double* Lb = L_bar;
  const bool direct_l = w.direct && aligned16(C) && aligned16(L_bar);
  if (!direct_l) {
    double *Cp = nullptr, *Lp = nullptr;
    if ((rc = ensure_mat(2, (size_t)w.N * w.Mp * sizeof(double), &Cp))) return rc;
    if ((rc = ensure_mat(3, (size_t)w.N * w.N * sizeof(double), &Lp))) return rc;
    CK(cudaMemsetAsync(Cp, 0, (size_t)w.N * w.Mp * sizeof(double), st));
    CK(cudaMemcpy2DAsync(Cp, w.Mp * sizeof(double), C, m * sizeof(double), m * sizeof(double), n,
                         cudaMemcpyDeviceToDevice, st));
    Cw = Cp;
    Lb = Lp;
  }
  const int64_t ldlb = direct_l ? n : w.N, ldc = direct_l ? m : w.Mp;
  CK(cudaMemsetAsync(Lb, 0, (size_t)w.N * ldlb * sizeof(double), st));
  CK(gemm_lower_nt((int)w.N, (int)w.Mp, w.Wx, w.ldw, Cw, ldc, Lb, ldlb, status, st));
  if (!direct_l) CK(copy_lower_out(Lb, w.N, L_bar, n, n, st));
  if (!w.direct)
    CK(cudaMemcpy2DAsync(B_bar, m * sizeof(double), w.Wx, w.ldw * sizeof(double), m * sizeof(double), n,
                         cudaMemcpyDeviceToDevice, st));
  return read_status();
}

int stan_cl_check_matrix(int64_t n, const double* A, int checks, double tol) {
  CallScope call_("stan_cl_check_matrix");
  if (n < 0 || (checks & ~7) || !(tol >= 0.0)) return STAN_CL_EINVAL;
  if (n == 0 || checks == 0) return 0;
  if (!A) return STAN_CL_EINVAL;
  int rc = ensure_ws(kHdr);
  if (rc) return rc;
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  CK(check_matrix(A, n, checks, tol, status, st));
  return read_status();
}

int stan_cl_trsv(int64_t n, const double* L, const double* b, double* x, int trans) {
  CallScope call_("stan_cl_trsv");
  if (n < 0) return STAN_CL_EINVAL;
  if (n == 0) return STAN_CL_OK;
  if (!L || !b || !x) return STAN_CL_EINVAL;
  const size_t vb = (size_t)n * sizeof(double);
  if (x != b && ranges_overlap(x, b, vb)) return STAN_CL_EINVAL;
  if (ranges_overlap2(x, vb, L, (size_t)n * vb)) return STAN_CL_EINVAL;
  int rc = ensure_ws(al(sizeof(int) * 64));
  if (rc) return rc;
  VecScratch v;
  if ((rc = vec_scratch(n, &v))) return rc;
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  CK(check_diag(L, n, n, status, st));
  CK(trsv(L, n, n, b, x, trans != 0, v.flags, status, st));
  return read_status();
}

int stan_cl_gp_lpdf_grad(int64_t n, const double* x, const double* y, double alpha, double rho, double sigma,
                         double* out, double* y_bar) {
  CallScope call_("stan_cl_gp_lpdf_grad");
  if (n < 0) return STAN_CL_EINVAL;
  if (n > 0 && (!x || !y || !out)) return STAN_CL_EINVAL;
  if (!(rho != 0.0) || !(rho - rho == 0.0) || !(alpha - alpha == 0.0) || !(sigma - sigma == 0.0))
    return STAN_CL_EINVAL;
  cudaStream_t st = g.stream;
  if (n == 0) {
    if (out) CK(cudaMemsetAsync(out, 0, 4 * sizeof(double), st));
    return STAN_CL_OK;
  }
  const size_t bytes = (size_t)n * (size_t)n * sizeof(double);
  double *K = nullptr, *W = nullptr;
  // size the shared workspace for the adjoint first: growing it later would
  // move the status word the kernels below are given
  int rc = ensure_ws(adj_plan(n).total);
  if (rc) return rc;
  if ((rc = ensure_mat(2, bytes, &K))) return rc;
  if ((rc = ensure_mat(3, bytes, &W))) return rc;
  VecScratch v;
  if ((rc = vec_scratch(n, &v))) return rc;
  // K = SE + sigma^2 I;  L = chol(K) in place (the hot path's forward)
  CK(se_cov(n, x, alpha, rho, sigma * sigma, K, st));
  if ((rc = cholesky_enqueue(n, K, K, nullptr))) return rc;
  if ((rc = read_status())) return rc;  // not positive definite: info
  int* status = (int*)g.ws;
  // z = L^-1 y, lp, a = L^-T z, L_bar
  CK(trsv(K, n, n, y, v.z, false, v.flags, status, st));
  CK(gp_lp(K, n, n, v.z, out, status, st));
  CK(trsv(K, n, n, v.z, v.a, true, v.flags, status, st));
  CK(gp_lbar(K, n, n, v.a, v.z, W, n, status, st));
  // A_bar = cholesky_adjoint(L, L_bar), in place (the hot path's adjoint)
  if ((rc = adjoint_enqueue(n, K, W, W, nullptr))) return rc;
  status = (int*)g.ws;
  CK(gp_hyper(W, n, n, x, alpha, rho, sigma, v.partial, out + 1, status, st));
  if (y_bar) CK(negate(v.a, y_bar, n, status, st));
  return read_status();
}

// ---- NEXT-4: batched small matrices ----------------------------------------
int stan_cl_cholesky_batched(int64_t batch, int64_t n, const double* A, double* L, int* info) {
  CallScope call_("stan_cl_cholesky_batched");
  if (batch < 0 || n < 0 || n > NB) return STAN_CL_EINVAL;
  if (batch == 0 || n == 0) return STAN_CL_OK;
  if (!A || !L) return STAN_CL_EINVAL;
  const size_t bytes = (size_t)batch * (size_t)n * (size_t)n * sizeof(double);
  if (A != L && ranges_overlap(A, L, bytes)) return STAN_CL_EINVAL;
  int rc = ensure_ws(al(sizeof(int) * 64));
  if (rc) return rc;
  int* inf = info;
  if (!inf) {
    double* p = nullptr;
    if ((rc = ensure_mat(4, sizeof(int) * (size_t)batch, &p))) return rc;
    inf = (int*)p;
  }
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  if (n <= 32) {
    CK(potrf_batched_w32(A, L, (int)n, batch, inf, st));
  } else if (n <= 64) {
    CK(potrf_batched_w64(A, L, (int)n, batch, inf, st));
  } else {
    CK(cudaMemsetAsync(inf, 0, sizeof(int) * (size_t)batch, st));
    CK(potrf_batched(A, L, (int)n, batch, inf, st));
  }
  CK(batched_first_fail(inf, batch, status, st));
  return read_status();
}

int stan_cl_cholesky_adjoint_batched(int64_t batch, int64_t n, const double* L, const double* L_bar,
                                     double* A_bar, int* info) {
  CallScope call_("stan_cl_cholesky_adjoint_batched");
  if (batch < 0 || n < 0 || n > NB) return STAN_CL_EINVAL;
  if (batch == 0 || n == 0) return STAN_CL_OK;
  if (!L || !L_bar || !A_bar) return STAN_CL_EINVAL;
  const size_t bytes = (size_t)batch * (size_t)n * (size_t)n * sizeof(double);
  if (L != A_bar && ranges_overlap(L, A_bar, bytes)) return STAN_CL_EINVAL;
  if (L_bar != A_bar && ranges_overlap(L_bar, A_bar, bytes)) return STAN_CL_EINVAL;
  int rc = ensure_ws(al(sizeof(int) * 64));
  if (rc) return rc;
  if (n <= 64) {  // one or two warps per matrix, no padded copies
    int* inf = info;
    if (!inf) {
      double* p = nullptr;
      if ((rc = ensure_mat(4, sizeof(int) * (size_t)batch, &p))) return rc;
      inf = (int*)p;
    }
    cudaStream_t st = g.stream;
    if (n <= 32) CK(adjoint_batched_w32(L, L_bar, A_bar, (int)n, batch, inf, st));
    else CK(adjoint_batched_w64(L, L_bar, A_bar, (int)n, batch, inf, st));
    CK(batched_first_fail(inf, batch, (int*)g.ws, st));
    return read_status();
  }
  // padded 128 x 128 work tiles: Lp, Wp (-> T2), Dinv, T1 (-> T3); chunks bound
  // the scratch and the 65535 grid-z limit of the batched products
  const int64_t chunk = batch < 4096 ? batch : 4096;
  const int64_t T2e = (int64_t)NB * NB;
  double* w = nullptr;
  if ((rc = ensure_mat(2, sizeof(double) * 4 * (size_t)chunk * (size_t)T2e, &w))) return rc;
  double *Lp = w, *Wp = w + chunk * T2e, *Dinv = w + 2 * chunk * T2e, *T1 = w + 3 * chunk * T2e;
  int* inf = info;
  if (!inf) {
    double* p = nullptr;
    if ((rc = ensure_mat(4, sizeof(int) * (size_t)batch, &p))) return rc;
    inf = (int*)p;
  }
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  CK(batched_check_diag(L, (int)n, batch, inf, st));
  const int64_t nn = n * n;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int64_t nb = batch - b0 < chunk ? batch - b0 : chunk;
    CK(batched_pad(L + b0 * nn, L_bar + b0 * nn, (int)n, nb, Lp, Wp, st));
    CK(tri_inverse_batched(Lp, NB, (int)nb, Dinv, status, st, NB, T2e, 1, T2e));
    // P = D^T D_bar (lower tiles, mirrored); S = D^-T sym(P) D^-1
    CK(gemm_small(NB, true, true, false, Lp, NB, Wp, NB, T1, NB, status, st, 1.0, (int)nb, T2e, T2e, T2e, true));
    CK(gemm_small(NB, true, false, false, Dinv, NB, T1, NB, Wp, NB, status, st, 1.0, (int)nb, T2e, T2e, T2e));
    CK(gemm_small(NB, false, false, false, Wp, NB, Dinv, NB, T1, NB, status, st, 1.0, (int)nb, T2e, T2e, T2e));
    // A_bar = Phi(sym S), leading n x n block
    CK(batched_phi_out(T1, (int)n, nb, A_bar + b0 * nn, st));
  }
  CK(batched_first_fail(inf, batch, status, st));
  return read_status();
}

int stan_cl_gp_exp_quad_cov(int64_t n, const double* x, double alpha, double rho, double jitter,
                            double* K) {
  if (n < 0) return STAN_CL_EINVAL;
  if (n == 0) return STAN_CL_OK;
  if (!x || !K) return STAN_CL_EINVAL;
  if (!(rho != 0.0) || !(rho - rho == 0.0)) return STAN_CL_EINVAL;
  CK(se_cov(n, x, alpha, rho, jitter, K, g.stream));
  return STAN_CL_OK;
}

// Host-buffer entry points: only the lower triangles cross PCIe (the paper's
// packed transfers), as one rectangle per 128-row block
// (rows r0..r1, columns 0..r1), and the transfers are streamed against the
// compute: the forward ships each panel's rows as soon as that panel is
// factored; the adjoint uploads row blocks bottom-up (the order the reverse
// sweep consumes them) and ships each column block of A_bar as soon as it is
// final.
int cholesky_host_enqueue(int64_t n, const double* A, double* L) {
  int64_t OB = g.nb;
  if (!OB) OB = fwd_outer_block(n);
  const int64_t N = round_up(n, OB);
  int rc = ensure_ws(al(sizeof(int) * 64));
  if (rc) return rc;
  if ((rc = ensure_copy(4))) return rc;
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  double* W = nullptr;
  if ((rc = ensure_mat(0, (size_t)N * N * sizeof(double), &W))) return rc;
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  CK(init_pad(W, n, N, 1.0, st));
  CK(cudaEventRecord(g.xev[0], st));
  CK(cudaStreamWaitEvent(g.h2d, g.xev[0], 0));
  for (int64_t r0 = 0; r0 < n; r0 += NB) {
    const int64_t r1 = std::min(r0 + NB, n);
    CK(cudaMemcpy2DAsync(W + r0 * N, N * sizeof(double), A + r0 * n, n * sizeof(double), r1 * sizeof(double),
                         r1 - r0, cudaMemcpyHostToDevice, g.h2d));
  }
  CK(cudaEventRecord(g.xev[1], g.h2d));
  CK(cudaStreamWaitEvent(st, g.xev[1], 0));
  HostOut out{L, n};
  rc = factor_inplace(W, N, N, OB, status, &out);
  if (rc) return rc;
  CK(cudaEventRecord(g.xev[2], g.d2h));
  CK(cudaStreamWaitEvent(st, g.xev[2], 0));
  return STAN_CL_OK;
}

// +0.0 into the strict upper triangle of a host output outside the 128 x 128
// diagonal tiles (the streamed copies write the lower rectangles and the
// diagonal tiles, include/stan_cl.h), by host threads while the device works:
// row r gets columns [end of r's 128-row tile, n), disjoint from every copy.
struct HostUpperZero {
  std::vector<std::thread> th;
  HostUpperZero(double* out, int64_t n) {
    if (n <= NB) return;
    const unsigned hc = std::thread::hardware_concurrency();
    const int T = (int)std::max(1u, std::min(8u, hc ? hc / 2 : 1u));
    // rows split by equal zero-fill volume: row r has about n - r entries to fill
    std::vector<int64_t> cut{0};
    const double total = 0.5 * (double)n * (double)n;
    int64_t r = 0;
    double acc = 0;
    for (int t = 1; t < T; ++t) {
      while (r < n && acc < total * t / T) acc += (double)(n - r++);
      cut.push_back(r);
    }
    cut.push_back(n);
    for (int t = 0; t < T; ++t)
      th.emplace_back([=] {
        for (int64_t i = cut[t]; i < cut[t + 1]; ++i) {
          const int64_t c0 = std::min(n, (i / NB + 1) * NB);
          if (c0 < n) memset(out + i * n + c0, 0, (size_t)(n - c0) * sizeof(double));
        }
      });
  }
  ~HostUpperZero() {
    for (auto& t : th) t.join();
  }
};

int stan_cl_cholesky_host(int64_t n, const double* A, double* L) {
  CallScope call_("stan_cl_cholesky_host");
  PdlOff pdl_off_;
  if (n < 0) return STAN_CL_EINVAL;
  if (n == 0) return STAN_CL_OK;
  if (!A || !L) return STAN_CL_EINVAL;
  if (A != L && ranges_overlap(A, L, (size_t)n * (size_t)n * sizeof(double))) return STAN_CL_EINVAL;
  HostUpperZero zero_(L, n);
  int rc = run_cached(GraphKey{2, n, {A, L, nullptr, nullptr}, g.nb, 0},
                      [&] { return cholesky_host_enqueue(n, A, L); });
  if (rc) return rc;
  return read_status();
}

int adjoint_host_enqueue(int64_t n, const double* L, const double* L_bar, double* A_bar) {
  const AdjPlan plan = adj_plan(n);
  const int64_t N = plan.N, nblk = N / NB;
  int rc = ensure_ws(plan.total);
  if (rc) return rc;
  if ((rc = ensure_copy(2 * nblk + 4))) return rc;
  int* status = (int*)g.ws;
  cudaStream_t st = g.stream;
  double *Lw = nullptr, *Wm = nullptr;
  if ((rc = ensure_mat(0, (size_t)N * N * sizeof(double), &Lw))) return rc;
  if ((rc = ensure_mat(1, (size_t)N * N * sizeof(double), &Wm))) return rc;
  CK(cudaMemsetAsync(status, 0, sizeof(int), st));
  CK(init_pad(Lw, n, N, 1.0, st));
  CK(init_pad(Wm, n, N, 0.0, st));
  cudaEvent_t* ready = g.xev.data() + 2;
  cudaEvent_t* col_done = ready + nblk;
  CK(cudaEventRecord(g.xev[0], st));
  CK(cudaStreamWaitEvent(g.h2d, g.xev[0], 0));
  for (int64_t b = nblk - 1; b >= 0; --b) {  // bottom-up: the order the reverse sweep needs
    const int64_t r0 = b * NB, r1 = std::min(r0 + NB, n);
    if (r0 < n) {
      CK(cudaMemcpy2DAsync(Lw + r0 * N, N * sizeof(double), L + r0 * n, n * sizeof(double), r1 * sizeof(double),
                           r1 - r0, cudaMemcpyHostToDevice, g.h2d));
      CK(cudaMemcpy2DAsync(Wm + r0 * N, N * sizeof(double), L_bar + r0 * n, n * sizeof(double),
                           r1 * sizeof(double), r1 - r0, cudaMemcpyHostToDevice, g.h2d));
    }
    CK(cudaEventRecord(ready[b], g.h2d));
  }
  HostOut out{A_bar, n};
  rc = adjoint_inplace(Lw, Wm, N, N, status, plan, ready, &out, col_done, nullptr, 0, n);
  if (rc) return rc;
  CK(cudaEventRecord(g.xev[1], g.d2h));
  CK(cudaStreamWaitEvent(st, g.xev[1], 0));
  return STAN_CL_OK;
}

int stan_cl_cholesky_adjoint_host(int64_t n, const double* L, const double* L_bar, double* A_bar) {
  CallScope call_("stan_cl_cholesky_adjoint_host");
  PdlOff pdl_off_;
  if (n < 0) return STAN_CL_EINVAL;
  if (n == 0) return STAN_CL_OK;
  if (!L || !L_bar || !A_bar) return STAN_CL_EINVAL;
  const size_t bytes = (size_t)n * (size_t)n * sizeof(double);
  if (ranges_overlap(L, A_bar, bytes)) return STAN_CL_EINVAL;
  if (L_bar != A_bar && ranges_overlap(L_bar, A_bar, bytes)) return STAN_CL_EINVAL;
  HostUpperZero zero_(A_bar, n);
  int rc = run_cached(GraphKey{3, n, {L, L_bar, A_bar, nullptr}, g.adj_nb, 0},
                      [&] { return adjoint_host_enqueue(n, L, L_bar, A_bar); });
  if (rc) return rc;
  return read_status();
}

int stan_cl_set_stream(void* s) {
  g.stream = (cudaStream_t)s;
  return STAN_CL_OK;
}

void* stan_cl_get_stream(void) { return (void*)g.stream; }

int stan_cl_set_block_size(int nb) {
  if (nb == 0 || nb == NB || nb == 2 * NB) {
    g.nb = nb;
    return STAN_CL_OK;
  }
  return STAN_CL_EINVAL;
}

int stan_cl_get_block_size(void) { return g.nb; }

int stan_cl_set_adjoint_block_size(int nb) {
  if (nb == 0 || nb == NB || nb == 2 * NB) {
    g.adj_nb = nb;
    return STAN_CL_OK;
  }
  return STAN_CL_EINVAL;
}

// Bytes of caller workspace the single-GPU entry points need at order n, laid
// out as CallScope / ensure_ws / ensure_mat carve them (16-byte aligned
// buffers assumed: an unaligned caller buffer takes the padded path, which
// needs the padded matrices below even when n divides the block).
size_t stan_cl_workspace_bytes(int64_t n) {
  if (n <= 0) return kHdr;
  const AdjPlan p = adj_plan(n);
  const int64_t OB = g.nb ? g.nb : fwd_outer_block(n);
  const size_t Nf = (size_t)round_up(n, OB), Na = (size_t)p.N, nn = (size_t)n;
  const size_t mat_f = al(Nf * Nf * sizeof(double)), mat_a = al(Na * Na * sizeof(double));
  const size_t vec = al((2 * nn + gp_hyper_scratch_doubles() + 8) * sizeof(double) + sizeof(int) * (nn / 64 + 4));
  const size_t adj_ws = al(std::max(p.total, kHdr));
  size_t need = kHdr + ((Nf == nn) ? 0 : mat_f);                     // cholesky
  need = std::max(need, adj_ws + ((Na == nn) ? 0 : 2 * mat_a));     // cholesky_adjoint
  need = std::max(need, kHdr + mat_f);                               // cholesky_host
  need = std::max(need, adj_ws + 2 * mat_a);                         // cholesky_adjoint_host
  need = std::max(need, kHdr + vec);                                 // trsv
  // gp_lpdf_grad: K, W (n x n), the O(n) scratch, then the padded matrices of
  // the inner cholesky / adjoint when n is not a block multiple
  const size_t pads = std::max((Nf == nn) ? 0 : mat_f, (Na == nn) ? 0 : 2 * mat_a);
  need = std::max(need, adj_ws + 2 * al(nn * nn * sizeof(double)) + vec + pads);
  // lower_triangular_inverse: padded L and X when n % 128 != 0, doubling scratch
  const size_t N128 = (size_t)round_up(n, NB);
  const size_t mat_128 = al(N128 * N128 * sizeof(double));
  need = std::max(need, kHdr + ((N128 == nn) ? 0 : 2 * mat_128) + al(trinv_scratch_doubles((int64_t)N128) * sizeof(double)));
  return need;
}

size_t stan_cl_trsm_workspace_bytes(int64_t n, int64_t m) {
  if (n <= 0) return kHdr;
  const int64_t Bk = trsm_block(n), N = round_up(n, Bk), Mp = round_up(std::max<int64_t>(m, 1), 64);
  const size_t ws = al(trsm_ws_bytes(n, std::max<int64_t>(m, 1)));
  const size_t Lp = al((size_t)N * N * sizeof(double)), Wp = al((size_t)N * Mp * sizeof(double));
  // trsm_adjoint, padded: L, right-hand sides, C and L_bar working copies
  return ws + 2 * Lp + 2 * Wp;
}

size_t stan_cl_batched_workspace_bytes(int64_t batch, int64_t n, int with_info) {
  if (batch <= 0 || n <= 0) return kHdr;
  const size_t inf = with_info ? 0 : al(sizeof(int) * (size_t)batch);
  if (n <= 64) return kHdr + inf;
  const size_t chunk = (size_t)std::min<int64_t>(batch, 4096);
  return kHdr + al(sizeof(double) * 4 * chunk * (size_t)NB * NB) + inf;
}

int stan_cl_set_workspace(void* dev_ptr, size_t bytes) {
  if (g.depth) return STAN_CL_EINVAL;
  if (dev_ptr && (((uintptr_t)dev_ptr & (kAlign - 1)) != 0 || bytes < kHdr)) return STAN_CL_EINVAL;
  // drop every library-owned buffer (the caller's memory bound is the point)
  CK(cudaDeviceSynchronize());
  clear_graphs();
  if (!g.user_ws && g.ws) CK(cudaFree(g.ws));
  for (int i = 0; i < 5; ++i)
    if (!g.user_ws && g.mat[i]) CK(cudaFree(g.mat[i]));
  for (int i = 0; i < 5; ++i) {
    g.mat[i] = nullptr;
    g.mat_cap[i] = 0;
  }
  g.ws = nullptr;
  g.ws_cap = 0;
  ++g.gen;
  g.user_ws = (char*)dev_ptr;
  g.user_cap = dev_ptr ? bytes : 0;
  g.user_next = 0;
  if (dev_ptr) {
    // the header (status word, grid-barrier counters) starts at zero; the
    // kernels leave the counters at zero
    CK(cudaMemset(dev_ptr, 0, kHdr));
    g.ws = g.user_ws;
    g.ws_cap = kHdr;
  }
  return STAN_CL_OK;
}

const char* stan_cl_status_string(int status) {
  switch (status) {
    case STAN_CL_OK: return "ok";
    case STAN_CL_EINVAL: return "invalid argument";
    case STAN_CL_ENOMEM: return g.last_err[0] ? g.last_err : "device workspace allocation failed";
    case STAN_CL_ECUDA: return g.last_err[0] ? g.last_err : "CUDA error";
    case STAN_CL_ENCCL: return "NCCL error";
    default: return status > 0 ? "numerical failure (not positive definite / bad diagonal)" : "unknown status";
  }
}

long long stan_cl_kernel_launches(void) { return launches(); }

int stan_cl_profile_enable(int mask) {
  prof_enable(mask == 1 ? ~0u : (unsigned)mask >> 1);
  return STAN_CL_OK;
}

int stan_cl_profile_reset(void) {
  prof_reset();
  return STAN_CL_OK;
}

int stan_cl_profile_read(int kind, double* ms, double* flops, long long* n) {
  if (kind < 0 || kind >= PROF_KINDS || !ms || !flops || !n) return STAN_CL_EINVAL;
  prof_read(kind, ms, flops, n);
  return STAN_CL_OK;
}

int stan_cl_profile_read_bytes(int kind, double* bytes) {
  if (kind < 0 || kind >= PROF_KINDS || !bytes) return STAN_CL_EINVAL;
  double ms, fl;
  long long n;
  prof_read(kind, &ms, &fl, &n, bytes);
  return STAN_CL_OK;
}

int stan_cl_trace_enable(int on) {
  if (on) trace_start(g.stream);
  else trace_stop();
  return STAN_CL_OK;
}

int stan_cl_trace_read(double* out, int max_records) {
  if (max_records < 0 || (max_records > 0 && !out)) return STAN_CL_EINVAL;
  return trace_read(out, max_records);
}

int stan_cl_finalize(void) {
  clear_graphs();
  if (g.cap) {
    cudaStreamDestroy(g.cap);
    g.cap = nullptr;
  }
  if (g.ws) {
    cudaStreamSynchronize(g.stream);
    if (!g.user_ws) cudaFree(g.ws);
    g.ws = nullptr;
    g.ws_cap = 0;
  }
  if (g.h_status) {
    cudaFreeHost(g.h_status);
    g.h_status = nullptr;
  }
  for (cudaEvent_t e : g.events) cudaEventDestroy(e);
  g.events.clear();
  for (cudaEvent_t e : g.xev) cudaEventDestroy(e);
  g.xev.clear();
  for (int i = 0; i < 5; ++i) {
    if (g.mat[i] && !g.user_ws) cudaFree(g.mat[i]);
    g.mat[i] = nullptr;
    g.mat_cap[i] = 0;
  }
  g.user_ws = nullptr;  // the caller's workspace is never freed by the library
  g.user_cap = g.user_next = 0;
  ++g.gen;
  if (g.h2d) {
    cudaStreamDestroy(g.h2d);
    g.h2d = nullptr;
  }
  if (g.d2h) {
    cudaStreamDestroy(g.d2h);
    g.d2h = nullptr;
  }
  if (g.side) {
    cudaStreamDestroy(g.side);
    g.side = nullptr;
  }
  if (g.aux) {
    cudaStreamDestroy(g.aux);
    g.aux = nullptr;
  }
  return STAN_CL_OK;
}

int stan_cl_version(void) { return 100; }

}  // extern "C"

// ============================================================ multi-GPU layer
// Distributed factorisation and adjoint over a P x Q process grid (one process
// per GPU), 2-D block-cyclic by 256 x 256 tiles (ScaLAPACK
// PDPOTRF style): tile (I, J) lives on rank (I % P, J % Q) = global rank
// (I % P) * Q + J % Q, as local tile (I / P, J / Q) of a row-major
// (R_p * 256) x (C_q * 256) array (R_p / C_q = number of block rows / columns
// with I % P == p / J % Q == q).  Only the lower tiles (I >= J) are read or
// written.  P = 1 is block-column cyclic (every rank holds whole columns).
//
//   forward step k
//     diagonal owner (k%P, k%Q): L_kk = chol(A_kk)   -> column broadcast
//     process column k%Q: L_Ik = A_Ik L_kk^-T for its rows I > k
//     row broadcast of those panel rows along every process row
//     column exchange: rank (p', q) sends the panel tiles L_Jk with J % Q == q
//       to its process column (P > 1 only)
//     every rank: A_IJ -= L_Ik L_Jk^T on its lower tiles I >= J > k
//   adjoint step for block jb
//     column broadcast of D^-1 (column jb%Q); C_bar D^-1 there
//     row broadcast of C_bar D^-1; column broadcast of L's row block jb
//     every rank: B_bar -= C_bar R on its tiles
//     every rank: partial C_bar^T [B C] over its rows; column reduce to the
//       owners of block row jb (P > 1)
//     diagonal owner: symbolic step -> sym(S)
//     row broadcast of sym(S) along process row jb%P: R_bar -= sym(S) R
// Collectives: ncclBroadcast / ncclReduce on the row and column communicators
// (ncclCommSplit of the world communicator), issued by every rank in the same
// global order.  The same code drives a single-process simulation of the P*Q
// ranks on one device (broadcast = device copies, reduce = fixed-order adds),
// which is what the tests exercise on a one-GPU box.
namespace {

constexpr int64_t DB = 2 * NB;  // distributed tile

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;  // optional
  ncclResult_t (*commAbort)(ncclComm_t) = nullptr;                        // optional
  bool load() {
    if (h) return true;
    const char* env = getenv("STAN_CL_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm) continue;
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    commSplit = (decltype(commSplit))dlsym(h, "ncclCommSplit");
    broadcast = (decltype(broadcast))dlsym(h, "ncclBroadcast");
    reduce = (decltype(reduce))dlsym(h, "ncclReduce");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    commGetAsyncError = (decltype(commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    commAbort = (decltype(commAbort))dlsym(h, "ncclCommAbort");
    return getUniqueId && commInitRank && commSplit && broadcast && reduce && allReduce && commDestroy;
  }
};
NcclApi g_nccl;

struct DistState {
  ncclComm_t comm = nullptr;     // world
  ncclComm_t rowc = nullptr;     // my process row (Q ranks, rank index = q)
  ncclComm_t colc = nullptr;     // my process column (P ranks, rank index = p)
  int G = 0, P = 0, Q = 0, rank = -1;
};
DistState g_dist;

// number of block indices I in [0, x) with I % P == p (= the local index of the
// first such I >= x)
inline int64_t below(int64_t x, int P, int p) { return p < x ? (x - p + P - 1) / P : 0; }

struct Grid {
  int64_t n, T;
  int P, Q;
  int64_t R(int p) const { return below(T, P, p); }  // local block rows of process row p
  int64_t C(int q) const { return below(T, Q, q); }  // local block columns of process column q
};

// per-rank device scratch (doubles), laid out by DistPlan
struct DistPlan {
  size_t pan, cbuf, stage, dinv, dbuf, lrow, part, z, sbuf, tmp, total;
  size_t pan_sz = 0, cbuf_sz = 0, stage_sz = 0;  // forward: two sets (lookahead double buffering)
  size_t lrow_sz = 0;                             // adjoint: pan and lrow doubled likewise
};
DistPlan dist_plan(const Grid& gr, int p, int q, bool adjoint) {
  DistPlan d{};
  const size_t t2 = (size_t)DB * DB;
  size_t o = 0;
  auto take = [&](size_t cnt) {
    size_t at = o;
    o += (cnt + 31) / 32 * 32;  // 256-B aligned
    return at;
  };
  const int64_t R = gr.R(p), C = gr.C(q);
  auto a32 = [](size_t c) { return (c + 31) / 32 * 32; };
  if (!adjoint) {  // two buffer sets: panel k+1 is formed while panel k is consumed
    d.pan_sz = a32((R + 1) * t2);  // [L_kk | panel rows]
    d.cbuf_sz = a32(C * t2);  // L_Jk of every local block column (one GEMM per step)
    d.stage_sz = a32(gr.P > 1 ? (size_t)gr.P * (C + 1) * t2 : 0);
    d.pan = take(2 * d.pan_sz);
    d.cbuf = take(2 * d.cbuf_sz);
    d.stage = take(2 * d.stage_sz);
  } else {
    d.pan_sz = a32((R + 1) * t2);  // C_bar D^-1 rows (two sets: the side stream still reads step jb+1's)
    d.lrow_sz = a32(gr.P > 1 ? C * t2 : 0);
    d.pan = take(2 * d.pan_sz);
    d.dinv = take(C * t2);
    d.dbuf = take(t2);
    d.lrow = take(2 * d.lrow_sz);
    size_t part = 0;
    for (int64_t jb = gr.T - 1; jb >= 0; --jb) {
      const int64_t mloc = (R - below(jb + 1, gr.P, p)) * DB, w2 = below(jb + 1, gr.Q, q) * DB;
      if (mloc == 0 || w2 == 0) continue;
      int s, kps;
      splitk_choice(mloc, w2, DB, &s, &kps);
      part = std::max(part, (size_t)s * DB * w2);
    }
    d.part = take(part);
    d.z = take(gr.P > 1 ? C * t2 : 0);
    d.sbuf = take(t2);
    d.tmp = take(std::max<size_t>(4 * t2, (size_t)C * NB * NB));  // also the batched D^-1 scratch (NB^2 per tile)
  }
  d.total = o;
  return d;
}

// ranks handled by this process: one (NCCL) or all P*Q (simulation)
struct Rank {
  int p, q;
  const double* L;  // local factor (adjoint) -- or nullptr
  double* W;        // local working matrix
  int64_t ld;
  double* base;     // scratch arena (DistPlan offsets)
  DistPlan pl;
  int* status;
  double* at(size_t off) const { return base + off; }
  double* pan(int b) const { return base + pl.pan + b * pl.pan_sz; }
  double* cbuf(int b) const { return base + pl.cbuf + b * pl.cbuf_sz; }
  double* stage(int b) const { return base + pl.stage + b * pl.stage_sz; }
  double* lrow(int b) const { return base + pl.lrow + b * pl.lrow_sz; }
};

// Collective trace (stan_cl_dist_trace): when set, the real (one rank per
// process) path records each NCCL call it would issue -- communicator, op,
// root, count, stream -- in host issue order instead of calling NCCL.
struct TraceEntry {
  int64_t comm_kind;  // 0 = row communicator, 1 = column, 2 = world
  int64_t comm_index; // p for a row, q for a column, 0 for the world
  int64_t op;         // 0 = broadcast, 1 = reduce (sum), 2 = all-reduce (max)
  int64_t root;       // root's index within the communicator (-1: none)
  int64_t count;      // elements
  int64_t stream;     // 0 = library stream, 1 = side (lookahead) stream, 2 = other
};
std::vector<TraceEntry>* g_trace = nullptr;
int64_t stream_role(cudaStream_t st) { return st == g.stream ? 0 : (st == g.side ? 1 : 2); }

struct Comm {
  bool sim;
  int P, Q;
  Rank* find(std::vector<Rank>& rs, int p, int q) {
    for (auto& r : rs)
      if (r.p == p && r.q == q) return &r;
    return nullptr;
  }
  // broadcast `count` doubles within process row p (row = true) or process
  // column q (row = false) from the member with index `root` (q resp. p);
  // ptr(rank) names the buffer on each member (the root's holds the data)
  template <class F>
  int bcast(std::vector<Rank>& rs, bool row, int idx, int root, F ptr, size_t count, cudaStream_t st) {
    const int members = row ? Q : P;
    if (members == 1 || count == 0) return STAN_CL_OK;
    if (sim) {
      Rank* src = row ? find(rs, idx, root) : find(rs, root, idx);
      for (int m = 0; m < members; ++m) {
        if (m == root) continue;
        Rank* dst = row ? find(rs, idx, m) : find(rs, m, idx);
        CK(cudaMemcpyAsync(ptr(*dst), ptr(*src), count * sizeof(double), cudaMemcpyDeviceToDevice, st));
      }
      return STAN_CL_OK;
    }
    Rank& me = rs[0];
    if ((row ? me.p : me.q) != idx) return STAN_CL_OK;
    double* b = ptr(me);
    if (g_trace) {
      g_trace->push_back(TraceEntry{row ? 0 : 1, idx, 0, root, (int64_t)count, stream_role(st)});
      return STAN_CL_OK;
    }
    if (g_nccl.broadcast(b, b, count, ncclFloat64, root, row ? g_dist.rowc : g_dist.colc, st) != ncclSuccess)
      return STAN_CL_ENCCL;
    return STAN_CL_OK;
  }
  // sum over process column q into the member with index `root` (fixed order in
  // the simulation: root, then p = 0, 1, ...)
  template <class F>
  int col_reduce(std::vector<Rank>& rs, int q, int root, F ptr, size_t count, cudaStream_t st) {
    if (P == 1 || count == 0) return STAN_CL_OK;
    if (sim) {
      Rank* dst = find(rs, root, q);
      for (int m = 0; m < P; ++m) {
        if (m == root) continue;
        CK(add_block(ptr(*find(rs, m, q)), (int64_t)count, ptr(*dst), (int64_t)count, 1, (int64_t)count, st));
      }
      return STAN_CL_OK;
    }
    Rank& me = rs[0];
    if (me.q != q) return STAN_CL_OK;
    double* b = ptr(me);
    if (g_trace) {
      g_trace->push_back(TraceEntry{1, q, 1, root, (int64_t)count, stream_role(st)});
      return STAN_CL_OK;
    }
    if (g_nccl.reduce(b, b, count, ncclFloat64, ncclSum, root, g_dist.colc, st) != ncclSuccess) return STAN_CL_ENCCL;
    return STAN_CL_OK;
  }
};

#define RC(x)                   \
  do {                          \
    int rc_ = (x);              \
    if (rc_) return rc_;        \
  } while (0)

// forward phases (a)-(d) of step k into buffer set b, on stream st
int dist_panel(std::vector<Rank>& rs, const Grid& gr, Comm& cm, int64_t k, int b, cudaStream_t st) {
  const int64_t T = gr.T, t2 = DB * DB;
  const int P = gr.P, Q = gr.Q;
  const int64_t Lc = std::lcm((int64_t)P, (int64_t)Q);
  const int pk = (int)(k % P), qk = (int)(k % Q);
  const int64_t c0 = k * DB;
  // (a) L_kk = chol(A_kk) on the diagonal owner, in place, then into pan[0]
  for (auto& r : rs) {
    if (r.p != pk || r.q != qk) continue;
    double* tile = r.W + (k / P) * DB * r.ld + (k / Q) * DB;
    RC(panel(tile - c0 * r.ld - c0, r.ld, c0, c0 + DB, DB, r.status, st));  // view: rows [c0, c0 + DB)
    CK(copy_block(tile, r.ld, r.pan(b), DB, DB, DB, st));
  }
  RC(cm.bcast(rs, false, qk, pk, [b](Rank& r) { return r.pan(b); }, (size_t)t2, st));
  // (b) process column qk: L_Ik = A_Ik L_kk^-T for the local rows I > k
  //     (two 128-wide substitutions with the cross update, as the forward panel)
  for (auto& r : rs) {
    if (r.q != qk) continue;
    const int64_t li0 = below(k + 1, P, r.p), mloc = (gr.R(r.p) - li0) * DB;
    if (mloc == 0) continue;
    double* pan = r.pan(b);
    double* A = r.W + li0 * DB * r.ld + (k / Q) * DB;
    CK(copy_block(A, r.ld, pan + t2, DB, mloc, DB, st));
    CK(trsm_panel(pan, DB, 0, DB, DB + mloc, r.status, st));
    CK(gemm_full(true, true, (int)mloc, NB, NB, -1.0, 1, pan + t2, DB, pan + NB * DB, DB, pan + t2 + NB, DB,
                 r.status, st, 0, PROF_LOOKAHEAD, /*allow_persistent=*/false));
    CK(trsm_panel(pan, DB, NB, DB, DB + mloc, r.status, st));
    CK(copy_block(pan + t2, DB, A, r.ld, mloc, DB, st));
  }
  // (c) row broadcast of the panel rows along every process row
  for (int p = 0; p < P; ++p) {
    const int64_t mloc = (gr.R(p) - below(k + 1, P, p)) * DB;
    RC(cm.bcast(rs, true, p, qk, [b](Rank& r) { return r.pan(b) + DB * DB; }, (size_t)mloc * DB, st));
  }
  // (d0) own tiles: L_Jk with J % P == p, J % Q == q, J > k from the panel rows into
  //      the column buffer (slot J / Q), so the trailing update is one GEMM per step
  for (auto& r : rs) {
    int64_t J0 = -1;
    for (int64_t J = k + 1; J < std::min(T, k + 1 + Lc); ++J)
      if (J % P == r.p && J % Q == r.q) {
        J0 = J;
        break;
      }
    if (J0 < 0) continue;
    const int64_t cnt = (T - 1 - J0) / Lc + 1, li0 = below(k + 1, P, r.p);
    CK(copy_tiles(r.pan(b) + t2, J0 / P - li0, Lc / P, r.cbuf(b), J0 / Q, Lc / Q, cnt, t2, st));
  }
  // (d) column exchange (P > 1): rank (p', q) sends the tiles L_Jk, J > k,
  //     J % P == p', J % Q == q (J = J0 + t * lcm(P, Q)) to its process column
  if (P > 1) {
    for (int q = 0; q < Q; ++q) {
      for (int pp = 0; pp < P; ++pp) {
        int64_t J0 = -1;
        for (int64_t J = k + 1; J < std::min(T, k + 1 + Lc); ++J)
          if (J % P == pp && J % Q == q) {
            J0 = J;
            break;
          }
        if (J0 < 0) continue;
        const int64_t cnt = (T - 1 - J0) / Lc + 1;
        Rank* root = cm.sim ? cm.find(rs, pp, q) : (rs[0].p == pp && rs[0].q == q ? &rs[0] : nullptr);
        const size_t soff = (size_t)pp * (gr.C(q) + 1) * t2;
        if (root) {
          const int64_t li0 = below(k + 1, P, pp);
          CK(copy_tiles(root->pan(b) + t2, J0 / P - li0, Lc / P, root->stage(b) + soff, 0, 1, cnt, t2, st));
        }
        RC(cm.bcast(rs, false, q, pp, [soff, b](Rank& r) { return r.stage(b) + soff; }, (size_t)cnt * t2, st));
        for (auto& r : rs) {
          if (r.q != q || r.p == pp) continue;
          CK(copy_tiles(r.stage(b) + soff, 0, 1, r.cbuf(b), J0 / Q, Lc / Q, cnt, t2, st));
        }
      }
    }
  }
  return STAN_CL_OK;
}

// forward phase (e) of step k (buffer set b): A_IJ -= L_Ik L_Jk^T on the local
// lower tiles I >= J with J in [Jlo, Jhi): one block-cyclic-masked GEMM per rank
// (rows from the first local block row that reaches the first column's diagonal)
int dist_update(std::vector<Rank>& rs, const Grid& gr, int64_t k, int b, int64_t Jlo, int64_t Jhi, cudaStream_t st,
                int reserve) {
  const int64_t t2 = DB * DB;
  const int P = gr.P, Q = gr.Q;
  for (auto& r : rs) {
    const int64_t li0 = below(k + 1, P, r.p), R = gr.R(r.p);
    const int64_t lj_lo = below(Jlo, Q, r.q), lj_hi = below(Jhi, Q, r.q);
    if (lj_hi <= lj_lo) continue;
    const int64_t li_f = below(lj_lo * Q + r.q, P, r.p);  // first local block row with I >= J of column lj_lo
    if (li_f >= R) continue;
    CK(gemm_cyclic_lower((int)((R - li_f) * DB), (int)((lj_hi - lj_lo) * DB), (int)DB, r.pan(b) + t2 + (li_f - li0) * t2,
                         DB, r.cbuf(b) + lj_lo * t2, DB, r.W + li_f * DB * r.ld + lj_lo * DB, r.ld, P, r.p, Q, r.q,
                         (int)li_f, (int)lj_lo, r.status, st, reserve));
  }
  return STAN_CL_OK;
}

// Right-looking distributed forward with one step of lookahead: the panel of
// step k+1 (diagonal factorization, panel solve, row broadcasts, column
// exchange) runs on the high-priority side stream while the main stream
// applies the rest of step k's trailing update, which leaves SMs free for the
// panel kernels and the NCCL kernels.  Buffer sets alternate by step parity.
//   main: wait panel k; update block column k+1 (the ranks of column (k+1)%Q)
//   side: wait that; panel k+1
//   main: update block columns > k+1
int dist_factor(std::vector<Rank>& rs, const Grid& gr, Comm& cm) {
  cudaStream_t main = g.stream;
  const int64_t T = gr.T;
  RC(ensure_side(2 * T + 2));
  cudaStream_t side = g.side;
  cudaEvent_t* ev = g.events.data();  // ev[0]: start; ev[1 + 2k]: panel k done; ev[2 + 2k]: column k+1 updated
  // SMs the bulk update leaves to the panel (and, with several ranks, the NCCL) kernels
  const int kReserve = gr.P * gr.Q > 1 ? 16 : 8;
  CK(cudaEventRecord(ev[0], main));
  CK(cudaStreamWaitEvent(side, ev[0], 0));
  RC(dist_panel(rs, gr, cm, 0, 0, side));
  CK(cudaEventRecord(ev[1], side));
  for (int64_t k = 0; k < T; ++k) {
    const int b = (int)(k & 1);
    CK(cudaStreamWaitEvent(main, ev[1 + 2 * k], 0));
    if (k + 1 == T) break;
    RC(dist_update(rs, gr, k, b, k + 1, k + 2, main, 0));
    CK(cudaEventRecord(ev[2 + 2 * k], main));
    CK(cudaStreamWaitEvent(side, ev[2 + 2 * k], 0));
    RC(dist_panel(rs, gr, cm, k + 1, b ^ 1, side));
    CK(cudaEventRecord(ev[1 + 2 * (k + 1)], side));
    RC(dist_update(rs, gr, k, b, k + 2, T, main, kReserve));
  }
  const int P = gr.P, Q = gr.Q;
  for (auto& r : rs)  // strict upper of the local diagonal tiles
    for (int64_t J = 0; J < T; ++J)
      if (J % P == r.p && J % Q == r.q) {
        double* tile = r.W + (J / P) * DB * r.ld + (J / Q) * DB;
        CK(zero_tile_upper(tile, r.ld, 0, (int)DB, main));
      }
  return STAN_CL_OK;
}

// B_bar -= C_bar R on the local tiles I > jb with global block column J in
// [Jlo, Jhi) (C_bar D^-1 rows in pan(b); R = L's row block jb: local for P = 1,
// else the broadcast copy lrow(b))
int dist_r3(std::vector<Rank>& rs, const Grid& gr, int64_t jb, int b, int64_t Jlo, int64_t Jhi, cudaStream_t st,
            int reserve) {
  const int P = gr.P, Q = gr.Q;
  for (auto& r : rs) {
    const int64_t li0 = below(jb + 1, P, r.p), mloc = (gr.R(r.p) - li0) * DB;
    const int64_t lj0 = below(std::max<int64_t>(Jlo, 0), Q, r.q), lj1 = below(std::min(Jhi, jb), Q, r.q);
    if (mloc == 0 || lj1 <= lj0) continue;
    const int64_t w = below(jb, Q, r.q) * DB;  // width of the R row block held / broadcast
    const double* Rr = P > 1 ? r.lrow(b) : r.L + jb * DB * r.ld;
    const int64_t ldr = P > 1 ? w : r.ld;
    CK(gemm_full(true, false, (int)mloc, (int)((lj1 - lj0) * DB), (int)DB, -1.0, 1, r.pan(b), DB, Rr + lj0 * DB, ldr,
                 r.W + li0 * DB * r.ld + lj0 * DB, r.ld, r.status, st, 0, PROF_GEMM, true, reserve));
  }
  return STAN_CL_OK;
}

// Reverse sweep over 256-wide blocks with lookahead: the
// bulk of each step's B_bar update (the largest GEMM) runs on the side stream
// while the main stream goes on with the latency-bound chain (split-K product
// and its column reduce, the symbolic diagonal step, sym(S) broadcast, R_bar
// update, the next step's D^-1 / C_bar D^-1 broadcasts).  Per step jb (buffer
// set b = jb & 1):
//   main: [wait side done with set b (step jb+2)] D^-1 bcast; C_bar D^-1 -> pan(b);
//         row bcast; L row bcast -> lrow(b); [wait side's column jb-1 update of
//         step jb+1] B_bar(:, jb-1) -= ...; event A
//   side: wait A; B_bar(:, jb-2) -= ... ; event P1; B_bar(:, < jb-2) -= ...; event R(b)
//   main: split-K partials, column reduce, symbolic step, sym(S) bcast, R_bar update
// The column the next step's C_bar needs (jb-1) is updated on the main stream,
// the one after it (jb-2) first on the side stream, so no two updates of the same
// tiles are ever in flight together.
int dist_adjoint(std::vector<Rank>& rs, const Grid& gr, Comm& cm) {
  cudaStream_t st = g.stream;
  const int64_t T = gr.T, t2 = DB * DB;
  const int P = gr.P, Q = gr.Q;
  RC(ensure_side(8));
  // one rank: no collectives to hide, and the two streams' persistent GEMMs only
  // compete for SMs (measured 108 vs 95 ms at n = 16384 on a 1 x 1 grid), so the
  // bulk update then stays in stream order
  const bool overlap = P * Q > 1;
  cudaStream_t side = overlap ? g.side : st;
  cudaEvent_t* ev = g.events.data();  // 0: start; 1, 2: side done with set 0 / 1; 3: column jb-2 done; 4: main ready
  const int kReserve = overlap ? 16 : 0;  // SMs the side-stream bulk update leaves to the main-stream chain / NCCL
  for (int i = 0; i < 4; ++i) CK(cudaEventRecord(ev[i], st));
  CK(cudaStreamWaitEvent(side, ev[0], 0));
  auto ltile = [&](const Rank& r, const double* M, int64_t I, int64_t J) {  // local tile (I, J) of M
    return M + (I / P) * DB * r.ld + (J / Q) * DB;
  };
  // D^-1 of the owned diagonal tiles J = J0 + t lcm(P, Q) (slot t), one batched
  // call per rank (consecutive owned tiles are a constant local stride apart);
  // they depend only on L
  const int64_t Lc = std::lcm((int64_t)P, (int64_t)Q);
  auto first_diag = [&](const Rank& r) -> int64_t {
    for (int64_t J = 0; J < std::min(T, Lc); ++J)
      if (J % P == r.p && J % Q == r.q) return J;
    return -1;
  };
  for (auto& r : rs) {
    const int64_t J0 = first_diag(r);
    if (J0 < 0) continue;
    const int64_t cnt = (T - 1 - J0) / Lc + 1;
    const int64_t stride = (Lc / P) * DB * r.ld + (Lc / Q) * DB;
    const double* D = ltile(r, r.L, J0, J0);
    RC(block_inverses(D, r.ld, DB, 0, cnt, r.at(r.pl.dinv), r.at(r.pl.tmp), r.status, st, stride));
  }
  for (int64_t jb = T - 1; jb >= 0; --jb) {
    const int pj = (int)(jb % P), qj = (int)(jb % Q);
    const int b = (int)(jb & 1);
    auto dinv_of = [&](Rank& r) {
      return r.p == pj ? r.at(r.pl.dinv) + ((jb - first_diag(r)) / Lc) * t2 : r.at(r.pl.dbuf);
    };
    if (jb < T - 1) {
      CK(cudaStreamWaitEvent(st, ev[1 + b], 0));  // the side stream is done with pan(b) / lrow(b) of step jb+2
      // R1: C_bar <- C_bar D^-1 on process column qj (D^-1 broadcast down it)
      RC(cm.bcast(rs, false, qj, pj, dinv_of, (size_t)t2, st));
      for (auto& r : rs) {
        if (r.q != qj) continue;
        const int64_t li0 = below(jb + 1, P, r.p), mloc = (gr.R(r.p) - li0) * DB;
        if (mloc == 0) continue;
        double* Cb = r.W + li0 * DB * r.ld + (jb / Q) * DB;
        CK(gemm_full(true, false, (int)mloc, (int)DB, (int)DB, 1.0, 0, Cb, r.ld, dinv_of(r), DB, r.pan(b), DB,
                     r.status, st, 0, PROF_TRMM, true, 0, TRI_B_LOWER));
        CK(copy_block(r.pan(b), DB, Cb, r.ld, mloc, DB, st));
      }
      for (int p = 0; p < P; ++p) {
        const int64_t mloc = (gr.R(p) - below(jb + 1, P, p)) * DB;
        RC(cm.bcast(rs, true, p, qj, [b](Rank& r) { return r.pan(b); }, (size_t)mloc * DB, st));
      }
      // L's row block jb (columns J < jb) down every process column (P > 1)
      if (P > 1) {
        for (int q = 0; q < Q; ++q) {
          const int64_t w = below(jb, Q, q) * DB;
          if (w == 0) continue;
          for (auto& r : rs)
            if (r.p == pj && r.q == q) CK(copy_block(r.L + (jb / P) * DB * r.ld, r.ld, r.lrow(b), w, DB, w, st));
          RC(cm.bcast(rs, false, q, pj, [b](Rank& r) { return r.lrow(b); }, (size_t)DB * w, st));
        }
      }
      // R3 on column jb-1 here (the next step's C_bar), after the side stream's
      // update of that column from step jb+1; the rest on the side stream
      if (overlap) {
        CK(cudaStreamWaitEvent(st, ev[3], 0));
        RC(dist_r3(rs, gr, jb, b, jb - 1, jb, st, 0));
        CK(cudaEventRecord(ev[4], st));
        CK(cudaStreamWaitEvent(side, ev[4], 0));
        RC(dist_r3(rs, gr, jb, b, jb - 2, jb - 1, side, 0));
        CK(cudaEventRecord(ev[3], side));
        RC(dist_r3(rs, gr, jb, b, 0, jb - 2, side, kReserve));
        CK(cudaEventRecord(ev[1 + b], side));
      } else {
        RC(dist_r3(rs, gr, jb, b, 0, jb, st, 0));  // one launch, in stream order
      }
      // R2: [R_bar D_bar] -= C_bar^T [B C]: local split-K partials over the rows
      //     I > jb, reduced down each process column to the owner of row block jb
      //     (large-k product PAPER.md:172-174)
      for (auto& r : rs) {
        const int64_t li0 = below(jb + 1, P, r.p), mloc = (gr.R(r.p) - li0) * DB, w2 = below(jb + 1, Q, r.q) * DB;
        if (w2 == 0) continue;
        double* dst = P > 1 ? r.at(r.pl.z) : r.W + jb * DB * r.ld;
        const int64_t ldd = P > 1 ? w2 : r.ld;
        if (P > 1) CK(cudaMemsetAsync(dst, 0, (size_t)DB * w2 * sizeof(double), st));
        if (mloc == 0) continue;
        int splits, kps;
        splitk_choice(mloc, w2, DB, &splits, &kps);
        CK(gemm_splitk_tn((int)DB, (int)w2, (int)mloc, splits, kps, r.pan(b), DB, r.L + li0 * DB * r.ld, r.ld,
                          r.at(r.pl.part), r.status, st));
        CK(splitk_reduce_sub(r.at(r.pl.part), splits, (int)DB, (int)w2, dst, ldd, r.status, st));
      }
      if (P > 1) {
        for (int q = 0; q < Q; ++q) {
          const int64_t w2 = below(jb + 1, Q, q) * DB;
          if (w2 == 0) continue;
          RC(cm.col_reduce(rs, q, pj, [](Rank& r) { return r.at(r.pl.z); }, (size_t)DB * w2, st));
          for (auto& r : rs)
            if (r.p == pj && r.q == q)
              CK(add_block(r.at(r.pl.z), w2, r.W + (jb / P) * DB * r.ld, r.ld, DB, w2, st));
        }
      }
    }
    // R4: symbolic diagonal step on the owner -> sym(S) in sbuf
    for (auto& r : rs) {
      if (r.p != pj || r.q != qj) continue;
      const double* D = ltile(r, r.L, jb, jb);
      double* Dbar = r.W + (jb / P) * DB * r.ld + (jb / Q) * DB;
      const double* Di = r.at(r.pl.dinv) + ((jb - first_diag(r)) / Lc) * t2;
      double* T1 = r.at(r.pl.tmp);
      CK(adj_diag_fused((int)DB, D, r.ld, Dbar, r.ld, Di, T1, T1 + t2, T1 + 2 * t2, r.at(r.pl.sbuf),
                        (unsigned*)r.status + 16, r.status, st));
    }
    // R5: R_bar -= sym(S) R on process row pj
    RC(cm.bcast(rs, true, pj, qj, [](Rank& r) { return r.at(r.pl.sbuf); }, (size_t)t2, st));
    for (auto& r : rs) {
      if (r.p != pj) continue;
      const int64_t w = below(jb, Q, r.q) * DB;
      if (w == 0) continue;
      CK(gemm_full(true, false, (int)DB, (int)w, (int)DB, -1.0, 1, r.at(r.pl.sbuf), DB, r.L + (jb / P) * DB * r.ld,
                   r.ld, r.W + (jb / P) * DB * r.ld, r.ld, r.status, st));
    }
  }
  // join: the last side-stream updates
  CK(cudaStreamWaitEvent(st, ev[1], 0));
  CK(cudaStreamWaitEvent(st, ev[2], 0));
  return STAN_CL_OK;
}

// nloc ranks in this process: all P*Q (sim) or the one at (p0, q0)
int dist_run(bool adjoint, int64_t n, int P, int Q, bool sim, int p0, int q0, const double* const* Ls,
             double* const* Ws, int64_t ld) {
  if (n == 0) return STAN_CL_OK;
  if (n < 0 || n % DB != 0 || P < 1 || Q < 1 || ld < 1) return STAN_CL_EINVAL;
  const Grid gr{n, n / DB, P, Q};
  const int nloc = sim ? P * Q : 1;
  std::vector<DistPlan> plans;
  size_t total = 0;
  for (int i = 0; i < nloc; ++i) {
    const int p = sim ? i / Q : p0, q = sim ? i % Q : q0;
    const bool owns = gr.R(p) > 0 && gr.C(q) > 0;  // a rank of a grid larger than the tile count may own none
    if (owns && (!Ws[i] || (adjoint && !Ls[i]))) return STAN_CL_EINVAL;
    if (gr.C(q) > 0 && ld < gr.C(q) * DB) return STAN_CL_EINVAL;
    plans.push_back(dist_plan(gr, p, q, adjoint));
    total += plans.back().total;
  }
  double* buf = nullptr;
  int rc = ensure_ws(al(sizeof(int) * 64) + NB * NB * sizeof(double));
  if (rc) return rc;
  rc = ensure_mat(0, std::max<size_t>(total, 1) * sizeof(double), &buf);
  if (rc) return rc;
  int* status = (int*)g.ws;
  CK(cudaMemsetAsync(status, 0, sizeof(int), g.stream));
  std::vector<Rank> rs;
  size_t off = 0;
  for (int i = 0; i < nloc; ++i) {
    const int p = sim ? i / Q : p0, q = sim ? i % Q : q0;
    rs.push_back(Rank{p, q, adjoint ? Ls[i] : nullptr, Ws[i], ld, buf + off, plans[i], status});
    off += plans[i].total;
  }
  if (adjoint)  // A_bar <- tril(L_bar): strict upper of the local diagonal tiles
    for (auto& r : rs)
      for (int64_t J = 0; J < gr.T; ++J)
        if (J % P == r.p && J % Q == r.q)
          CK(zero_tile_upper(r.W + (J / P) * DB * r.ld + (J / Q) * DB, r.ld, 0, (int)DB, g.stream));
  Comm cm{sim, P, Q};
  return adjoint ? dist_adjoint(rs, gr, cm) : dist_factor(rs, gr, cm);
}

}  // namespace

extern "C" {

int stan_cl_dist_get_unique_id(void* out128) {
  if (!out128) return STAN_CL_EINVAL;
  if (!g_nccl.load()) return STAN_CL_ENCCL;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return STAN_CL_ENCCL;
  memcpy(out128, &id, sizeof(id));
  return STAN_CL_OK;
}

int stan_cl_dist_init(int nranks, int rank, const void* id128, int P, int Q) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !id128 || P < 1 || Q < 1 || P * Q != nranks)
    return STAN_CL_EINVAL;
  if (!g_nccl.load()) return STAN_CL_ENCCL;
  if (g_dist.comm) return STAN_CL_EINVAL;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  if (g_nccl.commInitRank(&g_dist.comm, nranks, id, rank) != ncclSuccess) {
    g_dist.comm = nullptr;
    return STAN_CL_ENCCL;
  }
  const int p = rank / Q, q = rank % Q;
  // row communicator: same p, ordered by q; column communicator: same q, ordered by p
  if (g_nccl.commSplit(g_dist.comm, p, q, &g_dist.rowc, nullptr) != ncclSuccess ||
      g_nccl.commSplit(g_dist.comm, q, p, &g_dist.colc, nullptr) != ncclSuccess) {
    if (g_dist.rowc) g_nccl.commDestroy(g_dist.rowc);
    g_nccl.commDestroy(g_dist.comm);
    g_dist = DistState{};
    return STAN_CL_ENCCL;
  }
  g_dist.G = nranks;
  g_dist.P = P;
  g_dist.Q = Q;
  g_dist.rank = rank;
  return STAN_CL_OK;
}

// abort every communicator of the grid (after an asynchronous NCCL error or a
// timeout: a peer died or stopped issuing collectives); the grid must be
// re-initialised with stan_cl_dist_init
static void dist_abort(const char* why) {
  snprintf(g.last_err, sizeof(g.last_err), "NCCL: %s; communicators aborted", why);
  for (ncclComm_t* c : {&g_dist.rowc, &g_dist.colc, &g_dist.comm}) {
    if (*c) {
      if (g_nccl.commAbort) g_nccl.commAbort(*c);
      *c = nullptr;
    }
  }
  g_dist = DistState{};
}

// wait for the library stream while watching the communicators: returns
// STAN_CL_ENCCL (after aborting them) on an asynchronous NCCL error or when the
// stream has not drained within STAN_CL_NCCL_TIMEOUT_S seconds (default 1800;
// 0 = wait forever), instead of hanging in cudaStreamSynchronize
static int dist_wait() {
  static const double timeout_s = [] {
    const char* e = getenv("STAN_CL_NCCL_TIMEOUT_S");
    return e ? atof(e) : 1800.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned it = 0;; ++it) {
    const cudaError_t e = cudaStreamQuery(g.stream);
    if (e == cudaSuccess) return STAN_CL_OK;
    if (e != cudaErrorNotReady) return cuda_fail(e, "dist_wait");
    if (g_nccl.commGetAsyncError) {
      for (ncclComm_t c : {g_dist.comm, g_dist.rowc, g_dist.colc}) {
        ncclResult_t r = ncclSuccess;
        if (c && g_nccl.commGetAsyncError(c, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress) {
          dist_abort("asynchronous error");
          return STAN_CL_ENCCL;
        }
      }
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_s > 0 && el > timeout_s) {
      dist_abort("timeout waiting for the collectives");
      return STAN_CL_ENCCL;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(it < 1000 ? 20 : 500));
  }
}

static int dist_status_allreduce(int rc) {
  if (rc) return rc;
  // "did anything fail": status words are 0 or row+1; the max is a failing row
  int* status = (int*)g.ws;
  if (g_nccl.allReduce(status, status, 1, ncclInt32, ncclMax, g_dist.comm, g.stream) != ncclSuccess)
    return STAN_CL_ENCCL;
  if ((rc = dist_wait())) return rc;
  return read_status();
}

int stan_cl_dist_cholesky(int64_t n, int nb, double* A_local, int64_t ld_local) {
  CallScope call_("stan_cl_dist_cholesky");
  if (!g_dist.comm || (nb != 0 && nb != (int)DB)) return STAN_CL_EINVAL;
  double* Ws[1] = {A_local};
  const int p = g_dist.rank / g_dist.Q, q = g_dist.rank % g_dist.Q;
  int rc = dist_run(false, n, g_dist.P, g_dist.Q, false, p, q, nullptr, Ws, ld_local);
  return n == 0 ? rc : dist_status_allreduce(rc);
}

int stan_cl_dist_cholesky_adjoint(int64_t n, int nb, const double* L_local, double* Lbar_to_Abar_local,
                                  int64_t ld_local) {
  CallScope call_("stan_cl_dist_cholesky_adjoint");
  if (!g_dist.comm || (nb != 0 && nb != (int)DB)) return STAN_CL_EINVAL;
  const double* Ls[1] = {L_local};
  double* Ws[1] = {Lbar_to_Abar_local};
  const int p = g_dist.rank / g_dist.Q, q = g_dist.rank % g_dist.Q;
  int rc = dist_run(true, n, g_dist.P, g_dist.Q, false, p, q, Ls, Ws, ld_local);
  return n == 0 ? rc : dist_status_allreduce(rc);
}

int stan_cl_dist_trace(int64_t n, int P, int Q, int p, int q, int adjoint, const double* L_local,
                       double* A_local, int64_t ld_local, int64_t* out, int64_t max_entries) {
  CallScope call_("stan_cl_dist_trace");
  if (P < 1 || Q < 1 || p < 0 || p >= P || q < 0 || q >= Q || max_entries < 0 || (max_entries && !out))
    return STAN_CL_EINVAL;
  std::vector<TraceEntry> tr;
  g_trace = &tr;
  const double* Ls[1] = {L_local};
  double* Ws[1] = {A_local};
  int rc = dist_run(adjoint != 0, n, P, Q, false, p, q, adjoint ? Ls : nullptr, Ws, ld_local);
  g_trace = nullptr;
  if (rc) return rc;
  if (n > 0) tr.push_back(TraceEntry{2, 0, 2, -1, 1, 0});  // dist_status_allreduce
  CK(cudaStreamSynchronize(g.stream));
  const int64_t m = std::min<int64_t>((int64_t)tr.size(), max_entries);
  for (int64_t i = 0; i < m; ++i) memcpy(out + 6 * i, &tr[i], sizeof(TraceEntry));
  return (int)tr.size();
}

int stan_cl_dist_finalize(void) {
  if (g_dist.rowc) g_nccl.commDestroy(g_dist.rowc);
  if (g_dist.colc) g_nccl.commDestroy(g_dist.colc);
  if (g_dist.comm) g_nccl.commDestroy(g_dist.comm);
  g_dist = DistState{};
  return STAN_CL_OK;
}

int stan_cl_gp_exp_quad_cov_tiles(int64_t n, const double* x, double alpha, double rho, double jitter,
                                  double* K_local, int64_t ld_local, int P, int Q, int p, int q) {
  if (n < 0 || P < 1 || Q < 1 || p < 0 || p >= P || q < 0 || q >= Q || n % DB != 0) return STAN_CL_EINVAL;
  if (n == 0) return STAN_CL_OK;
  if (!x || !K_local) return STAN_CL_EINVAL;
  if (!(rho != 0.0) || !(rho - rho == 0.0)) return STAN_CL_EINVAL;
  if (ld_local < below(n / DB, Q, q) * DB) return STAN_CL_EINVAL;
  CK(se_cov_tiles(n, x, alpha, rho, jitter, K_local, ld_local, P, Q, p, q, g.stream));
  return STAN_CL_OK;
}

int stan_cl_gp_exp_quad_cov_cols(int64_t n, const double* x, double alpha, double rho, double jitter,
                                 double* K_local, int64_t ld_local, int G, int q) {
  return stan_cl_gp_exp_quad_cov_tiles(n, x, alpha, rho, jitter, K_local, ld_local, 1, G, 0, q);
}

int stan_cl_dist_sim2_cholesky(int64_t n, int P, int Q, double* const* A_locals, int64_t ld_local) {
  CallScope call_("stan_cl_dist_sim2_cholesky");
  if (!A_locals || P < 1 || Q < 1) return STAN_CL_EINVAL;
  int rc = dist_run(false, n, P, Q, true, 0, 0, nullptr, A_locals, ld_local);
  return (rc || n == 0) ? rc : read_status();
}

int stan_cl_dist_sim2_cholesky_adjoint(int64_t n, int P, int Q, const double* const* L_locals,
                                       double* const* W_locals, int64_t ld_local) {
  CallScope call_("stan_cl_dist_sim2_cholesky_adjoint");
  if (!L_locals || !W_locals || P < 1 || Q < 1) return STAN_CL_EINVAL;
  int rc = dist_run(true, n, P, Q, true, 0, 0, L_locals, W_locals, ld_local);
  return (rc || n == 0) ? rc : read_status();
}

int stan_cl_dist_sim_cholesky(int64_t n, int G, double* const* A_locals, int64_t ld_local) {
  return stan_cl_dist_sim2_cholesky(n, 1, G, A_locals, ld_local);
}

int stan_cl_dist_sim_cholesky_adjoint(int64_t n, int G, const double* const* L_locals, double* const* W_locals,
                                      int64_t ld_local) {
  return stan_cl_dist_sim2_cholesky_adjoint(n, 1, G, L_locals, W_locals, ld_local);
}

}  // extern "C"
