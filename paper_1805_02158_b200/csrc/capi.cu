// C ABI + native runtime: context, RED problem setup, device-resident solve
// schedule (solvers.py:288-399 re-expressed as a static kernel schedule with
// per-image masks), and the window-level VE entry point.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/redve_b200.h"
#include "kernels.cuh"
#include "rd.cuh"
#include "slab.cuh"
#include "sr.cuh"
#include "grad.cuh"
#include "spectral.cuh"
#include <cufft.h>

using namespace redve;

// Device-memory cache: problems are created per solve by the drop-in API, so
// their buffers (ring, spectra, traces ...) are recycled instead of going
// through cudaMalloc/cudaFree (which synchronise the device) every time.
struct MemPool {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free_blocks;  // (device, bytes) -> ptr
  static size_t round(size_t b) {
    const size_t g = b >= (1u << 20) ? (1u << 20) : 4096;
    return (b + g - 1) / g * g;
  }
  cudaError_t get(void** p, size_t bytes, size_t* got) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_blocks.lower_bound({dev, bytes});
      if (it != free_blocks.end() && it->first.first == dev && it->first.second <= 2 * bytes) {
        *p = it->second;
        *got = it->first.second;
        free_blocks.erase(it);
        return cudaSuccess;
      }
    }
    *got = bytes;
    return cudaMalloc(p, bytes);
  }
  void put(void* p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    free_blocks.insert({{dev, bytes}, p});
  }
  void release() {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& kv : free_blocks) cudaFree(kv.second);
    free_blocks.clear();
  }
};
static MemPool g_pool;

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;   // usable bytes requested
  size_t cap = 0; // bytes of the pooled block
  ~DevBuf() {
    if (p) g_pool.put(p, cap);
  }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) {
      n = bytes;
      return cudaSuccess;
    }
    if (p) g_pool.put(p, cap);
    p = nullptr;
    n = cap = 0;
    const size_t want = MemPool::round(bytes > 0 ? bytes : 16);
    size_t got = 0;
    cudaError_t e = g_pool.get(&p, want, &got);
    if (e == cudaSuccess) {
      n = bytes;
      cap = got;
    }
    return e;
  }
  template <class T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

static std::atomic<unsigned long long> g_launches{0};

struct ProfEvent {
  const char* name;
  cudaEvent_t a, b;
};

// A captured solve schedule.  Instantiated graphs are kept per context by
// topology (everything but buffer addresses): a problem of the same shape and
// configuration re-captures and UPDATES the instantiated graph in place
// (cudaGraphExecUpdate) instead of instantiating ~750 nodes again.  `owner` is
// the full key (problem serial + buffer addresses) the executable holds now.
struct GraphSlot {
  cudaGraphExec_t exec = nullptr;
  std::string owner;
  unsigned long long launches = 0;
};
static std::atomic<unsigned long long> g_problem_serial{0};

struct redve_ctx {
  bool profiling = false;
  std::map<std::string, GraphSlot> graphs;  // topology key -> executable graph
  void* hstage = nullptr;                   // pinned staging for trace read-back
  size_t hstage_bytes = 0;
  cudaStream_t cap_stream = nullptr;  // graph capture
  cudaEvent_t fork_ev = nullptr;
  std::vector<ProfEvent> prof;
  std::vector<cudaEvent_t> ev_pool;
  int device = 0;
  cudaStream_t stream = 0;
  std::string err;
  std::map<int, DevBuf*> twiddles, stage_twiddles;
  DevBuf scratch_taps, scratch_a, scratch_b, ve_ring, ve_state, ve_partials, ve_counters,
      ve_q, ve_trace;
  std::vector<double> taps_host;  // what scratch_taps holds (skip identical re-uploads)
  void* taps_dev = nullptr;
  bool taps_sep = false;          // scratch_taps is followed by the rank-one [u | v]
  // cuFFT plans by (H, W, batch), shared by the context's problems: a plan
  // costs milliseconds to create, a RedBatch per call must not pay it again
  std::map<std::tuple<int, int, int>, cufftHandle> fft_plans;
  ~redve_ctx() {
    for (auto& kv : fft_plans) cufftDestroy(kv.second);
    for (auto& kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (hstage) cudaFreeHost(hstage);
    for (auto& kv : twiddles) delete kv.second;
    for (auto& kv : stage_twiddles) delete kv.second;
    for (auto& e : prof) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    for (auto e : ev_pool) cudaEventDestroy(e);
  }
  cudaEvent_t ev() {
    cudaEvent_t e;
    if (!ev_pool.empty()) {
      e = ev_pool.back();
      ev_pool.pop_back();
    } else {
      cudaEventCreate(&e);
    }
    return e;
  }
  const cd* tws(int L) {  // stage-major table for compile-time plans
    if (!(L == 64 || L == 128 || L == 256 || L == 512 || L == 1024)) return nullptr;
    auto it = stage_twiddles.find(L);
    if (it != stage_twiddles.end()) return it->second->as<cd>();
    DevBuf* b = new DevBuf();
    if (b->ensure(sizeof(cd) * tw_stage_size(L)) != cudaSuccess) {
      delete b;
      return nullptr;
    }
    launch_stage_twiddles(b->as<cd>(), L, stream);
    g_launches.fetch_add(1);
    stage_twiddles[L] = b;
    return b->as<cd>();
  }
  const cd* tw(int L) {
    auto it = twiddles.find(L);
    if (it != twiddles.end()) return it->second->as<cd>();
    DevBuf* b = new DevBuf();
    if (b->ensure(sizeof(cd) * L) != cudaSuccess) {
      delete b;
      return nullptr;
    }
    launch_twiddles(b->as<cd>(), L, stream);
    g_launches.fetch_add(1);
    twiddles[L] = b;
    return b->as<cd>();
  }
};

static int fail(redve_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(ctx, REDVE_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_));      \
  } while (0)

// Every kernel launch goes through RUN: counts it and, when profiling, brackets
// it with CUDA events on the launching stream.
#define RUN(ctx_, name_, call_)                                                     \
  do {                                                                              \
    redve_ctx* c_ = (ctx_);                                                         \
    cudaEvent_t a_ = nullptr, b_ = nullptr;                                         \
    if (c_ && c_->profiling) {                                                      \
      a_ = c_->ev();                                                                \
      b_ = c_->ev();                                                                \
      cudaEventRecord(a_, c_->stream);                                              \
    }                                                                               \
    call_;                                                                          \
    g_launches.fetch_add(1, std::memory_order_relaxed);                             \
    if (a_) {                                                                       \
      cudaEventRecord(b_, c_->stream);                                              \
      c_->prof.push_back(ProfEvent{name_, a_, b_});                                 \
    }                                                                               \
  } while (0)

#define CKL()                                                                       \
  do {                                                                              \
    cudaError_t e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess)                                                          \
      return fail(ctx, REDVE_E_CUDA, "kernel launch: %s", cudaGetErrorString(e_));  \
  } while (0)

static int is_odd_pos(int k) { return k >= 1 && (k & 1); }

static bool graphs_enabled() {
  const char* e = getenv("REDVE_GRAPHS");
  return !(e && e[0] == '0');
}

// ------------------------------------------------------------------ problem
struct redve_problem {
  redve_ctx* ctx;
  int B, H, W, Hy, Wy, npairs;
  long long N;
  redve_operator_desc op;
  int dn_kind;
  int dn_ksize;
  double sigma, alpha;
  bool fourier;
  int lpc_row, lpc_col;
  int separable = 0;
  DevBuf hsep;  // [u | v] when the PSF is rank one
  int dn_api_kind = 0;  // REDVE_DN_* as requested
  int pw_pr = 1, pw_sr = 3, pw_iters = 20, pw_npos = 24;
  double pw_h = 110.0;
  int pw_w32 = 0;
  DevBuf w0, D0, D1, cgst, cr, cp, cq, cnt_cg, cnt_rec, part_cg;
  unsigned long long serial = ++g_problem_serial;  // never reused (graph ownership)
  unsigned long long captures = 0;  // graph (re)captures, for tests
  DevBuf x0bad;                     // device flag: x0 had a non-finite entry
  // gradient baselines: H^T H / sigma^2 stencil taps (circulant H), Nesterov y
  DevBuf gtaps, ybuf, part_grad, cnt_grad;
  int g_R = 0, g_sep = 0;
  // spectral route (linear denoisers): constant spectra, DFT staging, plans
  DevBuf sp_m, sp_hh, sp_wr, sp_xb, sp_yh, sp_rh, sp_stage, sp_part, sp_cnt;
  bool sp_ready = false;
  cufftHandle sp_plan = 0, sp_plan1 = 0;  // batch B / batch 1, [H][W] complex (ctx-owned)
  // CG fixed-point steps as graphs with a device-decided WHILE loop, keyed by
  // their views / phase / f buffer
  std::map<std::string, cudaGraphExec_t> cg_graphs;
  cudaStream_t cg_body_stream = nullptr;
  ~redve_problem() {
    for (auto& kv : cg_graphs) cudaGraphExecDestroy(kv.second);
    if (cg_body_stream) cudaStreamDestroy(cg_body_stream);
  }

  int rd_nf = 0, rd_fs = 0;
  double rd_tau = 0.0;
  DevBuf rd_filters, rd_scales;
  DevBuf htaps, dntaps, y, ref, hty, xb, g, Z, state, partials, cnt_inv, cnt_cost, cnt_ve,
      fbuf, ring, best, q, trace, vals;
  // Fourier-route cost identity: f(x_{k-1}) of cadence steps, second f buffer
  // for the precomputed denoisers, ||y||^2 per image
  DevBuf fprev, fcur, yy;
  bool has_ref = false;
  const cd* twH = nullptr;
  const cd* twW = nullptr;
  const cd* twsH = nullptr;
  const cd* twsW = nullptr;
  int ring_S = 0;
};

static DenoiseArgs dn_args(const redve_problem* p) {
  DenoiseArgs d;
  d.kind = p->dn_kind;
  d.ksize = p->dn_kind == DN_CONV ? p->dn_ksize : 0;
  d.radius = p->dn_kind == DN_CONV ? p->dn_ksize / 2 : (p->dn_kind == DN_MEDIAN3 ? 1 : 0);
  d.taps = p->dntaps.as<double>();
  return d;
}

static int lines_per_cta(int L) {
  int T = threads_per_line(L);
  int lpc = 128 / T;
  return lpc < 1 ? 1 : lpc;
}

static int col_lines_per_cta(int H, int W) {
  int T = threads_per_line(H);
  int lpc = 128 / T;
  if (lpc > 16) lpc = 16;
  if (lpc < 1) lpc = 1;
  return lpc;
}

static int map_dn_kind(int k) {
  switch (k) {
    case REDVE_DN_IDENTITY: return DN_IDENTITY;
    case REDVE_DN_CONV: return DN_CONV;
    case REDVE_DN_MEDIAN3: return DN_MEDIAN3;
    default: return DN_EXTERNAL;
  }
}

// Fourier solve pipeline on pairs: Z <- rowfwd(xin) ; col(scale) ; rowinv -> out
// The three Fourier kernels as separate pieces.
static int f_row_fwd(redve_problem* p, View xin, DenoiseArgs dn, cd* Z, int phase,
                     double* fout = nullptr) {
  redve_ctx* ctx = p->ctx;
  RowFwdArgs rf{p->B, p->H, p->W, p->lpc_row, xin, dn, Z, p->twW, p->twsW,
                p->state.as<ImgState>(), phase, fout};
  RUN(ctx, "row_fwd", launch_row_fwd(rf, p->npairs, ctx->stream));
  CKL();
  return REDVE_OK;
}
static int f_col(redve_problem* p, cd* Z, double scale, int phase) {
  redve_ctx* ctx = p->ctx;
  ColArgs ca{p->B, p->H, p->W, p->lpc_col, Z, p->twH, p->twsH, p->g.as<double>(),
             scale, p->state.as<ImgState>(), phase};
  RUN(ctx, "col", launch_col(ca, p->npairs, ctx->stream));
  CKL();
  return REDVE_OK;
}
static int f_row_inv(redve_problem* p, const cd* Z, View out, const double* base, int epilogue,
                     View xprev, StepCtl ctl, TraceBufs tr, int S) {
  redve_ctx* ctx = p->ctx;
  RowInvArgs ri;
  ri.B = p->B; ri.H = p->H; ri.W = p->W; ri.lpc = p->lpc_row;
  ri.Z = Z; ri.tw = p->twW; ri.tws = p->twsW; ri.out = out; ri.base = base; ri.xprev = xprev;
  ri.epilogue = epilogue; ri.S = S; ri.st = p->state.as<ImgState>(); ri.ctl = ctl; ri.tr = tr;
  ri.partials = p->partials.as<double>(); ri.counters = p->cnt_inv.as<unsigned>();
  RUN(ctx, "row_inv", launch_row_inv(ri, p->npairs, ctx->stream));
  CKL();
  return REDVE_OK;
}
static int fourier_pipeline(redve_problem* p, View xin, DenoiseArgs dn, double scale, View out,
                            const double* base, int epilogue, View xprev, StepCtl ctl,
                            TraceBufs tr, int S, int phase, double* fout = nullptr) {
  int r = f_row_fwd(p, xin, dn, p->Z.as<cd>(), phase, fout);
  if (r) return r;
  if ((r = f_col(p, p->Z.as<cd>(), scale, phase))) return r;
  return f_row_inv(p, p->Z.as<cd>(), out, base, epilogue, xprev, ctl, tr, S);
}

static View plain(const double* base, long long N) {
  View v;
  v.base = const_cast<double*>(base);
  v.img_stride = N;
  v.slot_stride = 0;
  v.S = 1;
  v.mode = 0;
  return v;
}

// f(x) into p->fbuf for the device denoisers the Fourier kernels do not fuse
// (PatchWeighted always; the stencils on the CG route).
static int denoise_to_fbuf(redve_problem* p, View x, int phase, double* out = nullptr) {
  redve_ctx* ctx = p->ctx;
  double* fdst = out ? out : p->fbuf.as<double>();
  if (p->dn_api_kind == REDVE_DN_FILTERBANK) {
    RdArgs a;
    a.B = p->B; a.H = p->H; a.W = p->W; a.nf = p->rd_nf; a.fs = p->rd_fs;
    a.filters = p->rd_filters.as<double>(); a.scales = p->rd_scales.as<double>(); a.tau = p->rd_tau;
    a.xin = x; a.out = fdst; a.st = p->state.as<ImgState>(); a.phase = phase;
    RUN(ctx, "filter_bank", launch_rd(a, ctx->stream));
  } else if (p->dn_api_kind == REDVE_DN_PATCH) {
    PwArgs a;
    a.B = p->B; a.H = p->H; a.W = p->W;
    a.pr = p->pw_pr; a.sr = p->pw_sr; a.npos = p->pw_npos; a.iters = p->pw_iters;
    a.inv_h2 = 1.0 / (p->pw_h * p->pw_h);
    a.xin = x;
    a.w0 = p->w0.as<double>(); a.w32 = p->pw_w32;
    a.D0 = p->D0.as<double>(); a.D1 = p->D1.as<double>();
    a.out = fdst;
    a.st = p->state.as<ImgState>(); a.phase = phase;
    int n = 0;
    RUN(ctx, "patch_weighted", launch_pw(a, ctx->stream, &n));
    g_launches.fetch_add(n - 1);
  } else {
    RUN(ctx, "denoise", launch_denoise_view(x, dn_args(p), fdst,
                                            p->state.as<ImgState>(), phase, p->B, p->H, p->W,
                                            ctx->stream));
  }
  CKL();
  return REDVE_OK;
}

static int cg_any_active(redve_problem* p, std::vector<CgState>& h) {
  redve_ctx* ctx = p->ctx;
  h.resize(p->B);
  CK(cudaMemcpyAsync(h.data(), p->cgst.p, sizeof(CgState) * p->B, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int b = 0; b < p->B; ++b)
    if (h[b].active) return 1;
  return 0;
}

// The CG solve of one fixed-point step as a graph: init (pre-check), then a
// WHILE node whose body is one CG iteration plus the device test "any image
// still active" (k_cg_continue sets the loop condition), then the b == 0 and
// maxiter residual epilogues.  No host round trip inside the solve.
static int cg_graph_build(redve_problem* p, const CgArgs& a, const CgArgs& rres,
                          cudaGraphExec_t* out) {
  redve_ctx* ctx = p->ctx;
  if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  if (!p->cg_body_stream) CK(cudaStreamCreateWithFlags(&p->cg_body_stream, cudaStreamNonBlocking));
  const cudaStream_t cs = ctx->cap_stream, bs = p->cg_body_stream;
  cudaGraph_t g = nullptr;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
  CK(cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  launch_cg_init(a, cs);
  launch_cg_continue(a, h, cs);
  cudaStreamCaptureStatus st;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(cs, &st, nullptr, nullptr, &deps, &nd);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode = nullptr;
  if (e == cudaSuccess) e = cudaGraphAddNode(&cnode, g, deps, nd, &cp);
  if (e == cudaSuccess)
    e = cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies);
  if (e == cudaSuccess) {
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      launch_cg_iter(a, bs);
      launch_cg_update(a, bs);
      launch_cg_continue(a, h, bs);
      cudaGraph_t body_out = nullptr;
      e = cudaStreamEndCapture(bs, &body_out);
    }
  }
  launch_cg_zero_b(a, cs);
  launch_cg_resid(rres, cs);
  cudaGraph_t gout = nullptr;
  const cudaError_t e2 = cudaStreamEndCapture(cs, &gout);
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, REDVE_E_CUDA, "CG graph: %s", cudaGetErrorString(e));
  }
  return REDVE_OK;
}

// One CG fixed-point step (objective.py:105-121, scipy cg semantics) from xin
// into xout; f_ext overrides the device denoiser (host plug-in).
static int fp_step_cg(redve_problem* p, View xin, View xout, int phase, const double* f_ext) {
  redve_ctx* ctx = p->ctx;
  const cudaStream_t s = ctx->stream;
  if (!f_ext) {
    int r = denoise_to_fbuf(p, xin, phase);
    if (r) return r;
  }
  CgArgs a;
  memset(&a, 0, sizeof(a));
  a.B = p->B; a.H = p->H; a.W = p->W; a.factor = p->op.factor; a.k = p->op.ksize;
  a.taps = p->htaps.as<double>();
  a.inv_sigma2 = 1.0 / (p->sigma * p->sigma); a.alpha = p->alpha;
  a.rtol = 1e-6; a.abort = 1e-4; a.maxiter = 200;  // objective.py:35-37
  a.row0 = 0; a.Hg = 0;
  a.huv = p->separable ? p->hsep.as<double>() : nullptr;
  a.xin = xin; a.xout = xout;
  a.hty = p->hty.as<double>(); a.f = f_ext ? f_ext : p->fbuf.as<double>();
  a.r = p->cr.as<double>(); a.p = p->cp.as<double>(); a.q = p->cq.as<double>();
  a.cg = p->cgst.as<CgState>(); a.st = p->state.as<ImgState>(); a.phase = phase;
  a.partials = p->part_cg.as<double>(); a.counters = p->cnt_cg.as<unsigned>();
  CgArgs rres = a;
  rres.xin = xout;
  if (!ctx->profiling && graphs_enabled()) {
    char key[256];
    snprintf(key, sizeof(key), "%p|%lld|%lld|%d|%d|%p|%lld|%lld|%d|%d|%d|%p", (void*)xin.base,
             xin.img_stride, xin.slot_stride, xin.S, xin.mode, (void*)xout.base,
             xout.img_stride, xout.slot_stride, xout.S, xout.mode, phase, (const void*)a.f);
    auto it = p->cg_graphs.find(key);
    if (it == p->cg_graphs.end()) {
      cudaGraphExec_t ge = nullptr;
      int r = cg_graph_build(p, a, rres, &ge);
      if (r) return r;
      it = p->cg_graphs.emplace(key, ge).first;
    }
    CK(cudaGraphLaunch(it->second, s));
    g_launches.fetch_add(4);  // init, continue, zero_b, resid (+3 per CG iteration)
    return REDVE_OK;
  }
  // profiling: the same kernels launched one by one (per-kernel events), the
  // loop test read back every 2 iterations
  RUN(ctx, "cg_init", launch_cg_init(a, s));
  CKL();
  std::vector<CgState> h;
  for (int it = 0; it < a.maxiter; ++it) {
    if (it % 2 == 0) {
      int any = cg_any_active(p, h);
      if (any > 1) return any;
      if (!any) break;
    }
    RUN(ctx, "cg_matvec", launch_cg_iter(a, s));
    RUN(ctx, "cg_update", launch_cg_update(a, s));
    CKL();
  }
  RUN(ctx, "cg_zero_b", launch_cg_zero_b(a, s));
  RUN(ctx, "cg_resid", launch_cg_resid(rres, s));
  CKL();
  return REDVE_OK;
}

extern "C" {

const char* redve_version(void) { return "redve_b200 0.1.0 (sm_100a)"; }

uint64_t redve_kernel_launches(void) { return g_launches.load(); }

void redve_release_cached_memory(void) { g_pool.release(); }

int redve_profile(redve_ctx* ctx, int enable) {
  ctx->profiling = enable != 0;
  return REDVE_OK;
}

int redve_profile_report(redve_ctx* ctx, int max_kinds, char* names, double* total_ms,
                         int64_t* count, int* n_kinds) {
  CK(cudaStreamSynchronize(ctx->stream));
  std::vector<std::string> kinds;
  std::vector<double> tot;
  std::vector<int64_t> cnt;
  for (auto& e : ctx->prof) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    size_t k = 0;
    while (k < kinds.size() && kinds[k] != e.name) ++k;
    if (k == kinds.size()) {
      kinds.push_back(e.name);
      tot.push_back(0.0);
      cnt.push_back(0);
    }
    tot[k] += ms;
    cnt[k] += 1;
    ctx->ev_pool.push_back(e.a);
    ctx->ev_pool.push_back(e.b);
  }
  ctx->prof.clear();
  int n = (int)kinds.size() < max_kinds ? (int)kinds.size() : max_kinds;
  for (int k = 0; k < n; ++k) {
    strncpy(names + 32 * k, kinds[k].c_str(), 31);
    names[32 * k + 31] = 0;
    total_ms[k] = tot[k];
    count[k] = cnt[k];
  }
  *n_kinds = n;
  return REDVE_OK;
}

int redve_create(redve_ctx** out, int device) {
  if (!out) return REDVE_E_VALUE;
  redve_ctx* c = new redve_ctx();
  c->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    *out = c;
    return fail(c, REDVE_E_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
  }
  int ce = configure_kernels();
  *out = c;
  if (ce != 0)
    return fail(c, REDVE_E_CUDA, "configuring kernels: %s", cudaGetErrorString((cudaError_t)ce));
  return REDVE_OK;
}

void redve_destroy(redve_ctx* ctx) { delete ctx; }

const char* redve_last_error(const redve_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

int redve_set_stream(redve_ctx* ctx, void* s) {
  ctx->stream = reinterpret_cast<cudaStream_t>(s);
  return REDVE_OK;
}

int redve_synchronize(redve_ctx* ctx) {
  CK(cudaStreamSynchronize(ctx->stream));
  return REDVE_OK;
}

// Rank-one PSF?  taps[a][b] == u[a] v[b] to 1e-15 of the largest tap (the
// uniform and Gaussian kernels are); uv = [u | v], v normalised at the peak.
static bool rank_one_split(const double* taps, int k, std::vector<double>& uv) {
  int a0 = 0, b0 = 0;
  double best = -1.0;
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b)
      if (std::fabs(taps[a * k + b]) > best) {
        best = std::fabs(taps[a * k + b]);
        a0 = a;
        b0 = b;
      }
  uv.assign(2 * k, 0.0);
  if (!(best > 0) || k <= 1) return false;
  for (int a = 0; a < k; ++a) uv[a] = taps[a * k + b0];
  for (int b = 0; b < k; ++b) uv[k + b] = taps[a0 * k + b] / taps[a0 * k + b0];
  for (int a = 0; a < k; ++a)
    for (int b = 0; b < k; ++b)
      if (std::fabs(uv[a] * uv[k + b] - taps[a * k + b]) > 1e-15 * best) return false;
  return true;
}

// k x k host taps into scratch_taps (followed by [u | v] when rank one);
// identical taps already resident are not re-sent (a pageable upload would
// serialise the stream with the host)
static int put_taps(redve_ctx* ctx, const double* taps, int k) {
  const size_t n = (size_t)k * k, kb = sizeof(double) * n;
  CK(ctx->scratch_taps.ensure(kb + sizeof(double) * 2 * k));
  if (ctx->taps_dev == ctx->scratch_taps.p && ctx->taps_host.size() == n &&
      memcmp(ctx->taps_host.data(), taps, kb) == 0)
    return REDVE_OK;
  std::vector<double> buf(taps, taps + n), uv;
  ctx->taps_sep = rank_one_split(taps, k, uv);
  buf.insert(buf.end(), uv.begin(), uv.end());
  CK(cudaMemcpyAsync(ctx->scratch_taps.p, buf.data(), sizeof(double) * buf.size(),
                     cudaMemcpyHostToDevice, ctx->stream));
  ctx->taps_host.assign(taps, taps + n);
  ctx->taps_dev = ctx->scratch_taps.p;
  return REDVE_OK;
}

// ctx->scratch_taps (k x k) through the rank-one two-pass stencil when the
// taps split, else the 2-D stencil kernels
static void conv_scratch(redve_ctx* ctx, const double* x, double* out, int B, int H, int W, int k,
                         int corr) {
  const double* taps = ctx->scratch_taps.as<double>();
  if (ctx->taps_sep &&
      launch_conv_rank1(x, out, B, H, W, taps + (size_t)k * k, k, corr, 1.0, ctx->stream))
    return;
  launch_conv(x, out, B, H, W, taps, k, corr, 1.0, ctx->stream);
}

// ------------------------------------------------------------------ denoise
int redve_denoise(redve_ctx* ctx, const redve_denoiser_desc* dn, int B, int H, int W,
                  const double* x, double* out) {
  if (B < 1 || H < 1 || W < 1) return fail(ctx, REDVE_E_VALUE, "bad batch shape");
  if (x == out) return fail(ctx, REDVE_E_VALUE, "out must not alias x (stencils read neighbours)");
  const long long N = (long long)H * W;
  switch (dn->kind) {
    case REDVE_DN_IDENTITY:
      CK(cudaMemcpyAsync(out, x, sizeof(double) * N * B, cudaMemcpyDeviceToDevice, ctx->stream));
      return REDVE_OK;
    case REDVE_DN_MEDIAN3:
      RUN(ctx, "median3", launch_median3(x, out, B, H, W, ctx->stream));
      CKL();
      return REDVE_OK;
    case REDVE_DN_CONV: {
      if (!is_odd_pos(dn->ksize)) return fail(ctx, REDVE_E_VALUE, "kernel size must be odd");
      if (dn->ksize > H || dn->ksize > W)
        return fail(ctx, REDVE_E_KERNEL, "%dx%d PSF on a %dx%d image", dn->ksize, dn->ksize, H, W);
      int rc = put_taps(ctx, dn->taps, dn->ksize);
      if (rc) return rc;
      RUN(ctx, "conv", conv_scratch(ctx, x, out, B, H, W, dn->ksize, 0));
      CKL();
      // taps buffer is reused by the next call: keep it alive until then
      CK(cudaStreamSynchronize(ctx->stream));
      return REDVE_OK;
    }
    case REDVE_DN_FILTERBANK: {
      if (dn->n_filters < 1 || !is_odd_pos(dn->fsize) || dn->fsize > 15)
        return fail(ctx, REDVE_E_VALUE, "filter bank needs n_filters >= 1 and an odd size <= 15");
      const size_t fb = sizeof(double) * dn->n_filters * dn->fsize * dn->fsize;
      CK(ctx->ve_state.ensure(sizeof(ImgState) * B));
      CK(ctx->scratch_a.ensure(fb + sizeof(double) * dn->n_filters));
      CK(cudaMemcpyAsync(ctx->scratch_a.p, dn->filters, fb, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(ctx->scratch_a.as<char>() + fb, dn->scales,
                         sizeof(double) * dn->n_filters, cudaMemcpyHostToDevice, ctx->stream));
      RdArgs a;
      a.B = B; a.H = H; a.W = W; a.nf = dn->n_filters; a.fs = dn->fsize;
      a.filters = ctx->scratch_a.as<double>();
      a.scales = reinterpret_cast<const double*>(ctx->scratch_a.as<char>() + fb);
      a.tau = dn->tau; a.xin = plain(x, N); a.out = out;
      a.st = ctx->ve_state.as<ImgState>(); a.phase = PH_SETUP;
      RUN(ctx, "filter_bank", launch_rd(a, ctx->stream));
      CKL();
      CK(cudaStreamSynchronize(ctx->stream));
      return REDVE_OK;
    }
    case REDVE_DN_PATCH: {
      if (dn->patch_radius < 0 || dn->search_radius < 1 || !(dn->h > 0) || dn->balance_iters < 1)
        return fail(ctx, REDVE_E_VALUE,
                    "need patch_radius >= 0, search_radius >= 1, h > 0, balance_iters >= 1");
      if (dn->weight_bits != 0 && dn->weight_bits != 32 && dn->weight_bits != 64)
        return fail(ctx, REDVE_E_VALUE, "weight_bits must be 32 or 64");
      const int npos = ((2 * dn->search_radius + 1) * (2 * dn->search_radius + 1) - 1) / 2;
      CK(ctx->ve_state.ensure(sizeof(ImgState) * B));
      CK(ctx->scratch_a.ensure(sizeof(double) * N * B * npos));
      CK(ctx->scratch_b.ensure(sizeof(double) * N * B * 2));
      PwArgs a;
      a.B = B; a.H = H; a.W = W;
      a.pr = dn->patch_radius; a.sr = dn->search_radius; a.npos = npos;
      a.iters = dn->balance_iters; a.inv_h2 = 1.0 / (dn->h * dn->h);
      a.xin = plain(x, N);
      a.w0 = ctx->scratch_a.as<double>();
      a.w32 = dn->weight_bits == 32;
      a.D0 = ctx->scratch_b.as<double>();
      a.D1 = ctx->scratch_b.as<double>() + N * B;
      a.out = out;
      a.st = ctx->ve_state.as<ImgState>();
      a.phase = PH_SETUP;
      int n = 0;
      RUN(ctx, "patch_weighted", launch_pw(a, ctx->stream, &n));
      g_launches.fetch_add(n - 1);
      CKL();
      return REDVE_OK;
    }
    default:
      return fail(ctx, REDVE_E_UNSUPPORTED, "denoiser kind %d not available in this build",
                  dn->kind);
  }
}

int redve_patch_weight_maps(redve_ctx* ctx, const redve_denoiser_desc* dn, int B, int H, int W,
                            const double* x, double* maps) {
  if (dn->kind != REDVE_DN_PATCH) return fail(ctx, REDVE_E_VALUE, "not a PatchWeighted descriptor");
  if (dn->patch_radius < 0 || dn->search_radius < 1 || !(dn->h > 0) || dn->balance_iters < 1)
    return fail(ctx, REDVE_E_VALUE,
                "need patch_radius >= 0, search_radius >= 1, h > 0, balance_iters >= 1");
  if (dn->weight_bits != 0 && dn->weight_bits != 32 && dn->weight_bits != 64)
    return fail(ctx, REDVE_E_VALUE, "weight_bits must be 32 or 64");
  const long long N = (long long)H * W;
  const int npos = ((2 * dn->search_radius + 1) * (2 * dn->search_radius + 1) - 1) / 2;
  CK(ctx->ve_state.ensure(sizeof(ImgState) * B));
  CK(ctx->scratch_a.ensure(sizeof(double) * N * B * npos));
  CK(ctx->scratch_b.ensure(sizeof(double) * N * B * 2));
  PwArgs a;
  a.B = B; a.H = H; a.W = W;
  a.pr = dn->patch_radius; a.sr = dn->search_radius; a.npos = npos;
  a.iters = dn->balance_iters; a.inv_h2 = 1.0 / (dn->h * dn->h);
  a.xin = plain(x, N);
  a.w0 = ctx->scratch_a.as<double>();
  a.w32 = dn->weight_bits == 32;
  a.D0 = ctx->scratch_b.as<double>();
  a.D1 = ctx->scratch_b.as<double>() + N * B;
  a.out = nullptr;
  a.st = ctx->ve_state.as<ImgState>();
  a.phase = PH_SETUP;
  int n = 0;
  RUN(ctx, "patch_maps", launch_pw_maps(a, ctx->stream, &n, maps));
  g_launches.fetch_add(n - 1);
  CKL();
  return REDVE_OK;
}

// ------------------------------------------------------------------ operators
static int op_check(redve_ctx* ctx, const redve_operator_desc* op, int H, int W) {
  if (!is_odd_pos(op->ksize)) return fail(ctx, REDVE_E_VALUE, "PSF size must be odd and >= 1");
  if (op->ksize > H || op->ksize > W)
    return fail(ctx, REDVE_E_KERNEL, "%dx%d PSF on a %dx%d image", op->ksize, op->ksize, H, W);
  if (op->kind == REDVE_OP_BLUR_DOWNSAMPLE && op->factor < 1)
    return fail(ctx, REDVE_E_VALUE, "downsample factor must be >= 1");
  if (op->kind != REDVE_OP_BLUR && op->kind != REDVE_OP_BLUR_DOWNSAMPLE)
    return fail(ctx, REDVE_E_VALUE, "unknown operator kind");
  return REDVE_OK;
}

static int upload_taps(redve_ctx* ctx, const redve_operator_desc* op) {
  return put_taps(ctx, op->taps, op->ksize);
}

int redve_operator_apply(redve_ctx* ctx, const redve_operator_desc* op, int B, int H, int W,
                         const double* x, double* out) {
  int rc = op_check(ctx, op, H, W);
  if (rc) return rc;
  if (x == out) return fail(ctx, REDVE_E_VALUE, "out must not alias x");
  if ((rc = upload_taps(ctx, op))) return rc;
  if (op->kind == REDVE_OP_BLUR) {
    RUN(ctx, "conv", conv_scratch(ctx, x, out, B, H, W, op->ksize, 0));
  } else {
    RUN(ctx, "decimate_conv", launch_decimate_conv(x, out, B, H, W, op->factor, ctx->scratch_taps.as<double>(), op->ksize,
                         ctx->stream));
  }
  CKL();
  CK(cudaStreamSynchronize(ctx->stream));
  return REDVE_OK;
}

int redve_operator_adjoint(redve_ctx* ctx, const redve_operator_desc* op, int B, int H, int W,
                           const double* z, double* out) {
  int rc = op_check(ctx, op, H, W);
  if (rc) return rc;
  if (z == out) return fail(ctx, REDVE_E_VALUE, "out must not alias z");
  if ((rc = upload_taps(ctx, op))) return rc;
  if (op->kind == REDVE_OP_BLUR) {
    RUN(ctx, "conv", conv_scratch(ctx, z, out, B, H, W, op->ksize, 1));
  } else {
    RUN(ctx, "upsample_corr", launch_upsample_corr(z, out, B, H, W, op->factor, ctx->scratch_taps.as<double>(), op->ksize,
                         1.0, ctx->stream));
  }
  CKL();
  CK(cudaStreamSynchronize(ctx->stream));
  return REDVE_OK;
}

// ------------------------------------------------------------------ problem
// Everything of a problem that depends on the measurements (and the PSNR
// reference): y, H^T y / sigma^2 (objective.py:70), x_b, ||y||^2, fresh image
// state.  Buffers, operator constants and the captured solve graph do not.
static int problem_measurements(redve_problem* p, const double* y, const double* reference) {
  redve_ctx* ctx = p->ctx;
  const cudaStream_t s = ctx->stream;
  const int B = p->B, H = p->H, W = p->W;
  const long long Ny = (long long)p->Hy * p->Wy;
  CK(cudaMemcpyAsync(p->y.p, y, sizeof(double) * Ny * B, cudaMemcpyDeviceToDevice, s));
  if (reference)
    CK(cudaMemcpyAsync(p->ref.p, reference, sizeof(double) * p->N * B, cudaMemcpyDeviceToDevice,
                       s));
  RUN(ctx, "init_state", launch_init_state(p->state.as<ImgState>(), B, s));
  const double is2 = 1.0 / (p->sigma * p->sigma);
  if (!p->fourier) {
    RUN(ctx, "upsample_corr", launch_upsample_corr(p->y.as<double>(), p->hty.as<double>(), B, H, W,
                                                   p->op.factor, p->htaps.as<double>(),
                                                   p->op.ksize, is2, s));
  } else {  // rank-one PSFs as two 1-D passes
    bool done = false;
    if (p->separable)
      RUN(ctx, "conv", done = launch_conv_rank1(p->y.as<double>(), p->hty.as<double>(), B, H, W,
                                                p->hsep.as<double>(), p->op.ksize, 1, is2, s));
    if (!done)
      RUN(ctx, "conv", launch_conv(p->y.as<double>(), p->hty.as<double>(), B, H, W,
                                   p->htaps.as<double>(), p->op.ksize, 1, is2, s));
  }
  CKL();
  if (p->fourier) {
    // x_b = IDFT(DFT(H^T y / sigma^2) / d)
    DenoiseArgs ident{DN_IDENTITY, 0, 0, nullptr};
    StepCtl ctl{PH_SETUP, 0, 0.0, 1, 0, 0};
    TraceBufs tr;
    memset(&tr, 0, sizeof(tr));
    int r = fourier_pipeline(p, plain(p->hty.as<double>(), p->N), ident, 1.0,
                             plain(p->xb.as<double>(), p->N), nullptr, 0, plain(nullptr, p->N),
                             ctl, tr, 1, PH_SETUP);
    if (r) return r;
    RUN(ctx, "sumsq", launch_sumsq(p->y.as<double>(), Ny, B, p->yy.as<double>(), s));
    CKL();
  }
  p->sp_ready = false;  // spectral constants hold DFT(x_b), DFT(y), DFT(ref)
  return REDVE_OK;
}

int redve_problem_create(redve_ctx* ctx, const redve_operator_desc* op,
                         const redve_denoiser_desc* dn, int B, int H, int W, const double* y,
                         double sigma, double alpha, const double* reference,
                         redve_problem** out) {
  *out = nullptr;
  if (!(sigma > 0)) return fail(ctx, REDVE_E_VALUE, "sigma must be > 0");
  if (!(alpha > 0)) return fail(ctx, REDVE_E_VALUE, "alpha must be > 0");
  if (B < 1 || H < 1 || W < 1) return fail(ctx, REDVE_E_VALUE, "bad batch shape");
  int rc = op_check(ctx, op, H, W);
  if (rc) return rc;
  if (op->kind == REDVE_OP_BLUR_DOWNSAMPLE && op->ksize > 31)
    return fail(ctx, REDVE_E_UNSUPPORTED, "the fused CG normal operator takes PSFs up to 31x31");
  if (dn->kind == REDVE_DN_CONV) {
    if (!is_odd_pos(dn->ksize)) return fail(ctx, REDVE_E_VALUE, "denoiser kernel must be odd");
    if (dn->ksize > H || dn->ksize > W)
      return fail(ctx, REDVE_E_KERNEL, "%dx%d PSF on a %dx%d image", dn->ksize, dn->ksize, H, W);
  }
  if (dn->kind != REDVE_DN_IDENTITY && dn->kind != REDVE_DN_CONV && dn->kind != REDVE_DN_MEDIAN3 &&
      dn->kind != REDVE_DN_EXTERNAL && dn->kind != REDVE_DN_PATCH &&
      dn->kind != REDVE_DN_FILTERBANK)
    return fail(ctx, REDVE_E_UNSUPPORTED, "denoiser kind %d not available in this build",
                dn->kind);
  if (dn->kind == REDVE_DN_PATCH &&
      (dn->patch_radius < 0 || dn->search_radius < 1 || !(dn->h > 0) || dn->balance_iters < 1))
    return fail(ctx, REDVE_E_VALUE,
                "need patch_radius >= 0, search_radius >= 1, h > 0, balance_iters >= 1");
  if (dn->kind == REDVE_DN_PATCH && dn->weight_bits != 0 && dn->weight_bits != 32 &&
      dn->weight_bits != 64)
    return fail(ctx, REDVE_E_VALUE, "weight_bits must be 32 or 64");
  if (dn->kind == REDVE_DN_FILTERBANK &&
      (dn->n_filters < 1 || !is_odd_pos(dn->fsize) || dn->fsize > 15 || !dn->filters || !dn->scales))
    return fail(ctx, REDVE_E_VALUE, "filter bank needs n_filters >= 1 and an odd size <= 15");
  if (op->kind == REDVE_OP_BLUR) {  // Fourier route limits
    if (H > 4096 || W > 4096) return fail(ctx, REDVE_E_UNSUPPORTED, "image side > 4096");
    if (!is_pow2(H) && H > 256) return fail(ctx, REDVE_E_UNSUPPORTED, "non power-of-two side > 256");
    if (!is_pow2(W) && W > 256) return fail(ctx, REDVE_E_UNSUPPORTED, "non power-of-two side > 256");
  }

  redve_problem* p = new redve_problem();
  p->ctx = ctx;
  p->B = B; p->H = H; p->W = W;
  p->N = (long long)H * W;
  p->op = *op;
  p->op.taps = nullptr;
  int f = op->kind == REDVE_OP_BLUR ? 1 : op->factor;
  p->Hy = (H + f - 1) / f;
  p->Wy = (W + f - 1) / f;
  p->npairs = (B + 1) / 2;
  p->dn_kind = map_dn_kind(dn->kind);
  p->dn_api_kind = dn->kind;
  if (dn->kind == REDVE_DN_PATCH) {
    p->pw_pr = dn->patch_radius;
    p->pw_sr = dn->search_radius;
    p->pw_iters = dn->balance_iters;
    p->pw_h = dn->h;
    p->pw_w32 = dn->weight_bits == 32;
    p->pw_npos = ((2 * dn->search_radius + 1) * (2 * dn->search_radius + 1) - 1) / 2;
  }
  p->dn_ksize = dn->kind == REDVE_DN_CONV ? dn->ksize : 0;
  p->sigma = sigma;
  p->alpha = alpha;
  p->fourier = op->kind == REDVE_OP_BLUR;
  p->lpc_row = lines_per_cta(W);
  if (p->lpc_row > H) p->lpc_row = H;
  p->lpc_col = col_lines_per_cta(H, W);
  if (p->lpc_col > W) p->lpc_col = W;

  auto bail = [&](int code) {
    delete p;
    return code;
  };
#define PK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      fail(ctx, REDVE_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_));             \
      return bail(REDVE_E_CUDA);                                                    \
    }                                                                               \
  } while (0)
  const cudaStream_t s = ctx->stream;
  const size_t kb = sizeof(double) * op->ksize * op->ksize;
  PK(p->htaps.ensure(kb));
  PK(cudaMemcpyAsync(p->htaps.p, op->taps, kb, cudaMemcpyHostToDevice, s));
  {  // rank-one PSF? taps[a][b] == u[a] v[b] (uniform and Gaussian kernels are)
    const int k = op->ksize;
    std::vector<double> uv;
    const bool sep = rank_one_split(op->taps, k, uv);
    if (sep && k > 1) {
      p->separable = 1;
      PK(p->hsep.ensure(sizeof(double) * 2 * k));
      PK(cudaMemcpy(p->hsep.p, uv.data(), sizeof(double) * 2 * k, cudaMemcpyHostToDevice));
    }
    if (op->kind == REDVE_OP_BLUR) {
      // H^T H = periodic convolution with the PSF autocorrelation a(d) =
      // sum_i h(i) h(i + d) (radius k - 1), scaled by 1/sigma^2; rank one when
      // h is: a = (u * u)(v * v)^T.  Used by the gradient baselines.
      const int R = k - 1, T = 2 * k - 1;
      const double is2 = 1.0 / (sigma * sigma);
      std::vector<double> at;
      if (sep && k > 1) {
        at.assign(2 * T, 0.0);  // [horizontal (v) | vertical (u) / sigma^2]
        for (int d = -R; d <= R; ++d) {
          double sv = 0.0, su = 0.0;
          for (int i = 0; i < k; ++i)
            if (i + d >= 0 && i + d < k) {
              sv += uv[k + i] * uv[k + i + d];
              su += uv[i] * uv[i + d];
            }
          at[d + R] = sv;
          at[T + d + R] = su * is2;
        }
      } else {
        at.assign((size_t)T * T, 0.0);
        for (int d1 = -R; d1 <= R; ++d1)
          for (int d2 = -R; d2 <= R; ++d2) {
            double sacc = 0.0;
            for (int i1 = 0; i1 < k; ++i1)
              for (int i2 = 0; i2 < k; ++i2)
                if (i1 + d1 >= 0 && i1 + d1 < k && i2 + d2 >= 0 && i2 + d2 < k)
                  sacc += op->taps[i1 * k + i2] * op->taps[(i1 + d1) * k + i2 + d2];
            at[(size_t)(d1 + R) * T + d2 + R] = sacc * is2;
          }
      }
      p->g_R = R;
      p->g_sep = sep && k > 1;
      PK(p->gtaps.ensure(sizeof(double) * at.size()));
      PK(cudaMemcpy(p->gtaps.p, at.data(), sizeof(double) * at.size(), cudaMemcpyHostToDevice));
    }
  }
  size_t db = dn->kind == REDVE_DN_CONV ? sizeof(double) * dn->ksize * dn->ksize : 8;
  PK(p->dntaps.ensure(db));
  if (dn->kind == REDVE_DN_CONV)
    PK(cudaMemcpyAsync(p->dntaps.p, dn->taps, db, cudaMemcpyHostToDevice, s));
  const long long Ny = (long long)p->Hy * p->Wy;
  PK(p->y.ensure(sizeof(double) * Ny * B));
  if (reference) {
    p->has_ref = true;
    PK(p->ref.ensure(sizeof(double) * p->N * B));
  }
  PK(p->state.ensure(sizeof(ImgState) * B));
  int nblk_row = (H + p->lpc_row - 1) / p->lpc_row;
  int nblk_cost = (H + cost_rows(H) - 1) / cost_rows(H);
  int nblk_fp = (H + cost_fp_rows(W) - 1) / cost_fp_rows(W);
  int nblk_max = nblk_row > nblk_cost ? nblk_row : nblk_cost;
  if (nblk_fp > nblk_max) nblk_max = nblk_fp;
  size_t part = (size_t)p->npairs * nblk_max * 8;
  if (part < (size_t)p->npairs * H * 6) part = (size_t)p->npairs * H * 6;  // any lines per CTA
  if (part < (size_t)B * 64 * 4) part = (size_t)B * 64 * 4;  // k_cost_fp: <= 64 CTAs per image
  PK(p->partials.ensure(sizeof(double) * part));
  PK(p->cnt_inv.ensure(sizeof(unsigned) * (B + 1)));
  PK(p->cnt_cost.ensure(sizeof(unsigned) * (B + 1)));
  PK(p->cnt_ve.ensure(sizeof(unsigned) * (B + 1)));
  PK(cudaMemsetAsync(p->cnt_inv.p, 0, sizeof(unsigned) * (B + 1), s));
  PK(cudaMemsetAsync(p->cnt_cost.p, 0, sizeof(unsigned) * (B + 1), s));
  PK(cudaMemsetAsync(p->cnt_ve.p, 0, sizeof(unsigned) * (B + 1), s));
  PK(p->vals.ensure(sizeof(double) * 3 * B));
  if (dn->kind == REDVE_DN_FILTERBANK) {
    p->rd_nf = dn->n_filters;
    p->rd_fs = dn->fsize;
    p->rd_tau = dn->tau;
    const size_t fb = sizeof(double) * dn->n_filters * dn->fsize * dn->fsize;
    PK(p->rd_filters.ensure(fb));
    PK(cudaMemcpyAsync(p->rd_filters.p, dn->filters, fb, cudaMemcpyHostToDevice, s));
    PK(p->rd_scales.ensure(sizeof(double) * dn->n_filters));
    PK(cudaMemcpyAsync(p->rd_scales.p, dn->scales, sizeof(double) * dn->n_filters,
                       cudaMemcpyHostToDevice, s));
    PK(cudaStreamSynchronize(s));  // host parameter arrays may go away
  }
  // device denoiser output / PatchWeighted fields
  if (dn->kind != REDVE_DN_EXTERNAL) PK(p->fbuf.ensure(sizeof(double) * p->N * B));
  if (dn->kind == REDVE_DN_PATCH) {
    PK(p->w0.ensure(sizeof(double) * p->N * B * p->pw_npos));
    PK(p->D0.ensure(sizeof(double) * p->N * B));
    PK(p->D1.ensure(sizeof(double) * p->N * B));
  }
  if (!p->fourier) {  // CG route
    PK(p->cgst.ensure(sizeof(CgState) * B));
    PK(p->cr.ensure(sizeof(double) * p->N * B));
    PK(p->cp.ensure(sizeof(double) * p->N * B));
    PK(p->cq.ensure(sizeof(double) * p->N * B));
    PK(p->cnt_cg.ensure(sizeof(unsigned) * (B + 1)));
    PK(cudaMemsetAsync(p->cnt_cg.p, 0, sizeof(unsigned) * (B + 1), s));
    PK(cudaMemsetAsync(p->cgst.p, 0, sizeof(CgState) * B, s));
    const int nb = cg_matvec_blocks(H, W), nu = cg_update_blocks(p->N);
    PK(p->part_cg.ensure(sizeof(double) * B * (size_t)(nb > nu ? nb : nu) * 3 + 64));
  }
  PK(p->cnt_rec.ensure(sizeof(unsigned) * (B + 1)));
  PK(cudaMemsetAsync(p->cnt_rec.p, 0, sizeof(unsigned) * (B + 1), s));
  PK(p->hty.ensure(sizeof(double) * p->N * B));
  if (p->fourier) {
    p->twH = ctx->tw(H);
    p->twW = ctx->tw(W);
    p->twsH = ctx->tws(H);
    p->twsW = ctx->tws(W);
    if (!p->twH || !p->twW) {
      fail(ctx, REDVE_E_CUDA, "twiddle allocation failed");
      return bail(REDVE_E_CUDA);
    }
    PK(p->g.ensure(sizeof(double) * p->N));
    RUN(ctx, "inv_denom", launch_inv_denom(p->g.as<double>(), H, W, p->htaps.as<double>(), op->ksize, sigma, alpha, s));
    PK(cudaGetLastError());
    PK(p->Z.ensure(sizeof(cd) * p->N * p->npairs));
    PK(p->xb.ensure(sizeof(double) * p->N * B));
    // cost identity on the Fourier route (cost.cu k_cost_fp)
    PK(p->fprev.ensure(sizeof(double) * p->N * B));
    PK(p->yy.ensure(sizeof(double) * B));
    if (dn->kind == REDVE_DN_PATCH || dn->kind == REDVE_DN_FILTERBANK)
      PK(p->fcur.ensure(sizeof(double) * p->N * B));
  }
  {
    const int r = problem_measurements(p, y, reference);
    if (r) return bail(r);
  }
#undef PK
  *out = p;
  return REDVE_OK;
}

void redve_problem_destroy(redve_problem* p) { delete p; }

int redve_problem_set_measurements(redve_problem* p, const double* y, const double* reference) {
  if (!p) return REDVE_E_VALUE;
  redve_ctx* ctx = p->ctx;
  if (!y) return fail(ctx, REDVE_E_VALUE, "y is null");
  if ((reference != nullptr) != p->has_ref)
    return fail(ctx, REDVE_E_VALUE,
                "a problem keeps its PSNR-reference mode: created %s a reference",
                p->has_ref ? "with" : "without");
  return problem_measurements(p, y, reference);
}

uint64_t redve_problem_graph_captures(const redve_problem* p) { return p ? p->captures : 0; }

static int fp_step_impl(redve_problem* p, const double* x, double* out, const double* f_ext,
                        double* f_out);

int redve_fp_step(redve_problem* p, const double* x, double* out, const double* f_ext) {
  return fp_step_impl(p, x, out, f_ext, nullptr);
}

int redve_fp_step_denoised(redve_problem* p, const double* x, double* out, double* f_out) {
  if (!p->fourier || p->dn_kind == DN_EXTERNAL)
    return fail(p->ctx, REDVE_E_UNSUPPORTED,
                "f(x) is fused into the first FFT pass only for the Fourier route's stencil denoisers");
  return fp_step_impl(p, x, out, nullptr, f_out);
}

static int fp_step_impl(redve_problem* p, const double* x, double* out, const double* f_ext,
                        double* f_out) {
  redve_ctx* ctx = p->ctx;
  const bool host_dn = p->dn_api_kind == REDVE_DN_EXTERNAL;
  if (host_dn && !f_ext) return fail(ctx, REDVE_E_VALUE, "external denoiser needs f(x)");
  RUN(ctx, "init_state", launch_init_state(p->state.as<ImgState>(), p->B, ctx->stream));
  if (!p->fourier) {
    int r = fp_step_cg(p, plain(x, p->N), plain(out, p->N), PH_SETUP, host_dn ? f_ext : nullptr);
    if (r) return r;
    std::vector<ImgState> hs(p->B);
    CK(cudaMemcpyAsync(hs.data(), p->state.p, sizeof(ImgState) * p->B, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int b = 0; b < p->B; ++b)
      if (hs[b].err == ERR_CG) return fail(ctx, REDVE_E_CG, "CG residual above 1e-4 ||rhs|| after 200 iterations");
    return REDVE_OK;
  }
  DenoiseArgs dn = dn_args(p);
  View xin = plain(x, p->N);
  if (p->dn_kind == DN_EXTERNAL) {  // host plug-in or PatchWeighted: f precomputed
    if (!host_dn) {
      int r = denoise_to_fbuf(p, plain(x, p->N), PH_SETUP);
      if (r) return r;
      f_ext = p->fbuf.as<double>();
    }
    dn.kind = DN_IDENTITY;
    dn.radius = 0;
    xin = plain(f_ext, p->N);
  }
  StepCtl ctl{PH_SETUP, 0, 0.0, 1, 0, 0};
  TraceBufs tr;
  memset(&tr, 0, sizeof(tr));
  return fourier_pipeline(p, xin, dn, p->alpha, plain(out, p->N), p->xb.as<double>(), 0,
                          plain(nullptr, p->N), ctl, tr, 1, PH_SETUP, f_out);
}

// grad E(x) = H^T (H x - y) / sigma^2 + alpha (x - f(x))  (objective.py:90-93)
int redve_gradient(redve_problem* p, const double* x, const double* f_ext, double* out) {
  redve_ctx* ctx = p->ctx;
  const cudaStream_t s = ctx->stream;
  const bool host_dn = p->dn_api_kind == REDVE_DN_EXTERNAL;
  if (host_dn && !f_ext) return fail(ctx, REDVE_E_VALUE, "external denoiser needs f(x)");
  RUN(ctx, "init_state", launch_init_state(p->state.as<ImgState>(), p->B, s));
  View xv = plain(x, p->N);
  if (!host_dn) {
    int r = denoise_to_fbuf(p, xv, PH_SETUP);
    if (r) return r;
    f_ext = p->fbuf.as<double>();
  }
  GradArgs ga;
  memset(&ga, 0, sizeof(ga));
  ga.B = p->B; ga.H = p->H; ga.W = p->W;
  ga.v = xv; ga.xprev = xv; ga.xout = xv;
  if (!p->fourier) {
    CgArgs ca;
    memset(&ca, 0, sizeof(ca));
    ca.B = p->B; ca.H = p->H; ca.W = p->W; ca.factor = p->op.factor; ca.k = p->op.ksize;
    ca.taps = p->htaps.as<double>();
    ca.inv_sigma2 = 1.0 / (p->sigma * p->sigma); ca.alpha = p->alpha;
    ca.huv = p->separable ? p->hsep.as<double>() : nullptr;
    ca.xin = xv; ca.q = p->cq.as<double>(); ca.cg = p->cgst.as<CgState>();
    ca.st = p->state.as<ImgState>(); ca.phase = PH_SETUP;
    RUN(ctx, "normal_matvec", launch_normal_matvec(ca, s));
    CKL();
    ga.Av = p->cq.as<double>();
  } else {
    const int T = 2 * p->g_R + 1;
    ga.R = p->g_R;
    if (p->g_sep) {
      ga.av = p->gtaps.as<double>();
      ga.au = ga.av + T;
    } else {
      ga.afull = p->gtaps.as<double>();
    }
  }
  ga.hty = p->hty.as<double>(); ga.f = f_ext; ga.alpha = p->alpha;
  ga.gout = out;
  ga.st = p->state.as<ImgState>();
  ga.ctl = StepCtl{PH_SETUP, 0, 0.0, 1, 0, 0};
  RUN(ctx, "gradient", launch_grad_step(ga, s));
  CKL();
  return REDVE_OK;
}

static CostArgs cost_args(redve_problem* p, View x, const double* f_ext, int mode, StepCtl ctl,
                          TraceBufs tr) {
  CostArgs a;
  a.B = p->B; a.H = p->H; a.W = p->W; a.rows = cost_rows(p->H);
  a.Hy = p->Hy; a.Wy = p->Wy;
  a.factor = p->op.kind == REDVE_OP_BLUR ? 1 : p->op.factor;
  a.x = x; a.y = p->y.as<double>(); a.ref = p->has_ref ? p->ref.as<double>() : nullptr;
  a.dn = dn_args(p);
  a.fext = f_ext;
  a.htaps = p->htaps.as<double>(); a.hk = p->op.ksize;
  a.separable = p->separable;
  a.hu = p->separable ? p->hsep.as<double>() : nullptr;
  a.hv = p->separable ? p->hsep.as<double>() + p->op.ksize : nullptr;
  a.sigma = p->sigma; a.alpha = p->alpha;
  a.mode = mode; a.out_vals = p->vals.as<double>();
  a.st = p->state.as<ImgState>(); a.ctl = ctl; a.tr = tr;
  a.partials = p->partials.as<double>(); a.counters = p->cnt_cost.as<unsigned>();
  return a;
}

int redve_cost(redve_problem* p, const double* x, const double* f_ext, double* cost,
               double* fid, double* reg, double* psnr) {
  redve_ctx* ctx = p->ctx;
  if (p->dn_api_kind == REDVE_DN_EXTERNAL && !f_ext)
    return fail(ctx, REDVE_E_VALUE, "external denoiser needs f(x)");
  if (p->dn_api_kind == REDVE_DN_PATCH || p->dn_api_kind == REDVE_DN_FILTERBANK) {
    RUN(ctx, "init_state", launch_init_state(p->state.as<ImgState>(), p->B, ctx->stream));
    int r = denoise_to_fbuf(p, plain(x, p->N), PH_SETUP);
    if (r) return r;
    f_ext = p->fbuf.as<double>();
  }
  StepCtl ctl{PH_SETUP, 0, 0.0, 1, 0, 0};
  TraceBufs tr;
  memset(&tr, 0, sizeof(tr));
  CostArgs a = cost_args(p, plain(x, p->N), f_ext, COST_VALUE, ctl, tr);
  RUN(ctx, "cost", launch_cost(a, p->npairs, ctx->stream));
  CKL();
  std::vector<double> v(3 * p->B);
  CK(cudaMemcpyAsync(v.data(), p->vals.p, sizeof(double) * 3 * p->B, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int b = 0; b < p->B; ++b) {
    double df = v[3 * b] / (2.0 * p->sigma * p->sigma);
    double rg = 0.5 * v[3 * b + 1];
    if (fid) fid[b] = df;
    if (reg) reg[b] = rg;
    if (cost) cost[b] = df + p->alpha * rg;
    if (psnr) {
      double mse = v[3 * b + 2] / (double)p->N;
      psnr[b] = !p->has_ref ? NAN : (mse == 0.0 ? INFINITY : (!std::isfinite(mse) ? -INFINITY
                                   : 10.0 * std::log10(255.0 * 255.0 / mse)));
    }
  }
  return REDVE_OK;
}

// CTAs per image for the VE passes (k_gram / k_combine, 256 threads, 2 resident
// per SM): minimise waves x (pixels per thread + the per-CTA reduction cost),
// so small batches still fill the GPU and large ones are not cut into slivers
// (configs[1] sweep: 4 CTAs/image -> gram 60 us, 9 -> 67, 32 -> 80).
static int ve_chunks(int B, long long N) {
  if (const char* e = getenv("REDVE_VE_CHUNKS")) {  // experiments
    const int c = atoi(e);
    if (c >= 1 && c <= 64) return c;
  }
  static long long resident = 0;  // 2 CTAs per SM (k_gram / k_combine at 128 registers)
  if (resident == 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident = 2LL * (sms > 0 ? sms : 148);
  }
  int best = 1;
  double best_cost = 1e300;
  for (int c = 1; c <= 64; ++c) {
    if ((long long)c * 256 > N && c > 1) break;
    const long long ctas = (long long)B * c;
    const double waves = (double)((ctas + resident - 1) / resident);
    const double cost = waves * ((double)N / (256.0 * c) + 24.0);  // 24: measured tail cost
    if (cost < best_cost * 0.999) {
      best_cost = cost;
      best = c;
    }
  }
  return best;
}

// ------------------------------------------------------------------ spectral route
static bool spectral_enabled() {
  const char* e = getenv("REDVE_SPECTRAL");
  return !(e && e[0] == '0');
}

// The spectral route applies to circulant operators with a linear shift-
// invariant denoiser (spectral.cuh).
static bool spectral_route(const redve_problem* p) {
  return p->fourier && (p->dn_api_kind == REDVE_DN_CONV || p->dn_api_kind == REDVE_DN_IDENTITY) &&
         spectral_enabled();
}

// Constant spectra, once per problem: m = a hf / d, H(k), 1 - Re hf, DFT(x_b),
// DFT(y), DFT(ref).
static int spectral_setup(redve_problem* p) {
  redve_ctx* ctx = p->ctx;
  const cudaStream_t s = ctx->stream;
  const int B = p->B;
  const long long N = p->N;
  auto plan = [&](int batch) -> cufftHandle {
    const auto key = std::make_tuple(p->H, p->W, batch);
    auto it = ctx->fft_plans.find(key);
    if (it != ctx->fft_plans.end()) return it->second;
    int n[2] = {p->H, p->W};
    cufftHandle h = 0;
    if (cufftPlanMany(&h, 2, n, nullptr, 1, (int)N, nullptr, 1, (int)N, CUFFT_Z2Z, batch) !=
        CUFFT_SUCCESS)
      return 0;
    ctx->fft_plans[key] = h;
    return h;
  };
  if (!p->sp_plan) {
    p->sp_plan = plan(B);
    p->sp_plan1 = plan(1);
    if (!p->sp_plan || !p->sp_plan1) return fail(ctx, REDVE_E_CUDA, "cufftPlanMany failed");
  }
  if (cufftSetStream(p->sp_plan, s) != CUFFT_SUCCESS || cufftSetStream(p->sp_plan1, s) != CUFFT_SUCCESS)
    return fail(ctx, REDVE_E_CUDA, "cufftSetStream failed");
  CK(p->sp_stage.ensure(sizeof(cd) * N * B));
  if (!p->sp_cnt.p || p->sp_cnt.n < sizeof(unsigned) * (B + 1)) {
    CK(p->sp_cnt.ensure(sizeof(unsigned) * (B + 1)));
    CK(cudaMemsetAsync(p->sp_cnt.p, 0, sizeof(unsigned) * (B + 1), s));
  }
  CK(p->sp_part.ensure(sizeof(double) * 6 * (size_t)B * spec_chunks(B, N)));
  if (p->sp_ready) return REDVE_OK;
  CK(p->sp_m.ensure(sizeof(cd) * N));
  CK(p->sp_hh.ensure(sizeof(cd) * N));
  CK(p->sp_wr.ensure(sizeof(double) * N));
  CK(p->sp_xb.ensure(sizeof(cd) * N * B));
  CK(p->sp_yh.ensure(sizeof(cd) * N * B));
  cd* stage = p->sp_stage.as<cd>();
  auto fwd = [&](cufftHandle plan, cd* z) {
    return cufftExecZ2Z(plan, reinterpret_cast<cufftDoubleComplex*>(z),
                        reinterpret_cast<cufftDoubleComplex*>(z), CUFFT_FORWARD) == CUFFT_SUCCESS;
  };
  // denoiser spectrum -> m, 1 - Re hf (stage[0] as scratch)
  const bool ident = p->dn_api_kind == REDVE_DN_IDENTITY;
  if (!ident) {
    RUN(ctx, "spec_embed", launch_spec_embed(p->dntaps.as<double>(), p->dn_ksize, p->H, p->W, stage, s));
    if (!fwd(p->sp_plan1, stage)) return fail(ctx, REDVE_E_CUDA, "cufftExecZ2Z failed");
  }
  RUN(ctx, "spec_consts", launch_spec_consts(ident ? nullptr : stage, p->g.as<double>(), p->alpha,
                                             N, p->sp_m.as<cd>(), p->sp_wr.as<double>(), s));
  // operator spectrum H(k)
  RUN(ctx, "spec_embed", launch_spec_embed(p->htaps.as<double>(), p->op.ksize, p->H, p->W,
                                           p->sp_hh.as<cd>(), s));
  if (!fwd(p->sp_plan1, p->sp_hh.as<cd>())) return fail(ctx, REDVE_E_CUDA, "cufftExecZ2Z failed");
  // DFT(x_b), DFT(y), DFT(ref)
  RUN(ctx, "spec_pack", launch_spec_pack(p->xb.as<double>(), B, N, p->sp_xb.as<cd>(), N, nullptr, s));
  if (!fwd(p->sp_plan, p->sp_xb.as<cd>())) return fail(ctx, REDVE_E_CUDA, "cufftExecZ2Z failed");
  RUN(ctx, "spec_pack", launch_spec_pack(p->y.as<double>(), B, N, p->sp_yh.as<cd>(), N, nullptr, s));
  if (!fwd(p->sp_plan, p->sp_yh.as<cd>())) return fail(ctx, REDVE_E_CUDA, "cufftExecZ2Z failed");
  if (p->has_ref) {
    CK(p->sp_rh.ensure(sizeof(cd) * N * B));
    RUN(ctx, "spec_pack", launch_spec_pack(p->ref.as<double>(), B, N, p->sp_rh.as<cd>(), N, nullptr, s));
    if (!fwd(p->sp_plan, p->sp_rh.as<cd>())) return fail(ctx, REDVE_E_CUDA, "cufftExecZ2Z failed");
  }
  CKL();
  p->sp_ready = true;
  return REDVE_OK;
}

// ------------------------------------------------------------------ solve
int redve_solve(redve_problem* p, const redve_solve_config* cfg, const double* x0, double* x_out,
                redve_trace* trace) {
  redve_ctx* ctx = p->ctx;
  cudaStream_t s = ctx->stream;
  if (cfg->method < REDVE_METHOD_FP || cfg->method > REDVE_METHOD_NESTEROV)
    return fail(ctx, REDVE_E_VALUE, "unknown method %d", cfg->method);
  const bool gradm = cfg->method == REDVE_METHOD_SD || cfg->method == REDVE_METHOD_SD_VE ||
                     cfg->method == REDVE_METHOD_NESTEROV;
  const bool nest = cfg->method == REDVE_METHOD_NESTEROV;
  if (gradm && !(cfg->step_size > 0))  // solvers.py:277-278, 323-324
    return fail(ctx, REDVE_E_VALUE, "this method needs a positive step_size");
  if (gradm && p->fourier && p->g_R > 64)
    return fail(ctx, REDVE_E_UNSUPPORTED, "gradient stencil radius %d too large", p->g_R);
  if (cfg->ve_method < 0 || cfg->ve_method > 2) return fail(ctx, REDVE_E_VALUE, "unknown VE method");
  if (cfg->kappa < 1) return fail(ctx, REDVE_E_VALUE, "kappa must be >= 1");
  if (cfg->kappa + 1 > MAXKP1) return fail(ctx, REDVE_E_UNSUPPORTED, "kappa > %d", MAXKP1 - 1);
  if (cfg->m < 0) return fail(ctx, REDVE_E_VALUE, "m must be >= 0");
  if (cfg->max_inner_steps < 1) return fail(ctx, REDVE_E_VALUE, "max_inner_steps must be >= 1");
  if (cfg->tol < 0) return fail(ctx, REDVE_E_VALUE, "tol must be >= 0");
  if (cfg->stabilization_iters < 0) return fail(ctx, REDVE_E_VALUE, "stabilization_iters < 0");
  if (!(cfg->rank_tolerance > 0)) return fail(ctx, REDVE_E_VALUE, "rank_tolerance must be > 0");
  const bool ve = cfg->method == REDVE_METHOD_FP_VE || cfg->method == REDVE_METHOD_SD_VE;
  if (ve && cfg->max_inner_steps < cfg->m + cfg->kappa + 2)
    return fail(ctx, REDVE_E_VALUE, "budget must admit at least one full cycle (m + kappa + 2)");
  if (p->dn_api_kind == REDVE_DN_EXTERNAL)
    return fail(ctx, REDVE_E_UNSUPPORTED, "device solve needs a device denoiser");
  const bool pw = p->dn_api_kind == REDVE_DN_PATCH || p->dn_api_kind == REDVE_DN_FILTERBANK;
  const bool spec = !gradm && spectral_route(p);
  if (spec) {
    int r = spectral_setup(p);
    if (r) return r;
  }

  const int B = p->B;
  const long long N = p->N;
  const long long NE = spec ? 2 * N : N;  // ring elements per iterate (doubles)
  const int budget = cfg->max_inner_steps;
  const int stab = ve ? cfg->stabilization_iters : 0;
  const int clen = cfg->m + cfg->kappa + 1;
  const int S = ve ? clen + 1 : 2;
  const int kp1 = cfg->kappa + 1;
  const int cap = budget + stab;
  const int ccap = budget / clen + 2;
  const int log_every = N <= 128 * 128 ? 1 : 5;  // solvers.py:34,213
  const bool track = ve;

  CK(p->ring.ensure(sizeof(double) * NE * S * B));
  if (track) CK(p->best.ensure(sizeof(double) * NE * B));
  const int chunks = ve_chunks(B, NE);
  if (ve) {
    CK(p->q.ensure(sizeof(double) * NE * kp1 * B));
    size_t need = (size_t)B * chunks * (MAXKP1 * (MAXKP1 + 1) / 2);
    if (need * sizeof(double) > p->partials.n)  // grow (the row kernels' share fits inside)
      CK(p->partials.ensure(need * sizeof(double) + 64));
  }
  if (gradm) {
    const int nb = grad_partials_per_image(p->H, p->W, p->fourier);
    CK(p->part_grad.ensure(sizeof(double) * 3 * (size_t)B * nb));
    if (p->cnt_grad.n < sizeof(unsigned) * (B + 1)) {
      CK(p->cnt_grad.ensure(sizeof(unsigned) * (B + 1)));
      CK(cudaMemsetAsync(p->cnt_grad.p, 0, sizeof(unsigned) * (B + 1), s));
    }
    if (nest) CK(p->ybuf.ensure(sizeof(double) * 2 * (size_t)B * N));
  }
  // Nesterov momentum t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2, beta_k = (t_k - 1) / t_{k+1}
  // (solvers.py:330-333): the same for every image, so a per-step launch argument
  std::vector<double> betas;
  if (nest) {
    double t = 1.0;
    for (int i = 0; i < budget; ++i) {
      const double tn = (1.0 + std::sqrt(1.0 + 4.0 * t * t)) / 2.0;
      betas.push_back((t - 1.0) / tn);
      t = tn;
    }
  }
  // trace buffers (device)
  const size_t nrec = (size_t)B * cap, ncyc = (size_t)B * ccap;
  size_t tbytes = sizeof(double) * (5 * nrec + ncyc * (1 + 2 * MAXKP1)) + sizeof(int) * ncyc * 4 +
                  sizeof(int) * nrec;
  CK(p->trace.ensure(tbytes));
  TraceBufs tr;
  {
    char* base = p->trace.as<char>();
    tr.cap = cap;
    tr.ccap = ccap;
    double* d = reinterpret_cast<double*>(base);
    tr.step_norm = d;
    tr.cost = d + nrec;
    tr.psnr = d + 2 * nrec;
    tr.gamma = d + 3 * nrec;
    tr.elapsed = d + 4 * nrec;
    tr.cyc_stab = d + 5 * nrec;
    tr.cyc_gamma = tr.cyc_stab + ncyc;
    tr.cyc_c = tr.cyc_gamma + ncyc * MAXKP1;
    tr.cyc_meta = reinterpret_cast<int*>(tr.cyc_c + ncyc * MAXKP1);
    tr.cg_iters = tr.cyc_meta + ncyc * 4;
  }
  // All device work of the solve.  Fourier route with tol == 0 has no host
  // decision inside, so it is captured once into a CUDA graph and replayed
  // (the CG route checks its per-image stop flags on the host).
  const bool use_graph = p->fourier && cfg->tol == 0 && !ctx->profiling && graphs_enabled();
  // The graph never sees the caller's x0 / x_out: x0 is loaded into ring slot 0
  // before it and the solution gathered after it, so repeated solves on one
  // problem replay a single capture whatever buffers the caller passes.
  char topo[512], keybuf[640];
  snprintf(topo, sizeof(topo), "%d|%d|%d|%d|%d|%d|%d|%d|%d|%d|%d|%d|%d|%d|%.17g|%d|%.17g|%.17g",
           p->B, p->H, p->W, p->op.kind, p->op.ksize, p->dn_api_kind, p->dn_ksize, (int)pw,
           (int)spec + (spec && spec_run_fits(p->B, p->N, ve ? kp1 : 2) ? 2 : 0),
           cfg->method, cfg->ve_method, cfg->m, cfg->kappa, cfg->max_inner_steps, cfg->tol,
           cfg->stabilization_iters, cfg->rank_tolerance, gradm ? cfg->step_size : 0.0);
  snprintf(keybuf, sizeof(keybuf), "%s|%llu|%p|%p|%p|%p", topo, p->serial, p->ring.p, p->trace.p,
           p->best.p, p->ybuf.p);
  CK(p->x0bad.ensure(sizeof(int)));
  CK(cudaMemsetAsync(p->x0bad.p, 0, sizeof(int), s));
  if (spec) {  // x0 -> DFT(x0) in ring slot 0
    cd* stage = p->sp_stage.as<cd>();
    RUN(ctx, "load_x0", launch_spec_pack(x0, B, N, stage, N, p->x0bad.as<int>(), s));
    CKL();
    if (cufftExecZ2Z(p->sp_plan, reinterpret_cast<cufftDoubleComplex*>(stage),
                     reinterpret_cast<cufftDoubleComplex*>(stage), CUFFT_FORWARD) != CUFFT_SUCCESS)
      return fail(ctx, REDVE_E_CUDA, "cufftExecZ2Z failed");
    CK(cudaMemcpy2DAsync(p->ring.p, sizeof(double) * NE * S, stage, sizeof(cd) * N, sizeof(cd) * N,
                         B, cudaMemcpyDeviceToDevice, s));
  } else {
    RUN(ctx, "load_x0", launch_load_x0(p->ring.as<double>(), N * S, x0, B, N, p->x0bad.as<int>(), s));
    CKL();
  }
  auto device_work = [&]() -> int {
    CK(cudaMemsetAsync(p->trace.p, 0xFF, sizeof(double) * 5 * nrec, s));  // NaN
    CK(cudaMemsetAsync(tr.cyc_stab, 0, sizeof(double) * ncyc * (1 + 2 * MAXKP1) +
                                           sizeof(int) * (ncyc * 4 + nrec), s));
    ImgState* st = p->state.as<ImgState>();
    RUN(ctx, "init_state", launch_init_state(st, B, s));
    CKL();

    View cur{p->ring.as<double>(), NE * S, NE, S, 1};
    View nxt{p->ring.as<double>(), NE * S, NE, S, 2};
    View bestv = plain(p->best.as<double>(), NE);
    DenoiseArgs dn = dn_args(p);
    SpecConsts sk;
    memset(&sk, 0, sizeof(sk));
    if (spec) {
      sk.m = p->sp_m.as<cd>(); sk.hh = p->sp_hh.as<cd>(); sk.wr = p->sp_wr.as<double>();
      sk.xb = p->sp_xb.as<cd>(); sk.yh = p->sp_yh.as<cd>();
      sk.rh = p->has_ref ? p->sp_rh.as<cd>() : nullptr;
    }
    StepCtl ctl{PH_MAIN, budget, cfg->tol, log_every, 0, track ? 1 : 0,
                (spec && cfg->tol == 0) ? 1 : 0};

    VeArgs va;
    memset(&va, 0, sizeof(va));
    va.B = B; va.N = NE; va.m = cfg->m; va.kp1 = kp1; va.S = S;
    va.ring = p->ring.as<double>(); va.img_stride = NE * S; va.slot_stride = NE;
    va.st = st; va.tr = tr; va.partials = p->partials.as<double>();
    va.counters = p->cnt_ve.as<unsigned>(); va.qscratch = p->q.as<double>();
    va.method = cfg->ve_method; va.rank_tol = cfg->rank_tolerance; va.chunks = chunks;
    va.stationary_continues = (spec && cfg->tol == 0) ? 1 : 0;
    va.mgs_cluster = mgs_cluster_pays(B) ? 1 : 0;

    // Cost of the current iterates.  Fourier route: cadence records use the
    // normal-equation identity (k_cost_fp) with f(x_{k-1}) kept by k_row_fwd
    // (fused denoisers) or by the step itself (precomputed denoisers).  For the
    // precomputed denoisers f(x_k) evaluated here is handed to the next step
    // when nothing changes the iterate in between (f_ready); the CG route
    // reuses it the same way.
    const bool ident = p->fourier && !gradm;  // the cost identity holds for FP steps only
    double* f_step = p->fbuf.as<double>();   // f of the current step's input
    double* f_spare = p->fcur.as<double>();  // f of the new iterate (cost)
    bool f_ready = false;
    auto cost_of_cur = [&](int mode, StepCtl c, const double* fprev_rec = nullptr) -> int {
      if (spec) {  // note_initial / finalize in the Fourier domain (records are fused)
        SpecCostArgs sa;
        sa.B = B; sa.H = p->H; sa.W = p->W; sa.x = cur; sa.k = sk; sa.mode = mode;
        sa.sigma = p->sigma; sa.alpha = p->alpha; sa.st = st; sa.ctl = c; sa.tr = tr;
        sa.partials = p->sp_part.as<double>(); sa.counters = p->sp_cnt.as<unsigned>();
        RUN(ctx, "spec_cost", launch_spec_cost(sa, s));
        CKL();
        return REDVE_OK;
      }
      const double* fe = nullptr;
      const int ph = mode == COST_RECORD ? c.phase : PH_SETUP;
      if (pw) {
        double* dst = ident ? f_spare : p->fbuf.as<double>();
        int r = denoise_to_fbuf(p, cur, ph, dst);
        if (r) return r;
        fe = dst;
      }
      CostArgs ca = cost_args(p, cur, fe, mode, c, tr);
      if (ident && mode == COST_RECORD) {
        ca.fprev = pw ? f_step : (fprev_rec ? fprev_rec : p->fprev.as<double>());
        ca.hty = p->hty.as<double>();
        ca.yy = p->yy.as<double>();
      }
      if (ident && mode == COST_RECORD && cost_fp_ok(ca)) {
        RUN(ctx, "cost", launch_cost_fp(ca, p->npairs, s));
      } else {
        RUN(ctx, "cost", launch_cost(ca, p->npairs, s));
      }
      CKL();
      if (pw && ident && mode != COST_FINAL) {  // f(cur) is ready for the next step
        std::swap(f_step, f_spare);
        f_ready = true;
      } else if (pw && !p->fourier && !gradm && mode != COST_FINAL) {
        f_ready = true;  // CG route: f(cur) sits in fbuf, where the next step reads it
      }
      return REDVE_OK;
    };

    if (nest)  // y_0 = x_0 (solvers.py:327)
      RUN(ctx, "copy_view", launch_copy_view(plain(p->ybuf.as<double>(), N), cur, B, N, st, 0, s));
    if (track) {  // note_initial (solvers.py:219-223)
      int r0 = cost_of_cur(COST_INIT, ctl);
      if (r0) return r0;
      RUN(ctx, "copy_view", launch_copy_view(bestv, cur, B, NE, st, 1, s));
      CKL();
    }

    cd* zcur = p->Z.as<cd>();
    int kk = 0;  // steps issued so far (Nesterov buffer parity / momentum index)
    auto step = [&](int phase, bool cadence) -> int {
      StepCtl c = ctl;
      c.phase = phase;
      c.defer_commit = cadence ? 1 : 0;
      int r = REDVE_OK;
      double* fp_this = p->fprev.as<double>();
      if (spec) {  // X+ = Xb + m X, cost fused on cadence steps (spectral.cuh)
        SpecStepArgs sa;
        sa.B = B; sa.H = p->H; sa.W = p->W; sa.cur = cur; sa.nxt = nxt; sa.k = sk;
        sa.cadence = cadence ? 1 : 0; sa.sigma = p->sigma; sa.alpha = p->alpha;
        sa.st = st; sa.ctl = c; sa.tr = tr; sa.S = S;
        sa.partials = p->sp_part.as<double>(); sa.counters = p->sp_cnt.as<unsigned>();
        RUN(ctx, "spec_step", launch_spec_step(sa, s));
        CKL();
        if (cadence && track) {
          RUN(ctx, "copy_view", launch_copy_view(bestv, cur, B, NE, st, 1, s));
          CKL();
        }
        ++kk;
        return REDVE_OK;
      }
      if (gradm) {  // x+ = v - s grad E(v)  (solvers.py:274-280, 315-337)
        double* y0 = nest ? p->ybuf.as<double>() : nullptr;
        const size_t half = (size_t)B * N;
        View vin = nest ? plain(y0 + (kk & 1) * half, N) : cur;
        r = denoise_to_fbuf(p, vin, phase);
        if (r) return r;
        GradArgs ga;
        memset(&ga, 0, sizeof(ga));
        ga.B = B; ga.H = p->H; ga.W = p->W;
        ga.v = vin; ga.xprev = cur; ga.xout = nxt;
        if (!p->fourier) {
          CgArgs ca;
          memset(&ca, 0, sizeof(ca));
          ca.B = B; ca.H = p->H; ca.W = p->W; ca.factor = p->op.factor; ca.k = p->op.ksize;
          ca.taps = p->htaps.as<double>();
          ca.inv_sigma2 = 1.0 / (p->sigma * p->sigma); ca.alpha = p->alpha;
          ca.huv = p->separable ? p->hsep.as<double>() : nullptr;
          ca.xin = vin; ca.q = p->cq.as<double>(); ca.cg = p->cgst.as<CgState>(); ca.st = st;
          ca.phase = phase;
          RUN(ctx, "normal_matvec", launch_normal_matvec(ca, s));
          CKL();
          ga.Av = p->cq.as<double>();
        } else {
          const int T = 2 * p->g_R + 1;
          ga.R = p->g_R;
          if (p->g_sep) {
            ga.av = p->gtaps.as<double>();
            ga.au = ga.av + T;
          } else {
            ga.afull = p->gtaps.as<double>();
          }
        }
        ga.hty = p->hty.as<double>(); ga.f = p->fbuf.as<double>();
        ga.alpha = p->alpha; ga.step = cfg->step_size;
        ga.beta = nest ? betas[kk < (int)betas.size() ? kk : (int)betas.size() - 1] : 0.0;
        ga.ynext = nest ? y0 + ((kk + 1) & 1) * half : nullptr;
        ga.st = st; ga.ctl = c; ga.tr = tr; ga.S = S;
        ga.partials = p->part_grad.as<double>(); ga.counters = p->cnt_grad.as<unsigned>();
        RUN(ctx, "grad_step", launch_grad_step(ga, s));
        CKL();
      } else if (p->fourier) {
        {
          View xin = cur;
          DenoiseArgs d = dn;
          if (pw) {
            if (!f_ready) {
              r = denoise_to_fbuf(p, cur, phase, f_step);
              if (r) return r;
            }
            xin = plain(f_step, N);
            d.kind = DN_IDENTITY;
            d.radius = 0;
          }
          f_ready = false;
          double* fout = (cadence && !pw) ? fp_this : nullptr;
          if ((r = f_row_fwd(p, xin, d, zcur, phase, fout))) return r;
        }
        if ((r = f_col(p, zcur, p->alpha, phase))) return r;
        r = f_row_inv(p, zcur, nxt, p->xb.as<double>(), 1, cur, c, tr, S);
      } else {
        // a cadence cost already denoised cur into fbuf (PatchWeighted: ~30%
        // of a configs[2] solve): the CG step takes it as its f
        r = fp_step_cg(p, cur, nxt, phase, f_ready ? p->fbuf.as<double>() : nullptr);
        f_ready = false;
        if (r) return r;
        RecordArgs ra;
        ra.cg = p->cgst.as<CgState>();
        ra.N = N; ra.xnew = nxt; ra.xprev = cur; ra.S = S; ra.st = st; ra.ctl = c; ra.tr = tr;
        ra.partials = p->part_cg.as<double>(); ra.counters = p->cnt_rec.as<unsigned>();
        RUN(ctx, "step_record", launch_step_record(ra, B, s));
        CKL();
      }
      if (r) return r;
      if (cadence) {
        r = cost_of_cur(COST_RECORD, c, fp_this);
        if (r) return r;
        if (track) {
          RUN(ctx, "copy_view", launch_copy_view(bestv, cur, B, NE, st, 1, s));
          CKL();
        }
      }
      ++kk;
      return REDVE_OK;
    };

    // spectral route, small batches: the whole schedule below (steps, cadence
    // costs, best copies, VE after every full cycle) as one cluster launch per
    // image (k_spec_run)
    const bool spec_fused = spec && spec_run_fits(B, N, ve ? kp1 : 2);
    auto spec_run = [&](int phase, int kstart, int kend, bool with_ve, bool all_cadence) -> int {
      StepCtl c = ctl;
      c.phase = phase;
      SpecStepArgs sa;
      sa.B = B; sa.H = p->H; sa.W = p->W; sa.cur = cur; sa.nxt = nxt; sa.k = sk;
      sa.cadence = 0; sa.sigma = p->sigma; sa.alpha = p->alpha;
      sa.st = st; sa.ctl = c; sa.tr = tr; sa.S = S;
      sa.partials = p->sp_part.as<double>(); sa.counters = p->sp_cnt.as<unsigned>();
      int rc = 0;
      RUN(ctx, "spec_run", rc = launch_spec_run(sa, va, kstart, kend, clen, with_ve ? 1 : 0,
                                                all_cadence ? 1 : 0, track ? 1 : 0,
                                                p->best.as<double>(), s));
      if (rc) return fail(ctx, REDVE_E_CUDA, "spec_run: %s", cudaGetErrorString((cudaError_t)rc));
      kk += kend - kstart;
      return REDVE_OK;
    };

    std::vector<ImgState> hst(B);
    auto any_running = [&]() -> int {
      CK(cudaMemcpyAsync(hst.data(), st, sizeof(ImgState) * B, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      int any = 0;
      for (int b = 0; b < B; ++b) any |= (hst[b].term == RUNNING);
      return any ? 1 : 0;
    };
    const int check_every = (cfg->tol > 0 || !p->fourier) ? 1 : 8;  // CG steps stop exactly

    int k = 0;
    if (spec_fused) {
      int r = spec_run(PH_MAIN, 0, budget, ve, false);
      if (r) return r;
      k = budget;
    } else if (!ve) {
      while (k < budget) {
        int r = step(PH_MAIN, ((k + 1) % log_every) == 0);
        if (r) return r;
        ++k;
        if (!use_graph && k % (check_every * clen) == 0 && k < budget) {
          int a = any_running();
          if (a < 0 || a > 1) return a;
          if (!a) break;
        }
      }
    } else {
      int cycles = 0;
      while (true) {
        int n = 0;
        for (int i = 0; i < clen; ++i) {
          int r = step(PH_MAIN, ((k + 1) % log_every) == 0);
          if (r) return r;
          ++k;
          ++n;
          if (k >= budget) break;
        }
        if (n == clen) {
          RUN(ctx, "gram", launch_gram(va, s));
          CKL();
          if (va.mgs_cluster) {
            RUN(ctx, "mgs_cluster", launch_mgs_cluster(va, s));
            CKL();
          }
          RUN(ctx, "combine", launch_combine(va, s));
          CKL();
          f_ready = false;  // the iterate may have been replaced
        }
        if (k >= budget) break;
        if (++cycles % check_every == 0 && !use_graph) {
          int a = any_running();
          if (a < 0 || a > 1) return a;
          if (!a) break;
        }
      }
    }
    if (spec_fused) {
      if (stab > 0) {
        int r = spec_run(PH_STAB, 0, stab, false, true);
        if (r) return r;
      }
    } else {
      for (int i = 0; i < stab; ++i) {
        int r = step(PH_STAB, true);
        if (r) return r;
      }
    }
    if (track) {  // finalize (solvers.py:255-262)
      int r = cost_of_cur(COST_FINAL, ctl);
      if (r) return r;
    }
    return REDVE_OK;
  };
  GraphSlot* slot = use_graph ? &ctx->graphs[topo] : nullptr;
  if (use_graph && slot->exec && slot->owner == keybuf) {
    CK(cudaGraphLaunch(slot->exec, s));
    g_launches.fetch_add(slot->launches);
  } else if (use_graph) {
    const cudaStream_t orig = s;
    if (!ctx->cap_stream) CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    if (!ctx->fork_ev) CK(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->fork_ev, orig));
    CK(cudaStreamWaitEvent(ctx->cap_stream, ctx->fork_ev, 0));
    s = ctx->cap_stream;
    ctx->stream = s;
    const unsigned long long l0 = g_launches.load();
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    int r = device_work();
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(s, &graph);
    ctx->stream = orig;
    s = orig;
    if (r) return r;
    if (ce != cudaSuccess) return fail(ctx, REDVE_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
    bool updated = false;
    if (slot->exec) {  // same topology, other buffers: patch the node parameters
      cudaGraphExecUpdateResultInfo info;
      updated = cudaGraphExecUpdate(slot->exec, graph, &info) == cudaSuccess;
      if (!updated) {
        cudaGetLastError();
        cudaGraphExecDestroy(slot->exec);
        slot->exec = nullptr;
      }
    }
    if (!updated) {
      if (ctx->graphs.size() > 16) {  // bound the cache: drop other topologies
        for (auto it = ctx->graphs.begin(); it != ctx->graphs.end();) {
          if (&it->second != slot) {
            if (it->second.exec) cudaGraphExecDestroy(it->second.exec);
            it = ctx->graphs.erase(it);
          } else {
            ++it;
          }
        }
      }
      ce = cudaGraphInstantiate(&slot->exec, graph, 0);
    }
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) {
      slot->exec = nullptr;
      slot->owner.clear();
      return fail(ctx, REDVE_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    }
    slot->owner = keybuf;
    slot->launches = g_launches.load() - l0;
    p->captures += 1;
    CK(cudaGraphLaunch(slot->exec, s));
  } else {
    int r = device_work();
    if (r) return r;
  }
  if (spec) {  // chosen spectrum -> inverse DFT -> x_out
    View cur{p->ring.as<double>(), NE * S, NE, S, 1};
    cd* stage = p->sp_stage.as<cd>();
    RUN(ctx, "gather", launch_spec_pick(stage, cur, track ? p->best.as<double>() : nullptr, B, N,
                                        p->state.as<ImgState>(), s));
    CKL();
    if (cufftExecZ2Z(p->sp_plan, reinterpret_cast<cufftDoubleComplex*>(stage),
                     reinterpret_cast<cufftDoubleComplex*>(stage), CUFFT_INVERSE) != CUFFT_SUCCESS)
      return fail(ctx, REDVE_E_CUDA, "cufftExecZ2Z failed");
    RUN(ctx, "gather", launch_spec_real(stage, x_out, B, N, 1.0 / (double)N, s));
    CKL();
  } else {
    View cur{p->ring.as<double>(), N * S, N, S, 1};
    RUN(ctx, "gather", launch_gather(x_out, cur, track ? p->best.as<double>() : nullptr, B, N,
                                     p->state.as<ImgState>(), s));
    CKL();
  }

  // trace back to the host: one pinned copy of [trace | state | x0 flag], then
  // host copies into the caller's arrays
  const size_t sbytes = sizeof(ImgState) * B;
  const size_t need = tbytes + sbytes + sizeof(int);
  if (ctx->hstage_bytes < need) {
    if (ctx->hstage) cudaFreeHost(ctx->hstage);
    ctx->hstage = nullptr;
    ctx->hstage_bytes = 0;
    CK(cudaHostAlloc(&ctx->hstage, need, cudaHostAllocDefault));
    ctx->hstage_bytes = need;
  }
  char* hs = static_cast<char*>(ctx->hstage);
  CK(cudaMemcpyAsync(hs, p->trace.p, tbytes, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hs + tbytes, p->state.p, sbytes, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hs + tbytes + sbytes, p->x0bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (*reinterpret_cast<int*>(hs + tbytes + sbytes))
    return fail(ctx, REDVE_E_VALUE, "x0 contains non-finite entries");
  const ImgState* hst = reinterpret_cast<const ImgState*>(hs + tbytes);
  auto host_ptr = [&](const void* dptr) {
    return hs + (static_cast<const char*>(dptr) - p->trace.as<char>());
  };
  auto cp2 = [&](void* dst, const void* dsrc, size_t elem, int hcols, int dcols) {
    if (!dst) return;
    const char* src = host_ptr(dsrc);
    const size_t w = elem * (size_t)(hcols < dcols ? hcols : dcols);
    for (int b = 0; b < B; ++b)
      memcpy(static_cast<char*>(dst) + elem * hcols * (size_t)b, src + elem * dcols * (size_t)b, w);
  };
  cp2(trace->step_norm, tr.step_norm, 8, trace->cap, cap);
  cp2(trace->cost, tr.cost, 8, trace->cap, cap);
  cp2(trace->psnr, tr.psnr, 8, trace->cap, cap);
  cp2(trace->gamma_abs_sum, tr.gamma, 8, trace->cap, cap);
  cp2(trace->elapsed_s, tr.elapsed, 8, trace->cap, cap);
  cp2(trace->cycle_meta, tr.cyc_meta, 16, trace->ccap, ccap);
  cp2(trace->cycle_stability, tr.cyc_stab, 8, trace->ccap, ccap);
  cp2(trace->cycle_gamma, tr.cyc_gamma, 8 * MAXKP1, trace->ccap, ccap);
  cp2(trace->cycle_c, tr.cyc_c, 8 * MAXKP1, trace->ccap, ccap);
  cp2(trace->cg_iters, tr.cg_iters, 4, trace->cap, cap);
  for (int b = 0; b < B; ++b) {
    if (trace->n_records) trace->n_records[b] = hst[b].k;
    if (trace->n_cycles) trace->n_cycles[b] = hst[b].ncycles;
    if (trace->returned_best) trace->returned_best[b] = hst[b].use_best;
    if (trace->status)
      trace->status[b] = hst[b].err == ERR_NONE ? REDVE_OK
                         : (hst[b].err == ERR_CG ? REDVE_E_CG : REDVE_E_NONFINITE);
  }
  return REDVE_OK;
}

// ------------------------------------------------------------------ window VE
int redve_extrapolate(redve_ctx* ctx, int B, int rows, int64_t n, const double* window,
                      int method, double rank_tol, double* out, redve_ve_result* res) {
  if (rows < 3) return fail(ctx, REDVE_E_VALUE, "window needs at least kappa+2 = 3 vectors");
  if (rows - 1 > MAXKP1) return fail(ctx, REDVE_E_UNSUPPORTED, "kappa > %d", MAXKP1 - 1);
  if (method < 0 || method > 2) return fail(ctx, REDVE_E_VALUE, "unknown VE method");
  if (!(rank_tol > 0)) return fail(ctx, REDVE_E_VALUE, "rank_tolerance must be positive");
  const cudaStream_t s = ctx->stream;
  const int kp1 = rows - 1;
  CK(ctx->ve_ring.ensure(sizeof(double) * n * rows * B));
  CK(cudaMemcpyAsync(ctx->ve_ring.p, window, sizeof(double) * n * rows * B,
                     cudaMemcpyDeviceToDevice, s));
  CK(ctx->ve_state.ensure(sizeof(ImgState) * B));
  ImgState* st = ctx->ve_state.as<ImgState>();
  RUN(ctx, "init_state", launch_init_state(st, B, s));
  CKL();
  RUN(ctx, "window_extrapolate_setup", launch_window_extrapolate_setup(st, B, rows, 0, s));
  CKL();
  const int chunks = ve_chunks(B, n);
  CK(ctx->ve_partials.ensure(sizeof(double) * B * chunks * (MAXKP1 * (MAXKP1 + 1) / 2) + 64));
  CK(ctx->ve_counters.ensure(sizeof(unsigned) * B));
  CK(cudaMemsetAsync(ctx->ve_counters.p, 0, sizeof(unsigned) * B, s));
  CK(ctx->ve_q.ensure(sizeof(double) * n * kp1 * B));
  const int ccap = 1;
  CK(ctx->ve_trace.ensure(sizeof(double) * (B * 2 + (size_t)B * ccap * (1 + 2 * MAXKP1)) +
                          sizeof(int) * B * ccap * 4));
  TraceBufs tr;
  {
    double* d = ctx->ve_trace.as<double>();
    tr.cap = 1; tr.ccap = ccap;
    tr.step_norm = tr.cost = tr.psnr = tr.elapsed = d;
    tr.gamma = d + B;
    tr.cyc_stab = d + 2 * B;
    tr.cyc_gamma = tr.cyc_stab + B * ccap;
    tr.cyc_c = tr.cyc_gamma + B * ccap * MAXKP1;
    tr.cyc_meta = reinterpret_cast<int*>(tr.cyc_c + B * ccap * MAXKP1);
  }
  CK(cudaMemsetAsync(ctx->ve_trace.p, 0, ctx->ve_trace.n, s));
  VeArgs va;
  memset(&va, 0, sizeof(va));
  va.B = B; va.N = n; va.m = 0; va.kp1 = kp1; va.S = rows;
  va.ring = ctx->ve_ring.as<double>(); va.img_stride = n * rows; va.slot_stride = n;
  va.st = st; va.tr = tr; va.partials = ctx->ve_partials.as<double>();
  va.counters = ctx->ve_counters.as<unsigned>(); va.qscratch = ctx->ve_q.as<double>();
  va.method = method; va.rank_tol = rank_tol; va.chunks = chunks;
  RUN(ctx, "gram", launch_gram(va, s));
  CKL();
  std::vector<ImgState> pre(B);
  CK(cudaMemcpyAsync(pre.data(), st, sizeof(ImgState) * B, cudaMemcpyDeviceToHost, s));
  RUN(ctx, "combine", launch_combine(va, s));
  CKL();
  View curv{ctx->ve_ring.as<double>(), n * rows, n, rows, 1};
  RUN(ctx, "gather", launch_gather(out, curv, nullptr, B, n, st, s));
  CKL();
  std::vector<ImgState> post(B);
  CK(cudaMemcpyAsync(post.data(), st, sizeof(ImgState) * B, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int b = 0; b < B; ++b) {
    redve_ve_result& r = res[b];
    memset(&r, 0, sizeof(r));
    const ImgState& q = pre[b];
    r.converged = q.ve_mode == VE_CONVERGED;
    r.extrapolated = q.ve_mode == VE_EXTRAPOLATE && post[b].ncycles == 1;
    if (q.ve_mode == VE_EXTRAPOLATE) {
      r.kappa_used = q.ve_k;
      r.method = q.ve_method;
      r.fallback = q.ve_fallback;
      r.stability_sum = q.ve_stab;
      for (int i = 0; i <= q.ve_k && i < 12; ++i) {
        r.gamma[i] = q.ve_gamma[i];
        r.c[i] = q.ve_c[i];
      }
    }
  }
  return REDVE_OK;
}

// ------------------------------------------------------------------ slab primitives
// (spatially partitioned solve, BASELINE.json configs[4]; the partial sums are
// combined across ranks by the caller's allreduce)
static int slab_scratch(redve_ctx* ctx, size_t bytes) {
  CK(ctx->scratch_b.ensure(bytes));
  return REDVE_OK;
}

int redve_sr_normal_matvec(redve_ctx* ctx, const redve_operator_desc* op, double sigma,
                           double alpha, int Hext, int W, int row0, int Hg, const double* w,
                           double* out) {
  if (op->kind != REDVE_OP_BLUR_DOWNSAMPLE || op->factor < 1 || !is_odd_pos(op->ksize))
    return fail(ctx, REDVE_E_VALUE, "normal matvec needs a BlurDownsample operator");
  if (op->ksize > 31)
    return fail(ctx, REDVE_E_UNSUPPORTED, "the fused normal operator takes PSFs up to 31x31");
  if (!(sigma > 0) || !(alpha > 0)) return fail(ctx, REDVE_E_VALUE, "sigma, alpha must be > 0");
  int rc = upload_taps(ctx, op);
  if (rc) return rc;
  CK(ctx->ve_state.ensure(sizeof(CgState) + sizeof(ImgState)));
  CgArgs a;
  memset(&a, 0, sizeof(a));
  a.B = 1; a.H = Hext; a.W = W; a.factor = op->factor; a.k = op->ksize;
  a.taps = ctx->scratch_taps.as<double>();
  a.huv = ctx->taps_sep ? a.taps + (size_t)op->ksize * op->ksize : nullptr;
  a.inv_sigma2 = 1.0 / (sigma * sigma); a.alpha = alpha;
  a.row0 = row0; a.Hg = Hg;
  a.xin = plain(w, (long long)Hext * W);
  a.q = out;
  a.cg = ctx->ve_state.as<CgState>();
  a.st = reinterpret_cast<ImgState*>(ctx->ve_state.as<char>() + sizeof(CgState));
  RUN(ctx, "normal_matvec", launch_normal_matvec(a, ctx->stream));
  CKL();
  return REDVE_OK;
}

static int vec_reduce(redve_ctx* ctx, int op, int64_t n, const double* x, const double* y,
                      double* out) {
  int rc = slab_scratch(ctx, sizeof(double) * (SLAB_BLOCKS + 2));
  if (rc) return rc;
  double* part = ctx->scratch_b.as<double>();
  RUN(ctx, "vec_reduce",
      launch_vec_reduce(op, n, x, y, part, part + SLAB_BLOCKS, ctx->stream));
  CKL();
  CK(cudaMemcpyAsync(out, part + SLAB_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return REDVE_OK;
}
int redve_vec_dot(redve_ctx* ctx, int64_t n, const double* x, const double* y, double* out) {
  return vec_reduce(ctx, 0, n, x, y, out);
}
int redve_vec_dist2(redve_ctx* ctx, int64_t n, const double* x, const double* y, double* out) {
  return vec_reduce(ctx, 1, n, x, y, out);
}
int redve_vec_axpby(redve_ctx* ctx, int64_t n, double a, const double* x, double b, double* y) {
  RUN(ctx, "vec_axpby", launch_vec_axpby(n, a, x, b, y, ctx->stream));
  CKL();
  return REDVE_OK;
}

int redve_enable_peer_access(redve_ctx* ctx, int peer) {
  if (!ctx) return REDVE_E_VALUE;
  if (peer == ctx->device) return REDVE_OK;
  int can = 0;
  CK(cudaSetDevice(ctx->device));
  CK(cudaDeviceCanAccessPeer(&can, ctx->device, peer));
  if (!can) return fail(ctx, REDVE_E_UNSUPPORTED, "no peer access %d -> %d", ctx->device, peer);
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return REDVE_OK;
  }
  CK(e);
  return REDVE_OK;
}

int redve_halo_push(redve_ctx* ctx, int rows, int W, int halo, const double* x, double* ext,
                    double* prev_bot, double* next_top) {
  if (rows <= 0 || W <= 0 || halo < 0 || halo > rows)
    return fail(ctx, REDVE_E_SHAPE, "halo_push: rows=%d W=%d halo=%d", rows, W, halo);
  if (!x || !ext || (halo > 0 && (!prev_bot || !next_top)))
    return fail(ctx, REDVE_E_VALUE, "halo_push: null buffer");
  RUN(ctx, "halo_push", launch_halo_push(rows, W, halo, x, ext, prev_bot, next_top, ctx->stream));
  CKL();
  return REDVE_OK;
}

int redve_sr_fidelity(redve_ctx* ctx, const redve_operator_desc* op, int Hext, int W, int row0,
                      int Hg, int halo, int rows, const double* x_ext, const double* yup_ext,
                      double* out) {
  int rc = upload_taps(ctx, op);
  if (rc) return rc;
  if ((rc = slab_scratch(ctx, sizeof(double) * (SLAB_BLOCKS + 2)))) return rc;
  double* part = ctx->scratch_b.as<double>();
  const int f = op->kind == REDVE_OP_BLUR ? 1 : op->factor;
  RUN(ctx, "fidelity", launch_fidelity(Hext, W, row0, Hg, halo, rows, f,
                                       ctx->scratch_taps.as<double>(), op->ksize, x_ext, yup_ext,
                                       part, part + SLAB_BLOCKS, ctx->stream));
  CKL();
  CK(cudaMemcpyAsync(out, part + SLAB_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return REDVE_OK;
}

int redve_window_gram(redve_ctx* ctx, int rows, int64_t n, const double* window, double* G) {
  if (rows < 3 || rows - 1 > MAXKP1) return fail(ctx, REDVE_E_VALUE, "window rows out of range");
  const int kp1 = rows - 1, ng = kp1 * (kp1 + 1) / 2;
  int rc = slab_scratch(ctx, sizeof(double) * (GRAM_BLOCKS * ng + kp1 * kp1 + 16));
  if (rc) return rc;
  double* part = ctx->scratch_b.as<double>();
  double* Gd = part + GRAM_BLOCKS * ng;
  RUN(ctx, "window_gram", launch_window_gram(rows, n, window, part, Gd, ctx->stream));
  CKL();
  CK(cudaMemcpyAsync(G, Gd, sizeof(double) * kp1 * kp1, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return REDVE_OK;
}

static void fill_result(const VeOut& o, redve_ve_result* res, double* xi) {
  memset(res, 0, sizeof(*res));
  res->converged = o.mode == VE_CONVERGED;
  res->extrapolated = o.mode == VE_EXTRAPOLATE;
  if (o.mode == VE_EXTRAPOLATE) {
    res->kappa_used = o.k_used;
    res->method = o.method;
    res->fallback = o.fallback;
    res->stability_sum = o.stab;
    for (int i = 0; i <= o.k_used && i < 12; ++i) {
      res->gamma[i] = o.gamma[i];
      res->c[i] = o.c[i];
      if (i < o.k_used) xi[i] = o.xi[i];
    }
  }
}

int redve_ve_decide(redve_ctx* ctx, int kp1, const double* G, int method, double rank_tol,
                    redve_ve_result* res, double* xi, int* needs_mgs) {
  if (kp1 < 2 || kp1 > MAXKP1) return fail(ctx, REDVE_E_VALUE, "window order out of range");
  VeOut o;
  decide_from_gram(G, kp1, method, rank_tol, o);
  *needs_mgs = o.mode == VE_MGS;
  fill_result(o, res, xi);
  return REDVE_OK;
}

int redve_ve_decide_r(redve_ctx* ctx, int kp1, const double* R, int rank, int method,
                      redve_ve_result* res, double* xi) {
  if (kp1 < 2 || kp1 > MAXKP1) return fail(ctx, REDVE_E_VALUE, "window order out of range");
  double Rm[MAXKP1][MAXKP1];
  for (int i = 0; i < kp1; ++i)
    for (int j = 0; j < kp1; ++j) Rm[i][j] = R[i * kp1 + j];
  VeOut o;
  decide_from_r(Rm, kp1, rank, method, o);
  fill_result(o, res, xi);
  return REDVE_OK;
}

int redve_window_combine(redve_ctx* ctx, int rows, int64_t n, const double* window, int ke,
                         const double* xi, double* out) {
  if (ke < 1 || ke > rows - 2) return fail(ctx, REDVE_E_VALUE, "bad extrapolation order");
  int rc = slab_scratch(ctx, sizeof(double) * MAXKP1);
  if (rc) return rc;
  CK(cudaMemcpyAsync(ctx->scratch_b.p, xi, sizeof(double) * ke, cudaMemcpyHostToDevice,
                     ctx->stream));
  RUN(ctx, "window_combine",
      launch_window_combine(n, window, ke, ctx->scratch_b.as<double>(), out, ctx->stream));
  CKL();
  CK(cudaStreamSynchronize(ctx->stream));
  return REDVE_OK;
}

}  // extern "C"
