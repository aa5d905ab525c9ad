/*
 * redve_b200 -- C ABI of the B200-native RED fixed-point / vector-extrapolation
 * solver.  Drop-in boundary for the reference package ``redve``
 * (/root/reference/pkg/src/redve); each entry point names the reference
 * interface it replaces.  The reference is Python, so its FFI for this path
 * is ctypes: the binding a maintainer adds is shown in INTEGRATION.md and is
 * what paper_1805_02158_b200/_native.py does.
 *
 * Conventions
 *  - plain C types only: pointers, sizes, doubles, ints; no torch types.
 *  - images are fp64, row-major, batched [B][H][W] (B independent problems
 *    that share operator, denoiser, sigma and alpha, like B calls to the
 *    reference with different measurements).
 *  - array arguments of compute calls are DEVICE pointers unless the field
 *    says HOST; calls are asynchronous on the context's stream unless they
 *    return host data (then they synchronise).
 *  - every call returns REDVE_OK (0) or an error code; redve_last_error()
 *    gives the message.  Codes map to the reference exceptions:
 *      REDVE_E_VALUE      -> ValueError            (objective.py:61-66, solvers.py:162-199)
 *      REDVE_E_SHAPE      -> ShapeMismatch         (imaging.py:27-28)
 *      REDVE_E_KERNEL     -> KernelTooLarge        (imaging.py:23-24, 119-120)
 *      REDVE_E_NONFINITE  -> NonFiniteIterate      (solvers.py:37-42, 249-252)
 *      REDVE_E_CG         -> CgNoConvergence       (objective.py:40-41, 114-120)
 *      REDVE_E_CUDA / REDVE_E_UNSUPPORTED -> RuntimeError
 *  - one context per thread/stream; contexts are independent (the
 *    reference's "sessions are pure" rule).
 */
#ifndef REDVE_B200_H
#define REDVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  REDVE_OK = 0,
  REDVE_E_VALUE = 1,
  REDVE_E_SHAPE = 2,
  REDVE_E_KERNEL = 3,
  REDVE_E_CUDA = 4,
  REDVE_E_NONFINITE = 5,
  REDVE_E_CG = 6,
  REDVE_E_UNSUPPORTED = 7
};

/* forward operators: imaging.py:147-204 */
enum { REDVE_OP_BLUR = 0, REDVE_OP_BLUR_DOWNSAMPLE = 1 };
/* denoisers: denoisers.py:21-129 + BASELINE.json plug-ins */
enum {
  REDVE_DN_IDENTITY = 0,   /* Identity        denoisers.py:21-27 */
  REDVE_DN_CONV = 1,       /* GaussianFilter  denoisers.py:30-46 (any k x k taps) */
  REDVE_DN_MEDIAN3 = 2,    /* periodic 3x3 median (configs[1]) */
  REDVE_DN_FILTERBANK = 3, /* seeded reaction-diffusion stage (configs[3]) */
  REDVE_DN_PATCH = 4,      /* PatchWeighted   denoisers.py:49-129 */
  REDVE_DN_EXTERNAL = 5    /* f(x) supplied by the caller (host plug-in) */
};
/* weight rules: extrapolation.py:35-38 */
enum { REDVE_VE_MPE = 0, REDVE_VE_RRE = 1, REDVE_VE_SVDMPE = 2 };
/* drivers: solvers.py:388-399 */
enum {
  REDVE_METHOD_FP = 0,       /* run_fixed_point      solvers.py:288-298 */
  REDVE_METHOD_FP_VE = 1,    /* run_ve_cycling (fp)  solvers.py:340-385 */
  REDVE_METHOD_SD = 2,       /* run_steepest_descent solvers.py:301-312 */
  REDVE_METHOD_SD_VE = 3,    /* run_ve_cycling (sd)  solvers.py:340-385 with _sd_map :274-280 */
  REDVE_METHOD_NESTEROV = 4  /* run_nesterov         solvers.py:315-337 */
};

typedef struct redve_ctx redve_ctx;
typedef struct redve_problem redve_problem;

/* Blur(psf, shape) / BlurDownsample(psf, factor, shape)  (imaging.py:147-204) */
typedef struct {
  int kind;            /* REDVE_OP_* */
  int ksize;           /* odd PSF size (Psf.size) */
  const double* taps;  /* HOST, ksize*ksize row-major (Psf.taps) */
  int factor;          /* decimation factor; 1 for REDVE_OP_BLUR */
} redve_operator_desc;

typedef struct {
  int kind;                  /* REDVE_DN_* */
  int ksize;                 /* CONV: kernel size */
  const double* taps;        /* CONV: HOST ksize*ksize taps (GaussianFilter.psf.taps) */
  int patch_radius;          /* PATCH (PatchWeighted.__init__, denoisers.py:68-81) */
  int search_radius;
  int balance_iters;
  double h;
  int n_filters;             /* FILTERBANK */
  int fsize;
  const double* filters;     /* HOST [n_filters][fsize][fsize] */
  const double* scales;      /* HOST [n_filters] */
  double tau;
  int weight_bits;           /* PATCH: storage of the raw-weight planes, 64 (0 = default)
                                or 32 (fp32 planes, fp64 arithmetic -- BASELINE.json
                                configs[2]/[4] "fp32 with fp64 accumulation") */
} redve_denoiser_desc;

/* SolveConfig (solvers.py:162-199) */
typedef struct {
  int method;            /* REDVE_METHOD_* ("fp" / "fp-ve" / "sd" / "sd-ve" / "nesterov") */
  int ve_method;         /* REDVE_VE_* */
  int m;
  int kappa;             /* 1 <= kappa <= 11 */
  int max_inner_steps;
  double tol;
  int stabilization_iters;
  double rank_tolerance;
  double step_size;      /* SD / SD-VE / Nesterov: > 0 (ignored by fp / fp-ve) */
} redve_solve_config;

/* IterationTrace (solvers.py:51-95), HOST arrays sized by the caller:
 * per-record arrays [B][cap], per-cycle arrays [B][ccap] (x12 for vectors). */
typedef struct {
  int cap;
  int ccap;
  int32_t* n_records;       /* [B] = inner steps taken */
  double* step_norm;        /* [B][cap] */
  double* cost;             /* [B][cap], NaN off the logging cadence */
  double* psnr;             /* [B][cap], NaN off cadence / without reference */
  double* gamma_abs_sum;    /* [B][cap], NaN unless an accepted cycle closed there */
  double* elapsed_s;        /* [B][cap], device time since the solve started */
  int32_t* n_cycles;        /* [B] accepted extrapolations */
  int32_t* cycle_meta;      /* [B][ccap][4]: rule used, fallback(0/1), kappa_used, record index */
  double* cycle_stability;  /* [B][ccap] sum|gamma| */
  double* cycle_gamma;      /* [B][ccap][12] */
  double* cycle_c;          /* [B][ccap][12] */
  int32_t* status;          /* [B] REDVE_OK / REDVE_E_NONFINITE / REDVE_E_CG */
  int32_t* returned_best;   /* [B] finalize returned the best plain iterate */
  int32_t* cg_iters;        /* [B][cap] scipy-cg iterations of each fixed-point step
                               (CG route; 0 on the Fourier route), or NULL */
} redve_trace;

/* ExtrapolationResult (extrapolation.py:132-146), HOST, one per window */
typedef struct {
  int converged;
  int extrapolated;
  int kappa_used;
  int method;               /* rule actually used */
  int fallback;             /* 1 if MPE/SVD-MPE fell back to RRE */
  double stability_sum;
  double gamma[12];
  double c[12];
} redve_ve_result;

/* ---- context ------------------------------------------------------------ */
int redve_create(redve_ctx** out, int device);
void redve_destroy(redve_ctx* ctx);
const char* redve_last_error(const redve_ctx* ctx);
int redve_set_stream(redve_ctx* ctx, void* cuda_stream); /* cudaStream_t, 0 = legacy default */
int redve_synchronize(redve_ctx* ctx);
const char* redve_version(void);
/* return the library's cached device blocks to the driver */
void redve_release_cached_memory(void);
/* total kernels this library has launched (all contexts) */
uint64_t redve_kernel_launches(void);
/* time every kernel with CUDA events on the context's stream (measurement aid) */
int redve_profile(redve_ctx* ctx, int enable);
/* per-kernel-kind totals since the last report: names is max_kinds x 32 chars */
int redve_profile_report(redve_ctx* ctx, int max_kinds, char* names, double* total_ms,
                         int64_t* count, int* n_kinds);

/* ---- denoisers: f(x) for a batch (denoisers.py __call__) ------------------- */
int redve_denoise(redve_ctx* ctx, const redve_denoiser_desc* dn, int B, int H, int W,
                  const double* x, double* out);

/* PatchWeighted.weight_maps (denoisers.py:83-111): the balanced map of every
 * search offset, raster order; maps: DEVICE [B][(2 sr + 1)^2][H][W] */
int redve_patch_weight_maps(redve_ctx* ctx, const redve_denoiser_desc* dn, int B, int H, int W,
                            const double* x, double* maps);

/* ---- operators: apply / adjoint (imaging.py Blur / BlurDownsample) -------- */
int redve_operator_apply(redve_ctx* ctx, const redve_operator_desc* op, int B, int H, int W,
                         const double* x, double* out);
int redve_operator_adjoint(redve_ctx* ctx, const redve_operator_desc* op, int B, int H, int W,
                           const double* z, double* out);

/* ---- RED objective (objective.py:44-135) ---------------------------------- */
/* RedObjective(forward, y, sigma, alpha, denoiser) for B measurements.
 * y: DEVICE [B][out_h][out_w]; reference: DEVICE [B][H][W] or NULL (PSNR). */
int redve_problem_create(redve_ctx* ctx, const redve_operator_desc* op,
                         const redve_denoiser_desc* dn, int B, int H, int W, const double* y,
                         double sigma, double alpha, const double* reference,
                         redve_problem** out);
void redve_problem_destroy(redve_problem* p);
/* New measurements (and PSNR reference) for an existing problem: the same
 * operator, denoiser, sigma, alpha and shapes as a fresh RedObjective
 * (objective.py:61-74 recomputes H^T y / sigma^2 per object), but the device
 * buffers and the captured solve graph are kept, so a stream of batches pays
 * neither allocation nor graph capture.  reference must be given iff the
 * problem was created with one.  y / reference: DEVICE, shapes as in create. */
int redve_problem_set_measurements(redve_problem* p, const double* y, const double* reference);
/* Number of times redve_solve captured (and instantiated) its CUDA graph for
 * this problem.  Repeated solves with the same configuration replay one
 * capture whatever x0 / x_out buffers they pass (no reference counterpart:
 * runtime introspection for tests). */
uint64_t redve_problem_graph_captures(const redve_problem* p);
/* fp_step (objective.py:100-121); f_ext: DEVICE f(x) for REDVE_DN_EXTERNAL, else NULL */
int redve_fp_step(redve_problem* p, const double* x, double* out, const double* f_ext);
/* fp_step whose first FFT pass also writes the denoiser output it fused in,
 * f(x) -> f_out (DEVICE [B][H][W]): the in-kernel median / convolution can be
 * checked directly against the standalone denoiser.  Fourier route, stencil
 * denoisers only (REDVE_E_UNSUPPORTED otherwise). */
int redve_fp_step_denoised(redve_problem* p, const double* x, double* out, double* f_out);
/* gradient (objective.py:90-93): out = H^T (H x - y) / sigma^2 + alpha (x - f(x));
 * x, out: DEVICE [B][H][W]; f_ext as for redve_fp_step */
int redve_gradient(redve_problem* p, const double* x, const double* f_ext, double* out);
/* data_fidelity / regularizer / cost (objective.py:78-88), HOST outputs [B] each */
int redve_cost(redve_problem* p, const double* x, const double* f_ext, double* cost,
               double* data_fidelity, double* regularizer, double* psnr);
/* solve / run_fixed_point / run_ve_cycling (solvers.py:288-399), whole batch on device.
 * x0, x_out: DEVICE [B][H][W].  Per-image outcome in trace->status. */
int redve_solve(redve_problem* p, const redve_solve_config* cfg, const double* x0, double* x_out,
                redve_trace* trace);

/* ---- vector extrapolation (extrapolation.py:319-386) ---------------------- */
/* extrapolate_once on B windows of `rows` = kappa+2 iterates of length n.
 * window: DEVICE [B][rows][n]; out: DEVICE [B][n]; res: HOST [B]. */
int redve_extrapolate(redve_ctx* ctx, int B, int rows, int64_t n, const double* window,
                      int method, double rank_tolerance, double* out, redve_ve_result* res);

/* ---- slab primitives: spatially partitioned solve (configs[4]) ------------ */
/* Every rank holds rows [row0, row0 + Hext) (mod Hg) of one huge image, i.e. its
 * slab plus halos; results on rows within reach of the buffer edge are not
 * valid.  Partial sums are returned to the host for the caller's allreduce. */
/* (H^T H / sigma^2 + alpha I) w on the extended slab, measurement lattice by
 * global row (objective.py:97-98 on a slab) */
int redve_sr_normal_matvec(redve_ctx* ctx, const redve_operator_desc* op, double sigma,
                           double alpha, int Hext, int W, int row0, int Hg, const double* w,
                           double* out);
/* deterministic partial reductions (HOST out) and an in-place update */
int redve_vec_dot(redve_ctx* ctx, int64_t n, const double* x, const double* y, double* out);
int redve_vec_dist2(redve_ctx* ctx, int64_t n, const double* x, const double* y, double* out);
int redve_vec_axpby(redve_ctx* ctx, int64_t n, double a, const double* x, double b, double* y);
/* halo exchange over peer memory (replaces the neighbour send/recv of the
 * slab ring; reference: none, the reference solves one image on one CPU).
 * x: DEVICE [rows][W] slab; ext: this rank's DEVICE [rows + 2 halo][W] buffer,
 * interior rows [halo, halo + rows) <- x; prev_bot: the previous rank's bottom
 * halo (its ext + (halo + rows_prev) W) <- x's first halo rows; next_top: the
 * next rank's top halo (its ext) <- x's last halo rows.  Peer pointers are
 * CUDA-IPC mappings of the neighbours' buffers; for one rank pass this rank's
 * own ext halos (periodic wrap).  Ordering against the neighbours' readers is
 * the caller's (stream sync + barrier on both sides). */
/* let the context's device load/store the memory of device `peer` (NVLink P2P);
 * idempotent, REDVE_E_UNSUPPORTED when the pair has no peer access */
int redve_enable_peer_access(redve_ctx* ctx, int peer);
int redve_halo_push(redve_ctx* ctx, int rows, int W, int halo, const double* x, double* ext,
                    double* prev_bot, double* next_top);
/* sum over interior rows [halo, halo + rows) of ((H x) - y_up)^2 at lattice points */
int redve_sr_fidelity(redve_ctx* ctx, const redve_operator_desc* op, int Hext, int W, int row0,
                      int Hg, int halo, int rows, const double* x_ext, const double* yup_ext,
                      double* out);
/* window Gram of differences (HOST G, (rows-1)^2), decision (host), recombination */
int redve_window_gram(redve_ctx* ctx, int rows, int64_t n, const double* window, double* G);
int redve_ve_decide(redve_ctx* ctx, int kp1, const double* G, int method, double rank_tol,
                    redve_ve_result* res, double* xi, int* needs_mgs);
int redve_ve_decide_r(redve_ctx* ctx, int kp1, const double* R, int rank, int method,
                      redve_ve_result* res, double* xi);
int redve_window_combine(redve_ctx* ctx, int rows, int64_t n, const double* window, int ke,
                         const double* xi, double* out);

#ifdef __cplusplus
}
#endif

#endif /* REDVE_B200_H */
