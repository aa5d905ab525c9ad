// Per-image solver state, trace buffers and batch views (device-resident driver).
//
// Mirrors the reference recorder / cycling driver state (solvers.py:206-262,
// 340-385): iteration count, termination, best plain iterate, the ring slot of
// the current iterate and of the cycle start, and the last extrapolation
// decision.  One ImgState per image; every kernel reads it so the whole solve
// runs without host round trips (and can be captured in a CUDA graph).
#pragma once

#include "common.cuh"

namespace redve {

constexpr int MAXKP1 = 12;  // kappa + 1 <= 12  (kappa <= 11)

enum Term : int { RUNNING = 0, CONVERGED = 1, BUDGET = 2, FAILED = 3 };
enum Err : int { ERR_NONE = 0, ERR_NONFINITE_X = 1, ERR_NONFINITE_COST = 2, ERR_CG = 3 };
enum VeMode : int { VE_SKIP = 0, VE_EXTRAPOLATE = 1, VE_CONVERGED = 2, VE_MGS = 3 };
enum Phase : int { PH_MAIN = 0, PH_STAB = 1, PH_SETUP = 2 };

struct ImgState {
  int term;       // Term
  int err;        // Err
  int k;          // baseline evaluations so far (trace records)
  int cur;        // ring slot of the current iterate
  int start;      // ring slot where the current cycle started
  int pending;    // termination decided by the last record, applied at commit
  int stepped;    // took part in the current step
  int copy_best;  // cost kernel asks for best_x <- x
  int has_best;
  int use_best;   // finalize chose the best plain iterate
  int ncycles;    // accepted extrapolations
  int cg_its;     // CG iterations of the last fp step
  int ve_mode;    // VeMode of the last decision
  int ve_k;       // kappa_used
  int ve_method;  // 0 mpe, 1 rre, 2 svdmpe (rule actually used)
  int ve_fallback;
  double best_cost;
  double ve_stab;
  double ve_xi[MAXKP1];
  double ve_gamma[MAXKP1];
  double ve_c[MAXKP1];
  unsigned long long t0;
};

// Host-visible trace buffers (device memory, copied back once per solve).
struct TraceBufs {
  int cap;            // records per image
  int ccap;           // cycle records per image
  double* step_norm;  // [B][cap]
  double* cost;       // [B][cap] NaN off cadence
  double* psnr;       // [B][cap]
  double* gamma;      // [B][cap] NaN unless an accepted cycle closed here
  double* elapsed;    // [B][cap] seconds since solve start (device globaltimer)
  int* cyc_meta;      // [B][ccap][4]: method, fallback, kappa_used, record index
  double* cyc_stab;   // [B][ccap]
  double* cyc_gamma;  // [B][ccap][MAXKP1]
  double* cyc_c;      // [B][ccap][MAXKP1]
  int* cg_iters;      // [B][cap] CG iterations of each fixed-point step (CG route)
};

// A batch of images living either in a plain array or in a per-image ring.
struct View {
  double* base;
  long long img_stride;   // elements between images
  long long slot_stride;  // elements between ring slots (0 for plain)
  int S;                  // ring length (1 for plain)
  int mode;               // 0 plain, 1 current slot, 2 next slot, 3 cycle start slot
  // as at(), from a copy of image b's state
  __device__ __forceinline__ double* at_state(int b, const ImgState& s) const {
    double* p = base + (long long)b * img_stride;
    if (mode == 1) p += (long long)s.cur * slot_stride;
    else if (mode == 2) p += (long long)((s.cur + 1) % S) * slot_stride;
    else if (mode == 3) p += (long long)s.start * slot_stride;
    return p;
  }
  __device__ __forceinline__ double* at(int b, const ImgState* st) const {
    double* p = base + (long long)b * img_stride;
    if (mode == 1) p += (long long)st[b].cur * slot_stride;
    else if (mode == 2) p += (long long)((st[b].cur + 1) % S) * slot_stride;
    else if (mode == 3) p += (long long)st[b].start * slot_stride;
    return p;
  }
};

struct StepCtl {
  int phase;          // Phase
  int budget;         // max_inner_steps
  double tol;
  int log_every;      // 1 or 5
  int defer_commit;   // the cost kernel commits this step
  int track_best;
  // spectral route with tol == 0: an exactly zero step (an exact fixed point of
  // the rounded Fourier-domain map, which the reference's FFT round trips never
  // reach) does not end the run -- the reference's tol = 0 contract is "run to
  // the budget" (solvers.py:170-172)
  int zero_step_continues;
};

__device__ __forceinline__ bool takes_step(const ImgState& s, int phase) {
  if (phase == PH_SETUP) return true;
  if (phase == PH_MAIN) return s.term == RUNNING;
  return s.err == ERR_NONE;  // stabilization
}

__device__ __forceinline__ void commit_step(ImgState& s, int phase) {
  if (!s.stepped) return;
  if (s.err != ERR_NONE) {
    s.term = FAILED;
  } else if (phase == PH_MAIN && s.pending != RUNNING) {
    s.term = s.pending;
  }
  s.pending = RUNNING;
}

// --------------------------------------------------------------- record
// solvers.py:225-253 (_Recorder.record) minus the cost/psnr part (k_cost).
__device__ inline void record_step(ImgState& s, int b, double d2, double x2, double nf, int S,
                            const StepCtl& ctl, const TraceBufs& tr) {
  s.stepped = 1;
  s.k += 1;
  s.cur = (s.cur + 1) % S;
  double den = sqrt(x2);
  if (den == 0.0) den = 1.0;
  const double sn = sqrt(d2) / den;
  const long long i = (long long)b * tr.cap + (s.k - 1);
  if (s.k - 1 < tr.cap) {
    tr.step_norm[i] = sn;
    tr.elapsed[i] = (double)(globaltimer_ns() - s.t0) * 1e-9;
  }
  if (nf > 0.0) s.err = ERR_NONFINITE_X;
  s.pending = RUNNING;
  if (ctl.phase == PH_MAIN) {
    if (sn <= ctl.tol && !(ctl.zero_step_continues && sn == 0.0)) s.pending = CONVERGED;
    else if (s.k >= ctl.budget) s.pending = BUDGET;
  }
  if (!ctl.defer_commit) commit_step(s, ctl.phase);
}


}  // namespace redve
