/*
 * pmap.h -- C ABI of the B200-native parallel continuous-time MAP trajectory
 * estimator (arXiv 2512.13319, Razavi, Garcia-Fernandez, Saerkkae).
 *
 * Citations: "P:n" = line n of the paper's LaTeX source.  Readings of
 * garbled or silent passages are listed in DESIGN.md ("R-*" ids).
 *
 * Problem: a partially observed SDE
 *     dx/dt = f(x, t) + L(t) w(t),     y(t) = h(x, t) + nu(t),
 * w, nu white with spectral densities W(t), R(t), x(t0) ~ N(m0, P0).  Its MAP
 * trajectory minimises the Onsager--Machlup functional, solved as the
 * time-reversed optimal-control / LQT problem by two parallel
 * associative scans:
 *   pass 1  backward (in tau = tf - t) scan of conditional value functions
 *           (A, b, C, eta, J) with the combination rule of P:395-407
 *           == the parallel Kalman--Bucy filter in information form;
 *   pass 2  forward (in tau) scan of affine transition elements (Phi, beta)
 *            == the parallel continuous-time RTS smoother.
 * The two-filter variant and the iterated Taylor linearisation for
 * nonlinear models run on the same engine.
 *
 * Discretisation (DESIGN.md R-ELEM): one element per grid node
 * t_i = t0 + i dt, i = 0..T, dt = (tf - t0)/T:
 *   E_0 = (0, 0, 0, P0^-1 m0 + dt H0^T R0^-1 (y0 - r0), P0^-1 + dt H0^T R0^-1 H0)
 *   E_i = (I - dt F_i, -dt c_i, dt Q_i, dt H_i^T R_i^-1 (y_i - r_i), dt H_i^T R_i^-1 H_i)
 * i.e. one explicit step of the element ODEs P:416-427 from the boundary
 * (I, 0, 0, 0, 0) of P:427.  The result is the exact MAP of that discrete model.
 *
 * Conventions
 *  - Array pointers passed to the solve calls may be DEVICE or HOST memory
 *    (detected per call).  Host buffers are staged through plan-owned device
 *    buffers with cudaMemcpyAsync on the plan's stream; the call then
 *    synchronises the stream before returning.  Device buffers: the call is
 *    asynchronous on the plan's stream.
 *  - All matrices are row-major, fp64 on the host (model arrays); the y / x
 *    buffers use the plan dtype (fp64 or fp32).
 *  - Time layout: y is [batch][T+1][ny], x is [batch][T+1][nx] (node index =
 *    grid index i, i.e. original time t_i; the time reversal of P:78 is realised
 *    by the scan operator, nothing is reversed in memory, R-FLIP).
 *  - Time sharding (world > 1, shard_mode 0): rank r owns the contiguous node
 *    range [a_r, a_{r+1}), a_r = floor(r (T+1) / world); the y / x buffers of the
 *    solve calls cover only the rank's own nodes.
 *  - Ownership: the caller owns every buffer it passes and the NCCL
 *    communicator; the plan owns its workspace (no allocation during solves).
 *  - Errors: argument errors are returned synchronously; numeric failures
 *    (non-finite values, singular pivots) are flagged on the device and reported
 *    by map_sync() (or by the next blocking call) as MAP_E_NUMERIC with the first
 *    offending node in map_last_error().  No exceptions cross the ABI.
 *  - Thread safety: a plan is not thread-safe; distinct plans are independent.
 */
#ifndef PMAP_H
#define PMAP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MAP_OK = 0,
  MAP_E_ARG = 1,         /* bad shape / stride / NULL / dt <= 0 / plan kind mismatch */
  MAP_E_UNSUPPORTED = 2, /* (nx, ny) combination or mode not compiled */
  MAP_E_CUDA = 3,        /* CUDA runtime error (message in map_last_error) */
  MAP_E_NCCL = 4,        /* NCCL error or NCCL not loaded in the process */
  MAP_E_NUMERIC = 5,     /* non-finite value / zero pivot; node in map_last_error */
  MAP_E_DIVERGED = 6     /* iterated linearisation did not reach tol */
} map_status;

typedef enum { MAP_F64 = 0, MAP_F32 = 1 } map_dtype;

typedef enum {
  MAP_NL_COORD_TURN = 1, /* nx = 5, ny = 2 (range, bearing); params unused */
  MAP_NL_VAN_DER_POL = 2 /* DESIGN.md R-VDP: nx = 2, ny = 1; params[0] = mu */
} map_nl_kind;

typedef struct map_plan_s* map_plan_t;

/* map_plan_desc.flags.  MAP_FLAG_MIXED: mixed-precision pass 2 -- on the
 * look-back path of an fp64 LTI plan, the per-node recursion of pass 2 (the value-function
 * update and the forward recovery of x*, R-FWD) runs in fp32 from fp64 run carries, while
 * pass 1, every scan / look-back, the plan tables and all I/O stay fp64.  Rounding then
 * does not accumulate across runs (each restarts from fp64 values): about 1e-6 relative
 * instead of 1e-15.  Ignored on other paths. */
#define MAP_FLAG_MIXED 1
/* map_plan_desc.flags.  MAP_FLAG_BATCH_SHARD (SURVEY section 8(b) shard_mode BATCH, 8(e)
 * "replicas"): with world > 1, rank r owns the trajectories [floor(r batch / world),
 * floor((r + 1) batch / world)) of the global batch and solves them as an independent
 * single-GPU plan -- no exchange, no communicator; the y / x buffers of every call cover
 * only the rank's trajectories (all of their T + 1 nodes).  MAP_E_ARG when a rank would
 * own no trajectory.  Without the flag, world > 1 shards time (below). */
#define MAP_FLAG_BATCH_SHARD 2

typedef struct {
  int32_t nx, ny, nw;  /* state, measurement, diffusion dims */
  int32_t dtype;       /* map_dtype: compute precision and dtype of y / x buffers */
  int64_t T;           /* GLOBAL number of grid steps; nodes 0..T (dt = (tf - t0)/T) */
  int64_t batch;       /* independent trajectories sharing the model (>= 1) */
  double t0, tf;       /* time span [t0, tf], tf > t0 */
  int32_t rank, world; /* time shard index / count (world == 1: single GPU) */
  int32_t substeps;    /* 0 or 1: one exact element per grid interval (DESIGN.md R-ELEM).
                          n > 1: the paper's Euler blocks (DESIGN.md R-EULER):
                          each interval is n explicit Euler substeps of the element ODEs
                          P:416-427 (dA/ds sign corrected) with a measurement at
                          every substep, so y rows hold n*ny values ([batch][T+1][n][ny],
                          block i's substep k = fine time t_{i-1} + (k+1) dt/n; row 0 holds
                          y(t_0) in its last sub-slot).  LTI linear models only (a time-varying
                          model with n > 1 -> MAP_E_UNSUPPORTED), world == 1, RTS
                          form (map_solve_linear / map_solve_sequential); compiled for n = 10
                          at (nx, ny) = (1, 1), (4, 2) (else MAP_E_UNSUPPORTED).  x_map is
                          returned at the block boundaries t_i. */
  int32_t flags;       /* MAP_FLAG_* (0 = none) */
  void* nccl_comm;     /* ncclComm_t borrowed from the caller (e.g. torch's
                          ProcessGroupNCCL._comm_ptr()); NULL when world == 1, or
                          when the caller drives the exchange (map_shard_phase) */
  void* stream;        /* cudaStream_t borrowed from the caller; NULL = legacy default */
} map_plan_desc;

/* Linear-affine model.  HOST pointers, row-major:
 *   F nx*nx, c nx (nullable = 0), L nx*nw, W nw*nw, H ny*nx, r ny (nullable = 0),
 *   R ny*ny (SPD), m0 nx, P0 nx*nx (SPD).
 * s* = number of doubles between consecutive grid nodes (0 = constant in time,
 * otherwise the array holds T+1 node samples).  Only Q = L W L^T >= 0 is
 * required (DESIGN.md R-QPSD; the paper's invertibility assumption P:70 is not
 * needed by the scan). */
typedef struct {
  const double *F, *c, *L, *W, *H, *r, *R, *m0, *P0;
  int64_t sF, sc, sL, sW, sH, sr, sR;
} map_linear_model;

/* Nonlinear model with built-in drift / measurement functions.
 * HOST pointers: L nx*nw, W nw*nw, R ny*ny, m0 nx, P0 nx*nx; params[nparams]. */
typedef struct {
  int32_t kind;     /* map_nl_kind */
  int32_t nparams;
  const double* params;
  const double *L, *W, *R, *m0, *P0;
} map_nl_model;

/* Create a plan.  Exactly one of `lin` / `nl` is non-NULL; its dimensions must
 * match desc->nx, ny, nw.  Allocates the plan workspace on the current device.
 * MAP_E_ARG on inconsistent arguments, MAP_E_UNSUPPORTED when (nx, ny) has no
 * compiled kernel (compiled: (1,1) (2,1) (2,2) (3,1) (3,2) (4,2) (5,2)). */
map_status map_plan(const map_plan_desc* desc, const map_linear_model* lin,
                    const map_nl_model* nl, map_plan_t* out);

/* Free the plan and its workspace (synchronises its stream).  NULL is a no-op. */
void map_plan_destroy(map_plan_t plan);

/* Linear MAP by the parallel RTS form: pass 1 (filter scan)
 * + pass 2 (transition scan).  y [batch][T+1][ny] -> x_map [batch][T+1][nx].
 * Optional outputs (nullable): filt_m [batch][T+1][nx] = S_i^-1 v_i and filt_P
 * [batch][T+1][nx*(nx+1)/2] (upper triangle, row-major) = S_i^-1, the
 * Kalman--Bucy filter mean / covariance.  Linear plans only. */
map_status map_solve_linear(map_plan_t plan, const void* y, void* x_map, void* filt_m, void* filt_P);

/* Linear MAP by the parallel RTS form with the smoother covariances (SURVEY f4, P:509,
 * DESIGN.md R-SCOV): x_map as map_solve_linear, smooth_P [batch][T+1][nx*(nx+1)/2]
 * (upper triangle, row-major) = Cov(x_i | y_0..y_T), the RTS covariance recursion
 * P^s_{i-1} = Phi_i P^s_i Phi_i^T + Sigma_i (Phi_i = (I + C_i S_{i-1})^-1 A_i,
 * Sigma_i = (I + C_i S_{i-1})^-1 C_i, P^s_T = S_T^-1).  Its maps P -> Phi P Phi^T + Sigma
 * compose associatively; for a time-invariant model they are data-independent, so the
 * plan scans them over the tiles once (first call) and pass 2 runs the recursion forward
 * inside each run (R-FWD).  Single-GPU LTI plans on the look-back path; otherwise
 * MAP_E_UNSUPPORTED (map_two_filter gives smoother covariances for every linear plan). */
map_status map_solve_linear_cov(map_plan_t plan, const void* y, void* x_map, void* smooth_P);

/* Euler-block plans (substeps = n > 1): x* at EVERY fine grid point, the
 * block boundaries from the parallel RTS solve and the n - 1 points inside each block by
 * the intra-block refinement of P:485-507 (DESIGN.md R-REFINE): the value function of the
 * block's first k substeps combined with the filter at the block start, then
 * the transition P:456-459 with the forward-HJB element (first three
 * equations; n - k Euler steps in reversed time) from x* at the block end.
 * y [batch][T+1][n*ny] (Euler rows, as map_solve_linear) -> x_fine [batch][n*T+1][nx]
 * (fine point j at t0 + j (tf - t0) / (n T)).  Host or device buffers.  Other plans:
 * MAP_E_UNSUPPORTED.  Workspace for the block solution and filter outputs is allocated
 * on the first call and owned by the plan. */
map_status map_solve_linear_fine(map_plan_t plan, const void* y, void* x_fine);

/* Linear MAP by the parallel two-filter form (information-form
 * backward filter, DESIGN.md R-TF): the backward-information suffix scan runs
 * concurrently with pass 1 and the per-node combine is fused into its epilogue.
 * smooth_P (nullable) [batch][T+1][nx*(nx+1)/2] (upper triangle, row-major)
 * receives the smoother covariance (S_i + Lam_i - J_i^m)^-1: the posterior
 * precision of x_i is the sum of the forward and backward filters' information
 * (SURVEY f4).  Linear plans only; single GPU (world == 1). */
map_status map_two_filter(map_plan_t plan, const void* y, void* x_map, void* smooth_P);

/* Sequential on-device baselines: the paper's "sequential counterparts"
 * of the parallel smoothers, one GPU thread per trajectory,
 * same element sources and register algebra as the parallel path.
 *   method 0: value-function recursion V_i = E_i (x) V_{i-1} (Kalman--Bucy filter
 *             in information form) then the RTS recursion
 *             x*_{i-1} = (I + C_i S_{i-1})^-1 (A_i x*_i + b_i + C_i v_{i-1})
 *              from x*_T = S_T^-1 v_T;
 *   method 1: the same forward recursion and the backward information filter over
 *             mirrored elements, combined per node (two-filter, R-TF).
 * smooth_P (nullable, layout as in map_two_filter): smoother covariance
 * (method 0: P^s_{i-1} = Phi_i P^s_i Phi_i^T + (I + C_i S_{i-1})^-1 C_i; method 1:
 * (S_i + Lam_i - J_i^m)^-1).  Nonlinear plans: method 0 only, `passes` iterated
 * linearisation passes from xbar^(0) = m0 (R-INIT); linear plans ignore
 * `passes`.  Single GPU (world == 1).  MAP_E_ARG on a bad method / plan kind. */
map_status map_solve_sequential(map_plan_t plan, int32_t method, const void* y, int32_t passes, void* x_map,
                                void* smooth_P);

/* Nonlinear MAP by iterated Taylor linearisation (IEKS): each pass
 * re-linearises f, h about the previous estimate on the device (F_i = df(xbar_i),
 * c_i = f(xbar_i) - F_i xbar_i, H_i = dh(xbar_i), r_i = h(xbar_i) - H_i xbar_i;
 * bearing residuals wrapped to (-pi, pi], R-WRAP) and runs the parallel RTS
 * solve.  x_init [batch][T+1][nx] nullable -> xbar^(0) = m0 at every node (R-INIT).
 * tol > 0: stop after the first pass whose max |x - xbar| < tol.  The test runs on the
 * device: the pass is the body of a CUDA-graph WHILE node whose condition a one-thread
 * kernel sets from the device-side max |dx|, so the call synchronises the host once per
 * solve (to report passes_run), not once per pass.  If `passes` passes run without
 * reaching tol, x_map holds the last iterate and the call returns MAP_E_DIVERGED
 * (map_last_error gives max |dx| and the pass count).  tol == 0: run exactly `passes`
 * passes with no host synchronisation (captured as one CUDA graph).  passes_run (host,
 * nullable) receives the number of passes executed.  A host x_init is read before the
 * call returns.  Nonlinear plans only. */
map_status map_solve_nonlinear(map_plan_t plan, const void* y, int32_t passes, double tol,
                               const void* x_init, void* x_map, int32_t* passes_run);

/* Time-sharded solves (world > 1) with a caller-driven
 * exchange.  map_solve_linear on a sharded plan runs the same three phases around
 * two ncclAllGather calls on desc->nccl_comm; these entry points let the caller
 * run the exchange itself (another communicator, or single-GPU virtual shards).
 * All buffers are DEVICE buffers; calls are asynchronous on the plan's stream.
 *   phase 1: y (this rank's nodes) -> payload: the rank's pass-1 chunk aggregate
 *            (an element (A, b, C, eta, J) per trajectory).
 *   phase 2: gathered = [world][payload1] in rank order -> payload: the rank's
 *            pass-2 chunk affine aggregate (Phi, beta) (+ x*_T on the last rank).
 *   phase 3: gathered = [world][payload2] -> x_map (+ optional filter outputs).
 * Filter outputs (filt_m, filt_P) are written at phase 3 and must also be passed
 * (non-NULL) at phase 2: without them phase 2 of a low-rank-diffusion model keeps only
 * the pass-2 records (DESIGN.md R-P2REC) and phase 3 then fails with MAP_E_ARG.
 * Sharded look-back (LTI model, batch == 1, every rank holding at least one full tile,
 * DESIGN.md section 8): the same three phases with smaller payloads -- phase 1 the v-part
 * of the value function leaving the chunk and the chunk's v-map (nx + nx^2 values),
 * phase 2 x at the node before the chunk for x = 0 at its end, the chunk's x-map and
 * x*_T (2 nx + nx^2); map_shard_payload_bytes reports the plan's sizes.  Phase 3 needs y
 * again: pass it, or pass NULL and keep the phase-2 y buffer valid.  Each phase must run
 * once per solve, in order (phase 2 updates phase 1's run values in place).
 * Unused pointers may be NULL.  Linear plans only. */
int64_t map_shard_payload_bytes(map_plan_t plan, int32_t phase /* 1 or 2 */);
map_status map_shard_phase(map_plan_t plan, int32_t phase, const void* y, const void* gathered, void* payload,
                           void* x_map, void* filt_m, void* filt_P);

/* Pipelined host-buffer solve (the map_solve_linear computation): enqueues the copy of y
 * (HOST, pinned for the copies to overlap) into one of two plan-owned staging slots on a
 * copy-in stream, the solve on the plan's stream and the copy of x back to x_host on a
 * copy-out stream, and returns without waiting.  Consecutive calls overlap one solve's
 * device-to-host copy with the next one's host-to-device copy (separate copy engines), so
 * a stream of solves runs at the PCIe rate of the larger direction instead of the sum of
 * both.  y_host must stay unchanged and x_host unread until map_sync returns (map_sync
 * waits for every solve in flight and reports numeric failures).  Not combined with
 * filter outputs; device buffers: use map_solve_linear (already asynchronous). */
map_status map_solve_linear_pipelined(map_plan_t plan, const void* y_host, void* x_host);

/* Wait for the plan's stream and surface device-side numeric flags. */
map_status map_sync(map_plan_t plan);

/* Last error message of the plan ("" if none); valid until the next call on it. */
const char* map_last_error(map_plan_t plan);

/* Static description of a status code. */
const char* map_status_string(map_status s);

/* Bytes of device workspace owned by the plan. */
int64_t map_workspace_bytes(map_plan_t plan);

/* Number of kernel launches issued by the most recent solve call on this plan. */
int64_t map_last_launch_count(map_plan_t plan);

/* Per-kernel CUDA-event timing of subsequent solve calls (enable != 0), for the
 * roofline report: each kernel launch is bracketed by two events recorded on the
 * stream it is launched on.  Disabling discards pending records. */
map_status map_profile_enable(map_plan_t plan, int32_t enable);

/* Synchronise and report the device time accumulated per kernel class since the
 * last read: names[i] (static strings), ms[i] total milliseconds, launches[i]
 * count, for at most nmax classes.  Returns the number of classes written, or -1
 * on error.  Resets the accumulation. */
int32_t map_profile_read(map_plan_t plan, const char** names, double* ms, int64_t* launches, int32_t nmax);

/* Diagnostics (tools/lb_timing.py): plans created with PMAP_LB_TIMING=1 in the
 * environment record per-tile %globaltimer stamps at the phase boundaries of the two
 * look-back kernels ([2 passes][tiles][8] uint64, ns).  Copies min(n, total) stamps of
 * the last solve to `out` (host) and returns the total, 0 if not recorded, -1 on error. */
int64_t map_debug_lb_timing(map_plan_t plan, uint64_t* out, int64_t n);

/* Library version string. */
const char* map_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PMAP_H */
