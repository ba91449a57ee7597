// pmap_runner.cuh -- host-side runner of the parallel MAP solve: workspace layout,
// launch sequencing per (dtype, nx, ny, model kind) instantiation, time-shard
// exchange.  Included by the ABI translation unit and by the instantiation units.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pmap.h"
#include "pmap_kernels.cuh"
#include "pmap_tf.cuh"
#include "pmap_lti.cuh"
#include "pmap_seq.cuh"
#include "pmap_lti_scan.cuh"
#include "pmap_lb.cuh"
#include "pmap_refine.cuh"
#include <cstdlib>
#include <type_traits>

using namespace pmap;

namespace pmap_rt {

constexpr int kNT = 64;  // runs (threads) per tile
// nodes per run K is a template parameter of the runner: 32 (tiles of 2048 nodes) for
// large problems, 8 (512-node tiles) when that leaves too few tiles to fill the GPU
constexpr int kKBig = 32;
constexpr int kKSmall = 8;
// nonlinear plans: the general pass-1 reduce runs a serial chain of K general combines
// per thread plus the in-tile scan, so short runs (more threads, shorter chains) pay
constexpr int kKTiny = 4;
// Structural-zero masks compiled in (R-MASK): the Wiener-velocity model of P:519-548,
// A = I - dt F with F = [[0, I], [0, 0]] (bits (i, j) -> 4 i + j) and U = sqrt(dt) L chol(W)
// with L = [0; I] (bits (i, a) -> 2 i + a).  Any (nx, ny, nw) = (4, 2, 2) model whose
// zeros include these zeros uses the specialised kernels.
constexpr uint32_t kWienerAMask = (1u << 0) | (1u << 2) | (1u << 5) | (1u << 7) | (1u << 10) | (1u << 15);
constexpr uint32_t kWienerUMask = (1u << 4) | (1u << 7);
// ... and the value function's S (R-SMASK): the two axes decouple, S has zeros at the packed
// (i, j) with i, j on different axes (axis x = states {0, 2}, axis y = {1, 3}); used when
// J and J0 have them too (the mask is closed under the node update for these A and U).
constexpr uint32_t kWienerSMask = (1u << 0) | (1u << 2) | (1u << 4) | (1u << 6) | (1u << 7) | (1u << 9);

enum class Kind { LTI, TV, NL };

// ---------------------------------------------------------------- host algebra
// O(nx^3) model preprocessing at plan time only (never per node).
using HMat = std::vector<double>;

inline bool h_inv(int n, const double* a, double* out) {  // Gauss-Jordan, partial pivoting
  std::vector<double> m(a, a + n * n);
  for (int i = 0; i < n * n; ++i) out[i] = (i % (n + 1) == 0) ? 1.0 : 0.0;
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(m[i * n + k]) > std::fabs(m[p * n + k])) p = i;
    if (m[p * n + k] == 0.0) return false;
    for (int j = 0; j < n; ++j) {
      std::swap(m[k * n + j], m[p * n + j]);
      std::swap(out[k * n + j], out[p * n + j]);
    }
    double d = 1.0 / m[k * n + k];
    for (int j = 0; j < n; ++j) { m[k * n + j] *= d; out[k * n + j] *= d; }
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      double f = m[i * n + k];
      for (int j = 0; j < n; ++j) { m[i * n + j] -= f * m[k * n + j]; out[i * n + j] -= f * out[k * n + j]; }
    }
  }
  return true;
}

inline bool h_is_finite(const double* a, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(a[i])) return false;
  return true;
}

// ---------------------------------------------------------------- workspace
template <typename R, int N, int K>
struct WsLayout {
  size_t run_incl, tile_agg1, tile_incl1, group_agg1, group_carry1, total1, sv, run_suf, tile_agg2,
      tile_sufx2, group_agg2, group_carry2, total2, carry_in, xend, svl, tf_run, tf_tile, tf_tincl, tf_gagg, tf_gcarry, bytes;
  void plan(const Geom& g, bool tf) {
    using E = Elem<R, N>;
    using V = VF<R, N>;
    using A = Aff<R, N>;
    const size_t nt = (size_t)(g.batch * g.tpt), ng = (size_t)(g.batch * g.gpt), B = (size_t)g.batch;
    size_t off = 0;
    auto take = [&](size_t elems) {
      size_t o = off;
      off += ((elems * sizeof(R) + 255) / 256) * 256;
      return o;
    };
    run_incl = take(2 * nt * E::SZ * kNT);  // [inclusive prefixes | run aggregates]
    tile_agg1 = take(nt * E::SZ);
    tile_incl1 = take(nt * E::SZ);
    group_agg1 = take(ng * E::SZ);
    group_carry1 = take(ng * V::SZ);
    total1 = take(B * E::SZ);
    sv = take(nt * V::SZ * K * kNT);
    run_suf = take(nt * A::SZ * kNT);
    tile_agg2 = take(nt * A::SZ);
    tile_sufx2 = take(nt * A::SZ);
    group_agg2 = take(ng * A::SZ);
    group_carry2 = take(ng * N);
    total2 = take(B * (A::SZ + N));
    carry_in = take(B * V::SZ);
    xend = take(B * N);
    svl = take(B * V::SZ);  // (S, v) of every trajectory's last local node
    if (tf) {
      tf_run = take(2 * nt * E::SZ * kNT);
      tf_tile = take(nt * E::SZ);
      tf_tincl = take(nt * E::SZ);
      tf_gagg = take(ng * E::SZ);
      tf_gcarry = take(ng * V::SZ);
    } else {
      tf_run = tf_tile = tf_tincl = tf_gagg = tf_gcarry = 0;
    }
    bytes = off;
  }
};

// ------------------------------------------------------------------ runners
struct PlanState;

struct Runner {
  virtual ~Runner() {}
  virtual size_t ws_bytes(const Geom& g, bool tf) const = 0;
  virtual void set_attrs() = 0;
  // plan-time device preparation (LTI tables); returns false on failure
  virtual bool prepare(PlanState& p) = 0;
  // one parallel-RTS solve (pass 1 + pass 2); xbar only for nonlinear sources
  virtual void rts(PlanState& p, const void* y, const void* xbar, void* x, void* fm, void* fP) = 0;
  virtual size_t payload_elems(int phase) const = 0;
  virtual void phase1(PlanState& p, const void* y, const void* xbar, void* payload) = 0;
  virtual void phase2(PlanState& p, const void* y, const void* xbar, const void* gathered, void* payload) = 0;
  virtual void phase3(PlanState& p, const void* y, const void* xbar, const void* gathered, void* x, void* fm,
                      void* fP) = 0;
  virtual void two_filter(PlanState& p, const void* y, void* x, void* Ps) = 0;
  // parallel RTS with smoother covariances (false + p.err when the plan cannot)
  virtual bool rts_cov(PlanState& p, const void* y, void* x, void* Ps) = 0;
  // sequential on-device baseline: method 0 = RTS, 1 = two-filter
  virtual void sequential(PlanState& p, int method, const void* y, const void* xbar, void* x, void* Ps) = 0;
  virtual void fill_m0(PlanState& p, void* xbar) = 0;
  // out <- max |a - b| (atomicMax of the bit pattern); copy: also a <- b
  virtual void maxdiff(PlanState& p, void* a, const void* b, unsigned long long* out, bool copy) = 0;
  virtual int sizeof_real() const = 0;
  // Euler-block plans: x* at every fine point from the block solution and the filter
  // outputs at the block nodes (R-REFINE); false + p.err for other plans
  virtual bool refine(PlanState& p, const void* y, const void* xb, const void* fm, const void* fP, void* xf) {
    return false;
  }
};

struct NcclApi {
  typedef int (*allgather_t)(const void*, void*, size_t, int, void*, cudaStream_t);
  allgather_t allgather = nullptr;
  bool load() {
    if (allgather) return true;
    allgather = (allgather_t)dlsym(RTLD_DEFAULT, "ncclAllGather");
    if (!allgather) {  // torch loads libnccl RTLD_LOCAL: look it up by soname without reloading
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (h) allgather = (allgather_t)dlsym(h, "ncclAllGather");
    }
    return allgather != nullptr;
  }
};

struct PlanState {
  map_plan_desc d{};
  Kind kind = Kind::LTI;
  int nl_kind = 0;
  Geom g{};
  cudaStream_t stream = nullptr;
  std::unique_ptr<Runner> runner;
  unsigned char* ws = nullptr;
  size_t ws_bytes = 0;
  bool ws_tf = false;
  unsigned long long* dflag = nullptr;  // [0] numeric flag, [1] max diff
  void* xbuf[2] = {nullptr, nullptr};   // nonlinear ping-pong
  void* stage_y = nullptr;
  void* stage_x = nullptr;
  void* stage_aux = nullptr;
  size_t stage_y_bytes = 0, stage_x_bytes = 0, stage_aux_bytes = 0;
  void* dev_tv = nullptr;  // time-varying model arrays
  double* m0_host = nullptr;
  void* m0_dev = nullptr;
  std::string err;
  int64_t launches = 0;
  NcclApi nccl;
  // linear-solve graph cache (map_solve_linear / map_two_filter on device buffers): a key
  // seen once runs eagerly, the second time it is captured, then replayed
  struct GraphEntry {
    const void* key[6];
    cudaGraphExec_t exec;
    int64_t launches;
    bool no_graph;
  };
  std::vector<GraphEntry> lgraphs;
  // nonlinear graph cache
  cudaGraphExec_t graph = nullptr;
  const void* graph_key[4] = {nullptr, nullptr, nullptr, nullptr};
  int graph_passes = -1;
  int64_t graph_launches = 0;
  // tol > 0 nonlinear graph: one CUDA-graph WHILE node around one pass
  cudaGraphExec_t wgraph = nullptr;
  const void* wgraph_key[4] = {nullptr, nullptr, nullptr, nullptr};
  double wgraph_tol = -1.0;
  int64_t wgraph_launches = 0;
  size_t elem_real = 8;
  bool want_filter = false;  // filter outputs requested for the current solve (full (S, v) storage)
  bool rec_done = false;     // phase 2 stored low-rank pass-2 records (R-P2REC) instead of (S, v)
  bool no_rec = false;       // PMAP_NO_P2REC=1: always store (S, v) (A/B checks)
  bool euler = false;        // paper-faithful Euler blocks: y rows of ny_row = substeps * ny
  int ny_row = 0;            // doubles of y per node
  bool force_shard = false;  // PMAP_FORCE_SHARD=1 with a communicator: run the NCCL path at world == 1 (tests)
  bool no_lb = false;        // PMAP_NO_LB=1: LTI plans use the multi-kernel scan hierarchy instead of look-back
  int lb_stress = 0;         // PMAP_LB_STRESS=1: delay injection in the look-back kernels (tests)
  bool mixed = false;        // MAP_FLAG_MIXED: fp32 node recursion in pass 2 (look-back path, fp64 plans)
  const void* lb_y = nullptr;  // sharded look-back: y of phase 2, reused by phase 3 when it passes none
  size_t lb_bytes = 0;       // look-back workspace
  unsigned long long* lb_tim = nullptr;  // PMAP_LB_TIMING=1: per-tile globaltimer stamps (diagnostics)
  size_t lb_tim_n = 0;
  std::vector<double> refine_host;  // Euler blocks: intra-block refinement tables (R-REFINE), host copy
  void* refine_tab = nullptr;       // ... on the device (R), uploaded on first map_solve_linear_fine
  void* fine_ws = nullptr;          // block x, filter m, P of map_solve_linear_fine
  size_t fine_ws_bytes = 0;
  // map_solve_linear_pipelined: host-buffer solves in flight on three streams (copy in,
  // compute = stream, copy out), two staging slots each for y and x
  cudaStream_t pipe_in = nullptr, pipe_out = nullptr;
  cudaEvent_t pipe_ev_in[2] = {nullptr, nullptr}, pipe_ev_comp[2] = {nullptr, nullptr},
              pipe_ev_out[2] = {nullptr, nullptr};
  void* pipe_y[2] = {nullptr, nullptr};
  void* pipe_x[2] = {nullptr, nullptr};
  size_t pipe_y_bytes = 0, pipe_x_bytes = 0;
  int64_t pipe_k = 0;
  cudaStream_t stream2 = nullptr;  // second stream of the two-filter fork
  cudaStream_t stream3 = nullptr, stream4 = nullptr;  // boundary-tile forks of stream / stream2
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_edge0 = nullptr, ev_edge1 = nullptr, ev_edge2 = nullptr, ev_edge3 = nullptr;
  // per-kernel CUDA-event profiling (map_profile_enable / map_profile_read)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Rec { int id; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  void* scratch = nullptr;  // shard payload / gather buffers
  size_t scratch_bytes = 0;
  void* shard_scratch(size_t bytes) {
    if (scratch_bytes < bytes) {
      cudaFree(scratch);
      scratch = nullptr;
      scratch_bytes = 0;
      if (cudaMalloc(&scratch, bytes) == cudaSuccess) scratch_bytes = bytes;
    }
    return scratch;
  }
  // frees everything the plan owns (map_plan_destroy and every map_plan error return)
  ~PlanState() {
    if (stream) cudaStreamSynchronize(stream);
    if (graph) cudaGraphExecDestroy(graph);
    if (wgraph) cudaGraphExecDestroy(wgraph);
    for (auto& ge : lgraphs)
      if (ge.exec) cudaGraphExecDestroy(ge.exec);
    runner.reset();
    for (void* q : {(void*)lb_tim, (void*)ws, (void*)dflag, xbuf[0], xbuf[1], stage_y, stage_x, stage_aux, dev_tv, scratch, m0_dev,
                    refine_tab, fine_ws})
      if (q) cudaFree(q);
    for (cudaStream_t s : {pipe_in, pipe_out})
      if (s) cudaStreamSynchronize(s);
    for (void* q : {pipe_y[0], pipe_y[1], pipe_x[0], pipe_x[1]})
      if (q) cudaFree(q);
    for (cudaEvent_t e : {pipe_ev_in[0], pipe_ev_in[1], pipe_ev_comp[0], pipe_ev_comp[1], pipe_ev_out[0], pipe_ev_out[1]})
      if (e) cudaEventDestroy(e);
    for (cudaStream_t s : {stream2, stream3, stream4, pipe_in, pipe_out})
      if (s) cudaStreamDestroy(s);
    for (cudaEvent_t e : {ev_edge0, ev_edge1, ev_edge2, ev_edge3, ev_fork, ev_join})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    delete[] m0_host;
  }
  cudaEvent_t ev_get() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
};

// kernel classes reported by map_profile_read
enum KernelId { K_P1_REDUCE = 0, K_P1_REDUCE_EDGE, K_P1_TILES, K_P1_GROUPS, K_P1_DOWN, K_P2_TILES, K_P2_GROUPS,
                K_P2_DOWN, K_FILTER_OUT, K_TF_REDUCE, K_TF_REDUCE_EDGE, K_TF_TILES, K_TF_GROUPS, K_TF_DOWN, K_SHARD,
                K_NL_MISC, K_SEQ, K_LB_P1, K_LB_P2, K_P1_REDUCE_LTI, K_LB_P1B, K_REFINE, K_COUNT };
inline const char* kernel_name(int id) {
  static const char* names[K_COUNT] = {"k_p1_reduce", "k_p1_reduce_lti_edge", "k_p1_tiles", "k_p1_groups",
                                       "k_p1_down", "k_p2_tiles", "k_p2_groups", "k_p2_down", "k_filter_out",
                                       "k_tf_reduce", "k_tf_reduce_lti_edge", "k_tf_tiles", "k_tf_groups",
                                       "k_tf_down", "k_shard_*", "k_fill_m0/k_maxdiff", "k_seq_rts/k_seq_tf",
                                       "k_lb_pass1a", "k_lb_pass2", "k_p1_reduce_lti", "k_lb_pass1b",
                                       "k_euler_refine"};
  return (id >= 0 && id < K_COUNT) ? names[id] : "?";
}

// Launch a kernel on stream S, counting it and (when profiling) bracketing it with events.
#define PM_LAUNCH(p, S, ID, ...)                         \
  do {                                                   \
    cudaEvent_t _pa = nullptr;                           \
    if ((p).prof) {                                      \
      _pa = (p).ev_get();                                \
      cudaEventRecord(_pa, (S));                         \
    }                                                    \
    __VA_ARGS__;                                         \
    if ((p).prof) {                                      \
      cudaEvent_t _pb = (p).ev_get();                    \
      cudaEventRecord(_pb, (S));                         \
      (p).recs.push_back({(ID), _pa, _pb});              \
    }                                                    \
    (p).launches++;                                      \
  } while (0)

inline map_status cuda_fail(PlanState& p, cudaError_t e, const char* where) {
  p.err = std::string(where) + ": " + cudaGetErrorString(e);
  return MAP_E_CUDA;
}

#define PM_CK(p, call)                                        \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return cuda_fail((p), _e, #call);  \
  } while (0)

// fp32 copy of an LTI source (mixed-precision pass 2); other sources have none
template <class Src, class = void>
struct LbSrcF {
  using type = Src;
};
template <class Src>
struct LbSrcF<Src, std::void_t<typename Src::template rebind<float>>> {
  using type = typename Src::template rebind<float>;
};

// Euler-block sources (SrcEulerLTI) expose their substep count (R-REFINE)
template <class Src, class = void>
struct SrcIsEuler : std::false_type {};
template <class Src>
struct SrcIsEuler<Src, std::void_t<decltype(Src::NSUB_)>> : std::true_type {};

template <typename R, int N, int NY, class Src, int K>
struct RunnerT : Runner {
  Src src;
  using E = Elem<R, N>;
  using V = VF<R, N>;
  using A = Aff<R, N>;
  static constexpr bool IS_LTI = Src::IS_LTI_SRC;
  // low-rank pass-2 records (R-P2REC) when they are smaller than (S, v)
  static constexpr bool kRec = Src::LOWRANK > 0 && Src::LOWRANK * (N + 1) < VF<R, N>::SZ;
  using Tab = LtiTables<R, N, kNT, K>;
  Tab* tab = nullptr;    // pass-1 tables (LTI only)
  LtiScanTables<R, N>* scan_tab = nullptr;    // data-only tile / group scans (LTI only)
  LtiScanTables<R, N>* scan_tab_m = nullptr;  // the same for the mirrored elements (two-filter pass B)
  Tab* tab_m = nullptr;  // mirrored-element tables (two-filter pass B)
  LtiNode<R, N, NY> lnode{}, lnode_m{};
  LtiFoldParams<R, N, NY, K, Log2<kNT>::value> fold{}, fold_m{};  // kernel-parameter copies of the fold tables
  bool use_lti = false;
  // single-pass decoupled look-back path (pmap_lb.cuh), LTI single-GPU plans
  bool use_lb = false;
  LbGeom lbg{};
  LbTileTab<R, N>* lbtab = nullptr;  // [tpt] plan tables
  R* lbprod = nullptr;               // look-back window products Pa [tpt][33][N][N], Pb (triangular)
  R* lbrun = nullptr;                // [tpt][LbRunTab::F][NT] plan run tables
  R* lbcov = nullptr;                // [tpt][NS][NT] smoother covariance before each run (built on first use)
  // the model in fp32 for the mixed-precision pass 2 (MAP_FLAG_MIXED)
  std::conditional_t<IS_LTI, typename LbSrcF<Src>::type, Src> srcf{};
  std::vector<double> lb_phit;       // pass-2 tile matrices (host copy, for the covariance chain)
  unsigned char* lbws = nullptr;     // workspace
  LbWs<R> lbw{};
  double lb_amp = 0.0;               // forward-recovery amplification bound over a run (R-FWD)
  // time-sharded look-back: this rank's chunk on the look-back path,
  // two small exchanges.  lbsh: [zeros N | v_in N | probe1 N | probe2 N | x_end N |
  // Gc N*N (v-map of the chunk) | Pc N*N (x-map of the chunk) | Phi_tile0 N*N]
  bool lb_shard = false;
  R* lbsh = nullptr;

  ~RunnerT() override {
    cudaFree(tab);
    cudaFree(tab_m);
    cudaFree(scan_tab);
    cudaFree(scan_tab_m);
    cudaFree(lbtab);
    cudaFree(lbprod);
    cudaFree(lbrun);
    cudaFree(lbcov);
    cudaFree(lbws);
    cudaFree(lbsh);
  }

  bool prepare(PlanState& p) override;
  bool prepare_lb(PlanState& p);

  // one look-back solve: k_lb_pass1a + k_lb_pass1b + k_lb_pass2 (3 launches); Ps != null:
  // smoother covariances (pass 2 with OUT = 2, plan tables built on first use)
  void lb_rts(PlanState& p, const void* yv, void* xv, void* fm, void* fP, void* Ps = nullptr) {
    if constexpr (IS_LTI) {
      const R* y = static_cast<const R*>(yv);
      R* x = static_cast<R*>(xv);
      const unsigned ntiles = (unsigned)(lbg.batch * lbg.tpt);
      cudaStream_t s = p.stream;
      PM_LAUNCH(p, s, K_LB_P1,
                (k_lb_pass1a<R, N, NY, kNT, K, Src><<<ntiles, kNT, 0, s>>>(fold, lbg, y, tab, lbtab, lbrun, lbw)));
      const unsigned n1b = (unsigned)((lb_ticket_count(ntiles, lbg.S1) + 3) / 4);
      const unsigned n2 = (unsigned)lb_ticket_count(ntiles, lbg.S2);
      PM_LAUNCH(p, s, K_LB_P1B,
                (k_lb_pass1b<R, N, NY, kNT, K, Src><<<n1b, 128, 0, s>>>(src, lbg, y, tab, lbtab, lbrun, lbw, p.dflag,
                                                                      p.lb_stress, nullptr, 0, nullptr)));
      if (Ps)
        PM_LAUNCH(p, s, K_LB_P2,
                  (k_lb_pass2<R, N, NY, kNT, K, Src, 2><<<n2, kNT, 0, s>>>(src, lbg, y, lbrun, lbw, x, nullptr,
                                                                         static_cast<R*>(Ps), lbcov, p.dflag,
                                                                         p.lb_stress, nullptr, 1, 0, nullptr,
                                                                         nullptr)));
      else if (fm || fP)
        PM_LAUNCH(p, s, K_LB_P2,
                  (k_lb_pass2<R, N, NY, kNT, K, Src, 1><<<n2, kNT, 0, s>>>(
                      src, lbg, y, lbrun, lbw, x, static_cast<R*>(fm), static_cast<R*>(fP), nullptr, p.dflag,
                      p.lb_stress, nullptr, 1, 0, nullptr, nullptr)));
      else if (p.mixed && std::is_same<R, double>::value)  // MAP_FLAG_MIXED: fp32 node recursion
        PM_LAUNCH(p, s, K_LB_P2,
                  (k_lb_pass2<R, N, NY, kNT, K, Src, 0, float><<<n2, kNT, 0, s>>>(
                      srcf, lbg, y, lbrun, lbw, x, nullptr, nullptr, nullptr, p.dflag, p.lb_stress, nullptr, 1, 0,
                      nullptr, nullptr)));
      else
        PM_LAUNCH(p, s, K_LB_P2,
                  (k_lb_pass2<R, N, NY, kNT, K, Src, 0><<<n2, kNT, 0, s>>>(src, lbg, y, lbrun, lbw, x, nullptr, nullptr,
                                                                         nullptr, p.dflag, p.lb_stress, nullptr, 1,
                                                                         0, nullptr, nullptr)));
    }
  }

  // ---- time-sharded look-back.  Rank r > 0 views its chunk with the
  // node before it (owned by rank r - 1) as local node 0, the carry-in; buffers are offset
  // by one node so the kernels keep their geometry.
  //   phase 1: k_lb_pass1a, then k_lb_pass1b in probe mode (last tile, v_in = 0 on r > 0,
  //            the true prior on rank 0) -> payload [v leaving the chunk | Gc]
  //   phase 2: v_in = fold of the gathered ranks < r; k_lb_pass1b with it; k_lb_pass2 in
  //            probe mode (tile 0, x at the chunk's end = 0) -> payload [x at local node 0
  //            | Pc | x*_T (meaningful on the last rank)]
  //   phase 3: x at the chunk's end = fold of the gathered ranks > r onto the last rank's
  //            x*_T; k_lb_pass2 from it.
  static constexpr size_t lbsh_elems() { return 5 * N + 3 * N * N; }
  size_t lb_payload(int phase) const { return phase == 1 ? (size_t)(N + N * N) : (size_t)(2 * N + N * N); }
  const R* lb_yview(PlanState& p, const void* y) const {
    return static_cast<const R*>(y) - (p.d.rank > 0 ? NY : 0);
  }
  R* lb_xview(PlanState& p, void* x, int w) const { return x ? static_cast<R*>(x) - (p.d.rank > 0 ? w : 0) : nullptr; }
  void lb_phase1(PlanState& p, const void* yv, void* payload) {
    if constexpr (IS_LTI) {
      const R* y = lb_yview(p, yv);
      cudaStream_t s = p.stream;
      const unsigned ntiles = (unsigned)(lbg.batch * lbg.tpt);
      PM_LAUNCH(p, s, K_LB_P1,
                (k_lb_pass1a<R, N, NY, kNT, K, Src><<<ntiles, kNT, 0, s>>>(fold, lbg, y, tab, lbtab, lbrun, lbw)));
      PM_LAUNCH(p, s, K_LB_P1B,
                (k_lb_pass1b<R, N, NY, kNT, K, Src><<<1, 128, 0, s>>>(src, lbg, y, tab, lbtab, lbrun, lbw, p.dflag, 0,
                                                                    p.d.rank > 0 ? lbsh : nullptr, 1,
                                                                    lbsh + 2 * N)));
      if (payload) {
        cudaMemcpyAsync(payload, lbsh + 2 * N, sizeof(R) * N, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(static_cast<R*>(payload) + N, lbsh + 5 * N, sizeof(R) * N * N, cudaMemcpyDeviceToDevice, s);
      }
    }
  }
  void lb_phase2(PlanState& p, const void* yv, const void* gathered, void* payload) {
    if constexpr (IS_LTI) {
      const R* y = lb_yview(p, yv);
      p.lb_y = yv;
      cudaStream_t s = p.stream;
      const unsigned ntiles = (unsigned)(lbg.batch * lbg.tpt);
      const unsigned n1b = (unsigned)((lb_ticket_count(ntiles, lbg.S1) + 3) / 4);
      if (p.d.rank > 0)
        PM_LAUNCH(p, s, K_SHARD,
                  (k_lb_shard_vin<R, N><<<1, 1, 0, s>>>(static_cast<const R*>(gathered), p.d.rank, lbsh + N)));
      PM_LAUNCH(p, s, K_LB_P1B,
                (k_lb_pass1b<R, N, NY, kNT, K, Src><<<n1b, 128, 0, s>>>(src, lbg, y, tab, lbtab, lbrun, lbw, p.dflag,
                                                                      p.lb_stress, p.d.rank > 0 ? lbsh + N : nullptr,
                                                                      0, nullptr)));
      PM_LAUNCH(p, s, K_LB_P2,
                (k_lb_pass2<R, N, NY, kNT, K, Src, 0><<<1, kNT, 0, s>>>(src, lbg, y, lbrun, lbw, nullptr, nullptr,
                                                                      nullptr, nullptr, p.dflag, 0, lbsh, 0, 1,
                                                                      lbsh + 3 * N, lbsh + 5 * N + 2 * N * N)));
      if (payload) {
        R* pl = static_cast<R*>(payload);
        cudaMemcpyAsync(pl, lbsh + 3 * N, sizeof(R) * N, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(pl + N, lbsh + 5 * N + N * N, sizeof(R) * N * N, cudaMemcpyDeviceToDevice, s);
        cudaMemcpyAsync(pl + N + N * N, lbw.seed, sizeof(R) * N, cudaMemcpyDeviceToDevice, s);
      }
    }
  }
  void lb_phase3(PlanState& p, const void* yv, const void* gathered, void* xv, void* fm, void* fP) {
    if constexpr (IS_LTI) {
      if (!yv) yv = p.lb_y;
      if (!yv) {
        p.err = "map_shard_phase: the look-back shard path needs y at phase 3 (or the phase-2 y still valid)";
        return;
      }
      const R* y = lb_yview(p, yv);
      R* x = lb_xview(p, xv, N);
      cudaStream_t s = p.stream;
      const unsigned ntiles = (unsigned)(lbg.batch * lbg.tpt);
      const unsigned n2 = (unsigned)lb_ticket_count(ntiles, lbg.S2);
      PM_LAUNCH(p, s, K_SHARD,
                (k_lb_shard_xend<R, N><<<1, 1, 0, s>>>(static_cast<const R*>(gathered), p.d.rank, p.d.world,
                                                       lbsh + 4 * N)));
      const int store0 = p.d.rank == 0 ? 1 : 0;
      if (fm || fP)
        PM_LAUNCH(p, s, K_LB_P2,
                  (k_lb_pass2<R, N, NY, kNT, K, Src, 1><<<n2, kNT, 0, s>>>(
                      src, lbg, y, lbrun, lbw, x, lb_xview(p, fm, N), lb_xview(p, fP, Dim<N>::NS), nullptr, p.dflag,
                      p.lb_stress, lbsh + 4 * N, store0, 0, nullptr, nullptr)));
      else
        PM_LAUNCH(p, s, K_LB_P2,
                  (k_lb_pass2<R, N, NY, kNT, K, Src, 0><<<n2, kNT, 0, s>>>(src, lbg, y, lbrun, lbw, x, nullptr, nullptr,
                                                                         nullptr, p.dflag, p.lb_stress, lbsh + 4 * N,
                                                                         store0, 0, nullptr, nullptr)));
    }
  }

  bool refine(PlanState& p, const void* y, const void* xb, const void* fm, const void* fP, void* xf) override {
    if constexpr (!SrcIsEuler<Src>::value) {
      p.err = "map_solve_linear_fine needs a plan with Euler blocks (substeps > 1)";
      return false;
    } else {
      constexpr int NSUB = Src::NSUB_, NYM = Src::NYM_;
      const Geom& g = p.g;
      const int64_t T = g.Nn - 1;
      if (!p.refine_tab) {  // plan tables in R, uploaded once
        std::vector<R> h(p.refine_host.size());
        for (size_t k = 0; k < h.size(); ++k) h[k] = (R)p.refine_host[k];
        if (cudaMalloc(&p.refine_tab, sizeof(R) * h.size()) != cudaSuccess ||
            cudaMemcpy(p.refine_tab, h.data(), sizeof(R) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
          p.err = "refinement tables: device allocation failed";
          return false;
        }
      }
      rts(p, y, nullptr, const_cast<void*>(xb), const_cast<void*>(fm), const_cast<void*>(fP));
      const int64_t n = g.batch * T;
      if (n > 0)
        PM_LAUNCH(p, p.stream, K_REFINE,
                  (k_euler_refine<R, N, NYM, NSUB><<<(unsigned)((n + 127) / 128), 128, 0, p.stream>>>(
                      static_cast<const R*>(p.refine_tab), T, g.batch, static_cast<const R*>(y),
                      static_cast<const R*>(xb), static_cast<const R*>(fm), static_cast<const R*>(fP),
                      static_cast<R*>(xf), p.dflag)));
      return true;
    }
  }

  // Parallel RTS with smoother covariances (map_solve_linear_cov): look-back plans only.
  bool rts_cov(PlanState& p, const void* y, void* x, void* Ps) override {
    if (!(use_lb && p.d.world == 1 && !p.force_shard && !p.no_lb)) {
      p.err = "smoother covariances of the parallel RTS need a single-GPU LTI look-back plan (map_two_filter gives them "
              "for every linear plan)";
      return false;
    }
    if (!lbcov && !prepare_lb_cov(p)) {
      p.err = "plan tables of the smoother covariance failed";
      return false;
    }
    lb_rts(p, y, x, nullptr, nullptr, Ps);
    return true;
  }
  bool prepare_lb_cov(PlanState& p);

  // interior (LTI-specialised) tile range [j_lo, j_hi) of a trajectory
  static int64_t lti_jlo(const Geom& g, bool rev) { return (rev || g.node0 == 0) ? 1 : 0; }
  static int64_t lti_jhi(const Geom& g) { return g.Nn / ((int64_t)kNT * K); }

  // Pass-1 reduce: LTI-specialised kernel on interior tiles, general kernel on the
  // boundary tiles (node 0 / terminal node, ragged last tile); all tiles otherwise.
  template <bool REV, class KS>
  void reduce1(PlanState& p, cudaStream_t s, int kid, const KS& ksrc,
               const LtiFoldParams<R, N, NY, K, Log2<kNT>::value>& fpar,
               const Tab* tb, const R* y, const R* xbar, R* run_incl, R* tile_agg) {
    const Geom& g = p.g;
    if (!(use_lti && tb)) {
      PM_LAUNCH(p, s, kid,
                (k_p1_reduce<R, N, NY, kNT, K, KS, REV><<<(unsigned)(g.batch * g.tpt), kNT, smem_reduce(), s>>>(
                    ksrc, g, y, xbar, run_incl, tile_agg, p.dflag, 0, 0, 0)));
      return;
    }
    if constexpr (IS_LTI) {
    const LtiNode<R, N, NY>& ln = fpar.node;
    const int64_t j_lo = lti_jlo(g, REV);
    const int64_t j_hi = lti_jhi(g);
    const int64_t n_int = j_hi > j_lo ? j_hi - j_lo : 0;
    int nsel = 0;
    int64_t js[2] = {0, 0};
    if (j_lo == 1) js[nsel++] = 0;
    if (j_hi < g.tpt && !(nsel == 1 && js[0] == g.tpt - 1)) js[nsel++] = g.tpt - 1;
    // boundary tiles on a forked stream, concurrently with the interior tiles
    cudaStream_t se = (s == p.stream) ? p.stream3 : p.stream4;
    cudaEvent_t e0 = (s == p.stream) ? p.ev_edge0 : p.ev_edge2, e1 = (s == p.stream) ? p.ev_edge1 : p.ev_edge3;
    if (nsel > 0) {
      cudaEventRecord(e0, s);
      cudaStreamWaitEvent(se, e0, 0);
      PM_LAUNCH(p, se, kid + 1,
                (k_p1_reduce_lti_edge<R, N, NY, kNT, K, KS, REV><<<(unsigned)(g.batch * nsel), kNT, smem_reduce(),
                                                                    se>>>(ksrc, ln, g, nsel, js[0], js[1], y, tb,
                                                                          run_incl, tile_agg, p.dflag)));
    }
    if (n_int > 0)
      PM_LAUNCH(p, s, kid == K_P1_REDUCE ? (int)K_P1_REDUCE_LTI : kid,
                (k_p1_reduce_lti<R, N, NY, kNT, K, REV><<<(unsigned)(g.batch * n_int), kNT, 0, s>>>(
                    fpar, g, j_lo, n_int, y, tb, run_incl, tile_agg)));
    if (nsel > 0) {
      cudaEventRecord(e1, se);
      cudaStreamWaitEvent(s, e1, 0);
    }
    }
  }

  // in-tile run-scan tables for the down-sweeps (reduce stores run aggregates only, R-LTI)
  const R* uwc(bool rev) const {
#ifndef PM_REDUCE_TREE
    (void)rev;
    return nullptr;
#else
    const Tab* t = rev ? tab_m : tab;
    return (use_lti && t) ? t->UWc : nullptr;
#endif
  }
  const R* ux(bool rev) const {
    const Tab* t = rev ? tab_m : tab;
    return (use_lti && t) ? &t->UX[0][0][0][0] : nullptr;
  }
  // Scans of tile aggregates within groups and of group aggregates (carries): the
  // data-only LTI kernels (pmap_lti_scan.cuh) when the plan has their tables and the
  // trajectory has at most kScanB groups, else the general kernels.
  bool lti_scan(const PlanState& p, bool rev) const {
    const char* e = getenv("PMAP_NO_LTI_SCAN");
    return use_lti && (rev ? scan_tab_m : scan_tab) && p.g.gpt <= kScanB && smem_scan() <= 180 * 1024 &&
           !(e && e[0] == '1');
  }
  void tiles1(PlanState& p, cudaStream_t s, int kid, bool rev, R* tile_agg, R* tile_incl, R* group_agg) {
    const Geom& g = p.g;
    if (lti_scan(p, rev))
      PM_LAUNCH(p, s, kid,
                (k_p1_tiles_lti<R, N><<<(unsigned)(g.batch * g.gpt), kScanB, smem_scan(), s>>>(
                    g, tile_agg, tile_incl, group_agg, rev ? scan_tab_m : scan_tab, lti_jlo(g, rev), lti_jhi(g),
                    p.dflag)));
    else
      PM_LAUNCH(p, s, kid,
                (k_p1_tiles<R, N><<<(unsigned)(g.batch * g.gpt), NT2, smem_tiles(), s>>>(g, tile_agg, tile_incl,
                                                                                         group_agg, p.dflag)));
  }
  void groups1(PlanState& p, cudaStream_t s, int kid, bool rev, R* group_agg, const R* gathered, R* carry_out,
               R* group_carry, R* total) {
    const Geom& g = p.g;
    if (lti_scan(p, rev))
      PM_LAUNCH(p, s, kid,
                (k_p1_groups_lti<R, N><<<(unsigned)g.batch, kScanB, smem_scan(), s>>>(
                    g, group_agg, gathered, p.d.rank, carry_out, group_carry, total, rev ? scan_tab_m : scan_tab,
                    lti_jlo(g, rev), lti_jhi(g), p.dflag)));
    else
      PM_LAUNCH(p, s, kid,
                (k_p1_groups<R, N><<<(unsigned)g.batch, NT3, smem_groups(), s>>>(
                    g, group_agg, gathered, p.d.rank, carry_out, group_carry, total, p.dflag)));
  }

  size_t ws_bytes(const Geom& g, bool tf) const override {
    WsLayout<R, N, K> L;
    L.plan(g, tf);
    return L.bytes;
  }
  int sizeof_real() const override { return (int)sizeof(R); }

  static size_t smem_reduce() { return sizeof(R) * E::SZ * kNT; }
  static size_t smem_scan() { return sizeof(R) * E::SZ * kScanB; }
  static size_t smem_tiles() { return sizeof(R) * E::SZ * NT2; }
  static size_t smem_groups() { return sizeof(R) * E::SZ * NT3; }
  static size_t smem_down() { return sizeof(R) * (A::SZ * kNT > V::SZ ? A::SZ * kNT : V::SZ); }
  static size_t smem_p2tiles() { return sizeof(R) * A::SZ * NT2; }
  static size_t smem_p2groups() { return sizeof(R) * (A::SZ * NT4 + N); }

  void set_attrs() override {
    cudaFuncSetAttribute(k_p1_reduce<R, N, NY, kNT, K, Src, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_reduce());
    cudaFuncSetAttribute(k_p1_tiles<R, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tiles());
    cudaFuncSetAttribute(k_p1_groups<R, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_groups());
    cudaFuncSetAttribute(k_p1_down<R, N, NY, kNT, K, Src, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_down());
    cudaFuncSetAttribute(k_p2_tiles<R, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_p2tiles());
    cudaFuncSetAttribute(k_p2_groups<R, N, kNT, K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem_p2groups());
    if constexpr (IS_LTI) {
      if (smem_scan() <= 180 * 1024) {
        cudaFuncSetAttribute(k_p1_tiles_lti<R, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_scan());
        cudaFuncSetAttribute(k_p1_groups_lti<R, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_scan());
      }
      // the LTI reduce is latency bound: let as many 17.5 KB CTAs reside as registers allow
      cudaFuncSetAttribute(k_p1_reduce_lti<R, N, NY, kNT, K, false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           100);
      cudaFuncSetAttribute(k_p1_reduce_lti<R, N, NY, kNT, K, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           100);
      cudaFuncSetAttribute(k_p1_reduce_lti_edge<R, N, NY, kNT, K, Src, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_reduce());
      cudaFuncSetAttribute(k_p1_reduce_lti_edge<R, N, NY, kNT, K, Mirror<Src>, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_reduce());
    }
    if constexpr (Src::HAS_MIRROR) {
      cudaFuncSetAttribute(k_p1_reduce<R, N, NY, kNT, K, Mirror<Src>, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_reduce());
      cudaFuncSetAttribute(k_p1_down<R, N, NY, kNT, K, Src, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem_down());
      cudaFuncSetAttribute(k_tf_down<R, N, NY, kNT, K, Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem_down());
    }
  }

  // ---------------------------------------------------------------------------
  // Parallel RTS solve (pass 1 + pass 2).  Time-sharded plans (world > 1) run it
  // as three phases around two all-gathers of chunk carries:
  //   phase 1: local pass-1 reduce -> payload1 = this rank's chunk aggregate
  //   phase 2: fold gathered aggregates of ranks < r into the carry (S, v), local
  //            pass-1 down-sweep + pass-2 reduce -> payload2 = chunk affine aggregate
  //            (+ x*_T on the last rank)
  //   phase 3: fold gathered affine aggregates of ranks > r onto x*_T, local pass 2.
  // map_solve_linear drives the exchange with ncclAllGather; map_shard_phase lets
  // the caller drive it (other communicators, single-GPU virtual shards in tests).
  size_t payload_elems(int phase) const override {
    if (lb_shard) return lb_payload(phase);
    return phase == 1 ? (size_t)E::SZ : (size_t)(A::SZ + N);
  }

  void phase1(PlanState& p, const void* yv, const void* xbarv, void* payload) override {
    if (lb_shard) {
      lb_phase1(p, yv, payload);
      return;
    }
    const Geom& g = p.g;
    WsLayout<R, N, K> L;
    L.plan(g, p.ws_tf);
    auto W = [&](size_t off) { return reinterpret_cast<R*>(p.ws + off); };
    const R* y = static_cast<const R*>(yv);
    const R* xbar = static_cast<const R*>(xbarv);
    cudaStream_t s = p.stream;
    reduce1<false>(p, s, K_P1_REDUCE, src, fold, tab, y, xbar, W(L.run_incl), W(L.tile_agg1));
    tiles1(p, s, K_P1_TILES, false, W(L.tile_agg1), W(L.tile_incl1), W(L.group_agg1));
    if (payload)  // chunk aggregate only (group carries are recomputed in phase 2)
      groups1(p, s, K_P1_GROUPS, false, W(L.group_agg1), nullptr, nullptr, W(L.group_carry1),
              static_cast<R*>(payload));
  }

  void phase2(PlanState& p, const void* yv, const void* xbarv, const void* gathered, void* payload) override {
    if (lb_shard) {
      lb_phase2(p, yv, gathered, payload);
      return;
    }
    const Geom& g = p.g;
    WsLayout<R, N, K> L;
    L.plan(g, p.ws_tf);
    auto W = [&](size_t off) { return reinterpret_cast<R*>(p.ws + off); };
    const R* y = static_cast<const R*>(yv);
    const R* xbar = static_cast<const R*>(xbarv);
    const unsigned ntiles = (unsigned)(g.batch * g.tpt);
    cudaStream_t s = p.stream;
    groups1(p, s, K_P1_GROUPS, false, W(L.group_agg1), static_cast<const R*>(gathered), W(L.carry_in),
            W(L.group_carry1), nullptr);
    const R* span1 = (use_lti && tab) ? tab->E1 : nullptr;
    const R* sf = (use_lti && tab) ? &tab->SF[0][0] : nullptr;
    p.rec_done = false;
    if constexpr (kRec) p.rec_done = !p.want_filter && !p.no_rec;
    if (p.rec_done) {
      if constexpr (kRec)
        PM_LAUNCH(p, s, K_P1_DOWN,
                  (k_p1_down<R, N, NY, kNT, K, Src, true, true><<<ntiles, kNT, smem_down(), s>>>(
                      src, g, y, xbar, W(L.run_incl), W(L.tile_incl1), W(L.group_carry1), W(L.sv), W(L.run_suf),
                      W(L.tile_agg2), p.dflag, span1, sf, lti_jlo(g, false), lti_jhi(g), W(L.svl), uwc(false), ux(false))));
    } else {
      PM_LAUNCH(p, s, K_P1_DOWN,
                (k_p1_down<R, N, NY, kNT, K, Src, true><<<ntiles, kNT, smem_down(), s>>>(
                    src, g, y, xbar, W(L.run_incl), W(L.tile_incl1), W(L.group_carry1), W(L.sv), W(L.run_suf),
                    W(L.tile_agg2), p.dflag, span1, sf, lti_jlo(g, false), lti_jhi(g), W(L.svl), uwc(false), ux(false))));
    }
    PM_LAUNCH(p, s, K_P2_TILES,
              (k_p2_tiles<R, N><<<(unsigned)(g.batch * g.gpt), NT2, smem_p2tiles(), s>>>(
                  g, W(L.tile_agg2), W(L.tile_sufx2), W(L.group_agg2))));
    if (payload) {
      PM_LAUNCH(p, s, K_P2_GROUPS,
                (k_p2_groups<R, N, kNT, K><<<(unsigned)g.batch, NT4, smem_p2groups(), s>>>(
                    g, W(L.svl), W(L.group_agg2), nullptr, p.d.rank, p.d.world, W(L.group_carry2),
                    static_cast<R*>(payload), p.dflag)));
    }
  }

  void phase3(PlanState& p, const void* yv, const void* xbarv, const void* gathered, void* xv, void* fm,
              void* fP) override {
    if (lb_shard) {
      lb_phase3(p, yv, gathered, xv, fm, fP);
      return;
    }
    const Geom& g = p.g;
    WsLayout<R, N, K> L;
    L.plan(g, p.ws_tf);
    auto W = [&](size_t off) { return reinterpret_cast<R*>(p.ws + off); };
    const R* xbar = static_cast<const R*>(xbarv);
    const R* y = static_cast<const R*>(yv);
    R* x = static_cast<R*>(xv);
    const unsigned ntiles = (unsigned)(g.batch * g.tpt);
    cudaStream_t s = p.stream;
    PM_LAUNCH(p, s, K_P2_GROUPS,
              (k_p2_groups<R, N, kNT, K><<<(unsigned)g.batch, NT4, smem_p2groups(), s>>>(
                  g, W(L.svl), W(L.group_agg2), static_cast<const R*>(gathered), p.d.rank, p.d.world,
                  W(L.group_carry2), nullptr, p.dflag)));
    if ((fm || fP) && p.rec_done) {
      p.err = "filter outputs need full (S, v) storage: pass filt_m/filt_P at phase 2 as well";
      return;
    }
    if (p.rec_done) {
      if constexpr (kRec)
        PM_LAUNCH(p, s, K_P2_DOWN,
                  (k_p2_down<R, N, kNT, K, Src, true><<<ntiles, kNT, 0, s>>>(src, g, y, xbar, W(L.sv), W(L.run_suf),
                                                                           W(L.tile_sufx2), W(L.group_carry2),
                                                                           W(L.carry_in), x, p.dflag)));
    } else {
      PM_LAUNCH(p, s, K_P2_DOWN,
                (k_p2_down<R, N, kNT, K, Src><<<ntiles, kNT, 0, s>>>(src, g, y, xbar, W(L.sv), W(L.run_suf),
                                                                    W(L.tile_sufx2), W(L.group_carry2),
                                                                    W(L.carry_in), x, p.dflag)));
    }
    if (fm || fP) {
      const int64_t n = g.batch * g.Nn;
      PM_LAUNCH(p, s, K_FILTER_OUT,
                (k_filter_out<R, N, kNT, K><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(g, W(L.sv), (R*)fm,
                                                                                        (R*)fP, p.dflag)));
    }
  }

  void rts(PlanState& p, const void* y, const void* xbar, void* x, void* fm, void* fP) override {
    p.want_filter = fm || fP;
    if (use_lb && p.d.world == 1 && !p.force_shard && !p.no_lb) {
      lb_rts(p, y, x, fm, fP);
      return;
    }
    if (p.d.world == 1 && !p.force_shard) {
      phase1(p, y, xbar, nullptr);
      phase2(p, y, xbar, nullptr, nullptr);
      phase3(p, y, xbar, nullptr, x, fm, fP);
      return;
    }
    // NCCL-driven exchange: two all-gathers of chunk carries per solve
    const size_t per1 = (size_t)p.g.batch * payload_elems(1), per2 = (size_t)p.g.batch * payload_elems(2);
    R* buf = static_cast<R*>(p.shard_scratch(((per1 + per2) * (p.d.world + 1)) * sizeof(R)));
    R* pay1 = buf;
    R* gat1 = pay1 + per1;
    R* pay2 = gat1 + per1 * p.d.world;
    R* gat2 = pay2 + per2;
    const int nt = sizeof(R) == 8 ? 8 /*ncclFloat64*/ : 7 /*ncclFloat32*/;
    phase1(p, y, xbar, pay1);
    if (!p.nccl.load() || p.nccl.allgather(pay1, gat1, per1, nt, p.d.nccl_comm, p.stream) != 0) {
      p.err = "ncclAllGather failed or NCCL not loaded in the process";
      return;
    }
    phase2(p, y, xbar, gat1, pay2);
    if (p.nccl.allgather(pay2, gat2, per2, nt, p.d.nccl_comm, p.stream) != 0) {
      p.err = "ncclAllGather failed";
      return;
    }
    phase3(p, y, xbar, gat2, x, fm, fP);
  }

  // Two-filter (R-TF): pass A = pass-1 kernels without the pass-2 fold on the plan
  // stream; pass B = mirrored suffix scan with the fused combine on a forked stream.
  void two_filter(PlanState& p, const void* yv, void* xv, void* Psv) override {
    if constexpr (Src::HAS_MIRROR) {
      const Geom& g = p.g;
      WsLayout<R, N, K> L;
      L.plan(g, true);
      auto W = [&](size_t off) { return reinterpret_cast<R*>(p.ws + off); };
      const R* y = static_cast<const R*>(yv);
      R* x = static_cast<R*>(xv);
      const unsigned ntiles = (unsigned)(g.batch * g.tpt);
      cudaStream_t s = p.stream, s2 = p.stream2;
      cudaEventRecord(p.ev_fork, s);
      cudaStreamWaitEvent(s2, p.ev_fork, 0);
      // pass A: forward filter (S_i, v_i)
      reduce1<false>(p, s, K_P1_REDUCE, src, fold, tab, y, nullptr, W(L.run_incl), W(L.tile_agg1));
      tiles1(p, s, K_P1_TILES, false, W(L.tile_agg1), W(L.tile_incl1), W(L.group_agg1));
      groups1(p, s, K_P1_GROUPS, false, W(L.group_agg1), nullptr, nullptr, W(L.group_carry1), nullptr);
      PM_LAUNCH(p, s, K_P1_DOWN,
                (k_p1_down<R, N, NY, kNT, K, Src, false><<<ntiles, kNT, smem_down(), s>>>(
                    src, g, y, nullptr, W(L.run_incl), W(L.tile_incl1), W(L.group_carry1), W(L.sv), nullptr,
                    nullptr, p.dflag, nullptr, (use_lti && tab) ? &tab->SF[0][0] : nullptr, lti_jlo(g, false),
                    lti_jhi(g), nullptr, uwc(false), ux(false))));
      // pass B: backward information filter over mirrored elements (reverse node order)
      Mirror<Src> mir{src, g.node0 + g.Nn - 1};
      reduce1<true>(p, s2, K_TF_REDUCE, mir, fold_m, tab_m, y, nullptr, W(L.tf_run), W(L.tf_tile));
      tiles1(p, s2, K_TF_TILES, true, W(L.tf_tile), W(L.tf_tincl), W(L.tf_gagg));
      groups1(p, s2, K_TF_GROUPS, true, W(L.tf_gagg), nullptr, nullptr, W(L.tf_gcarry), nullptr);
      cudaEventRecord(p.ev_join, s);
      cudaStreamWaitEvent(s2, p.ev_join, 0);
      PM_LAUNCH(p, s2, K_TF_DOWN,
                (k_tf_down<R, N, NY, kNT, K, Src><<<ntiles, kNT, smem_down(), s2>>>(
                    mir, g, y, W(L.tf_run), W(L.tf_tincl), W(L.tf_gcarry), W(L.sv), x, static_cast<R*>(Psv), p.dflag,
                    (use_lti && tab_m) ? &tab_m->SF[0][0] : nullptr, lti_jlo(g, true), lti_jhi(g), uwc(true),
                    ux(true))));
      cudaEventRecord(p.ev_fork, s2);
      cudaStreamWaitEvent(s, p.ev_fork, 0);
    } else {
      p.err = "two-filter not available for this model kind";
    }
  }
  void sequential(PlanState& p, int method, const void* yv, const void* xbarv, void* xv, void* Psv) override {
    const Geom& g = p.g;
    WsLayout<R, N, K> L;
    L.plan(g, p.ws_tf);
    R* ws = reinterpret_cast<R*>(p.ws + L.sv);  // V_i of every node: [Nn][SZ][batch] fits the (S, v) planes
    const R* y = static_cast<const R*>(yv);
    const R* xbar = static_cast<const R*>(xbarv);
    R* x = static_cast<R*>(xv);
    R* Ps = static_cast<R*>(Psv);
    cudaStream_t s = p.stream;
    const unsigned nb = (unsigned)((g.batch + 31) / 32);
    const unsigned nt = (unsigned)(g.batch < 32 ? g.batch : 32);
    if (method == 0) {
      PM_LAUNCH(p, s, K_SEQ, (k_seq_rts<R, N, NY, Src><<<nb, nt, 0, s>>>(src, g, y, xbar, ws, x, Ps, p.dflag)));
    } else if constexpr (Src::HAS_MIRROR) {
      PM_LAUNCH(p, s, K_SEQ, (k_seq_tf<R, N, NY, Src><<<nb, nt, 0, s>>>(src, g, y, ws, x, Ps, p.dflag)));
    } else {
      p.err = "sequential two-filter not available for this model kind";
    }
  }
  void fill_m0(PlanState& p, void* xbar) override {
    const int64_t n = p.g.batch * p.g.Nn * N;
    PM_LAUNCH(p, p.stream, K_NL_MISC,
              (k_fill_m0<R, N><<<(unsigned)((n + 255) / 256), 256, 0, p.stream>>>(
                  n, static_cast<const R*>(p.m0_dev), static_cast<R*>(xbar))));
  }
  void maxdiff(PlanState& p, void* a, const void* b, unsigned long long* out, bool copy) override {
    const int64_t n = p.g.batch * p.g.Nn * N;
    if (copy)
      PM_LAUNCH(p, p.stream, K_NL_MISC,
                (k_maxdiff<R, true><<<296, 256, 0, p.stream>>>(n, static_cast<R*>(a), static_cast<const R*>(b), out)));
    else
      PM_LAUNCH(p, p.stream, K_NL_MISC,
                (k_maxdiff<R, false><<<296, 256, 0, p.stream>>>(n, static_cast<R*>(a), static_cast<const R*>(b), out)));
  }
};

template <typename R, int N, int NY, class Src, int K>
bool RunnerT<R, N, NY, Src, K>::prepare(PlanState& p) {
  if constexpr (IS_LTI) {
    const char* gen = getenv("PMAP_GENERAL");
    if (gen && gen[0] == '1') return true;  // force the general reduce (A/B checks)
    auto fill = [&](LtiNode<R, N, NY>& ln, bool mirror) {
      for (int i = 0; i < N; ++i) {
        for (int j = 0; j < N; ++j) ln.A[i][j] = mirror ? src.Am[i][j] : src.A[i][j];
        ln.b[i] = mirror ? src.bm[i] : src.b[i];
        ln.h0[i] = src.h0[i];
        for (int k = 0; k < NY; ++k) ln.K[i][k] = src.K[i][k];
      }
      for (int k = 0; k < Dim<N>::NS; ++k) {
        ln.C[k] = mirror ? src.Cm[k] : src.C[k];
        ln.J[k] = src.J[k];
      }
    };
    fill(lnode, false);
    fill(lnode_m, true);
    int* dok = nullptr;
    if (cudaMalloc(&tab, sizeof(Tab)) != cudaSuccess || cudaMalloc(&tab_m, sizeof(Tab)) != cudaSuccess ||
        cudaMalloc(&dok, 2 * sizeof(int)) != cudaSuccess)
      return false;
    k_lti_setup<R, N, NY, kNT, K><<<1, 1>>>(lnode, tab, dok);
    k_lti_setup<R, N, NY, kNT, K><<<1, 1>>>(lnode_m, tab_m, dok + 1);
    int* dok2 = nullptr;
    if (cudaMalloc(&scan_tab, sizeof(LtiScanTables<R, N>)) == cudaSuccess &&
        cudaMalloc(&scan_tab_m, sizeof(LtiScanTables<R, N>)) == cudaSuccess &&
        cudaMalloc(&dok2, 2 * sizeof(int)) == cudaSuccess) {
      k_lti_scan_setup<R, N, kNT, K><<<1, 1>>>(tab, scan_tab, dok2);
      k_lti_scan_setup<R, N, kNT, K><<<1, 1>>>(tab_m, scan_tab_m, dok2 + 1);
      int ok2[2] = {0, 0};
      if (cudaMemcpy(ok2, dok2, sizeof ok2, cudaMemcpyDeviceToHost) != cudaSuccess || !ok2[0] || !ok2[1]) {
        cudaGetLastError();
        cudaFree(scan_tab);
        cudaFree(scan_tab_m);
        scan_tab = scan_tab_m = nullptr;  // general scans
      }
    } else {
      cudaGetLastError();
      cudaFree(scan_tab);
      scan_tab = scan_tab_m = nullptr;
    }
    cudaFree(dok2);
    int ok[2] = {0, 0};
    cudaError_t e = cudaMemcpy(ok, dok, sizeof ok, cudaMemcpyDeviceToHost);
    cudaFree(dok);
    if (e != cudaSuccess) return false;
    use_lti = ok[0] && ok[1];  // a failed setup (singular pivot) falls back to the general kernels
    if (use_lti) {
      auto pull = [&](LtiFoldParams<R, N, NY, K, Log2<kNT>::value>& fpp, const LtiNode<R, N, NY>& ln,
                      const Tab* t) {
        fpp.node = ln;
        bool okc = true;
        for (int lg = 0; lg < Log2<kNT>::value; ++lg) {
          const int idx = 2 * (1 << lg) - 2;
          okc = okc && cudaMemcpy(fpp.Uf[lg][0], t->U1[idx], sizeof(R) * N * N, cudaMemcpyDeviceToHost) == cudaSuccess &&
                cudaMemcpy(fpp.Uf[lg][1], t->U2[idx], sizeof(R) * N * N, cudaMemcpyDeviceToHost) == cudaSuccess &&
                cudaMemcpy(fpp.Uf[lg][2], t->U3[idx], sizeof(R) * N * N, cudaMemcpyDeviceToHost) == cudaSuccess &&
                cudaMemcpy(fpp.Uf[lg][3], t->U4[idx], sizeof(R) * N * N, cudaMemcpyDeviceToHost) == cudaSuccess;
        }
        if (!okc || cudaMemcpy(fpp.crun, t->crun, sizeof fpp.crun, cudaMemcpyDeviceToHost) != cudaSuccess)
          return false;
        for (int m = 0; m < K; ++m)
          for (int i = 0; i < 2 * N; ++i)
            if (cudaMemcpy(fpp.GK[m][i], t->GK[m][i], sizeof(R) * NY, cudaMemcpyDeviceToHost) != cudaSuccess)
              return false;
        return true;
      };
      if (!pull(fold, lnode, tab) || !pull(fold_m, lnode_m, tab_m)) return false;
      if (getenv("PMAP_PLAN_TIMING")) fprintf(stderr, "[pmap plan]   LTI setup kernels + table pulls done\n");
      if (!prepare_lb(p)) {
        cudaGetLastError();
        use_lb = false;
      }
    }
  }
  (void)p;
  return true;
}

// Plan-time tables of the look-back path (pmap_lb.cuh), host fp64: S entering every tile
// (the data-independent Riccati part of the value function, chained over the tile span
// element (A_L, C_L, J_L) of k_lti_setup from S_0 = J_0), Gt_j = A_L^T (I + S_j C_L)^-1,
// Hs_j = Gt_j S_j, the group products of Gt, and the forward-recovery amplification
// bound max_j || A^-1 (I + C S_j) ||_2^K (R-FWD) that decides whether the path is used.
template <typename R, int N, int NY, class Src, int K>
bool RunnerT<R, N, NY, Src, K>::prepare_lb(PlanState& p) {
  if constexpr (!IS_LTI) {
    return false;
  } else {
    // time-sharded plans (world > 1, or the 1-rank NCCL test path) take the sharded look-back
    // for single trajectories when every rank holds at least one full tile; the decision
    // uses global quantities only, so every rank makes the same one
    const bool shard = p.d.world > 1 || p.force_shard;
    lb_shard = false;
    if (shard && (p.g.batch != 1 || p.no_lb || p.d.T + 1 < (int64_t)p.d.world * kNT * K)) return false;
    const bool ptime = getenv("PMAP_PLAN_TIMING") != nullptr;
    auto tnow = [] { return std::chrono::steady_clock::now(); };
    auto t0 = tnow();
    auto tlog = [&](const char* what) {
      if (ptime) {
        cudaDeviceSynchronize();
        fprintf(stderr, "[pmap plan]   lb: %-22s %8.2f ms\n", what,
                std::chrono::duration<double, std::milli>(tnow() - t0).count());
        t0 = tnow();
      }
    };
    constexpr int NS = Dim<N>::NS;
    const int64_t L = (int64_t)kNT * K;
    LbGeom g{};
    g.Nn = p.g.Nn + ((shard && p.d.rank > 0) ? 1 : 0);  // rank r > 0: local node 0 = the node before the chunk
    g.batch = p.g.batch;
    const int64_t M = g.Nn - 1;  // interior nodes
    if (M < 1) return false;
    g.tpt = (M + L - 1) / L;
    g.gpt = (g.tpt + kLbGroup - 1) / kLbGroup;
    // tile span element (matrix parts of NT full runs)
    R sa[N][N], sc[NS], sj[NS];
    if (cudaMemcpy(sa, tab->SA[kNT - 1], sizeof sa, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(sc, tab->SC[kNT - 1], sizeof sc, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(sj, tab->SJ[kNT - 1], sizeof sj, cudaMemcpyDeviceToHost) != cudaSuccess)
      return false;
    auto full = [&](const R* pk, double* m) {
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) m[i * N + j] = (double)pk[i <= j ? sidx(i, j, N) : sidx(j, i, N)];
    };
    double AL[N * N], CL[N * N], JL[N * N], S[N * N], Cn[N * N], Am[N * N];
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        AL[i * N + j] = (double)sa[i][j];
        Am[i * N + j] = (double)src.Am[i][j];
      }
    full(sc, CL);
    full(sj, JL);
    full(src.J0, S);
    full(src.C, Cn);
    double An[N * N], Jn[N * N];  // one interior node's element (LTI)
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) An[i * N + j] = (double)src.A[i][j];
    full(src.J, Jn);
    auto mm = [&](const double* X, const double* Y, double* Z) {
      double T[N * N];
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
          double a = 0;
          for (int k = 0; k < N; ++k) a += X[i * N + k] * Y[k * N + j];
          T[i * N + j] = a;
        }
      memcpy(Z, T, sizeof T);
    };
    // S <- J + A^T S (I + C S)^-1 A (an element of matrix parts (A, C, J) applied to S)
    auto vstep = [&](const double* Ax, const double* Cx, const double* Jx, double* Sx) -> bool {
      double M2[N * N], M2i[N * N], X[N * N], Y[N * N], Sn[N * N], At[N * N];
      mm(Cx, Sx, M2);
      for (int i = 0; i < N; ++i) M2[i * N + i] += 1.0;
      if (!h_inv(N, M2, M2i)) return false;
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) At[i * N + c] = Ax[c * N + i];
      mm(M2i, Ax, X);
      mm(Sx, X, Y);
      mm(At, Y, Sn);
      for (int i = 0; i < N * N; ++i) Sn[i] += Jx[i];
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) Sx[i * N + c] = 0.5 * (Sn[i * N + c] + Sn[c * N + i]);
      return h_is_finite(Sx, N * N);
    };
    // forward-recovery step map A^-1 (I + C S) at S: spectral norm by power iteration, ^K
    auto amp_of = [&](const double* Sx) -> double {
      double CS[N * N], Mf[N * N];
      mm(Cn, Sx, CS);
      for (int i = 0; i < N; ++i) CS[i * N + i] += 1.0;
      mm(Am, CS, Mf);
      double v[N], w2[N], nrm = 0;
      for (int i = 0; i < N; ++i) v[i] = 1.0 / std::sqrt((double)N);
      for (int it = 0; it < 60; ++it) {  // v <- M^T M v / |M^T M v|;  |M|_2^2 = |M^T M v| at convergence
        double u[N];
        for (int i = 0; i < N; ++i) {
          u[i] = 0;
          for (int k = 0; k < N; ++k) u[i] += Mf[i * N + k] * v[k];
        }
        double s2 = 0;
        for (int i = 0; i < N; ++i) {
          w2[i] = 0;
          for (int k = 0; k < N; ++k) w2[i] += Mf[k * N + i] * u[k];
          s2 += w2[i] * w2[i];
        }
        s2 = std::sqrt(s2);
        if (!(s2 > 0)) break;
        nrm = std::sqrt(s2);
        for (int i = 0; i < N; ++i) v[i] = w2[i] / s2;
      }
      return std::pow(nrm, (double)K);
    };
    double amp_global = 0.0;
    if (shard) {
      // the decision: the amplification bound over the GLOBAL tile chain (same on every rank)
      double Sg[N * N];
      memcpy(Sg, S, sizeof Sg);
      const int64_t gt_tiles = (p.d.T + L - 1) / L;
      for (int64_t t = 0; t < gt_tiles; ++t) {
        amp_global = std::max(amp_global, amp_of(Sg));
        if (!vstep(AL, CL, JL, Sg)) return false;
      }
      // S after global node c0 - 1 (rank r > 0): whole global tiles, then node by node
      if (p.d.rank > 0) {
        const int64_t nint = p.g.node0 - 1;
        for (int64_t t = 0; t < nint / L; ++t)
          if (!vstep(AL, CL, JL, S)) return false;
        for (int64_t t = 0; t < nint % L; ++t)
          if (!vstep(An, Cn, Jn, S)) return false;
      }
    }
    std::vector<LbTileTab<R, N>> ht((size_t)g.tpt);
    std::vector<double> gt((size_t)g.tpt * N * N);
    double amp = 0.0;
    for (int64_t j = 0; j < g.tpt; ++j) {
      LbTileTab<R, N>& e = ht[(size_t)j];
      for (int i = 0; i < N; ++i)
        for (int c = i; c < N; ++c) e.S[sidx(i, c, N)] = (R)(0.5 * (S[i * N + c] + S[c * N + i]));
      if constexpr (src_smask<Src>() != ~0u) {  // R-SMASK: the chain keeps S's structural zeros exactly
        for (int k = 0; k < NS; ++k)
          if (!mask_nz(src_smask<Src>(), k) && e.S[k] != R(0)) return false;
      }
      // Gt = A^T (I + S C)^-1, Hs = Gt S
      double M1[N * N], Mi[N * N], G[N * N], H[N * N];
      mm(S, CL, M1);
      for (int i = 0; i < N; ++i) M1[i * N + i] += 1.0;
      if (!h_inv(N, M1, Mi)) return false;
      double At[N * N];
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) At[i * N + c] = AL[c * N + i];
      mm(At, Mi, G);
      mm(G, S, H);
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) {
          e.Gt[i][c] = (R)G[i * N + c];
          e.Hs[i][c] = (R)H[i * N + c];
          gt[(size_t)j * N * N + i * N + c] = G[i * N + c];
        }
      // forward-recovery step map A^-1 (I + C S) at this S: spectral norm by power iteration
      {
        double CS[N * N], Mf[N * N];
        mm(Cn, S, CS);
        for (int i = 0; i < N; ++i) CS[i * N + i] += 1.0;
        mm(Am, CS, Mf);
        double v[N], w2[N], nrm = 0;
        for (int i = 0; i < N; ++i) v[i] = 0.5;  // unit vector (N <= 4) or close to it; renormalised below
        {
          double s0 = 0;
          for (int i = 0; i < N; ++i) s0 += v[i] * v[i];
          for (int i = 0; i < N; ++i) v[i] /= std::sqrt(s0);
        }
        for (int it = 0; it < 60; ++it) {  // v <- M^T M v / |M^T M v|;  |M|_2^2 = |M^T M v| at convergence
          double u[N];
          for (int i = 0; i < N; ++i) {
            u[i] = 0;
            for (int k = 0; k < N; ++k) u[i] += Mf[i * N + k] * v[k];
          }
          double s2 = 0;
          for (int i = 0; i < N; ++i) {
            w2[i] = 0;
            for (int k = 0; k < N; ++k) w2[i] += Mf[k * N + i] * u[k];
            s2 += w2[i] * w2[i];
          }
          s2 = std::sqrt(s2);
          if (!(s2 > 0)) break;
          nrm = std::sqrt(s2);
          for (int i = 0; i < N; ++i) v[i] = w2[i] / s2;
        }
        if (!shard) amp = std::max(amp, std::pow(nrm, (double)K));
      }
      // S_{j+1} = J_L + A_L^T S (I + C_L S)^-1 A_L
      double M2[N * N], M2i[N * N], X[N * N], Y[N * N], Sn[N * N];
      mm(CL, S, M2);
      for (int i = 0; i < N; ++i) M2[i * N + i] += 1.0;
      if (!h_inv(N, M2, M2i)) return false;
      mm(M2i, AL, X);
      mm(S, X, Y);
      mm(At, Y, Sn);
      for (int i = 0; i < N * N; ++i) Sn[i] += JL[i];
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) S[i * N + c] = 0.5 * (Sn[i * N + c] + Sn[c * N + i]);
      if (!h_is_finite(S, N * N)) return false;
    }
    if (shard) amp = amp_global;
    lb_amp = amp;
    tlog("S chain (host)");
    const char* ma = getenv("PMAP_LB_MAX_AMP");
    const double max_amp = ma ? atof(ma) : 1e6;
    if (!(amp <= max_amp)) return false;  // forward recovery would amplify rounding: keep the scan hierarchy
    // group maps GtG_G = Gt_{32G+31} ... Gt_{32G} (host) and Pb[G][l] = GtG_{G-1} ... GtG_{G-l}
    // (l = 0..G); the per-tile window products Pa, Qa are built on the device below
    constexpr int W1 = kLbGroup + 1;
    const size_t npa = (size_t)g.tpt * W1 * N * N, npb = (size_t)(g.gpt * (g.gpt + 1) / 2) * N * N;
    std::vector<double> pb(npb, 0.0), gtg((size_t)g.gpt * N * N, 0.0);
    for (int64_t G = 0; G + 1 < g.gpt; ++G) {  // full groups (every group before the last)
      double P[N * N];
      for (int i = 0; i < N * N; ++i) P[i] = (i % (N + 1) == 0) ? 1.0 : 0.0;
      for (int64_t k = G * kLbGroup; k < (G + 1) * kLbGroup; ++k) mm(&gt[(size_t)k * N * N], P, P);
      memcpy(&gtg[(size_t)G * N * N], P, sizeof P);
    }
    for (int64_t G = 0; G < g.gpt; ++G) {
      double P[N * N];
      for (int i = 0; i < N * N; ++i) P[i] = (i % (N + 1) == 0) ? 1.0 : 0.0;
      const size_t base = (size_t)(G * (G + 1) / 2);
      for (int64_t l = 0; l <= G; ++l) {
        memcpy(&pb[(base + l) * N * N], P, sizeof P);
        if (l < G) mm(P, &gtg[(size_t)(G - 1 - l) * N * N], P);
      }
    }
    tlog("Pa, Pb (host)");
    if (cudaMalloc(&lbtab, sizeof(LbTileTab<R, N>) * g.tpt) != cudaSuccess) return false;
    cudaMemcpy(lbtab, ht.data(), sizeof(LbTileTab<R, N>) * g.tpt, cudaMemcpyHostToDevice);
    {  // per-run tables, one device thread per (tile, run)
      const size_t rb = sizeof(R) * LbRunTab<N>::F * kNT * (size_t)g.tpt;
      int* dok = nullptr;
      if (cudaMalloc(&lbrun, rb) != cudaSuccess || cudaMalloc(&dok, sizeof(int)) != cudaSuccess) return false;
      const int one = 1;
      cudaMemcpy(dok, &one, sizeof one, cudaMemcpyHostToDevice);
      const int64_t nthr = g.tpt * kNT;
      k_lb_setup_runs<R, N, NY, kNT, K><<<(unsigned)((nthr + 127) / 128), 128>>>(tab, lbtab, g.tpt, g.Nn, lbrun, dok);
      int okh = 0;
      const cudaError_t e = cudaMemcpy(&okh, dok, sizeof okh, cudaMemcpyDeviceToHost);
      cudaFree(dok);
      if (e != cudaSuccess || !okh) return false;
      p.lb_bytes += rb;
    }
    tlog("run tables (device)");
    // QB per run and the pass-2 tile matrices Phi_tile(j) (device, one thread per tile),
    // then the window products Qa[j][l] = Phi_{j+1} ... Phi_{j+l} (l = 0..kLbGroup), the
    // group matrices PhiG_G = Qa[32G - 1][group size] (G >= 1, the last group included)
    // and Qb[G][l] = PhiG_{G+1} ... PhiG_{G+l} (l = 0..gpt-1-G; the last one multiplies x*_T)
    std::vector<double> phit((size_t)g.tpt * N * N);
    {
      R* dphi = nullptr;
      if (cudaMalloc(&dphi, sizeof(R) * N * N * g.tpt) != cudaSuccess) return false;
      k_lb_setup_tiles<R, N, kNT, K><<<(unsigned)((g.tpt + 127) / 128), 128>>>(tab, lbrun, g.tpt, g.Nn, dphi);
      std::vector<R> hphi((size_t)g.tpt * N * N);
      const cudaError_t e = cudaMemcpy(hphi.data(), dphi, sizeof(R) * N * N * g.tpt, cudaMemcpyDeviceToHost);
      cudaFree(dphi);
      if (e != cudaSuccess) return false;
      for (size_t i = 0; i < hphi.size(); ++i) phit[i] = (double)hphi[i];
    }
    lb_phit = phit;
    if (shard) {  // the chunk's v-map Gc and x-map Pc, plan constants of the two exchanges
      double Gc[N * N], Pc[N * N];
      for (int i = 0; i < N * N; ++i) Gc[i] = Pc[i] = (i % (N + 1) == 0) ? 1.0 : 0.0;
      for (int64_t j = 0; j + 1 < g.tpt; ++j) mm(&gt[(size_t)j * N * N], Gc, Gc);
      {  // the last tile node by node: G_node = A^T (I + S C)^-1, then S <- the node's update
        double Sx[N * N];
        const LbTileTab<R, N>& e = ht[(size_t)g.tpt - 1];
        for (int i = 0; i < N; ++i)
          for (int c = 0; c < N; ++c) Sx[i * N + c] = (double)e.S[i <= c ? sidx(i, c, N) : sidx(c, i, N)];
        const int64_t nlast = (g.Nn - 1) - (g.tpt - 1) * L;
        for (int64_t t = 0; t < nlast; ++t) {
          double M1[N * N], Mi[N * N], At[N * N], Gn[N * N];
          mm(Sx, Cn, M1);
          for (int i = 0; i < N; ++i) M1[i * N + i] += 1.0;
          if (!h_inv(N, M1, Mi)) return false;
          for (int i = 0; i < N; ++i)
            for (int c = 0; c < N; ++c) At[i * N + c] = An[c * N + i];
          mm(At, Mi, Gn);
          mm(Gn, Gc, Gc);
          if (!vstep(An, Cn, Jn, Sx)) return false;
        }
      }
      for (int64_t j = 0; j < g.tpt; ++j) mm(Pc, &phit[(size_t)j * N * N], Pc);
      std::vector<R> h(lbsh_elems(), R(0));
      for (int i = 0; i < N * N; ++i) {
        h[5 * N + i] = (R)Gc[i];
        h[5 * N + N * N + i] = (R)Pc[i];
        h[5 * N + 2 * N * N + i] = (R)phit[i];
      }
      if (cudaMalloc(&lbsh, sizeof(R) * h.size()) != cudaSuccess ||
          cudaMemcpy(lbsh, h.data(), sizeof(R) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return false;
    }
    const size_t nqa = (size_t)g.tpt * W1 * N * N, nqb = (size_t)(g.gpt * (g.gpt + 1) / 2) * N * N;
    std::vector<double> qb(nqb, 0.0), phig((size_t)g.gpt * N * N, 0.0);
    for (int64_t G = 1; G < g.gpt; ++G) {  // PhiG_G = Phi_{32G} ... Phi_{32G + n_G - 1} (the last group included)
      const int64_t cntG = std::min<int64_t>(kLbGroup, g.tpt - G * kLbGroup);
      double P[N * N];
      for (int i = 0; i < N * N; ++i) P[i] = (i % (N + 1) == 0) ? 1.0 : 0.0;
      for (int64_t k = G * kLbGroup; k < G * kLbGroup + cntG; ++k) mm(P, &phit[(size_t)k * N * N], P);
      memcpy(&phig[(size_t)G * N * N], P, sizeof P);
    }
    for (int64_t G = 0; G < g.gpt; ++G) {
      double P[N * N];
      for (int i = 0; i < N * N; ++i) P[i] = (i % (N + 1) == 0) ? 1.0 : 0.0;
      const size_t base = (size_t)(G * g.gpt - G * (G - 1) / 2);
      for (int64_t l = 0; l < g.gpt - G; ++l) {
        memcpy(&qb[(base + l) * N * N], P, sizeof P);
        if (G + 1 + l < g.gpt) mm(P, &phig[(size_t)(G + 1 + l) * N * N], P);
      }
    }
    tlog("Phi_tile, Pb, Qb (host)");
    if (cudaMalloc(&lbprod, sizeof(R) * (npa + npb + nqa + nqb)) != cudaSuccess) return false;
    {
      std::vector<R> small(npb + nqb);
      for (size_t i = 0; i < npb; ++i) small[i] = (R)pb[i];
      for (size_t i = 0; i < nqb; ++i) small[npb + i] = (R)qb[i];
      cudaMemset(lbprod, 0, sizeof(R) * (npa + nqa));
      cudaMemcpy(lbprod + npa, small.data(), sizeof(R) * npb, cudaMemcpyHostToDevice);
      cudaMemcpy(lbprod + npa + npb + nqa, small.data() + npb, sizeof(R) * nqb, cudaMemcpyHostToDevice);
      R* dphi = nullptr;  // Phi_tile again (device) for the window products
      std::vector<R> hphi(phit.size());
      for (size_t i = 0; i < phit.size(); ++i) hphi[i] = (R)phit[i];
      if (cudaMalloc(&dphi, sizeof(R) * hphi.size()) != cudaSuccess) return false;
      cudaMemcpy(dphi, hphi.data(), sizeof(R) * hphi.size(), cudaMemcpyHostToDevice);
      k_lb_setup_window<R, N><<<(unsigned)((g.tpt + 127) / 128), 128>>>(lbtab, dphi, g.tpt, lbprod, lbprod + npa + npb);
      const cudaError_t e = cudaDeviceSynchronize();
      cudaFree(dphi);
      if (e != cudaSuccess) return false;
      p.lb_bytes += sizeof(R) * (npa + npb + nqa + nqb);
    }
    tlog("upload products");
    // workspace
    const size_t tiles = (size_t)(g.batch * g.tpt), groups = (size_t)(g.batch * g.gpt);
    size_t off = 0;
    auto take = [&](size_t bytes) {
      size_t o = off;
      off += (bytes + 255) / 256 * 256;
      return o;
    };
    const size_t o_a1 = take(tiles * N * sizeof(R)), o_p1 = take(tiles * N * sizeof(R)),
                 o_g1 = take(groups * N * sizeof(R)), o_rc = take(tiles * N * kNT * sizeof(R)),
                 o_ri = take(tiles * Aff<R, N>::SZ * kNT * sizeof(R)), o_a2 = take(tiles * N * sizeof(R)),
                 o_g2 = take(groups * N * sizeof(R)), o_p2 = take(tiles * N * sizeof(R)),
                 o_sd = take((size_t)g.batch * N * sizeof(R)), o_sr = take((size_t)g.batch * 2 * N * sizeof(R));
    const size_t f0 = off;
    const size_t o_f1 = take(tiles * 4), o_gf1 = take(groups * 4), o_gc1 = take(groups * 4), o_gc2 = take(groups * 4),
                 o_f2 = take(tiles * 4), o_ct = take(8);
    if (cudaMalloc(&lbws, off) != cudaSuccess) return false;
    if (cudaMemset(lbws + f0, 0, off - f0) != cudaSuccess) return false;
    auto RP = [&](size_t o) { return reinterpret_cast<R*>(lbws + o); };
    auto UP = [&](size_t o) { return reinterpret_cast<unsigned*>(lbws + o); };
    lbw.agg1 = RP(o_a1);
    lbw.pub1 = RP(o_p1);
    lbw.gagg1 = RP(o_g1);
    lbw.rcv = RP(o_rc);
    lbw.ri = RP(o_ri);
    lbw.agg2 = RP(o_a2);
    lbw.gagg2 = RP(o_g2);
    lbw.pub2 = RP(o_p2);
    lbw.seed = RP(o_sd);
    lbw.seedrb = RP(o_sr);
    lbw.flag1 = UP(o_f1);
    lbw.gflag1 = UP(o_gf1);
    lbw.gcnt1 = UP(o_gc1);
    lbw.gcnt2 = UP(o_gc2);
    lbw.flag2 = UP(o_f2);
    lbw.ctr = UP(o_ct);
    lbw.Pa = lbprod;
    lbw.Pb = lbprod + npa;
    lbw.Qa = lbprod + npa + npb;
    lbw.tim = nullptr;
    {
      const char* tm = getenv("PMAP_LB_TIMING");
      if (tm && tm[0] == '1') {
        if (cudaMalloc(&lbw.tim, sizeof(unsigned long long) * 16 * tiles) != cudaSuccess) return false;
        cudaMemset(lbw.tim, 0, sizeof(unsigned long long) * 16 * tiles);
        p.lb_tim = lbw.tim;
        p.lb_tim_n = 16 * tiles;
      }
    }
    lbw.Qb = lbprod + npa + npb + nqa;
    // ticket strides = resident CTAs (warps) of the look-back kernels on this device
    {
      int dev = 0, nsm = 148, b1 = 0, b2 = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k_lb_pass1b<R, N, NY, kNT, K, Src>, 128, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k_lb_pass2<R, N, NY, kNT, K, Src, 0>, kNT, 0);
      const char* sd = getenv("PMAP_LB_STRIDE");  // "0": plain (unstrided) ticket order (A/B checks)
      const bool plain = sd && sd[0] == '0';
      g.S1 = plain ? (int64_t)1 << 40 : std::max<int64_t>(1, (int64_t)b1 * 4 * nsm);
      g.S2 = plain ? (int64_t)1 << 40 : std::max<int64_t>(1, (int64_t)b2 * nsm);
      if (plain) g.S1 = g.S2 = std::max<int64_t>(1, g.batch * g.tpt);
      const char* sg1 = getenv("PMAP_LB_STAGGER1_NS");  // first-wave stagger steps (lb_stagger); "0" = off
      const char* sg2 = getenv("PMAP_LB_STAGGER2_NS");
      g.stagger1 = sg1 ? atoi(sg1) : 1100;
      g.stagger2 = sg2 ? atoi(sg2) : 3000;
      g.stmod1 = 8;
      g.stmod2 = 6;
      const char* sg1b = getenv("PMAP_LB_STAGGER1B_NS");
      g.stagger1b = sg1b ? atoi(sg1b) : 800;
    }
    lbg = g;
    p.lb_bytes += off;
    srcf = src.template cast<float>();
    tlog("workspace");
    use_lb = true;
    lb_shard = shard;
    return true;
  }
}

// Plan tables of the smoother covariance (R-SCOV, look-back path), on first use: the
// covariance maps of the tiles (k_lb_cov_tiles), P^s_T = S_T^-1 (S_T from the last run's
// S and its element), the backward chain P^s at every tile end (host fp64:
// P_end(j-1) = Phi_j P_end(j) Phi_j^T + Sigma_j), then P^s before every run (k_lb_cov_runs).
template <typename R, int N, int NY, class Src, int K>
bool RunnerT<R, N, NY, Src, K>::prepare_lb_cov(PlanState& p) {
  if constexpr (!IS_LTI) {
    return false;
  } else {
    (void)p;
    const LbGeom& g = lbg;
    const int64_t tpt = g.tpt;
    double* dsig = nullptr;
    double* dpend = nullptr;
    if (cudaMalloc(&dsig, sizeof(double) * N * N * tpt) != cudaSuccess) return false;
    k_lb_cov_tiles<R, N, kNT, K><<<(unsigned)((tpt + 127) / 128), 128>>>(tab, lbrun, tpt, g.Nn, dsig);
    std::vector<double> sig((size_t)tpt * N * N);
    if (cudaMemcpy(sig.data(), dsig, sizeof(double) * sig.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaFree(dsig);
      return false;
    }
    cudaFree(dsig);
    // S_T: the last run's S and its element (one full run or the partial run of q nodes)
    const int64_t L = (int64_t)kNT * K, n0 = 1 + (tpt - 1) * L, nvalid = g.Nn - n0;
    const int rT = (int)((nvalid - 1) / K), q = (int)(nvalid - (int64_t)rT * K);
    constexpr int NS = Dim<N>::NS;
    R sp[NS], ea[N][N], ec[NS], ej[NS];
    for (int k = 0; k < NS; ++k)
      if (cudaMemcpy(&sp[k], lbrun + ((tpt - 1) * (int64_t)LbRunTab<N>::F + LbRunTab<N>::SP + k) * kNT + rT, sizeof(R),
                     cudaMemcpyDeviceToHost) != cudaSuccess)
        return false;
    if (q == K) {
      R e1[N * N + 2 * N + 2 * NS];
      if (cudaMemcpy(e1, tab->E1, sizeof e1, cudaMemcpyDeviceToHost) != cudaSuccess) return false;
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) ea[i][c] = e1[i * N + c];
      for (int k = 0; k < NS; ++k) {
        ec[k] = e1[N * N + N + k];
        ej[k] = e1[N * N + 2 * N + NS + k];
      }
    } else if (cudaMemcpy(ea, tab->PA[q - 1], sizeof ea, cudaMemcpyDeviceToHost) != cudaSuccess ||
               cudaMemcpy(ec, tab->PC[q - 1], sizeof ec, cudaMemcpyDeviceToHost) != cudaSuccess ||
               cudaMemcpy(ej, tab->PJ[q - 1], sizeof ej, cudaMemcpyDeviceToHost) != cudaSuccess) {
      return false;
    }
    auto full = [&](const R* pk, double* m) {
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) m[i * N + c] = (double)pk[i <= c ? sidx(i, c, N) : sidx(c, i, N)];
    };
    auto mm = [&](const double* X, const double* Y, double* Z) {
      double T[N * N];
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) {
          double a = 0;
          for (int k = 0; k < N; ++k) a += X[i * N + k] * Y[k * N + c];
          T[i * N + c] = a;
        }
      memcpy(Z, T, sizeof T);
    };
    double S[N * N], C[N * N], J[N * N], A[N * N], At[N * N], M1[N * N], M1i[N * N], X[N * N], ST[N * N], PT[N * N];
    full(sp, S);
    full(ec, C);
    full(ej, J);
    for (int i = 0; i < N; ++i)
      for (int c = 0; c < N; ++c) {
        A[i * N + c] = (double)ea[i][c];
        At[c * N + i] = (double)ea[i][c];
      }
    mm(C, S, M1);  // S_T = A^T S (I + C S)^-1 A + J
    for (int i = 0; i < N; ++i) M1[i * N + i] += 1.0;
    if (!h_inv(N, M1, M1i)) return false;
    mm(M1i, A, X);
    mm(S, X, X);
    mm(At, X, ST);
    for (int i = 0; i < N * N; ++i) ST[i] += J[i];
    if (!h_inv(N, ST, PT)) return false;
    std::vector<double> pend((size_t)tpt * N * N);
    for (int i = 0; i < N; ++i)
      for (int c = 0; c < N; ++c) pend[((size_t)(tpt - 1) * N + i) * N + c] = 0.5 * (PT[i * N + c] + PT[c * N + i]);
    for (int64_t j = tpt - 1; j >= 1; --j) {
      const double* Ph = &lb_phit[(size_t)j * N * N];
      double T1[N * N], T2[N * N], Pht[N * N];
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) Pht[c * N + i] = Ph[i * N + c];
      mm(Ph, &pend[(size_t)j * N * N], T1);
      mm(T1, Pht, T2);
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < N; ++c) {
          const double v = T2[i * N + c] + sig[((size_t)j * N + i) * N + c];
          const double w = T2[c * N + i] + sig[((size_t)j * N + c) * N + i];
          pend[((size_t)(j - 1) * N + i) * N + c] = 0.5 * (v + w);
        }
    }
    if (cudaMalloc(&dpend, sizeof(double) * pend.size()) != cudaSuccess ||
        cudaMalloc(&lbcov, sizeof(R) * NS * kNT * tpt) != cudaSuccess) {
      cudaFree(dpend);
      return false;
    }
    cudaMemcpy(dpend, pend.data(), sizeof(double) * pend.size(), cudaMemcpyHostToDevice);
    k_lb_cov_runs<R, N, kNT, K><<<(unsigned)((tpt + 127) / 128), 128>>>(tab, lbrun, tpt, g.Nn, dpend, lbcov);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaFree(dpend);
    return e == cudaSuccess;
  }
}

// ---------------------------------------------------------- instantiation
// Factories are declared here and explicitly instantiated, one (dtype, shape,
// model kind) per translation unit, in inst.cu (see pmap_make.cuh).
template <typename R, int N, int NY, int KR, int NWC, uint32_t AM, uint32_t UM, uint32_t SM = ~0u>
Runner* make_lti(const double* A, const double* b, const double* C, const double* J, const double* K,
                 const double* h0, const double* J0, const double* h00, const double* Am, const double* bm,
                 const double* Cm, const double* U);
template <typename R, int N, int NY, int KR>
Runner* make_tv(const R* F, const R* c, const R* L, const R* Wm, const R* H, const R* r, const R* Rm,
                const int64_t* str, int nw, double dt, const double* P0i, const double* P0im0);
template <typename R, int N, int NYM, int NSUB, int KR>
Runner* make_euler(const double* A, const double* C, const double* J, const double* b0, const double* h0,
                   const double* Kb, const double* Ke, const double* J0, const double* h00, const double* K0);
template <typename R, int N, int NY, int KIND, int KR>
Runner* make_nl(double dt, double mu, double om_div, const double* C, const double* Ri, const double* P0i,
                const double* P0im0);

#define PM_SHAPES(X) X(1, 1) X(2, 1) X(2, 2) X(3, 1) X(3, 2) X(4, 2) X(5, 2)

}  // namespace pmap_rt
