// pmap_lb.cuh -- single-pass decoupled look-back solve for time-invariant (LTI) models.
//
// Three kernels per solve ("look-back path"):
//
//   k_lb_pass1a pass 1 (value functions, P:260-341 / P:382-409), one CTA per tile (NT = 64
//               runs x K interior nodes), no waiting: the y tile into shared memory, the run
//               folds of the node elements' data parts (LTI impulse responses, R-LTI), the
//               tile aggregate (and, by each group's last arriver, the group aggregate), the
//               in-tile run scan and every run's pass-2 map (R-RUNAGG) with its in-tile
//               suffix composition -- as affine functions of the still unknown value
//               function entering the tile.
//   k_lb_pass1b one warp per tile: the decoupled look-back over the tile aggregates for
//               the value function entering the tile (all aggregates are in memory, so it
//               never waits; a published prefix only shortens the walk), then the run
//               values and maps are finished with one mat-vec per run, and the tiles' and
//               groups' pass-2 offsets and x*_T are written for pass 2.
//   k_lb_pass2  pass 2 (trajectory), one CTA of two warps per tile, tiles in
//               reverse order: the y tile into shared memory while warp 0 looks back over
//               the following tiles for x* at the tile's last node (again never waiting),
//               then per run x*_{s-1} from its suffix map and a FORWARD sweep over the
//               run's nodes that recomputes (S_i, v_i) from the run's value function and y
//               and recovers x*_i (R-FWD):
//                   x*_i = A_i^-1 [ x*_{i-1} - b_i + C_i (S_{i-1} x*_{i-1} - v_{i-1}) ],
//               the transition x*_{i-1} = (I + C_i S_{i-1})^-1 (A_i x*_i + b_i + C_i v_{i-1})
//               of R-TRANS solved for x*_i.  Nothing per node is stored between the
//               passes: the schedule moves y twice and x once (+ O(1/K) run data).
//
// Plan tables (R-LTI).  Node 0 (E_0 = prior + y_0) is the carry-in, so every tile holds
// only interior nodes: tile j covers nodes [1 + jL, 1 + (j+1)L), L = NT K, and every
// tile but a ragged last one has the same matrix parts.  The value function entering
// tile j has a data-independent S_j and a v that is affine in the v entering tile j-1:
// v_end(j) = Gt_j v_end(j-1) + g_j with Gt_j = A^T (I + S_j C)^-1 and g_j = eta_j -
// Gt_j S_j b_j from the tile's data parts (b_j, eta_j).  Every S-dependent matrix (per
// tile, per run, and the products of Gt and of the tiles' pass-2 matrices Phi over
// look-back windows) is computed once in map_plan, so the per-solve work is data parts,
// mat-vecs and the node recursion.
//
// Look-back (passes 1b and 2, two levels): a tile first looks at the tiles of its group
// of kLbGroup tiles (one warp window), then at whole groups, whose aggregates the
// previous kernel wrote, so a walk is at most a few windows even for the first wave;
// each window is one mat-vec per lane with a plan-time product and a warp sum.  Every
// aggregate exists before the look-back runs, so nothing ever waits: prefix status
// words (0 = none, 2 = inclusive prefix; written with st.release after the payload,
// read relaxed, one acquire fence before a prefix payload is read through L2) only cut
// a walk short.  Tiles run in ticket order (atomic counter), so the tiles a look-back
// reaches first are the ones most likely done.  Flags are cleared by the other kernel
// of the solve, counters by their last user, so repeated solves (and CUDA-graph
// replays) need no memset.
#pragma once
#include <type_traits>

#include "pmap_lti.cuh"

namespace pmap {

constexpr int kLbGroup = 32;  // tiles per look-back group (one warp window)
#ifndef PM_LB2_MAXREG
#define PM_LB2_MAXREG 168
#endif

struct LbGeom {
  int64_t Nn;     // nodes per trajectory (this launch)
  int64_t tpt;    // tiles per trajectory
  int64_t gpt;    // groups per trajectory
  int64_t batch;
  int64_t S1, S2;  // ticket strides of pass 1b (warps) and pass 2 (CTAs): the resident counts
  int stagger1, stagger2;  // first-wave start stagger of passes 1a / 2 (ns per step; 0 = off), lb_stagger
  int stmod1, stmod2;      // ... and its number of distinct start offsets
  int stagger1b;           // ... of pass 1b (per warp, 8 offsets)
};

// Strided ticket order of the look-back kernels: ticket t -> tile (t mod S) C + t div S,
// C = ceil(total / S), a bijection of [0, S C).  With S = the number of CTAs (warps)
// resident at once, a tile's neighbour in the scan direction was taken one full wave
// earlier, so its prefix is usually published by the time the tile looks back: the
// look-back is then one status read and one payload read.  Tickets past `total` map to
// tiles >= total and their CTAs (warps) exit at once.
__host__ __device__ inline int64_t lb_stride_map(int64_t t, int64_t total, int64_t S) {
  const int64_t C = (total + S - 1) / S;
  return (t % S) * C + t / S;
}
__host__ __device__ inline int64_t lb_ticket_count(int64_t total, int64_t S) { return ((total + S - 1) / S) * S; }

// Plan-time, data-independent quantities of tile j (shared by every trajectory).
template <typename R, int N>
struct LbTileTab {
  R S[Dim<N>::NS];  // S of the value function entering tile j (after node jL)
  R Gt[N][N];       // A_L^T (I + S C_L)^-1 (full tiles)
  R Hs[N][N];       // Gt S
};

// Plan-time, data-independent quantities of run r of tile j, stored field-major
// [tpt][F][NT] (lane r reads field f of its run coalesced):
//   GP  = A_p^T (I + S_in C_p)^-1   v-map of the exclusive prefix of r runs (span element
//                                    (A_p, C_p, J_p) of SF, S_in = S entering the tile):
//                                    v_{s-1} = GP (v_in - S_in pb) + ph
//   WR  = (I + C_R S_{s-1})^-1      the run's transition solve (R-RUNAGG, run element R)
//   PHI = WR A_R                    the run's pass-2 matrix
//   QB  = sum_{k >= r} Phi_r..Phi_{k-1} WR_k C_Rk GP_k   the v_in-coefficient of the run's
//                                    suffix offset (beta_k = WR_k (rb_k + C_Rk v_{s-1,k}))
//   SP  = S_{s-1}                   S entering the run (pass 2 restarts the node recursion there)
//   PS  = Phi_r Phi_{r+1} ... Phi_{NT-1}  the matrix of the run's in-tile suffix map (x at the
//                                    tile's last node -> x*_{s-1}); data-free, so pass 1a
//                                    writes only the map's offset and pass 2 reads PS here
// Empty runs of a ragged last tile are identity maps (PHI = I, WR = QB... = 0).
template <int N>
struct LbRunTab {
  static constexpr int GP = 0, WR = N * N, PHI = 2 * N * N, QB = 3 * N * N, SP = 4 * N * N,
                       PS = 4 * N * N + Dim<N>::NS, F = 5 * N * N + Dim<N>::NS;
};

// One thread per (tile, run): GP, WR, PHI, SP from the tile's S and the LTI span tables.
template <typename R, int N, int NY, int NT, int K>
__global__ void k_lb_setup_runs(const LtiTables<R, N, NT, K>* __restrict__ tab, const LbTileTab<R, N>* __restrict__ lt,
                                int64_t tpt, int64_t Nn, R* __restrict__ lrt, int* okflag) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= tpt * NT) return;
  const int64_t j = idx / NT;
  const int r = (int)(idx % NT);
  const int64_t n0 = 1 + j * (int64_t)NT * K;
  const int q = (int)max((int64_t)0, min((int64_t)K, Nn - n0 - (int64_t)r * K));
  R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;
  bool ok = true;
  VF<R, N> cur;
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) cur.S[k] = lt[j].S[k];
#pragma unroll
  for (int i = 0; i < N; ++i) cur.v[i] = R(0);
  R Gp[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) Gp[i][c] = (i == c) ? R(1) : R(0);
  if (r > 0 && q > 0) {
    Elem<R, N> p;
    int f = 0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int jj = 0; jj < N; ++jj) p.A[i][jj] = tab->SF[f++][r - 1];
#pragma unroll
    for (int k = 0; k < Dim<N>::NS; ++k) p.C[k] = tab->SF[f++][r - 1];
#pragma unroll
    for (int k = 0; k < Dim<N>::NS; ++k) p.J[k] = tab->SF[f++][r - 1];
#pragma unroll
    for (int i = 0; i < N; ++i) p.b[i] = p.h[i] = R(0);
    // GP^T = (I + C_p S_in)^-1 A_p  (= vapply's transition matrix X1)
    Aff<R, N> tr;
    VF<R, N> out;
    vapply<R, N, true>(p, cur, out, &tr, ok);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) Gp[i][c] = tr.P[c][i];
    cur = out;
  }
  R Wr[N][N], Phi[N][N];
  if (q == 0) {  // empty run: identity map
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        Wr[i][c] = R(0);
        Phi[i][c] = (i == c) ? R(1) : R(0);
      }
  } else {
    // run element R: one full run, or the partial run of the ragged last tile
    Elem<R, N> ra;
    if (q == K) {
      load(ra, tab->E1, 1);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int jj = 0; jj < N; ++jj) ra.A[i][jj] = tab->PA[q - 1][i][jj];
#pragma unroll
      for (int k = 0; k < Dim<N>::NS; ++k) {
        ra.C[k] = tab->PC[q - 1][k];
        ra.J[k] = tab->PJ[q - 1][k];
      }
    }
    // Wr = (I + C_R S)^-1 column by column, Phi = Wr A_R
    LUF<R, N> fct;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        R s = (i == c) ? R(1) : R(0);
#pragma unroll
        for (int k = 0; k < N; ++k)
          s = fma(ra.C[i <= k ? sidx(i, k, N) : sidx(k, i, N)], cur.S[k <= c ? sidx(k, c, N) : sidx(c, k, N)], s);
        fct.a[i][c] = s;
      }
    lu_factor(fct, ok);
#pragma unroll
    for (int c = 0; c < N; ++c) {
      R t[N], u[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        t[i] = (i == c) ? R(1) : R(0);
        u[i] = ra.A[i][c];
      }
      lu_solve(fct, t);
      lu_solve(fct, u);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        Wr[i][c] = t[i];
        Phi[i][c] = u[i];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      rt[(LbRunTab<N>::GP + i * N + c) * NT] = Gp[i][c];
      rt[(LbRunTab<N>::WR + i * N + c) * NT] = Wr[i][c];
      rt[(LbRunTab<N>::PHI + i * N + c) * NT] = Phi[i][c];
    }
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) rt[(LbRunTab<N>::SP + k) * NT] = cur.S[k];
  if (!ok) atomicExch(okflag, 0);
}

// One thread per tile, serial over the runs: the suffix coefficients QB_r (backwards),
// and the tile's pass-2 matrix Phi_tile = Phi_0 Phi_1 ... Phi_{NT-1} (x at the tile's
// last node -> x at the node before it).
template <typename R, int N, int NT, int K>
__global__ void k_lb_setup_tiles(const LtiTables<R, N, NT, K>* __restrict__ tab, R* __restrict__ lrt, int64_t tpt,
                                 int64_t Nn, R* __restrict__ phit) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= tpt) return;
  const int64_t n0 = 1 + j * (int64_t)NT * K;
  R Q[N][N], P[N][N];  // running QB (suffix) and Phi product (suffix: Phi_r ... Phi_{NT-1})
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      Q[i][c] = R(0);
      P[i][c] = (i == c) ? R(1) : R(0);
    }
  for (int r = NT - 1; r >= 0; --r) {
    R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;
    const int q = (int)max((int64_t)0, min((int64_t)K, Nn - n0 - (int64_t)r * K));
    if (q == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          rt[(LbRunTab<N>::QB + i * N + c) * NT] = R(0);
          rt[(LbRunTab<N>::PS + i * N + c) * NT] = P[i][c];  // an empty run: the suffix product so far
        }
      continue;
    }
    R CR[Dim<N>::NS];
#pragma unroll
    for (int k = 0; k < Dim<N>::NS; ++k) CR[k] = (q == K) ? tab->E1[N * N + N + k] : tab->PC[q - 1][k];
    R Wr[N][N], Ph[N][N], Gp[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        Wr[i][c] = rt[(LbRunTab<N>::WR + i * N + c) * NT];
        Ph[i][c] = rt[(LbRunTab<N>::PHI + i * N + c) * NT];
        Gp[i][c] = rt[(LbRunTab<N>::GP + i * N + c) * NT];
      }
    // B = Wr C_R Gp ; QB_r = B + Phi_r QB_{r+1}
    R WC[N][N], Nq[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        R a = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) a = fma(Wr[i][k], CR[k <= c ? sidx(k, c, N) : sidx(c, k, N)], a);
        WC[i][c] = a;
      }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        R a = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) {
          a = fma(WC[i][k], Gp[k][c], a);
          a = fma(Ph[i][k], Q[k][c], a);
        }
        Nq[i][c] = a;
      }
    R Np[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        R a = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) a = fma(Ph[i][k], P[k][c], a);
        Np[i][c] = a;
      }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        Q[i][c] = Nq[i][c];
        P[i][c] = Np[i][c];
        rt[(LbRunTab<N>::QB + i * N + c) * NT] = Q[i][c];
        rt[(LbRunTab<N>::PS + i * N + c) * NT] = P[i][c];
      }
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) phit[(j * N + i) * N + c] = P[i][c];
}

// One thread per tile: the look-back window products (fp64 accumulation)
//   Pa[j][l] = Gt_{j-1} Gt_{j-2} ... Gt_{j-l},   Qa[j][l] = Phi_{j+1} ... Phi_{j+l},
// l = 0..kLbGroup (entries reaching past the trajectory stay as the caller zeroed them).
template <typename R, int N>
__global__ void k_lb_setup_window(const LbTileTab<R, N>* __restrict__ lt, const R* __restrict__ phit, int64_t tpt,
                                  R* __restrict__ Pa, R* __restrict__ Qa) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= tpt) return;
  constexpr int W1 = kLbGroup + 1;
  for (int which = 0; which < 2; ++which) {
    double P[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) P[i][c] = (i == c) ? 1.0 : 0.0;
    R* out = (which == 0 ? Pa : Qa) + j * W1 * N * N;
    for (int l = 0; l < W1; ++l) {
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) out[(l * N + i) * N + c] = (R)P[i][c];
      const int64_t k = which == 0 ? j - 1 - l : j + 1 + l;
      if (k < 0 || k >= tpt) break;
      double T[N][N];
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          double a = 0.0;
#pragma unroll
          for (int m = 0; m < N; ++m)
            a = fma(P[i][m], (double)(which == 0 ? lt[k].Gt[m][c] : phit[(k * N + m) * N + c]), a);
          T[i][c] = a;
        }
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) P[i][c] = T[i][c];
    }
  }
}

// Workspace pointers of the look-back path.
template <typename R>
struct LbWs {
  R* agg1;    // [tiles][N]              g_j (pass-1 tile aggregate, data part)
  R* pub1;    // [tiles][N]              v_end(j)
  R* gagg1;   // [groups][N]             group g
  R* rcv;     // [tiles][N][NT]          v entering each run (pass 1 -> pass 2)
  R* ri;      // [tiles][Aff::SZ][NT]    run suffix maps: x at the tile's last node -> x_{s-1}
  R* agg2;    // [tiles][N]              tile pass-2 offsets beta_tile (Phi_tile: plan)
  R* gagg2;   // [groups][N]             group pass-2 offsets
  R* pub2;    // [tiles][N]              x at the last node of tile j - 1 (pass-2 prefix)
  R* seed;    // [batch][N]              x*_T = S_T^-1 v_T
  R* seedrb;  // [batch][2N]             data parts of the run ending at node T (pass 1a -> 1b)
  unsigned* flag1;   // [tiles]
  unsigned* gflag1;  // [groups]
  unsigned* gcnt1;   // [groups]
  unsigned* gcnt2;   // [groups]
  unsigned* flag2;   // [tiles]
  unsigned* ctr;     // [2] tickets of pass 1 / pass 2
  const R* Pa;       // [tpt][kLbGroup + 1][N][N] plan: Pa[j][l] = Gt_{j-1} Gt_{j-2} ... Gt_{j-l}
  const R* Pb;       // triangular [gpt][G + 1][N][N]: Pb[G][l] = GtG_{G-1} ... GtG_{G-l}
  const R* Qa;       // [tpt][kLbGroup + 1][N][N] plan: Qa[j][l] = Phi_{j+1} Phi_{j+2} ... Phi_{j+l}
  const R* Qb;       // triangular [gpt][gpt - G][N][N]: Qb[G][l] = PhiG_{G+1} ... PhiG_{G+l}
  unsigned long long* tim;  // [2][tiles][8] globaltimer stamps (PMAP_LB_TIMING=1 diagnostics), else null
};

PM_INLINE unsigned long long lb_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define LB_STAMP(PASS, K)                                                                 \
  do {                                                                                   \
    if (w.tim && threadIdx.x == 0) w.tim[((PASS) * g.batch * g.tpt + tile) * 8 + (K)] = lb_now(); \
  } while (0)

// Status words are polled with relaxed gpu-scope loads (LDG.STRONG.GPU, no L1
// invalidation per poll: an ld.acquire would emit CCTL.IVALL on every iteration and
// flush the SM's L1 under the other CTAs' feet); once the warp has seen what it needs,
// one fence.acq_rel.gpu orders the payload loads (read through L2) after the polls.
PM_INLINE unsigned lb_ld_status(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PM_INLINE void lb_fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Group arrival counter: acq_rel, so the payload this thread published is visible to the
// last arriver, which reads every tile's payload of the group after its own arrival.
PM_INLINE unsigned lb_arrive(unsigned* p) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}
// Bulk L2 prefetch (cp.async.bulk.prefetch, UBLKPF): pulls a contiguous block (16-B
// aligned, size a multiple of 16) into L2 without registers or shared memory, so the
// plan-table rows a tile reads later are L2 hits instead of DRAM round trips.
PM_INLINE void lb_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
PM_INLINE void lb_st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <typename R>
PM_INLINE R lb_ldcg(const R* p) {
  return __ldcg(p);
}

// First-wave stagger: with several waves of tiles, the CTAs of the first wave would run their
// phases in lock step (all staging y, then all looking back, then all storing x), so DRAM
// sees bursts of reads and of writes instead of a mix.  Delaying the start of the first
// wave's CTAs by (slot mod m) steps spreads the phases (C3, A/B on one box: pass 1a
// 0.1327 -> 0.1272 ms with m = 8, 1.1 us steps; pass 2 0.1361 -> 0.1291 ms with m = 6, 3 us
// steps; pass 1b, per warp, 0.0471 -> 0.0455 ms with m = 8, 0.8 us steps); later waves
// inherit the spread.  Off for problems of < 2 waves, whose CTAs would
// only wait.
PM_INLINE void lb_stagger(int64_t slot, int64_t resident, int64_t total, int step_ns, int mod) {
  if (step_ns > 0 && mod > 1 && total >= 2 * resident && slot < resident) {
    const unsigned ns = (unsigned)(slot % mod) * (unsigned)step_ns;
    for (unsigned t = 0; t < ns; t += 250u) __nanosleep(250u);
  }
}

// Optional delay injection for the look-back stress test (PMAP_LB_STRESS): a
// pseudo-random pause of up to ~16 us before a publication.
PM_INLINE void lb_stress(int stress, int64_t key, int salt) {
  if (stress) {
    unsigned h = (unsigned)(key * 2654435761ull) ^ (unsigned)(salt * 40503);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    const unsigned ns = (h & 7u) * 2000u;
    for (unsigned t = 0; t < ns; t += 1000u) __nanosleep(1000u);
  }
}

// The tile's y rows (nodes [n0, n0 + nvalid)) into padded shared-memory run rows,
// one cp.async (LDGSTS) per node row, consecutive threads on consecutive rows.
template <typename R, int NY, int NT, int K>
struct LbYStage {
  static constexpr int BYTES = NY * (int)sizeof(R);
  static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16 || BYTES % 16 == 0, "row size");
  static constexpr int ROW = ((K * NY * (int)sizeof(R) + 15) / 16 * 16 + 16) / (int)sizeof(R);
  static PM_INLINE void issue(R* ys, const R* src_y, int nvalid, int tid, int nthreads) {
    for (int q = tid; q < nvalid; q += nthreads) {
      const int run = q / K, mm = q - run * K;
      R* dst = ys + run * ROW + mm * NY;
      const R* srcp = src_y + (int64_t)q * NY;
      const unsigned sdst = (unsigned)__cvta_generic_to_shared(dst);
      if constexpr (BYTES % 16 == 0) {
#pragma unroll
        for (int c = 0; c < BYTES / 16; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst + 16 * c),
                       "l"(srcp + c * (16 / sizeof(R))));
      } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(sdst), "l"(srcp), "n"(BYTES));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  static PM_INLINE void wait() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
};


// Barrier of warps 1-2 (the 64 run threads of k_lb_pass1); warp 0 never joins it.
PM_INLINE void lb_bar_runs() { asm volatile("bar.sync 1, 64;" ::: "memory"); }

// Tile total of the NT = 64 run aggregates' data parts (r = run index 0..63, called by
// the 64 run threads only): a tree over aligned equal spans with the constant-bank
// coefficient sets of lti_run_reduce; run 63 ends with the total.
template <typename R, int N, int NY, int K>
PM_INLINE void lb_run_reduce64(const LtiFoldParams<R, N, NY, K, 6>& fp, int r, R (&bb)[N], R (&hh)[N], R* s_tot) {
  const int lane = r & 31;
  const unsigned FULL = 0xffffffffu;
  auto step = [&](int lg, const R (&b2)[N], const R (&h2)[N]) {
    R nb[N], nh[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R sb = b2[i], sb2 = R(0), sh_ = hh[i], sh2 = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        sb = fma(fp.Uf[lg][0][i][k], bb[k], sb);
        sb2 = fma(fp.Uf[lg][1][i][k], h2[k], sb2);
        sh_ = fma(fp.Uf[lg][2][i][k], h2[k], sh_);
        sh2 = fma(-fp.Uf[lg][3][i][k], bb[k], sh2);
      }
      nb[i] = sb + sb2;
      nh[i] = sh_ + sh2;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      bb[i] = nb[i];
      hh[i] = nh[i];
    }
  };
#pragma unroll
  for (int lg = 0; lg < 5; ++lg) {
    const int d = 1 << lg;
    R b2[N], h2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      b2[i] = __shfl_up_sync(FULL, bb[i], d);
      h2[i] = __shfl_up_sync(FULL, hh[i], d);
    }
    if (((lane + 1) & (2 * d - 1)) == 0) step(lg, b2, h2);  // lane ends an aligned span of 2d runs
  }
  if (r == 31) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      s_tot[i] = bb[i];
      s_tot[N + i] = hh[i];
    }
  }
  lb_bar_runs();
  if (r == 63) {
    R b2[N], h2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      b2[i] = s_tot[i];
      h2[i] = s_tot[N + i];
    }
    step(5, b2, h2);
  }
  lb_bar_runs();  // s_tot is reused
}

// Inclusive scan of the 64 run aggregates' data parts (run threads only; the warp-
// synchronous Kogge-Stone of lti_run_scan with the compact coefficient tables, the
// cross-warp step through s_tot and the run barrier).
template <typename R, int N>
PM_INLINE void lb_run_scan64(const R* __restrict__ UWc, const R* __restrict__ UX, int r, R (&bb)[N], R (&hh)[N],
                             R* s_tot) {
  const int lane = r & 31;
  const unsigned FULL = 0xffffffffu;
  auto step = [&](const R* __restrict__ U, int stride, int slot, const R (&b2)[N], const R (&h2)[N]) {
    R nb[N], nh[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R sb = b2[i], sb2 = R(0), sh_ = hh[i], sh2 = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        sb = fma(__ldg(U + ((0 * N + i) * N + k) * stride + slot), bb[k], sb);
        sb2 = fma(__ldg(U + ((1 * N + i) * N + k) * stride + slot), h2[k], sb2);
        sh_ = fma(__ldg(U + ((2 * N + i) * N + k) * stride + slot), h2[k], sh_);
        sh2 = fma(-__ldg(U + ((3 * N + i) * N + k) * stride + slot), bb[k], sh2);
      }
      nb[i] = sb + sb2;
      nh[i] = sh_ + sh2;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      bb[i] = nb[i];
      hh[i] = nh[i];
    }
  };
#pragma unroll
  for (int lg = 0; lg < 5; ++lg) {
    const int d = 1 << lg;
    R b2[N], h2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      b2[i] = __shfl_up_sync(FULL, bb[i], d);
      h2[i] = __shfl_up_sync(FULL, hh[i], d);
    }
    if (lane >= d) step(UWc + (d - 1) * 4 * N * N, d, min(lane - d, d - 1), b2, h2);
  }
  if (r == 31) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      s_tot[i] = bb[i];
      s_tot[N + i] = hh[i];
    }
  }
  lb_bar_runs();
  if (r >= 32) {
    R b2[N], h2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      b2[i] = s_tot[i];
      h2[i] = s_tot[N + i];
    }
    step(UX, 32, lane, b2, h2);
  }
}

template <typename R, int N>
PM_INLINE void lb_matvec(const R* __restrict__ P, const R (&x)[N], R (&o)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R a = R(0);
#pragma unroll
    for (int c = 0; c < N; ++c) a = fma(__ldg(P + i * N + c), x[c], a);
    o[i] = a;
  }
}

template <typename R, int N>
PM_INLINE void lb_warp_sum(R (&s)[N]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < N; ++i) s[i] += __shfl_xor_sync(0xffffffffu, s[i], o);
}

// ------------------------------------------------------------------ pass 1a
// Per tile, no waiting: the run folds of the node elements' data parts (LTI impulse
// responses, R-LTI), the tile aggregate g_j (tree over the runs) and, by the group's last
// arriver, the group aggregate g_G; then the in-tile run scan and every run's pass-2 map
// as an affine function of the still unknown v entering the tile:
//   v_{s-1} = GP v_in + c,   c = ph - GP S_in pb,
//   beta = WR (rb + C_R v_{s-1}) = beta0 + WR C_R GP v_in,   beta0 = WR (rb + C_R c);
// the suffix composition of (PHI, beta0) is each run's map with v_in = 0 (its offset's
// v_in-coefficient QB is a plan table).  Stored: c (rcv), the maps (ri), g_j.
template <typename R, int N, int NY, int NT, int K, class Src>
__global__ void __launch_bounds__(NT, 6)
    k_lb_pass1a(const __grid_constant__ LtiFoldParams<R, N, NY, K, Log2<NT>::value> fp, const LbGeom g,
                const R* __restrict__ y, const LtiTables<R, N, NT, K>* __restrict__ tab,
                const LbTileTab<R, N>* __restrict__ lt, const R* __restrict__ lrt, const LbWs<R> w) {
  using A = Aff<R, N>;
  using YS = LbYStage<R, NY, NT, K>;
  constexpr int L = NT * K;
  constexpr int NS = Dim<N>::NS;
  static_assert(NT == 64, "64 run threads per tile");
  __shared__ __align__(16) R ys[NT * YS::ROW];
  __shared__ R s_tot[2 * N];  // cross-warp step of the run reduce / scan
  __shared__ R s_a32[A::SZ];  // runs 32..63 suffix map (cross-warp)
  const int r = threadIdx.x, lane = r & 31;
  const unsigned FULL = 0xffffffffu;
  const int64_t tile = blockIdx.x;
  const int64_t b = tile / g.tpt, j = tile % g.tpt;
  const int64_t G = j / kLbGroup;
  const bool last = (j == g.tpt - 1);
  lb_stagger((int64_t)blockIdx.x, g.S2, (int64_t)gridDim.x, g.stagger1, g.stmod1);
  LB_STAMP(0, 0);
  const int64_t n0 = 1 + j * (int64_t)L;
  const int nvalid = (int)min((int64_t)L, g.Nn - n0);
  const R* yb = y + b * g.Nn * NY;
  if (r == 0)  // this tile's run tables GP, WR, PHI (read after the scan) into L2 now
    lb_prefetch_l2(lrt + j * (int64_t)LbRunTab<N>::F * NT, (unsigned)(sizeof(R) * 3 * N * N * NT));
  YS::issue(ys, yb + n0 * NY, nvalid, r, NT);
  YS::wait();
  __syncthreads();
  LB_STAMP(0, 1);
  const int q = max(0, min(K, nvalid - r * K));
  R rb[N], rh[N], bb[N], hh[N];
  {
    const R* yr = ys + r * YS::ROW;
    if (q == K) {
      R acc0[2 * N], acc1[2 * N];
#pragma unroll
      for (int i = 0; i < 2 * N; ++i) {
        acc0[i] = fp.crun[i];
        acc1[i] = R(0);
      }
#pragma unroll
      for (int m = 0; m < K; m += 2) {
#pragma unroll
        for (int i = 0; i < 2 * N; ++i)
#pragma unroll
          for (int k = 0; k < NY; ++k) {
            acc0[i] = fma(fp.GK[m][i][k], yr[m * NY + k], acc0[i]);
            acc1[i] = fma(fp.GK[m + 1][i][k], yr[(m + 1) * NY + k], acc1[i]);
          }
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        rb[i] = acc0[i] + acc1[i];
        rh[i] = acc0[N + i] + acc1[N + i];
      }
    } else if (q > 0) {
      lti_fold_data<R, N, NY, NT, K>(fp.node, tab, q, [&](int m) { return yr + m * NY; }, rb, rh);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) rb[i] = rh[i] = R(0);
    }
  }
  if (!last) {  // every tile but the last is full: g_j from the tile total (tree over the runs)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      bb[i] = rb[i];
      hh[i] = rh[i];
    }
    lb_run_reduce64<R, N, NY, K>(fp, r, bb, hh, s_tot);
    if (r == NT - 1) {
      R gj[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        R s = hh[i];
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(-__ldg(&lt[j].Hs[i][k]), bb[k], s);
        gj[i] = s;
      }
#pragma unroll
      for (int i = 0; i < N; ++i) w.agg1[tile * N + i] = gj[i];
    }
  }
  const bool full_group = (G + 1) * kLbGroup <= g.tpt - 1;  // every tile of the group precedes the last tile
  LB_STAMP(0, 2);
  // in-tile inclusive scan; exclusive prefix (pb, ph) of run r (0 for run 0)
#pragma unroll
  for (int i = 0; i < N; ++i) {
    bb[i] = rb[i];
    hh[i] = rh[i];
  }
  lb_run_scan64<R, N>(tab->UWc, &tab->UX[0][0][0][0], r, bb, hh, s_tot);
  R pb[N], ph[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    pb[i] = __shfl_up_sync(FULL, bb[i], 1);
    ph[i] = __shfl_up_sync(FULL, hh[i], 1);
  }
  __syncthreads();
  if (r == 32) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      pb[i] = s_tot[i];
      ph[i] = s_tot[N + i];
    }
  }
  if (r == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) pb[i] = ph[i] = R(0);
  }
  const R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;  // field f of run r at rt[f * NT]
  R cvec[N];
  {
    R u[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(-__ldg(&lt[j].S[i <= k ? sidx(i, k, N) : sidx(k, i, N)]), pb[k], s);
      u[i] = s;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = ph[i];
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(__ldg(rt + (LbRunTab<N>::GP + i * N + k) * NT), u[k], s);
      cvec[i] = s;
    }
  }
  A agg;
  set_identity(agg);
  if (q > 0) {
    R CR[NS];  // C of the run element: one full run (E1) or the partial run of q nodes
#pragma unroll
    for (int k = 0; k < NS; ++k) CR[k] = (q == K) ? __ldg(&tab->E1[N * N + N + k]) : __ldg(&tab->PC[q - 1][k]);
    R t2[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = rb[i];
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(CR[i <= k ? sidx(i, k, N) : sidx(k, i, N)], cvec[k], s);
      t2[i] = s;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(__ldg(rt + (LbRunTab<N>::WR + i * N + k) * NT), t2[k], s);
      agg.q[i] = s;
#pragma unroll
      for (int c = 0; c < N; ++c) agg.P[i][c] = __ldg(rt + (LbRunTab<N>::PHI + i * N + c) * NT);
    }
  }
  // in-tile suffix composition: Incl_r = agg_r o ... o agg_{NT-1}
#pragma unroll 1
  for (int d = 1; d < 32; d <<= 1) {
    A o;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int c = 0; c < N; ++c) o.P[i][c] = __shfl_down_sync(FULL, agg.P[i][c], d);
      o.q[i] = __shfl_down_sync(FULL, agg.q[i], d);
    }
    if (lane + d < 32) compose(agg, o, agg);
  }
  if (r == 32) store(agg, s_a32, 1);
  __syncthreads();
  if (r < 32) {
    A o;
    load(o, s_a32, 1);
    compose(agg, o, agg);
  }
#pragma unroll
  for (int i = 0; i < N; ++i) w.rcv[(tile * N + i) * NT + r] = cvec[i];
#pragma unroll
  for (int i = 0; i < N; ++i) w.ri[(tile * (int64_t)A::SZ + N * N + i) * NT + r] = agg.q[i];  // the matrix is PS
  if (last && q > 0 && n0 + (int64_t)r * K + q == g.Nn) {  // the run ending at node T: keep its data parts
#pragma unroll
    for (int i = 0; i < N; ++i) {
      w.seedrb[b * 2 * N + i] = rb[i];
      w.seedrb[b * 2 * N + N + i] = rh[i];
    }
  }
  // the group aggregate, by the group's last arriver (after everything else of the tile,
  // so the atomic's round trip is off the tile's critical path):
  //   g_G = sum_l Pa[32G + 32][l] g_{32G + 31 - l}
  if (full_group && r >= 32) {
    unsigned gl = 0;
    if (r == NT - 1) gl = lb_arrive(&w.gcnt1[b * g.gpt + G]) == kLbGroup - 1;
    gl = __shfl_sync(FULL, gl, 31);
    if (gl) {
      R x[N], sg[N];
#pragma unroll
      for (int i = 0; i < N; ++i) x[i] = lb_ldcg(w.agg1 + (b * g.tpt + G * kLbGroup + kLbGroup - 1 - lane) * N + i);
      lb_matvec<R, N>(w.Pa + (((G + 1) * kLbGroup) * (kLbGroup + 1) + lane) * N * N, x, sg);
      lb_warp_sum<R, N>(sg);
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) w.gagg1[(b * g.gpt + G) * N + i] = sg[i];
        atomicExch(&w.gcnt1[b * g.gpt + G], 0u);
      }
    }
  }
  LB_STAMP(0, 3);
}

// The value function leaving the run that ends at the trajectory's (chunk's) last node,
// from the value function entering it (S from the plan's run table, v = vp) and the run's
// element (full or partial run; data parts kept by pass 1a in seedrb).
template <typename R, int N, int NT, int K>
PM_INLINE void lb_run_vend(const LtiTables<R, N, NT, K>* __restrict__ tab, const R* __restrict__ rt, const R (&vp)[N],
                           int q, const R* __restrict__ seedrb, VF<R, N>& vend, bool& ok) {
  constexpr int NS = Dim<N>::NS;
  VF<R, N> cur;
#pragma unroll
  for (int k = 0; k < NS; ++k) cur.S[k] = __ldg(rt + (LbRunTab<N>::SP + k) * NT);
#pragma unroll
  for (int i = 0; i < N; ++i) cur.v[i] = vp[i];
  Elem<R, N> ra;
  if (q == K) {
    load(ra, tab->E1, 1);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int jj = 0; jj < N; ++jj) ra.A[i][jj] = __ldg(&tab->PA[q - 1][i][jj]);
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      ra.C[k] = __ldg(&tab->PC[q - 1][k]);
      ra.J[k] = __ldg(&tab->PJ[q - 1][k]);
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    ra.b[i] = seedrb[i];
    ra.h[i] = seedrb[N + i];
  }
  vapply<R, N, false>(ra, cur, vend, nullptr, ok);
}

// ------------------------------------------------------------------ pass 1b
// One warp per tile: the decoupled look-back for v entering the tile over the tile
// aggregates g (pass 1a wrote every g and group g_G, so nothing is waited for; a
// published prefix only shortens the walk):
//   v_end(j-1) = sum_{l < l*} Pa[j][l] g_{j-1-l} + Pa[j][l*] v_end(j-1-l*)
// over the tiles of j's group, else + Pa[j][cnt] v_end(32G - 1) with
//   v_end(32G - 1) = sum_{l < l*} Pb[G][l] g_{G-1-l} + Pb[G][l*] v_end(group G-1-l*)
// over whole groups (group -1 = node 0); then the finished run values for pass 2:
// v_{s-1} = GP v_in + c (rcv), the maps' offsets q += QB v_in (ri), the tile's pass-2
// offset beta_tile (agg2), the group's (last arriver, agg2 -> gagg2), and x*_T.
template <typename R, int N, int NY, int NT, int K, class Src>
__global__ void __launch_bounds__(128)
    k_lb_pass1b(const __grid_constant__ Src src, const LbGeom g, const R* __restrict__ y,
                const LtiTables<R, N, NT, K>* __restrict__ tab, const LbTileTab<R, N>* __restrict__ lt,
                const R* __restrict__ lrt, const LbWs<R> w, unsigned long long* flag, int stress,
                const R* __restrict__ vin0, int probe, R* __restrict__ probe_out) {
  // vin0 (nullable): v entering the chunk (a time shard's carry-in)
  // instead of node 0's prior + y_0.  probe: one warp, the last tile only, no publication:
  // the value function's v leaving the chunk -> probe_out (a shard's pass-1 payload).
  using E = Elem<R, N>;
  using V = VF<R, N>;
  using A = Aff<R, N>;
  constexpr int NS = Dim<N>::NS;
  constexpr int L = NT * K;
  static_assert(NT == 64, "two runs per lane");
  __shared__ int s_ticket[4];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const int64_t total = g.batch * g.tpt;
  int64_t u;
  if (probe) {
    if (blockIdx.x != 0 || wid != 0) return;
    u = g.tpt - 1;  // trajectory 0 (probes run on batch-1 plans), last tile
  } else {
    const int64_t nticket = lb_ticket_count(total, g.S1);
    if ((int64_t)blockIdx.x * 4 + wid >= nticket) return;  // no ticket for the grid's spare warps
    if (lane == 0) {
      const unsigned t = atomicAdd(&w.ctr[0], 1u);
      if (t == nticket - 1) atomicExch(&w.ctr[0], 0u);  // every ticket is taken: reset for the next solve
      s_ticket[wid] = (int)t;
    }
    __syncwarp();
    const int64_t t = s_ticket[wid];
    if (t >= nticket) return;
    u = lb_stride_map(t, total, g.S1);
    if (u >= total) return;
    lb_stagger(t, g.S1, total, g.stagger1b, 8);
  }
  const int64_t b = u / g.tpt, j = u % g.tpt;
  const int64_t tile = b * g.tpt + j;
  const int64_t G = j / kLbGroup;
  const bool last = (j == g.tpt - 1);
  const int64_t n0 = 1 + j * (int64_t)L;
  if (lane == 0) {
    if (!probe) w.flag2[tile] = 0u;  // pass-2 prefix status of the previous solve
    if (w.tim) w.tim[tile * 8 + 4] = lb_now();
    // what the run values need after the look-back, into L2 now: GP, QB, c, the maps' offsets
    const R* rt0 = lrt + j * (int64_t)LbRunTab<N>::F * NT;
    lb_prefetch_l2(rt0 + LbRunTab<N>::GP * NT, (unsigned)(sizeof(R) * N * N * NT));
    lb_prefetch_l2(rt0 + LbRunTab<N>::QB * NT, (unsigned)(sizeof(R) * N * N * NT));
    lb_prefetch_l2(w.rcv + tile * (int64_t)N * NT, (unsigned)(sizeof(R) * N * NT));
    lb_prefetch_l2(w.ri + tile * (int64_t)A::SZ * NT + N * N * NT, (unsigned)(sizeof(R) * N * NT));
  }
  const R* yb = y + b * g.Nn * NY;
  R eta0[N];  // v of node 0: P0^-1 m0 + K y_0 - K r (E_0's data), or the chunk's carry-in
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = src.h00[i];
    if (vin0) {
      s = vin0[b * N + i];
    } else {
#pragma unroll
      for (int k = 0; k < NY; ++k) s = fma(src.K[i][k], __ldg(yb + k), s);
    }
    eta0[i] = s;
  }
  R vin[N];
  bool quick = false;
  if (j > 0) {  // the usual case (strided tickets): the previous tile's prefix is v_in
    unsigned s0 = 0;
    if (lane == 0) s0 = lb_ld_status(&w.flag1[b * g.tpt + j - 1]);
    s0 = __shfl_sync(FULL, s0, 0);
    if (s0 == 2u) {
      lb_fence_acquire();
#pragma unroll
      for (int i = 0; i < N; ++i) vin[i] = lb_ldcg(w.pub1 + (b * g.tpt + j - 1) * N + i);
      quick = true;
    }
  }
  if (j == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) vin[i] = eta0[i];
  } else if (!quick) {
    const int cnt = (int)(j - G * kLbGroup);
    const int64_t ka = j - 1 - lane;
    const int64_t Gp = G - 1 - lane;
    R Pa_l[N][N], Pb_l[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        Pa_l[i][c] = __ldg(w.Pa + ((j * (kLbGroup + 1) + lane) * N + i) * N + c);
        Pb_l[i][c] = (lane <= G) ? __ldg(w.Pb + ((G * (G + 1) / 2 + lane) * N + i) * N + c) : R(0);
      }
    // (b) status of group Gp: 2 = its last tile's prefix, 1 = its aggregate (written by
    // pass 1a), 3 = node 0
    auto group_status = [&](int64_t Gx) -> unsigned {
      if (Gx < -1) return 0u;
      if (Gx == -1) return 3u;
      return lb_ld_status(&w.flag1[b * g.tpt + Gx * kLbGroup + kLbGroup - 1]) == 2u ? 2u : 1u;
    };
    const unsigned sta = lane < cnt ? lb_ld_status(&w.flag1[b * g.tpt + ka]) : 0u;
    const unsigned prea = __ballot_sync(FULL, sta == 2u);
    const unsigned stb = prea ? 0u : group_status(Gp);
    const unsigned preb = prea ? 0u : __ballot_sync(FULL, stb >= 2u);
    if (prea || preb) lb_fence_acquire();
    const int la = prea ? __ffs(prea) - 1 : cnt;
    R sa[N];
    {
      R x[N];
      const bool use = lane < la || (lane == la && prea);
#pragma unroll
      for (int i = 0; i < N; ++i)
        x[i] = !use ? R(0)
                    : (lane < la ? w.agg1[(b * g.tpt + ka) * N + i] : lb_ldcg(w.pub1 + (b * g.tpt + ka) * N + i));
#pragma unroll
      for (int i = 0; i < N; ++i) {
        R t2 = R(0);
#pragma unroll
        for (int c = 0; c < N; ++c) t2 = fma(Pa_l[i][c], x[c], t2);
        sa[i] = t2;
      }
    }
    if (!prea) {
      R sb[N];
      const int lb = preb ? __ffs(preb) - 1 : 32;
      {
        R x[N];
        const bool use = lane < lb || (lane == lb && preb);
#pragma unroll
        for (int i = 0; i < N; ++i)
          x[i] = !use ? R(0)
                      : (stb == 3u ? eta0[i]
                                   : (lane < lb ? w.gagg1[(b * g.gpt + Gp) * N + i]
                                                : lb_ldcg(w.pub1 + (b * g.tpt + Gp * kLbGroup + kLbGroup - 1) * N + i)));
#pragma unroll
        for (int i = 0; i < N; ++i) {
          R t2 = R(0);
#pragma unroll
          for (int c = 0; c < N; ++c) t2 = fma(Pb_l[i][c], x[c], t2);
          sb[i] = t2;
        }
      }
      if (!preb) {  // more than 32 groups to the nearest prefix (or node 0)
        const R* PbG = w.Pb + (G * (G + 1) / 2) * N * N;
        for (int64_t l0 = 32;; l0 += 32) {
          const int64_t l = l0 + lane;
          const int64_t Gq = G - 1 - l;
          const unsigned st = group_status(Gq);
          const unsigned pre = __ballot_sync(FULL, st >= 2u);
          if (pre) lb_fence_acquire();
          const int lstar = pre ? __ffs(pre) - 1 : 32;
          if (lane <= lstar && Gq >= -1) {
            R x[N], o[N];
#pragma unroll
            for (int i = 0; i < N; ++i)
              x[i] = st == 3u ? eta0[i]
                              : (lane < lstar ? w.gagg1[(b * g.gpt + Gq) * N + i]
                                              : lb_ldcg(w.pub1 + (b * g.tpt + Gq * kLbGroup + kLbGroup - 1) * N + i));
            lb_matvec<R, N>(PbG + l * N * N, x, o);
#pragma unroll
            for (int i = 0; i < N; ++i) sb[i] += o[i];
          }
          if (pre) break;
        }
      }
      lb_warp_sum<R, N>(sb);
      R o[N];  // + Pa[j][cnt] v_end(32G - 1): Pa[j][cnt] is lane cnt's Pa_l
#pragma unroll
      for (int i = 0; i < N; ++i) {
        R t2 = R(0);
#pragma unroll
        for (int c = 0; c < N; ++c) t2 = fma(__shfl_sync(FULL, Pa_l[i][c], cnt), sb[c], t2);
        o[i] = t2;
      }
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) sa[i] += o[i];
      }
    }
    lb_warp_sum<R, N>(sa);
#pragma unroll
    for (int i = 0; i < N; ++i) vin[i] = sa[i];
  }
  if (lane == 0 && w.tim) w.tim[tile * 8 + 5] = lb_now();
  if (probe) {  // v leaving the chunk: the run ending at its last node (read-only)
    bool okp = true;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      const int q = (int)max((int64_t)0, min((int64_t)K, g.Nn - n0 - (int64_t)r * K));
      if (q > 0 && n0 + (int64_t)r * K + q == g.Nn) {
        const R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;
        const R* cv = w.rcv + tile * (int64_t)N * NT + r;
        R vp[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          R s = cv[i * NT];
#pragma unroll
          for (int k = 0; k < N; ++k) s = fma(__ldg(rt + (LbRunTab<N>::GP + i * N + k) * NT), vin[k], s);
          vp[i] = s;
        }
        V vend;
        lb_run_vend<R, N, NT, K>(tab, rt, vp, q, w.seedrb + b * 2 * N, vend, okp);
#pragma unroll
        for (int i = 0; i < N; ++i) probe_out[b * N + i] = vend.v[i];
      }
    }
    if (!okp) atomicMin(flag, (unsigned long long)(g.Nn - 1));
    return;
  }
  if (lane == 0 && !last) {  // inclusive prefix: v leaving the tile
    lb_stress(stress, tile, 3);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = w.agg1[tile * N + i];
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(__ldg(&lt[j].Gt[i][k]), vin[k], s);
      w.pub1[tile * N + i] = s;
    }
    lb_st_release(&w.flag1[tile], 2u);
  }
  // finish the run values: two runs per lane
  bool ok = true;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = lane + 32 * h;
    const R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;
    R* cv = w.rcv + tile * (int64_t)N * NT + r;
    R* qv = w.ri + tile * (int64_t)A::SZ * NT + N * N * NT + r;  // the offset fields of the run's map
    R vp[N], qn[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = cv[i * NT], s2 = qv[i * NT];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s = fma(__ldg(rt + (LbRunTab<N>::GP + i * N + k) * NT), vin[k], s);
        s2 = fma(__ldg(rt + (LbRunTab<N>::QB + i * N + k) * NT), vin[k], s2);
      }
      vp[i] = s;
      qn[i] = s2;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      cv[i * NT] = vp[i];
      qv[i * NT] = qn[i];
    }
    if (r == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i) w.agg2[tile * N + i] = qn[i];  // run 0's map = the tile's pass-2 map
    }
    const int q = (int)max((int64_t)0, min((int64_t)K, g.Nn - n0 - (int64_t)r * K));
    if (last && q > 0 && n0 + (int64_t)r * K + q == g.Nn) {  // the run ending at node T: x*_T = S_T^-1 v_T
      V vend;
      lb_run_vend<R, N, NT, K>(tab, rt, vp, q, w.seedrb + b * 2 * N, vend, ok);
      R xT[N];
      spd_solve<R, N>(vend.S, vend.v, xT, ok);
#pragma unroll
      for (int i = 0; i < N; ++i) w.seed[b * N + i] = xT[i];
    }
  }
  // the group's pass-2 offset, by its last arriver: beta_G = sum_l Qa[32G - 1][l] beta_{32G + l}
  if (G >= 1) {
    const int gcount = (int)min((int64_t)kLbGroup, g.tpt - G * kLbGroup);
    unsigned gl = 0;
    if (lane == 0) gl = lb_arrive(&w.gcnt2[b * g.gpt + G]) == (unsigned)(gcount - 1);
    gl = __shfl_sync(FULL, gl, 0);
    if (gl) {
      R s[N];
#pragma unroll
      for (int i = 0; i < N; ++i) s[i] = R(0);
      if (lane < gcount) {
        R x[N];
#pragma unroll
        for (int i = 0; i < N; ++i) x[i] = lb_ldcg(w.agg2 + (b * g.tpt + G * kLbGroup + lane) * N + i);
        lb_matvec<R, N>(w.Qa + ((G * kLbGroup - 1) * (kLbGroup + 1) + lane) * N * N, x, s);
      }
      lb_warp_sum<R, N>(s);
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) w.gagg2[(b * g.gpt + G) * N + i] = s[i];
        atomicExch(&w.gcnt2[b * g.gpt + G], 0u);
      }
    }
  }
  if (lane == 0 && w.tim) w.tim[tile * 8 + 6] = lb_now();
  if (!ok) atomicMin(flag, (unsigned long long)(g.Nn - 1));
}

// The structural-zero mask of S a source's pass-2 node recursion may rely on (R-SMASK;
// SrcLTI::SMASK, ~0u = dense for every other source).
template <class Src, class = void>
struct SrcSMask {
  static constexpr uint32_t value = ~0u;
};
template <class Src>
struct SrcSMask<Src, std::void_t<decltype(Src::SMASK)>> {
  static constexpr uint32_t value = Src::SMASK;
};
template <class Src>
__host__ __device__ constexpr uint32_t src_smask() {
  return SrcSMask<Src>::value;
}

// One forward node step (R-FWD + the node update): x <- A^-1 [x - b + C (S x - v)] with
// the value function V = V_{i-1} entering node i, then V <- E_i (x) V (Woodbury form
// for a low-rank diffusion C = U U^T, R-LOWRANK; the general update otherwise).
template <typename R, int N, class Src>
PM_INLINE void lb_node_step(const Src& src, const Elem<R, N>& e, VF<R, N>& V, R (&x)[N], bool& ok) {
  constexpr int NW = Src::LOWRANK > 0 ? Src::LOWRANK : 1;
  R z[N];
  if constexpr (Src::LOWRANK > 0) {
    // u = U^T (S x - v)
    R u[NW];
#pragma unroll
    for (int a = 0; a < NW; ++a) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (mask_nz(Src::UMASK, k * NW + a)) {
          R t = -V.v[k];
#pragma unroll
          for (int l = 0; l < N; ++l)
            if (sm_nz(src_smask<Src>(), k, l, N)) t = fma(V.S[sidx(k, l, N)], x[l], t);
          s = fma(src.U[k][a], t, s);
        }
      u[a] = s;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = src.zero_b ? x[i] : x[i] - src.b[i];
#pragma unroll
      for (int a = 0; a < NW; ++a)
        if (mask_nz(Src::UMASK, i * NW + a)) s = fma(src.U[i][a], u[a], s);
      z[i] = s;
    }
  } else {
    R t[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      R s = -V.v[k];
#pragma unroll
      for (int l = 0; l < N; ++l) s = fma(V.S[sidx(k, l, N)], x[l], s);
      t[k] = s;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = x[i] - src.b[i];
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(src.C[sidx(i, k, N)], t[k], s);
      z[i] = s;
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (mask_nz(Src::AMASK, i * N + k)) s = fma(src.Am[i][k], z[k], s);  // A^-1 shares A's masked pattern
    x[i] = s;
  }
  if constexpr (Src::LOWRANK > 0)
    vapply_lowrank<R, N, Src::LOWRANK, Src::AMASK, Src::UMASK, src_smask<Src>()>(e, src.U, V, V, ok, nullptr, 0,
                                                                                src.zero_b != 0);
  else
    vapply<R, N, false>(e, V, V, nullptr, ok);
}

template <typename R, int N>
PM_INLINE void lb_store_x(R* __restrict__ dst, const R (&x)[N]) {
  if constexpr (N == 4 && sizeof(R) == 8) {
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(x[0]), "d"(x[1]), "d"(x[2]), "d"(x[3])
                 : "memory");
  } else if constexpr (N == 4 && sizeof(R) == 4) {
    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3])
                 : "memory");
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) dst[i] = x[i];
  }
}


// Smoother covariance, forward inside a run (R-FWD applied to the RTS covariance
// recursion P^s_{i-1} = Phi_i P^s_i Phi_i^T + Sigma_i, Phi_i = M^-1 A_i, Sigma_i = M^-1 C_i,
// M = I + C_i S_{i-1}, R-SCOV):  P^s_i = A_i^-1 (M P^s_{i-1} M^T - C_i M^T) A_i^-T,
// C M^T = C + C S C (symmetric).  S = S_{i-1}; the upper triangle only.
template <typename R, int N, class Src>
PM_INLINE void lb_cov_step(const Src& src, const R (&S)[Dim<N>::NS], R (&P)[Dim<N>::NS]) {
  R Cf[N][N], Sf[N][N], Pf[N][N], M[N][N], CS[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      Cf[i][c] = src.C[i <= c ? sidx(i, c, N) : sidx(c, i, N)];
      Sf[i][c] = S[i <= c ? sidx(i, c, N) : sidx(c, i, N)];
      Pf[i][c] = P[i <= c ? sidx(i, c, N) : sidx(c, i, N)];
    }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      R a = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) a = fma(Cf[i][k], Sf[k][c], a);
      CS[i][c] = a;
      M[i][c] = a + (i == c ? R(1) : R(0));
    }
  R MP[N][N], Tm[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      R a = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) a = fma(M[i][k], Pf[k][c], a);
      MP[i][c] = a;
    }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      R a = -Cf[i][c];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        a = fma(MP[i][k], M[c][k], a);
        a = fma(-CS[i][k], Cf[k][c], a);
      }
      Tm[i][c] = a;
    }
  R AT[N][N];  // A^-1 Tm
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) {
      R a = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (mask_nz(Src::AMASK, i * N + k)) a = fma(src.Am[i][k], Tm[k][c], a);
      AT[i][c] = a;
    }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = i; c < N; ++c) {
      R a = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (mask_nz(Src::AMASK, c * N + k)) a = fma(AT[i][k], src.Am[c][k], a);
      P[sidx(i, c, N)] = a;
    }
}

// Plan time, one thread per tile: the run maps of the covariance recursion, Phi_r and
// Sigma_r = WR_r C_R, composed over the tile (run 0 outermost): Sigma_tile (Phi_tile is
// k_lb_setup_tiles').  (Phi_a, Sigma_a) o (Phi_b, Sigma_b) = (Phi_a Phi_b, Phi_a Sigma_b Phi_a^T + Sigma_a).
template <typename R, int N, int NT, int K>
__global__ void k_lb_cov_tiles(const LtiTables<R, N, NT, K>* __restrict__ tab, const R* __restrict__ lrt, int64_t tpt,
                               int64_t Nn, double* __restrict__ sig_tile) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= tpt) return;
  const int64_t n0 = 1 + j * (int64_t)NT * K;
  double Sg[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) Sg[i][c] = 0.0;
  for (int r = NT - 1; r >= 0; --r) {
    const int q = (int)max((int64_t)0, min((int64_t)K, Nn - n0 - (int64_t)r * K));
    if (q == 0) continue;
    const R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;
    double Ph[N][N], Wr[N][N], Cr[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        Ph[i][c] = (double)rt[(LbRunTab<N>::PHI + i * N + c) * NT];
        Wr[i][c] = (double)rt[(LbRunTab<N>::WR + i * N + c) * NT];
        const int kk = i <= c ? sidx(i, c, N) : sidx(c, i, N);
        Cr[i][c] = (double)((q == K) ? tab->E1[N * N + N + kk] : tab->PC[q - 1][kk]);
      }
    double T[N][N], U[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) a = fma(Ph[i][k], Sg[k][c], a);
        T[i][c] = a;
      }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          a = fma(T[i][k], Ph[c][k], a);
          a = fma(Wr[i][k], Cr[k][c], a);
        }
        U[i][c] = a;
      }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = 0; c < N; ++c) Sg[i][c] = 0.5 * (U[i][c] + U[c][i]);
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) sig_tile[(j * N + i) * N + c] = Sg[i][c];
}

// Plan time, one thread per tile: from P^s at the tile's last node, backwards over the
// runs, P^s at the node before each run (the start value of the forward recursion).
template <typename R, int N, int NT, int K>
__global__ void k_lb_cov_runs(const LtiTables<R, N, NT, K>* __restrict__ tab, const R* __restrict__ lrt, int64_t tpt,
                              int64_t Nn, const double* __restrict__ pend, R* __restrict__ lcov) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= tpt) return;
  const int64_t n0 = 1 + j * (int64_t)NT * K;
  double P[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int c = 0; c < N; ++c) P[i][c] = pend[(j * N + i) * N + c];
  for (int r = NT - 1; r >= 0; --r) {
    const int q = (int)max((int64_t)0, min((int64_t)K, Nn - n0 - (int64_t)r * K));
    if (q > 0) {
      const R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;
      double Ph[N][N], Wr[N][N], Cr[N][N], T[N][N], U[N][N];
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          Ph[i][c] = (double)rt[(LbRunTab<N>::PHI + i * N + c) * NT];
          Wr[i][c] = (double)rt[(LbRunTab<N>::WR + i * N + c) * NT];
          const int kk = i <= c ? sidx(i, c, N) : sidx(c, i, N);
          Cr[i][c] = (double)((q == K) ? tab->E1[N * N + N + kk] : tab->PC[q - 1][kk]);
        }
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          double a = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) a = fma(Ph[i][k], P[k][c], a);
          T[i][c] = a;
        }
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          double a = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            a = fma(T[i][k], Ph[c][k], a);
            a = fma(Wr[i][k], Cr[k][c], a);
          }
          U[i][c] = a;
        }
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) P[i][c] = 0.5 * (U[i][c] + U[c][i]);
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int c = i; c < N; ++c) lcov[(j * Dim<N>::NS + sidx(i, c, N)) * NT + r] = (R)P[i][c];
  }
}

// ------------------------------------------------------------------ time shards
// The two exchanges of the sharded look-back, one thread each (batch 1).
// v entering rank r's chunk: v = (v leaving rank 0, absolute); v = Gc_s v + v0_s for s = 1..r-1,
// gathered = [world][v0 (N) | Gc (N*N)].
template <typename R, int N>
__global__ void k_lb_shard_vin(const R* __restrict__ gathered, int rank, R* __restrict__ vin) {
  constexpr int P1 = N + N * N;
  R v[N];
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = gathered[i];
  for (int sr = 1; sr < rank; ++sr) {
    const R* pl = gathered + (int64_t)sr * P1;
    R nv[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R a = pl[i];
#pragma unroll
      for (int c = 0; c < N; ++c) a = fma(pl[N + i * N + c], v[c], a);
      nv[i] = a;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = nv[i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) vin[i] = v[i];
}
// x at rank r's last node: x = x*_T (the last rank's); x = Pc_s x + beta_s for s = world-1 .. r+1,
// gathered = [world][beta (N) | Pc (N*N) | x*_T (N)].
template <typename R, int N>
__global__ void k_lb_shard_xend(const R* __restrict__ gathered, int rank, int world, R* __restrict__ xend) {
  constexpr int P2 = 2 * N + N * N;
  R x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = gathered[(int64_t)(world - 1) * P2 + N + N * N + i];
  for (int sr = world - 1; sr > rank; --sr) {
    const R* pl = gathered + (int64_t)sr * P2;
    R nx[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R a = pl[i];
#pragma unroll
      for (int c = 0; c < N; ++c) a = fma(pl[N + i * N + c], x[c], a);
      nx[i] = a;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = nx[i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) xend[i] = x[i];
}

// ------------------------------------------------------------------ pass 2
// OUT = 1: also write the filter outputs m_i = S_i^-1 v_i, P_i = S_i^-1 to
// (fm, fP); OUT = 2: the smoother covariances P^s_i (R-SCOV) to fP, forward inside each run
// from the plan's P^s at the node before the run (lcov).
// RC: precision of the per-node recursion (R, or float from an fp64 plan: MAP_FLAG_MIXED,
// where every run restarts from fp64 carries and x leaves as fp64).
template <typename R, int N, int NY, int NT, int K, class Src, int OUT, typename RC = R>
__global__ void __maxnreg__(PM_LB2_MAXREG)
    k_lb_pass2(const __grid_constant__ typename Src::template rebind<RC> src, const LbGeom g, const R* __restrict__ y,
               const R* __restrict__ lrt, const LbWs<R> w, R* __restrict__ x_out, R* __restrict__ fm,
               R* __restrict__ fP, const R* __restrict__ lcov, unsigned long long* flag, int stress,
               const R* __restrict__ seed_in, int store0, int probe, R* __restrict__ probe_out,
               const R* __restrict__ phit) {
  // seed_in (nullable): x* at the chunk's last node (a time shard's carry from the ranks
  // after it) instead of x*_T from pass 1b; store0: write node 0 (rank 0 only).  probe: one
  // CTA, tile 0 only, no publication, no node loop: x* at node 0 for x* = seed_in at the
  // chunk's end -> probe_out (a shard's pass-2 payload; phit = the tiles' pass-2 matrices).
  constexpr bool FO = OUT == 1;
  constexpr bool MIXED = !std::is_same<R, RC>::value;
  static_assert(!MIXED || OUT == 0, "mixed precision: trajectory only");
  using SrcC = typename Src::template rebind<RC>;
  using E = Elem<R, N>;
  using V = VF<R, N>;
  using A = Aff<R, N>;
  using YS = LbYStage<R, NY, NT, K>;
  constexpr int L = NT * K;
  constexpr int NS = Dim<N>::NS;
  static_assert(NT == 64, "two warps per tile");
  __shared__ __align__(16) R ys[NT * YS::ROW];
  __shared__ int s_ticket;
  __shared__ R s_x[N];  // x at the tile's last node
  const int r = threadIdx.x, lane = r & 31;
  const unsigned FULL = 0xffffffffu;
  const int64_t total = g.batch * g.tpt;
  int64_t ur;
  if (probe) {
    if (blockIdx.x != 0 || r >= 32) return;
    ur = 0;  // trajectory 0, tile 0
  } else {
    const int64_t nticket = lb_ticket_count(total, g.S2);
    if (r == 0) {
      const unsigned t = atomicAdd(&w.ctr[1], 1u);
      if (t == nticket - 1) atomicExch(&w.ctr[1], 0u);
      s_ticket = (int)t;
    }
    __syncthreads();
    lb_stagger(s_ticket, g.S2, total, g.stagger2, g.stmod2);
    const int64_t u = lb_stride_map(s_ticket, total, g.S2);
    if (u >= total) return;
    ur = total - 1 - u;  // reverse order
  }
  const int64_t b = ur / g.tpt, j = ur % g.tpt;
  const int64_t tile = b * g.tpt + j;
  const int64_t G = j / kLbGroup;
  const bool last = (j == g.tpt - 1);
  const int64_t n0 = 1 + j * (int64_t)L;
  const int nvalid = (int)min((int64_t)L, g.Nn - n0);
  const R* yb = y + b * g.Nn * NY;
  LB_STAMP(1, 0);
  if (r == 0) {  // what the runs read after the look-back, into L2 now: S, the maps, v
    lb_prefetch_l2(lrt + j * (int64_t)LbRunTab<N>::F * NT + LbRunTab<N>::SP * NT,
                   (unsigned)(sizeof(R) * (NS + N * N) * NT));  // SP and PS
    lb_prefetch_l2(w.ri + (tile * (int64_t)A::SZ + N * N) * NT, (unsigned)(sizeof(R) * N * NT));
    lb_prefetch_l2(w.rcv + tile * (int64_t)N * NT, (unsigned)(sizeof(R) * N * NT));
  }
  if (!probe) YS::issue(ys, yb + n0 * NY, nvalid, r, NT);  // lands while warp 0 looks back
  if (r < 32) {
    if (lane == 0 && !probe) {  // pass-1 status of this solve (that kernel has finished): clear for the next one
      w.flag1[tile] = 0u;
      if (j % kLbGroup == 0) w.gflag1[b * g.gpt + G] = 0u;
    }
    // look-back for x at the tile's last node.  Every map already exists (pass 1 wrote
    // the tiles' and groups' offsets beta; their matrices are the plan products Qa, Qb),
    // so nothing is waited for: a published prefix only shortens the walk.
    //   x_last(j) = sum_{l < l*} Qa[j][l] beta_{j+1+l} + Qa[j][l*] x_last(j + l*)
    // over (a) the following tiles of the group (x_last(k - 1) = tile k's prefix, the last
    // tile's successor = the seed x*_T), else + Qa[j][cnt] x_end(group G) with (b)
    // x_end(G) = sum_{l < l*} Qb[G][l] beta_{G+1+l} + Qb[G][l*] x_end(group G + l*) over
    // whole groups (past the last group: the seed).  Both windows' status words are read
    // once, one fence, one round of payload loads.
    R seed[N], Phj[N][N], bej[N];  // x*_T; this tile's map (Phi_j = Qa[j-1][1], beta_j) for its prefix
#pragma unroll
    for (int i = 0; i < N; ++i) {
      seed[i] = seed_in ? seed_in[b * N + i] : w.seed[b * N + i];
      bej[i] = j > 0 ? w.agg2[tile * N + i] : R(0);
#pragma unroll
      for (int c = 0; c < N; ++c) Phj[i][c] = j > 0 ? __ldg(w.Qa + (((j - 1) * (kLbGroup + 1) + 1) * N + i) * N + c) : R(0);
    }
    R xl[N];
    if (last) {
#pragma unroll
      for (int i = 0; i < N; ++i) xl[i] = seed[i];
    } else {
      const int64_t gend = min((G + 1) * kLbGroup, g.tpt) - 1;
      const int cnt = (int)(gend - j);  // following tiles in the group
      const R* QbG = w.Qb + (G * g.gpt - G * (G - 1) / 2) * N * N;
      bool quick = false;
      if (cnt > 0) {  // the usual case (strided tickets): the next tile's prefix is x_last(j)
        unsigned s0 = 0;
        if (lane == 0) s0 = lb_ld_status(&w.flag2[b * g.tpt + j + 1]);
        s0 = __shfl_sync(FULL, s0, 0);
        if (s0 == 2u) {
          lb_fence_acquire();
#pragma unroll
          for (int i = 0; i < N; ++i) xl[i] = lb_ldcg(w.pub2 + (b * g.tpt + j + 1) * N + i);
          quick = true;
        }
      }
      if (!quick) {
      R Qa_l[N][N], Qb_l[N][N];
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int c = 0; c < N; ++c) {
          Qa_l[i][c] = __ldg(w.Qa + ((j * (kLbGroup + 1) + lane) * N + i) * N + c);
          Qb_l[i][c] = (lane < g.gpt - G) ? __ldg(QbG + (lane * N + i) * N + c) : R(0);
        }
      const int64_t ka = j + 1 + lane;
      const int64_t Gp = G + 1 + lane;
      const unsigned sta = lane < cnt ? lb_ld_status(&w.flag2[b * g.tpt + ka]) : 0u;
      // (b) status: 2 = prefix of the group's first tile, 1 = the group's map, 3 = the seed
      const unsigned stb =
          Gp < g.gpt ? (lb_ld_status(&w.flag2[b * g.tpt + Gp * kLbGroup]) == 2u ? 2u : 1u) : (Gp == g.gpt ? 3u : 0u);
      const unsigned prea = __ballot_sync(FULL, sta == 2u);
      const bool terma = !prea && gend == g.tpt - 1;  // the window reaches the last tile: the seed follows it
      const unsigned preb = (prea || terma) ? 0u : __ballot_sync(FULL, stb >= 2u);
      if (prea || preb) lb_fence_acquire();
      const int la = prea ? __ffs(prea) - 1 : cnt;
      R sa[N];
      {
        R x[N];
        const bool use = lane < la || (lane == la && (prea || terma));
#pragma unroll
        for (int i = 0; i < N; ++i)
          x[i] = !use ? R(0)
                      : (lane < la ? lb_ldcg(w.agg2 + (b * g.tpt + ka) * N + i)
                                   : (prea ? lb_ldcg(w.pub2 + (b * g.tpt + ka) * N + i) : seed[i]));
#pragma unroll
        for (int i = 0; i < N; ++i) {
          R t2 = R(0);
#pragma unroll
          for (int c = 0; c < N; ++c) t2 = fma(Qa_l[i][c], x[c], t2);
          sa[i] = t2;
        }
      }
      if (!prea && !terma) {
        R sb[N];
        const int lb = preb ? __ffs(preb) - 1 : 32;
        {
          R x[N];
          const bool use = lane < lb || (lane == lb && preb);
#pragma unroll
          for (int i = 0; i < N; ++i)
            x[i] = !use ? R(0)
                        : (stb == 3u ? seed[i]
                                     : (lane < lb ? lb_ldcg(w.gagg2 + (b * g.gpt + Gp) * N + i)
                                                  : lb_ldcg(w.pub2 + (b * g.tpt + Gp * kLbGroup) * N + i)));
#pragma unroll
          for (int i = 0; i < N; ++i) {
            R t2 = R(0);
#pragma unroll
            for (int c = 0; c < N; ++c) t2 = fma(Qb_l[i][c], x[c], t2);
            sb[i] = t2;
          }
        }
        if (!preb) {  // more than 32 groups to the nearest prefix (or the seed)
          for (int64_t l0 = 32;; l0 += 32) {
            const int64_t l = l0 + lane;
            const int64_t Gq = G + 1 + l;
            unsigned st = 0;
            if (Gq < g.gpt)
              st = lb_ld_status(&w.flag2[b * g.tpt + Gq * kLbGroup]) == 2u ? 2u : 1u;
            else if (Gq == g.gpt)
              st = 3u;
            const unsigned pre = __ballot_sync(FULL, st >= 2u);
            if (pre) lb_fence_acquire();
            const int lstar = pre ? __ffs(pre) - 1 : 32;
            if (lane <= lstar && Gq <= g.gpt) {
              R x[N], o[N];
#pragma unroll
              for (int i = 0; i < N; ++i)
                x[i] = st == 3u ? seed[i]
                                : (lane < lstar ? lb_ldcg(w.gagg2 + (b * g.gpt + Gq) * N + i)
                                                : lb_ldcg(w.pub2 + (b * g.tpt + Gq * kLbGroup) * N + i));
              lb_matvec<R, N>(QbG + l * N * N, x, o);
#pragma unroll
              for (int i = 0; i < N; ++i) sb[i] += o[i];
            }
            if (pre) break;
          }
        }
        lb_warp_sum<R, N>(sb);
        R o[N];  // + Qa[j][cnt] x_end(G): Qa[j][cnt] is lane cnt's Qa_l
#pragma unroll
        for (int i = 0; i < N; ++i) {
          R t2 = R(0);
#pragma unroll
          for (int c = 0; c < N; ++c) t2 = fma(__shfl_sync(FULL, Qa_l[i][c], cnt), sb[c], t2);
          o[i] = t2;
        }
        if (lane == 0) {
#pragma unroll
          for (int i = 0; i < N; ++i) sa[i] += o[i];
        }
      }
      lb_warp_sum<R, N>(sa);
#pragma unroll
      for (int i = 0; i < N; ++i) xl[i] = sa[i];
      }
    }
    LB_STAMP(1, 1);
    if (probe) {  // x* at node 0 = Phi_tile0 x_last(0) + beta_0
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          R a = w.agg2[tile * N + i];
#pragma unroll
          for (int c = 0; c < N; ++c) a = fma(__ldg(phit + (j * N + i) * N + c), xl[c], a);
          probe_out[b * N + i] = a;
        }
      }
      return;
    }
    if (lane == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i) s_x[i] = xl[i];
      if (j > 0) {  // prefix: x at the last node of tile j - 1 = Phi_j x_last(j) + beta_j
        lb_stress(stress, tile, 4);
#pragma unroll
        for (int i = 0; i < N; ++i) {
          R a = bej[i];
#pragma unroll
          for (int c = 0; c < N; ++c) a = fma(Phj[i][c], xl[c], a);
          w.pub2[tile * N + i] = a;
        }
        lb_st_release(&w.flag2[tile], 2u);
      }
    }
  }
  YS::wait();
  __syncthreads();
  LB_STAMP(1, 2);
  const int q = max(0, min(K, nvalid - r * K));
  bool ok = true;
  if (q > 0) {
    // x_{s-1} of the run from its suffix map; the value function entering the run (S from
    // the plan's run table, v from pass 1); then the forward sweep over the run's nodes
    RC x[N];
    {
      A inc;  // the run's in-tile suffix map: matrix from the plan (PS), offset from pass 1
      {
        const R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;
        const R* qv = w.ri + (tile * (int64_t)A::SZ + N * N) * NT + r;
#pragma unroll
        for (int i = 0; i < N; ++i) {
#pragma unroll
          for (int c = 0; c < N; ++c) inc.P[i][c] = __ldg(rt + (LbRunTab<N>::PS + i * N + c) * NT);
          inc.q[i] = qv[i * NT];
        }
      }
      R xr[N];
#pragma unroll
      for (int i = 0; i < N; ++i) xr[i] = s_x[i];
      apply(inc, xr);
#pragma unroll
      for (int i = 0; i < N; ++i) x[i] = (RC)xr[i];
    }
    VF<RC, N> cur;
    {
      const R* rt = lrt + j * (int64_t)LbRunTab<N>::F * NT + r;
#pragma unroll
      for (int k = 0; k < NS; ++k) cur.S[k] = (RC)__ldg(rt + (LbRunTab<N>::SP + k) * NT);
#pragma unroll
      for (int i = 0; i < N; ++i) cur.v[i] = (RC)w.rcv[(tile * N + i) * NT + r];
    }
    R* xo = x_out + b * g.Nn * N;
    const int64_t s0 = n0 + (int64_t)r * K;
    R Ps[OUT == 2 ? NS : 1];  // smoother covariance at the current node
    if constexpr (OUT == 2) {
#pragma unroll
      for (int k = 0; k < NS; ++k) Ps[k] = __ldg(lcov + (j * NS + k) * NT + r);
    }
    auto store_x = [&](R* dst) {
      if constexpr (MIXED) {
        R xr[N];
#pragma unroll
        for (int i = 0; i < N; ++i) xr[i] = (R)x[i];
        lb_store_x<R, N>(dst, xr);
      } else {
        lb_store_x<R, N>(dst, x);
      }
    };
    if (s0 == 1 && store0) {  // node 0 (the carry-in of the first tile; a later shard's belongs to the rank before)
      store_x(xo);
      if constexpr (OUT == 2) {
#pragma unroll
        for (int k = 0; k < NS; ++k) fP[(b * g.Nn) * NS + k] = Ps[k];
      }
      if constexpr (FO) {
        R m[N];
        spd_solve<R, N>(cur.S, cur.v, m, ok);
        R P[NS];
        spd_inverse<R, N>(cur.S, P, ok);
#pragma unroll
        for (int i = 0; i < N; ++i)
          if (fm) fm[(b * g.Nn) * N + i] = m[i];  // either filter output may be absent
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (fP) fP[(b * g.Nn) * NS + k] = P[k];
      }
    }
    const R* yr = ys + r * YS::ROW;
#pragma unroll 1
    for (int m = 0; m < q; ++m) {
      Elem<RC, N> e;
      if constexpr (MIXED) {
        RC yc[NY];
#pragma unroll
        for (int k = 0; k < NY; ++k) yc[k] = (RC)yr[m * NY + k];
        src.node_interior(s0 + m, yc, nullptr, e);
      } else {
        src.node_interior(s0 + m, yr + m * NY, nullptr, e);
      }
      if constexpr (OUT == 2) {
        lb_cov_step<R, N, SrcC>(src, cur.S, Ps);  // with S_{i-1}, before the node update
#pragma unroll
        for (int k = 0; k < NS; ++k) fP[(b * g.Nn + s0 + m) * NS + k] = Ps[k];
      }
      lb_node_step<RC, N, SrcC>(src, e, cur, x, ok);
      store_x(xo + (s0 + m) * N);
      if constexpr (FO) {
        R mm[N];
        spd_solve<R, N>(cur.S, cur.v, mm, ok);
        R P[NS];
        spd_inverse<R, N>(cur.S, P, ok);
        const int64_t idx = b * g.Nn + s0 + m;
#pragma unroll
        for (int i = 0; i < N; ++i)
          if (fm) fm[idx * N + i] = mm[i];
#pragma unroll
        for (int k = 0; k < NS; ++k)
          if (fP) fP[idx * NS + k] = P[k];
      }
    }
    RC s = RC(0);
#pragma unroll
    for (int i = 0; i < N; ++i) s += x[i];
    if (!(s - s == RC(0))) ok = false;
  }
  if (!ok) atomicMin(flag, (unsigned long long)(n0 + (int64_t)r * K));
  LB_STAMP(1, 3);
}

}  // namespace pmap
