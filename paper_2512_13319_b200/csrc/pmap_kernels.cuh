// pmap_kernels.cuh -- the scan kernels of the parallel MAP solve (arXiv 2512.13319).
//
// Tiling: a trajectory of Nn local nodes is cut into tiles of NT runs x K nodes.
// Thread r of a tile owns the contiguous run of K nodes [l0, l0 + K).  Nothing is
// reversed in memory: the suffix-in-tau scan of P:249-258 / P:333-336 is a prefix
// scan in node (time) order with the flipped operator acc_i = E_i (x) acc_{i-1}
// (R-FLIP), and the forward-in-tau recovery scan of P:348-353 / P:448-459 is a
// suffix scan in node order.
//
//   pass 1 (value functions, P:323-341 / P:382-409)
//     k_p1_reduce  per run: serial fold of node elements (fused element build);
//                  per tile: Kogge-Stone inclusive scan of the run aggregates
//     k_p1_tiles   per group of NT2 tiles: inclusive scan of tile aggregates
//     k_p1_groups  per trajectory: value-function carries of every group
//     k_p1_down    per run: carry -> (S_i, v_i) at every node (vapply), fused with
//                  the pass-2 transition build and the per-run affine fold, plus
//                  the per-tile suffix scan of the affine run aggregates
//   pass 2 (trajectory)
//     k_p2_tiles   per group of NT2 tiles: suffix composition of tile aggregates
//     k_p2_groups  per trajectory: x* at each group's last node (seeded with
//                  x*_T = S_T^-1 v_T)
//     k_p2_down    per run: x*_{i-1} = (I + C_i S_{i-1})^-1 (A_i x*_i + b_i + C_i v_{i-1})
// Workspace layouts are SoA "field-major" so that a warp touches consecutive
// addresses.
#pragma once
#include "pmap_sources.cuh"

namespace pmap {

struct Geom {
  int64_t Nn;     // local nodes per trajectory (this launch)
  int64_t node0;  // global index of local node 0 (time shard offset)
  int64_t tpt;    // tiles per trajectory
  int64_t gpt;    // tile groups per trajectory
  int64_t batch;
};

#ifndef PM_DOWN_UNROLL
#define PM_DOWN_UNROLL 1
#endif
constexpr int kDownUnroll = PM_DOWN_UNROLL;  // node-loop unroll of k_p1_down
constexpr int NT2 = 128;  // tiles per group (k_p1_tiles block size)
constexpr int NT3 = 128;  // k_p1_groups block size
constexpr int NT4 = 256;  // k_p2_groups block size

PM_INLINE void flag_node(unsigned long long* flag, int64_t node) {
  atomicMin(flag, (unsigned long long)node);
}

template <typename R, int N>
PM_INLINE bool finite_vf(const VF<R, N>& V) {
  R s = R(0);
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) s += V.S[k];
#pragma unroll
  for (int i = 0; i < N; ++i) s += V.v[i];
  return s - s == R(0);
}

// Inclusive run prefix r of a tile (row pointer already offset by the run): on LTI
// interior tiles the reduce stores only its data parts and the matrix parts come from
// the plan table (sf = SF + run, field-major over A, C, J), else the full element.
template <typename R, int N, int NT>
PM_INLINE void load_prefix(Elem<R, N>& p, const R* __restrict__ row, const R* __restrict__ sf) {
  if (sf) {
    int f = 0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) p.A[i][j] = __ldg(sf + (f++) * NT);
#pragma unroll
    for (int k = 0; k < Dim<N>::NS; ++k) p.C[k] = __ldg(sf + (f++) * NT);
#pragma unroll
    for (int k = 0; k < Dim<N>::NS; ++k) p.J[k] = __ldg(sf + (f++) * NT);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      p.b[i] = row[(N * N + i) * NT];
      p.h[i] = row[(N * N + N + Dim<N>::NS + i) * NT];
    }
  } else {
    load(p, row, NT);
  }
}

// Inclusive scan over the NT runs of a tile, data parts (b, eta) only (R-LTI): warp-
// synchronous Kogge-Stone with shuffles and the compact coefficient tables (UWc: lanes
// d..2d-2 read consecutive slots, the rest one broadcast slot), then one cross-warp step
// with warp 0's total (UX).  Thread r holds its run's aggregate on entry, the inclusive
// prefix of runs 0..r on exit.
template <typename R, int N, int NT>
PM_INLINE void lti_run_scan(const R* __restrict__ UWc, const R* __restrict__ UX, int r, R (&bb)[N], R (&hh)[N]) {
  static_assert(NT == 32 || NT == 64, "tile of one or two warps");
  const int lane = r & 31;
  const unsigned FULL = 0xffffffffu;
  auto step = [&](const R* __restrict__ U, int stride, int slot, const R (&b2)[N], const R (&h2)[N]) {
    // U = [4][N][N][stride] (slot-indexed): b = U1 b1 + U2 eta2 + b2 ; eta = U3 eta2 - U4 b1 + eta1
    R nb[N], nh[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      // two independent accumulators per output (halves the dependent FMA chain)
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
  if (NT == 64) {
    __shared__ R tot[2 * N];
    if (r == 31) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        tot[i] = bb[i];
        tot[N + i] = hh[i];
      }
    }
    __syncthreads();
    if (r >= 32) {
      R b2[N], h2[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        b2[i] = tot[i];
        h2[i] = tot[N + i];
      }
      step(UX, 32, lane, b2, h2);
    }
  }
}

// ----------------------------------------------------------------- pass 1a
// nsel > 0: only the listed tiles {jsel0, jsel1} of each trajectory (the boundary
// tiles left over by the LTI-specialised reduce), else every tile.
template <typename R, int N, int NY, int NT, int K, class Src, bool REV>
__global__ void __launch_bounds__(NT) k_p1_reduce(const __grid_constant__ Src src, const Geom g,
                                                  const R* __restrict__ y, const R* __restrict__ xbar,
                                                  R* __restrict__ run_incl, R* __restrict__ tile_agg,
                                                  unsigned long long* flag, int nsel, int64_t jsel0, int64_t jsel1) {
  using E = Elem<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);  // [E::SZ][NT]
  int64_t b, j;
  if (nsel > 0) {
    b = blockIdx.x / nsel;
    j = (blockIdx.x % nsel == 0) ? jsel0 : jsel1;
  } else {
    b = blockIdx.x / g.tpt;
    j = blockIdx.x % g.tpt;
  }
  const int64_t tile = b * g.tpt + j;
  const int r = threadIdx.x;
  const int64_t l0 = (j * NT + r) * (int64_t)K;
  const R* yb = y + b * g.Nn * NY;
  const R* xb = Src::NEEDS_XBAR ? xbar + b * g.Nn * N : nullptr;
  bool ok = true;
  E acc, acc_x0;  // acc_x0: the run's fold without global node 0 (pass-2 aggregate of that run)
  set_identity(acc);
  set_identity(acc_x0);
  const bool has_node0 = !REV && (g.node0 + l0 == 0);
#pragma unroll 1
  for (int m = 0; m < K; ++m) {
    const int64_t lr = l0 + m;
    if (lr >= g.Nn) break;
    const int64_t l = REV ? g.Nn - 1 - lr : lr;  // REV: suffix scan (two-filter pass B)
    E e;
    src.node(g.node0 + l, yb + l * NY, Src::NEEDS_XBAR ? xb + l * N : nullptr, e);
    if (m == 0) {
      acc = e;
    } else if constexpr (N >= 5) {
      // acc = E_l (x) acc (R-FLIP) with the right operand read in place from this thread's
      // shared-memory slot: two register-resident nx = 5 elements spill at 255 registers
      store(acc, sh + r, NT);
      combine_g(e, ElemRef<R, N>{sh + r, NT}, acc, ok);
    } else {
      combine(e, acc, acc, ok);  // acc = E_l (x) acc   (R-FLIP)
    }
    if (has_node0 && m >= 1) {
      if (m == 1)
        acc_x0 = e;
      else
        combine(e, acc_x0, acc_x0, ok);
    }
  }
  // the run's own aggregate (pass 2 derives its transition from it, R-RUNAGG)
  store(has_node0 ? acc_x0 : acc, run_incl + (g.batch * g.tpt + tile) * (int64_t)E::SZ * NT + r, NT);
  // inclusive Kogge-Stone scan over the runs of the tile: In_r = In_r (x) In_{r-d}
  // (the partner read in place from its shared-memory slot, combine_g)
  __syncthreads();
#pragma unroll 1
  for (int d = 1; d < NT; d <<= 1) {
    store(acc, sh + r, NT);
    __syncthreads();
    if (r >= d) combine_g(acc, ElemRef<R, N>{sh + r - d, NT}, acc, ok);
    __syncthreads();
  }
  store(acc, run_incl + tile * (int64_t)E::SZ * NT + r, NT);
  if (r == NT - 1) store(acc, tile_agg + tile * (int64_t)E::SZ, 1);
  if (!ok) flag_node(flag, g.node0 + l0);
}

// ----------------------------------------------------------------- pass 1b
// Inclusive scan of tile aggregates within groups of NT2 tiles.
template <typename R, int N>
__global__ void __launch_bounds__(NT2) k_p1_tiles(const Geom g, const R* __restrict__ tile_agg,
                                                  R* __restrict__ tile_incl, R* __restrict__ group_agg,
                                                  unsigned long long* flag) {
  using E = Elem<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);
  const int64_t grp = blockIdx.x;
  const int64_t b = grp / g.gpt, gg = grp % g.gpt;
  const int t = threadIdx.x;
  const int64_t jt = gg * NT2 + t;
  const bool valid = jt < g.tpt;
  const int cnt = (int)min((int64_t)NT2, g.tpt - gg * NT2);  // valid tiles in this group
  bool ok = true;
  E acc;
  if (valid)
    load(acc, tile_agg + (b * g.tpt + jt) * E::SZ, 1);
  else
    set_identity(acc);
#pragma unroll 1
  for (int d = 1; d < cnt; d <<= 1) {
    store(acc, sh + t, NT2);
    __syncthreads();
    if (t >= d) combine_g(acc, ElemRef<R, N>{sh + t - d, NT2}, acc, ok);  // partner read in place
    __syncthreads();
  }
  if (valid) store(acc, tile_incl + (b * g.tpt + jt) * E::SZ, 1);
  if (t == cnt - 1) store(acc, group_agg + grp * E::SZ, 1);
  if (!ok) flag_node(flag, g.node0 + jt);
}

// ----------------------------------------------------------------- pass 1c
// Value-function carry entering every group: carry_g = GroupExcl_g (.) carry_in,
// carry_in = the trajectory's incoming value function ((0,0) on rank 0).  Time shards
// (gathered != nullptr): thread 0 first folds the gathered chunk
// aggregates of the ranks before this one, carry_in = Agg_{r-1} (x) ... (x) Agg_0 (.) (0, 0),
// and stores it to carry_out (read by k_p2_down at the rank's first node).
template <typename R, int N>
__global__ void __launch_bounds__(NT3) k_p1_groups(const Geom g, const R* __restrict__ group_agg,
                                                   const R* __restrict__ gathered, int rank,
                                                   R* __restrict__ carry_out, R* __restrict__ group_carry,
                                                   R* __restrict__ total_agg, unsigned long long* flag) {
  using E = Elem<R, N>;
  using V = VF<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t c = (g.gpt + NT3 - 1) / NT3;
  const int64_t k0 = t * c, k1 = min(g.gpt, k0 + c);
  const int nact = (int)((g.gpt + c - 1) / c);  // threads holding groups
  bool ok = true;
  E acc;
  set_identity(acc);
  for (int64_t k = k0; k < k1; ++k) {
    E p;
    load(p, group_agg + (b * g.gpt + k) * E::SZ, 1);
    if (k == k0)
      acc = p;
    else
      combine(p, acc, acc, ok);
  }
#pragma unroll 1
  for (int d = 1; d < nact; d <<= 1) {
    store(acc, sh + t, NT3);
    __syncthreads();
    if (t >= d) combine_g(acc, ElemRef<R, N>{sh + t - d, NT3}, acc, ok);  // partner read in place
    __syncthreads();
  }
  store(acc, sh + t, NT3);
  __shared__ R shc[V::SZ];
  if (t == 0) {
    V c0;
    set_zero(c0);
    if (gathered) {
      for (int q = 0; q < rank; ++q) {
        E a;
        load(a, gathered + ((int64_t)q * g.batch + b) * E::SZ, 1);
        vapply<R, N, false>(a, c0, c0, nullptr, ok);
      }
      store(c0, carry_out + b * V::SZ, 1);
    }
    store(c0, shc, 1);
  }
  __syncthreads();
  V cin;
  load(cin, shc, 1);
  if (t == nact - 1 && total_agg) store(acc, total_agg + b * E::SZ, 1);
  V cur = cin;
  if (t > 0) {
    E p;
    load(p, sh + t - 1, NT3);
    vapply<R, N, false>(p, cin, cur, nullptr, ok);
  }
  for (int64_t k = k0; k < k1; ++k) {
    store(cur, group_carry + (b * g.gpt + k) * V::SZ, 1);
    if (k + 1 < k1) {
      E p;
      load(p, group_agg + (b * g.gpt + k) * E::SZ, 1);
      vapply<R, N, false>(p, cur, cur, nullptr, ok);
    }
  }
  if (!ok) flag_node(flag, g.node0);
}

// Value function entering run r of a tile: cur (the tile carry) advanced over runs
// 0..r-1.  LTI interior tiles (uwc != nullptr): the exclusive run prefix is scanned here
// from the stored run aggregates, data parts only (lti_run_scan; matrix parts from the
// plan table sf); otherwise the reduce stored the inclusive prefixes (load_prefix).
template <typename R, int N, int NT>
PM_INLINE void run_carry(const R* __restrict__ run_incl, const Geom& g, int64_t tile, int r, bool interior,
                         const R* __restrict__ sf, const R* __restrict__ uwc, const R* __restrict__ ux,
                         VF<R, N>& cur, bool& ok) {
  using E = Elem<R, N>;
#ifdef PM_REDUCE_TREE
  if (interior && uwc) {  // block-uniform
    const R* pa = run_incl + (g.batch * g.tpt + tile) * (int64_t)E::SZ * NT + r;  // run aggregates
    R bb[N], hh[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      bb[i] = pa[(N * N + i) * NT];
      hh[i] = pa[(N * N + N + Dim<N>::NS + i) * NT];
    }
    lti_run_scan<R, N, NT>(uwc, ux, r, bb, hh);
    // exclusive prefix of run r = inclusive prefix of run r - 1
    __shared__ R x31[2 * N];
    if (r == 31) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        x31[i] = bb[i];
        x31[N + i] = hh[i];
      }
    }
    R pb[N], ph[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      pb[i] = __shfl_up_sync(0xffffffffu, bb[i], 1);
      ph[i] = __shfl_up_sync(0xffffffffu, hh[i], 1);
    }
    __syncthreads();
    if (r == 32) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        pb[i] = x31[i];
        ph[i] = x31[N + i];
      }
    }
    if (r > 0) {
      E p;
      const R* sfr = sf + (r - 1);
      int f = 0;
#pragma unroll
      for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < N; ++j) p.A[i][j] = __ldg(sfr + (f++) * NT);
#pragma unroll
      for (int k = 0; k < Dim<N>::NS; ++k) p.C[k] = __ldg(sfr + (f++) * NT);
#pragma unroll
      for (int k = 0; k < Dim<N>::NS; ++k) p.J[k] = __ldg(sfr + (f++) * NT);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        p.b[i] = pb[i];
        p.h[i] = ph[i];
      }
      vapply<R, N, false>(p, cur, cur, nullptr, ok);
    }
    return;
  }
#else
  (void)uwc;
  (void)ux;
#endif
  if (r > 0) {
    E p;
    load_prefix<R, N, NT>(p, run_incl + tile * (int64_t)E::SZ * NT + (r - 1), interior ? sf + (r - 1) : nullptr);
    vapply<R, N, false>(p, cur, cur, nullptr, ok);
  }
}

// ----------------------------------------------------------------- pass 1d
// 6 resident 64-thread CTAs per SM for nx <= 4 (<= 168 registers: measured 10 %
// faster than the unconstrained 186-register build at nx = 4); nx = 5 unconstrained.
#ifdef PM_DOWN_MINB
#define PM_DOWN_LB(NT) __launch_bounds__(NT, PM_DOWN_MINB)
#else
#define PM_DOWN_LB(NT) __launch_bounds__(NT, (N <= 4 ? 6 : 1))
#endif
// REC (low-rank sources only, R-P2REC): instead of (S_i, v_i) store at node i the
// pass-2 record [S_{i-1} U | U^T v_{i-1}] of the value function the node consumes
// (N*NW + NW values instead of N(N+1)/2 + N); (S, v) of the last node always goes to svl.
template <typename R, int N, int NY, int NT, int K, class Src, bool P2, bool REC = false>
__global__ void PM_DOWN_LB(NT) k_p1_down(const __grid_constant__ Src src, const Geom g,
                                                const R* __restrict__ y, const R* __restrict__ xbar,
                                                const R* __restrict__ run_incl, const R* __restrict__ tile_incl,
                                                const R* __restrict__ group_carry, R* __restrict__ sv,
                                                R* __restrict__ run_suf, R* __restrict__ tile_agg2,
                                                unsigned long long* flag, const R* __restrict__ span1,
                                                const R* __restrict__ sf, int64_t j_lo, int64_t j_hi,
                                                R* __restrict__ svl, const R* __restrict__ uwc = nullptr,
                                                const R* __restrict__ ux = nullptr) {
  static_assert(!REC || Src::LOWRANK > 0, "pass-2 records need a low-rank source");
  using E = Elem<R, N>;
  using V = VF<R, N>;
  using A = Aff<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);  // [A::SZ][NT] (reused for the tile carry)
  const int64_t tile = blockIdx.x;
  const int64_t b = tile / g.tpt, j = tile % g.tpt;
  const int r = threadIdx.x;
  const int64_t l0 = (j * NT + r) * (int64_t)K;
  const R* yb = y + b * g.Nn * NY;
  const R* xb = Src::NEEDS_XBAR ? xbar + b * g.Nn * N : nullptr;
  bool ok = true;
  // tile carry
  if (r == 0) {
    const int64_t gg = j / NT2, lj = j % NT2;
    V c;
    load(c, group_carry + (b * g.gpt + gg) * V::SZ, 1);
    if (lj > 0) {
      E p;
      load(p, tile_incl + (b * g.tpt + j - 1) * E::SZ, 1);
      vapply<R, N, false>(p, c, c, nullptr, ok);
    }
    store(c, sh, 1);
  }
  __syncthreads();
  V cur;
  load(cur, sh, 1);
  __syncthreads();
  const bool interior = sf && j >= j_lo && j < j_hi;
  run_carry<R, N, NT>(run_incl, g, tile, r, interior, sf, uwc, ux, cur, ok);
  // Pass-2 aggregate of the run (maps x*_e -> x*_{s-1}), R-RUNAGG: by dynamic
  // programming it is the argmin of V_{s-1}(x) + R(x_e; x) over x for the run's own
  // aggregate element R, i.e. the transition of vapply(R, V_{s-1}) -- one solve per
  // run instead of one affine composition per node.  The run holding global node 0
  // (no transition into it) composes per node instead.
  const bool node0_run = (g.node0 + l0 == 0);
  if (P2) {
    A agg;
    E ra;
    const R* pa = run_incl + (g.batch * g.tpt + tile) * (int64_t)E::SZ * NT + r;
    if (span1 && j >= j_lo && j < j_hi) {
      // LTI interior tile: matrix parts of one full run from the plan table, data parts stored
      load(ra, span1, 1);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        ra.b[i] = pa[(N * N + i) * NT];
        ra.h[i] = pa[(N * N + N + Dim<N>::NS + i) * NT];
      }
    } else {
      load(ra, pa, NT);  // (the run holding node 0 stores its fold without node 0)
    }
    V vin = cur;
    if (node0_run) {  // no transition into node 0: the DP starts from V_0 = E_0 (.) (0, 0)
      E e0;
      src.node(0, yb, Src::NEEDS_XBAR ? xb : nullptr, e0);
#pragma unroll
      for (int k = 0; k < Dim<N>::NS; ++k) vin.S[k] = e0.J[k];
#pragma unroll
      for (int i = 0; i < N; ++i) vin.v[i] = e0.h[i];
    }
    V vend;
    vapply<R, N, true>(ra, vin, vend, &agg, ok);
    store(agg, sh + r, NT);  // parked in shared memory across the node loop
  }
  R* svt = sv + tile * (int64_t)V::SZ * K * NT;
  // measurements prefetched two nodes ahead with cp.async (LDGSTS) into a per-thread
  // ring in shared memory: consecutive threads own runs K nodes apart, so a y row is one
  // half-used sector per thread and mostly misses L1; an asynchronous copy keeps the
  // latency off the recursion without a register dependency
  constexpr int YB = NY * (int)sizeof(R);
  constexpr bool kPF = (YB == 4 || YB == 8 || YB == 16);
  __shared__ __align__(16) R yring[kPF ? NT : 1][4][kPF ? NY : 1];
  auto ypf = [&](int m) {  // issue the copy of node l0 + m into slot m & 3 (one commit group)
    if constexpr (kPF) {
      if (m < K && l0 + m < g.Nn) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(&yring[r][m & 3][0]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(dst), "l"(yb + (l0 + m) * NY), "n"(YB));
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
  };
  ypf(0);
  ypf(1);
#pragma unroll kDownUnroll
  for (int m = 0; m < K; ++m) {
    const int64_t l = l0 + m;
    if (l >= g.Nn) break;
    const int64_t gi = g.node0 + l;
    const R* yrow = yb + l * NY;
    if constexpr (kPF) {
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // node m's copy has landed
      yrow = &yring[r][m & 3][0];
      ypf(m + 2);
    }
    E e;
    if (gi == 0) {
      src.node(gi, yrow, Src::NEEDS_XBAR ? xb + l * N : nullptr, e);
#pragma unroll
      for (int k = 0; k < Dim<N>::NS; ++k) cur.S[k] = e.J[k];
#pragma unroll
      for (int i = 0; i < N; ++i) cur.v[i] = e.h[i];
    } else {
      src.node_interior(gi, yrow, Src::NEEDS_XBAR ? xb + l * N : nullptr, e);
      if constexpr (Src::LOWRANK > 0)
        vapply_lowrank<R, N, Src::LOWRANK, Src::AMASK, Src::UMASK>(e, src.U, cur, cur, ok, REC ? svt + m * NT + r : nullptr,
                                           (int64_t)K * NT, src.zero_b != 0);
      else
        vapply<R, N, false>(e, cur, cur, nullptr, ok);
    }
    if (!REC) store(cur, svt + m * NT + r, (int64_t)K * NT);
    if (l == g.Nn - 1 && svl) store(cur, svl + b * V::SZ, 1);
  }
  if constexpr (kPF) asm volatile("cp.async.wait_all;\n" ::: "memory");
  if (!finite_vf(cur)) ok = false;
  if (!P2) {
    if (!ok) flag_node(flag, g.node0 + l0);
    return;
  }
  // exclusive suffix scan of the run aggregates within the tile
  A agg;
  load(agg, sh + r, NT);
  __syncthreads();
#pragma unroll 1
  for (int d = 1; d < NT; d <<= 1) {
    store(agg, sh + r, NT);
    __syncthreads();
    if (r + d < NT) {
      A p;
      load(p, sh + r + d, NT);
      compose(agg, p, agg);
    }
    __syncthreads();
  }
  store(agg, sh + r, NT);
  __syncthreads();
  A ex;
  if (r + 1 < NT)
    load(ex, sh + r + 1, NT);
  else
    set_identity(ex);
  store(ex, run_suf + tile * (int64_t)A::SZ * NT + r, NT);
  if (r == 0) store(agg, tile_agg2 + tile * (int64_t)A::SZ, 1);
  if (!ok) flag_node(flag, g.node0 + l0);
}

// (S, v) of local node l of trajectory b in the tiled SoA layout
template <typename R, int N, int NT, int K>
PM_INLINE void load_sv(const R* sv, const Geom& g, int64_t b, int64_t l, VF<R, N>& V) {
  const int64_t L = (int64_t)NT * K;
  const int64_t j = l / L, q = l % L;
  const int64_t rr = q / K, m = q % K;
  load(V, sv + (b * g.tpt + j) * (int64_t)VF<R, N>::SZ * K * NT + m * NT + rr, (int64_t)K * NT);
}

// ----------------------------------------------------------------- pass 2a
// Exclusive suffix composition of tile affine aggregates within groups of NT2 tiles.
template <typename R, int N>
__global__ void __launch_bounds__(NT2) k_p2_tiles(const Geom g, const R* __restrict__ tile_agg2,
                                                  R* __restrict__ tile_sufx, R* __restrict__ group_agg2) {
  using A = Aff<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);  // [A::SZ][NT2]
  const int64_t grp = blockIdx.x;
  const int64_t b = grp / g.gpt, gg = grp % g.gpt;
  const int t = threadIdx.x;
  const int64_t jt = gg * NT2 + t;
  const bool valid = jt < g.tpt;
  const int cnt = (int)min((int64_t)NT2, g.tpt - gg * NT2);
  A acc;
  if (valid)
    load(acc, tile_agg2 + (b * g.tpt + jt) * A::SZ, 1);
  else
    set_identity(acc);
#pragma unroll 1
  for (int d = 1; d < cnt; d <<= 1) {
    store(acc, sh + t, NT2);
    __syncthreads();
    if (t + d < NT2) {
      A p;
      load(p, sh + t + d, NT2);
      compose(acc, p, acc);
    }
    __syncthreads();
  }
  store(acc, sh + t, NT2);
  __syncthreads();
  if (valid) {
    A ex;
    if (t + 1 < NT2)
      load(ex, sh + t + 1, NT2);
    else
      set_identity(ex);
    store(ex, tile_sufx + (b * g.tpt + jt) * A::SZ, 1);
  }
  if (t == 0) store(acc, group_agg2 + grp * A::SZ, 1);
}

// x* at the last node of every tile group (exclusive suffix over group aggregates,
// seeded with x_end = S_T^-1 v_T on the rank holding node T, or the shard carry).
// Time shards: payload != nullptr (phase 2) -> thread 0 writes
// this rank's chunk affine aggregate (+ x*_T = S_T^-1 v_T on the last rank) to payload;
// gathered != nullptr (phase 3) -> x at the rank's last node is
// Agg_{r+1} o ... o Agg_{G-1} (x*_T) from the gathered payloads.
template <typename R, int N, int NT, int K>
__global__ void __launch_bounds__(NT4) k_p2_groups(const Geom g, const R* __restrict__ svl,
                                                   const R* __restrict__ group_agg2, const R* __restrict__ gathered,
                                                   int rank, int world, R* __restrict__ group_carry,
                                                   R* __restrict__ payload, unsigned long long* flag) {
  using A = Aff<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);  // [A::SZ][NT4] + N
  R* shx = sh + A::SZ * NT4;
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  bool ok = true;
  if (t == 0) {
    R x[N];
    if (gathered) {
      const int64_t PS = A::SZ + N;
#pragma unroll
      for (int i = 0; i < N; ++i) x[i] = gathered[((int64_t)(world - 1) * g.batch + b) * PS + A::SZ + i];
      for (int q = world - 1; q > rank; --q) {
        A a;
        load(a, gathered + ((int64_t)q * g.batch + b) * PS, 1);
        apply(a, x);
      }
    } else {
      VF<R, N> V;
      load(V, svl + b * VF<R, N>::SZ, 1);
      spd_solve<R, N>(V.S, V.v, x, ok);  // x*_T = S_T^-1 v_T
    }
#pragma unroll
    for (int i = 0; i < N; ++i) shx[i] = x[i];
  }
  const int64_t c = (g.gpt + NT4 - 1) / NT4;
  const int64_t k0 = t * c, k1 = min(g.gpt, k0 + c);
  const int nact = (int)((g.gpt + c - 1) / c);
  A acc;
  set_identity(acc);
  for (int64_t k = k1 - 1; k >= k0; --k) {
    A p;
    load(p, group_agg2 + (b * g.gpt + k) * A::SZ, 1);
    compose(p, acc, acc);
  }
#pragma unroll 1
  for (int d = 1; d < nact; d <<= 1) {
    store(acc, sh + t, NT4);
    __syncthreads();
    if (t + d < NT4) {
      A p;
      load(p, sh + t + d, NT4);
      compose(acc, p, acc);
    }
    __syncthreads();
  }
  store(acc, sh + t, NT4);
  __syncthreads();
  if (t == 0 && payload) {
    R* pp = payload + b * (A::SZ + N);
    store(acc, pp, 1);
    if (rank == world - 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) pp[A::SZ + i] = shx[i];
    }
  }
  R x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = shx[i];
  if (t + 1 < NT4) {
    A p;
    load(p, sh + t + 1, NT4);
    apply(p, x);
  }
  for (int64_t k = k1 - 1; k >= k0; --k) {
#pragma unroll
    for (int i = 0; i < N; ++i) group_carry[(b * g.gpt + k) * N + i] = x[i];
    A p;
    load(p, group_agg2 + (b * g.gpt + k) * A::SZ, 1);
    apply(p, x);
  }
  if (!ok) flag_node(flag, g.node0 + g.Nn - 1);
}

// ----------------------------------------------------------------- pass 2b
// Backward sweep of each run.  (S, v) of the next node is prefetched one step
// ahead (coalesced SoA loads), and x is staged through shared memory in chunks of
// KC nodes so that it leaves as contiguous 8*KC*N-byte segments per run.
template <typename R, int N, int NT, int K, class Src, bool REC = false>
__global__ void __launch_bounds__(NT) k_p2_down(const __grid_constant__ Src src, const Geom g,
                                                const R* __restrict__ y, const R* __restrict__ xbar,
                                                const R* __restrict__ sv,
                                                const R* __restrict__ run_suf, const R* __restrict__ tile_sufx,
                                                const R* __restrict__ group_carry, const R* __restrict__ carry_in,
                                                R* __restrict__ x_out, unsigned long long* flag) {
  using V = VF<R, N>;
  using A = Aff<R, N>;
  constexpr int KC = K < 8 ? K : 8;  // nodes per staged chunk
  static_assert(K % KC == 0, "chunking");
  __shared__ R xs[NT][KC * N + 1];
  const int64_t tile = blockIdx.x;
  const int64_t b = tile / g.tpt, j = tile % g.tpt;
  const int r = threadIdx.x;
  const int64_t l0 = (j * NT + r) * (int64_t)K;
  const R* xb = Src::NEEDS_XBAR ? xbar + b * g.Nn * N : nullptr;
  const R* yb = Src::TRANS_Y ? y + b * g.Nn * Src::NYROW : nullptr;
  bool ok = true;
  R x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = group_carry[(b * g.gpt + j / NT2) * N + i];
  {
    A s;
    load(s, tile_sufx + tile * (int64_t)A::SZ, 1);  // x at the tile's last node
    apply(s, x);
    load(s, run_suf + tile * (int64_t)A::SZ * NT + r, NT);  // x at the run's last node
    apply(s, x);
  }
  R* xo = x_out + b * g.Nn * N;
  const R* svt = sv + tile * (int64_t)V::SZ * K * NT;
  if constexpr (REC) {
    // pass-2 records (R-P2REC): the record of step m sits in the run's own slot m
    constexpr int NW = Src::LOWRANK > 0 ? Src::LOWRANK : 1;
    constexpr bool CR = CompactRec<N, NW, Src::UMASK>::value;
    constexpr int RS = CR ? CompactRec<N, NW, Src::UMASK>::SIZE : N * NW + NW;
    R rn[RS], rn2[RS];  // records of the next two steps (two nodes of loads in flight)
    auto fetch_rec = [&](int m, R (&rr)[RS]) {
#pragma unroll
      for (int f = 0; f < RS; ++f) rr[f] = svt[(int64_t)f * K * NT + m * NT + r];
    };
    fetch_rec(K - 1, rn);
    fetch_rec(K - 2, rn2);
#pragma unroll 1
    for (int c = K / KC - 1; c >= 0; --c) {
#pragma unroll 1
      for (int mm = KC - 1; mm >= 0; --mm) {
        const int m = c * KC + mm;
        const int64_t l = l0 + m;
        const bool valid = l < g.Nn;
        R rc[RS];
#pragma unroll
        for (int f = 0; f < RS; ++f) {
          rc[f] = rn[f];
          rn[f] = rn2[f];
        }
        if (m > 1) fetch_rec(m - 2, rn2);
#pragma unroll
        for (int i = 0; i < N; ++i) xs[r][mm * N + i] = x[i];
        const int64_t gi = g.node0 + l;
        if (valid && gi != 0) {
          R At[N][N], bt[N], Ct[Dim<N>::NS], SU[N][NW], u[NW];
          src.trans(gi, nullptr, nullptr, At, bt, Ct);
          if constexpr (CR) {  // columns 2, 3 of S and v2, v3 (CompactRec)
            const R c0 = src.U[N > 2 ? 2 : 0][0], c1 = src.U[N > 3 ? 3 : 0][NW > 1 ? 1 : 0];
            const R s2[4] = {rc[0], rc[1], rc[2], rc[5]}, s3[4] = {rc[3], rc[4], rc[5], rc[6]};
#pragma unroll
            for (int i = 0; i < N; ++i) {
              SU[i][0] = s2[i < 4 ? i : 0] * c0;
              SU[i][NW > 1 ? 1 : 0] = s3[i < 4 ? i : 0] * c1;
            }
            u[0] = c0 * rc[7];
            u[NW > 1 ? 1 : 0] = c1 * rc[8 < RS ? 8 : 0];
          } else {
#pragma unroll
            for (int i = 0; i < N; ++i)
#pragma unroll
              for (int a = 0; a < NW; ++a) SU[i][a] = rc[i * NW + a];
#pragma unroll
            for (int a = 0; a < NW; ++a) u[a] = rc[N * NW + a];
          }
          trans_step_rec<R, N, NW, Src::AMASK, Src::UMASK>(At, bt, src.U, SU, u, x, ok);
        }
      }
      __syncthreads();
      for (int rr = r >> 5; rr < NT; rr += NT / 32) {
        const int64_t lb = (j * NT + rr) * (int64_t)K + c * KC;
        for (int q = r & 31; q < KC * N; q += 32) {
          const int64_t node = lb + q / N;
          if (node < g.Nn) xo[lb * N + q] = xs[rr][q];
        }
      }
      __syncthreads();
    }
  } else {
  // (S, v) of node l-1 for step m (m >= 1: same run, SoA slot m-1)
  auto fetch = [&](int m, V& Vp) {
    const int64_t l = l0 + m;
    if (m >= 1) {
      load(Vp, svt + (m - 1) * NT + r, (int64_t)K * NT);
    } else if (l > 0) {
      load_sv<R, N, NT, K>(sv, g, b, l - 1, Vp);
    } else {
      load(Vp, carry_in + b * V::SZ, 1);  // previous rank's last node (time shard)
    }
  };
  V Vn;
  fetch(K - 1, Vn);
#pragma unroll 1
  for (int c = K / KC - 1; c >= 0; --c) {
#pragma unroll 1
    for (int mm = KC - 1; mm >= 0; --mm) {
      const int m = c * KC + mm;
      const int64_t l = l0 + m;
      const bool valid = l < g.Nn;
      V Vp = Vn;
      if (m > 0) fetch(m - 1, Vn);  // prefetch the next step's (S, v)
#pragma unroll
      for (int i = 0; i < N; ++i) xs[r][mm * N + i] = x[i];
      const int64_t gi = g.node0 + l;
      if (valid && gi != 0) {
        R At[N][N], bt[N], Ct[Dim<N>::NS];
        src.trans(gi, Src::TRANS_Y ? yb + l * Src::NYROW : nullptr, Src::NEEDS_XBAR ? xb + l * N : nullptr, At, bt,
                  Ct);
        trans_step<R, N>(At, bt, Ct, Vp, x, ok);
      }
    }
    __syncthreads();
    // cooperative store of the chunk: one run's KC*N contiguous doubles per pass
    for (int rr = r >> 5; rr < NT; rr += NT / 32) {
      const int64_t lb = (j * NT + rr) * (int64_t)K + c * KC;
      for (int q = r & 31; q < KC * N; q += 32) {
        const int64_t node = lb + q / N;
        if (node < g.Nn) xo[lb * N + q] = xs[rr][q];
      }
    }
    __syncthreads();
  }
  }
  R s = R(0);
#pragma unroll
  for (int i = 0; i < N; ++i) s += x[i];
  if (!(s - s == R(0))) ok = false;
  if (!ok) flag_node(flag, g.node0 + l0);
}

// ---------------------------------------------------------- filter outputs
// m_i = S_i^-1 v_i, P_i = S_i^-1 (packed upper triangle).
template <typename R, int N, int NT, int K>
__global__ void k_filter_out(const Geom g, const R* __restrict__ sv, R* __restrict__ fm, R* __restrict__ fP,
                             unsigned long long* flag) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= g.batch * g.Nn) return;
  const int64_t b = idx / g.Nn, l = idx % g.Nn;
  VF<R, N> V;
  load_sv<R, N, NT, K>(sv, g, b, l, V);
  bool ok = true;
  R m[N];
  spd_solve<R, N>(V.S, V.v, m, ok);
  if (fm) {
#pragma unroll
    for (int i = 0; i < N; ++i) fm[idx * N + i] = m[i];
  }
  if (fP) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      R e[N], col[N];
#pragma unroll
      for (int i = 0; i < N; ++i) e[i] = (i == c) ? R(1) : R(0);
      spd_solve<R, N>(V.S, e, col, ok);
#pragma unroll
      for (int i = 0; i <= c; ++i) fP[idx * Dim<N>::NS + sidx(i, c, N)] = col[i];
    }
  }
  if (!ok) flag_node(flag, g.node0 + l);
}

// --------------------------------------------------- iterated linearisation
template <typename R, int N>
__global__ void k_fill_m0(int64_t count, const R* __restrict__ m0, R* __restrict__ xbar) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx < count) xbar[idx] = m0[idx % N];
}

// max |a - b| as the bit pattern of a non-negative double (order-preserving).
// COPY: also a <- b (the iterated-linearisation loop of a CUDA-graph while node keeps
// xbar in one buffer: pass k reads a, writes b, then a takes b's values).
template <typename R, bool COPY = false>
__global__ void k_maxdiff(int64_t count, R* __restrict__ a, const R* __restrict__ b, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const R bv = b[i];
    double d = fabs((double)a[i] - (double)bv);
    m = (d > m || d != d) ? d : m;
    if (COPY) a[i] = bv;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

}  // namespace pmap
