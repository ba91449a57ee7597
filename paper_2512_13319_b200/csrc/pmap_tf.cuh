// pmap_tf.cuh -- parallel two-filter smoother.
//
// Reading R-TF: the paper's forward scan over e (x) a_0 (x) ...
// needs J_0^-1 of a one-node element, which is singular whenever ny < nx.  The
// same backward-filter information is obtained exactly by the combination rule
// of P:395-407 applied, in reverse node order, to "mirrored" elements
//   M_i = ((I - dt F_{i+1})^-1, (I - dt F_{i+1})^-1 dt c_{i+1},
//          (I - dt F_{i+1})^-1 dt Q_{i+1} (I - dt F_{i+1})^-T, eta_i^m, J_i^m),
//   M_T = (0, 0, 0, eta_T^m, J_T^m)          (zero prior information at t_T),
// whose suffix products acc_i = M_i (x) acc_{i+1} carry in (J, eta) the backward
// information filter (Lam_i, xi_i) of y_i..y_T.  The two filters are combined per
// node (P:462-466 in information form, C_bar = Lam^-1, b_bar = Lam^-1 xi):
//   x_i = (S_i + Lam_i - J_i^m)^-1 (v_i + xi_i - eta_i^m)   (y_i counted once, R-TF),
// and, optionally, the smoother covariance P^s_i = (S_i + Lam_i - J_i^m)^-1 (the
// posterior precision of x_i is the sum of both filters' information).
// Pass A (forward filter, the pass-1 kernels without the pass-2 fold) and pass B
// (this suffix scan, with the combine fused into its epilogue) are independent
// and run on two streams.
#pragma once
#include "pmap_kernels.cuh"

namespace pmap {

// Adapter: presents the mirrored elements of `Src` as a prefix scan over the
// reversed local index (k_p1_reduce<REV=true> passes the original node index).
template <class Src>
struct Mirror {
  Src s;
  int64_t Tg;  // global index of the last node
  static constexpr bool NEEDS_XBAR = false;
  template <typename R, int N>
  PM_INLINE void node(int64_t gi, const R* yrow, const R* /*xrow*/, Elem<R, N>& e) const {
    s.mirror(gi, Tg, yrow, e);
  }
};

template <typename R, int N, int NY, int NT, int K, class Src>
__global__ void __launch_bounds__(NT) k_tf_down(const __grid_constant__ Mirror<Src> mir, const Geom g,
                                                const R* __restrict__ y, const R* __restrict__ run_incl,
                                                const R* __restrict__ tile_incl, const R* __restrict__ group_carry,
                                                const R* __restrict__ sv, R* __restrict__ x_out,
                                                R* __restrict__ Ps_out, unsigned long long* flag, const R* __restrict__ sf, int64_t j_lo,
                                                int64_t j_hi, const R* __restrict__ uwc = nullptr,
                                                const R* __restrict__ ux = nullptr) {
  using E = Elem<R, N>;
  using V = VF<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);
  const int64_t tile = blockIdx.x;
  const int64_t b = tile / g.tpt, j = tile % g.tpt;
  const int r = threadIdx.x;
  const int64_t l0 = (j * NT + r) * (int64_t)K;  // reversed local index
  const R* yb = y + b * g.Nn * NY;
  R* xo = x_out + b * g.Nn * N;
  bool ok = true;
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
  run_carry<R, N, NT>(run_incl, g, tile, r, sf && j >= j_lo && j < j_hi, sf, uwc, ux, cur, ok);
  // x is staged in shared memory in chunks of KC nodes and stored as contiguous segments
  constexpr int KC = K < 8 ? K : 8;
  static_assert(K % KC == 0, "chunking");
  __shared__ R xs[NT][KC * N + 1];
#pragma unroll 1
  for (int c = 0; c < K / KC; ++c) {
#pragma unroll 1
    for (int mm = 0; mm < KC; ++mm) {
      const int64_t lr = l0 + c * KC + mm;
      if (lr < g.Nn) {
        const int64_t l = g.Nn - 1 - lr;
        V Va;
        load_sv<R, N, NT, K>(sv, g, b, l, Va);  // issued early: independent of the recursion
        E e;
        mir.template node<R, N>(g.node0 + l, yb + l * NY, nullptr, e);
        if constexpr (Src::LOWRANK > 0) {  // mirrored diffusion Cm = (Am U)(Am U)^T
          if (g.node0 + l != mir.Tg)
            vapply_lowrank<R, N, Src::LOWRANK>(e, mir.s.Um, cur, cur, ok, nullptr, 0, mir.s.zero_bm != 0);
          else
            vapply<R, N, false>(e, cur, cur, nullptr, ok);
        } else {
          vapply<R, N, false>(e, cur, cur, nullptr, ok);  // (Lam_l, xi_l)
        }
        R Ssum[Dim<N>::NS], rhs[N], xv[N];
#pragma unroll
        for (int k = 0; k < Dim<N>::NS; ++k) Ssum[k] = Va.S[k] + (cur.S[k] - e.J[k]);
#pragma unroll
        for (int i = 0; i < N; ++i) rhs[i] = Va.v[i] + (cur.v[i] - e.h[i]);
        spd_solve_ldl<R, N>(Ssum, rhs, xv, ok);
#pragma unroll
        for (int i = 0; i < N; ++i) xs[r][mm * N + i] = xv[i];
        if (Ps_out) {  // smoother covariance (S_l + Lam_l - J_l^m)^-1
          R P[Dim<N>::NS];
          spd_inverse<R, N>(Ssum, P, ok);
          R* po = Ps_out + (b * g.Nn + l) * Dim<N>::NS;
#pragma unroll
          for (int k = 0; k < Dim<N>::NS; ++k) po[k] = P[k];
        }
      }
    }
    __syncthreads();
    // run rr's chunk holds nodes Nn-1-(l0_rr + c KC + mm), mm = 0..KC-1 (descending)
    for (int rr = r >> 5; rr < NT; rr += NT / 32) {
      const int64_t lrb = (j * NT + rr) * (int64_t)K + c * KC;
      for (int q = r & 31; q < KC * N; q += 32) {
        const int mm = q / N, i = q - mm * N;
        const int64_t lr = lrb + mm;
        if (lr < g.Nn) xo[(g.Nn - 1 - lr) * N + i] = xs[rr][q];
      }
    }
    __syncthreads();
  }
  if (!ok) flag_node(flag, g.node0 + g.Nn - 1 - l0);
}

}  // namespace pmap
