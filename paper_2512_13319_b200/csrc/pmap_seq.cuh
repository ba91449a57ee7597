// pmap_seq.cuh -- sequential on-device baselines: the paper's
// "sequential counterparts" of the parallel scans, run on the
// same B200 with one thread per trajectory.
//
//   k_seq_rts  forward: V_i = E_i (x) V_{i-1} (the value-function recursion, i.e. the
//              Kalman--Bucy filter in information form), stored per
//              node; backward: x*_T = S_T^-1 v_T and the RTS recursion
//              x*_{i-1} = (I + C_i S_{i-1})^-1 (A_i x*_i + b_i + C_i v_{i-1})
//              (DESIGN.md R-TRANS).  Optionally the smoother
//              covariance P^s_{i-1} = Phi_i P^s_i Phi_i^T + Sigma_i with
//              Phi_i = (I + C_i S_{i-1})^-1 A_i, Sigma_i = (I + C_i S_{i-1})^-1 C_i
//              (the covariance of x_{i-1} given x_i and y_0..y_{i-1}), P^s_T = S_T^-1.
//   k_seq_tf   forward as above; backward: the information filter over the mirrored
//              elements (DESIGN.md R-TF), (Lam_i, xi_i) = M_i (x) (Lam_{i+1}, xi_{i+1}),
//              combined per node x*_i = (S_i + Lam_i - J_i^m)^-1 (v_i + xi_i - eta_i^m)
//              (P:462-466), smoother covariance (S_i + Lam_i - J_i^m)^-1.
// Same element sources and register algebra as the parallel path, so the parallel /
// sequential ratio isolates the scan (the comparison the paper makes on its A100).
#pragma once
#include "pmap_tf.cuh"

namespace pmap {

// One backward RTS step in place: x <- (I + C S)^-1 (A x + b + C v); Ps (nullable)
// <- Phi Ps Phi^T + Sigma (packed upper triangles).
template <typename R, int N>
PM_INLINE void rts_back_step(const R (&A)[N][N], const R (&b)[N], const R (&C)[Dim<N>::NS], const VF<R, N>& V,
                             R (&x)[N], R* Ps, bool& ok) {
  constexpr int NS = Dim<N>::NS;
  LUF<R, N> f;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = (i == j) ? R(1) : R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(C[sidx(i, k, N)], V.S[sidx(k, j, N)], s);
      f.a[i][j] = s;
    }
  lu_factor(f, ok);
  R t[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = b[i];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      s = fma(A[i][k], x[k], s);
      s = fma(C[sidx(i, k, N)], V.v[k], s);
    }
    t[i] = s;
  }
  lu_solve(f, t);
  if (Ps) {
    R Phi[N][N], Sig[N][N];
#pragma unroll
    for (int c = 0; c < N; ++c) {
      R u[N], w[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        u[i] = A[i][c];
        w[i] = C[sidx(i, c, N)];
      }
      lu_solve(f, u);
      lu_solve(f, w);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        Phi[i][c] = u[i];
        Sig[i][c] = w[i];
      }
    }
    R M[N][N];  // Phi Ps
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        R s = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(Phi[i][k], Ps[sidx(k, j, N)], s);
        M[i][j] = s;
      }
    R o[NS];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i; j < N; ++j) {
        R s = Sig[i][j];
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(M[i][k], Phi[j][k], s);
        o[sidx(i, j, N)] = s;
      }
#pragma unroll
    for (int k = 0; k < NS; ++k) Ps[k] = o[k];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = t[i];
}

// Forward value-function recursion of one trajectory; V_l stored field-major across
// the batch (ws[(l * SZ + f) * B + b]) so a warp of trajectories stores coalesced.
template <typename R, int N, int NY, class Src>
PM_INLINE void seq_forward(const Src& src, const Geom& g, int64_t b, const R* __restrict__ yb,
                           const R* __restrict__ xb, R* __restrict__ ws, VF<R, N>& cur, bool& ok) {
  using V = VF<R, N>;
  const int64_t B = g.batch;
  set_zero(cur);
  R yn[NY];
#pragma unroll
  for (int k = 0; k < NY; ++k) yn[k] = yb[k];
#pragma unroll 1
  for (int64_t l = 0; l < g.Nn; ++l) {
    R yc[NY];
#pragma unroll
    for (int k = 0; k < NY; ++k) yc[k] = yn[k];
    if (l + 1 < g.Nn) {  // prefetch the next measurement (off the recursion's critical path)
#pragma unroll
      for (int k = 0; k < NY; ++k) yn[k] = yb[(l + 1) * NY + k];
    }
    Elem<R, N> e;
    src.node(g.node0 + l, yc, xb ? xb + l * N : nullptr, e);
    vapply<R, N, false>(e, cur, cur, nullptr, ok);
    store(cur, ws + (l * V::SZ) * B + b, B);
  }
}

template <typename R, int N, int NY, class Src>
__global__ void __launch_bounds__(32) k_seq_rts(const __grid_constant__ Src src, const Geom g,
                                                const R* __restrict__ y, const R* __restrict__ xbar,
                                                R* __restrict__ ws, R* __restrict__ x_out, R* __restrict__ Ps_out,
                                                unsigned long long* flag) {
  using V = VF<R, N>;
  constexpr int NS = Dim<N>::NS;
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= g.batch) return;
  const int64_t B = g.batch;
  const R* yb = y + b * g.Nn * NY;
  const R* xb = xbar ? xbar + b * g.Nn * N : nullptr;
  R* xo = x_out + b * g.Nn * N;
  R* po = Ps_out ? Ps_out + b * g.Nn * NS : nullptr;
  bool ok = true;
  V cur;
  seq_forward<R, N, NY, Src>(src, g, b, yb, xb, ws, cur, ok);
  R x[N], Ps[NS];
  spd_solve<R, N>(cur.S, cur.v, x, ok);  // x*_T = S_T^-1 v_T
  const int64_t last = g.Nn - 1;
#pragma unroll
  for (int i = 0; i < N; ++i) xo[last * N + i] = x[i];
  if (po) {
    spd_inverse<R, N>(cur.S, Ps, ok);
#pragma unroll
    for (int k = 0; k < NS; ++k) po[last * NS + k] = Ps[k];
  }
  V Vn;  // V_{l-1}, loaded one step ahead (independent of the recursion)
  if (last >= 1) load(Vn, ws + ((last - 1) * V::SZ) * B + b, B);
#pragma unroll 1
  for (int64_t l = last; l >= 1; --l) {
    const V Vp = Vn;
    if (l >= 2) load(Vn, ws + ((l - 2) * V::SZ) * B + b, B);
    R At[N][N], bt[N], Ct[NS];
    src.trans(g.node0 + l, yb + l * NY, xb ? xb + l * N : nullptr, At, bt, Ct);
    rts_back_step<R, N>(At, bt, Ct, Vp, x, po ? Ps : nullptr, ok);
#pragma unroll
    for (int i = 0; i < N; ++i) xo[(l - 1) * N + i] = x[i];
    if (po) {
#pragma unroll
      for (int k = 0; k < NS; ++k) po[(l - 1) * NS + k] = Ps[k];
    }
  }
  R s = R(0);
#pragma unroll
  for (int i = 0; i < N; ++i) s += x[i];
  if (!(s - s == R(0))) ok = false;
  if (!ok) flag_node(flag, g.node0);
}

template <typename R, int N, int NY, class Src>
__global__ void __launch_bounds__(32) k_seq_tf(const __grid_constant__ Src src, const Geom g,
                                               const R* __restrict__ y, R* __restrict__ ws, R* __restrict__ x_out,
                                               R* __restrict__ Ps_out, unsigned long long* flag) {
  using V = VF<R, N>;
  constexpr int NS = Dim<N>::NS;
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= g.batch) return;
  const int64_t B = g.batch;
  const R* yb = y + b * g.Nn * NY;
  R* xo = x_out + b * g.Nn * N;
  R* po = Ps_out ? Ps_out + b * g.Nn * NS : nullptr;
  bool ok = true;
  V lam;
  seq_forward<R, N, NY, Src>(src, g, b, yb, nullptr, ws, lam, ok);
  const int64_t Tg = g.node0 + g.Nn - 1;
  set_zero(lam);
  V Vn;  // V_l, loaded one step ahead
  load(Vn, ws + ((g.Nn - 1) * V::SZ) * B + b, B);
#pragma unroll 1
  for (int64_t l = g.Nn - 1; l >= 0; --l) {
    const V Va = Vn;
    if (l >= 1) load(Vn, ws + ((l - 1) * V::SZ) * B + b, B);
    Elem<R, N> e;
    src.mirror(g.node0 + l, Tg, yb + l * NY, e);
    vapply<R, N, false>(e, lam, lam, nullptr, ok);  // (Lam_l, xi_l): y_l..y_T
    R Ssum[NS], rhs[N], xv[N];
#pragma unroll
    for (int k = 0; k < NS; ++k) Ssum[k] = Va.S[k] + (lam.S[k] - e.J[k]);
#pragma unroll
    for (int i = 0; i < N; ++i) rhs[i] = Va.v[i] + (lam.v[i] - e.h[i]);
    spd_solve_ldl<R, N>(Ssum, rhs, xv, ok);
#pragma unroll
    for (int i = 0; i < N; ++i) xo[l * N + i] = xv[i];
    if (po) {
      R P[NS];
      spd_inverse<R, N>(Ssum, P, ok);
#pragma unroll
      for (int k = 0; k < NS; ++k) po[l * NS + k] = P[k];
    }
  }
  if (!ok) flag_node(flag, g.node0);
}

}  // namespace pmap
