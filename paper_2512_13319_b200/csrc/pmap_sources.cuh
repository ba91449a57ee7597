// pmap_sources.cuh -- per-node element builders ("element sources") for the scans.
//
// A source turns the model and the data of one grid node i into the node element
// (DESIGN.md R-ELEM; one explicit step of the element ODEs P:416-427 from the
// boundary (I, 0, 0, 0, 0) of P:427, measurement attached to its own node, R-NODE):
//   E_0 = (0, 0, 0, P0^-1 m0 + K_0 (y_0 - r_0), P0^-1 + K_0 H_0)
//   E_i = (I - dt F_i, -dt c_i, dt Q_i, K_i (y_i - r_i), K_i H_i),  K_i = dt H_i^T R_i^-1
// and, for pass 2, the transition data (A_i, b_i, C_i) of node i >= 1.
// Sources are passed to kernels by value (__grid_constant__): model constants sit
// in the kernel-parameter constant bank and are broadcast to all threads.
#pragma once
#include "pmap_algebra.cuh"

namespace pmap {

// ---------------------------------------------------------------- LTI model
// F, c, L, W, H, r, R constant in time (all strides 0).  Everything but the
// y-dependent eta is precomputed on the host at plan time.
// NWC > 0: the diffusion has low rank, C = dt Q = U U^T with U (N x NWC), and the
// per-node value-function update uses the Woodbury form (vapply_lowrank, R-LOWRANK).
template <typename R, int N, int NY, int NWC = 0, uint32_t AM = ~0u, uint32_t UM = ~0u, uint32_t SM = ~0u>
struct SrcLTI {
  static constexpr int NS = Dim<N>::NS;
  static constexpr bool IS_LTI_SRC = true;
  static constexpr int LOWRANK = NWC;
  // structural-zero masks of A (N x N) and U (N x NWC) this instantiation is specialised
  // for (R-MASK); the plan picks it only when the model's zeros cover the mask's zeros
  static constexpr uint32_t AMASK = AM;
  static constexpr uint32_t UMASK = UM;
  // structural zeros of S the look-back pass-2 node recursion skips (R-SMASK): closed under
  // the low-rank update (static_assert in vapply_lowrank); J's and J0's zeros, and those of
  // the plan's S chain, are checked at plan time
  static constexpr uint32_t SMASK = SM;
  static constexpr int NXB = N;  // row width of the nominal trajectory (unused)
  static constexpr bool NEEDS_XBAR = false;
  static constexpr int NYROW = NY;         // doubles of y per node
  static constexpr bool TRANS_Y = false;   // the pass-2 transition does not depend on y
  R A[N][N];
  R b[N];
  R C[NS];
  R J[NS];
  R K[N][NY];  // dt H^T R^-1
  R h0[N];     // -K r          (eta offset, nodes >= 1)
  R J0[NS];    // P0^-1 + K H
  R h00[N];    // P0^-1 m0 - K r
  R Am[N][N];  // (I - dt F)^-1             (two-filter mirrored element, R-TF)
  R bm[N];     // (I - dt F)^-1 dt c
  R Cm[NS];    // (I - dt F)^-1 dt Q (I - dt F)^-T
  R U[N][NWC > 0 ? NWC : 1];   // dt Q = U U^T (NWC > 0)
  R Um[N][NWC > 0 ? NWC : 1];  // mirrored: Cm = (Am U)(Am U)^T
  int zero_b = 0, zero_bm = 0;  // b == 0 / bm == 0 (c == 0): the node updates skip S b
  static constexpr bool HAS_MIRROR = true;

  // the same model in another precision (mixed-precision pass 2, MAP_FLAG_MIXED)
  template <typename R2>
  using rebind = SrcLTI<R2, N, NY, NWC, AM, UM, SM>;
  template <typename R2>
  __host__ rebind<R2> cast() const {
    rebind<R2> o;
    for (int i = 0; i < N; ++i) {
      for (int j = 0; j < N; ++j) {
        o.A[i][j] = (R2)A[i][j];
        o.Am[i][j] = (R2)Am[i][j];
      }
      o.b[i] = (R2)b[i];
      o.bm[i] = (R2)bm[i];
      o.h0[i] = (R2)h0[i];
      o.h00[i] = (R2)h00[i];
      for (int k = 0; k < NY; ++k) o.K[i][k] = (R2)K[i][k];
      for (int a = 0; a < (NWC > 0 ? NWC : 1); ++a) {
        o.U[i][a] = (R2)U[i][a];
        o.Um[i][a] = (R2)Um[i][a];
      }
    }
    for (int k = 0; k < NS; ++k) {
      o.C[k] = (R2)C[k];
      o.J[k] = (R2)J[k];
      o.J0[k] = (R2)J0[k];
      o.Cm[k] = (R2)Cm[k];
    }
    o.zero_b = zero_b;
    o.zero_bm = zero_bm;
    return o;
  }

  // Mirrored element M_i of node gi (R-TF); the terminal node Tg has no transition.
  PM_INLINE void mirror(int64_t gi, int64_t Tg, const R* yrow, Elem<R, N>& e) const {
    R yv[NY];
#pragma unroll
    for (int k = 0; k < NY; ++k) yv[k] = yrow[k];
    const bool last = (gi == Tg);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = h0[i];
#pragma unroll
      for (int k = 0; k < NY; ++k) s = fma(K[i][k], yv[k], s);
      e.h[i] = s;
#pragma unroll
      for (int j = 0; j < N; ++j) e.A[i][j] = last ? R(0) : Am[i][j];
      e.b[i] = last ? R(0) : bm[i];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      e.C[k] = last ? R(0) : Cm[k];
      e.J[k] = J[k];
    }
  }

  PM_INLINE void node(int64_t gi, const R* yrow, const R* /*xrow*/, Elem<R, N>& e) const {
    R yv[NY];
#pragma unroll
    for (int k = 0; k < NY; ++k) yv[k] = yrow[k];
    const bool first = (gi == 0);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = first ? h00[i] : h0[i];
#pragma unroll
      for (int k = 0; k < NY; ++k) s = fma(K[i][k], yv[k], s);
      e.h[i] = s;
#pragma unroll
      for (int j = 0; j < N; ++j) e.A[i][j] = first ? R(0) : A[i][j];
      e.b[i] = first ? R(0) : b[i];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      e.C[k] = first ? R(0) : C[k];
      e.J[k] = first ? J0[k] : J[k];
    }
  }
  // element of a node gi >= 1 (no node-0 selects: constants stay constant-bank operands)
  PM_INLINE void node_interior(int64_t /*gi*/, const R* yrow, const R* /*xrow*/, Elem<R, N>& e) const {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = h0[i];
#pragma unroll
      for (int k = 0; k < NY; ++k) s = fma(K[i][k], yrow[k], s);
      e.h[i] = s;
#pragma unroll
      for (int j = 0; j < N; ++j) e.A[i][j] = A[i][j];
      e.b[i] = b[i];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      e.C[k] = C[k];
      e.J[k] = J[k];
    }
  }
  PM_INLINE void trans(int64_t /*gi*/, const R* /*yrow*/, const R* /*xrow*/, R (&At)[N][N], R (&bt)[N],
                       R (&Ct)[NS]) const {
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) At[i][j] = A[i][j];
      bt[i] = b[i];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) Ct[k] = C[k];
  }
};

// ------------------------------------------------------- time-varying model
// Per-node device arrays (converted to R at plan time); stride 0 = constant.
template <typename R, int N, int NY>
struct SrcTV {
  static constexpr int NS = Dim<N>::NS;
  static constexpr bool IS_LTI_SRC = false;
  static constexpr int LOWRANK = 0;
  static constexpr bool NEEDS_XBAR = false;
  static constexpr bool HAS_MIRROR = true;
  static constexpr int NYROW = NY;
  static constexpr bool TRANS_Y = false;
  const R *F, *c, *L, *W, *H, *r, *Rm;
  int64_t sF, sc, sL, sW, sH, sr, sR;
  int nw;
  R dt;
  R P0i[NS];
  R P0im0[N];

  PM_INLINE void model(int64_t gi, R (&Ft)[N][N], R (&ct)[N], R (&Q)[NS]) const {
    const R* Fp = F + gi * sF;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) Ft[i][j] = Fp[i * N + j];
      ct[i] = c ? c[gi * sc + i] : R(0);
    }
    const R* Lp = L + gi * sL;
    const R* Wp = W + gi * sW;
    // Q = L W L^T, nw <= N
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i; j < N; ++j) {
        R s = R(0);
        for (int a = 0; a < nw; ++a) {
          R t = R(0);
          for (int bb = 0; bb < nw; ++bb) t = fma(Wp[a * nw + bb], Lp[j * nw + bb], t);
          s = fma(Lp[i * nw + a], t, s);
        }
        Q[sidx(i, j, N)] = s;
      }
  }
  // K = dt H^T R^-1 and the offset-corrected measurement at node gi
  PM_INLINE void meas(int64_t gi, R (&Kt)[N][NY], R (&Hm)[NY][N], R (&rr)[NY]) const {
    const R* Hp = H + gi * sH;
    const R* Rp = Rm + gi * sR;
#pragma unroll
    for (int a = 0; a < NY; ++a) {
#pragma unroll
      for (int j = 0; j < N; ++j) Hm[a][j] = Hp[a * N + j];
      rr[a] = r ? r[gi * sr + a] : R(0);
    }
    // R^-1 H via LU (NY small)
    LUF<R, NY> f;
#pragma unroll
    for (int a = 0; a < NY; ++a)
#pragma unroll
      for (int bb = 0; bb < NY; ++bb) f.a[a][bb] = Rp[a * NY + bb];
    bool ok = true;
    lu_factor(f, ok);
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R t[NY];
#pragma unroll
      for (int a = 0; a < NY; ++a) t[a] = Hm[a][j];
      lu_solve(f, t);  // column j of R^-1 H  ->  K[j][:] = dt (R^-1 H)[:, j]  (R symmetric)
#pragma unroll
      for (int a = 0; a < NY; ++a) Kt[j][a] = dt * t[a];
    }
  }
  PM_INLINE void node(int64_t gi, const R* yrow, const R* /*xrow*/, Elem<R, N>& e) const {
    R Kt[N][NY], Hm[NY][N], rr[NY];
    meas(gi, Kt, Hm, rr);
    R res[NY];
#pragma unroll
    for (int a = 0; a < NY; ++a) res[a] = yrow[a] - rr[a];
    const bool first = (gi == 0);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = first ? P0im0[i] : R(0);
#pragma unroll
      for (int a = 0; a < NY; ++a) s = fma(Kt[i][a], res[a], s);
      e.h[i] = s;
#pragma unroll
      for (int j = i; j < N; ++j) {
        R t = first ? P0i[sidx(i, j, N)] : R(0);
#pragma unroll
        for (int a = 0; a < NY; ++a) t = fma(Kt[i][a], Hm[a][j], t);
        e.J[sidx(i, j, N)] = t;
      }
    }
    if (first) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) e.A[i][j] = R(0);
        e.b[i] = R(0);
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) e.C[k] = R(0);
    } else {
      R Ft[N][N], ct[N], Q[NS];
      model(gi, Ft, ct, Q);
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) e.A[i][j] = ((i == j) ? R(1) : R(0)) - dt * Ft[i][j];
        e.b[i] = -dt * ct[i];
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) e.C[k] = dt * Q[k];
    }
  }
  PM_INLINE void node_interior(int64_t gi, const R* yrow, const R* xrow, Elem<R, N>& e) const {
    node(gi, yrow, xrow, e);
  }
  PM_INLINE void trans(int64_t gi, const R* /*yrow*/, const R* /*xrow*/, R (&At)[N][N], R (&bt)[N],
                       R (&Ct)[NS]) const {
    R Ft[N][N], ct[N], Q[NS];
    model(gi, Ft, ct, Q);
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) At[i][j] = ((i == j) ? R(1) : R(0)) - dt * Ft[i][j];
      bt[i] = -dt * ct[i];
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) Ct[k] = dt * Q[k];
  }
  // Mirrored element (R-TF): transition of node gi+1 inverted, measurement of node gi.
  PM_INLINE void mirror(int64_t gi, int64_t Tg, const R* yrow, Elem<R, N>& e) const {
    R Kt[N][NY], Hm[NY][N], rr[NY];
    meas(gi, Kt, Hm, rr);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = R(0);
#pragma unroll
      for (int a = 0; a < NY; ++a) s = fma(Kt[i][a], yrow[a] - rr[a], s);
      e.h[i] = s;
#pragma unroll
      for (int j = i; j < N; ++j) {
        R t = R(0);
#pragma unroll
        for (int a = 0; a < NY; ++a) t = fma(Kt[i][a], Hm[a][j], t);
        e.J[sidx(i, j, N)] = t;
      }
    }
    if (gi == Tg) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) e.A[i][j] = R(0);
        e.b[i] = R(0);
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) e.C[k] = R(0);
      return;
    }
    R Ft[N][N], ct[N], Q[NS];
    model(gi + 1, Ft, ct, Q);
    LUF<R, N> f;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) f.a[i][j] = ((i == j) ? R(1) : R(0)) - dt * Ft[i][j];
    bool ok = true;
    lu_factor(f, ok);
    R Am[N][N], T1[N][N];
#pragma unroll
    for (int c = 0; c < N; ++c) {
      R t[N];
#pragma unroll
      for (int i = 0; i < N; ++i) t[i] = (i == c) ? R(1) : R(0);
      lu_solve(f, t);
#pragma unroll
      for (int i = 0; i < N; ++i) Am[i][c] = t[i];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(Am[i][k], dt * ct[k], s);
      e.b[i] = s;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        e.A[i][j] = Am[i][j];
        R t = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) t = fma(Am[i][k], dt * Q[sidx(k, j, N)], t);
        T1[i][j] = t;
      }
    }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i; j < N; ++j) {
        R t = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) t = fma(T1[i][k], Am[j][k], t);
        e.C[sidx(i, j, N)] = t;
      }
  }
};

// --------------------------------------------- nonlinear: linearise at xbar_i
// Taylor linearisation of P:513 (R-LIN): F_i = df(xbar_i), c_i = f(xbar_i) - F_i xbar_i,
// H_i = dh(xbar_i), r_i = h(xbar_i) - H_i xbar_i, so that
//   y_i - r_i = wrap(y_i - h(xbar_i)) + H_i xbar_i     (bearing residual wrapped, R-WRAP).
template <typename R>
PM_INLINE R wrap_pi(R a) {  // to (-pi, pi]
  const R TWO_PI = R(6.28318530717958647692);
  const R PI = R(3.14159265358979323846);
  return a - TWO_PI * ceil((a - PI) / TWO_PI);
}

template <typename R, int N, int NY, int KIND>
struct SrcNL {
  static constexpr int NS = Dim<N>::NS;
  static constexpr bool IS_LTI_SRC = false;
  static constexpr int LOWRANK = 0;
  static constexpr bool NEEDS_XBAR = true;
  static constexpr bool HAS_MIRROR = false;
  static constexpr int NYROW = NY;
  static constexpr bool TRANS_Y = false;
  R dt;
  R mu;           // Van der Pol parameter
  int om_div = 0;  // keep the OM divergence term 1/2 div f linearised into eta
  R C[NS];        // dt Q, Q = L W L^T
  R Ri[NY][NY];   // R^-1
  R P0i[NS];
  R P0im0[N];

  // drift f and Jacobian F at x
  PM_INLINE void drift(const R (&x)[N], R (&f)[N], R (&F)[N][N]) const {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) F[i][j] = R(0);
    if (KIND == 1) {  // coordinated turn
      f[0] = x[2];
      f[1] = x[3];
      f[2] = -x[4] * x[3];
      f[3] = x[4] * x[2];
      f[4] = R(0);
      F[0][2] = R(1);
      F[1][3] = R(1);
      F[2][3] = -x[4];
      F[2][4] = -x[3];
      F[3][2] = x[4];
      F[3][4] = x[2];
    } else {  // Van der Pol (R-VDP)
      f[0] = x[1];
      f[1] = mu * (R(1) - x[0] * x[0]) * x[1] - x[0];
      F[0][1] = R(1);
      F[1][0] = -R(2) * mu * x[0] * x[1] - R(1);
      F[1][1] = mu * (R(1) - x[0] * x[0]);
    }
  }
  // measurement h and Jacobian H at x
  PM_INLINE void meas(const R (&x)[N], R (&h)[NY], R (&H)[NY][N]) const {
#pragma unroll
    for (int a = 0; a < NY; ++a)
#pragma unroll
      for (int j = 0; j < N; ++j) H[a][j] = R(0);
    if (KIND == 1) {  // range / bearing, P:600 (atan2, G13)
      R r2 = x[0] * x[0] + x[1] * x[1];
      R rr = sqrt(r2);
      h[0] = rr;
      h[1] = atan2(x[1], x[0]);
      H[0][0] = x[0] / rr;
      H[0][1] = x[1] / rr;
      H[1][0] = -x[1] / r2;
      H[1][1] = x[0] / r2;
    } else {
      h[0] = x[0];
      H[0][0] = R(1);
    }
  }
  PM_INLINE void node(int64_t gi, const R* yrow, const R* xrow, Elem<R, N>& e) const {
    R x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = xrow[i];
    R h[NY], H[NY][N];
    meas(x, h, H);
    R res[NY];
#pragma unroll
    for (int a = 0; a < NY; ++a) {
      R d = yrow[a] - h[a];
      if (KIND == 1 && a == 1) d = wrap_pi(d);
      R hx = R(0);
#pragma unroll
      for (int j = 0; j < N; ++j) hx = fma(H[a][j], x[j], hx);
      res[a] = d + hx;  // = y_eff - r
    }
    R Kt[N][NY];  // dt H^T R^-1
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int bb = 0; bb < NY; ++bb) {
        R s = R(0);
#pragma unroll
        for (int a = 0; a < NY; ++a) s = fma(H[a][i], Ri[a][bb], s);
        Kt[i][bb] = dt * s;
      }
    const bool first = (gi == 0);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = first ? P0im0[i] : R(0);
#pragma unroll
      for (int a = 0; a < NY; ++a) s = fma(Kt[i][a], res[a], s);
      e.h[i] = s;
#pragma unroll
      for (int j = i; j < N; ++j) {
        R t = first ? P0i[sidx(i, j, N)] : R(0);
#pragma unroll
        for (int a = 0; a < NY; ++a) t = fma(Kt[i][a], H[a][j], t);
        e.J[sidx(i, j, N)] = t;
      }
    }
    if (KIND == 2 && om_div && !first) {
      // OM cost of interval i: + dt/2 div f(x_i), div f = mu (1 - x_0^2) for VdP.  Its
      // Taylor linearisation about xbar_i adds dt/2 grad(div f)(xbar_i)^T x_i to the node
      // cost, i.e. eta_i -= dt/2 grad(div f) = eta_i + (dt mu xbar_0, 0).
      e.h[0] = fma(dt * mu, x[0], e.h[0]);
    }
    if (first) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = 0; j < N; ++j) e.A[i][j] = R(0);
        e.b[i] = R(0);
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) e.C[k] = R(0);
    } else {
      R f[N], F[N][N];
      drift(x, f, F);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        R c = f[i];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          c = fma(-F[i][j], x[j], c);
          e.A[i][j] = ((i == j) ? R(1) : R(0)) - dt * F[i][j];
        }
        e.b[i] = -dt * c;
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) e.C[k] = C[k];
    }
  }
  PM_INLINE void node_interior(int64_t gi, const R* yrow, const R* xrow, Elem<R, N>& e) const {
    node(gi, yrow, xrow, e);
  }
  PM_INLINE void trans(int64_t /*gi*/, const R* /*yrow*/, const R* xrow, R (&At)[N][N], R (&bt)[N],
                       R (&Ct)[NS]) const {
    R x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = xrow[i];
    R f[N], F[N][N];
    drift(x, f, F);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R c = f[i];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        c = fma(-F[i][j], x[j], c);
        At[i][j] = ((i == j) ? R(1) : R(0)) - dt * F[i][j];
      }
      bt[i] = -dt * c;
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) Ct[k] = C[k];
  }
};

// ------------------------------------------- paper-faithful Euler blocks (f2)
// Each grid interval (t_{i-1}, t_i] is a block of NSUB explicit Euler substeps
// (n = 10) of the element ODEs P:416-427 in s (tau time), integrated from the
// boundary (I, 0, 0, 0, 0) of P:427 with the sign of dA/ds corrected (SURVEY G6:
// dA/ds = +A Q J - A F~).  Substep k (k = 0..NSUB-1) uses the measurement at the fine
// time t_{i-1} + (k+1) dt/NSUB (DESIGN.md R-EULER); node 0 carries the prior and y(t_0).
// For LTI models A, C, J of a block are data independent and (b, eta) are affine in
// the block's NSUB measurements, so the plan integrates the ODEs once (host, fp64) into
// constants plus data-coefficient matrices (the same superposition as R-LTI); the
// kernels evaluate b = b0 + Kb y_blk, eta = h0 + Ke y_blk.  y rows hold NSUB*NYM
// values: [NSUB][NYM] per block, node 0's y(t_0) in its last sub-slot.
template <typename R, int N, int NYM, int NSUB>
struct SrcEulerLTI {
  static constexpr int NS = Dim<N>::NS;
  static constexpr int NYROW = NSUB * NYM;
  static constexpr int NSUB_ = NSUB, NYM_ = NYM;  // refinement (R-REFINE)
  static constexpr bool IS_LTI_SRC = false;
  static constexpr int LOWRANK = 0;
  static constexpr bool NEEDS_XBAR = false;
  static constexpr bool HAS_MIRROR = false;
  static constexpr bool TRANS_Y = true;  // b of a block depends on its measurements
  R A[N][N];
  R C[NS];
  R J[NS];
  R b0[N];
  R h0[N];
  R Kb[N][NYROW];
  R Ke[N][NYROW];
  R J0[NS];     // P0^-1 + delta H^T R^-1 H
  R h00[N];     // P0^-1 m0 - delta H^T R^-1 r
  R K0[N][NYM]; // delta H^T R^-1

  PM_INLINE void data_parts(const R* yrow, R (&b)[N], R (&h)[N]) const {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R sb = b0[i], sh = h0[i];
#pragma unroll
      for (int k = 0; k < NYROW; ++k) {
        const R yk = yrow[k];
        sb = fma(Kb[i][k], yk, sb);
        sh = fma(Ke[i][k], yk, sh);
      }
      b[i] = sb;
      h[i] = sh;
    }
  }
  PM_INLINE void node(int64_t gi, const R* yrow, const R* /*xrow*/, Elem<R, N>& e) const {
    if (gi == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        R s = h00[i];
#pragma unroll
        for (int a = 0; a < NYM; ++a) s = fma(K0[i][a], yrow[(NSUB - 1) * NYM + a], s);
        e.h[i] = s;
        e.b[i] = R(0);
#pragma unroll
        for (int j = 0; j < N; ++j) e.A[i][j] = R(0);
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        e.C[k] = R(0);
        e.J[k] = J0[k];
      }
      return;
    }
    data_parts(yrow, e.b, e.h);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) e.A[i][j] = A[i][j];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      e.C[k] = C[k];
      e.J[k] = J[k];
    }
  }
  PM_INLINE void node_interior(int64_t gi, const R* yrow, const R* xrow, Elem<R, N>& e) const {
    node(gi, yrow, xrow, e);
  }
  PM_INLINE void trans(int64_t /*gi*/, const R* yrow, const R* /*xrow*/, R (&At)[N][N], R (&bt)[N],
                       R (&Ct)[NS]) const {
    R h[N];
    data_parts(yrow, bt, h);
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) At[i][j] = A[i][j];
#pragma unroll
    for (int k = 0; k < NS; ++k) Ct[k] = C[k];
  }
};

}  // namespace pmap
