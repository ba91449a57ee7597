// pmap_algebra.cuh -- register-resident small-matrix algebra of the parallel MAP scans.
//
// Element types and operators of arXiv 2512.13319 (P:n = PAPER.md line n):
//   Elem  (A, b, C, eta, J)  conditional value function
//   VF    (S, v)             value function V = 1/2 x^T S x - v^T x
//   Aff   (Phi, beta)        affine transition x -> Phi x + beta
// combine()  = the combination rule of P:395-407 (left operand e1 on [s, gamma],
//              right operand e2 on [gamma, t]);
// vapply()   = combine() with a value function (A = b = C = 0) on the right;
// compose()  = P:448-449.
// All matrices are N x N with N a compile-time constant so every loop unrolls
// and every value lives in registers.  C and J (and S) are symmetric and stored
// as packed upper triangles; only the upper triangle of a symmetric result is
// ever computed, so symmetry is exact.  The shared inverse (I + C1 J2)^-1 is
// never formed: one LU factorisation with partial pivoting (DESIGN.md R-PIVOT,
// SURVEY G26) serves the P x = r and P^T x = r solves.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pmap {

#define PM_INLINE __device__ __forceinline__

// Compact pass-2 record (R-P2REC with R-MASK): when every column a of U has exactly one
// structural non-zero, at row ka (the Wiener-velocity factor U = c [0; I]: rows 2, 3),
// S U = S[:, ka] U[ka][a] and U^T v = U[ka][a] v[ka], so the record stores the columns
// S[:, ka] (symmetric duplicates once) and v[ka] instead of the products: 9 values instead
// of 10 at nx = 4, bit-identical after the pass-2 reconstruction (the products are
// single roundings either way).
template <int N, int NW, uint32_t UM>
struct CompactRec {
  static constexpr bool value = (N == 4 && NW == 2 && UM == ((1u << 4) | (1u << 7)));
  static constexpr int SIZE = 9;
};

// Structural-zero masks (DESIGN.md R-MASK): bit (i * cols + j) set = entry (i, j) may be
// non-zero.  Inside fully unrolled loops the test folds at compile time, so the terms
// of entries that are structurally zero are never issued -- bit-identical results
// (fma(x, 0, s) == s for finite x), fewer FP64 instructions.  ~0u = dense.
__host__ __device__ constexpr bool mask_nz(uint32_t m, int bit) { return ((m >> bit) & 1u) != 0u; }

template <int N>
struct Dim {
  static constexpr int NS = N * (N + 1) / 2;
};

// packed upper-triangle index of (i, j), i <= j, row-major
__host__ __device__ constexpr int sidx(int i, int j, int N) {
  return i <= j ? i * N - (i * (i - 1)) / 2 + (j - i) : j * N - (j * (j - 1)) / 2 + (i - j);
}

// Structural zeros of the value function's S (R-SMASK): SM is a mask over the packed
// upper triangle.  Given the zeros of S, U and A, these are the entries of S U, of
// G = I + U^T S U, of its LDL^T factor L, of Y = L^-1 (S U)^T and of B A (B = S - S U
// G^-1 U^T S) that can be non-zero; closed(): the low-rank node update maps an S with
// zeros outside SM to one with zeros outside SM whenever J has them (checked at plan
// time), so the pass-2 node recursion never computes those entries.
__host__ __device__ constexpr bool sm_nz(uint32_t sm, int i, int j, int N) { return mask_nz(sm, sidx(i, j, N)); }
__host__ __device__ constexpr uint32_t lr_su_mask(int N, int NW, uint32_t UM, uint32_t SM) {
  uint32_t m = 0;
  for (int i = 0; i < N; ++i)
    for (int a = 0; a < NW; ++a)
      for (int k = 0; k < N; ++k)
        if (sm_nz(SM, i, k, N) && mask_nz(UM, k * NW + a)) m |= 1u << (i * NW + a);
  return m;
}
__host__ __device__ constexpr uint32_t lr_g_mask(int N, int NW, uint32_t UM, uint32_t SU) {
  uint32_t m = 0;
  for (int a = 0; a < NW; ++a)
    for (int c = 0; c <= a; ++c) {
      bool nz = a == c;
      for (int k = 0; k < N; ++k)
        if (mask_nz(UM, k * NW + a) && mask_nz(SU, k * NW + c)) nz = true;
      if (nz) m |= 1u << (a * NW + c);
    }
  return m;
}
__host__ __device__ constexpr uint32_t lr_l_mask(int NW, uint32_t G) {
  uint32_t m = 0;
  for (int c = 0; c < NW; ++c)
    for (int a = c + 1; a < NW; ++a) {
      bool nz = mask_nz(G, a * NW + c);
      for (int k = 0; k < c; ++k)
        if (mask_nz(m, a * NW + k) && mask_nz(m, c * NW + k)) nz = true;
      if (nz) m |= 1u << (a * NW + c);
    }
  return m;
}
__host__ __device__ constexpr uint32_t lr_y_mask(int N, int NW, uint32_t SU, uint32_t L) {
  uint32_t m = 0;
  for (int a = 0; a < NW; ++a)
    for (int j = 0; j < N; ++j) {
      bool nz = mask_nz(SU, j * NW + a);
      for (int c = 0; c < a; ++c)
        if (mask_nz(L, a * NW + c) && mask_nz(m, c * N + j)) nz = true;
      if (nz) m |= 1u << (a * N + j);
    }
  return m;
}
__host__ __device__ constexpr uint32_t lr_ba_mask(int N, uint32_t AM, uint32_t SM) {
  uint32_t m = 0;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j)
      for (int k = 0; k < N; ++k)
        if (sm_nz(SM, i, k, N) && mask_nz(AM, k * N + j)) m |= 1u << (i * N + j);
  return m;
}
__host__ __device__ constexpr bool lr_closed(int N, int NW, uint32_t AM, uint32_t SM, uint32_t Y, uint32_t BA) {
  for (int i = 0; i < N; ++i)
    for (int j = i; j < N; ++j) {
      if (sm_nz(SM, i, j, N)) continue;
      for (int a = 0; a < NW; ++a)  // B = S - Ys^T Y
        if (mask_nz(Y, a * N + i) && mask_nz(Y, a * N + j)) return false;
      for (int k = 0; k < N; ++k)  // S' = A^T (B A) + J
        if (mask_nz(AM, k * N + i) && mask_nz(BA, k * N + j)) return false;
    }
  return true;
}
template <int N, int NW, uint32_t AM, uint32_t UM, uint32_t SM>
struct LrMasks {
  static constexpr uint32_t SU = lr_su_mask(N, NW, UM, SM);
  static constexpr uint32_t G = lr_g_mask(N, NW, UM, SU);
  static constexpr uint32_t L = lr_l_mask(NW, G);
  static constexpr uint32_t Y = lr_y_mask(N, NW, SU, L);
  static constexpr uint32_t BA = lr_ba_mask(N, AM, SM);
  static constexpr bool closed = lr_closed(N, NW, AM, SM, Y, BA);
};

template <typename R, int N>
struct Elem {
  static constexpr int NS = Dim<N>::NS;
  static constexpr int SZ = N * N + N + NS + N + NS;
  R A[N][N];
  R b[N];
  R C[NS];
  R h[N];  // eta
  R J[NS];
};

template <typename R, int N>
struct VF {
  static constexpr int NS = Dim<N>::NS;
  static constexpr int SZ = NS + N;
  R S[NS];
  R v[N];
};

template <typename R, int N>
struct Aff {
  static constexpr int SZ = N * N + N;
  R P[N][N];
  R q[N];
};

// ---------------------------------------------------------------- identities
template <typename R, int N>
PM_INLINE void set_identity(Elem<R, N>& e) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) e.A[i][j] = (i == j) ? R(1) : R(0);
    e.b[i] = R(0);
    e.h[i] = R(0);
  }
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) {
    e.C[k] = R(0);
    e.J[k] = R(0);
  }
}

template <typename R, int N>
PM_INLINE void set_identity(Aff<R, N>& a) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) a.P[i][j] = (i == j) ? R(1) : R(0);
    a.q[i] = R(0);
  }
}

template <typename R, int N>
PM_INLINE void set_zero(VF<R, N>& V) {
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) V.S[k] = R(0);
#pragma unroll
  for (int i = 0; i < N; ++i) V.v[i] = R(0);
}

// ------------------------------------------------- strided load / store (SoA)
// Field f of an object lives at p[f * stride]; the field order is the struct order.
template <typename R, int N>
PM_INLINE void store(const Elem<R, N>& e, R* p, int64_t s) {
  int f = 0;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) p[(f++) * s] = e.A[i][j];
#pragma unroll
  for (int i = 0; i < N; ++i) p[(f++) * s] = e.b[i];
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) p[(f++) * s] = e.C[k];
#pragma unroll
  for (int i = 0; i < N; ++i) p[(f++) * s] = e.h[i];
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) p[(f++) * s] = e.J[k];
}

template <typename R, int N>
PM_INLINE void load(Elem<R, N>& e, const R* p, int64_t s) {
  int f = 0;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) e.A[i][j] = p[(f++) * s];
#pragma unroll
  for (int i = 0; i < N; ++i) e.b[i] = p[(f++) * s];
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) e.C[k] = p[(f++) * s];
#pragma unroll
  for (int i = 0; i < N; ++i) e.h[i] = p[(f++) * s];
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) e.J[k] = p[(f++) * s];
}

template <typename R, int N>
PM_INLINE void store(const VF<R, N>& V, R* p, int64_t s) {
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) p[k * s] = V.S[k];
#pragma unroll
  for (int i = 0; i < N; ++i) p[(Dim<N>::NS + i) * s] = V.v[i];
}

template <typename R, int N>
PM_INLINE void load(VF<R, N>& V, const R* p, int64_t s) {
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) V.S[k] = p[k * s];
#pragma unroll
  for (int i = 0; i < N; ++i) V.v[i] = p[(Dim<N>::NS + i) * s];
}

template <typename R, int N>
PM_INLINE void store(const Aff<R, N>& a, R* p, int64_t s) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) p[(i * N + j) * s] = a.P[i][j];
#pragma unroll
  for (int i = 0; i < N; ++i) p[(N * N + i) * s] = a.q[i];
}

template <typename R, int N>
PM_INLINE void load(Aff<R, N>& a, const R* p, int64_t s) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) a.P[i][j] = p[(i * N + j) * s];
#pragma unroll
  for (int i = 0; i < N; ++i) a.q[i] = p[(N * N + i) * s];
}

// ------------------------------------------------------ LU, partial pivoting
template <typename R, int N>
struct LUF {
  R a[N][N];   // strictly lower: L multipliers; upper incl. diagonal: U
  R dinv[N];   // 1 / U[i][i]
  int piv[N];  // row swapped with row k at step k
  bool nopiv;  // no swap happened (fast path)
};

PM_INLINE double pm_abs(double x) { return fabs(x); }
PM_INLINE float pm_abs(float x) { return fabsf(x); }

// correctly rounded reciprocal (bit-identical to 1/x, without the division slow path)
PM_INLINE double pm_rcp(double x) { return __drcp_rn(x); }
PM_INLINE float pm_rcp(float x) { return __frcp_rn(x); }

// Reciprocal of a normal number >= 1 (the LDL pivots of G = I + U^T S U): the
// hardware approximation refined by two Newton steps (error ~1 ulp; no slow path).
PM_INLINE double pm_rcp_ge1(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
PM_INLINE float pm_rcp_ge1(float x) { return __frcp_rn(x); }

// G = L D L^T of the small SPD matrix G = I + U^T (S U) (NW x NW, pivots >= 1),
// sqrt-free.  In: SU = S U.  Out: unit lower L (strict part), Dinv = D^-1.
// ldl_gram with the structural zeros of S U (SUM) and of L (LM) skipped (R-SMASK).
template <typename R, int N, int NW, uint32_t UM, uint32_t SUM, uint32_t LM>
PM_INLINE void ldl_gram_m(const R (&U)[N][NW], const R (&SU)[N][NW], R (&L)[NW][NW], R (&Dinv)[NW], bool& ok) {
  R G[NW][NW];
#pragma unroll
  for (int a = 0; a < NW; ++a)
#pragma unroll
    for (int c = 0; c <= a; ++c) {
      R s = (a == c) ? R(1) : R(0);
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (mask_nz(UM, k * NW + a) && mask_nz(SUM, k * NW + c)) s = fma(U[k][a], SU[k][c], s);
      G[a][c] = s;
    }
  R D[NW];
#pragma unroll
  for (int c = 0; c < NW; ++c) {
    R d = G[c][c];
#pragma unroll
    for (int k = 0; k < c; ++k)
      if (mask_nz(LM, c * NW + k)) d = fma(-L[c][k] * D[k], L[c][k], d);
    ok = ok && (d > R(0));
    D[c] = d;
    Dinv[c] = pm_rcp_ge1(d);
#pragma unroll
    for (int a = c + 1; a < NW; ++a) {
      if (!mask_nz(LM, a * NW + c)) {
        L[a][c] = R(0);
        continue;
      }
      R t = G[a][c];
#pragma unroll
      for (int k = 0; k < c; ++k)
        if (mask_nz(LM, a * NW + k) && mask_nz(LM, c * NW + k)) t = fma(-L[a][k] * D[k], L[c][k], t);
      L[a][c] = t * Dinv[c];
    }
  }
}

template <typename R, int N, int NW, uint32_t UM = ~0u>
PM_INLINE void ldl_gram(const R (&U)[N][NW], const R (&SU)[N][NW], R (&L)[NW][NW], R (&Dinv)[NW], bool& ok) {
  ldl_gram_m<R, N, NW, UM, ~0u, ~0u>(U, SU, L, Dinv, ok);
}

// q <- G^-1 q with G = L D L^T from ldl_gram.
template <typename R, int NW>
PM_INLINE void ldl_solve(const R (&L)[NW][NW], const R (&Dinv)[NW], R (&q)[NW]) {
#pragma unroll
  for (int a = 0; a < NW; ++a) {
    R s = q[a];
#pragma unroll
    for (int c = 0; c < a; ++c) s = fma(-L[a][c], q[c], s);
    q[a] = s;
  }
#pragma unroll
  for (int a = NW - 1; a >= 0; --a) {
    R s = q[a] * Dinv[a];
#pragma unroll
    for (int c = a + 1; c < NW; ++c) s = fma(-L[c][a], q[c], s);
    q[a] = s;
  }
}

// Factorise f.a in place.  Row swaps are predicated selects (no dynamic
// register indexing).  `ok` is cleared on a zero or non-finite pivot.
// Fast path: if the matrix is column diagonally dominant, Gaussian elimination
// keeps it so and partial pivoting (strict ">" test) never swaps -- the
// unpivoted factorisation below is then bit-identical to the pivoted one and
// skips every select.  The (I + C J) matrices of the per-node updates are
// dominant for small dt; general aggregates fall back to the pivoted path.
template <typename R, int N>
PM_INLINE void lu_factor(LUF<R, N>& f, bool& ok) {
#ifdef PM_LU_SPEC
  // speculative unpivoted factorisation; the dominance test runs alongside it and
  // only a non-dominant matrix (rare) is refactorised with pivoting
  R orig[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) orig[i][j] = f.a[i][j];
  bool okf = true;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    f.piv[k] = k;
    R d = f.a[k][k];
    okf = okf && (d != R(0)) && (d == d);
    R di = pm_rcp(d);
    f.dinv[k] = di;
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      R l = f.a[i][k] * di;
      f.a[i][k] = l;
#pragma unroll
      for (int j = k + 1; j < N; ++j) f.a[i][j] = fma(-l, f.a[k][j], f.a[i][j]);
    }
  }
  bool dom = true;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    R off = R(0);
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (i != k) off += pm_abs(orig[i][k]);
    dom = dom && (pm_abs(orig[k][k]) >= off);
  }
  f.nopiv = dom;
  if (dom) {
    ok = ok && okf;
    return;
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) f.a[i][j] = orig[i][j];
#else
  bool dom = true;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    R off = R(0);
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (i != k) off += pm_abs(f.a[i][k]);
    dom = dom && (pm_abs(f.a[k][k]) >= off);
  }
  f.nopiv = dom;
  if (dom) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      f.piv[k] = k;
      R d = f.a[k][k];
      ok = ok && (d != R(0)) && (d == d);
      R di = pm_rcp(d);
      f.dinv[k] = di;
#pragma unroll
      for (int i = k + 1; i < N; ++i) {
        R l = f.a[i][k] * di;
        f.a[i][k] = l;
#pragma unroll
        for (int j = k + 1; j < N; ++j) f.a[i][j] = fma(-l, f.a[k][j], f.a[i][j]);
      }
    }
    return;
  }
#endif
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int p = k;
    R amax = pm_abs(f.a[k][k]);
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      R t = pm_abs(f.a[i][k]);
      bool gt = t > amax;
      p = gt ? i : p;
      amax = gt ? t : amax;
    }
    f.piv[k] = p;
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      bool sw = (p == i);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        R rk = f.a[k][j], ri = f.a[i][j];
        f.a[k][j] = sw ? ri : rk;
        f.a[i][j] = sw ? rk : ri;
      }
    }
    R d = f.a[k][k];
    ok = ok && (d != R(0)) && (d == d);
    R di = pm_rcp(d);
    f.dinv[k] = di;
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      R l = f.a[i][k] * di;
      f.a[i][k] = l;
#pragma unroll
      for (int j = k + 1; j < N; ++j) f.a[i][j] = fma(-l, f.a[k][j], f.a[i][j]);
    }
  }
}

// x <- P^{-1} x   where P = Pi^T L U
template <typename R, int N>
PM_INLINE void lu_solve(const LUF<R, N>& f, R (&x)[N]) {
  if (!f.nopiv) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      bool sw = (f.piv[k] == i);
      R xk = x[k], xi = x[i];
      x[k] = sw ? xi : xk;
      x[i] = sw ? xk : xi;
    }
  }
  }
#pragma unroll
  for (int i = 1; i < N; ++i)
#pragma unroll
    for (int j = 0; j < i; ++j) x[i] = fma(-f.a[i][j], x[j], x[i]);
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
#pragma unroll
    for (int j = i + 1; j < N; ++j) x[i] = fma(-f.a[i][j], x[j], x[i]);
    x[i] *= f.dinv[i];
  }
}

// x <- P^{-T} x   (P^T = U^T L^T Pi)
template <typename R, int N>
PM_INLINE void lu_solve_t(const LUF<R, N>& f, R (&x)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < i; ++j) x[i] = fma(-f.a[j][i], x[j], x[i]);
    x[i] *= f.dinv[i];
  }
#pragma unroll
  for (int i = N - 2; i >= 0; --i)
#pragma unroll
    for (int j = i + 1; j < N; ++j) x[i] = fma(-f.a[j][i], x[j], x[i]);
  if (f.nopiv) return;
#pragma unroll
  for (int k = N - 1; k >= 0; --k) {
#pragma unroll
    for (int i = k + 1; i < N; ++i) {
      bool sw = (f.piv[k] == i);
      R xk = x[k], xi = x[i];
      x[k] = sw ? xi : xk;
      x[i] = sw ? xk : xi;
    }
  }
}

// ----------------------------------------------------------- the operators
// Combination rule, P:395-407 (e1 on [s, gamma] left, e2 on [gamma, t] right):
//   A = A2 (I + C1 J2)^-1 A1
//   b = A2 (I + C1 J2)^-1 (b1 + C1 eta2) + b2
//   C = A2 (I + C1 J2)^-1 C1 A2^T + C2
//   eta = A1^T (I + J2 C1)^-1 (eta2 - J2 b1) + eta1
//   J = A1^T (I + J2 C1)^-1 J2 A1 + J1
// using (I + J2 C1)^-1 = (I + C1 J2)^-T and (I + J2 C1)^-1 J2 = J2 (I + C1 J2)^-1.
template <typename R, int N>
PM_INLINE void combine(const Elem<R, N>& e1, const Elem<R, N>& e2, Elem<R, N>& out, bool& ok) {
  LUF<R, N> f;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = (i == j) ? R(1) : R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(e1.C[sidx(i, k, N)], e2.J[sidx(k, j, N)], s);
      f.a[i][j] = s;
    }
  lu_factor(f, ok);
  R X1[N][N], X3[N][N], x2[N], z[N];
#pragma unroll
  for (int c = 0; c < N; ++c) {
    R t[N], u[N];
#pragma unroll
    for (int i = 0; i < N; ++i) { t[i] = e1.A[i][c]; u[i] = e1.C[sidx(i, c, N)]; }
    lu_solve(f, t);
    lu_solve(f, u);
#pragma unroll
    for (int i = 0; i < N; ++i) { X1[i][c] = t[i]; X3[i][c] = u[i]; }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = e1.b[i], w = e2.h[i];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      s = fma(e1.C[sidx(i, k, N)], e2.h[k], s);
      w = fma(-e2.J[sidx(i, k, N)], e1.b[k], w);
    }
    x2[i] = s;
    z[i] = w;
  }
  lu_solve(f, x2);
  lu_solve_t(f, z);
  Elem<R, N> o;
  // A, b
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(e2.A[i][k], X1[k][j], s);
      o.A[i][j] = s;
    }
    R s = e2.b[i];
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(e2.A[i][k], x2[k], s);
    o.b[i] = s;
  }
  // C = (A2 X3) A2^T + C2 (upper triangle)
  {
    R T1[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        R s = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(e2.A[i][k], X3[k][j], s);
        T1[i][j] = s;
      }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i; j < N; ++j) {
        R s = e2.C[sidx(i, j, N)];
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(T1[i][k], e2.A[j][k], s);
        o.C[sidx(i, j, N)] = s;
      }
  }
  // J = A1^T (J2 X1) + J1 (upper triangle); eta = A1^T z + eta1
  {
    R Y[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        R s = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(e2.J[sidx(i, k, N)], X1[k][j], s);
        Y[i][j] = s;
      }
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = i; j < N; ++j) {
        R s = e1.J[sidx(i, j, N)];
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(e1.A[k][i], Y[k][j], s);
        o.J[sidx(i, j, N)] = s;
      }
      R s = e1.h[i];
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(e1.A[k][i], z[k], s);
      o.h[i] = s;
    }
  }
  out = o;
}

// Right operand of combine_g read in place from a field-major (SoA) element, e.g. a
// partner's slot in shared memory: field f at p[f * s].  Keeps the partner out of
// registers (the register-resident combine of two elements spills at 255 registers).
template <typename R, int N>
struct ElemRef {
  const R* p;
  int64_t s;
  PM_INLINE R A(int i, int j) const { return p[(i * N + j) * s]; }
  PM_INLINE R b(int i) const { return p[(N * N + i) * s]; }
  PM_INLINE R C(int k) const { return p[(N * N + N + k) * s]; }
  PM_INLINE R h(int i) const { return p[(N * N + N + Dim<N>::NS + i) * s]; }
  PM_INLINE R J(int k) const { return p[(N * N + 2 * N + Dim<N>::NS + k) * s]; }
};

template <typename R, int N, class E2>
PM_INLINE void combine_g(const Elem<R, N>& e1, const E2& e2, Elem<R, N>& out, bool& ok) {
  LUF<R, N> f;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = (i == j) ? R(1) : R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(e1.C[sidx(i, k, N)], e2.J(sidx(k, j, N)), s);
      f.a[i][j] = s;
    }
  lu_factor(f, ok);
  R X1[N][N], X3[N][N], x2[N], z[N];
#pragma unroll
  for (int c = 0; c < N; ++c) {
    R t[N], u[N];
#pragma unroll
    for (int i = 0; i < N; ++i) { t[i] = e1.A[i][c]; u[i] = e1.C[sidx(i, c, N)]; }
    lu_solve(f, t);
    lu_solve(f, u);
#pragma unroll
    for (int i = 0; i < N; ++i) { X1[i][c] = t[i]; X3[i][c] = u[i]; }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = e1.b[i], w = e2.h(i);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      s = fma(e1.C[sidx(i, k, N)], e2.h(k), s);
      w = fma(-e2.J(sidx(i, k, N)), e1.b[k], w);
    }
    x2[i] = s;
    z[i] = w;
  }
  lu_solve(f, x2);
  lu_solve_t(f, z);
  Elem<R, N> o;
  // A, b
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(e2.A(i, k), X1[k][j], s);
      o.A[i][j] = s;
    }
    R s = e2.b(i);
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(e2.A(i, k), x2[k], s);
    o.b[i] = s;
  }
  // C = (A2 X3) A2^T + C2 (upper triangle)
  {
    R T1[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        R s = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(e2.A(i, k), X3[k][j], s);
        T1[i][j] = s;
      }
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i; j < N; ++j) {
        R s = e2.C(sidx(i, j, N));
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(T1[i][k], e2.A(j, k), s);
        o.C[sidx(i, j, N)] = s;
      }
  }
  // J = A1^T (J2 X1) + J1 (upper triangle); eta = A1^T z + eta1
  {
    R Y[N][N];
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        R s = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(e2.J(sidx(i, k, N)), X1[k][j], s);
        Y[i][j] = s;
      }
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = i; j < N; ++j) {
        R s = e1.J[sidx(i, j, N)];
#pragma unroll
        for (int k = 0; k < N; ++k) s = fma(e1.A[k][i], Y[k][j], s);
        o.J[sidx(i, j, N)] = s;
      }
      R s = e1.h[i];
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(e1.A[k][i], z[k], s);
      o.h[i] = s;
    }
  }
  out = o;
}

// e1 (x) (0, 0, 0, v, S): the value function of P:333-336 one interval earlier.
//   S' = A1^T S (I + C1 S)^-1 A1 + J1,  v' = A1^T (I + S C1)^-1 (v - S b1) + eta1.
// Also returns the pass-2 transition of the same interval (P:163-198 discretised,
// DESIGN.md R-TRANS):  Phi = (I + C1 S)^-1 A1,  beta = (I + C1 S)^-1 (b1 + C1 v).
template <typename R, int N, bool WANT_TRANS>
PM_INLINE void vapply(const Elem<R, N>& e1, const VF<R, N>& V, VF<R, N>& out, Aff<R, N>* tr, bool& ok) {
  LUF<R, N> f;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = (i == j) ? R(1) : R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(e1.C[sidx(i, k, N)], V.S[sidx(k, j, N)], s);
      f.a[i][j] = s;
    }
  lu_factor(f, ok);
  R X1[N][N], z[N], bt[N];
#pragma unroll
  for (int c = 0; c < N; ++c) {
    R t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] = e1.A[i][c];
    lu_solve(f, t);
#pragma unroll
    for (int i = 0; i < N; ++i) X1[i][c] = t[i];
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R w = V.v[i], s = e1.b[i];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      w = fma(-V.S[sidx(i, k, N)], e1.b[k], w);
      s = fma(e1.C[sidx(i, k, N)], V.v[k], s);
    }
    z[i] = w;
    bt[i] = s;
  }
  lu_solve_t(f, z);
  if (WANT_TRANS) {
    lu_solve(f, bt);
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) tr->P[i][j] = X1[i][j];
      tr->q[i] = bt[i];
    }
  }
  R Y[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(V.S[sidx(i, k, N)], X1[k][j], s);
      Y[i][j] = s;
    }
  VF<R, N> o;
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = i; j < N; ++j) {
      R s = e1.J[sidx(i, j, N)];
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(e1.A[k][i], Y[k][j], s);
      o.S[sidx(i, j, N)] = s;
    }
    R s = e1.h[i];
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(e1.A[k][i], z[k], s);
    o.v[i] = s;
  }
  out = o;
}

// vapply without transition for a node element whose C = U U^T has rank NW < N
// (R-LOWRANK, Woodbury):  (S^-1 + C)^-1 = S - S U G^-1 U^T S =: B,  G = I + U^T S U
// (NW x NW, SPD, G = L D L^T), (I + S C)^-1 = I - S U G^-1 U^T, so
//   S' = A^T B A + J,   v' = A^T [w - S U G^-1 U^T w] + eta,   w = v - S b.
// Same value function as vapply (up to rounding); the N x N pivoted LU becomes an
// NW x NW sqrt-free LDL^T.  zero_b: b == 0 (skips S b).  rec (nullable): pass-2
// record [S U | U^T v] of the input value function (R-P2REC), field stride rstride.
template <typename R, int N, int NW, uint32_t AM = ~0u, uint32_t UM = ~0u, uint32_t SM = ~0u>
PM_INLINE void vapply_lowrank(const Elem<R, N>& e1, const R (&U)[N][NW], const VF<R, N>& V, VF<R, N>& out,
                              bool& ok, R* rec = nullptr, int64_t rstride = 0, bool zero_b = false) {
  using MK = LrMasks<N, NW, AM, UM, SM>;
  static_assert(SM == ~0u || MK::closed, "S mask not closed under the low-rank node update");
  R SU[N][NW];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int a = 0; a < NW; ++a) {
      R s = R(0);
      bool first = true;
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (mask_nz(UM, k * NW + a) && sm_nz(SM, i, k, N)) {
          s = first ? V.S[sidx(i, k, N)] * U[k][a] : fma(V.S[sidx(i, k, N)], U[k][a], s);
          first = false;
        }
      SU[i][a] = s;
    }
  if (rec && CompactRec<N, NW, UM>::value) {
    // columns 2 and 3 of S (S23 once) and v2, v3 -- see CompactRec
    rec[0 * rstride] = V.S[sidx(0, 2, N)];
    rec[1 * rstride] = V.S[sidx(1, 2, N)];
    rec[2 * rstride] = V.S[sidx(2, 2, N)];
    rec[3 * rstride] = V.S[sidx(0, 3, N)];
    rec[4 * rstride] = V.S[sidx(1, 3, N)];
    rec[5 * rstride] = V.S[sidx(2, 3, N)];
    rec[6 * rstride] = V.S[sidx(3, 3, N)];
    rec[7 * rstride] = V.v[N > 2 ? 2 : 0];
    rec[8 * rstride] = V.v[N > 3 ? 3 : 0];
  } else if (rec) {
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int a = 0; a < NW; ++a) rec[(i * NW + a) * rstride] = SU[i][a];
#pragma unroll
    for (int a = 0; a < NW; ++a) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (mask_nz(UM, k * NW + a)) s = fma(U[k][a], V.v[k], s);
      rec[(N * NW + a) * rstride] = s;
    }
  }
  R Lg[NW][NW], dinv[NW];
  ldl_gram_m<R, N, NW, UM, MK::SU, MK::L>(U, SU, Lg, dinv, ok);
  // Y = L^-1 (S U)^T, Ys = D^-1 Y:  S U G^-1 (S U)^T = Ys^T Y
  R Y[NW][N], Ys[NW][N];
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int a = 0; a < NW; ++a) {
      if (!mask_nz(MK::Y, a * N + j)) {
        Y[a][j] = Ys[a][j] = R(0);
        continue;
      }
      R s = SU[j][a];
#pragma unroll
      for (int c = 0; c < a; ++c)
        if (mask_nz(MK::L, a * NW + c) && mask_nz(MK::Y, c * N + j)) s = fma(-Lg[a][c], Y[c][j], s);
      Y[a][j] = s;
      Ys[a][j] = s * dinv[a];
    }
  // B = S - Ys^T Y (symmetric, full for the product below)
  R B[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      if (!sm_nz(SM, i, j, N)) {  // closed mask: B has S's zeros
        B[i][j] = B[j][i] = R(0);
        continue;
      }
      R s = V.S[sidx(i, j, N)];
#pragma unroll
      for (int a = 0; a < NW; ++a)
        if (mask_nz(MK::Y, a * N + i) && mask_nz(MK::Y, a * N + j)) s = fma(-Ys[a][i], Y[a][j], s);
      B[i][j] = s;
      B[j][i] = s;
    }
  // w = v - S b ; q = G^-1 U^T w ; w2 = w - S U q
  R w[N], q[NW];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = V.v[i];
    if (!zero_b) {
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (sm_nz(SM, i, k, N)) s = fma(-V.S[sidx(i, k, N)], e1.b[k], s);
    }
    w[i] = s;
  }
#pragma unroll
  for (int a = 0; a < NW; ++a) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (mask_nz(UM, k * NW + a)) s = fma(U[k][a], w[k], s);
    q[a] = s;
  }
  ldl_solve<R, NW>(Lg, dinv, q);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = w[i];
#pragma unroll
    for (int a = 0; a < NW; ++a)
      if (mask_nz(MK::SU, i * NW + a)) s = fma(-SU[i][a], q[a], s);
    w[i] = s;
  }
  // BA = B A ; S' = A^T (B A) + J (upper triangle) ; v' = A^T w2 + eta
  R BA[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (mask_nz(AM, k * N + j) && sm_nz(SM, i, k, N)) s = fma(B[i][k], e1.A[k][j], s);
      BA[i][j] = s;
    }
  VF<R, N> o;
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = i; j < N; ++j) {
      if (!sm_nz(SM, i, j, N)) {  // closed mask (J's zeros checked at plan time)
        o.S[sidx(i, j, N)] = R(0);
        continue;
      }
      R s = e1.J[sidx(i, j, N)];
#pragma unroll
      for (int k = 0; k < N; ++k)
        if (mask_nz(AM, k * N + i) && mask_nz(MK::BA, k * N + j)) s = fma(e1.A[k][i], BA[k][j], s);
      o.S[sidx(i, j, N)] = s;
    }
    R s = e1.h[i];
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (mask_nz(AM, k * N + i)) s = fma(e1.A[k][i], w[k], s);
    o.v[i] = s;
  }
  out = o;
}

// Pass-2 single step (P:456-459 with the transition of vapply):
//   x_{i-1} = (I + C_i S_{i-1})^-1 (A_i x_i + b_i + C_i v_{i-1}).
template <typename R, int N>
PM_INLINE void trans_step(const R (&A)[N][N], const R (&b)[N], const R (&C)[Dim<N>::NS], const VF<R, N>& V,
                          R (&x)[N], bool& ok) {
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
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = t[i];
}

// Pass-2 step from the low-rank record of V_{i-1} (R-P2REC, C_i = U U^T):
//   w = A_i x_i + b_i + U (U^T v_{i-1}),  x_{i-1} = w - U G^-1 (S U)^T w,  G = I + U^T (S U),
// which is (I + C_i S_{i-1})^-1 (A_i x_i + b_i + C_i v_{i-1}) by the Woodbury identity.
template <typename R, int N, int NW, uint32_t AM = ~0u, uint32_t UM = ~0u>
PM_INLINE void trans_step_rec(const R (&A)[N][N], const R (&b)[N], const R (&U)[N][NW], const R (&SU)[N][NW],
                              const R (&u)[NW], R (&x)[N], bool& ok) {
  R w[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = b[i];
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (mask_nz(AM, i * N + k)) s = fma(A[i][k], x[k], s);
#pragma unroll
    for (int a = 0; a < NW; ++a)
      if (mask_nz(UM, i * NW + a)) s = fma(U[i][a], u[a], s);
    w[i] = s;
  }
  R Lg[NW][NW], dinv[NW], q[NW];
  ldl_gram<R, N, NW, UM>(U, SU, Lg, dinv, ok);
#pragma unroll
  for (int a = 0; a < NW; ++a) {
    R s = R(0);
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(SU[k][a], w[k], s);
    q[a] = s;
  }
  ldl_solve<R, NW>(Lg, dinv, q);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = w[i];
#pragma unroll
    for (int a = 0; a < NW; ++a)
      if (mask_nz(UM, i * NW + a)) s = fma(-U[i][a], q[a], s);
    x[i] = s;
  }
}

// (f o g)(x) = f(g(x)):  (P_f P_g, P_f q_g + q_f).
template <typename R, int N>
PM_INLINE void compose(const Aff<R, N>& f, const Aff<R, N>& g, Aff<R, N>& out) {
  Aff<R, N> o;
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(f.P[i][k], g.P[k][j], s);
      o.P[i][j] = s;
    }
    R s = f.q[i];
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(f.P[i][k], g.q[k], s);
    o.q[i] = s;
  }
  out = o;
}

template <typename R, int N>
PM_INLINE void apply(const Aff<R, N>& f, R (&x)[N]) {
  R t[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = f.q[i];
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(f.P[i][k], x[k], s);
    t[i] = s;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = t[i];
}

// Symmetric positive-definite solve S x = v by Cholesky (x* = S^-1 v).
template <typename R, int N>
PM_INLINE void spd_solve(const R (&S)[Dim<N>::NS], const R (&v)[N], R (&x)[N], bool& ok) {
  R Lm[N][N], di[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    R d = S[sidx(j, j, N)];
#pragma unroll
    for (int k = 0; k < j; ++k) d = fma(-Lm[j][k], Lm[j][k], d);
    ok = ok && (d > R(0));
    R s = sqrt(d);
    Lm[j][j] = s;
    R si = pm_rcp(s);
    di[j] = si;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      R t = S[sidx(i, j, N)];
#pragma unroll
      for (int k = 0; k < j; ++k) t = fma(-Lm[i][k], Lm[j][k], t);
      Lm[i][j] = t * si;
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R t = v[i];
#pragma unroll
    for (int k = 0; k < i; ++k) t = fma(-Lm[i][k], x[k], t);
    x[i] = t * di[i];
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    R t = x[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) t = fma(-Lm[k][i], x[k], t);
    x[i] = t * di[i];
  }
}

// Symmetric positive-definite solve S x = v by LDL^T (no square roots).
template <typename R, int N>
PM_INLINE void spd_solve_ldl(const R (&S)[Dim<N>::NS], const R (&v)[N], R (&x)[N], bool& ok) {
  R Lm[N][N], D[N], Di[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    R d = S[sidx(j, j, N)];
#pragma unroll
    for (int k = 0; k < j; ++k) d = fma(-Lm[j][k] * D[k], Lm[j][k], d);
    ok = ok && (d > R(0));
    D[j] = d;
    Di[j] = pm_rcp(d);
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      R t = S[sidx(i, j, N)];
#pragma unroll
      for (int k = 0; k < j; ++k) t = fma(-Lm[i][k] * D[k], Lm[j][k], t);
      Lm[i][j] = t * Di[j];
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R t = v[i];
#pragma unroll
    for (int k = 0; k < i; ++k) t = fma(-Lm[i][k], x[k], t);
    x[i] = t;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] *= Di[i];
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    R t = x[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) t = fma(-Lm[k][i], x[k], t);
    x[i] = t;
  }
}

// Packed inverse of a symmetric positive-definite S (covariance P = S^-1 from an
// information matrix, P:202 / P:509): one LDL^T factorisation, N unit-vector solves.
template <typename R, int N>
PM_INLINE void spd_inverse(const R (&S)[Dim<N>::NS], R (&P)[Dim<N>::NS], bool& ok) {
  R Lm[N][N], D[N], Di[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    R d = S[sidx(j, j, N)];
#pragma unroll
    for (int k = 0; k < j; ++k) d = fma(-Lm[j][k] * D[k], Lm[j][k], d);
    ok = ok && (d > R(0));
    D[j] = d;
    Di[j] = pm_rcp(d);
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      R t = S[sidx(i, j, N)];
#pragma unroll
      for (int k = 0; k < j; ++k) t = fma(-Lm[i][k] * D[k], Lm[j][k], t);
      Lm[i][j] = t * Di[j];
    }
  }
#pragma unroll
  for (int c = 0; c < N; ++c) {
    R x[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R t = (i == c) ? R(1) : R(0);
#pragma unroll
      for (int k = 0; k < i; ++k) t = fma(-Lm[i][k], x[k], t);
      x[i] = t;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] *= Di[i];
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
      R t = x[i];
#pragma unroll
      for (int k = i + 1; k < N; ++k) t = fma(-Lm[k][i], x[k], t);
      x[i] = t;
    }
#pragma unroll
    for (int i = 0; i <= c; ++i) P[sidx(i, c, N)] = x[i];
  }
}

}  // namespace pmap
