// pmap_lti.cuh -- pass-1 reduce specialised for time-invariant (LTI) linear models.
//
// For an LTI model every interior node element is E_i = (A, b, C, eta_i, J) with
// only eta_i = K y_i - K r depending on the data (R-ELEM).  The combination rule
// P:395-407 is affine in the data parts (b, eta) with coefficient matrices that
// depend only on the matrix parts (A, C, J) of the two operands:
//   b   = [A2 M] b1 + [A2 M C1] eta2 + b2
//   eta = [A1^T M^T] eta2 - [A1^T M^T J2] b1 + eta1,      M = (I + C1 J2)^-1.
// In an interior tile (all runs full, node 0 not included) the matrix parts of
// every run fold prefix and of every Kogge-Stone span are therefore identical
// across runs and tiles: they are computed once at plan time by k_lti_setup (a
// one-thread device kernel; model-only data, O(K + NT) combines), and the
// per-solve reduce k_p1_reduce_lti only propagates the data parts: ~40 FMA per
// node (fold) + 4 N x N mat-vecs per Kogge-Stone round, instead of one general
// combine (580 FMA at nx = 4) per node.  Boundary tiles (the one holding node 0,
// a ragged last tile) use the general k_p1_reduce.  Output format (run_incl,
// tile_agg) is identical to k_p1_reduce, so every later kernel is shared.
#pragma once
#include "pmap_kernels.cuh"

namespace pmap {

template <typename R, int N, int NT, int K>
struct LtiTables {
  static constexpr int NS = Dim<N>::NS;
  // run fold, step m = 1..K-1 (index m):  b' = b + Wb eta + cb ;  eta' = We eta + ce + eta_m
  R Wb[K][N][N];
  R cb[K][N];
  R We[K][N][N];
  R ce[K][N];
  // the fold is linear in the measurements: (b, eta)_run = crun + sum_m GK[m] y_m
  R GK[K][2 * N][8];  // [m][state][measurement] (NY <= 8)
  R crun[2 * N];
  // matrix parts of the fold prefix of m + 1 nodes, m = 0..K-1
  R PA[K][N][N];
  R PC[K][NS];
  R PJ[K][NS];
  // matrix parts of a span of l full runs, l = 1..NT (index l-1)
  R SA[NT][N][N];
  R SC[NT][NS];
  R SJ[NT][NS];
  // one full run as an element in the Elem field order (data parts zero)
  R E1[N * N + 2 * N + 2 * NS];
  // the same, field-major: SF[f][l-1] (f over A, C, J) so lane r reads column r coalesced
  R SF[N * N + 2 * NS][NT];
  // warp-synchronous Kogge-Stone coefficient sets (compact, so they stay L1-resident):
  //   UWc: round d = 2^lg (< 32) at offset (d - 1) * 4 N^2, layout [u][i][k][slot], slot =
  //        partner span - 1 in 0..d-1 (own span d); lane l >= d reads slot min(l - d, d - 1),
  //        so the d - 1 partial lanes read consecutive doubles and the rest one broadcast slot
  //   UX[u][i][k][lane]: cross-warp step, own span lane+1 (in warp 1), partner span 32
  R UWc[31 * 4 * N * N];
  R UX[4][N][N][32];
  // Kogge-Stone round d (1, 2, 4, ..), partner span l2 in 1..d: index d + l2 - 2
  R U1[NT - 1][N][N];
  R U2[NT - 1][N][N];
  R U3[NT - 1][N][N];
  R U4[NT - 1][N][N];
};

// M = (I + C1 J2)^-1 explicitly (plan-time only), via the pivoted LU of pmap_algebra.
template <typename R, int N>
PM_INLINE void inv_ICJ(const R (&C1)[Dim<N>::NS], const R (&J2)[Dim<N>::NS], R (&M)[N][N]) {
  LUF<R, N> f;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = (i == j) ? R(1) : R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(C1[sidx(i, k, N)], J2[sidx(k, j, N)], s);
      f.a[i][j] = s;
    }
  bool ok = true;
  lu_factor(f, ok);
#pragma unroll
  for (int c = 0; c < N; ++c) {
    R t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] = (i == c) ? R(1) : R(0);
    lu_solve(f, t);
#pragma unroll
    for (int i = 0; i < N; ++i) M[i][c] = t[i];
  }
}

template <typename R, int N>
PM_INLINE void matmul(const R (&X)[N][N], const R (&Y)[N][N], R (&Z)[N][N]) {
  R T[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) {
      R s = R(0);
#pragma unroll
      for (int k = 0; k < N; ++k) s = fma(X[i][k], Y[k][j], s);
      T[i][j] = s;
    }
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) Z[i][j] = T[i][j];
}

template <typename R, int N>
PM_INLINE void unpack(const R (&P)[Dim<N>::NS], R (&M)[N][N]) {
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) M[i][j] = P[sidx(i, j, N)];
}

// Matrix parts of an interior LTI node element and its measurement map.
template <typename R, int N, int NY>
struct LtiNode {
  R A[N][N];
  R b[N];
  R C[Dim<N>::NS];
  R J[Dim<N>::NS];
  R K[N][NY];  // eta_i = K y_i + h0
  R h0[N];
};

// Kernel-parameter copy of the node data and the run-fold tables: read through the
// constant bank, so the fully unrolled fold uses them as DFMA constant operands
// (no load instructions; ~10.7 KB at nx = 4, within the 32 KB parameter limit).
template <typename R, int N, int NY, int K, int LOGNT>
struct LtiFoldParams {
  LtiNode<R, N, NY> node;
  R GK[K][2 * N][NY];  // impulse response of the run fold to y_m
  R crun[2 * N];       // the fold of a run with y = 0
  // Kogge-Stone coefficient sets of round 2^k with a full partner span (the
  // common case): U1..U4 of table index 2 * 2^k - 2
  R Uf[LOGNT][4][N][N];
};

template <int NT>
struct Log2 {
  static constexpr int value = NT <= 1 ? 0 : 1 + Log2<NT / 2>::value;
};

// Plan-time tables (one thread; model-only quantities).
template <typename R, int N, int NY, int NT, int K>
__global__ void k_lti_setup(const LtiNode<R, N, NY> src, LtiTables<R, N, NT, K>* tab, int* okflag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  using E = Elem<R, N>;
  bool ok = true;
  E node;  // interior node element with zero data parts
#pragma unroll
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < N; ++j) node.A[i][j] = src.A[i][j];
    node.b[i] = src.b[i];
    node.h[i] = R(0);
  }
#pragma unroll
  for (int k = 0; k < Dim<N>::NS; ++k) {
    node.C[k] = src.C[k];
    node.J[k] = src.J[k];
  }
  R Am[N][N], Cm[N][N];
  unpack<R, N>(node.C, Cm);
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) Am[i][j] = node.A[i][j];
  E acc = node;
  auto put_prefix = [&](int m) {
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) tab->PA[m][i][j] = acc.A[i][j];
    for (int k = 0; k < Dim<N>::NS; ++k) {
      tab->PC[m][k] = acc.C[k];
      tab->PJ[m][k] = acc.J[k];
    }
  };
  put_prefix(0);
  for (int m = 1; m < K; ++m) {
    R M[N][N], A2M[N][N], T[N][N], J2m[N][N];
    inv_ICJ<R, N>(node.C, acc.J, M);
    matmul<R, N>(acc.A, M, A2M);
    matmul<R, N>(A2M, Cm, T);
    unpack<R, N>(acc.J, J2m);
    for (int i = 0; i < N; ++i) {
      R s = R(0);
      for (int k = 0; k < N; ++k) s = fma(A2M[i][k], node.b[k], s);
      tab->cb[m][i] = s;
      for (int j = 0; j < N; ++j) tab->Wb[m][i][j] = T[i][j];
    }
    // We = A^T M^T ;  ce = -A^T M^T J2 b
    R AtMt[N][N];
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        R s = R(0);
        for (int k = 0; k < N; ++k) s = fma(Am[k][i], M[j][k], s);
        AtMt[i][j] = s;
      }
    R J2b[N];
    for (int i = 0; i < N; ++i) {
      R s = R(0);
      for (int k = 0; k < N; ++k) s = fma(J2m[i][k], node.b[k], s);
      J2b[i] = s;
    }
    for (int i = 0; i < N; ++i) {
      R s = R(0);
      for (int k = 0; k < N; ++k) s = fma(-AtMt[i][k], J2b[k], s);
      tab->ce[m][i] = s;
      for (int j = 0; j < N; ++j) tab->We[m][i][j] = AtMt[i][j];
    }
    combine(node, acc, acc, ok);
    put_prefix(m);
  }
  // impulse response of the run fold (state s = (b, eta), s' = T_m s + [0; eta_m] + c_m,
  // T_m = [[I, Wb_m], [0, We_m]]):  G_m = (T_{K-1} ... T_{m+1})[:, N:2N],  GK_m = G_m K.
  {
    R P[2 * N][2 * N];
    for (int i = 0; i < 2 * N; ++i)
      for (int j = 0; j < 2 * N; ++j) P[i][j] = (i == j) ? R(1) : R(0);
    for (int m = K - 1; m >= 0; --m) {
      for (int i = 0; i < 2 * N; ++i)
        for (int k = 0; k < NY; ++k) {
          R sacc = R(0);
          for (int j = 0; j < N; ++j) sacc = fma(P[i][N + j], src.K[j][k], sacc);
          tab->GK[m][i][k] = sacc;
        }
      if (m >= 1) {  // P <- P T_m
        R Q[2 * N][2 * N];
        for (int i = 0; i < 2 * N; ++i)
          for (int j = 0; j < 2 * N; ++j) {
            R sacc = R(0);
            if (j < N) {
              sacc = P[i][j];  // T_m[:, j] = e_j for the b columns
            } else {
              const int jj = j - N;
              for (int k = 0; k < N; ++k) sacc = fma(P[i][k], tab->Wb[m][k][jj], sacc);
              for (int k = 0; k < N; ++k) sacc = fma(P[i][N + k], tab->We[m][k][jj], sacc);
            }
            Q[i][j] = sacc;
          }
        for (int i = 0; i < 2 * N; ++i)
          for (int j = 0; j < 2 * N; ++j) P[i][j] = Q[i][j];
      }
    }
    // constant part: the data fold with y = 0
    R bb[N], hh[N];
    for (int i = 0; i < N; ++i) {
      bb[i] = src.b[i];
      hh[i] = src.h0[i];
    }
    for (int m = 1; m < K; ++m) {
      R nb[N], nh[N];
      for (int i = 0; i < N; ++i) {
        R s1 = bb[i] + tab->cb[m][i], t1 = src.h0[i] + tab->ce[m][i];
        for (int k = 0; k < N; ++k) {
          s1 = fma(tab->Wb[m][i][k], hh[k], s1);
          t1 = fma(tab->We[m][i][k], hh[k], t1);
        }
        nb[i] = s1;
        nh[i] = t1;
      }
      for (int i = 0; i < N; ++i) {
        bb[i] = nb[i];
        hh[i] = nh[i];
      }
    }
    for (int i = 0; i < N; ++i) {
      tab->crun[i] = bb[i];
      tab->crun[N + i] = hh[i];
    }
  }
  {
    E e1 = acc;
    for (int i = 0; i < N; ++i) {
      e1.b[i] = R(0);
      e1.h[i] = R(0);
    }
    store(e1, tab->E1, 1);
  }
  // spans of l full runs (flipped: later span on the left)
  E run = acc, span = acc;
  for (int l = 1; l <= NT; ++l) {
    if (l > 1) combine(run, span, span, ok);
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) tab->SA[l - 1][i][j] = span.A[i][j];
    for (int k = 0; k < Dim<N>::NS; ++k) {
      tab->SC[l - 1][k] = span.C[k];
      tab->SJ[l - 1][k] = span.J[k];
    }
    int f = 0;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) tab->SF[f++][l - 1] = span.A[i][j];
    for (int k = 0; k < Dim<N>::NS; ++k) tab->SF[f++][l - 1] = span.C[k];
    for (int k = 0; k < Dim<N>::NS; ++k) tab->SF[f++][l - 1] = span.J[k];
  }
  // Kogge-Stone coefficient sets: own span d (left), partner span l2 (right)
  for (int d = 1; d < NT; d <<= 1) {
    for (int l2 = 1; l2 <= d; ++l2) {
      const int idx = d + l2 - 2;
      R C1[Dim<N>::NS], J2[Dim<N>::NS], A1[N][N], A2[N][N], C1m[N][N], J2m[N][N], M[N][N], A2M[N][N], T[N][N];
      for (int k = 0; k < Dim<N>::NS; ++k) {
        C1[k] = tab->SC[d - 1][k];
        J2[k] = tab->SJ[l2 - 1][k];
      }
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
          A1[i][j] = tab->SA[d - 1][i][j];
          A2[i][j] = tab->SA[l2 - 1][i][j];
        }
      unpack<R, N>(C1, C1m);
      unpack<R, N>(J2, J2m);
      inv_ICJ<R, N>(C1, J2, M);
      matmul<R, N>(A2, M, A2M);
      matmul<R, N>(A2M, C1m, T);
      R AtMt[N][N], U4[N][N];
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
          R s = R(0);
          for (int k = 0; k < N; ++k) s = fma(A1[k][i], M[j][k], s);
          AtMt[i][j] = s;
        }
      matmul<R, N>(AtMt, J2m, U4);
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) {
          tab->U1[idx][i][j] = A2M[i][j];
          tab->U2[idx][i][j] = T[i][j];
          tab->U3[idx][i][j] = AtMt[i][j];
          tab->U4[idx][i][j] = U4[i][j];
        }
    }
  }
  // lane-indexed copies for the warp-synchronous scan
  auto coeff = [&](int l1, int l2, int slot, R* dst, int stride) {
    // own span l1 (left), partner span l2 (right): U1 = A2 M, U2 = A2 M C1, U3 = A1^T M^T, U4 = A1^T M^T J2
    R C1[Dim<N>::NS], J2[Dim<N>::NS], A1[N][N], A2[N][N], C1m[N][N], J2m[N][N], M[N][N], A2M[N][N], T[N][N];
    for (int k = 0; k < Dim<N>::NS; ++k) {
      C1[k] = tab->SC[l1 - 1][k];
      J2[k] = tab->SJ[l2 - 1][k];
    }
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        A1[i][j] = tab->SA[l1 - 1][i][j];
        A2[i][j] = tab->SA[l2 - 1][i][j];
      }
    unpack<R, N>(C1, C1m);
    unpack<R, N>(J2, J2m);
    inv_ICJ<R, N>(C1, J2, M);
    matmul<R, N>(A2, M, A2M);
    matmul<R, N>(A2M, C1m, T);
    R AtMt[N][N], U4[N][N];
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        R sacc = R(0);
        for (int k = 0; k < N; ++k) sacc = fma(A1[k][i], M[j][k], sacc);
        AtMt[i][j] = sacc;
      }
    matmul<R, N>(AtMt, J2m, U4);
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        dst[((0 * N + i) * N + j) * stride + slot] = A2M[i][j];
        dst[((1 * N + i) * N + j) * stride + slot] = T[i][j];
        dst[((2 * N + i) * N + j) * stride + slot] = AtMt[i][j];
        dst[((3 * N + i) * N + j) * stride + slot] = U4[i][j];
      }
  };
  for (int lg = 0; lg < 5; ++lg) {
    const int d = 1 << lg;
    R* base = tab->UWc + (d - 1) * 4 * N * N;
    for (int slot = 0; slot < d; ++slot) {
      if (d > NT / 2) {
        for (int q = 0; q < 4 * N * N; ++q) base[q * d + slot] = R(0);
        continue;
      }
      coeff(d, slot + 1, slot, base, d);
    }
  }
  for (int lane = 0; lane < 32; ++lane) {
    if (NT > 32)
      coeff(lane + 1, 32, lane, &tab->UX[0][0][0][0], 32);
    else
      for (int u = 0; u < 4; ++u)
        for (int i = 0; i < N; ++i)
          for (int j = 0; j < N; ++j) tab->UX[u][i][j][lane] = R(0);
  }
  *okflag = ok ? 1 : 0;
}

template <typename R, int N>
PM_INLINE void matvec_acc(const R* __restrict__ M, const R (&x)[N], R (&y)[N]) {  // y += M x (row-major)
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = y[i];
#pragma unroll
    for (int k = 0; k < N; ++k) s = fma(__ldg(M + i * N + k), x[k], s);
    y[i] = s;
  }
}

// Total of the NT run aggregates of a tile (data parts): a binary tree over aligned,
// equal spans, so every combine uses the full-span coefficient set of its level
// (fp.Uf, constant-bank operands; no table loads).  Thread NT-1 ends with the total.
template <typename R, int N, int NY, int NT, int K>
PM_INLINE void lti_run_reduce(const LtiFoldParams<R, N, NY, K, Log2<NT>::value>& fp, int r, R (&bb)[N],
                              R (&hh)[N]) {
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
    if (r == 63) {
      R b2[N], h2[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        b2[i] = tot[i];
        h2[i] = tot[N + i];
      }
      step(5, b2, h2);
    }
  }
}

// Interior tiles only: blockIdx.x -> (trajectory b, tile j = j_lo + blockIdx.x % n_int).
// REV: reversed node order (two-filter pass B over mirrored elements).
// The tile's y block is staged through shared memory (coalesced global reads, a
// padded row per run so the per-run reads are bank-conflict free).
#ifndef PM_REDUCE_MINB
#define PM_REDUCE_MINB 8
#endif
template <typename R, int N, int NY, int NT, int K, bool REV>
__global__ void __launch_bounds__(NT, PM_REDUCE_MINB) k_p1_reduce_lti(const __grid_constant__ LtiFoldParams<R, N, NY, K, Log2<NT>::value> fp,
                                                      const Geom g, int64_t j_lo, int64_t n_int,
                                                      const R* __restrict__ y,
                                                      const LtiTables<R, N, NT, K>* __restrict__ tab,
                                                      R* __restrict__ run_incl, R* __restrict__ tile_agg) {
  using E = Elem<R, N>;
  // The tile's y block is staged in two halves (KH nodes of every run at a time) to keep
  // shared memory small (more CTAs per SM and room in L1 for the scan tables).
  // Padded run rows: 16-byte aligned, consecutive runs 4 banks apart.
#ifndef PM_REDUCE_SPLIT
#define PM_REDUCE_SPLIT 2
#endif
  constexpr int NSPLIT = (K / PM_REDUCE_SPLIT) % 2 == 0 ? PM_REDUCE_SPLIT : 2;
  constexpr int KH = K / NSPLIT;
  static_assert(K % 4 == 0, "run length");
  constexpr int ROW = ((KH * NY * (int)sizeof(R) + 15) / 16 * 16 + 16) / (int)sizeof(R);
  __shared__ __align__(16) R ys[NT * ROW];
  const LtiNode<R, N, NY>& src = fp.node;
  const int64_t b = blockIdx.x / n_int;
  const int64_t j = j_lo + blockIdx.x % n_int;
  const int64_t tile = b * g.tpt + j;
  const int r = threadIdx.x;
  const int64_t base = REV ? (g.Nn - (j + 1) * (int64_t)NT * K) : j * (int64_t)NT * K;
  const R* src_y = y + (b * g.Nn + base) * NY;
  constexpr int BYTES = NY * (int)sizeof(R);
  static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16 || BYTES % 16 == 0, "row size");
  const R* yr = ys + r * ROW;
  // run fold as a sum of independent terms: (b, eta) = crun + sum_m GK[m] y_m
  R acc0[2 * N], acc1[2 * N];
#pragma unroll
  for (int i = 0; i < 2 * N; ++i) {
    acc0[i] = fp.crun[i];
    acc1[i] = R(0);
  }
#pragma unroll
  for (int h = 0; h < NSPLIT; ++h) {
    // one cp.async (LDGSTS) per node row, all in flight at once
#pragma unroll 4
    for (int q = r; q < NT * KH; q += NT) {
      const int run = q / KH, mm = q - run * KH;
      const int tpos = run * K + h * KH + mm;            // position in tile (scan order)
      const int node = REV ? NT * K - 1 - tpos : tpos;   // position in memory
      R* dst = ys + run * ROW + mm * NY;
      const R* srcp = src_y + (int64_t)node * NY;
      const unsigned sdst = (unsigned)__cvta_generic_to_shared(dst);
      if constexpr (BYTES % 16 == 0) {
#pragma unroll
        for (int c = 0; c < BYTES / 16; ++c)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sdst + 16 * c), "l"(srcp + c * (16 / sizeof(R))));
      } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(sdst), "l"(srcp), "n"(BYTES));
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int mm = 0; mm < KH; mm += 2) {
      const int m = h * KH + mm;
      R y0[NY], y1[NY];
#pragma unroll
      for (int k = 0; k < NY; ++k) {
        y0[k] = yr[mm * NY + k];
        y1[k] = yr[(mm + 1) * NY + k];
      }
#pragma unroll
      for (int i = 0; i < 2 * N; ++i)
#pragma unroll
        for (int k = 0; k < NY; ++k) {
          acc0[i] = fma(fp.GK[m][i][k], y0[k], acc0[i]);
          acc1[i] = fma(fp.GK[m + 1][i][k], y1[k], acc1[i]);
        }
    }
    if (h + 1 < NSPLIT) __syncthreads();  // the buffer is refilled by the next part
  }
  R bb[N], hh[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    bb[i] = acc0[i] + acc1[i];
    hh[i] = acc0[N + i] + acc1[N + i];
  }
  // the run's own aggregate, R-RUNAGG: data parts only (the matrix parts of a full
  // interior run are the plan constant tab->SA[0] etc., read by k_p1_down)
  {
    R* oa = run_incl + (g.batch * g.tpt + tile) * (int64_t)E::SZ * NT + r;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      oa[(N * N + i) * NT] = bb[i];
      oa[(N * N + N + Dim<N>::NS + i) * NT] = hh[i];
    }
  }
#ifndef PM_REDUCE_TREE
  // inclusive run prefixes here (the down-sweeps then read them)
  lti_run_scan<R, N, NT>(tab->UWc, &tab->UX[0][0][0][0], r, bb, hh);
  R* out = run_incl + tile * (int64_t)E::SZ * NT + r;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    out[(N * N + i) * NT] = bb[i];
    out[(N * N + N + Dim<N>::NS + i) * NT] = hh[i];
  }
#else
  // PM_REDUCE_TREE (measured slower at C3: the scan moved into the occupancy-limited
  // down-sweep costs more than it saves here): only the tile aggregate, a tree over
  // aligned equal spans with uniform (constant-bank) coefficients; the down-sweeps scan
  // the stored run aggregates themselves (run_carry)
  lti_run_reduce<R, N, NY, NT, K>(fp, r, bb, hh);
#endif
  if (r == NT - 1) {
    E e;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int jj = 0; jj < N; ++jj) e.A[i][jj] = tab->SA[NT - 1][i][jj];
      e.b[i] = bb[i];
      e.h[i] = hh[i];
    }
#pragma unroll
    for (int k = 0; k < Dim<N>::NS; ++k) {
      e.C[k] = tab->SC[NT - 1][k];
      e.J[k] = tab->SJ[NT - 1][k];
    }
    store(e, tile_agg + tile * (int64_t)E::SZ, 1);
  }
}

// Data parts (b, eta) of the fold of q consecutive interior nodes whose first row is
// yrow(0) (LTI recurrence, steps 1..q-1 of the tables).
template <typename R, int N, int NY, int NT, int K, class YRow>
PM_INLINE void lti_fold_data(const LtiNode<R, N, NY>& src, const LtiTables<R, N, NT, K>* __restrict__ tab, int q,
                             YRow yrow, R (&bb)[N], R (&hh)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    R s = src.h0[i];
#pragma unroll
    for (int k = 0; k < NY; ++k) s = fma(src.K[i][k], yrow(0)[k], s);
    hh[i] = s;
    bb[i] = src.b[i];
  }
  for (int m = 1; m < q; ++m) {
    R yv[NY];
#pragma unroll
    for (int k = 0; k < NY; ++k) yv[k] = yrow(m)[k];
    R nb[N], nh[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      R s = bb[i] + __ldg(&tab->cb[m][i]);
      R t = src.h0[i] + __ldg(&tab->ce[m][i]);
#pragma unroll
      for (int k = 0; k < NY; ++k) t = fma(src.K[i][k], yv[k], t);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        s = fma(__ldg(&tab->Wb[m][i][k]), hh[k], s);
        t = fma(__ldg(&tab->We[m][i][k]), hh[k], t);
      }
      nb[i] = s;
      nh[i] = t;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      bb[i] = nb[i];
      hh[i] = nh[i];
    }
  }
}

// Boundary tiles of an LTI model (the tile holding node 0 / the terminal node, a
// ragged last tile): run elements from the LTI data recurrence and the fold-prefix
// matrix tables (plus one general combine with E_0 / M_T for the run holding it),
// then a general Kogge-Stone over the runs.  blockIdx.x -> (b, jsel[k]).
template <typename R, int N, int NY, int NT, int K, class Src, bool REV>
__global__ void __launch_bounds__(NT) k_p1_reduce_lti_edge(const __grid_constant__ Src gsrc,
                                                           const __grid_constant__ LtiNode<R, N, NY> src, const Geom g,
                                                           int nsel, int64_t jsel0, int64_t jsel1,
                                                           const R* __restrict__ y,
                                                           const LtiTables<R, N, NT, K>* __restrict__ tab,
                                                           R* __restrict__ run_incl, R* __restrict__ tile_agg,
                                                           unsigned long long* flag) {
  using E = Elem<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);  // [E::SZ][NT]
  const int64_t b = blockIdx.x / nsel;
  const int64_t j = (blockIdx.x % nsel == 0) ? jsel0 : jsel1;
  const int64_t tile = b * g.tpt + j;
  const int r = threadIdx.x;
  const int64_t l0 = (j * NT + r) * (int64_t)K;
  const R* yb = y + b * g.Nn * NY;
  auto lidx = [&](int64_t lr) { return REV ? (g.Nn - 1 - lr) : lr; };
  const int64_t rem = g.Nn - l0;
  const int q = rem <= 0 ? 0 : (rem >= K ? K : (int)rem);
  const bool first = (l0 == 0) && (REV || g.node0 == 0);  // run holds E_0 (or M_T)
  bool ok = true;
  E acc;
  set_identity(acc);
  if (q > 0) {
    const int qf = first ? q - 1 : q;  // interior nodes of the run
    const int64_t s0 = first ? l0 + 1 : l0;
    if (qf > 0) {
      R bb[N], hh[N];
      lti_fold_data<R, N, NY, NT, K>(src, tab, qf, [&](int m) { return yb + lidx(s0 + m) * NY; }, bb, hh);
#pragma unroll
      for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int jj = 0; jj < N; ++jj) acc.A[i][jj] = tab->PA[qf - 1][i][jj];
        acc.b[i] = bb[i];
        acc.h[i] = hh[i];
      }
#pragma unroll
      for (int k = 0; k < Dim<N>::NS; ++k) {
        acc.C[k] = tab->PC[qf - 1][k];
        acc.J[k] = tab->PJ[qf - 1][k];
      }
    }
    // run aggregate for pass 2 (R-RUNAGG): the run holding node 0 stores its fold
    // without node 0 (no transition into node 0)
    store(acc, run_incl + (g.batch * g.tpt + tile) * (int64_t)E::SZ * NT + r, NT);
    if (first) {
      const int64_t l = lidx(l0);
      E e0;
      gsrc.node(g.node0 + l, yb + l * NY, (const R*)nullptr, e0);
      if (qf > 0)
        combine(acc, e0, acc, ok);  // later nodes on the left (R-FLIP)
      else
        acc = e0;
    }
  } else {
    store(acc, run_incl + (g.batch * g.tpt + tile) * (int64_t)E::SZ * NT + r, NT);
  }
#pragma unroll 1
  for (int d = 1; d < NT; d <<= 1) {
    store(acc, sh + r, NT);
    __syncthreads();
    if (r >= d) combine_g(acc, ElemRef<R, N>{sh + r - d, NT}, acc, ok);
    __syncthreads();
  }
  store(acc, run_incl + tile * (int64_t)E::SZ * NT + r, NT);
  if (r == NT - 1) store(acc, tile_agg + tile * (int64_t)E::SZ, 1);
  if (!ok) atomicMin(flag, (unsigned long long)(g.node0 + l0));
}

}  // namespace pmap
