// pmap_refine.cuh -- intra-block refinement of the Euler-block method (
// DESIGN.md R-REFINE).
//
// With Euler blocks of NSUB substeps the solve gives x* at the block boundaries t_i.  The
// fine points t_k = t_{i-1} + k delta (k = 1 .. NSUB-1) inside block i get
//   V_k   = E_pre(k) (x) V_{i-1}      E_pre(k): the element of the block's first k substeps
//                                     (P:416-427 from the boundary of P:427, k Euler steps)
//   x*_k  = (I + C_k S_k)^-1 (A_k x*_i + b_k + C_k v_k)      (R-TRANS)
// with (A_k, b_k, C_k) the element from t_k to t_i by the forward HJB equation
// ("we only need the first three equations"), NSUB - k explicit Euler steps in reversed
// time from the boundary (I, 0, 0).  For an LTI model every matrix part is data-free and
// b, eta are affine in the block's measurements: the plan integrates both ODEs once per k
// with the data parts as coefficient matrices (as R-EULER does for the block element) and
// this kernel evaluates them.  V_{i-1} comes from the solve's filter outputs
// (S = P^-1, v = S m at the block nodes).
#pragma once
#include "pmap_algebra.cuh"

namespace pmap {

// Table of one k (row-major, doubles converted to R), NR = NSUB * NYM:
//   Apre N*N | Cpre NS | Jpre NS | bpre N | hpre N | Kbpre N*NR | Kepre N*NR |
//   Asuf N*N | Csuf NS | bsuf N | Kbsuf N*NR
template <int N, int NR>
struct RefineTab {
  static constexpr int NS = Dim<N>::NS;
  static constexpr int APRE = 0, CPRE = N * N, JPRE = CPRE + NS, BPRE = JPRE + NS, HPRE = BPRE + N,
                       KBPRE = HPRE + N, KEPRE = KBPRE + N * NR, ASUF = KEPRE + N * NR, CSUF = ASUF + N * N,
                       BSUF = CSUF + NS, KBSUF = BSUF + N, F = KBSUF + N * NR;
};

// One thread per (trajectory, block i >= 1).  y: [batch][T+1][NSUB*NYM] (Euler rows);
// xb, fm: [batch][T+1][N]; fP: [batch][T+1][NS] packed; xf: [batch][NSUB*T+1][N].
template <typename R, int N, int NYM, int NSUB>
__global__ void __launch_bounds__(128) k_euler_refine(const R* __restrict__ tab, int64_t T, int64_t batch,
                                                      const R* __restrict__ y, const R* __restrict__ xb,
                                                      const R* __restrict__ fm, const R* __restrict__ fP,
                                                      R* __restrict__ xf, unsigned long long* flag) {
  constexpr int NS = Dim<N>::NS;
  constexpr int NR = NSUB * NYM;
  using TB = RefineTab<N, NR>;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= batch * T) return;
  const int64_t b = idx / T, i = 1 + idx % T;
  const int64_t Nn = T + 1, Nf = (int64_t)NSUB * T + 1;
  const R* yr = y + (b * Nn + i) * NR;
  R yv[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) yv[k] = __ldg(yr + k);
  R xi[N];
#pragma unroll
  for (int a = 0; a < N; ++a) xi[a] = xb[(b * Nn + i) * N + a];
  R* xo = xf + b * Nf * N;
#pragma unroll
  for (int a = 0; a < N; ++a) xo[(int64_t)i * NSUB * N + a] = xi[a];
  if (i == 1) {
#pragma unroll
    for (int a = 0; a < N; ++a) xo[a] = xb[b * Nn * N + a];
  }
  // V_{i-1} from the filter outputs: S = P^-1, v = S m
  bool ok = true;
  VF<R, N> V;
  {
    R P[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) P[k] = fP[(b * Nn + i - 1) * NS + k];
    spd_inverse<R, N>(P, V.S, ok);
    R m[N];
#pragma unroll
    for (int a = 0; a < N; ++a) m[a] = fm[(b * Nn + i - 1) * N + a];
#pragma unroll
    for (int a = 0; a < N; ++a) {
      R s = R(0);
#pragma unroll
      for (int c = 0; c < N; ++c) s = fma(V.S[a <= c ? sidx(a, c, N) : sidx(c, a, N)], m[c], s);
      V.v[a] = s;
    }
  }
#pragma unroll 1
  for (int k = 1; k < NSUB; ++k) {
    const R* t = tab + (int64_t)(k - 1) * TB::F;
    Elem<R, N> e;
#pragma unroll
    for (int a = 0; a < N; ++a) {
#pragma unroll
      for (int c = 0; c < N; ++c) e.A[a][c] = __ldg(t + TB::APRE + a * N + c);
      R sb = __ldg(t + TB::BPRE + a), sh = __ldg(t + TB::HPRE + a);
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        sb = fma(__ldg(t + TB::KBPRE + a * NR + q), yv[q], sb);
        sh = fma(__ldg(t + TB::KEPRE + a * NR + q), yv[q], sh);
      }
      e.b[a] = sb;
      e.h[a] = sh;
    }
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      e.C[q] = __ldg(t + TB::CPRE + q);
      e.J[q] = __ldg(t + TB::JPRE + q);
    }
    VF<R, N> Vk;
    vapply<R, N, false>(e, V, Vk, nullptr, ok);
    R As[N][N], bs[N], Cs[NS];
#pragma unroll
    for (int a = 0; a < N; ++a) {
#pragma unroll
      for (int c = 0; c < N; ++c) As[a][c] = __ldg(t + TB::ASUF + a * N + c);
      R sb = __ldg(t + TB::BSUF + a);
#pragma unroll
      for (int q = 0; q < NR; ++q) sb = fma(__ldg(t + TB::KBSUF + a * NR + q), yv[q], sb);
      bs[a] = sb;
    }
#pragma unroll
    for (int q = 0; q < NS; ++q) Cs[q] = __ldg(t + TB::CSUF + q);
    R x[N];
#pragma unroll
    for (int a = 0; a < N; ++a) x[a] = xi[a];
    trans_step<R, N>(As, bs, Cs, Vk, x, ok);
#pragma unroll
    for (int a = 0; a < N; ++a) xo[((i - 1) * NSUB + k) * N + a] = x[a];
  }
  if (!ok) atomicMin(flag, (unsigned long long)i);
}

}  // namespace pmap
