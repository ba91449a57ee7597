// pmap_make.cuh -- factory definitions, included only by inst.cu.
#pragma once
#include "pmap_runner.cuh"

namespace pmap_rt {

template <typename R, int N, int NY, int KR, int NWC, uint32_t AM, uint32_t UM, uint32_t SM>
Runner* make_lti(const double* A, const double* b, const double* C, const double* J, const double* K,
                 const double* h0, const double* J0, const double* h00, const double* Am, const double* bm,
                 const double* Cm, const double* U) {
  auto* rn = new RunnerT<R, N, NY, SrcLTI<R, N, NY, NWC, AM, UM, SM>, KR>();
  auto& s = rn->src;
  constexpr int NS = Dim<N>::NS;
  for (int i = 0; i < N; ++i) {
    for (int jj = 0; jj < N; ++jj) s.A[i][jj] = (R)A[i * N + jj];
    s.b[i] = (R)b[i];
    s.h0[i] = (R)h0[i];
    s.h00[i] = (R)h00[i];
    for (int k = 0; k < NY; ++k) s.K[i][k] = (R)K[i * NY + k];
  }
  for (int k = 0; k < NS; ++k) {
    s.C[k] = (R)C[k];
    s.J[k] = (R)J[k];
    s.J0[k] = (R)J0[k];
    s.Cm[k] = (R)Cm[k];
  }
  for (int i = 0; i < N; ++i) {
    s.bm[i] = (R)bm[i];
    for (int jj = 0; jj < N; ++jj) s.Am[i][jj] = (R)Am[i * N + jj];
    for (int a = 0; a < (NWC > 0 ? NWC : 1); ++a) {
      s.U[i][a] = NWC > 0 ? (R)U[i * NWC + a] : R(0);
      double t = 0;
      for (int k = 0; k < N && NWC > 0; ++k) t += Am[i * N + k] * U[k * (NWC > 0 ? NWC : 1) + a];
      s.Um[i][a] = (R)t;
    }
  }
  s.zero_b = s.zero_bm = 1;
  for (int i = 0; i < N; ++i) {
    if (s.b[i] != R(0)) s.zero_b = 0;
    if (s.bm[i] != R(0)) s.zero_bm = 0;
  }
  return rn;
}

template <typename R, int N, int NY, int KR>
Runner* make_tv(const R* F, const R* c, const R* L, const R* Wm, const R* H, const R* r, const R* Rm,
                       const int64_t* str, int nw, double dt, const double* P0i, const double* P0im0) {
  auto* rn = new RunnerT<R, N, NY, SrcTV<R, N, NY>, KR>();
  auto& s = rn->src;
  s.F = F; s.c = c; s.L = L; s.W = Wm; s.H = H; s.r = r; s.Rm = Rm;
  s.sF = str[0]; s.sc = str[1]; s.sL = str[2]; s.sW = str[3]; s.sH = str[4]; s.sr = str[5]; s.sR = str[6];
  s.nw = nw;
  s.dt = (R)dt;
  for (int k = 0; k < Dim<N>::NS; ++k) s.P0i[k] = (R)P0i[k];
  for (int i = 0; i < N; ++i) s.P0im0[i] = (R)P0im0[i];
  return rn;
}

template <typename R, int N, int NY, int KIND, int KR>
Runner* make_nl(double dt, double mu, double om_div, const double* C, const double* Ri, const double* P0i,
                const double* P0im0) {
  auto* rn = new RunnerT<R, N, NY, SrcNL<R, N, NY, KIND>, KR>();
  auto& s = rn->src;
  s.dt = (R)dt;
  s.mu = (R)mu;
  s.om_div = om_div != 0.0 ? 1 : 0;
  for (int k = 0; k < Dim<N>::NS; ++k) { s.C[k] = (R)C[k]; s.P0i[k] = (R)P0i[k]; }
  for (int i = 0; i < N; ++i) s.P0im0[i] = (R)P0im0[i];
  for (int a = 0; a < NY; ++a)
    for (int bb = 0; bb < NY; ++bb) s.Ri[a][bb] = (R)Ri[a * NY + bb];
  return rn;
}


template <typename R, int N, int NYM, int NSUB, int KR>
Runner* make_euler(const double* A, const double* C, const double* J, const double* b0, const double* h0,
                   const double* Kb, const double* Ke, const double* J0, const double* h00, const double* K0) {
  using S = SrcEulerLTI<R, N, NYM, NSUB>;
  auto* rn = new RunnerT<R, N, S::NYROW, S, KR>();
  auto& s = rn->src;
  constexpr int NS = Dim<N>::NS;
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j < N; ++j) s.A[i][j] = (R)A[i * N + j];
    s.b0[i] = (R)b0[i];
    s.h0[i] = (R)h0[i];
    s.h00[i] = (R)h00[i];
    for (int k = 0; k < S::NYROW; ++k) {
      s.Kb[i][k] = (R)Kb[i * S::NYROW + k];
      s.Ke[i][k] = (R)Ke[i * S::NYROW + k];
    }
    for (int a = 0; a < NYM; ++a) s.K0[i][a] = (R)K0[i * NYM + a];
  }
  for (int k = 0; k < NS; ++k) {
    s.C[k] = (R)C[k];
    s.J[k] = (R)J[k];
    s.J0[k] = (R)J0[k];
  }
  return rn;
}

}  // namespace pmap_rt
