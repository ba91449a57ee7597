// Latency of one general combine / vapply on a single thread (tools only; B200 probe).
#include <cstdio>
#include "../paper_2512_13319_b200/csrc/pmap_algebra.cuh"
using namespace pmap;
template <int N>
__global__ void k(int reps, double* out, long long* cyc, const double* src) {
  Elem<double, N> e, acc;
  set_identity(e);
  const double dt = 1e-3;
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j < N; ++j) e.A[i][j] = (i == j ? 1.0 : 0.0) + ((j == i + N / 2) ? -dt : 0.0);
    e.b[i] = 0.01 * i;
    e.h[i] = 0.1 * (i + 1);
  }
  for (int k2 = 0; k2 < Dim<N>::NS; ++k2) {
    e.C[k2] = (k2 == Dim<N>::NS - 1 || k2 == 0) ? 4 * dt : 0.0;
    e.J[k2] = (k2 == 0) ? 100 * dt : 0.0;
  }
  if (src) load(e, src, 1);  // opaque operands: no constant folding
  acc = e;
  bool ok = true;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) combine(e, acc, acc, ok);
  long long t1 = clock64();
  VF<double, N> V;
  for (int k2 = 0; k2 < Dim<N>::NS; ++k2) V.S[k2] = acc.J[k2] + (k2 == 0 ? 1.0 : 0.0);
  for (int i = 0; i < N; ++i) V.v[i] = acc.h[i];
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) vapply<double, N, false>(e, V, V, nullptr, ok);
  long long t3 = clock64();
  out[0] = acc.J[0] + V.S[0] + (ok ? 0 : 1);
  cyc[0] = (t1 - t0) / reps;
  cyc[1] = (t3 - t2) / reps;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 16);
  long long h[2];
  // an interior-like element as opaque data
  double hs[128] = {0};
  const double dt = 1e-3;
  int f = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) hs[f++] = (i == j) + ((j == i + 2) ? -dt : 0.0) + 1e-7 * (i + 2 * j);
  for (int i = 0; i < 4; ++i) hs[f++] = 0.01 * i;
  for (int q = 0; q < 10; ++q) hs[f++] = (q == 0 || q == 9 || q == 7) ? 4 * dt : 1e-9 * q;
  for (int i = 0; i < 4; ++i) hs[f++] = 0.1 * (i + 1);
  for (int q = 0; q < 10; ++q) hs[f++] = (q == 0 || q == 4) ? 100 * dt : 1e-9 * q;
  double* ds; cudaMalloc(&ds, sizeof hs); cudaMemcpy(ds, hs, sizeof hs, cudaMemcpyHostToDevice);
  k<4><<<1, 1>>>(64, d, c, nullptr); cudaDeviceSynchronize();
  k<4><<<1, 1>>>(256, d, c, nullptr); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("N=4 const combine %lld cycles, vapply %lld cycles\n", h[0], h[1]);
  k<4><<<1, 1>>>(256, d, c, ds); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("N=4 opaque combine %lld cycles, vapply %lld cycles\n", h[0], h[1]);
  k<4><<<1, 32>>>(256, d, c, ds); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("N=4 opaque 32 lanes combine %lld cycles, vapply %lld cycles\n", h[0], h[1]);
  k<4><<<1, 128>>>(256, d, c, ds); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("N=4 opaque 128 thr combine %lld cycles, vapply %lld cycles\n", h[0], h[1]);
  return 0;
}
