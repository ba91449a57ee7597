// Isolated timing of k_p1_tiles / k_p1_groups at the C3 geometry (tools only; B200 probe).
#include <cstdio>
#include <vector>
#include "../paper_2512_13319_b200/csrc/pmap_kernels.cuh"
using namespace pmap;
// copy of k_p1_tiles with stages switchable (MODE bit0: skip combine, bit1: skip global load/store,
// bit2: time stages with clock64 into dbg)
template <typename R, int N, int MODE>
__global__ void __launch_bounds__(NT2) k_tiles_probe(const Geom g, const R* __restrict__ tile_agg,
                                                  R* __restrict__ tile_incl, R* __restrict__ group_agg,
                                                  unsigned long long* flag, long long* dbg) {
  using E = Elem<R, N>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sh = reinterpret_cast<R*>(smem_raw);
  const int64_t grp = blockIdx.x;
  const int64_t b = grp / g.gpt, gg = grp % g.gpt;
  const int t = threadIdx.x;
  const int64_t jt = gg * NT2 + t;
  const bool valid = jt < g.tpt;
  const int cnt = (int)min((int64_t)NT2, g.tpt - gg * NT2);
  bool ok = true;
  long long c0 = clock64();
  E acc;
  if (valid && !(MODE & 2))
    load(acc, tile_agg + (b * g.tpt + jt) * E::SZ, 1);
  else
    set_identity(acc);
  long long c1 = clock64();
#pragma unroll 1
  for (int d = 1; d < cnt; d <<= 1) {
    store(acc, sh + t, NT2);
    __syncthreads();
    if (t >= d && !(MODE & 1)) {
      if (MODE & 8) {
        E p;
        load(p, sh + t - d, NT2);
        combine(acc, p, acc, ok);
      } else {
        combine_g(acc, ElemRef<R, N>{sh + t - d, NT2}, acc, ok);
      }
    }
    __syncthreads();
  }
  long long c2 = clock64();
  if (valid && !(MODE & 2)) store(acc, tile_incl + (b * g.tpt + jt) * E::SZ, 1);
  if (t == cnt - 1) store(acc, group_agg + grp * E::SZ, 1);
  long long c3 = clock64();
  if (!ok) flag_node(flag, g.node0 + jt);
  if (t == 0 && grp == 0 && (MODE & 4)) { dbg[0] = c1 - c0; dbg[1] = c2 - c1; dbg[2] = c3 - c2; }
}
int main() {
  Geom g{};
  g.Nn = 10000001; g.node0 = 0; g.batch = 1; g.tpt = (g.Nn + 2047) / 2048; g.gpt = (g.tpt + NT2 - 1) / NT2;
  using E = Elem<double, 4>;
  std::vector<double> h(g.tpt * E::SZ);
  const double dt = 2048 * 5e-7;
  for (int64_t t = 0; t < g.tpt; ++t) {
    double* e = &h[t * E::SZ];
    int f = 0;
    for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) e[f++] = (i == j) + ((j == i + 2) ? -dt : 0.0);
    for (int i = 0; i < 4; ++i) e[f++] = 0.01 * i;
    for (int q = 0; q < 10; ++q) e[f++] = (q == 0 || q == 9 || q == 7 || q == 4) ? 4 * dt : 0;
    for (int i = 0; i < 4; ++i) e[f++] = 0.1 * (i + 1);
    for (int q = 0; q < 10; ++q) e[f++] = (q == 0 || q == 4) ? 100 * dt : 0;
  }
  double *agg, *incl, *gagg, *gcar; unsigned long long* flag;
  cudaMalloc(&agg, h.size() * 8); cudaMalloc(&incl, h.size() * 8); cudaMalloc(&gagg, g.gpt * E::SZ * 8);
  cudaMalloc(&gcar, g.gpt * 14 * 8); cudaMalloc(&flag, 8);
  cudaMemcpy(agg, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const int sm = E::SZ * NT2 * 8;
  cudaFuncSetAttribute(k_p1_tiles<double, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_p1_groups<double, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, E::SZ * NT3 * 8);
  cudaEvent_t a, b, c;
  cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c);
  for (int it = 0; it < 3; ++it) {
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) k_p1_tiles<double, 4><<<(unsigned)g.gpt, NT2, sm>>>(g, agg, incl, gagg, flag);
    cudaEventRecord(b);
    for (int r = 0; r < 20; ++r)
      k_p1_groups<double, 4><<<1, NT3, E::SZ * NT3 * 8>>>(g, gagg, nullptr, 0, nullptr, gcar, nullptr, flag);
    cudaEventRecord(c);
    cudaEventSynchronize(c);
    float t1, t2;
    cudaEventElapsedTime(&t1, a, b);
    cudaEventElapsedTime(&t2, b, c);
    printf("k_p1_tiles %.2f us/launch, k_p1_groups %.2f us/launch (%s)\n", t1 * 1e3 / 20, t2 * 1e3 / 20,
           cudaGetErrorString(cudaGetLastError()));
  }
  long long* dbg; cudaMalloc(&dbg, 64);
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(a);
      for (int r = 0; r < 20; ++r) kern<<<(unsigned)g.gpt, NT2, sm>>>(g, agg, incl, gagg, flag, dbg);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float t1;
      cudaEventElapsedTime(&t1, a, b);
      long long hd[3];
      cudaMemcpy(hd, dbg, 24, cudaMemcpyDeviceToHost);
      printf("%s %.2f us/launch  stages(cycles, CTA 0 thread 0): load %lld scan %lld store %lld\n", name, t1 * 1e3 / 20, hd[0], hd[1], hd[2]);
    }
  };
  run(k_tiles_probe<double, 4, 4>, "full   ");
  run(k_tiles_probe<double, 4, 5>, "nocomb ");
  run(k_tiles_probe<double, 4, 6>, "noglob ");
  run(k_tiles_probe<double, 4, 12>, "reg-p  ");
  return 0;
}
