// pmap_abi.cu -- C ABI (include/pmap.h) of the B200 parallel MAP library.
//
// Plan creation (model preprocessing, workspace), dispatch over the compiled
// (nx, ny, model kind, dtype) instantiations, host<->device staging, launch
// sequencing on the caller's stream, CUDA-graph capture of the nonlinear pass
// loop, device numeric flags, and the time-sharded (multi-GPU) protocol with
// NCCL all-gathers of chunk carries.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/pmap.h"
#include "pmap_kernels.cuh"
#include "pmap_tf.cuh"

#include "pmap_runner.cuh"

using namespace pmap;
using namespace pmap_rt;

namespace {

// One counting step of the device-side IEKS stop (map_solve_nonlinear, tol > 0):
// f[1] = max |dx| of the pass just run (bit pattern), f[2] = passes run, f[3] = that
// dmax; the WHILE condition (when h != 0) stays set while dmax >= tol and passes remain.
__global__ void k_ieks_decide(unsigned long long* f, double tol, int passes, cudaGraphConditionalHandle h,
                              int use_h) {
  const unsigned long long bits = f[1];
  double dmax;
  memcpy(&dmax, &bits, sizeof dmax);
  const unsigned long long run = f[2] + 1;
  f[2] = run;
  f[3] = bits;
  f[1] = 0;
  if (use_h) cudaGraphSetConditional(h, (dmax >= tol && run < (unsigned long long)passes) ? 1u : 0u);
}

static void launch_ieks_decide(cudaStream_t s, unsigned long long* f, double tol, int passes,
                               cudaGraphConditionalHandle h, bool use_h) {
  k_ieks_decide<<<1, 1, 0, s>>>(f, tol, passes, h, use_h ? 1 : 0);
}

// ------------------------------------------------------------- dispatch
template <typename R>
static Runner* dispatch_lti(int kr, int nx, int ny, int lowrank, const double* A, const double* b,
                            const double* C, const double* J, const double* K, const double* h0, const double* J0,
                            const double* h00, const double* Am, const double* bm, const double* Cm,
                            const double* U) {
  if (nx == 4 && ny == 2 && lowrank == 2) {
    // structural zeros (R-MASK): specialised kernels when the model's zeros cover the mask's
    uint32_t am = 0, um = 0;
    for (int i = 0; i < 16; ++i) am |= (A[i] != 0.0 ? 1u : 0u) << i;
    for (int i = 0; i < 8; ++i) um |= (U[i] != 0.0 ? 1u : 0u) << i;
    uint32_t sm = 0;  // packed entries where J or J0 is non-zero (R-SMASK)
    for (int k = 0; k < 10; ++k) sm |= ((J[k] != 0.0 || J0[k] != 0.0) ? 1u : 0u) << k;
    const char* nm = getenv("PMAP_NO_MASK");
    const char* nsm = getenv("PMAP_NO_SMASK");
    const bool masked = !(nm && nm[0] == '1') && (am & ~kWienerAMask) == 0 && (um & ~kWienerUMask) == 0;
    if (masked && !(nsm && nsm[0] == '1') && (sm & ~kWienerSMask) == 0)
      return kr == kKBig ? make_lti<R, 4, 2, kKBig, 2, kWienerAMask, kWienerUMask, kWienerSMask>(
                               A, b, C, J, K, h0, J0, h00, Am, bm, Cm, U)
                         : make_lti<R, 4, 2, kKSmall, 2, kWienerAMask, kWienerUMask, kWienerSMask>(
                               A, b, C, J, K, h0, J0, h00, Am, bm, Cm, U);
    if (masked)
      return kr == kKBig ? make_lti<R, 4, 2, kKBig, 2, kWienerAMask, kWienerUMask>(A, b, C, J, K, h0, J0, h00, Am,
                                                                                   bm, Cm, U)
                         : make_lti<R, 4, 2, kKSmall, 2, kWienerAMask, kWienerUMask>(A, b, C, J, K, h0, J0, h00,
                                                                                     Am, bm, Cm, U);
    return kr == kKBig ? make_lti<R, 4, 2, kKBig, 2, ~0u, ~0u>(A, b, C, J, K, h0, J0, h00, Am, bm, Cm, U)
                       : make_lti<R, 4, 2, kKSmall, 2, ~0u, ~0u>(A, b, C, J, K, h0, J0, h00, Am, bm, Cm, U);
  }
#define PM_CASE(NXV, NYV)                                                                                    \
  if (nx == NXV && ny == NYV)                                                                                \
    return kr == kKBig ? make_lti<R, NXV, NYV, kKBig, 0, ~0u, ~0u>(A, b, C, J, K, h0, J0, h00, Am, bm, Cm, U) \
                       : make_lti<R, NXV, NYV, kKSmall, 0, ~0u, ~0u>(A, b, C, J, K, h0, J0, h00, Am, bm, Cm, U);
  PM_SHAPES(PM_CASE)
#undef PM_CASE
  return nullptr;
}

template <typename R>
static Runner* dispatch_euler(int kr, int nx, int ny, int nsub, const double* A, const double* C, const double* J,
                              const double* b0, const double* h0, const double* Kb, const double* Ke,
                              const double* J0, const double* h00, const double* K0) {
  if (nsub != 10) return nullptr;  // compiled for the paper's n = 10 (build.py EULER_NSUB)
#define PM_CASE(NXV, NYV)                                                                                    \
  if (nx == NXV && ny == NYV)                                                                                \
    return kr == kKBig ? make_euler<R, NXV, NYV, 10, kKBig>(A, C, J, b0, h0, Kb, Ke, J0, h00, K0)            \
                       : make_euler<R, NXV, NYV, 10, kKSmall>(A, C, J, b0, h0, Kb, Ke, J0, h00, K0);
  PM_CASE(1, 1)
  PM_CASE(4, 2)
#undef PM_CASE
  return nullptr;
}

// Euler-block element of one grid interval (DESIGN.md R-EULER): NSUB explicit
// Euler substeps, in s, of the element ODEs P:416-427 (dA/ds sign corrected)
// from the boundary (I, 0, 0, 0, 0) of P:427, for an LTI model (F~ = -F, c~ = -c, Q~ = Q).
// b and eta are affine in the block's measurements: carried as nx x (1 + nsub*ny)
// matrices whose column 0 is the data-free part and column 1 + k*ny + a the coefficient
// of measurement component a at substep k (fine time t_{i-1} + (k+1) delta).
static void euler_block(int nx, int ny, int nsub, double dt, const double* F, const double* c, const double* Q,
                        const double* H, const double* r, const double* Ri, std::vector<double>& A,
                        std::vector<double>& C, std::vector<double>& J, std::vector<double>& B,
                        std::vector<double>& E) {
  const int M = 1 + nsub * ny;
  const double de = dt / nsub;
  auto I = [&](int i, int j) { return i == j ? 1.0 : 0.0; };
  A.assign(nx * nx, 0.0);
  for (int i = 0; i < nx; ++i) A[i * nx + i] = 1.0;
  C.assign(nx * nx, 0.0);
  J.assign(nx * nx, 0.0);
  B.assign(nx * M, 0.0);
  E.assign(nx * M, 0.0);
  std::vector<double> Ft(nx * nx), ct(nx), HRi(nx * ny, 0.0), HRH(nx * nx, 0.0), HRr(nx, 0.0);
  for (int i = 0; i < nx * nx; ++i) Ft[i] = -F[i];
  for (int i = 0; i < nx; ++i) ct[i] = c ? -c[i] : 0.0;
  for (int i = 0; i < nx; ++i)
    for (int a = 0; a < ny; ++a)
      for (int q = 0; q < ny; ++q) HRi[i * ny + a] += H[q * nx + i] * Ri[q * ny + a];
  for (int i = 0; i < nx; ++i) {
    for (int j = 0; j < nx; ++j)
      for (int a = 0; a < ny; ++a) HRH[i * nx + j] += HRi[i * ny + a] * H[a * nx + j];
    for (int a = 0; a < ny; ++a) HRr[i] += HRi[i * ny + a] * (r ? r[a] : 0.0);
  }
  auto mm = [&](const std::vector<double>& X, const double* Y, int m, std::vector<double>& Z) {  // Z = X Y, Y nx x m
    Z.assign(nx * m, 0.0);
    for (int i = 0; i < nx; ++i)
      for (int k = 0; k < nx; ++k)
        for (int j = 0; j < m; ++j) Z[i * m + j] += X[i * nx + k] * Y[k * m + j];
  };
  std::vector<double> AQ, JQ, dA(nx * nx), dB(nx * M), dC(nx * nx), dE(nx * M), dJ(nx * nx), t1, t2;
  for (int k = 0; k < nsub; ++k) {
    mm(A, Q, nx, AQ);
    mm(J, Q, nx, JQ);
    // dA/ds = A Q~ J - A F~
    mm(AQ, J.data(), nx, t1);
    mm(A, Ft.data(), nx, t2);
    for (int i = 0; i < nx * nx; ++i) dA[i] = t1[i] - t2[i];
    // db/ds = -A Q~ eta - A c~
    mm(AQ, E.data(), M, t1);
    for (int i = 0; i < nx * M; ++i) dB[i] = -t1[i];
    for (int i = 0; i < nx; ++i) {
      double s = 0;
      for (int j = 0; j < nx; ++j) s += A[i * nx + j] * ct[j];
      dB[i * M] -= s;
    }
    // dC/ds = -A Q~ A^T
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < nx; ++j) {
        double s = 0;
        for (int q = 0; q < nx; ++q) s += AQ[i * nx + q] * A[j * nx + q];
        dC[i * nx + j] = -s;
      }
    // deta/ds = J Q~ eta - F~^T eta - H^T R^-1 (y - r) + J c~
    mm(JQ, E.data(), M, t1);
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < M; ++j) {
        double s = t1[i * M + j];
        for (int q = 0; q < nx; ++q) s -= Ft[q * nx + i] * E[q * M + j];
        dE[i * M + j] = s;
      }
    for (int i = 0; i < nx; ++i) {
      double s = HRr[i];
      for (int j = 0; j < nx; ++j) s += J[i * nx + j] * ct[j];
      dE[i * M] += s;
      for (int a = 0; a < ny; ++a) dE[i * M + 1 + k * ny + a] -= HRi[i * ny + a];
    }
    // dJ/ds = J Q~ J - J F~ - F~^T J - H^T R^-1 H
    mm(JQ, J.data(), nx, t1);
    mm(J, Ft.data(), nx, t2);
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < nx; ++j) {
        double s = t1[i * nx + j] - t2[i * nx + j] - HRH[i * nx + j];
        for (int q = 0; q < nx; ++q) s -= Ft[q * nx + i] * J[q * nx + j];
        dJ[i * nx + j] = s;
      }
    // explicit Euler step backwards in s: X(s - delta) = X(s) - delta dX/ds
    for (int i = 0; i < nx * nx; ++i) {
      A[i] -= de * dA[i];
      C[i] -= de * dC[i];
      J[i] -= de * dJ[i];
    }
    for (int i = 0; i < nx * M; ++i) {
      B[i] -= de * dB[i];
      E[i] -= de * dE[i];
    }
  }
  (void)I;
}

// Forward-HJB element of the last m substeps of a block (R-REFINE, the first
// three equations): (A, b, C)(s, tau) integrated in reversed time tau by m explicit Euler
// steps of length de from the boundary (I, 0, 0), every right-hand side at the current
// state:  dA = -C M A + F~ A,  db = C H^T R^-1 (y - r) + F~ b + c~ - C M b,
// dC = -C M C + Q~ + F~ C + C F~^T  (M = H^T R^-1 H; F~ = -F, c~ = -c, Q~ = Q).  Step j
// reads the measurement of substep nsub - 1 - j (fine time t_i - j de).  b is affine in the
// block's measurements: B is nx x (1 + nsub*ny), column 0 data-free, column 1 + k*ny + a
// the coefficient of component a of substep k (the layout of euler_block).
static void hjb_block(int nx, int ny, int nsub, int m, double de, const double* F, const double* c,
                      const double* Q, const double* H, const double* r, const double* Ri, std::vector<double>& A,
                      std::vector<double>& C, std::vector<double>& B) {
  const int M = 1 + nsub * ny;
  A.assign(nx * nx, 0.0);
  for (int i = 0; i < nx; ++i) A[i * nx + i] = 1.0;
  C.assign(nx * nx, 0.0);
  B.assign(nx * M, 0.0);
  std::vector<double> Ft(nx * nx), ct(nx), HRi(nx * ny, 0.0), HRH(nx * nx, 0.0), HRr(nx, 0.0);
  for (int i = 0; i < nx * nx; ++i) Ft[i] = -F[i];
  for (int i = 0; i < nx; ++i) ct[i] = c ? -c[i] : 0.0;
  for (int i = 0; i < nx; ++i)
    for (int a = 0; a < ny; ++a)
      for (int q = 0; q < ny; ++q) HRi[i * ny + a] += H[q * nx + i] * Ri[q * ny + a];
  for (int i = 0; i < nx; ++i) {
    for (int j = 0; j < nx; ++j)
      for (int a = 0; a < ny; ++a) HRH[i * nx + j] += HRi[i * ny + a] * H[a * nx + j];
    for (int a = 0; a < ny; ++a) HRr[i] += HRi[i * ny + a] * (r ? r[a] : 0.0);
  }
  auto mm = [&](const double* X, int xc, const double* Y, int yc, std::vector<double>& Z) {  // Z = X Y
    Z.assign(nx * yc, 0.0);
    for (int i = 0; i < nx; ++i)
      for (int k = 0; k < xc; ++k)
        for (int j = 0; j < yc; ++j) Z[i * yc + j] += X[i * xc + k] * Y[k * yc + j];
  };
  std::vector<double> CM, t1, t2, dA(nx * nx), dB(nx * M), dC(nx * nx);
  for (int j = 0; j < m; ++j) {
    const int ks = nsub - 1 - j;
    mm(C.data(), nx, HRH.data(), nx, CM);
    mm(CM.data(), nx, A.data(), nx, t1);
    mm(Ft.data(), nx, A.data(), nx, t2);
    for (int i = 0; i < nx * nx; ++i) dA[i] = -t1[i] + t2[i];
    mm(Ft.data(), nx, B.data(), M, t1);
    mm(CM.data(), nx, B.data(), M, t2);
    for (int i = 0; i < nx * M; ++i) dB[i] = t1[i] - t2[i];
    for (int i = 0; i < nx; ++i) {
      double s = ct[i];
      for (int q = 0; q < nx; ++q) s -= C[i * nx + q] * HRr[q];
      dB[i * M] += s;
      for (int a = 0; a < ny; ++a) {
        double u = 0;
        for (int q = 0; q < nx; ++q) u += C[i * nx + q] * HRi[q * ny + a];
        dB[i * M + 1 + ks * ny + a] += u;
      }
    }
    mm(CM.data(), nx, C.data(), nx, t1);
    mm(Ft.data(), nx, C.data(), nx, t2);
    for (int i = 0; i < nx; ++i)
      for (int q = 0; q < nx; ++q) {
        double s = -t1[i * nx + q] + Q[i * nx + q] + t2[i * nx + q];
        for (int l = 0; l < nx; ++l) s += C[i * nx + l] * Ft[q * nx + l];  // C F~^T
        dC[i * nx + q] = s;
      }
    for (int i = 0; i < nx * nx; ++i) {
      A[i] += de * dA[i];
      C[i] += de * dC[i];
    }
    for (int i = 0; i < nx * M; ++i) B[i] += de * dB[i];
  }
  for (int i = 0; i < nx; ++i)
    for (int q = i + 1; q < nx; ++q) C[i * nx + q] = C[q * nx + i] = 0.5 * (C[i * nx + q] + C[q * nx + i]);
}

// Refinement tables of every k = 1 .. nsub - 1 (layout RefineTab in pmap_refine.cuh).
static std::vector<double> refine_tables(int nx, int ny, int nsub, double dt, const double* F, const double* c,
                                         const double* Q, const double* H, const double* r, const double* Ri) {
  const int NS = nx * (nx + 1) / 2, NR = nsub * ny, M = 1 + NR;
  const double de = dt / nsub;
  const int FR = 2 * nx * nx + 3 * NS + 3 * nx + 3 * nx * NR;
  std::vector<double> out((size_t)(nsub - 1) * FR, 0.0);
  std::vector<double> A, C, J, B, E, As, Cs, Bs, Cp(NS), Jp(NS), Csp(NS);
  auto sym_pack = [&](const double* Mf, double* P) {  // upper triangle, row-major
    for (int i = 0, k = 0; i < nx; ++i)
      for (int j = i; j < nx; ++j) P[k++] = 0.5 * (Mf[i * nx + j] + Mf[j * nx + i]);
  };
  for (int k = 1; k < nsub; ++k) {
    double* t = out.data() + (size_t)(k - 1) * FR;
    euler_block(nx, ny, k, k * de, F, c, Q, H, r, Ri, A, C, J, B, E);  // the first k substeps
    hjb_block(nx, ny, nsub, nsub - k, de, F, c, Q, H, r, Ri, As, Cs, Bs);
    sym_pack(C.data(), Cp.data());
    sym_pack(J.data(), Jp.data());
    sym_pack(Cs.data(), Csp.data());
    const int Mk = 1 + k * ny;  // euler_block's coefficient columns for k substeps
    double* p = t;
    for (int i = 0; i < nx * nx; ++i) *p++ = A[i];
    for (int i = 0; i < NS; ++i) *p++ = Cp[i];
    for (int i = 0; i < NS; ++i) *p++ = Jp[i];
    for (int i = 0; i < nx; ++i) *p++ = B[i * Mk];
    for (int i = 0; i < nx; ++i) *p++ = E[i * Mk];
    for (int i = 0; i < nx; ++i)
      for (int q = 0; q < NR; ++q) *p++ = q < k * ny ? B[i * Mk + 1 + q] : 0.0;
    for (int i = 0; i < nx; ++i)
      for (int q = 0; q < NR; ++q) *p++ = q < k * ny ? E[i * Mk + 1 + q] : 0.0;
    for (int i = 0; i < nx * nx; ++i) *p++ = As[i];
    for (int i = 0; i < NS; ++i) *p++ = Csp[i];
    for (int i = 0; i < nx; ++i) *p++ = Bs[i * M];
    for (int i = 0; i < nx; ++i)
      for (int q = 0; q < NR; ++q) *p++ = Bs[i * M + 1 + q];
  }
  return out;
}

template <typename R>
static Runner* dispatch_tv(int kr, int nx, int ny, const R* F, const R* c, const R* L, const R* Wm, const R* H,
                           const R* r, const R* Rm, const int64_t* str, int nw, double dt, const double* P0i,
                           const double* P0im0) {
#define PM_CASE(NXV, NYV)                                                                                    \
  if (nx == NXV && ny == NYV)                                                                                \
    return kr == kKBig ? make_tv<R, NXV, NYV, kKBig>(F, c, L, Wm, H, r, Rm, str, nw, dt, P0i, P0im0)         \
                       : make_tv<R, NXV, NYV, kKSmall>(F, c, L, Wm, H, r, Rm, str, nw, dt, P0i, P0im0);
  PM_SHAPES(PM_CASE)
#undef PM_CASE
  return nullptr;
}

template <typename R>
static Runner* dispatch_nl(int kr, int kind, double dt, double mu, double dv, const double* C, const double* Ri,
                           const double* P0i, const double* P0im0) {
  if (kind == MAP_NL_COORD_TURN)
    return kr == kKBig     ? make_nl<R, 5, 2, 1, kKBig>(dt, mu, dv, C, Ri, P0i, P0im0)
           : kr == kKTiny ? make_nl<R, 5, 2, 1, kKTiny>(dt, mu, dv, C, Ri, P0i, P0im0)
                          : make_nl<R, 5, 2, 1, kKSmall>(dt, mu, dv, C, Ri, P0i, P0im0);
  if (kind == MAP_NL_VAN_DER_POL)
    return kr == kKBig     ? make_nl<R, 2, 1, 2, kKBig>(dt, mu, dv, C, Ri, P0i, P0im0)
           : kr == kKTiny ? make_nl<R, 2, 1, 2, kKTiny>(dt, mu, dv, C, Ri, P0i, P0im0)
                          : make_nl<R, 2, 1, 2, kKSmall>(dt, mu, dv, C, Ri, P0i, P0im0);
  return nullptr;
}

// Run length: 2048-node tiles when they give >= 4 tiles per SM-slot-row of the GPU
// (148 SMs), else 512-node tiles so small problems still fill the machine.
static int choose_run_length(int64_t Nn, int64_t batch, bool nonlinear) {
  const char* e = getenv("PMAP_K");
  if (e && atoi(e) == kKSmall) return kKSmall;
  if (e && atoi(e) == kKBig) return kKBig;
  if (e && atoi(e) == kKTiny && nonlinear) return kKTiny;
  const int64_t tiles_big = batch * ((Nn + (int64_t)kNT * kKBig - 1) / ((int64_t)kNT * kKBig));
  if (nonlinear) {  // general combines: the chain length decides; tiny runs until the GPU is full
    const int64_t tiles_tiny = batch * ((Nn + (int64_t)kNT * kKTiny - 1) / ((int64_t)kNT * kKTiny));
    return tiles_tiny <= 16 * 148 ? kKTiny : (tiles_big >= 4 * 148 ? kKBig : kKSmall);
  }
  return tiles_big >= 4 * 148 ? kKBig : kKSmall;
}

static bool is_device_ptr(const void* ptr) {
  if (!ptr) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static map_status check_flag(PlanState& p) {
  unsigned long long f = ULLONG_MAX;
  cudaError_t e = cudaMemcpyAsync(&f, p.dflag, sizeof f, cudaMemcpyDeviceToHost, p.stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p.stream);
  if (e != cudaSuccess) return cuda_fail(p, e, "map_sync");
  if (f != ULLONG_MAX) {
    char buf[160];
    snprintf(buf, sizeof buf, "numeric failure (non-finite value or zero pivot) at or after node %llu", f);
    p.err = buf;
    const unsigned long long reset = ULLONG_MAX;
    cudaMemcpyAsync(p.dflag, &reset, sizeof reset, cudaMemcpyHostToDevice, p.stream);
    cudaStreamSynchronize(p.stream);
    return MAP_E_NUMERIC;
  }
  return MAP_OK;
}

// Run `body` (which launches one solve on p.stream) through the plan's graph cache:
// the first call with a key runs eagerly (it also sizes any lazily allocated scratch),
// the second captures the launches (kernels, fork/join events, NCCL all-gathers) into a
// CUDA graph on a private stream, later calls replay it on p.stream.  Profiling or
// PMAP_NO_GRAPH=1 run eagerly; a failed capture falls back to eager launches for good.
template <class Body>
static map_status graph_run(PlanState& p, const void* const (&key)[6], Body body) {
  const char* ng = getenv("PMAP_NO_GRAPH");
  if (p.prof || (ng && ng[0] == '1')) {
    body();
    return MAP_OK;
  }
  PlanState::GraphEntry* e = nullptr;
  for (auto& g : p.lgraphs)
    if (memcmp(g.key, key, sizeof g.key) == 0) e = &g;
  if (!e) {
    if (p.lgraphs.size() >= 8) {  // bounded cache: drop the oldest entry
      if (p.lgraphs.front().exec) cudaGraphExecDestroy(p.lgraphs.front().exec);
      p.lgraphs.erase(p.lgraphs.begin());
    }
    PlanState::GraphEntry ne{};
    memcpy(ne.key, key, sizeof ne.key);
    p.lgraphs.push_back(ne);
    body();
    return MAP_OK;
  }
  if (e->no_graph) {
    body();
    return MAP_OK;
  }
  if (!e->exec) {
    cudaStream_t cs;
    PM_CK(p, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaStream_t saved = p.stream;
    p.stream = cs;
    const int64_t l0 = p.launches;
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      body();
      ok = cudaStreamEndCapture(cs, &graph) == cudaSuccess && p.err.empty();
    }
    p.stream = saved;
    cudaStreamDestroy(cs);
    if (ok) ok = cudaGraphInstantiate(&e->exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {  // capture unsupported here: eager from now on
      cudaGetLastError();
      e->exec = nullptr;
      e->no_graph = true;
      p.err.clear();
      p.launches = l0;
      body();
      return MAP_OK;
    }
    e->launches = p.launches - l0;
    p.launches = l0;
  }
  PM_CK(p, cudaGraphLaunch(e->exec, p.stream));
  p.launches += e->launches;
  return MAP_OK;
}

static map_status ensure_stage(PlanState& p, void** buf, size_t* have, size_t need) {
  if (*have >= need) return MAP_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *have = 0;
  PM_CK(p, cudaMalloc(buf, need));
  *have = need;
  return MAP_OK;
}

}  // namespace

struct map_plan_s : PlanState {};

// NVTX range around every ABI entry point (host-side timeline of plans, solves and shard
// phases in Nsight tools; header-only NVTX3, a no-op when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

extern "C" {

const char* map_version(void) { return "pmap 0.1 (sm_100a)"; }

const char* map_status_string(map_status s) {
  switch (s) {
    case MAP_OK: return "ok";
    case MAP_E_ARG: return "invalid argument";
    case MAP_E_UNSUPPORTED: return "unsupported configuration";
    case MAP_E_CUDA: return "CUDA error";
    case MAP_E_NCCL: return "NCCL error";
    case MAP_E_NUMERIC: return "numeric failure";
    case MAP_E_DIVERGED: return "iteration did not converge";
  }
  return "unknown status";
}

static int hi_prio() {
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  return hi;
}

map_status map_plan(const map_plan_desc* desc, const map_linear_model* lin, const map_nl_model* nl,
                    map_plan_t* out) {
  NvtxRange nvtx_("pmap:map_plan");
  if (!desc || !out || (!lin) == (!nl)) return MAP_E_ARG;
  *out = nullptr;
  map_plan_desc dd = *desc;
  if (dd.nx < 1 || dd.ny < 1 || dd.nw < 1 || dd.nw > dd.nx || dd.T < 1 || dd.batch < 1 || !(dd.tf > dd.t0) ||
      (dd.dtype != MAP_F64 && dd.dtype != MAP_F32) || dd.world < 1 || dd.rank < 0 || dd.rank >= dd.world)
    return MAP_E_ARG;
  if ((dd.flags & MAP_FLAG_BATCH_SHARD) && dd.world > 1) {
    // BATCH shard mode: rank r owns trajectories [r B / world, (r + 1) B / world) and solves
    // them as an independent single-GPU plan (no exchange, no communicator)
    const int64_t b0 = dd.batch * dd.rank / dd.world, b1 = dd.batch * (dd.rank + 1) / dd.world;
    if (b1 <= b0) return MAP_E_ARG;  // more ranks than trajectories
    dd.batch = b1 - b0;
    dd.rank = 0;
    dd.world = 1;
    dd.nccl_comm = nullptr;
  }
  const map_plan_desc& d = dd;
  if (d.substeps < 0 || (d.substeps > 1 && (!lin || d.world != 1))) return MAP_E_ARG;
  std::unique_ptr<map_plan_s> p(new map_plan_s());
  p->d = d;
  p->ny_row = d.ny;
  p->stream = static_cast<cudaStream_t>(d.stream);
  {
    const char* fs = getenv("PMAP_FORCE_SHARD");
    p->force_shard = fs && fs[0] == '1' && d.nccl_comm;
    const char* nr = getenv("PMAP_NO_P2REC");
    p->no_rec = nr && nr[0] == '1';
    const char* nlb = getenv("PMAP_NO_LB");
    p->no_lb = nlb && nlb[0] == '1';
    p->mixed = (d.flags & MAP_FLAG_MIXED) != 0 && d.dtype == MAP_F64;
    const char* lbs = getenv("PMAP_LB_STRESS");
    p->lb_stress = (lbs && lbs[0] == '1') ? 1 : 0;
  }
  const int nx = d.nx, ny = d.ny, nw = d.nw;
  const int NS = nx * (nx + 1) / 2;
  const double dt = (d.tf - d.t0) / (double)d.T;
  const bool f32 = d.dtype == MAP_F32;
  // time shard geometry
  const int64_t Ntot = d.T + 1;
  const int64_t a0 = (int64_t)((__int128)d.rank * Ntot / d.world);
  const int64_t a1 = (int64_t)((__int128)(d.rank + 1) * Ntot / d.world);
  Geom& g = p->g;
  g.Nn = a1 - a0;
  g.node0 = a0;
  g.batch = d.batch;
  const int kr = choose_run_length(g.Nn, g.batch, nl != nullptr);
  const int64_t L = (int64_t)kNT * kr;
  g.tpt = (g.Nn + L - 1) / L;
  g.gpt = (g.tpt + NT2 - 1) / NT2;
  if (g.Nn < 1) return MAP_E_ARG;

  auto sym_pack = [&](const double* M, double* P) {
    for (int i = 0, k = 0; i < nx; ++i)
      for (int j = i; j < nx; ++j, ++k) P[k] = 0.5 * (M[i * nx + j] + M[j * nx + i]);
  };
  const double* m0 = lin ? lin->m0 : nl->m0;
  const double* P0 = lin ? lin->P0 : nl->P0;
  if (!m0 || !P0 || !h_is_finite(m0, nx) || !h_is_finite(P0, nx * nx)) return MAP_E_ARG;
  std::vector<double> P0i(nx * nx), P0ip(NS), P0im0(nx, 0.0);
  if (!h_inv(nx, P0, P0i.data())) return MAP_E_ARG;
  sym_pack(P0i.data(), P0ip.data());
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < nx; ++j) P0im0[i] += P0i[i * nx + j] * m0[j];
  p->m0_host = new double[nx];
  memcpy(p->m0_host, m0, sizeof(double) * nx);

  Runner* rn = nullptr;
  if (lin) {
    if (!lin->F || !lin->L || !lin->W || !lin->H || !lin->R) return MAP_E_ARG;
    const bool tv = lin->sF || lin->sc || lin->sL || lin->sW || lin->sH || lin->sr || lin->sR;
    if (tv && d.substeps > 1) {
      // Euler blocks are built for time-invariant models only (R-EULER): the kernels would
      // read y rows of substeps * ny values as [T+1][ny] and return wrong trajectories
      return MAP_E_UNSUPPORTED;
    }
    if (!tv && d.substeps > 1) {  // paper-faithful Euler blocks of d.substeps substeps
      p->kind = Kind::LTI;
      p->euler = true;
      const int nsub = d.substeps;
      const double de = dt / nsub;
      std::vector<double> Q(nx * nx, 0.0), Ri(ny * ny), A, C, J, B, E, Cp(NS), Jp(NS);
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nx; ++j)
          for (int a = 0; a < nw; ++a)
            for (int c = 0; c < nw; ++c) Q[i * nx + j] += lin->L[i * nw + a] * lin->W[a * nw + c] * lin->L[j * nw + c];
      if (!h_inv(ny, lin->R, Ri.data())) return MAP_E_ARG;
      euler_block(nx, ny, nsub, dt, lin->F, lin->c, Q.data(), lin->H, lin->r, Ri.data(), A, C, J, B, E);
      sym_pack(C.data(), Cp.data());
      sym_pack(J.data(), Jp.data());
      const int M = 1 + nsub * ny, NR = nsub * ny;
      std::vector<double> b0(nx), h0(nx), Kb(nx * NR), Ke(nx * NR), K0(nx * ny, 0.0), J0f(nx * nx, 0.0), J0(NS),
          h00(nx);
      for (int i = 0; i < nx; ++i) {
        b0[i] = B[i * M];
        h0[i] = E[i * M];
        for (int k = 0; k < NR; ++k) {
          Kb[i * NR + k] = B[i * M + 1 + k];
          Ke[i * NR + k] = E[i * M + 1 + k];
        }
      }
      // node 0: prior and the measurement at t_0 with the fine weight delta
      for (int i = 0; i < nx; ++i)
        for (int a = 0; a < ny; ++a)
          for (int q = 0; q < ny; ++q) K0[i * ny + a] += de * lin->H[q * nx + i] * Ri[q * ny + a];
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nx; ++j) {
          J0f[i * nx + j] = P0i[i * nx + j];
          for (int a = 0; a < ny; ++a) J0f[i * nx + j] += K0[i * ny + a] * lin->H[a * nx + j];
        }
      sym_pack(J0f.data(), J0.data());
      for (int i = 0; i < nx; ++i) {
        h00[i] = P0im0[i];
        for (int a = 0; a < ny; ++a) h00[i] -= K0[i * ny + a] * (lin->r ? lin->r[a] : 0.0);
      }
      p->ny_row = NR;
      p->refine_host = refine_tables(nx, ny, nsub, dt, lin->F, lin->c, Q.data(), lin->H, lin->r, Ri.data());
      rn = f32 ? dispatch_euler<float>(kr, nx, ny, nsub, A.data(), Cp.data(), Jp.data(), b0.data(), h0.data(),
                                       Kb.data(), Ke.data(), J0.data(), h00.data(), K0.data())
               : dispatch_euler<double>(kr, nx, ny, nsub, A.data(), Cp.data(), Jp.data(), b0.data(), h0.data(),
                                        Kb.data(), Ke.data(), J0.data(), h00.data(), K0.data());
    } else if (!tv) {
      p->kind = Kind::LTI;
      std::vector<double> A(nx * nx), b(nx, 0.0), Q(nx * nx, 0.0), Cp(NS), Ri(ny * ny), K(nx * ny, 0.0),
          Jf(nx * nx, 0.0), Jp(NS), h0(nx, 0.0), J0(NS), h00(nx);
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nx; ++j) A[i * nx + j] = (i == j ? 1.0 : 0.0) - dt * lin->F[i * nx + j];
      for (int i = 0; i < nx; ++i) b[i] = lin->c ? -dt * lin->c[i] : 0.0;
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nx; ++j)
          for (int a = 0; a < nw; ++a)
            for (int c = 0; c < nw; ++c) Q[i * nx + j] += lin->L[i * nw + a] * lin->W[a * nw + c] * lin->L[j * nw + c];
      for (int i = 0; i < nx * nx; ++i) Q[i] *= dt;
      sym_pack(Q.data(), Cp.data());
      if (!h_inv(ny, lin->R, Ri.data())) return MAP_E_ARG;
      for (int i = 0; i < nx; ++i)
        for (int k = 0; k < ny; ++k)
          for (int a = 0; a < ny; ++a) K[i * ny + k] += dt * lin->H[a * nx + i] * Ri[a * ny + k];
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nx; ++j)
          for (int k = 0; k < ny; ++k) Jf[i * nx + j] += K[i * ny + k] * lin->H[k * nx + j];
      sym_pack(Jf.data(), Jp.data());
      for (int i = 0; i < nx; ++i)
        for (int k = 0; k < ny; ++k) h0[i] -= K[i * ny + k] * (lin->r ? lin->r[k] : 0.0);
      for (int k = 0; k < NS; ++k) J0[k] = P0ip[k] + Jp[k];
      for (int i = 0; i < nx; ++i) h00[i] = P0im0[i] + h0[i];
      // mirrored transition (R-TF): Am = A^-1, bm = -Am b, Cm = Am (dt Q) Am^T
      std::vector<double> Am(nx * nx), bm(nx, 0.0), T1(nx * nx, 0.0), Cmf(nx * nx, 0.0), Cmp(NS);
      if (!h_inv(nx, A.data(), Am.data())) return MAP_E_ARG;
      for (int i = 0; i < nx; ++i)
        for (int k = 0; k < nx; ++k) bm[i] -= Am[i * nx + k] * b[k];
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nx; ++j)
          for (int k = 0; k < nx; ++k) T1[i * nx + j] += Am[i * nx + k] * Q[k * nx + j];
      for (int i = 0; i < nx; ++i)
        for (int j = 0; j < nx; ++j)
          for (int k = 0; k < nx; ++k) Cmf[i * nx + j] += T1[i * nx + k] * Am[j * nx + k];
      sym_pack(Cmf.data(), Cmp.data());
      // low-rank diffusion factor U = sqrt(dt) L chol(W) (dt Q = U U^T), R-LOWRANK
      std::vector<double> Lw(nw * nw, 0.0), U(nx * nw, 0.0);
      bool wpd = true;
      for (int j = 0; j < nw && wpd; ++j) {
        double d = lin->W[j * nw + j];
        for (int k = 0; k < j; ++k) d -= Lw[j * nw + k] * Lw[j * nw + k];
        if (!(d > 0)) { wpd = false; break; }
        Lw[j * nw + j] = std::sqrt(d);
        for (int i = j + 1; i < nw; ++i) {
          double t = lin->W[i * nw + j];
          for (int k = 0; k < j; ++k) t -= Lw[i * nw + k] * Lw[j * nw + k];
          Lw[i * nw + j] = t / Lw[j * nw + j];
        }
      }
      for (int i = 0; i < nx; ++i)
        for (int a = 0; a < nw; ++a) {
          double t = 0;
          for (int k = 0; k < nw; ++k) t += lin->L[i * nw + k] * Lw[k * nw + a];
          U[i * nw + a] = std::sqrt(dt) * t;
        }
      const char* nlr = getenv("PMAP_NO_LOWRANK");
      const int lowrank = (wpd && nw < nx && !(nlr && nlr[0] == '1')) ? nw : 0;
      rn = f32 ? dispatch_lti<float>(kr, nx, ny, lowrank, A.data(), b.data(), Cp.data(), Jp.data(), K.data(),
                                     h0.data(), J0.data(), h00.data(), Am.data(), bm.data(), Cmp.data(), U.data())
               : dispatch_lti<double>(kr, nx, ny, lowrank, A.data(), b.data(), Cp.data(), Jp.data(), K.data(),
                                      h0.data(), J0.data(), h00.data(), Am.data(), bm.data(), Cmp.data(), U.data());
    } else {
      p->kind = Kind::TV;
      // copy node arrays (global node indexing) to the device in the plan dtype
      const int64_t cnt[7] = {(int64_t)nx * nx, nx, (int64_t)nx * nw, (int64_t)nw * nw, (int64_t)ny * nx, ny,
                              (int64_t)ny * ny};
      const double* src[7] = {lin->F, lin->c, lin->L, lin->W, lin->H, lin->r, lin->R};
      const int64_t str[7] = {lin->sF, lin->sc, lin->sL, lin->sW, lin->sH, lin->sr, lin->sR};
      size_t total = 0;
      int64_t len[7];
      for (int k = 0; k < 7; ++k) {
        if (str[k] && str[k] != cnt[k]) return MAP_E_ARG;
        len[k] = src[k] ? (str[k] ? (d.T + 1) * cnt[k] : cnt[k]) : 0;
        total += len[k];
      }
      const size_t es = f32 ? 4 : 8;
      if (cudaMalloc(&p->dev_tv, total * es + 64) != cudaSuccess) return MAP_E_CUDA;
      size_t off = 0;
      const void* dptr[7];
      for (int k = 0; k < 7; ++k) {
        if (!src[k]) { dptr[k] = nullptr; continue; }
        char* dst = static_cast<char*>(p->dev_tv) + off * es;
        if (f32) {
          std::vector<float> tmp(src[k], src[k] + len[k]);
          cudaMemcpy(dst, tmp.data(), len[k] * 4, cudaMemcpyHostToDevice);
        } else {
          cudaMemcpy(dst, src[k], len[k] * 8, cudaMemcpyHostToDevice);
        }
        dptr[k] = dst;
        off += len[k];
      }
      if (f32)
        rn = dispatch_tv<float>(kr, nx, ny, (const float*)dptr[0], (const float*)dptr[1], (const float*)dptr[2],
                                (const float*)dptr[3], (const float*)dptr[4], (const float*)dptr[5],
                                (const float*)dptr[6], str, nw, dt, P0ip.data(), P0im0.data());
      else
        rn = dispatch_tv<double>(kr, nx, ny, (const double*)dptr[0], (const double*)dptr[1], (const double*)dptr[2],
                                 (const double*)dptr[3], (const double*)dptr[4], (const double*)dptr[5],
                                 (const double*)dptr[6], str, nw, dt, P0ip.data(), P0im0.data());
    }
  } else {
    p->kind = Kind::NL;
    p->nl_kind = nl->kind;
    if (!nl->L || !nl->W || !nl->R) return MAP_E_ARG;
    if (nl->kind == MAP_NL_COORD_TURN && (nx != 5 || ny != 2)) return MAP_E_ARG;
    if (nl->kind == MAP_NL_VAN_DER_POL && (nx != 2 || ny != 1 || nl->nparams < 1 || !nl->params)) return MAP_E_ARG;
    std::vector<double> Q(nx * nx, 0.0), Cp(NS), Ri(ny * ny);
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < nx; ++j)
        for (int a = 0; a < nw; ++a)
          for (int c = 0; c < nw; ++c) Q[i * nx + j] += nl->L[i * nw + a] * nl->W[a * nw + c] * nl->L[j * nw + c];
    for (int i = 0; i < nx * nx; ++i) Q[i] *= dt;
    sym_pack(Q.data(), Cp.data());
    if (!h_inv(ny, nl->R, Ri.data())) return MAP_E_ARG;
    const double mu = (nl->nparams >= 1 && nl->params) ? nl->params[0] : 0.0;
    // Van der Pol params[1] != 0: keep the Onsager--Machlup divergence term
    const double dv = (nl->kind == MAP_NL_VAN_DER_POL && nl->nparams >= 2 && nl->params) ? nl->params[1] : 0.0;
    rn = f32 ? dispatch_nl<float>(kr, nl->kind, dt, mu, dv, Cp.data(), Ri.data(), P0ip.data(), P0im0.data())
             : dispatch_nl<double>(kr, nl->kind, dt, mu, dv, Cp.data(), Ri.data(), P0ip.data(), P0im0.data());
  }
  if (!rn) return MAP_E_UNSUPPORTED;
  p->runner.reset(rn);
  p->elem_real = rn->sizeof_real();
  const bool ptime = getenv("PMAP_PLAN_TIMING") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto t0 = tnow();
  auto tlog = [&](const char* what) {
    if (ptime) {
      cudaDeviceSynchronize();
      fprintf(stderr, "[pmap plan] %-28s %8.2f ms\n", what,
              std::chrono::duration<double, std::milli>(tnow() - t0).count());
      t0 = tnow();
    }
  };
  tlog("model preprocessing");
  rn->set_attrs();
  tlog("set_attrs");
  if (!rn->prepare(*p)) {
    cudaGetLastError();
    p->err = "plan preparation (LTI tables) failed";
    return MAP_E_CUDA;
  }
  // workspace
  p->ws_tf = (p->kind != Kind::NL) && d.world == 1;
  tlog("prepare (LTI + look-back tables)");
  p->ws_bytes = rn->ws_bytes(g, p->ws_tf);
  if (cudaMalloc(&p->ws, p->ws_bytes) != cudaSuccess) {
    cudaGetLastError();
    p->err = "workspace allocation failed";
    return MAP_E_CUDA;
  }
  if (cudaMalloc(&p->dflag, 4 * sizeof(unsigned long long)) != cudaSuccess) return MAP_E_CUDA;
  const unsigned long long init[4] = {ULLONG_MAX, 0ull, 0ull, 0ull};
  cudaMemcpy(p->dflag, init, sizeof init, cudaMemcpyHostToDevice);
  if (p->kind == Kind::NL) {
    const size_t xb = (size_t)g.batch * g.Nn * nx * p->elem_real;
    if (cudaMalloc(&p->xbuf[0], xb) != cudaSuccess || cudaMalloc(&p->xbuf[1], xb) != cudaSuccess) return MAP_E_CUDA;
    if (cudaMalloc(&p->m0_dev, nx * p->elem_real) != cudaSuccess) return MAP_E_CUDA;
    if (f32) {
      std::vector<float> t(m0, m0 + nx);
      cudaMemcpy(p->m0_dev, t.data(), nx * 4, cudaMemcpyHostToDevice);
    } else {
      cudaMemcpy(p->m0_dev, m0, nx * 8, cudaMemcpyHostToDevice);
    }
  }
  if (cudaStreamCreateWithFlags(&p->stream2, cudaStreamNonBlocking) != cudaSuccess ||
      // boundary-tile forks at the highest priority: their CTAs are dispatched ahead of
      // the interior reduce's pending CTAs, keeping the short serial chain off the
      // critical path of pass 1
      cudaStreamCreateWithPriority(&p->stream3, cudaStreamNonBlocking, hi_prio()) != cudaSuccess ||
      cudaStreamCreateWithPriority(&p->stream4, cudaStreamNonBlocking, hi_prio()) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_edge0, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_edge1, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_edge2, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_edge3, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess)
    return MAP_E_CUDA;
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    p->err = cudaGetErrorString(e);
    return MAP_E_CUDA;
  }
  tlog("workspace, streams, events");
  *out = p.release();
  return MAP_OK;
}

void map_plan_destroy(map_plan_t p) {
  delete p;  // ~PlanState synchronises the stream and frees everything the plan owns
}

// Resolve y (input) and x (output) to device buffers, staging host memory.
struct IoGuard {
  PlanState& p;
  const void* y_host = nullptr;
  void* x_host = nullptr;
  size_t ybytes = 0, xbytes = 0;
  bool blocking = false;
  explicit IoGuard(PlanState& pp) : p(pp) {}
};

static map_status stage_in(PlanState& p, const void* y, size_t ybytes, const void** ydev, bool* blocking) {
  if (is_device_ptr(y)) {
    *ydev = y;
    return MAP_OK;
  }
  *blocking = true;
  map_status st = ensure_stage(p, &p.stage_y, &p.stage_y_bytes, ybytes);
  if (st) return st;
  PM_CK(p, cudaMemcpyAsync(p.stage_y, y, ybytes, cudaMemcpyHostToDevice, p.stream));
  *ydev = p.stage_y;
  return MAP_OK;
}

static map_status stage_out_buf(PlanState& p, void* x, size_t xbytes, void** buf, size_t* have, void** xdev,
                                bool* blocking) {
  if (!x) {
    *xdev = nullptr;
    return MAP_OK;
  }
  if (is_device_ptr(x)) {
    *xdev = x;
    return MAP_OK;
  }
  *blocking = true;
  map_status st = ensure_stage(p, buf, have, xbytes);
  if (st) return st;
  *xdev = *buf;
  return MAP_OK;
}

static map_status finish(PlanState& p, bool blocking, const std::vector<std::pair<void*, std::pair<void*, size_t>>>& outs) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(p, e, "kernel launch");
  if (!p.err.empty() && p.err.rfind("nccl", 0) == 0) return MAP_E_NCCL;
  if (p.err.rfind("ncclAllGather", 0) == 0) return MAP_E_NCCL;
  for (auto& o : outs)
    if (o.first != o.second.first) PM_CK(p, cudaMemcpyAsync(o.first, o.second.first, o.second.second,
                                                           cudaMemcpyDeviceToHost, p.stream));
  if (blocking) return check_flag(p);
  return MAP_OK;
}

map_status map_solve_linear(map_plan_t p, const void* y, void* x_map, void* filt_m, void* filt_P) {
  NvtxRange nvtx_("pmap:map_solve_linear");
  if (!p || !y || !x_map) return MAP_E_ARG;
  if (p->kind == Kind::NL) {
    p->err = "map_solve_linear called on a nonlinear plan";
    return MAP_E_ARG;
  }
  p->err.clear();
  p->launches = 0;
  const Geom& g = p->g;
  const size_t es = p->elem_real;
  const int nx = p->d.nx, ny = p->d.ny;
  const size_t yb = (size_t)g.batch * g.Nn * p->ny_row * es, xb = (size_t)g.batch * g.Nn * nx * es;
  const size_t mb = xb, Pb = (size_t)g.batch * g.Nn * (nx * (nx + 1) / 2) * es;
  bool blocking = false;
  const void* yd;
  void *xd, *md, *Pd;
  map_status st = stage_in(*p, y, yb, &yd, &blocking);
  if (!st) st = stage_out_buf(*p, x_map, xb, &p->stage_x, &p->stage_x_bytes, &xd, &blocking);
  if (!st && (filt_m || filt_P)) {
    // staging for optional outputs shares one aux buffer: [m | P]
    const bool mh = filt_m && !is_device_ptr(filt_m), Ph = filt_P && !is_device_ptr(filt_P);
    if (mh || Ph) {
      st = ensure_stage(*p, &p->stage_aux, &p->stage_aux_bytes, mb + Pb);
      blocking = true;
    }
    md = filt_m ? (mh ? p->stage_aux : filt_m) : nullptr;
    Pd = filt_P ? (Ph ? static_cast<char*>(p->stage_aux) + mb : filt_P) : nullptr;
  } else {
    md = Pd = nullptr;
  }
  if (st) return st;
  if (p->d.world > 1 && !p->d.nccl_comm) {
    p->err = "time-sharded plan without an NCCL communicator: drive the exchange with map_shard_phase";
    return MAP_E_NCCL;
  }
  {
    const void* key[6] = {yd, xd, md, Pd, nullptr, "rts"};
    map_status gs = graph_run(*p, key, [&] { p->runner->rts(*p, yd, nullptr, xd, md, Pd); });
    if (gs) return gs;
  }
  std::vector<std::pair<void*, std::pair<void*, size_t>>> outs;
  outs.push_back({x_map, {xd, xb}});
  if (filt_m) outs.push_back({filt_m, {md, mb}});
  if (filt_P) outs.push_back({filt_P, {Pd, Pb}});
  return finish(*p, blocking, outs);
}

map_status map_solve_linear_fine(map_plan_t p, const void* y, void* x_fine) {
  NvtxRange nvtx_("pmap:map_solve_linear_fine");
  if (!p || !y || !x_fine) return MAP_E_ARG;
  if (p->kind == Kind::NL || !p->euler) {
    p->err = "map_solve_linear_fine needs a linear plan with Euler blocks (substeps > 1)";
    return MAP_E_UNSUPPORTED;
  }
  if (p->d.world > 1) {
    p->err = "map_solve_linear_fine: single-GPU plans only";
    return MAP_E_UNSUPPORTED;
  }
  p->err.clear();
  p->launches = 0;
  const Geom& g = p->g;
  const size_t es = p->elem_real;
  const int nx = p->d.nx, NS = nx * (nx + 1) / 2;
  const int64_t T = g.Nn - 1, Nf = (int64_t)p->d.substeps * T + 1;
  const size_t yb = (size_t)g.batch * g.Nn * p->ny_row * es, xfb = (size_t)g.batch * Nf * nx * es;
  const size_t xbb = (size_t)g.batch * g.Nn * nx * es, Pbb = (size_t)g.batch * g.Nn * NS * es;
  bool blocking = false;
  const void* yd;
  void* xd;
  map_status st = stage_in(*p, y, yb, &yd, &blocking);
  if (!st) st = stage_out_buf(*p, x_fine, xfb, &p->stage_x, &p->stage_x_bytes, &xd, &blocking);
  if (st) return st;
  if (p->fine_ws_bytes < 2 * xbb + Pbb) {  // block x, filter m, filter P
    cudaFree(p->fine_ws);
    p->fine_ws = nullptr;
    p->fine_ws_bytes = 0;
    if (cudaMalloc(&p->fine_ws, 2 * xbb + Pbb) != cudaSuccess) {
      p->err = "map_solve_linear_fine: workspace allocation failed";
      return MAP_E_CUDA;
    }
    p->fine_ws_bytes = 2 * xbb + Pbb;
  }
  char* w = static_cast<char*>(p->fine_ws);
  void *xbd = w, *md = w + xbb, *Pd = w + 2 * xbb;
  bool ok = true;
  {
    const void* key[6] = {yd, xd, nullptr, nullptr, nullptr, "fine"};
    map_status gs = graph_run(*p, key, [&] { ok = p->runner->refine(*p, yd, xbd, md, Pd, xd); });
    if (gs) return gs;
  }
  if (!ok) return MAP_E_UNSUPPORTED;
  std::vector<std::pair<void*, std::pair<void*, size_t>>> outs;
  outs.push_back({x_fine, {xd, xfb}});
  return finish(*p, blocking, outs);
}
map_status map_solve_linear_cov(map_plan_t p, const void* y, void* x_map, void* smooth_P) {
  NvtxRange nvtx_("pmap:map_solve_linear_cov");
  if (!p || !y || !x_map || !smooth_P) return MAP_E_ARG;
  if (p->kind == Kind::NL || p->euler) {
    p->err = "map_solve_linear_cov needs a linear plan without Euler blocks";
    return MAP_E_ARG;
  }
  p->err.clear();
  p->launches = 0;
  const Geom& g = p->g;
  const size_t es = p->elem_real;
  const size_t yb = (size_t)g.batch * g.Nn * p->ny_row * es, xb = (size_t)g.batch * g.Nn * p->d.nx * es;
  const size_t Pb = (size_t)g.batch * g.Nn * (p->d.nx * (p->d.nx + 1) / 2) * es;
  bool blocking = false;
  const void* yd;
  void *xd, *Pd = nullptr;
  map_status st = stage_in(*p, y, yb, &yd, &blocking);
  if (!st) st = stage_out_buf(*p, x_map, xb, &p->stage_x, &p->stage_x_bytes, &xd, &blocking);
  if (!st) st = stage_out_buf(*p, smooth_P, Pb, &p->stage_aux, &p->stage_aux_bytes, &Pd, &blocking);
  if (st) return st;
  bool ok = true;
  {
    const void* key[6] = {yd, xd, Pd, nullptr, nullptr, "cov"};
    map_status gs = graph_run(*p, key, [&] { ok = p->runner->rts_cov(*p, yd, xd, Pd); });
    if (gs) return gs;
  }
  if (!ok) return MAP_E_UNSUPPORTED;
  std::vector<std::pair<void*, std::pair<void*, size_t>>> outs;
  outs.push_back({x_map, {xd, xb}});
  outs.push_back({smooth_P, {Pd, Pb}});
  return finish(*p, blocking, outs);
}

map_status map_two_filter(map_plan_t p, const void* y, void* x_map, void* smooth_P) {
  NvtxRange nvtx_("pmap:map_two_filter");
  if (!p || !y || !x_map) return MAP_E_ARG;
  if (p->euler) {
    p->err = "two-filter is not available with Euler blocks (the block element mixes dynamics and measurements)";
    return MAP_E_UNSUPPORTED;
  }
  if (p->kind == Kind::NL || p->d.world != 1) {
    p->err = "map_two_filter needs a linear single-GPU plan";
    return MAP_E_ARG;
  }
  p->err.clear();
  p->launches = 0;
  const Geom& g = p->g;
  const size_t es = p->elem_real;
  const size_t yb = (size_t)g.batch * g.Nn * p->ny_row * es, xb = (size_t)g.batch * g.Nn * p->d.nx * es;
  const size_t Pb = (size_t)g.batch * g.Nn * (p->d.nx * (p->d.nx + 1) / 2) * es;
  bool blocking = false;
  const void* yd;
  void *xd, *Pd = nullptr;
  map_status st = stage_in(*p, y, yb, &yd, &blocking);
  if (!st) st = stage_out_buf(*p, x_map, xb, &p->stage_x, &p->stage_x_bytes, &xd, &blocking);
  if (!st) st = stage_out_buf(*p, smooth_P, Pb, &p->stage_aux, &p->stage_aux_bytes, &Pd, &blocking);
  if (st) return st;
  {
    const void* key[6] = {yd, xd, Pd, nullptr, nullptr, "tf"};
    map_status gs = graph_run(*p, key, [&] { p->runner->two_filter(*p, yd, xd, Pd); });
    if (gs) return gs;
  }
  std::vector<std::pair<void*, std::pair<void*, size_t>>> outs;
  outs.push_back({x_map, {xd, xb}});
  if (smooth_P) outs.push_back({smooth_P, {Pd, Pb}});
  return finish(*p, blocking, outs);
}

map_status map_solve_sequential(map_plan_t p, int32_t method, const void* y, int32_t passes, void* x_map,
                                void* smooth_P) {
  NvtxRange nvtx_("pmap:map_solve_sequential");
  if (!p || !y || !x_map || (method != 0 && method != 1)) return MAP_E_ARG;
  if (p->d.world != 1) {
    p->err = "map_solve_sequential needs a single-GPU plan (world == 1)";
    return MAP_E_ARG;
  }
  const bool nl = p->kind == Kind::NL;
  if (nl && (method != 0 || passes < 1)) {
    p->err = "nonlinear plans: sequential RTS (method 0) with passes >= 1";
    return MAP_E_ARG;
  }
  p->err.clear();
  p->launches = 0;
  const Geom& g = p->g;
  const size_t es = p->elem_real;
  const size_t yb = (size_t)g.batch * g.Nn * p->ny_row * es, xb = (size_t)g.batch * g.Nn * p->d.nx * es;
  const size_t Pb = (size_t)g.batch * g.Nn * (p->d.nx * (p->d.nx + 1) / 2) * es;
  bool blocking = false;
  const void* yd;
  void *xd, *Pd = nullptr;
  map_status st = stage_in(*p, y, yb, &yd, &blocking);
  if (!st) st = stage_out_buf(*p, x_map, xb, &p->stage_x, &p->stage_x_bytes, &xd, &blocking);
  if (!st) st = stage_out_buf(*p, smooth_P, Pb, &p->stage_aux, &p->stage_aux_bytes, &Pd, &blocking);
  if (st) return st;
  if (!nl) {
    p->runner->sequential(*p, method, yd, nullptr, xd, Pd);
  } else {  // sequential IEKS: xbar^(0) = m0 (R-INIT), re-linearised every pass
    p->runner->fill_m0(*p, p->xbuf[0]);
    for (int k = 0; k < passes; ++k) {
      void* out = (k == passes - 1) ? xd : p->xbuf[(k + 1) & 1];
      p->runner->sequential(*p, 0, yd, p->xbuf[k & 1], out, (k == passes - 1) ? Pd : nullptr);
    }
  }
  if (!p->err.empty()) return MAP_E_ARG;
  std::vector<std::pair<void*, std::pair<void*, size_t>>> outs;
  outs.push_back({x_map, {xd, xb}});
  if (smooth_P) outs.push_back({smooth_P, {Pd, Pb}});
  return finish(*p, blocking, outs);
}

map_status map_solve_nonlinear(map_plan_t p, const void* y, int32_t passes, double tol, const void* x_init,
                               void* x_map, int32_t* passes_run) {
  NvtxRange nvtx_("pmap:map_solve_nonlinear");
  if (!p || !y || !x_map || passes < 1 || tol < 0) return MAP_E_ARG;
  if (p->kind != Kind::NL) {
    p->err = "map_solve_nonlinear called on a linear plan";
    return MAP_E_ARG;
  }
  p->err.clear();
  p->launches = 0;
  const Geom& g = p->g;
  const size_t es = p->elem_real;
  const size_t yb = (size_t)g.batch * g.Nn * p->ny_row * es, xb = (size_t)g.batch * g.Nn * p->d.nx * es;
  bool blocking = false;
  const void* yd;
  void* xd;
  map_status st = stage_in(*p, y, yb, &yd, &blocking);
  if (!st) st = stage_out_buf(*p, x_map, xb, &p->stage_x, &p->stage_x_bytes, &xd, &blocking);
  if (st) return st;
  // xbar^(0)
  if (x_init) {
    if (is_device_ptr(x_init)) {
      PM_CK(*p, cudaMemcpyAsync(p->xbuf[0], x_init, xb, cudaMemcpyDeviceToDevice, p->stream));
    } else {
      // host buffer: the caller may reuse it once we return, so wait for the copy
      PM_CK(*p, cudaMemcpyAsync(p->xbuf[0], x_init, xb, cudaMemcpyHostToDevice, p->stream));
      blocking = true;
    }
  } else {
    p->runner->fill_m0(*p, p->xbuf[0]);
  }
  // graph capture (private stream; p->stream / p->prof restored on every exit)
  struct CaptureScope {
    PlanState& p;
    cudaStream_t cs = nullptr, saved;
    bool saved_prof;
    explicit CaptureScope(PlanState& pp) : p(pp), saved(pp.stream), saved_prof(pp.prof) {}
    cudaError_t begin() {
      cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
      if (e == cudaSuccess) {
        p.stream = cs;
        p.prof = false;
      }
      return e;
    }
    ~CaptureScope() {
      p.stream = saved;
      p.prof = saved_prof;
      if (cs) {
        cudaStreamCaptureStatus cst;
        if (cudaStreamIsCapturing(cs, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
          cudaGraph_t junk = nullptr;
          cudaStreamEndCapture(cs, &junk);
          if (junk) cudaGraphDestroy(junk);
        }
        cudaStreamDestroy(cs);
      }
    }
  };
  const bool capture = p->d.world == 1 && !p->force_shard && !p->prof;  // profiling: plain launches
  int run = 0;
  if (tol == 0.0) {
    // fixed number of passes, no host synchronisation: one CUDA graph
    const void* key[4] = {yd, xd, (const void*)(intptr_t)passes, nullptr};
    if (capture && !(p->graph && memcmp(key, p->graph_key, sizeof key) == 0)) {
      if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
      }
      CaptureScope sc(*p);
      PM_CK(*p, sc.begin());
      const int64_t l0 = p->launches;
      PM_CK(*p, cudaStreamBeginCapture(sc.cs, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < passes; ++k) {
        void* out = (k == passes - 1) ? xd : p->xbuf[(k + 1) & 1];
        p->runner->rts(*p, yd, p->xbuf[k & 1], out, nullptr, nullptr);
      }
      cudaGraph_t graph = nullptr;
      PM_CK(*p, cudaStreamEndCapture(sc.cs, &graph));
      cudaError_t ie = cudaGraphInstantiate(&p->graph, graph, 0);
      cudaGraphDestroy(graph);
      if (ie != cudaSuccess) {
        p->graph = nullptr;
        return cuda_fail(*p, ie, "graph instantiate");
      }
      memcpy(p->graph_key, key, sizeof key);
      p->graph_launches = p->launches - l0;
      p->launches = l0;
    }
    if (capture) {
      PM_CK(*p, cudaGraphLaunch(p->graph, p->stream));
      p->launches += p->graph_launches;
    } else {
      for (int k = 0; k < passes; ++k) {
        void* out = (k == passes - 1) ? xd : p->xbuf[(k + 1) & 1];
        p->runner->rts(*p, yd, p->xbuf[k & 1], out, nullptr, nullptr);
      }
    }
    run = passes;
    if (passes_run) *passes_run = run;
    return finish(*p, blocking, {{x_map, {xd, xb}}});
  }
  // tol > 0: device-side stop.  One pass = rts(xbuf0 -> xbuf1), then
  // dflag[1] = max |xbuf1 - xbuf0| with xbuf0 <- xbuf1, then k_ieks_decide (one thread)
  // counts the pass in dflag[2], keeps dmax in dflag[3] and sets the loop condition
  // (dmax >= tol and passes left).  Captured as the body of a CUDA-graph WHILE node, so a
  // solve costs one host synchronisation (to report passes_run / divergence) instead of
  // one per pass; eager host loop when profiling or time-sharded.
  PM_CK(*p, cudaMemsetAsync(p->dflag + 1, 0, 3 * sizeof(unsigned long long), p->stream));
  const void* key[4] = {yd, (const void*)(intptr_t)passes, nullptr, nullptr};
  bool use_graph = capture;
  if (use_graph && !(p->wgraph && memcmp(key, p->wgraph_key, sizeof key) == 0 && p->wgraph_tol == tol)) {
    if (p->wgraph) {
      cudaGraphExecDestroy(p->wgraph);
      p->wgraph = nullptr;
    }
    cudaGraph_t top = nullptr;
    PM_CK(*p, cudaGraphCreate(&top, 0));
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, top, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    if (e == cudaSuccess) e = cudaGraphAddNode(&cn, top, nullptr, 0, &cp);
    const int64_t l0 = p->launches;
    if (e == cudaSuccess) {
      CaptureScope sc(*p);
      e = sc.begin();
      if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(sc.cs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) {
        p->runner->rts(*p, yd, p->xbuf[0], p->xbuf[1], nullptr, nullptr);
        p->runner->maxdiff(*p, p->xbuf[0], p->xbuf[1], p->dflag + 1, true);
        launch_ieks_decide(sc.cs, p->dflag, tol, passes, h, true);
        p->launches++;
        cudaGraph_t body = nullptr;
        e = cudaStreamEndCapture(sc.cs, &body);
      }
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&p->wgraph, top, 0);
    cudaGraphDestroy(top);
    if (e != cudaSuccess || !p->err.empty()) {  // conditional nodes unavailable: host loop
      cudaGetLastError();
      p->wgraph = nullptr;
      p->err.clear();
      use_graph = false;
    } else {
      memcpy(p->wgraph_key, key, sizeof key);
      p->wgraph_tol = tol;
      p->wgraph_launches = p->launches - l0;
    }
    p->launches = l0;
  } else if (use_graph && !p->wgraph) {
    use_graph = false;
  }
  unsigned long long cnt[2] = {0, 0};
  if (use_graph) {
    PM_CK(*p, cudaGraphLaunch(p->wgraph, p->stream));
    p->launches += p->wgraph_launches;  // per pass
    PM_CK(*p, cudaMemcpyAsync(xd, p->xbuf[1], xb, cudaMemcpyDeviceToDevice, p->stream));
    PM_CK(*p, cudaMemcpyAsync(cnt, p->dflag + 2, sizeof cnt, cudaMemcpyDeviceToHost, p->stream));
    PM_CK(*p, cudaStreamSynchronize(p->stream));
  } else {
    for (int k = 0; k < passes; ++k) {
      p->runner->rts(*p, yd, p->xbuf[0], p->xbuf[1], nullptr, nullptr);
      p->runner->maxdiff(*p, p->xbuf[0], p->xbuf[1], p->dflag + 1, true);
      launch_ieks_decide(p->stream, p->dflag, tol, passes, 0, false);
      p->launches++;
      PM_CK(*p, cudaMemcpyAsync(cnt, p->dflag + 2, sizeof cnt, cudaMemcpyDeviceToHost, p->stream));
      PM_CK(*p, cudaStreamSynchronize(p->stream));
      double dm;
      memcpy(&dm, &cnt[1], sizeof dm);
      if (!(dm >= tol)) break;
    }
    PM_CK(*p, cudaMemcpyAsync(xd, p->xbuf[1], xb, cudaMemcpyDeviceToDevice, p->stream));
  }
  run = (int)cnt[0];
  double dmax;
  memcpy(&dmax, &cnt[1], sizeof dmax);
  if (passes_run) *passes_run = run;
  map_status fs = finish(*p, blocking, {{x_map, {xd, xb}}});
  if (fs != MAP_OK) return fs;
  if (!(dmax < tol)) {
    char buf[160];
    snprintf(buf, sizeof buf, "iterated linearisation did not reach tol %.3g: max |dx| = %.3g after %d passes", tol,
             dmax, run);
    p->err = buf;
    return MAP_E_DIVERGED;  // x_map holds the last iterate
  }
  return MAP_OK;
}

int64_t map_shard_payload_bytes(map_plan_t p, int32_t phase) {
  if (!p || (phase != 1 && phase != 2)) return -1;
  return (int64_t)(p->runner->payload_elems(phase) * p->g.batch * p->elem_real);
}

map_status map_shard_phase(map_plan_t p, int32_t phase, const void* y, const void* gathered, void* payload,
                           void* x_map, void* filt_m, void* filt_P) {
  NvtxRange nvtx_("pmap:map_shard_phase");
  if (!p || phase < 1 || phase > 3) return MAP_E_ARG;
  if (p->kind == Kind::NL || p->d.world < 2) {
    p->err = "map_shard_phase needs a linear time-sharded plan (world > 1)";
    return MAP_E_ARG;
  }
  const bool dev_ok = (phase == 3 ? (!y || is_device_ptr(y)) : is_device_ptr(y)) && (phase == 1 || is_device_ptr(gathered)) &&
                      (phase == 3 || is_device_ptr(payload)) && (phase != 3 || is_device_ptr(x_map)) &&
                      (!filt_m || is_device_ptr(filt_m)) && (!filt_P || is_device_ptr(filt_P));
  if (!dev_ok) {
    p->err = "map_shard_phase takes device buffers only";
    return MAP_E_ARG;
  }
  p->err.clear();
  p->launches = 0;
  if (phase == 1)
    p->runner->phase1(*p, y, nullptr, payload);
  else if (phase == 2) {
    p->want_filter = filt_m || filt_P;
    p->runner->phase2(*p, y, nullptr, gathered, payload);
  } else {
    p->runner->phase3(*p, y, nullptr, gathered, x_map, filt_m, filt_P);
    if (!p->err.empty()) return MAP_E_ARG;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(*p, e, "kernel launch");
  return MAP_OK;
}

map_status map_sync(map_plan_t p) {
  if (!p) return MAP_E_ARG;
  for (cudaStream_t s : {p->pipe_in, p->pipe_out})  // pipelined host-buffer solves in flight
    if (s) {
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return cuda_fail(*p, e, "map_sync");
    }
  return check_flag(*p);
}

map_status map_solve_linear_pipelined(map_plan_t p, const void* y_host, void* x_host) {
  NvtxRange nvtx_("pmap:map_solve_linear_pipelined");
  if (!p || !y_host || !x_host) return MAP_E_ARG;
  if (p->kind == Kind::NL) {
    p->err = "map_solve_linear_pipelined called on a nonlinear plan";
    return MAP_E_ARG;
  }
  if (is_device_ptr(y_host) || is_device_ptr(x_host)) {
    p->err = "map_solve_linear_pipelined takes host buffers (pinned, for the copies to overlap)";
    return MAP_E_ARG;
  }
  if (p->d.world > 1 && !p->d.nccl_comm) {
    p->err = "time-sharded plan without an NCCL communicator: drive the exchange with map_shard_phase";
    return MAP_E_NCCL;
  }
  p->err.clear();
  p->launches = 0;
  const Geom& g = p->g;
  const size_t es = p->elem_real;
  const size_t yb = (size_t)g.batch * g.Nn * p->ny_row * es, xb = (size_t)g.batch * g.Nn * p->d.nx * es;
  if (!p->pipe_in) {
    PM_CK(*p, cudaStreamCreateWithFlags(&p->pipe_in, cudaStreamNonBlocking));
    PM_CK(*p, cudaStreamCreateWithFlags(&p->pipe_out, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t* e : {&p->pipe_ev_in[k], &p->pipe_ev_comp[k], &p->pipe_ev_out[k]})
        PM_CK(*p, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  if (p->pipe_y_bytes < yb || p->pipe_x_bytes < xb) {  // (re)size the staging slots
    for (cudaStream_t s : {p->pipe_in, p->pipe_out, p->stream}) cudaStreamSynchronize(s);
    for (int k = 0; k < 2; ++k) {
      cudaFree(p->pipe_y[k]);
      cudaFree(p->pipe_x[k]);
      p->pipe_y[k] = p->pipe_x[k] = nullptr;
    }
    p->pipe_y_bytes = p->pipe_x_bytes = 0;
    for (int k = 0; k < 2; ++k) {
      PM_CK(*p, cudaMalloc(&p->pipe_y[k], yb));
      PM_CK(*p, cudaMalloc(&p->pipe_x[k], xb));
    }
    p->pipe_y_bytes = yb;
    p->pipe_x_bytes = xb;
    p->pipe_k = 0;
  }
  const int sl = (int)(p->pipe_k & 1);
  const bool reuse = p->pipe_k >= 2;  // the slot served solve k - 2
  // copy in: after solve k - 2 has read the y slot
  if (reuse) PM_CK(*p, cudaStreamWaitEvent(p->pipe_in, p->pipe_ev_comp[sl], 0));
  PM_CK(*p, cudaMemcpyAsync(p->pipe_y[sl], y_host, yb, cudaMemcpyHostToDevice, p->pipe_in));
  PM_CK(*p, cudaEventRecord(p->pipe_ev_in[sl], p->pipe_in));
  // compute: after the copy in, and after the copy out of solve k - 2 has drained the x slot
  PM_CK(*p, cudaStreamWaitEvent(p->stream, p->pipe_ev_in[sl], 0));
  if (reuse) PM_CK(*p, cudaStreamWaitEvent(p->stream, p->pipe_ev_out[sl], 0));
  {
    const void* key[6] = {p->pipe_y[sl], p->pipe_x[sl], nullptr, nullptr, nullptr, "rts"};
    map_status gs = graph_run(*p, key, [&] { p->runner->rts(*p, p->pipe_y[sl], nullptr, p->pipe_x[sl], nullptr, nullptr); });
    if (gs) return gs;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(*p, e, "kernel launch");
  if (!p->err.empty()) return p->err.rfind("ncclAllGather", 0) == 0 ? MAP_E_NCCL : MAP_E_ARG;
  PM_CK(*p, cudaEventRecord(p->pipe_ev_comp[sl], p->stream));
  // copy out: after the solve
  PM_CK(*p, cudaStreamWaitEvent(p->pipe_out, p->pipe_ev_comp[sl], 0));
  PM_CK(*p, cudaMemcpyAsync(x_host, p->pipe_x[sl], xb, cudaMemcpyDeviceToHost, p->pipe_out));
  PM_CK(*p, cudaEventRecord(p->pipe_ev_out[sl], p->pipe_out));
  ++p->pipe_k;
  return MAP_OK;
}

const char* map_last_error(map_plan_t p) { return p ? p->err.c_str() : "null plan"; }

map_status map_profile_enable(map_plan_t p, int32_t enable) {
  if (!p) return MAP_E_ARG;
  p->prof = enable != 0;
  if (!p->prof) {
    p->recs.clear();
    p->ev_used = 0;
  }
  return MAP_OK;
}

int32_t map_profile_read(map_plan_t p, const char** names, double* ms, int64_t* launches, int32_t nmax) {
  if (!p || nmax < 0) return -1;
  double acc[K_COUNT] = {0};
  int64_t cnt[K_COUNT] = {0};
  for (auto& r : p->recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return -1;
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) return -1;
    acc[r.id] += t;
    cnt[r.id]++;
  }
  p->recs.clear();
  p->ev_used = 0;
  int32_t k = 0;
  for (int id = 0; id < K_COUNT && k < nmax; ++id) {
    if (!cnt[id]) continue;
    if (names) names[k] = kernel_name(id);
    if (ms) ms[k] = acc[id];
    if (launches) launches[k] = cnt[id];
    ++k;
  }
  return k;
}

int64_t map_workspace_bytes(map_plan_t p) { return p ? (int64_t)(p->ws_bytes + p->lb_bytes) : 0; }

int64_t map_last_launch_count(map_plan_t p) { return p ? p->launches : 0; }

int64_t map_debug_lb_timing(map_plan_t p, uint64_t* out, int64_t n) {
  if (!p || !p->lb_tim) return 0;
  const int64_t m = n < (int64_t)p->lb_tim_n ? n : (int64_t)p->lb_tim_n;
  if (out && m > 0 && cudaMemcpy(out, p->lb_tim, sizeof(uint64_t) * m, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return (int64_t)p->lb_tim_n;
}

}  // extern "C"
