/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, sequential CPU reference for arXiv 2512.13319 ("Temporal
 * parallelisation of continuous-time MAP trajectory estimation").  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load, call or link this file.  It shares no code, header,
 * table or helper with the CUDA product path in paper_2512_13319_b200/.
 *
 * Citations: "P:n" = line n of the paper's LaTeX; readings of the
 * paper are listed in DESIGN.md ("R-" ids) and SURVEY.md section 8(c) ("G" ids).
 *
 * What it computes:
 *   The linear-affine SDE of P:134-140 discretised on the grid t_i = t0 + i*dt,
 *   i = 0..T, dt = (tf - t0)/T, one node per grid point:
 *     x_{i-1} = (I - dt F_i) x_i - dt c_i + w_i,   w_i ~ N(0, dt Q_i), Q = L W L^T
 *     y_i     = H_i x_i + r_i + nu_i,             nu_i ~ N(0, R_i / dt)
 *     x_0     ~ N(m0, P0)
 *   i.e. the forward transition x_i = Phi_i (x_{i-1} + dt c_i) + Phi_i w_i with
 *   Phi_i = (I - dt F_i)^{-1}.  Its MAP trajectory (= posterior mean, the minimiser
 *   of the discretised Onsager--Machlup / LQT objective P:63-97 for linear models)
 *   is computed by the textbook sequential Kalman filter + RTS smoother, the
 *   discrete counterpart of the Kalman--Bucy filter and continuous RTS smoother
 *   of P:200-226.  The two-filter variant uses the textbook
 *   backward information filter.  The nonlinear variant is the
 *   iterated extended Kalman smoother (Gauss--Newton): re-linearise f, h about the
 *   previous trajectory and re-run the linear smoother.
 *
 * All arithmetic in REAL (double by default; -DORA_LONG_DOUBLE builds the
 * long-double self-check used by pin P10).  Inputs/outputs are double.
 */
#include <stdlib.h>
#include <string.h>
#include <tgmath.h>

#ifdef ORA_LONG_DOUBLE
typedef long double REAL;
#else
typedef double REAL;
#endif

#define MAXN 8

typedef struct {
  int nx, ny, nw;
  long T;            /* grid steps; nodes 0..T */
  double t0, tf;
  const double *F, *c, *L, *W, *H, *r, *R; /* per-node arrays, row-major */
  long sF, sc, sL, sW, sH, sr, sR;          /* element stride between nodes (0 = constant) */
  const double *m0, *P0;
  const double* g;   /* nullable [T+1][nx]: linear node cost g_i^T x_i (OM divergence term) */
} ora_model;

/* ---------------- small dense helpers (row-major, n <= MAXN) ---------------- */

static void mat_mul(int n, int k, int m, const REAL* A, const REAL* B, REAL* C) {
  /* C(n x m) = A(n x k) B(k x m) */
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) {
      REAL s = 0;
      for (int l = 0; l < k; ++l) s += A[i * k + l] * B[l * m + j];
      C[i * m + j] = s;
    }
}

static void mat_mul_bt(int n, int k, int m, const REAL* A, const REAL* B, REAL* C) {
  /* C(n x m) = A(n x k) B(m x k)^T */
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < m; ++j) {
      REAL s = 0;
      for (int l = 0; l < k; ++l) s += A[i * k + l] * B[j * k + l];
      C[i * m + j] = s;
    }
}

static void mat_vec(int n, int k, const REAL* A, const REAL* x, REAL* y) {
  for (int i = 0; i < n; ++i) {
    REAL s = 0;
    for (int l = 0; l < k; ++l) s += A[i * k + l] * x[l];
    y[i] = s;
  }
}

static void symmetrize(int n, REAL* P) {
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      REAL a = (P[i * n + j] + P[j * n + i]) / 2;
      P[i * n + j] = a;
      P[j * n + i] = a;
    }
}

/* Solve A X = B (A n x n, B n x m) by Gaussian elimination with partial
 * pivoting; A and B are overwritten (X returned in B).  Returns 0 on success. */
static int lu_solve(int n, int m, REAL* A, REAL* B) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (fabs(A[i * n + k]) > fabs(A[p * n + k])) p = i;
    if (A[p * n + k] == 0) return 1;
    if (p != k) {
      for (int j = 0; j < n; ++j) { REAL t = A[k * n + j]; A[k * n + j] = A[p * n + j]; A[p * n + j] = t; }
      for (int j = 0; j < m; ++j) { REAL t = B[k * m + j]; B[k * m + j] = B[p * m + j]; B[p * m + j] = t; }
    }
    for (int i = k + 1; i < n; ++i) {
      REAL f = A[i * n + k] / A[k * n + k];
      for (int j = k; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
      for (int j = 0; j < m; ++j) B[i * m + j] -= f * B[k * m + j];
    }
  }
  for (int k = n - 1; k >= 0; --k)
    for (int j = 0; j < m; ++j) {
      REAL s = B[k * m + j];
      for (int l = k + 1; l < n; ++l) s -= A[k * n + l] * B[l * m + j];
      B[k * m + j] = s / A[k * n + k];
    }
  return 0;
}

/* Solve S X = B for symmetric positive definite S via Cholesky; S, B overwritten.
 * Returns 0 on success, 1 if S is not positive definite. */
static int chol_solve(int n, int m, REAL* S, REAL* B) {
  for (int j = 0; j < n; ++j) {
    REAL d = S[j * n + j];
    for (int k = 0; k < j; ++k) d -= S[j * n + k] * S[j * n + k];
    if (!(d > 0)) return 1;
    d = sqrt(d);
    S[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      REAL s = S[i * n + j];
      for (int k = 0; k < j; ++k) s -= S[i * n + k] * S[j * n + k];
      S[i * n + j] = s / d;
    }
  }
  for (int c = 0; c < m; ++c) {
    for (int i = 0; i < n; ++i) { /* L z = b */
      REAL s = B[i * m + c];
      for (int k = 0; k < i; ++k) s -= S[i * n + k] * B[k * m + c];
      B[i * m + c] = s / S[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) { /* L^T x = z */
      REAL s = B[i * m + c];
      for (int k = i + 1; k < n; ++k) s -= S[k * n + i] * B[k * m + c];
      B[i * m + c] = s / S[i * n + i];
    }
  }
  return 0;
}

static void load(int cnt, const double* src, REAL* dst) {
  for (int i = 0; i < cnt; ++i) dst[i] = (REAL)src[i];
}

/* Model quantities at node i (P:134-140 sampled at t_i). */
typedef struct {
  REAL F[MAXN * MAXN], c[MAXN], Q[MAXN * MAXN], H[MAXN * MAXN], r[MAXN], R[MAXN * MAXN];
} node_model;

static void model_at(const ora_model* m, long i, node_model* nm) {
  int nx = m->nx, ny = m->ny, nw = m->nw;
  REAL L[MAXN * MAXN], W[MAXN * MAXN], LW[MAXN * MAXN];
  load(nx * nx, m->F + i * m->sF, nm->F);
  if (m->c) load(nx, m->c + i * m->sc, nm->c); else memset(nm->c, 0, sizeof nm->c);
  load(nx * nw, m->L + i * m->sL, L);
  load(nw * nw, m->W + i * m->sW, W);
  mat_mul(nx, nw, nw, L, W, LW);
  mat_mul_bt(nx, nw, nx, LW, L, nm->Q); /* Q = L W L^T */
  symmetrize(nx, nm->Q);
  load(ny * nx, m->H + i * m->sH, nm->H);
  if (m->r) load(ny, m->r + i * m->sr, nm->r); else memset(nm->r, 0, sizeof nm->r);
  load(ny * ny, m->R + i * m->sR, nm->R);
}

/* Prediction to node i (i >= 1) from the filter moments (m, P) at node i-1:
 *   Phi = (I - dt F_i)^{-1};  mp = Phi (m + dt c_i);  Pp = Phi (P + dt Q_i) Phi^T. */
static int predict(int nx, REAL dt, const node_model* nm, const REAL* m, const REAL* P,
                   REAL* Phi, REAL* mp, REAL* Pp) {
  REAL A[MAXN * MAXN], t[MAXN], PQ[MAXN * MAXN], T1[MAXN * MAXN];
  for (int a = 0; a < nx; ++a)
    for (int b = 0; b < nx; ++b) {
      A[a * nx + b] = (a == b ? 1 : 0) - dt * nm->F[a * nx + b];
      Phi[a * nx + b] = (a == b ? 1 : 0);
    }
  if (lu_solve(nx, nx, A, Phi)) return 1;
  for (int a = 0; a < nx; ++a) t[a] = m[a] + dt * nm->c[a];
  mat_vec(nx, nx, Phi, t, mp);
  for (int a = 0; a < nx * nx; ++a) PQ[a] = P[a] + dt * nm->Q[a];
  mat_mul(nx, nx, nx, Phi, PQ, T1);
  mat_mul_bt(nx, nx, nx, T1, Phi, Pp);
  symmetrize(nx, Pp);
  return 0;
}

/* Kalman update at node i with measurement y (noise covariance R_i/dt). */
static int update(int nx, int ny, REAL dt, const node_model* nm, const double* y,
                  const REAL* mp, const REAL* Pp, REAL* m, REAL* P) {
  REAL HP[MAXN * MAXN], Sy[MAXN * MAXN], Kt[MAXN * MAXN], e[MAXN], Hm[MAXN];
  mat_mul(ny, nx, nx, nm->H, Pp, HP);             /* H Pp */
  mat_mul_bt(ny, nx, ny, HP, nm->H, Sy);          /* H Pp H^T */
  for (int a = 0; a < ny * ny; ++a) Sy[a] += nm->R[a] / dt;
  memcpy(Kt, HP, sizeof(REAL) * ny * nx);
  if (chol_solve(ny, nx, Sy, Kt)) return 1;       /* Kt = Sy^{-1} H Pp = K^T */
  mat_vec(ny, nx, nm->H, mp, Hm);
  for (int a = 0; a < ny; ++a) e[a] = (REAL)y[a] - Hm[a] - nm->r[a];
  for (int a = 0; a < nx; ++a) {
    REAL s = mp[a];
    for (int b = 0; b < ny; ++b) s += Kt[b * nx + a] * e[b];
    m[a] = s;
  }
  /* P = Pp - K H Pp */
  for (int a = 0; a < nx; ++a)
    for (int b = 0; b < nx; ++b) {
      REAL s = Pp[a * nx + b];
      for (int l = 0; l < ny; ++l) s -= Kt[l * nx + a] * HP[l * nx + b];
      P[a * nx + b] = s;
    }
  symmetrize(nx, P);
  return 0;
}

/* Forward Kalman filter over nodes 0..T; stores m_i, P_i (full). */
static int kf_forward(const ora_model* md, const double* y, REAL* ms, REAL* Ps) {
  int nx = md->nx, ny = md->ny;
  REAL dt = ((REAL)md->tf - (REAL)md->t0) / (REAL)md->T;
  REAL mp[MAXN], Pp[MAXN * MAXN], Phi[MAXN * MAXN];
  node_model nm;
  for (long i = 0; i <= md->T; ++i) {
    model_at(md, i, &nm);
    if (i == 0) {
      load(nx, md->m0, mp);
      load(nx * nx, md->P0, Pp);
    } else if (predict(nx, dt, &nm, ms + (i - 1) * nx, Ps + (i - 1) * nx * nx, Phi, mp, Pp)) {
      return 1;
    }
    if (update(nx, ny, dt, &nm, y + i * ny, mp, Pp, ms + i * nx, Ps + i * nx * nx)) return 1;
    if (md->g) {
      /* a linear cost term g_i^T x_i multiplies the filtering density by exp(-g_i^T x_i):
       * N(x; m, P) exp(-g^T x) is proportional to N(x; m - P g, P) (completing the square) */
      REAL t[MAXN], gi[MAXN];
      load(nx, md->g + i * nx, gi);
      mat_vec(nx, nx, Ps + i * nx * nx, gi, t);
      for (int a = 0; a < nx; ++a) ms[i * nx + a] -= t[a];
    }
  }
  return 0;
}

/* RTS smoother: x_T = m_T; x_i = m_i + G_i (x_{i+1} - mp_{i+1}),
 * G_i = P_i Phi_{i+1}^T Pp_{i+1}^{-1}  (discrete counterpart of P:219-223).
 * PsS (nullable): smoother covariances, textbook RTS form
 * PsS_T = P_T,  PsS_i = P_i + G_i (PsS_{i+1} - Pp_{i+1}) G_i^T. */
static int rts_backward(const ora_model* md, const REAL* ms, const REAL* Ps, REAL* xs, REAL* PsS) {
  int nx = md->nx;
  REAL dt = ((REAL)md->tf - (REAL)md->t0) / (REAL)md->T;
  REAL mp[MAXN], Pp[MAXN * MAXN], Phi[MAXN * MAXN], Gt[MAXN * MAXN], d[MAXN];
  REAL D[MAXN * MAXN], DG[MAXN * MAXN];
  node_model nm;
  long T = md->T;
  memcpy(xs + T * nx, ms + T * nx, sizeof(REAL) * nx);
  if (PsS) memcpy(PsS + T * nx * nx, Ps + T * nx * nx, sizeof(REAL) * nx * nx);
  for (long i = T - 1; i >= 0; --i) {
    model_at(md, i + 1, &nm);
    if (predict(nx, dt, &nm, ms + i * nx, Ps + i * nx * nx, Phi, mp, Pp)) return 1;
    mat_mul_bt(nx, nx, nx, Phi, Ps + i * nx * nx, Gt); /* Phi P_i (P_i symmetric) = (P_i Phi^T)^T */
    if (PsS)
      for (int a = 0; a < nx * nx; ++a) D[a] = PsS[(i + 1) * nx * nx + a] - Pp[a];
    if (chol_solve(nx, nx, Pp, Gt)) return 1;          /* Gt = Pp^{-1} Phi P_i = G^T */
    for (int a = 0; a < nx; ++a) d[a] = xs[(i + 1) * nx + a] - mp[a];
    for (int a = 0; a < nx; ++a) {
      REAL s = ms[i * nx + a];
      for (int b = 0; b < nx; ++b) s += Gt[b * nx + a] * d[b];
      xs[i * nx + a] = s;
    }
    if (PsS) {
      /* PsS_i = P_i + G D G^T with G = Gt^T:  DG = D Gt,  PsS_i = P_i + Gt^T DG */
      mat_mul(nx, nx, nx, D, Gt, DG);
      for (int a = 0; a < nx; ++a)
        for (int b = 0; b < nx; ++b) {
          REAL s = Ps[i * nx * nx + a * nx + b];
          for (int l = 0; l < nx; ++l) s += Gt[l * nx + a] * DG[l * nx + b];
          PsS[i * nx * nx + a * nx + b] = s;
        }
      symmetrize(nx, PsS + i * nx * nx);
    }
  }
  return 0;
}

static void store(long cnt, const REAL* src, double* dst) {
  for (long i = 0; i < cnt; ++i) dst[i] = (double)src[i];
}

/* Linear MAP (RTS form).  y: [T+1][ny]; x_map: [T+1][nx]; filt_m: [T+1][nx] or
 * NULL; filt_P: [T+1][nx][nx] or NULL.  Returns 0, or 1 on a numeric failure. */
int ora_kf_rts(const ora_model* md, const double* y, double* x_map, double* filt_m, double* filt_P) {
  long N = md->T + 1;
  int nx = md->nx;
  if (nx > MAXN || md->ny > MAXN || md->nw > MAXN || md->T < 1) return 2;
  REAL* ms = malloc(sizeof(REAL) * N * nx);
  REAL* Ps = malloc(sizeof(REAL) * N * nx * nx);
  REAL* xs = malloc(sizeof(REAL) * N * nx);
  int rc = (!ms || !Ps || !xs) ? 3 : kf_forward(md, y, ms, Ps);
  if (!rc) rc = rts_backward(md, ms, Ps, xs, NULL);
  if (!rc) {
    store(N * nx, xs, x_map);
    if (filt_m) store(N * nx, ms, filt_m);
    if (filt_P) store(N * nx * nx, Ps, filt_P);
  }
  free(ms); free(Ps); free(xs);
  return rc;
}

/* Linear MAP and smoother covariances (RTS form).  smooth_P: [T+1][nx][nx]. */
int ora_kf_rts_cov(const ora_model* md, const double* y, double* x_map, double* smooth_P) {
  long N = md->T + 1;
  int nx = md->nx;
  if (nx > MAXN || md->ny > MAXN || md->nw > MAXN || md->T < 1) return 2;
  REAL* ms = malloc(sizeof(REAL) * N * nx);
  REAL* Ps = malloc(sizeof(REAL) * N * nx * nx);
  REAL* xs = malloc(sizeof(REAL) * N * nx);
  REAL* PsS = malloc(sizeof(REAL) * N * nx * nx);
  int rc = (!ms || !Ps || !xs || !PsS) ? 3 : kf_forward(md, y, ms, Ps);
  if (!rc) rc = rts_backward(md, ms, Ps, xs, PsS);
  if (!rc) {
    store(N * nx, xs, x_map);
    store(N * nx * nx, PsS, smooth_P);
  }
  free(ms); free(Ps); free(xs); free(PsS);
  return rc;
}

/* Two-filter MAP: forward filter (S_i = P_i^{-1}, v_i = S_i m_i)
 * combined with the backward information filter (Lb_i, xb_i) = information on
 * x_i from y_{i+1..T}:  x_i = (S_i + Lb_i)^{-1} (v_i + xb_i).
 * Backward recursion (textbook information form): start Lb_T = 0, xb_T = 0;
 * add measurement i:  Lu = Lb_i + dt H^T R^{-1} H,  xu = xb_i + dt H^T R^{-1} (y_i - r_i);
 * predict through x_i = M x_{i-1} + d + e, M = Phi_i, d = Phi_i dt c_i,
 * e ~ N(0, Sig), Sig = Phi_i dt Q_i Phi_i^T:
 *   Lt = (I + Lu Sig)^{-1} Lu,  xt = (I + Lu Sig)^{-1} xu,
 *   Lb_{i-1} = M^T Lt M,  xb_{i-1} = M^T (xt - Lt d). */
int ora_two_filter(const ora_model* md, const double* y, double* x_map) {
  long N = md->T + 1, T = md->T;
  int nx = md->nx, ny = md->ny;
  if (nx > MAXN || ny > MAXN || md->nw > MAXN || T < 1 || md->g) return 2;
  REAL dt = ((REAL)md->tf - (REAL)md->t0) / (REAL)T;
  REAL* ms = malloc(sizeof(REAL) * N * nx);
  REAL* Ps = malloc(sizeof(REAL) * N * nx * nx);
  int rc = (!ms || !Ps) ? 3 : kf_forward(md, y, ms, Ps);
  REAL Lb[MAXN * MAXN] = {0}, xb[MAXN] = {0};
  node_model nm;
  for (long i = T; i >= 0 && !rc; --i) {
    /* combine */
    REAL S[MAXN * MAXN], Sm[MAXN * MAXN], v[MAXN];
    for (int a = 0; a < nx * nx; ++a) { S[a] = (a % (nx + 1) == 0) ? 1 : 0; Sm[a] = Ps[i * nx * nx + a]; }
    if (chol_solve(nx, nx, Sm, S)) { rc = 1; break; } /* S = P_i^{-1} */
    symmetrize(nx, S);
    mat_vec(nx, nx, S, ms + i * nx, v);
    REAL Ssum[MAXN * MAXN], rhs[MAXN];
    for (int a = 0; a < nx * nx; ++a) Ssum[a] = S[a] + Lb[a];
    for (int a = 0; a < nx; ++a) rhs[a] = v[a] + xb[a];
    if (chol_solve(nx, 1, Ssum, rhs)) { rc = 1; break; }
    store(nx, rhs, x_map + i * nx);
    if (i == 0) break;
    /* measurement i */
    model_at(md, i, &nm);
    REAL Rinv[MAXN * MAXN], Rm[MAXN * MAXN], HtRi[MAXN * MAXN], e[MAXN];
    for (int a = 0; a < ny * ny; ++a) { Rinv[a] = (a % (ny + 1) == 0) ? 1 : 0; Rm[a] = nm.R[a]; }
    if (chol_solve(ny, ny, Rm, Rinv)) { rc = 1; break; }
    for (int a = 0; a < nx; ++a)
      for (int b = 0; b < ny; ++b) {
        REAL s = 0;
        for (int l = 0; l < ny; ++l) s += nm.H[l * nx + a] * Rinv[l * ny + b];
        HtRi[a * ny + b] = dt * s; /* dt H^T R^{-1} */
      }
    REAL Lu[MAXN * MAXN], xu[MAXN];
    mat_mul(nx, ny, nx, HtRi, nm.H, Lu);
    for (int a = 0; a < nx * nx; ++a) Lu[a] += Lb[a];
    for (int a = 0; a < ny; ++a) e[a] = (REAL)y[i * ny + a] - nm.r[a];
    mat_vec(nx, ny, HtRi, e, xu);
    for (int a = 0; a < nx; ++a) xu[a] += xb[a];
    /* predict through the transition into node i */
    REAL A[MAXN * MAXN], M[MAXN * MAXN], d[MAXN], t[MAXN], Sig[MAXN * MAXN], T1[MAXN * MAXN];
    for (int a = 0; a < nx; ++a)
      for (int b = 0; b < nx; ++b) {
        A[a * nx + b] = (a == b ? 1 : 0) - dt * nm.F[a * nx + b];
        M[a * nx + b] = (a == b ? 1 : 0);
      }
    if (lu_solve(nx, nx, A, M)) { rc = 1; break; }
    for (int a = 0; a < nx; ++a) t[a] = dt * nm.c[a];
    mat_vec(nx, nx, M, t, d);
    for (int a = 0; a < nx * nx; ++a) T1[a] = dt * nm.Q[a];
    REAL T2[MAXN * MAXN];
    mat_mul(nx, nx, nx, M, T1, T2);
    mat_mul_bt(nx, nx, nx, T2, M, Sig);
    REAL IL[MAXN * MAXN], RHS[MAXN * (MAXN + 1)];
    mat_mul(nx, nx, nx, Lu, Sig, IL);
    for (int a = 0; a < nx; ++a) IL[a * nx + a] += 1;
    for (int a = 0; a < nx; ++a) {
      for (int b = 0; b < nx; ++b) RHS[a * (nx + 1) + b] = Lu[a * nx + b];
      RHS[a * (nx + 1) + nx] = xu[a];
    }
    if (lu_solve(nx, nx + 1, IL, RHS)) { rc = 1; break; }
    REAL Lt[MAXN * MAXN], xt[MAXN], Ltd[MAXN], u[MAXN];
    for (int a = 0; a < nx; ++a) {
      for (int b = 0; b < nx; ++b) Lt[a * nx + b] = RHS[a * (nx + 1) + b];
      xt[a] = RHS[a * (nx + 1) + nx];
    }
    symmetrize(nx, Lt);
    mat_vec(nx, nx, Lt, d, Ltd);
    for (int a = 0; a < nx; ++a) u[a] = xt[a] - Ltd[a];
    REAL LtM[MAXN * MAXN];
    mat_mul(nx, nx, nx, Lt, M, LtM);
    for (int a = 0; a < nx; ++a) {
      for (int b = 0; b < nx; ++b) {
        REAL s = 0;
        for (int l = 0; l < nx; ++l) s += M[l * nx + a] * LtM[l * nx + b];
        Lb[a * nx + b] = s;
      }
      REAL s = 0;
      for (int l = 0; l < nx; ++l) s += M[l * nx + a] * u[l];
      xb[a] = s;
    }
    symmetrize(nx, Lb);
  }
  free(ms); free(Ps);
  return rc;
}

/* ---------------- nonlinear models (P:588-623 and DESIGN.md R-VDP) ---------------- */

/* Coordinated turn: x = (xi, zeta, xi_dot, zeta_dot, omega),
 * f = (xi_dot, zeta_dot, -omega zeta_dot, omega xi_dot, 0),
 * h = (sqrt(xi^2 + zeta^2), atan2(zeta, xi))  (G13: arctan(zeta/xi) read as atan2). */
void ora_ct_f(const double* x, double* f) {
  f[0] = x[2]; f[1] = x[3]; f[2] = -x[4] * x[3]; f[3] = x[4] * x[2]; f[4] = 0;
}
void ora_ct_dfdx(const double* x, double* J) {
  for (int a = 0; a < 25; ++a) J[a] = 0;
  J[0 * 5 + 2] = 1;
  J[1 * 5 + 3] = 1;
  J[2 * 5 + 3] = -x[4]; J[2 * 5 + 4] = -x[3];
  J[3 * 5 + 2] = x[4];  J[3 * 5 + 4] = x[2];
}
void ora_ct_h(const double* x, double* h) {
  h[0] = sqrt(x[0] * x[0] + x[1] * x[1]);
  h[1] = atan2(x[1], x[0]);
}
void ora_ct_dhdx(const double* x, double* J) {
  double r2 = x[0] * x[0] + x[1] * x[1], r = sqrt(r2);
  for (int a = 0; a < 10; ++a) J[a] = 0;
  J[0] = x[0] / r;   J[1] = x[1] / r;
  J[5] = -x[1] / r2; J[6] = x[0] / r2;
}
/* Van der Pol (not in the paper; DESIGN.md R-VDP): x = (x1, x2),
 * f = (x2, mu (1 - x1^2) x2 - x1), h = x1. */
void ora_vdp_f(double mu, const double* x, double* f) {
  f[0] = x[1]; f[1] = mu * (1 - x[0] * x[0]) * x[1] - x[0];
}
void ora_vdp_dfdx(double mu, const double* x, double* J) {
  J[0] = 0; J[1] = 1;
  J[2] = -2 * mu * x[0] * x[1] - 1; J[3] = mu * (1 - x[0] * x[0]);
}

static double wrap_pi(double a) { /* to (-pi, pi] */
  const double PI = 3.14159265358979323846, TWO_PI = 6.28318530717958647692;
  while (a > PI) a -= TWO_PI;
  while (a <= -PI) a += TWO_PI;
  return a;
}

/* Iterated linearisation (IEKS).  kind 1 = coordinated turn,
 * kind 2 = Van der Pol (params[0] = mu).  Pass p linearises about xbar:
 *   F_i = df(xbar_i), c_i = f(xbar_i) - F_i xbar_i, H_i = dh(xbar_i),
 *   r_i = h(xbar_i) - H_i xbar_i,
 * and replaces y_i by y_eff_i = r_i + H_i xbar_i + wrap(y_i - h(xbar_i)) (bearing
 * residual wrapped, G13), then solves the linear MAP with ora_kf_rts.
 * xbar^(0) = x_init, or m0 at every node when x_init is NULL (G18).
 * delta[p] = max_i |x^(p) - x^(p-1)|_inf.  Returns 0 on success. */
int ora_ieks(int kind, const double* params, int nx, int ny, int nw, long T, double t0, double tf,
             const double* L, const double* W, const double* R, const double* m0, const double* P0,
             const double* y, int passes, const double* x_init, double* x_map, double* delta) {
  long N = T + 1;
  if ((kind == 1 && (nx != 5 || ny != 2)) || (kind == 2 && (nx != 2 || ny != 1)) || kind < 1 || kind > 2)
    return 2;
  double *F = malloc(sizeof(double) * N * nx * nx), *c = malloc(sizeof(double) * N * nx);
  double *H = malloc(sizeof(double) * N * ny * nx), *r = malloc(sizeof(double) * N * ny);
  double *ye = malloc(sizeof(double) * N * ny), *xb = malloc(sizeof(double) * N * nx);
  /* Van der Pol with params[1] != 0: keep the OM divergence term 1/2 div f of
   * every interval i >= 1, dt/2 mu (1 - x_{i,0}^2), linearised about the nominal: its
   * gradient dt/2 (-2 mu xbar_{i,0}, 0) becomes a linear node cost. */
  const int om_div = (kind == 2 && params[1] != 0.0);
  double* gdiv = om_div ? calloc(N * nx, sizeof(double)) : NULL;
  int rc = (!F || !c || !H || !r || !ye || !xb || (om_div && !gdiv)) ? 3 : 0;
  for (long i = 0; i < N && !rc; ++i)
    for (int a = 0; a < nx; ++a) xb[i * nx + a] = x_init ? x_init[i * nx + a] : m0[a];
  for (int p = 0; p < passes && !rc; ++p) {
    for (long i = 0; i < N; ++i) {
      const double* xi = xb + i * nx;
      double f[MAXN], h[MAXN];
      double* Fi = F + i * nx * nx; double* Hi = H + i * ny * nx;
      if (kind == 1) { ora_ct_f(xi, f); ora_ct_dfdx(xi, Fi); ora_ct_h(xi, h); ora_ct_dhdx(xi, Hi); }
      else { ora_vdp_f(params[0], xi, f); ora_vdp_dfdx(params[0], xi, Fi); h[0] = xi[0]; Hi[0] = 1; Hi[1] = 0; }
      for (int a = 0; a < nx; ++a) {
        double s = f[a];
        for (int b = 0; b < nx; ++b) s -= Fi[a * nx + b] * xi[b];
        c[i * nx + a] = s;
      }
      for (int a = 0; a < ny; ++a) {
        double hx = 0;
        for (int b = 0; b < nx; ++b) hx += Hi[a * nx + b] * xi[b];
        r[i * ny + a] = h[a] - hx;
        double res = y[i * ny + a] - h[a];
        if (kind == 1 && a == 1) res = wrap_pi(res);
        ye[i * ny + a] = r[i * ny + a] + hx + res;
      }
      if (om_div && i >= 1) gdiv[i * nx + 0] = 0.5 * ((tf - t0) / T) * (-2.0 * params[0] * xi[0]);
    }
    ora_model md = {nx, ny, nw, T, t0, tf, F, c, L, W, H, r, R,
                    nx * nx, nx, 0, 0, ny * nx, ny, 0, m0, P0, gdiv};
    rc = ora_kf_rts(&md, ye, x_map, NULL, NULL);
    if (rc) break;
    double dmax = 0;
    for (long i = 0; i < N * nx; ++i) {
      double d = fabs(x_map[i] - xb[i]);
      if (d > dmax) dmax = d;
      xb[i] = x_map[i];
    }
    if (delta) delta[p] = dmax;
  }
  free(F); free(c); free(H); free(r); free(ye); free(xb); free(gdiv);
  return rc;
}

/* ------------------------------------------------------------------------
 * Paper-faithful Euler blocks (DESIGN.md R-EULER).  Followed step by
 * step in the paper's order and notation:
 *  1. each grid interval (t_{i-1}, t_i], i = 1..T, is a block; its conditional value
 *     function element (A, b, C, eta, J) is obtained by n explicit Euler substeps in s of
 *     the backward ODEs P:416-427 from the boundary A = I, b = C = eta = J = 0,
 *     with F~ = -F, c~ = -c, Q~ = Q and dA/ds = A Q~ J - A F~
 *     (the printed -A Q~ J^T is kept behind `g6_printed` only so the pins can
 *     show that they detect it).  Substep k uses y at the fine time t_{i-1} + (k+1) delta.
 *  2. the terminal element a_T at node 0: (0, 0, 0, P0^-1 m0 + delta H^T R^-1 (y_0 - r),
 *     P0^-1 + delta H^T R^-1 H);
 *  3. value functions at the block boundaries, V_i = E_i (x) V_{i-1} (P:333-336 with the
 *     combination rule P:395-407, right operand a value function), sequentially;
 *  4. x_T = S_T^-1 v_T, x_{i-1} = (I + C_i S_{i-1})^-1 (A_i x_i + b_i + C_i v_{i-1})
 *     (DESIGN.md R-TRANS).
 * y_fine: [n T + 1][ny]; x_map: [T + 1][nx] at the block boundaries.  LTI models only. */
static void mm_(int n, const REAL* X, const REAL* Y, REAL* Z) { mat_mul(n, n, n, X, Y, Z); }

/* Step 1 of the Euler-block method: the element (A, b, C, eta, J) of one block of
 * nsub explicit Euler substeps of length de of the backward ODEs P:416-427, from the
 * boundary (I, 0, 0, 0, 0) of P:427; substep k reads y_sub[k] (fine time
 * t_{i-1} + (k+1) de).  Ft = -F, ct = -c, HRi = H^T R^-1, HRH = H^T R^-1 H. */
static void euler_block(int nx, int ny, int nsub, REAL de, const node_model* nm, const REAL* Ft, const REAL* ct,
                        const REAL* HRi, const REAL* HRH, const double* y_sub, int g6_printed, REAL* A, REAL* b,
                        REAL* C, REAL* eta, REAL* J) {
  for (int a = 0; a < nx * nx; ++a) {
    A[a] = (a % (nx + 1) == 0) ? 1 : 0;
    C[a] = J[a] = 0;
  }
  for (int a = 0; a < nx; ++a) b[a] = eta[a] = 0;
  for (int k = 0; k < nsub; ++k) {
    const double* yk = y_sub + (long)k * ny;
    REAL AQ[MAXN * MAXN], JQ[MAXN * MAXN], t1[MAXN * MAXN], t2[MAXN * MAXN], JT[MAXN * MAXN];
    REAL dA[MAXN * MAXN], db[MAXN], dC[MAXN * MAXN], deta[MAXN], dJ[MAXN * MAXN], u[MAXN];
    mm_(nx, A, nm->Q, AQ);
    mm_(nx, J, nm->Q, JQ);
    for (int a = 0; a < nx; ++a)
      for (int c = 0; c < nx; ++c) JT[a * nx + c] = J[c * nx + a];
    mm_(nx, AQ, g6_printed ? JT : J, t1);
    mm_(nx, A, Ft, t2);
    for (int a = 0; a < nx * nx; ++a) dA[a] = (g6_printed ? -t1[a] : t1[a]) - t2[a];   /* dA/ds */
    mat_vec(nx, nx, AQ, eta, u);
    mat_vec(nx, nx, A, ct, db);
    for (int a = 0; a < nx; ++a) db[a] = -u[a] - db[a];                               /* db/ds */
    mat_mul_bt(nx, nx, nx, AQ, A, dC);
    for (int a = 0; a < nx * nx; ++a) dC[a] = -dC[a];                                 /* dC/ds */
    for (int a = 0; a < nx; ++a) {                                                    /* deta/ds */
      REAL s = 0;
      for (int c = 0; c < nx; ++c) s += JQ[a * nx + c] * eta[c] - Ft[c * nx + a] * eta[c] + J[a * nx + c] * ct[c];
      for (int q = 0; q < ny; ++q) s -= HRi[a * ny + q] * ((REAL)yk[q] - nm->r[q]);
      deta[a] = s;
    }
    mm_(nx, JQ, J, t1);                                                               /* dJ/ds */
    mm_(nx, J, Ft, t2);
    for (int a = 0; a < nx; ++a)
      for (int c = 0; c < nx; ++c) {
        REAL s = t1[a * nx + c] - t2[a * nx + c] - HRH[a * nx + c];
        for (int l = 0; l < nx; ++l) s -= Ft[l * nx + a] * J[l * nx + c];
        dJ[a * nx + c] = s;
      }
    for (int a = 0; a < nx * nx; ++a) { A[a] -= de * dA[a]; C[a] -= de * dC[a]; J[a] -= de * dJ[a]; }
    for (int a = 0; a < nx; ++a) { b[a] -= de * db[a]; eta[a] -= de * deta[a]; }
  }
  symmetrize(nx, C);
  symmetrize(nx, J);
}

/* Model quantities of the Euler-block ODEs (LTI): F~ = -F, c~ = -c,
 * H^T R^-1 and H^T R^-1 H. */
static int euler_setup(const ora_model* md, node_model* nm, REAL* Ft, REAL* ct, REAL* HRi, REAL* HRH) {
  int nx = md->nx, ny = md->ny;
  REAL Ri[MAXN * MAXN];
  model_at(md, 0, nm);
  for (int a = 0; a < nx * nx; ++a) Ft[a] = -nm->F[a];
  for (int a = 0; a < nx; ++a) ct[a] = -nm->c[a];
  for (int a = 0; a < ny * ny; ++a) Ri[a] = (a % (ny + 1) == 0) ? 1 : 0;
  { REAL Rc[MAXN * MAXN]; memcpy(Rc, nm->R, sizeof Rc); if (lu_solve(ny, ny, Rc, Ri)) return 1; }
  for (int a = 0; a < nx; ++a)            /* H^T R^-1 (nx x ny) */
    for (int q = 0; q < ny; ++q) {
      REAL s = 0;
      for (int l = 0; l < ny; ++l) s += nm->H[l * nx + a] * Ri[l * ny + q];
      HRi[a * ny + q] = s;
    }
  mat_mul(nx, ny, nx, HRi, nm->H, HRH);
  return 0;
}

/* The block element alone (pins, tests/test_oracle_pins.py): one block of length
 * (tf - t0) / T split into nsub substeps, measurements y_sub [nsub][ny]; outputs
 * A, C, J (nx x nx), b, eta (nx). */
int ora_euler_block(const ora_model* md, int nsub, const double* y_sub, double* A, double* b, double* C,
                    double* eta, double* J, int g6_printed) {
  int nx = md->nx, ny = md->ny;
  if (nx > MAXN || ny > MAXN || md->T < 1 || nsub < 1) return 2;
  node_model nm;
  REAL Ft[MAXN * MAXN], ct[MAXN], HRi[MAXN * MAXN], HRH[MAXN * MAXN];
  if (euler_setup(md, &nm, Ft, ct, HRi, HRH)) return 1;
  REAL de = ((REAL)md->tf - (REAL)md->t0) / (REAL)md->T / nsub;
  REAL A_[MAXN * MAXN], b_[MAXN], C_[MAXN * MAXN], e_[MAXN], J_[MAXN * MAXN];
  euler_block(nx, ny, nsub, de, &nm, Ft, ct, HRi, HRH, y_sub, g6_printed, A_, b_, C_, e_, J_);
  store(nx * nx, A_, A);
  store(nx, b_, b);
  store(nx * nx, C_, C);
  store(nx, e_, eta);
  store(nx * nx, J_, J);
  return 0;
}

int ora_euler_rts(const ora_model* md, int nsub, const double* y_fine, double* x_map, int g6_printed) {
  int nx = md->nx, ny = md->ny;
  long T = md->T, N = T + 1;
  if (nx > MAXN || ny > MAXN || md->nw > MAXN || T < 1 || nsub < 1 || md->g || md->sF || md->sc || md->sL ||
      md->sW || md->sH || md->sr || md->sR)
    return 2;
  REAL dt = ((REAL)md->tf - (REAL)md->t0) / (REAL)T, de = dt / nsub;
  node_model nm;
  REAL Ft[MAXN * MAXN], ct[MAXN], HRi[MAXN * MAXN], HRH[MAXN * MAXN];
  if (euler_setup(md, &nm, Ft, ct, HRi, HRH)) return 1;
  REAL* EA = malloc(sizeof(REAL) * N * nx * nx);
  REAL* Eb = malloc(sizeof(REAL) * N * nx);
  REAL* EC = malloc(sizeof(REAL) * N * nx * nx);
  REAL* Vs = malloc(sizeof(REAL) * N * nx * nx);
  REAL* Vv = malloc(sizeof(REAL) * N * nx);
  REAL* xs = malloc(sizeof(REAL) * N * nx);
  int rc = (!EA || !Eb || !EC || !Vs || !Vv || !xs) ? 3 : 0;
  /* node 0: a_T of P:329 plus the measurement at t_0 */
  if (!rc) {
    REAL P0[MAXN * MAXN], P0i[MAXN * MAXN], m0[MAXN], e[MAXN];
    load(nx * nx, md->P0, P0);
    load(nx, md->m0, m0);
    for (int a = 0; a < nx * nx; ++a) P0i[a] = (a % (nx + 1) == 0) ? 1 : 0;
    if (lu_solve(nx, nx, P0, P0i)) rc = 1;
    for (int q = 0; q < ny; ++q) e[q] = (REAL)y_fine[q] - nm.r[q];
    for (int a = 0; a < nx && !rc; ++a) {
      REAL s = 0;
      for (int c = 0; c < nx; ++c) s += P0i[a * nx + c] * m0[c];
      for (int q = 0; q < ny; ++q) s += de * HRi[a * ny + q] * e[q];
      Vv[a] = s;                                   /* V_0 = E_0 (x) 0: v_0 = eta_0, S_0 = J_0 */
      for (int c = 0; c < nx; ++c) Vs[a * nx + c] = P0i[a * nx + c] + de * HRH[a * nx + c];
    }
    symmetrize(nx, Vs);
  }
  for (long i = 1; i <= T && !rc; ++i) {
    /* 1. block element by n Euler substeps of P:416-427 (backwards in s from the boundary) */
    REAL A[MAXN * MAXN], b[MAXN], C[MAXN * MAXN], eta[MAXN], J[MAXN * MAXN];
    euler_block(nx, ny, nsub, de, &nm, Ft, ct, HRi, HRH, y_fine + ((i - 1) * nsub + 1) * ny, g6_printed, A, b, C,
                eta, J);
    memcpy(EA + i * nx * nx, A, sizeof(REAL) * nx * nx);
    memcpy(Eb + i * nx, b, sizeof(REAL) * nx);
    memcpy(EC + i * nx * nx, C, sizeof(REAL) * nx * nx);
    /* 3. V_i = E_i (x) V_{i-1}:  S = A^T S (I + C S)^-1 A + J,  v = A^T (I + S C)^-1 (v - S b) + eta */
    const REAL* S = Vs + (i - 1) * nx * nx;
    const REAL* v = Vv + (i - 1) * nx;
    REAL M[MAXN * MAXN], Mt[MAXN * MAXN], X[MAXN * MAXN], w[MAXN * MAXN], Sb[MAXN], t[MAXN * MAXN];
    mm_(nx, C, S, M);
    for (int a = 0; a < nx * nx; ++a) M[a] += (a % (nx + 1) == 0) ? 1 : 0;               /* I + C S */
    for (int a = 0; a < nx; ++a)
      for (int c = 0; c < nx; ++c) Mt[a * nx + c] = M[c * nx + a];                      /* I + S C */
    memcpy(X, A, sizeof A);
    if (lu_solve(nx, nx, M, X)) { rc = 1; break; }                                      /* (I + C S)^-1 A */
    mm_(nx, S, X, t);
    for (int a = 0; a < nx; ++a)
      for (int c = 0; c < nx; ++c) {
        REAL s = J[a * nx + c];
        for (int l = 0; l < nx; ++l) s += A[l * nx + a] * t[l * nx + c];
        Vs[i * nx * nx + a * nx + c] = s;
      }
    symmetrize(nx, Vs + i * nx * nx);
    mat_vec(nx, nx, S, b, Sb);
    for (int a = 0; a < nx; ++a) w[a] = v[a] - Sb[a];
    if (lu_solve(nx, 1, Mt, w)) { rc = 1; break; }
    for (int a = 0; a < nx; ++a) {
      REAL s = eta[a];
      for (int l = 0; l < nx; ++l) s += A[l * nx + a] * w[l];
      Vv[i * nx + a] = s;
    }
  }
  /* 4. x_T = S_T^-1 v_T, then the transitions backwards */
  if (!rc) {
    REAL Sc[MAXN * MAXN], xv[MAXN];
    memcpy(Sc, Vs + T * nx * nx, sizeof(REAL) * nx * nx);
    memcpy(xv, Vv + T * nx, sizeof(REAL) * nx);
    if (chol_solve(nx, 1, Sc, xv)) rc = 1;
    memcpy(xs + T * nx, xv, sizeof(REAL) * nx);
  }
  for (long i = T; i >= 1 && !rc; --i) {
    const REAL* S = Vs + (i - 1) * nx * nx;
    const REAL* v = Vv + (i - 1) * nx;
    const REAL *A = EA + i * nx * nx, *b = Eb + i * nx, *C = EC + i * nx * nx;
    REAL M[MAXN * MAXN], r_[MAXN], Ax[MAXN], Cv[MAXN];
    mm_(nx, C, S, M);
    for (int a = 0; a < nx * nx; ++a) M[a] += (a % (nx + 1) == 0) ? 1 : 0;
    mat_vec(nx, nx, A, xs + i * nx, Ax);
    mat_vec(nx, nx, C, v, Cv);
    for (int a = 0; a < nx; ++a) r_[a] = Ax[a] + b[a] + Cv[a];
    if (lu_solve(nx, 1, M, r_)) { rc = 1; break; }
    memcpy(xs + (i - 1) * nx, r_, sizeof(REAL) * nx);
  }
  if (!rc) store(N * nx, xs, x_map);
  free(EA); free(Eb); free(EC); free(Vs); free(Vv); free(xs);
  return rc;
}

/* ---------------------------------------------------------------------------
 * Intra-block refinement of the Euler-block method (
 * DESIGN.md R-REFINE): x* at the n - 1 fine points inside every block, from
 *   - the value function at the fine point t_k = t_{i-1} + k de: V_k = E_pre (x) V_{i-1},
 *     E_pre = the element of the block's first k substeps (step 1 of ora_euler_rts with
 *     k substeps: P:416-427 from the boundary of P:427);
 *   - the element (A, b, C) from t_k to the block end t_i by the FORWARD HJB equation
 *     of P:490-505 ("in practice, we only need the first three equations"), integrated
 *     in tau (reversed time) by n - k explicit Euler steps from the boundary (I, 0, 0);
 *   - the transition of R-TRANS with x* at the block end:
 *     x*(t_k) = (I + C S_k)^-1 (A x*_i + b + C v_k).
 * y_fine [n T + 1][ny]; x_fine [n T + 1][nx] (block boundaries: ora_euler_rts's x). */

/* V' = E (x) V (P:333-336 with the combination rule P:395-407, right operand a value
 * function):  S' = A^T S (I + C S)^-1 A + J,  v' = A^T (I + S C)^-1 (v - S b) + eta. */
static int vf_combine(int nx, const REAL* A, const REAL* b, const REAL* C, const REAL* eta, const REAL* J,
                      const REAL* S, const REAL* v, REAL* So, REAL* vo) {
  REAL M[MAXN * MAXN], Mt[MAXN * MAXN], X[MAXN * MAXN], w[MAXN], Sb[MAXN], t[MAXN * MAXN];
  mm_(nx, C, S, M);
  for (int a = 0; a < nx * nx; ++a) M[a] += (a % (nx + 1) == 0) ? 1 : 0;             /* I + C S */
  for (int a = 0; a < nx; ++a)
    for (int c = 0; c < nx; ++c) Mt[a * nx + c] = M[c * nx + a];                    /* I + S C */
  memcpy(X, A, sizeof(REAL) * nx * nx);
  if (lu_solve(nx, nx, M, X)) return 1;                                             /* (I + C S)^-1 A */
  mm_(nx, S, X, t);
  for (int a = 0; a < nx; ++a)
    for (int c = 0; c < nx; ++c) {
      REAL s = J[a * nx + c];
      for (int l = 0; l < nx; ++l) s += A[l * nx + a] * t[l * nx + c];
      So[a * nx + c] = s;
    }
  symmetrize(nx, So);
  mat_vec(nx, nx, S, b, Sb);
  for (int a = 0; a < nx; ++a) w[a] = v[a] - Sb[a];
  if (lu_solve(nx, 1, Mt, w)) return 1;
  for (int a = 0; a < nx; ++a) {
    REAL s = eta[a];
    for (int l = 0; l < nx; ++l) s += A[l * nx + a] * w[l];
    vo[a] = s;
  }
  return 0;
}

/* The forward-HJB element (A, b, C)(s, tau) of P:490-505 as a function of its end time
 * tau, m explicit Euler steps of length de in tau from the boundary (I, 0, 0) at tau = s:
 *   dA/dtau = -C H~^T R~^-1 H~ A + F~ A
 *   db/dtau =  C H~^T R~^-1 (y~ - r~) + F~ b + c~ - C H~^T R~^-1 H~ b
 *   dC/dtau = -C H~^T R~^-1 H~ C + Q~ + F~ C + C F~^T
 * (F~ = -F, c~ = -c, Q~ = Q, H~ = H, R~ = R: P:78-102).  tau runs backwards in t from the
 * block end t_i: step j reads y~ at its start, y at the fine time t_i - j de, which is
 * y_blk[nsub - 1 - j] (the measurement placement of R-EULER: every fine point once). */
static void hjb_suffix(int nx, int ny, int m, int nsub, REAL de, const node_model* nm, const REAL* Ft,
                       const REAL* ct, const REAL* HRi, const REAL* HRH, const double* y_blk, REAL* A, REAL* b,
                       REAL* C) {
  for (int a = 0; a < nx * nx; ++a) {
    A[a] = (a % (nx + 1) == 0) ? 1 : 0;
    C[a] = 0;
  }
  for (int a = 0; a < nx; ++a) b[a] = 0;
  for (int j = 0; j < m; ++j) {
    const double* yk = y_blk + (long)(nsub - 1 - j) * ny;
    REAL CM[MAXN * MAXN], t1[MAXN * MAXN], t2[MAXN * MAXN], dA[MAXN * MAXN], dC[MAXN * MAXN], db[MAXN];
    REAL u[MAXN], e[MAXN], t3[MAXN];
    mm_(nx, C, HRH, CM);                                     /* C H^T R^-1 H */
    mm_(nx, CM, A, t1);
    mm_(nx, Ft, A, t2);
    for (int a = 0; a < nx * nx; ++a) dA[a] = -t1[a] + t2[a];
    for (int q = 0; q < ny; ++q) e[q] = (REAL)yk[q] - nm->r[q];
    mat_vec(nx, ny, HRi, e, u);                              /* H^T R^-1 (y - r) */
    mat_vec(nx, nx, C, u, db);
    mat_vec(nx, nx, Ft, b, t3);
    for (int a = 0; a < nx; ++a) db[a] += t3[a] + ct[a];
    mat_vec(nx, nx, CM, b, t3);
    for (int a = 0; a < nx; ++a) db[a] -= t3[a];
    mm_(nx, CM, C, t1);
    mm_(nx, Ft, C, t2);
    mat_mul_bt(nx, nx, nx, C, Ft, dC);                       /* C F~^T */
    for (int a = 0; a < nx * nx; ++a) dC[a] += -t1[a] + nm->Q[a] + t2[a];
    for (int a = 0; a < nx * nx; ++a) { A[a] += de * dA[a]; C[a] += de * dC[a]; }
    for (int a = 0; a < nx; ++a) b[a] += de * db[a];
  }
  symmetrize(nx, C);
}

/* The forward-HJB element alone (pin P16): one block of length (tf - t0) / T, m Euler
 * steps in tau; y_sub [m][ny] in the block's fine order (y_sub[k] at t_start + (k+1) de). */
int ora_hjb_element(const ora_model* md, int m, const double* y_sub, double* A, double* b, double* C) {
  int nx = md->nx;
  if (nx > MAXN || md->ny > MAXN || md->T < 1 || m < 1) return 2;
  node_model nm;
  REAL Ft[MAXN * MAXN], ct[MAXN], HRi[MAXN * MAXN], HRH[MAXN * MAXN];
  if (euler_setup(md, &nm, Ft, ct, HRi, HRH)) return 1;
  REAL de = ((REAL)md->tf - (REAL)md->t0) / (REAL)md->T / m;
  REAL A_[MAXN * MAXN], b_[MAXN], C_[MAXN * MAXN];
  hjb_suffix(nx, md->ny, m, m, de, &nm, Ft, ct, HRi, HRH, y_sub, A_, b_, C_);
  store(nx * nx, A_, A);
  store(nx, b_, b);
  store(nx * nx, C_, C);
  return 0;
}

int ora_euler_refine(const ora_model* md, int nsub, const double* y_fine, double* x_fine) {
  int nx = md->nx, ny = md->ny;
  long T = md->T, N = T + 1;
  if (nx > MAXN || ny > MAXN || md->nw > MAXN || T < 1 || nsub < 1 || md->g || md->sF || md->sc || md->sL ||
      md->sW || md->sH || md->sr || md->sR)
    return 2;
  REAL dt = ((REAL)md->tf - (REAL)md->t0) / (REAL)T, de = dt / nsub;
  node_model nm;
  REAL Ft[MAXN * MAXN], ct[MAXN], HRi[MAXN * MAXN], HRH[MAXN * MAXN];
  if (euler_setup(md, &nm, Ft, ct, HRi, HRH)) return 1;
  double* xb = malloc(sizeof(double) * N * nx);
  REAL* Vs = malloc(sizeof(REAL) * N * nx * nx);
  REAL* Vv = malloc(sizeof(REAL) * N * nx);
  int rc = (!xb || !Vs || !Vv) ? 3 : 0;
  if (!rc) rc = ora_euler_rts(md, nsub, y_fine, xb, 0);      /* x* at the block boundaries */
  /* value functions at the block boundaries (steps 2-3 of ora_euler_rts) */
  if (!rc) {
    REAL P0[MAXN * MAXN], P0i[MAXN * MAXN], m0[MAXN], e[MAXN];
    load(nx * nx, md->P0, P0);
    load(nx, md->m0, m0);
    for (int a = 0; a < nx * nx; ++a) P0i[a] = (a % (nx + 1) == 0) ? 1 : 0;
    if (lu_solve(nx, nx, P0, P0i)) rc = 1;
    for (int q = 0; q < ny; ++q) e[q] = (REAL)y_fine[q] - nm.r[q];
    for (int a = 0; a < nx && !rc; ++a) {
      REAL s = 0;
      for (int c = 0; c < nx; ++c) s += P0i[a * nx + c] * m0[c];
      for (int q = 0; q < ny; ++q) s += de * HRi[a * ny + q] * e[q];
      Vv[a] = s;
      for (int c = 0; c < nx; ++c) Vs[a * nx + c] = P0i[a * nx + c] + de * HRH[a * nx + c];
    }
    symmetrize(nx, Vs);
  }
  for (long i = 1; i <= T && !rc; ++i) {
    REAL A[MAXN * MAXN], b[MAXN], C[MAXN * MAXN], eta[MAXN], J[MAXN * MAXN];
    euler_block(nx, ny, nsub, de, &nm, Ft, ct, HRi, HRH, y_fine + ((i - 1) * nsub + 1) * ny, 0, A, b, C, eta, J);
    if (vf_combine(nx, A, b, C, eta, J, Vs + (i - 1) * nx * nx, Vv + (i - 1) * nx, Vs + i * nx * nx, Vv + i * nx))
      rc = 1;
  }
  if (!rc) {
    memcpy(x_fine, xb, sizeof(double) * nx);
    for (long i = 1; i <= T; ++i) memcpy(x_fine + i * nsub * nx, xb + i * nx, sizeof(double) * nx);
  }
  for (long i = 1; i <= T && !rc; ++i) {
    const double* y_blk = y_fine + ((i - 1) * nsub + 1) * ny;
    REAL xi[MAXN];
    load(nx, xb + i * nx, xi);
    for (int k = 1; k < nsub && !rc; ++k) {
      REAL A[MAXN * MAXN], b[MAXN], C[MAXN * MAXN], eta[MAXN], J[MAXN * MAXN], Sk[MAXN * MAXN], vk[MAXN];
      euler_block(nx, ny, k, de, &nm, Ft, ct, HRi, HRH, y_blk, 0, A, b, C, eta, J);   /* first k substeps */
      if (vf_combine(nx, A, b, C, eta, J, Vs + (i - 1) * nx * nx, Vv + (i - 1) * nx, Sk, vk)) { rc = 1; break; }
      REAL As[MAXN * MAXN], bs[MAXN], Cs[MAXN * MAXN];
      hjb_suffix(nx, ny, nsub - k, nsub, de, &nm, Ft, ct, HRi, HRH, y_blk, As, bs, Cs);
      REAL M[MAXN * MAXN], r_[MAXN], Ax[MAXN], Cv[MAXN];
      mm_(nx, Cs, Sk, M);
      for (int a = 0; a < nx * nx; ++a) M[a] += (a % (nx + 1) == 0) ? 1 : 0;
      mat_vec(nx, nx, As, xi, Ax);
      mat_vec(nx, nx, Cs, vk, Cv);
      for (int a = 0; a < nx; ++a) r_[a] = Ax[a] + bs[a] + Cv[a];
      if (lu_solve(nx, 1, M, r_)) { rc = 1; break; }
      store(nx, r_, x_fine + ((i - 1) * nsub + k) * nx);
    }
  }
  free(xb); free(Vs); free(Vv);
  return rc;
}

/* Batched linear MAP: `batch` independent trajectories sharing the model;
 * y: [batch][T+1][ny], x_map: [batch][T+1][nx].  mode 0 = RTS, 1 = two-filter.
 * OpenMP over trajectories (each recursion is sequential).  Returns the
 * first non-zero per-trajectory status. */
int ora_batch(const ora_model* md, long batch, const double* y, double* x_map, int mode) {
  long N = md->T + 1;
  int rc = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(max : rc)
  for (long b = 0; b < batch; ++b) {
    int r = mode ? ora_two_filter(md, y + b * N * md->ny, x_map + b * N * md->nx)
                 : ora_kf_rts(md, y + b * N * md->ny, x_map + b * N * md->nx, NULL, NULL);
    if (r > rc) rc = r;
  }
  return rc;
}

int ora_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
