// pmap_lti_scan.cuh -- data-only scans of tile and group aggregates for LTI models.
//
// For a time-invariant model every interior tile (NT full runs of K interior nodes)
// has the same matrix parts (A, C, J); only its data parts (b, eta) depend on the
// measurements, and the combination rule of P:395-407 is affine in the data parts
// with coefficients fixed by the matrix parts of the two operands (DESIGN.md R-LTI).
// The Kogge-Stone scans over the tiles of a group and over the groups of a trajectory
// therefore propagate only (b, eta) with plan-time coefficient sets -- 4 N x N
// mat-vecs per round instead of a general combine (an N x N pivoted LU and ~10 N^3
// flops on the critical path).  The boundary blocks -- the one holding node 0 (its
// prefixes are value functions, A = b = C = 0) and a ragged last one -- are joined by
// one general combine each after the scan (depth 1).  Same results up to rounding.
#pragma once
#include "pmap_lti.cuh"

namespace pmap {

constexpr int kScanB = 128;  // blocks per scan (tiles per group = NT2, groups per trajectory)

// One scan level: blocks of equal (interior) span.
template <typename R, int N>
struct LtiBlockTables {
  static constexpr int NS = Dim<N>::NS;
  // matrix parts of a span of s blocks, s = 1..kScanB (index s - 1)
  R TA[kScanB][N][N];
  R TC[kScanB][NS];
  R TJ[kScanB][NS];
  // Kogge-Stone round d (own span d, d = 1, 2, .., kScanB / 2), partner span r = 1..d:
  // set (d, r) at offset (d - 1) * 4 N^2, layout [u][i][k][r - 1] (see UWc, pmap_lti.cuh)
  R U[(kScanB - 1) * 4 * N * N];
};

template <typename R, int N>
struct LtiScanTables {
  LtiBlockTables<R, N> tile;   // block = one interior tile
  LtiBlockTables<R, N> group;  // block = one group of kScanB interior tiles
};

// Coefficients of (own span l1 on the left) (x) (partner span l2 on the right) for the
// data parts: b = U1 b1 + U2 eta2 + b2, eta = U3 eta2 - U4 b1 + eta1 (as in pmap_lti.cuh).
template <typename R, int N>
PM_INLINE void lti_coeff(const R (&A1)[N][N], const R (&C1)[Dim<N>::NS], const R (&A2)[N][N],
                         const R (&J2)[Dim<N>::NS], R* dst, int stride, int slot) {
  R M[N][N], A2M[N][N], T[N][N], C1m[N][N], J2m[N][N], AtMt[N][N], U4[N][N];
  unpack<R, N>(C1, C1m);
  unpack<R, N>(J2, J2m);
  inv_ICJ<R, N>(C1, J2, M);
  matmul<R, N>(A2, M, A2M);
  matmul<R, N>(A2M, C1m, T);
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      R s = R(0);
      for (int k = 0; k < N; ++k) s = fma(A1[k][i], M[j][k], s);
      AtMt[i][j] = s;
    }
  matmul<R, N>(AtMt, J2m, U4);
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      dst[((0 * N + i) * N + j) * stride + slot] = A2M[i][j];
      dst[((1 * N + i) * N + j) * stride + slot] = T[i][j];
      dst[((2 * N + i) * N + j) * stride + slot] = AtMt[i][j];
      dst[((3 * N + i) * N + j) * stride + slot] = U4[i][j];
    }
}

template <typename R, int N>
PM_INLINE void lti_level_setup(const Elem<R, N>& unit, LtiBlockTables<R, N>* t, Elem<R, N>& span_full, bool& ok) {
  Elem<R, N> acc = unit;
  for (int s = 0; s < kScanB; ++s) {
    if (s > 0) combine(unit, acc, acc, ok);  // later block on the left
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) t->TA[s][i][j] = acc.A[i][j];
    for (int k = 0; k < Dim<N>::NS; ++k) {
      t->TC[s][k] = acc.C[k];
      t->TJ[s][k] = acc.J[k];
    }
  }
  span_full = acc;
  for (int d = 1; d < kScanB; d <<= 1) {
    R* base = t->U + (d - 1) * 4 * N * N;
    for (int r = 1; r <= d; ++r) lti_coeff<R, N>(t->TA[d - 1], t->TC[d - 1], t->TA[r - 1], t->TJ[r - 1], base, d, r - 1);
  }
}

// Plan-time tables (one thread): tile = NT runs (tab->SA/SC/SJ[NT - 1]), group = kScanB tiles.
template <typename R, int N, int NT, int K>
__global__ void k_lti_scan_setup(const LtiTables<R, N, NT, K>* __restrict__ tab, LtiScanTables<R, N>* st,
                                 int* okflag) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  bool ok = true;
  Elem<R, N> unit, full;
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j < N; ++j) unit.A[i][j] = tab->SA[NT - 1][i][j];
    unit.b[i] = R(0);
    unit.h[i] = R(0);
  }
  for (int k = 0; k < Dim<N>::NS; ++k) {
    unit.C[k] = tab->SC[NT - 1][k];
    unit.J[k] = tab->SJ[NT - 1][k];
  }
  lti_level_setup<R, N>(unit, &st->tile, full, ok);
  for (int i = 0; i < N; ++i) {
    full.b[i] = R(0);
    full.h[i] = R(0);
  }
  lti_level_setup<R, N>(full, &st->group, unit, ok);
  *okflag = ok ? 1 : 0;
}

// Inclusive scan (later blocks on the left, R-FLIP) of up to kScanB block aggregates
// held one per thread: lanes [0, s0) = the special first block (s0 <= 1), [s0, s1) =
// interior blocks (data-only Kogge-Stone), [s1, cnt) = the special last block (at most
// one).  `own` is the thread's aggregate; returns its inclusive prefix in `res`.
// shd: 2 N * kScanB doubles; she: Elem::SZ doubles.
// shown: the thread's own aggregate, field-major in shared memory (field f at shown[f * kScanB]),
// so that only the running prefix occupies registers.
template <typename R, int N>
PM_INLINE void lti_block_scan(const LtiBlockTables<R, N>* T, int t, int cnt, int s0, int s1,
                              const R* shown, Elem<R, N>& res, R* shd, R* she, bool& ok) {
  using E = Elem<R, N>;
  const bool interior = t >= s0 && t < s1;
  const int p = t - s0;
  const int nint = s1 - s0;
  const ElemRef<R, N> own{shown, kScanB};
  R bb[N], hh[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    bb[i] = own.b(i);
    hh[i] = own.h(i);
  }
#pragma unroll 1
  for (int d = 1; d < nint; d <<= 1) {
    __syncthreads();
#pragma unroll
    for (int i = 0; i < N; ++i) {
      shd[i * kScanB + t] = bb[i];
      shd[(N + i) * kScanB + t] = hh[i];
    }
    __syncthreads();
    if (interior && p >= d) {
      const R* U = T->U + (d - 1) * 4 * N * N;
      const int slot = min(p - d, d - 1);  // partner span - 1
      R b2[N], h2[N], nb[N], nh[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        b2[i] = shd[i * kScanB + t - d];
        h2[i] = shd[(N + i) * kScanB + t - d];
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        R sb = b2[i], sb2 = R(0), sh_ = hh[i], sh2 = R(0);
#pragma unroll
        for (int k = 0; k < N; ++k) {
          sb = fma(__ldg(U + ((0 * N + i) * N + k) * d + slot), bb[k], sb);
          sb2 = fma(__ldg(U + ((1 * N + i) * N + k) * d + slot), h2[k], sb2);
          sh_ = fma(__ldg(U + ((2 * N + i) * N + k) * d + slot), h2[k], sh_);
          sh2 = fma(-__ldg(U + ((3 * N + i) * N + k) * d + slot), bb[k], sh2);
        }
        nb[i] = sb + sb2;
        nh[i] = sh_ + sh2;
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        bb[i] = nb[i];
        hh[i] = nh[i];
      }
    }
  }
  if (interior) {  // the interior prefix as a full element (matrix parts of span p + 1)
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
      for (int j = 0; j < N; ++j) res.A[i][j] = T->TA[p][i][j];
      res.b[i] = bb[i];
      res.h[i] = hh[i];
    }
#pragma unroll
    for (int k = 0; k < Dim<N>::NS; ++k) {
      res.C[k] = T->TC[p][k];
      res.J[k] = T->TJ[p][k];
    }
  } else {
    load(res, shown, kScanB);
  }
  // join the special first block: prefix = interior prefix (x) first (lane 0's slot)
  __syncthreads();
  if (s0 == 1 && interior) combine_g(res, ElemRef<R, N>{shown - t, kScanB}, res, ok);
  // the special last block: its prefix = last (x) prefix of the lane before it
  if (s1 < cnt) {
    __syncthreads();
    if (t == s1 - 1) store(res, she, 1);
    __syncthreads();
    if (t == s1 && s1 > 0) {
      E last;
      load(last, shown, kScanB);
      combine_g(last, ElemRef<R, N>{she, 1}, res, ok);
    }
  }
}

// Inclusive scan of the tile aggregates within groups of kScanB tiles (LTI interior
// tiles data-only); same outputs as k_p1_tiles.
template <typename R, int N>
__global__ void __launch_bounds__(kScanB) k_p1_tiles_lti(const Geom g, const R* __restrict__ tile_agg,
                                                         R* __restrict__ tile_incl, R* __restrict__ group_agg,
                                                         const LtiScanTables<R, N>* __restrict__ st, int64_t j_lo,
                                                         int64_t j_hi, unsigned long long* flag) {
  using E = Elem<R, N>;
  __shared__ R shd[2 * N * kScanB];
  __shared__ R she[E::SZ];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sho = reinterpret_cast<R*>(smem_raw);  // the aggregates, field-major (dynamic)
  const LtiBlockTables<R, N>* Ts = &st->tile;
  const int64_t grp = blockIdx.x;
  const int64_t b = grp / g.gpt, gg = grp % g.gpt;
  const int t = threadIdx.x;
  const int64_t j0 = gg * kScanB;
  const int cnt = (int)min((int64_t)kScanB, g.tpt - j0);
  // lanes: [0, s0) first special (tile 0 when j_lo == 1), [s0, s1) interior, [s1, cnt) last
  const int s0 = (j0 < j_lo) ? (int)(j_lo - j0) : 0;
  const int s1 = (int)max((int64_t)s0, min((int64_t)cnt, j_hi - j0));
  bool ok = true;
  const R* src = tile_agg + (b * g.tpt + j0) * E::SZ;  // cnt contiguous aggregates
  for (int q = t; q < cnt * E::SZ; q += kScanB) sho[(q % E::SZ) * kScanB + q / E::SZ] = src[q];
  if (t >= cnt) {
    E id;
    set_identity(id);
    store(id, sho + t, kScanB);
  }
  __syncthreads();
  E res;
  lti_block_scan<R, N>(Ts, t, cnt, s0, s1, sho + t, res, shd, she, ok);
  if (t < cnt) store(res, tile_incl + (b * g.tpt + j0 + t) * E::SZ, 1);
  if (t == cnt - 1) store(res, group_agg + grp * E::SZ, 1);
  if (!ok) flag_node(flag, g.node0 + j0 + t);
}

// Group carries (as k_p1_groups) with the data-only scan over interior groups; one lane
// per group (gpt <= kScanB).  A group is interior when all of its kScanB tiles are.
template <typename R, int N>
__global__ void __launch_bounds__(kScanB) k_p1_groups_lti(const Geom g, const R* __restrict__ group_agg,
                                                          const R* __restrict__ gathered, int rank,
                                                          R* __restrict__ carry_out, R* __restrict__ group_carry,
                                                          R* __restrict__ total_agg,
                                                          const LtiScanTables<R, N>* __restrict__ st, int64_t j_lo,
                                                          int64_t j_hi, unsigned long long* flag) {
  using E = Elem<R, N>;
  using V = VF<R, N>;
  __shared__ R shd[2 * N * kScanB];
  __shared__ R she[E::SZ];
  __shared__ R shc[V::SZ];
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* sho = reinterpret_cast<R*>(smem_raw);  // the aggregates, field-major (dynamic)
  const LtiBlockTables<R, N>* Ts = &st->group;
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x;
  const int cnt = (int)g.gpt;
  // interior groups: [ceil(j_lo / B), floor(j_hi / B))
  const int s0 = (int)min((int64_t)cnt, (j_lo + kScanB - 1) / kScanB);
  const int s1 = (int)max((int64_t)s0, min((int64_t)cnt, j_hi / kScanB));
  bool ok = true;
  if (t == 0) {
    V c0;
    set_zero(c0);
    if (gathered) {  // time shards: fold the chunk aggregates of the ranks before this one
      for (int q = 0; q < rank; ++q) {
        E a;
        load(a, gathered + ((int64_t)q * g.batch + b) * E::SZ, 1);
        vapply<R, N, false>(a, c0, c0, nullptr, ok);
      }
      store(c0, carry_out + b * V::SZ, 1);
    }
    store(c0, shc, 1);
  }
  const R* src = group_agg + (b * g.gpt) * E::SZ;
  for (int q = t; q < cnt * E::SZ; q += kScanB) sho[(q % E::SZ) * kScanB + q / E::SZ] = src[q];
  if (t >= cnt) {
    E id;
    set_identity(id);
    store(id, sho + t, kScanB);
  }
  __syncthreads();
  E res;
  lti_block_scan<R, N>(Ts, t, cnt, s0, s1, sho + t, res, shd, she, ok);
  if (t == cnt - 1 && total_agg) store(res, total_agg + b * E::SZ, 1);
  __syncthreads();
  V cin;
  load(cin, shc, 1);
  if (t == 0) store(cin, group_carry + (b * g.gpt) * V::SZ, 1);
  if (t + 1 < cnt) {  // carry of group t + 1 = (groups 0..t) (.) carry_in
    V c;
    vapply<R, N, false>(res, cin, c, nullptr, ok);
    store(c, group_carry + (b * g.gpt + t + 1) * V::SZ, 1);
  }
  if (!ok) flag_node(flag, g.node0);
}

}  // namespace pmap
