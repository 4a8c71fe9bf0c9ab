// nodal.cuh -- the B200-native row-lane kernels (GTS_LAYOUT_NODAL), DESIGN.md §4.
//
// Lanes = rows (R rows per lane, 32R rows per warp).  A block of W warps
// stages one chunk of paths into shared memory; every warp walks all of the
// chunk's paths for its own rows, so each (row, path) pair is one lane's
// private EXTEND/UNWIND of the permutation-weight polynomial (Algorithm 1,
// PAPER.md:54-118), evaluated in the nodal basis:
//
//   U_i = sum_m m!(k-1-m)!/k! [t^m] prod_{s != i} (z_s + o_s t)
//       = int_0^1 prod_{s != i} (z_s + (o_s - z_s) t) dt          (Beta integral)
//       = sum_q w_q P(t_q) / f_i(t_q),  P(t) = prod_s f_s(t)       (Gauss-Legendre,
//                                                                   exact for Q = ceil(k/2))
// EXTEND(s) is "P(t_q) *= f_s(t_q)" at Q nodes (f_s = A_sq when o_s = 1, B_sq
// when o_s = 0; we start from prod A and multiply by rho = B/A for o_s = 0),
// UNWIND(i) is the division by f_i, folded into per-element constants:
//   phi_i = v (o_i - z_i) U_i = sum_q P_q C_iq        (o_i = 1)
//         = sum_q P_q d_q  (same for every o_i = 0)
// Interactions (Eq. 3, conditioning only on path features):
//   phi_ij = sum_q (v w_q P_q / 2) u_iq u_jq,  u = (o - z)/f,
//   phi_ii = sum_q (v w_q P_q / 2) u_iq (2 - sum_j u_jq + u_iq)    (Eq. 6)
//
// Paths of a chunk are ordered by (Q, feature set), so consecutive paths with
// the same feature set ("runs") share slots: their contributions accumulate in
// registers and reach the shared-memory phi tile once per run.
#pragma once
#include "blob_format.h"

namespace gts {
namespace nodal {

extern __shared__ __align__(16) unsigned char g_smem[];

template <int Q>
struct QP_ {
  static constexpr int v = (Q + 3) & ~3;
};

__device__ __forceinline__ int tri_row_base(int a, int S) { return a * (2 * S - a - 1) / 2; }

template <typename T, int N>
__device__ __forceinline__ void lds_vec(T (&dst)[N], const T* src) {
  // src is 16-byte aligned; N <= padded row length
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(src + i);
      dst[i] = v.x;
      if (i + 1 < N) dst[i + 1] = v.y;
      if (i + 2 < N) dst[i + 2] = v.z;
      if (i + 3 < N) dst[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const double2 v = *reinterpret_cast<const double2*>(src + i);
      dst[i] = v.x;
      if (i + 1 < N) dst[i + 1] = v.y;
    }
  }
}

template <typename T>
__device__ __forceinline__ bool one_fraction(T x, int4 rec) {
  // o = [lower <= x < upper]  (half-open bounds, reading G1)
  return (x >= (T)__int_as_float(rec.y)) & (x < (T)__int_as_float(rec.z));
}

// --------------------------------------------------------------------- SHAP

// A run of n_run paths with one feature set; k in {2Q-1, 2Q}; fully unrolled.
template <typename T, int Q, int R>
__device__ __forceinline__ void shap_run(int k, int n_run, const int4* __restrict__ E, const T* __restrict__ tab,
                                         const int (&xb)[R], const int (&ab)[R]) {
  constexpr int QP = QP_<Q>::v, KM = 2 * Q;
  T* const sT = reinterpret_cast<T*>(g_smem);
  const int words = 2 * QP * (k + 1);
  int slot[KM];
  T acc[R][KM], xv[R][KM];  // the run's slots and this lane's x values, loaded once per run
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    slot[s] = (s < KM - 1 || s < k) ? E[s].x : 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r][s] = (T)0;
      xv[r][s] = sT[xb[r] + slot[s]];
    }
  }
  for (int p = 0; p < n_run; ++p) {
    const int4* Ep = E + p * k;
    const T* tp = tab + p * words;
    T P[R][Q];
    {
      T c[Q];
      lds_vec(c, tp);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < Q; ++q) P[r][q] = c[q];
    }
    uint32_t om[R];
#pragma unroll
    for (int r = 0; r < R; ++r) om[r] = 0u;
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        const int4 rec = Ep[s];
        T rho[Q];
        lds_vec(rho, tp + 2 * QP + s * 2 * QP);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool o = one_fraction(xv[r][s], rec);
          if (o) om[r] |= 1u << s;
          if (!o) {
#pragma unroll
            for (int q = 0; q < Q; ++q) P[r][q] *= rho[q];  // EXTEND: f_s = B_s for o_s = 0
          }
        }
      }
    }
    T ph0[R];
    {
      T d[Q];
      lds_vec(d, tp + QP);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        T a = (T)0;
#pragma unroll
        for (int q = 0; q < Q; ++q) a = fma(P[r][q], d[q], a);
        ph0[r] = a;
      }
    }
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        T C[Q];
        lds_vec(C, tp + 2 * QP + s * 2 * QP + QP);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          T a = (T)0;
#pragma unroll
          for (int q = 0; q < Q; ++q) a = fma(P[r][q], C[q], a);  // UNWIND(s) folded into C
          acc[r][s] += ((om[r] >> s) & 1u) ? a : ph0[r];
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < KM; ++s)
    if (s < KM - 1 || s < k)
#pragma unroll
      for (int r = 0; r < R; ++r) sT[ab[r] + slot[s]] += acc[r][s];
}

// One path, element loop not unrolled (large Q); accumulates per element.
template <typename T, int Q, int R>
__device__ __forceinline__ void shap_path_dyn(int k, const int4* __restrict__ E, const T* __restrict__ tab,
                                              const int (&xb)[R], const int (&ab)[R]) {
  constexpr int QP = QP_<Q>::v;
  T* const sT = reinterpret_cast<T*>(g_smem);
  T P[R][Q];
  {
    T c[Q];
    lds_vec(c, tab);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int q = 0; q < Q; ++q) P[r][q] = c[q];
  }
  uint32_t om[R];
#pragma unroll
  for (int r = 0; r < R; ++r) om[r] = 0u;
#pragma unroll 1
  for (int s = 0; s < k; ++s) {
    const int4 rec = E[s];
    T rho[Q];
    lds_vec(rho, tab + 2 * QP + s * 2 * QP);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool o = one_fraction(sT[xb[r] + rec.x], rec);
      om[r] |= (uint32_t)o << s;
      if (!o) {
#pragma unroll
        for (int q = 0; q < Q; ++q) P[r][q] *= rho[q];
      }
    }
  }
  T ph0[R];
  {
    T d[Q];
    lds_vec(d, tab + QP);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      T a = (T)0;
#pragma unroll
      for (int q = 0; q < Q; ++q) a = fma(P[r][q], d[q], a);
      ph0[r] = a;
    }
  }
#pragma unroll 1
  for (int s = 0; s < k; ++s) {
    const int sl = E[s].x;
    T C[Q];
    lds_vec(C, tab + 2 * QP + s * 2 * QP + QP);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      T a = (T)0;
#pragma unroll
      for (int q = 0; q < Q; ++q) a = fma(P[r][q], C[q], a);
      sT[ab[r] + sl] += ((om[r] >> s) & 1u) ? a : ph0[r];
    }
  }
}

// ------------------------------------------------------------- interactions

// P(t_q) for one path and R rows; returns the o-bits.
template <typename T, int Q, int R, bool kUnroll>
__device__ __forceinline__ void inter_extend(int k, const int4* __restrict__ E, const T* __restrict__ tp,
                                             const int (&xb)[R], T (&P)[R][Q], uint32_t (&om)[R]) {
  constexpr int QP = QP_<Q>::v, KM = 2 * Q;
  T* const sT = reinterpret_cast<T*>(g_smem);
  {
    T c[Q];
    lds_vec(c, tp);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int q = 0; q < Q; ++q) P[r][q] = c[q];
  }
#pragma unroll
  for (int r = 0; r < R; ++r) om[r] = 0u;
  auto body = [&](int s) {
    const int4 rec = E[s];
    T rho[Q];
    lds_vec(rho, tp + 2 * QP + s * 2 * QP);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool o = one_fraction(sT[xb[r] + rec.x], rec);
      om[r] |= (uint32_t)o << s;
      if (!o) {
#pragma unroll
        for (int q = 0; q < Q; ++q) P[r][q] *= rho[q];
      }
    }
  };
  if constexpr (kUnroll) {
#pragma unroll
    for (int s = 0; s < KM; ++s)
      if (s < KM - 1 || s < k) body(s);
  } else {
#pragma unroll 1
    for (int s = 0; s < k; ++s) body(s);
  }
}

// A run of paths with one feature set (k in {2Q-1, 2Q}, fully unrolled).  Per
// path and row: P by EXTEND, u_s = (o_s - z_s)/f_s at every node (cached in
// registers), phi_ij = sum_q W_q u_iq u_jq for i < j, and the diagonal by
// Eq. 6 from row sums: phi_ii = phi_i - sum_{j != i} phi_ij with
// phi_i = 2 sum_q W_q u_iq.  kRegAcc: the run's cells accumulate in registers
// and reach the shared tile once per run (small Q); otherwise per path.
template <typename T, int Q, int R, bool kRegAcc>
__device__ __forceinline__ void inter_run(int k, int n_run, const int4* __restrict__ E, const T* __restrict__ tab,
                                          const T* __restrict__ gam, const int (&xb)[R], const int (&ab)[R]) {
  constexpr int QP = QP_<Q>::v, KM = 2 * Q, NC = KM * (KM + 1) / 2;
  T* const sT = reinterpret_cast<T*>(g_smem);
  const int words = 2 * QP * (k + 1);
  T G[Q];
  lds_vec(G, gam);
  int slot[KM], rb[KM];
  T xv[R][KM];
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    const bool valid = (s < KM - 1 || s < k);
    const int4 e = valid ? E[s] : make_int4(0, 0, 0, 0);
    slot[s] = e.x;
    rb[s] = e.w;
#pragma unroll
    for (int r = 0; r < R; ++r) xv[r][s] = sT[xb[r] + e.x];
  }
  T acc[R][kRegAcc ? NC : 1];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < (kRegAcc ? NC : 1); ++c) acc[r][c] = (T)0;
  auto add = [&](int r, int c, int i, int j, T v) {
    if constexpr (kRegAcc) acc[r][c] += v;
    else sT[ab[r] + rb[i] + slot[j]] += v;
  };
  for (int p = 0; p < n_run; ++p) {
    const int4* Ep = E + p * k;
    const T* tp = tab + p * words;
    T P[R][Q];
    uint32_t om[R];
    {
      T c0[Q];
      lds_vec(c0, tp);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        om[r] = 0u;
#pragma unroll
        for (int q = 0; q < Q; ++q) P[r][q] = c0[q];
      }
    }
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        const int4 rec = Ep[s];
        T rho[Q];
        lds_vec(rho, tp + 2 * QP + s * 2 * QP);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool o = one_fraction(xv[r][s], rec);
          if (o) om[r] |= 1u << s;
          if (!o) {
#pragma unroll
            for (int q = 0; q < Q; ++q) P[r][q] *= rho[q];  // EXTEND at the nodes
          }
        }
      }
    }
    T W[R][Q];
    {
      T h[Q];
      lds_vec(h, tp + QP);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < Q; ++q) W[r][q] = h[q] * P[r][q];
    }
    T u[R][KM][Q];
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        T al[Q];
        lds_vec(al, tp + 2 * QP + s * 2 * QP + QP);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool o = (om[r] >> s) & 1u;
#pragma unroll
          for (int q = 0; q < Q; ++q) u[r][s][q] = o ? al[q] : G[q];  // UNWIND(s) folded into u
        }
      }
    }
    int c = 0;
#pragma unroll
    for (int i = 0; i < KM; ++i) {
      if (i < KM - 1 || i < k) {
        T y[R][Q], phi[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          T a = (T)0;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            y[r][q] = W[r][q] * u[r][i][q];
            a += y[r][q];
          }
          phi[r] = a + a;  // phi_i
        }
        const int cdiag = c++;
#pragma unroll
        for (int j = i + 1; j < KM; ++j) {
          if (j < KM - 1 || j < k) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              T v = (T)0;
#pragma unroll
              for (int q = 0; q < Q; ++q) v = fma(y[r][q], u[r][j][q], v);
              add(r, c, i, j, v);
            }
          }
          ++c;
        }
        // the diagonal cell collects phi_i; Eq. 6 subtracts the row sums when
        // the tile is flushed (linear in the paths, so it holds per tile)
#pragma unroll
        for (int r = 0; r < R; ++r) add(r, cdiag, i, i, phi[r]);
      } else {
        c += KM - i;
      }
    }
  }
  if constexpr (kRegAcc) {
    int c = 0;
#pragma unroll
    for (int i = 0; i < KM; ++i) {
#pragma unroll
      for (int j = i; j < KM; ++j) {
        if ((i < KM - 1 || i < k) && (j < KM - 1 || j < k))
#pragma unroll
          for (int r = 0; r < R; ++r) sT[ab[r] + rb[i] + slot[j]] += acc[r][c];
        ++c;
      }
    }
  }
}

// One path, pair cells accumulated straight into the shared tile.
template <typename T, int Q, int R, bool kUnroll>
__device__ __forceinline__ void inter_path(int k, const int4* __restrict__ E, const T* __restrict__ tp,
                                           const T* __restrict__ gam, const int (&xb)[R], const int (&ab)[R]) {
  constexpr int QP = QP_<Q>::v, KM = 2 * Q;
  T* const sT = reinterpret_cast<T*>(g_smem);
  T G[Q];
  lds_vec(G, gam);
  T P[R][Q];
  uint32_t om[R];
  inter_extend<T, Q, R, kUnroll>(k, E, tp, xb, P, om);
  T W[R][Q];
  {
    T h[Q];
    lds_vec(h, tp + QP);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int q = 0; q < Q; ++q) W[r][q] = h[q] * P[r][q];
  }
#pragma unroll 1
  for (int i = 0; i < k; ++i) {
    const int4 ri = E[i];
    T ai[Q];
    lds_vec(ai, tp + 2 * QP + i * 2 * QP + QP);
    T y[R][Q], yg[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool oi = (om[r] >> i) & 1u;
      T phi = (T)0, g = (T)0;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const T u = oi ? ai[q] : G[q];
        y[r][q] = W[r][q] * u;
        phi += y[r][q];
        g = fma(y[r][q], G[q], g);
      }
      yg[r] = g;
      sT[ab[r] + ri.w + ri.x] += phi + phi;  // phi_i; Eq. 6 applied at flush
    }
#pragma unroll 1
    for (int j = i + 1; j < k; ++j) {
      const int cell = ri.w + E[j].x;
      T aj[Q];
      lds_vec(aj, tp + 2 * QP + j * 2 * QP + QP);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        T s1 = (T)0;
#pragma unroll
        for (int q = 0; q < Q; ++q) s1 = fma(y[r][q], aj[q], s1);
        sT[ab[r] + cell] += ((om[r] >> j) & 1u) ? s1 : yg[r];
      }
    }
  }
}

// ------------------------------------------------------------- dispatch

// Small Q: all R rows of the lane at once (shared table loads, R-way ILP).
// Larger Q: the lane's rows one after the other, which bounds the register
// footprint of the whole kernel by the small-Q instantiations.
template <typename T, int R, bool kInter>
__device__ __forceinline__ void run_dispatch(int4 ph, const int4* __restrict__ E0, const T* __restrict__ table,
                                             const T* __restrict__ gauss, const int (&xb)[R], const int (&ab)[R]) {
  const int k = ph.x & 0xff, n_run = ph.x >> 16, q = ph.y;
  const int4* E = E0 + ph.z;
  const T* tab = table + ph.w;
  const int words = 2 * ((q + 3) & ~3) * (k + 1);
  if constexpr (!kInter) {
    switch (q) {
#define GTS_RUN(QQ) case QQ: shap_run<T, QQ, R>(k, n_run, E, tab, xb, ab); break;
      GTS_RUN(1) GTS_RUN(2) GTS_RUN(3) GTS_RUN(4)
#undef GTS_RUN
      default:
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
          const int xb1[1] = {xb[r]}, ab1[1] = {ab[r]};
          switch (q) {
#define GTS_RUN1(QQ) case QQ: shap_run<T, QQ, 1>(k, n_run, E, tab, xb1, ab1); break;
            GTS_RUN1(5) GTS_RUN1(6) GTS_RUN1(7) GTS_RUN1(8)
#undef GTS_RUN1
            default:
              for (int p = 0; p < n_run; ++p) {
                switch (q) {
#define GTS_DYN(QQ) case QQ: shap_path_dyn<T, QQ, 1>(k, E + p * k, tab + p * words, xb1, ab1); break;
                  GTS_DYN(9) GTS_DYN(10) GTS_DYN(11) GTS_DYN(12) GTS_DYN(13) GTS_DYN(14) GTS_DYN(15) GTS_DYN(16)
#undef GTS_DYN
                  default: break;
                }
              }
          }
        }
    }
  } else {
    const T* gam = gauss + (q - 1) * 3 * kQMax + 2 * kQMax;
    switch (q) {
      case 1: inter_run<T, 1, R, true>(k, n_run, E, tab, gam, xb, ab); break;
      case 2: inter_run<T, 2, R, true>(k, n_run, E, tab, gam, xb, ab); break;
      default:
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
          const int xb1[1] = {xb[r]}, ab1[1] = {ab[r]};
          switch (q) {
            case 3: inter_run<T, 3, 1, true>(k, n_run, E, tab, gam, xb1, ab1); break;
            case 4: inter_run<T, 4, 1, false>(k, n_run, E, tab, gam, xb1, ab1); break;
            case 5: inter_run<T, 5, 1, false>(k, n_run, E, tab, gam, xb1, ab1); break;
            case 6:
              if constexpr (sizeof(T) == 4) { inter_run<T, 6, 1, false>(k, n_run, E, tab, gam, xb1, ab1); break; }
              [[fallthrough]];
            case 7:
              if constexpr (sizeof(T) == 4) {
                if (q == 7) { inter_run<T, 7, 1, false>(k, n_run, E, tab, gam, xb1, ab1); break; }
              }
              [[fallthrough]];
            default:
              for (int p = 0; p < n_run; ++p) {
                switch (q) {
#define GTS_IP(QQ) case QQ: inter_path<T, QQ, 1, false>(k, E + p * k, tab + p * words, gam, xb1, ab1); break;
                  GTS_IP(6) GTS_IP(7) GTS_IP(8) GTS_IP(9) GTS_IP(10) GTS_IP(11) GTS_IP(12) GTS_IP(13)
                  GTS_IP(14) GTS_IP(15) GTS_IP(16)
#undef GTS_IP
                  default: break;
                }
              }
          }
        }
    }
  }
}

// ------------------------------------------------------------------ kernel

struct Args {
  const char* blob;
  const void* X;
  int64_t n_rows, ld_x;
  void* out;
  int n_splits;
  int M, G;
  int64_t n_chunks;
  int max_elems, max_paths, max_words;
};

template <bool kInter>
__host__ __device__ constexpr int acc_width(int S) { return kInter ? S * (S + 1) / 2 : S; }

template <typename T, int S, int R, bool kInter>
__host__ __device__ constexpr int tile_words_per_warp() {
  return R * 32 * ((S + 1) + (acc_width<kInter>(S) | 1));
}

// Launch shape per (dtype, kernel, slot width): R rows per lane and W warps
// per block, chosen so that two blocks (tiles + chunk staging) share an SM.
template <typename T, bool kInter, int S>
struct Cfg {
  static constexpr int R = (sizeof(T) == 4 && (kInter ? S <= 8 : S <= 16)) ? 2 : 1;
  static constexpr int tile_bytes = (int)sizeof(T) * tile_words_per_warp<T, S, R, kInter>();
  static constexpr int W = tile_bytes * 8 <= 74 * 1024 ? 8 : (tile_bytes * 4 <= 80 * 1024 ? 4 : 2);
  static constexpr int kMinBlocks = 2;
};

// shared-memory layout (T words unless noted): gauss | X tiles | phi tiles | table | elems (int4) | paths (int4)
template <typename T, int S, int W, int R, bool kInter>
__host__ __device__ constexpr int table_word_offset() {
  return ((kQMax * 3 * kQMax + W * tile_words_per_warp<T, S, R, kInter>()) + 3) & ~3;
}

// Stage chunk c: element records, path headers, nodal tables (computed in fp64
// from the blob's fp64 zero fractions, rounded once to T).
template <typename T, bool kInter>
__device__ __forceinline__ void stage_chunk(const ChunkRec& c, const PathRec* __restrict__ gpaths,
                                            const ElemRec* __restrict__ gelems, int S, int o_table, int b_elem,
                                            int b_path, int nwarps) {
  T* const sT = reinterpret_cast<T*>(g_smem);
  int4* const sE = reinterpret_cast<int4*>(g_smem + b_elem);
  int4* const sP = reinterpret_cast<int4*>(g_smem + b_path);
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int e = tid; e < c.n_elems; e += nth) {
    const ElemRec er = gelems[c.elem_begin + e];
    sE[e] = make_int4(er.slot, __float_as_int(er.lo), __float_as_int(er.hi), tri_row_base(er.slot, S));
  }
  for (int p = tid; p < c.n_paths; p += nth) {
    const PathRec pr = gpaths[c.path_begin + p];
    sP[p] = make_int4(pr.k, pr.q, pr.elem, pr.table);  // pr.k holds k | run_len << 16
  }
  const int warp = tid >> 5, lane = tid & 31;
  const T* gauss = sT;
  for (int p = warp; p < c.n_paths; p += nwarps) {
    const PathRec pr = gpaths[c.path_begin + p];
    const int k = pr.k & 0xff, Q = pr.q, QP = (Q + 3) & ~3;
    const ElemRec* el = gelems + c.elem_begin + pr.elem;
    T* tab = sT + o_table + pr.table;
    const T* g = gauss + (Q - 1) * 3 * kQMax;
    for (int idx = lane; idx < k * Q; idx += 32) {
      const int s = idx / Q, q = idx - s * Q;
      const double z = el[s].z, t = (double)g[q];
      const double A = z + (1.0 - z) * t;  // f_s(t_q), o_s = 1
      const double B = z * (1.0 - t);      // f_s(t_q), o_s = 0
      T* row = tab + 2 * QP + s * 2 * QP;
      row[q] = (T)(B / A);                 // rho
      if (kInter) row[QP + q] = (T)((1.0 - z) / A);                          // alpha
      else row[QP + q] = (T)(pr.v * (double)g[kQMax + q] * (1.0 - z) / A);   // C
    }
    if (lane < Q) {
      const int q = lane;
      const double t = (double)g[q], w = (double)g[kQMax + q];
      double cq = 1.0;
      for (int s = 0; s < k; ++s) {
        const double z = el[s].z;
        cq *= z + (1.0 - z) * t;
      }
      tab[q] = (T)cq;
      if (kInter) tab[QP + q] = (T)(0.5 * pr.v * w);
      else tab[QP + q] = (T)(-pr.v * w / (1.0 - t));
    }
  }
}

template <typename T, int S, int W, int R, bool kInter>
__global__ void __launch_bounds__(W * 32, (W >= 8 ? 2 : 1)) nodal_kernel(Args a) {
  constexpr int XS = S + 1;
  constexpr int AW = acc_width<kInter>(S);
  constexpr int AS = AW | 1;
  constexpr int ROWS = 32 * R;
  constexpr int o_x = kQMax * 3 * kQMax;
  constexpr int o_acc = o_x + W * ROWS * XS;
  constexpr int o_table = table_word_offset<T, S, W, R, kInter>();
  const int b_elem = (o_table + a.max_words) * (int)sizeof(T);
  const int b_path = b_elem + 16 * a.max_elems;

  const BlobHeader* hdr = reinterpret_cast<const BlobHeader*>(a.blob);
  const ChunkRec* chunks = reinterpret_cast<const ChunkRec*>(a.blob + hdr->off_units);
  const double* work = reinterpret_cast<const double*>(a.blob + hdr->off_work) + (kInter ? (a.n_chunks + 1) : 0);
  const int32_t* slotmap = reinterpret_cast<const int32_t*>(a.blob + hdr->off_slotmap);
  const PathRec* gpaths = reinterpret_cast<const PathRec*>(a.blob + hdr->off_paths);
  const ElemRec* gelems = reinterpret_cast<const ElemRec*>(a.blob + hdr->off_elems);
  const T* X = static_cast<const T*>(a.X);
  T* out = static_cast<T*>(a.out);
  T* const sT = reinterpret_cast<T*>(g_smem);
  const int4* const sE = reinterpret_cast<const int4*>(g_smem + b_elem);
  const int4* const sP = reinterpret_cast<const int4*>(g_smem + b_path);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row_tile = blockIdx.x / a.n_splits;
  const int split = blockIdx.x % a.n_splits;
  const int64_t row0 = row_tile * (W * ROWS) + (int64_t)warp * ROWS;

  const double wtot = work[a.n_chunks];
  auto split_begin = [&](int s) -> int64_t {
    if (s >= a.n_splits) return a.n_chunks;
    const double target = wtot * (double)s / (double)a.n_splits;
    int64_t lo = 0, hi = a.n_chunks;  // first c with work[c] >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (work[mid] < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  const int64_t c_begin = split_begin(split), c_end = split_begin(split + 1);

  const T* gsrc = reinterpret_cast<const T*>(a.blob + hdr->off_gauss);
  for (int i = tid; i < kQMax * 3 * kQMax; i += blockDim.x) sT[i] = gsrc[i];
  int xb[R], ab[R];
  int64_t row[R];
  bool ok[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int lr = warp * ROWS + r * 32 + lane;
    xb[r] = o_x + lr * XS;
    ab[r] = o_acc + lr * AS;
    row[r] = row0 + r * 32 + lane;
    ok[r] = row[r] < a.n_rows;
    for (int i = 0; i < AW; ++i) sT[ab[r] + i] = (T)0;
  }
  const int M1 = a.M + 1;
  int cur_map = -1, cur_group = -1, cur_slots = 0;
  int64_t cur_map_begin = 0;
  bool dirty = false;

  // one atomic per non-zero (row, group, feature) cell of this lane's tiles
  auto flush = [&]() {
    if (dirty) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!ok[r]) continue;
        if constexpr (kInter) {
          T* base = out + ((size_t)row[r] * a.G + cur_group) * (size_t)M1 * M1;
          for (int i = 0; i < cur_slots; ++i) {
            // the diagonal cell holds sum phi_i; Eq. 6: phi_ii = phi_i - sum_{j != i} phi_ij
            T rowsum = (T)0;
            for (int j = 0; j < cur_slots; ++j)
              if (j != i) rowsum += sT[ab[r] + (j < i ? tri_row_base(j, S) + i : tri_row_base(i, S) + j)];
            const int fi = slotmap[cur_map_begin + i];
            const T d = sT[ab[r] + tri_row_base(i, S) + i] - rowsum;
            if (d != (T)0) atomicAdd(base + (size_t)fi * M1 + fi, d);
          }
          for (int i = 0; i < cur_slots; ++i) {
            const int fi = slotmap[cur_map_begin + i];
            const int rb = tri_row_base(i, S);
            sT[ab[r] + rb + i] = (T)0;
            for (int j = i + 1; j < cur_slots; ++j) {
              const T v = sT[ab[r] + rb + j];
              if (v != (T)0) {
                const int fj = slotmap[cur_map_begin + j];
                atomicAdd(base + (size_t)fi * M1 + fj, v);
                atomicAdd(base + (size_t)fj * M1 + fi, v);
                sT[ab[r] + rb + j] = (T)0;
              }
            }
          }
        } else {
          T* base = out + ((size_t)row[r] * a.G + cur_group) * (size_t)M1;
          for (int i = 0; i < cur_slots; ++i) {
            const T v = sT[ab[r] + i];
            if (v != (T)0) {
              atomicAdd(base + slotmap[cur_map_begin + i], v);
              sT[ab[r] + i] = (T)0;
            }
          }
        }
      }
    }
    dirty = false;
  };

  for (int64_t ci = c_begin; ci < c_end; ++ci) {
    const ChunkRec c = chunks[ci];
    __syncthreads();  // previous chunk's tables no longer in use
    stage_chunk<T, kInter>(c, gpaths, gelems, S, o_table, b_elem, b_path, W);
    if (c.map_id != cur_map || c.group != cur_group) {
      flush();
      if (c.map_id != cur_map) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          for (int i = 0; i < c.n_slots; ++i)
            sT[xb[r] + i] = ok[r] ? X[(size_t)row[r] * a.ld_x + slotmap[c.slotmap_begin + i]] : (T)0;
      }
      cur_map = c.map_id;
      cur_group = c.group;
      cur_slots = c.n_slots;
      cur_map_begin = c.slotmap_begin;
    }
    __syncthreads();  // tables staged
    if (row0 < a.n_rows) {
      for (int p = 0; p < c.n_paths;) {
        const int4 ph = sP[p];
        run_dispatch<T, R, kInter>(ph, sE, sT + o_table, sT, xb, ab);
        p += ph.x >> 16;
      }
      dirty = true;
    }
  }
  flush();
}

}  // namespace nodal
}  // namespace gts
