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
// (the table stores C' = C - d, see shap_run)
// Interactions (Eq. 3, conditioning only on path features):
//   phi_ij = sum_q (v w_q P_q / 2) u_iq u_jq,  u = (o - z)/f,
//   phi_ii = sum_q (v w_q P_q / 2) u_iq (2 - sum_j u_jq + u_iq)    (Eq. 6)
//
// Paths of a chunk are ordered by (Q, feature set), so consecutive paths with
// the same feature set ("runs") share slots: their contributions accumulate in
// registers and reach the shared-memory phi tile once per run.
#pragma once
#include "blob_format.h"

#ifndef GTS_X2
#define GTS_X2 1  // fp32 SHAP runs on paired Gauss nodes (FFMA2 / FMUL2)
#endif
#ifndef GTS_INTER_R8
#define GTS_INTER_R8 1  // rows per lane of the fp32 interaction kernel with 8 slots
                        // (measured: 1 row, 8 warps per block beats 2 rows, 4 warps by 8 %; profiles/r01h)
#endif
#ifndef GTS_INTER_PAIRED
#define GTS_INTER_PAIRED ((1 << 2) | (1 << 4))  // bit Q: fp32 interaction runs with Q nodes use paired
                                                // Gauss nodes (inter_run_q2).  Measured: Q = 4 +3 % cal_housing,
                                                // +10 % adult (profiles/r01i); Q = 2 another +3 % cal_housing;
                                                // Q = 3 (pair + scalar tail) -4 %, padded to 4 nodes -14 %
                                                // (profiles/r01n, r01i)
#endif
#ifndef GTS_INTER_CACHEU_QMAX
#define GTS_INTER_CACHEU_QMAX 5  // interaction runs up to this Q keep u_sq of every element in registers
                                 // (5 over 4: adult-large both +11 %, covtype interactions +5 %, profiles/r02k)
                                 // (measured in a session lost with the earlier container: 5, 6, 7 cost adult 12-16 %; a paired-node
                                 // per-path variant for Q >= 5 cost 28 %)
#endif
#ifndef GTS_INTER_RMW_BLOCK
#define GTS_INTER_RMW_BLOCK 4  // interaction runs without register cells: tile read-modify-writes per block of cells
#endif
#ifndef GTS_INTER_REGACC
#define GTS_INTER_REGACC 0  // bit Q: interaction runs with Q nodes keep the run's pair cells in registers
#endif
#ifndef GTS_X2_R2_QMAX
#define GTS_X2_R2_QMAX 6  // largest Q whose paired-node SHAP run keeps both rows of a lane in flight
                          // (measured: adult SHAP +19 % for 6 over 4; profiles/r01h)
#endif
#ifndef GTS_SHAP_R_WIDE
#define GTS_SHAP_R_WIDE 1  // rows per lane of the fp32 SHAP kernel with 32 or 64 slots
#endif
#ifndef GTS_SHAP_R8
#define GTS_SHAP_R8 4  // rows per lane of the fp32 SHAP kernel with 8 slots (measured: 4 > 2)
#endif

namespace gts {
namespace nodal {

extern __shared__ __align__(16) unsigned char g_smem[];

#ifndef GTS_RMW_REGS
#define GTS_RMW_REGS 8  // registers per lane for grouped tile read-modify-writes (R rows x cells)
#endif

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

// N float2 pairs from a 16-byte aligned row (table rows are padded to 4 words):
// LDS.128 per two pairs instead of LDS.64 per pair.
template <int N>
__device__ __forceinline__ void lds_pairs(float2 (&dst)[N], const float* src) {
#pragma unroll
  for (int h = 0; h < N; h += 2) {
    const float4 v = *reinterpret_cast<const float4*>(src + 2 * h);
    dst[h] = make_float2(v.x, v.y);
    if (h + 1 < N) dst[h + 1] = make_float2(v.z, v.w);
  }
}

// Offsets (T words) inside a path's nodal table (blob_format.h): element s's
// rho row (with the split bounds at BO), its C' row (SHAP) and alpha row
// (interactions; NT = 3).
template <int Q, int NT>
struct Lay {
  static constexpr bool kInRow = (Q & 3) == 1 || (Q & 3) == 2;
  static constexpr int QP = (Q + 3) & ~3, BO = (Q + 1) & ~1, RW = kInRow ? (BO + 2 + 3) & ~3 : QP,
                       BW = kInRow ? 0 : 4 * Q, ES = RW + (NT - 1) * QP;
  static_assert(kInRow == nodal_inrow(Q) && BO == nodal_bo(Q) && RW == nodal_rw(Q) && BW == nodal_bw(Q) &&
                    ES == nodal_es(Q, NT),
                "table layout");
  __device__ static __forceinline__ int bnd(int s) { return NT * QP + 2 * s; }  // bounds block (!kInRow)
  __device__ static __forceinline__ int rho(int s) { return NT * QP + BW + s * ES; }
  __device__ static __forceinline__ int cp(int s) { return rho(s) + RW; }
  __device__ static __forceinline__ int al(int s) { return rho(s) + RW + QP; }
};

// 16 bytes of bounds: two fp32 elements' {lo, hi} or one fp64 element's
template <typename T>
struct BQ;
template <>
struct BQ<float> { using type = float4; };
template <>
struct BQ<double> { using type = double2; };

// The first NW words of a 16-byte aligned row by 16-byte loads (an 8-byte
// load for a trailing pair of fp32 words).
template <typename T, int NW>
__device__ __forceinline__ void lds_words(T (&w)[NW], const T* src) {
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < NW; i += 4) {
      if (i + 4 <= NW) {
        const float4 v = *reinterpret_cast<const float4*>(src + i);
        w[i] = v.x, w[i + 1] = v.y, w[i + 2] = v.z, w[i + 3] = v.w;
      } else {
        const float2 v = *reinterpret_cast<const float2*>(src + i);
        w[i] = v.x, w[i + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < NW; i += 2) {
      const double2 v = *reinterpret_cast<const double2*>(src + i);
      w[i] = v.x, w[i + 1] = v.y;
    }
  }
}

// The split bounds of element s from the bounds block (fp32: one 16-byte load
// for elements s, s + 1, kept in bq -- callers walk s upwards from 0).
template <typename T, int Q, int NT>
__device__ __forceinline__ void lds_bounds(T& lo, T& hi, const T* tp, int s, typename BQ<T>::type& bq) {
  using L = Lay<Q, NT>;
  if constexpr (sizeof(T) == 4) {
    if ((s & 1) == 0) bq = *reinterpret_cast<const float4*>(tp + L::bnd(s));
    lo = (s & 1) ? bq.z : bq.x;
    hi = (s & 1) ? bq.w : bq.y;
  } else {
    bq = *reinterpret_cast<const double2*>(tp + L::bnd(s));
    lo = bq.x;
    hi = bq.y;
  }
}

// rho_s at the Q nodes and the split bounds of element s of the path table at tp.
template <typename T, int Q, int NT>
__device__ __forceinline__ void lds_rho(T (&rho)[Q], T& lo, T& hi, const T* tp, int s, typename BQ<T>::type& bq) {
  using L = Lay<Q, NT>;
  if constexpr (L::kInRow) {
    T w[L::BO + 2];
    lds_words(w, tp + L::rho(s));
#pragma unroll
    for (int q = 0; q < Q; ++q) rho[q] = w[q];
    lo = w[L::BO];
    hi = w[L::BO + 1];
  } else {
    lds_vec(rho, tp + L::rho(s));
    lds_bounds<T, Q, NT>(lo, hi, tp, s, bq);
  }
}

// fp32: rho_s on packed node pairs (odd Q: the zero pad completes the last pair) and the bounds.
template <int Q, int NT>
__device__ __forceinline__ void lds_rho_pairs(float2 (&rh)[(Q + 1) / 2], float& lo, float& hi, const float* tp, int s,
                                              float4& bq) {
  using L = Lay<Q, NT>;
  if constexpr (L::kInRow) {
    float w[L::BO + 2];
    lds_words(w, tp + L::rho(s));
#pragma unroll
    for (int h = 0; h < (Q + 1) / 2; ++h) rh[h] = make_float2(w[2 * h], w[2 * h + 1]);
    lo = w[L::BO];
    hi = w[L::BO + 1];
  } else {
    lds_pairs(rh, tp + L::rho(s));
    lds_bounds<float, Q, NT>(lo, hi, tp, s, bq);
  }
}

template <typename T>
__device__ __forceinline__ bool in_bounds(T x, T lo, T hi) {
  return (x >= lo) & (x < hi);  // o = [lower <= x < upper]  (reading G1)
}

template <typename T>
__device__ __forceinline__ bool one_fraction(T x, int4 rec) {
  // o = [lower <= x < upper]  (half-open bounds, reading G1)
  return (x >= (T)__int_as_float(rec.x)) & (x < (T)__int_as_float(rec.y));
}

// x value of lane-row xb for element record rec: from the warp's shared X
// tile (xb = tile row base, rec.z = slot), or, for kXg kernels, straight from
// a feature-major copy of X in global memory (xb = the row, rec.w = the
// feature; consecutive lanes read consecutive rows of one feature: one
// coalesced, L1-resident line per warp instruction; the launcher keeps
// feature * cs + row within 32 bits).  SHAP-only records (NT = 2) hold the
// slot as a byte offset into a tile row.
// kXg = 2 (fp32 SHAP with identity maps of <= 64 features): the block's X
// rows live in tensor memory (TMEM, 12-cycle loads instead of L2 misses: the
// L1 left beside three blocks' shared memory cannot hold their X rows); each
// thread owns one TMEM lane, its row r's features at columns r * 64 + f, so
// cs = the warp's TMEM address (lane quarter) and xb = r * 64.
//
// tcgen05.ld / st (.sync.aligned: warp-uniform control flow only, which the
// row-lane runs are) complete asynchronously: tm_wait_ld, then tm_pin on each
// loaded value, so that no use of it is scheduled above the wait.
__device__ __forceinline__ float tm_ld(uint32_t taddr) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
  return __uint_as_float(v);
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_pin(float& v) { asm volatile("" : "+f"(v)); }
__device__ __forceinline__ void tm_pin(double& v) { asm volatile("" : "+d"(v)); }
__device__ __forceinline__ void tm_st(uint32_t taddr, float v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(__float_as_uint(v)) : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// TMEM column of an element's x within its row's block: the feature (kXg = 2,
// identity maps) or the slot (kXg = 3, per-chunk maps; NT = 2 records hold the
// slot's byte offset).
template <typename T, int kXg>
__device__ __forceinline__ int tm_col(int4 rec) {
  return kXg == 2 ? rec.w : rec.z / (int)sizeof(T);
}

template <typename T, int NT, int kXg>
__device__ __forceinline__ T load_x(const T* sT, int xb, int4 rec, const T* __restrict__ xg, int cs) {
  if constexpr (kXg >= 2) {
    T v = (T)tm_ld((uint32_t)cs + (uint32_t)(xb + tm_col<T, kXg>(rec)));
    tm_wait_ld();
    tm_pin(v);
    return v;
  } else if constexpr (kXg) {
    return __ldg(xg + (uint32_t)(rec.w * cs + xb));
  } else {
    return sT[xb + (NT == 2 ? rec.z / (int)sizeof(T) : rec.z)];
  }
}

// The phi tile cell of lane-row ab (word index of its tile row) at a slot
// (NT = 2: byte offset; else word index).
template <typename T, int NT>
__device__ __forceinline__ T& tile_at(int ab, int slot) {
  if constexpr (NT == 2) return *reinterpret_cast<T*>(g_smem + ab * (int)sizeof(T) + slot);
  else return reinterpret_cast<T*>(g_smem)[ab + slot];
}

// --------------------------------------------------------------------- SHAP

// A run of n_run paths with one feature set; k in {2Q-1, 2Q}; fully unrolled.
// UNWIND is folded into the table as C'_sq = C_sq - d_q, so that
//   phi_s = ph0 + o_s sum_q P_q C'_sq,   ph0 = sum_q P_q d_q,
// i.e. an o_s = 1 element costs one predicated FMA chain straight into its
// accumulator and an o_s = 0 element costs nothing; ph0 is summed once per
// path into one register per row and added to every slot of the run at its end.
template <typename T, int Q, int R, int NT, int kXg>
__device__ __forceinline__ void shap_run(int k, int n_run, const int4* __restrict__ E, const T* __restrict__ tab,
                                         const int (&xb)[R], const int (&ab)[R], const T* __restrict__ xg, int cs) {
  constexpr int QP = QP_<Q>::v, KM = 2 * Q;
  constexpr int kRmw = GTS_RMW_REGS / R > 1 ? GTS_RMW_REGS / R : 1;
  T* const sT = reinterpret_cast<T*>(g_smem);
  const int words = nodal_path_words(k, Q, NT);
  T acc[R][KM], xv[R][KM], ph0[R];  // this lane's x values, loaded once per run
#pragma unroll
  for (int r = 0; r < R; ++r) ph0[r] = (T)0;
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    const bool valid = (s < KM - 1 || s < k);
    const int4 e = valid ? E[s] : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r][s] = (T)0;
      if constexpr (kXg >= 2) xv[r][s] = (T)tm_ld((uint32_t)cs + (uint32_t)(xb[r] + tm_col<T, kXg>(e)));
      else if constexpr (kXg) xv[r][s] = __ldg(xg + (uint32_t)(e.w * cs + xb[0]) + r * 32);  // a lane's rows: 32 apart
      else xv[r][s] = sT[xb[r] + (NT == 2 ? e.z / (int)sizeof(T) : e.z)];
    }
  }
  if constexpr (kXg >= 2) {
    tm_wait_ld();
#pragma unroll
    for (int s = 0; s < KM; ++s)
#pragma unroll
      for (int r = 0; r < R; ++r) tm_pin(xv[r][s]);
  }
  using L = Lay<Q, NT>;
  for (int p = 0; p < n_run; ++p) {
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
    typename BQ<T>::type bq;
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        T rho[Q], lo, hi;
        lds_rho<T, Q, NT>(rho, lo, hi, tp, s, bq);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool o = in_bounds(xv[r][s], lo, hi);
          om[r] |= (uint32_t)o << s;
          if (!o) {
#pragma unroll
            for (int q = 0; q < Q; ++q) P[r][q] *= rho[q];  // EXTEND: f_s = B_s for o_s = 0
          }
        }
      }
    }
    {
      T d[Q];
      lds_vec(d, tp + QP);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < Q; ++q) ph0[r] = fma(P[r][q], d[q], ph0[r]);
    }
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        T C[Q];
        lds_vec(C, tp + L::cp(s));
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if ((om[r] >> s) & 1u) {
#pragma unroll
            for (int q = 0; q < Q; ++q) acc[r][s] = fma(P[r][q], C[q], acc[r][s]);  // UNWIND(s) folded into C'
          }
        }
      }
    }
  }
  // The run's slots are distinct features (merged paths), so the tile cells are
  // updated in groups of kRmw: kRmw loads, then kRmw stores, instead of each
  // read-modify-write waiting for the previous store (the compiler cannot
  // prove runtime slots distinct, so it keeps them in program order).  The
  // slots are re-read from the run head's records here rather than held in
  // registers through the run.
#pragma unroll
  for (int s0 = 0; s0 < KM; s0 += kRmw) {
    T old[R][kRmw];
    int slot[kRmw];
#pragma unroll
    for (int b = 0; b < kRmw; ++b) {
      const int s = s0 + b;
      if (s < KM && (s < KM - 1 || s < k)) {
        slot[b] = E[s].z;
#pragma unroll
        for (int r = 0; r < R; ++r) old[r][b] = tile_at<T, NT>(ab[r], slot[b]);
      }
    }
#pragma unroll
    for (int b = 0; b < kRmw; ++b) {
      const int s = s0 + b;
      if (s < KM && (s < KM - 1 || s < k))
#pragma unroll
        for (int r = 0; r < R; ++r) tile_at<T, NT>(ab[r], slot[b]) = old[r][b] + (acc[r][s] + ph0[r]);
    }
  }
}

// fp32 variant of shap_run on packed pairs of Gauss nodes: {P_q, P_q+1} live
// in one 64-bit register pair and EXTEND / UNWIND use the sm_100 paired FP32
// instructions (FMUL2 / FFMA2: one issue slot for two lanes' worth of FMA-pipe
// work), predicated per row as before.  Pads (q >= Q) are zero in the table,
// so P_pad = 0 and they contribute nothing.  acc keeps even/odd node partial
// sums, folded once per run.
template <int Q, int R, int NT, int kXg>
__device__ __forceinline__ void shap_run_x2(int k, int n_run, const int4* __restrict__ E,
                                            const float* __restrict__ tab, const int (&xb)[R], const int (&ab)[R],
                                            const float* __restrict__ xg, int cs) {
  constexpr int QP = QP_<Q>::v, KM = 2 * Q, QH = (Q + 1) / 2;
  constexpr int kRmw = GTS_RMW_REGS / R > 1 ? GTS_RMW_REGS / R : 1;
  float* const sT = reinterpret_cast<float*>(g_smem);
  const int words = nodal_path_words(k, Q, NT);
  float xv[R][KM];
  float2 acc[R][KM], ph0[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ph0[r] = make_float2(0.f, 0.f);
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    const bool valid = (s < KM - 1 || s < k);
    const int4 e = valid ? E[s] : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      acc[r][s] = make_float2(0.f, 0.f);
      if constexpr (kXg >= 2) xv[r][s] = tm_ld((uint32_t)cs + (uint32_t)(xb[r] + tm_col<float, kXg>(e)));
      else if constexpr (kXg) xv[r][s] = __ldg(xg + (uint32_t)(e.w * cs + xb[0]) + r * 32);  // a lane's rows: 32 apart
      else xv[r][s] = sT[xb[r] + (NT == 2 ? e.z / (int)sizeof(float) : e.z)];
    }
  }
  if constexpr (kXg >= 2) {
    tm_wait_ld();
#pragma unroll
    for (int s = 0; s < KM; ++s)
#pragma unroll
      for (int r = 0; r < R; ++r) tm_pin(xv[r][s]);
  }
  using L = Lay<Q, NT>;
  for (int p = 0; p < n_run; ++p) {
    const float* tp = tab + p * words;
    float2 P[R][QH];
    {
      float2 c[QH];
      lds_pairs(c, tp);
#pragma unroll
      for (int h = 0; h < QH; ++h)
#pragma unroll
        for (int r = 0; r < R; ++r) P[r][h] = c[h];
    }
    uint32_t om[R];
#pragma unroll
    for (int r = 0; r < R; ++r) om[r] = 0u;
    float4 bq;
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        float2 rh[QH];
        float lo, hi;
        lds_rho_pairs<Q, NT>(rh, lo, hi, tp, s, bq);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool o = in_bounds(xv[r][s], lo, hi);
          om[r] |= (uint32_t)o << s;
          if (!o) {
#pragma unroll
            for (int h = 0; h < QH; ++h) P[r][h] = __fmul2_rn(P[r][h], rh[h]);  // EXTEND, f_s = B_s
          }
        }
      }
    }
    {
      float2 d[QH];
      lds_pairs(d, tp + QP);
#pragma unroll
      for (int h = 0; h < QH; ++h)
#pragma unroll
        for (int r = 0; r < R; ++r) ph0[r] = __ffma2_rn(P[r][h], d[h], ph0[r]);
    }
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        float2 Ch[QH];
        lds_pairs(Ch, tp + L::cp(s));
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if ((om[r] >> s) & 1u) {
#pragma unroll
            for (int h = 0; h < QH; ++h) acc[r][s] = __ffma2_rn(P[r][h], Ch[h], acc[r][s]);  // UNWIND via C'
          }
        }
      }
    }
  }
#pragma unroll
  for (int s0 = 0; s0 < KM; s0 += kRmw) {  // grouped read-modify-writes, see shap_run
    float old[R][kRmw];
    int slot[kRmw];
#pragma unroll
    for (int b = 0; b < kRmw; ++b) {
      const int s = s0 + b;
      if (s < KM && (s < KM - 1 || s < k)) {
        slot[b] = E[s].z;
#pragma unroll
        for (int r = 0; r < R; ++r) old[r][b] = tile_at<float, NT>(ab[r], slot[b]);
      }
    }
#pragma unroll
    for (int b = 0; b < kRmw; ++b) {
      const int s = s0 + b;
      if (s < KM && (s < KM - 1 || s < k))
#pragma unroll
        for (int r = 0; r < R; ++r)
          tile_at<float, NT>(ab[r], slot[b]) = old[r][b] + ((acc[r][s].x + acc[r][s].y) + (ph0[r].x + ph0[r].y));
    }
  }
}

// One path, element loop not unrolled (large Q); accumulates per element.
template <typename T, int Q, int R, int NT, int kXg>
__device__ __forceinline__ void shap_path_dyn(int k, const int4* __restrict__ E, const T* __restrict__ tab,
                                              const int (&xb)[R], const int (&ab)[R], const T* __restrict__ xg,
                                              int cs) {
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
  typename BQ<T>::type bq;
#pragma unroll 1
  for (int s = 0; s < k; ++s) {
    const int4 rec = E[s];  // the run head's record: x source
    T rho[Q], lo, hi;
    lds_rho<T, Q, NT>(rho, lo, hi, tab, s, bq);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool o = in_bounds(load_x<T, NT, kXg>(sT, xb[r], rec, xg, cs), lo, hi);
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
    const int sl = E[s].z;
    T C[Q];
    lds_vec(C, tab + Lay<Q, NT>::cp(s));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      T a = ph0[r];
      if ((om[r] >> s) & 1u) {
#pragma unroll
        for (int q = 0; q < Q; ++q) a = fma(P[r][q], C[q], a);
      }
      tile_at<T, NT>(ab[r], sl) += a;
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
  typename BQ<T>::type bq;
  auto body = [&](int s) {
    const int4 rec = E[s];  // the run head's record: x source
    T rho[Q], lo, hi;
    lds_rho<T, Q, 3>(rho, lo, hi, tp, s, bq);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const bool o = in_bounds(sT[xb[r] + rec.z], lo, hi);
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
  const int words = nodal_path_words(k, Q);
  T G[Q];
  lds_vec(G, gam);
  int slot[KM], rb[KM];
  T xv[R][KM];
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    const bool valid = (s < KM - 1 || s < k);
    const int4 e = valid ? E[s] : make_int4(0, 0, 0, 0);
    slot[s] = e.z;
    rb[s] = e.w;
#pragma unroll
    for (int r = 0; r < R; ++r) xv[r][s] = sT[xb[r] + e.z];
  }
  T acc[R][kRegAcc ? NC : 1];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < (kRegAcc ? NC : 1); ++c) acc[r][c] = (T)0;
  using L = Lay<Q, 3>;
  for (int p = 0; p < n_run; ++p) {
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
    typename BQ<T>::type bq;
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        T rho[Q], lo, hi;
        lds_rho<T, Q, 3>(rho, lo, hi, tp, s, bq);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool o = in_bounds(xv[r][s], lo, hi);
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
      lds_vec(h, tp + 2 * QP);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int q = 0; q < Q; ++q) W[r][q] = h[q] * P[r][q];
    }
    // u_s = (o_s - z_s)/f_s(t_q): cached in registers for small paths; for
    // larger ones the partner's u is applied as a select on the dot product
    constexpr bool kCacheU = Q <= GTS_INTER_CACHEU_QMAX;  // u of every element in registers
    T u[R][kCacheU ? KM : 1][Q];
    if constexpr (kCacheU) {
#pragma unroll
      for (int s = 0; s < KM; ++s) {
        if (s < KM - 1 || s < k) {
          T al[Q];
          lds_vec(al, tp + L::al(s));
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const bool o = (om[r] >> s) & 1u;
#pragma unroll
            for (int q = 0; q < Q; ++q) u[r][s][q] = o ? al[q] : G[q];  // UNWIND(s) folded into u
          }
        }
      }
    }
    int c = 0;
#pragma unroll
    for (int i = 0; i < KM; ++i) {
      if (i < KM - 1 || i < k) {
        T y[R][Q], phi[R], yg[R];
        T ai[Q];
        if constexpr (!kCacheU) lds_vec(ai, tp + L::al(i));
        const int cdiag = c++;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          T a = kRegAcc ? acc[r][cdiag] : (T)0, g = (T)0;
          const bool oi = (om[r] >> i) & 1u;
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            T ui;
            if constexpr (kCacheU) ui = u[r][i][q];
            else ui = oi ? ai[q] : G[q];
            y[r][q] = W[r][q] * ui;
            a = fma(y[r][q], (T)2, a);  // phi_i = 2 sum_q W_q u_iq
            if constexpr (!kCacheU) g = fma(y[r][q], G[q], g);
          }
          phi[r] = a;
          yg[r] = g;
        }
        // !kRegAcc: the cells (i, j) of one path are distinct, so they are
        // updated in blocks of kB: kB values, kB loads, then kB stores (in
        // program order the compiler must assume a store may alias the next load)
        constexpr int kB = GTS_INTER_RMW_BLOCK;
        T pv[R][kRegAcc ? 1 : kB];
#pragma unroll
        for (int j = i + 1; j < KM; ++j) {
          if (j < KM - 1 || j < k) {
            T aj[Q];
            if constexpr (!kCacheU) lds_vec(aj, tp + L::al(j));
#pragma unroll
            for (int r = 0; r < R; ++r) {
              if constexpr (kRegAcc) {
                // the pair's dot product accumulates straight into its register
                if constexpr (kCacheU) {
#pragma unroll
                  for (int q = 0; q < Q; ++q) acc[r][c] = fma(y[r][q], u[r][j][q], acc[r][c]);
                } else if ((om[r] >> j) & 1u) {
#pragma unroll
                  for (int q = 0; q < Q; ++q) acc[r][c] = fma(y[r][q], aj[q], acc[r][c]);
                } else {
                  acc[r][c] += yg[r];
                }
              } else {
                T v = (T)0;
                if constexpr (kCacheU) {
#pragma unroll
                  for (int q = 0; q < Q; ++q) v = fma(y[r][q], u[r][j][q], v);
                } else {
#pragma unroll
                  for (int q = 0; q < Q; ++q) v = fma(y[r][q], aj[q], v);
                  v = ((om[r] >> j) & 1u) ? v : yg[r];
                }
                if constexpr (kB > 1) pv[r][(j - i - 1) % kB] = v;
                else sT[ab[r] + rb[i] + slot[j]] += v;
              }
            }
          }
          if constexpr (!kRegAcc && kB > 1) {
            // flush the block after its last pair (or after the row's last pair)
            if ((j - i) % kB == 0 || j == KM - 1) {
              const int j0 = j - ((j - i - 1) % kB);
              T old[R][kB];
#pragma unroll
              for (int b = 0; b < kB; ++b) {
                const int jj = j0 + b;
                if (jj <= j && (jj < KM - 1 || jj < k))
#pragma unroll
                  for (int r = 0; r < R; ++r) old[r][b] = sT[ab[r] + rb[i] + slot[jj]];
              }
#pragma unroll
              for (int b = 0; b < kB; ++b) {
                const int jj = j0 + b;
                if (jj <= j && (jj < KM - 1 || jj < k))
#pragma unroll
                  for (int r = 0; r < R; ++r) sT[ab[r] + rb[i] + slot[jj]] = old[r][b] + pv[r][b];
              }
            }
          }
          ++c;
        }
        // the diagonal cell collects phi_i; Eq. 6 subtracts the row sums when
        // the tile is flushed (linear in the paths, so it holds per tile)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if constexpr (kRegAcc) acc[r][cdiag] = phi[r];
          else sT[ab[r] + rb[i] + slot[i]] += phi[r];
        }
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

// fp32, one row: inter_run on packed pairs of Gauss nodes.  Every cell keeps
// an {even node, odd node} partial sum, so the pair products, the diagonal
// sums, W and y run on paired FP32 instructions (FFMA2 / FMUL2) and the run's
// cells stay in registers.  Odd Q: the last node is a scalar "tail" whose
// products accumulate into the .x half of the same cell (no padded node).
template <int Q>
__device__ __forceinline__ void inter_run_q2(int k, int n_run, const int4* __restrict__ E,
                                             const float* __restrict__ tab, const float* __restrict__ gam,
                                             const int (&xb)[1], const int (&ab)[1]) {
  constexpr int QP = QP_<Q>::v, KM = 2 * Q, NC = KM * (KM + 1) / 2, NP = Q / 2;
  constexpr bool kTail = (Q & 1) != 0;
  constexpr int TQ = Q - 1;  // the tail node (odd Q)
  float* const sT = reinterpret_cast<float*>(g_smem);
  const int words = nodal_path_words(k, Q);
  float2 G[NP > 0 ? NP : 1];
#pragma unroll
  for (int h = 0; h < NP; ++h) G[h] = make_float2(gam[2 * h], gam[2 * h + 1]);
  const float Gt = kTail ? gam[TQ] : 0.f;
  float xv[KM];
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    const bool valid = (s < KM - 1 || s < k);
    xv[s] = sT[xb[0] + (valid ? E[s].z : 0)];
  }
  float2 acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = make_float2(0.f, 0.f);
  using L = Lay<Q, 3>;
  for (int p = 0; p < n_run; ++p) {
    const float* tf = tab + p * words;
    const float2* tp = reinterpret_cast<const float2*>(tf);
    float2 P[NP > 0 ? NP : 1];
#pragma unroll
    for (int h = 0; h < NP; ++h) P[h] = tp[h];
    float Pt = kTail ? tf[TQ] : 0.f;
    uint32_t om = 0u;
    float4 bq;
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        float w[Q], lo, hi;
        lds_rho<float, Q, 3>(w, lo, hi, tf, s, bq);
        const bool o = in_bounds(xv[s], lo, hi);
        om |= (uint32_t)o << s;
        if (!o) {
#pragma unroll
          for (int h = 0; h < NP; ++h) P[h] = __fmul2_rn(P[h], make_float2(w[2 * h], w[2 * h + 1]));  // EXTEND
          if constexpr (kTail) Pt *= w[TQ];
        }
      }
    }
    float2 W[NP > 0 ? NP : 1];
#pragma unroll
    for (int h = 0; h < NP; ++h) W[h] = __fmul2_rn(P[h], tp[QP + h]);  // h_q = v w_q / 2
    const float Wt = kTail ? Pt * tf[2 * QP + TQ] : 0.f;
    float2 u[KM][NP > 0 ? NP : 1];
    float ut[KM];
#pragma unroll
    for (int s = 0; s < KM; ++s) {
      if (s < KM - 1 || s < k) {
        const float* al = tf + L::al(s);
        const bool o = (om >> s) & 1u;
#pragma unroll
        for (int h = 0; h < NP; ++h) {
          const float2 a = reinterpret_cast<const float2*>(al)[h];
          u[s][h] = make_float2(o ? a.x : G[h].x, o ? a.y : G[h].y);  // UNWIND(s) folded into u
        }
        if constexpr (kTail) ut[s] = o ? al[TQ] : Gt;
      }
    }
    int c = 0;
#pragma unroll
    for (int i = 0; i < KM; ++i) {
      if (i < KM - 1 || i < k) {
        float2 y[NP > 0 ? NP : 1];
        const int cdiag = c++;
        float2 a = acc[cdiag];
#pragma unroll
        for (int h = 0; h < NP; ++h) {
          y[h] = __fmul2_rn(W[h], u[i][h]);
          a = __ffma2_rn(y[h], make_float2(2.f, 2.f), a);  // phi_i = 2 sum_q W_q u_iq
        }
        float yt = 0.f;
        if constexpr (kTail) {
          yt = Wt * ut[i];
          a.x = fmaf(yt, 2.f, a.x);
        }
#pragma unroll
        for (int j = i + 1; j < KM; ++j) {
          if (j < KM - 1 || j < k) {
#pragma unroll
            for (int h = 0; h < NP; ++h) acc[c] = __ffma2_rn(y[h], u[j][h], acc[c]);
            if constexpr (kTail) acc[c].x = fmaf(yt, ut[j], acc[c].x);
          }
          ++c;
        }
        acc[cdiag] = a;  // Eq. 6 subtracts the row sums when the tile is flushed
      } else {
        c += KM - i;
      }
    }
  }
  // the slots (and tri-row bases) are read back from the run head's records
  // only now, when the path registers are dead
  int slot[KM], rb[KM];
#pragma unroll
  for (int s = 0; s < KM; ++s) {
    const int4 e = (s < KM - 1 || s < k) ? E[s] : make_int4(0, 0, 0, 0);
    slot[s] = e.z;
    rb[s] = e.w;
  }
  int c = 0;
#pragma unroll
  for (int i = 0; i < KM; ++i) {
#pragma unroll
    for (int j = i; j < KM; ++j) {
      if ((i < KM - 1 || i < k) && (j < KM - 1 || j < k)) sT[ab[0] + rb[i] + slot[j]] += acc[c].x + acc[c].y;
      ++c;
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
    lds_vec(h, tp + 2 * QP);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int q = 0; q < Q; ++q) W[r][q] = h[q] * P[r][q];
  }
#pragma unroll 1
  for (int i = 0; i < k; ++i) {
    const int4 ri = E[i];
    T ai[Q];
    lds_vec(ai, tp + Lay<Q, 3>::al(i));
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
      sT[ab[r] + ri.w + ri.z] += phi + phi;  // phi_i; Eq. 6 applied at flush
    }
#pragma unroll 1
    for (int j = i + 1; j < k; ++j) {
      const int cell = ri.w + E[j].z;
      T aj[Q];
      lds_vec(aj, tp + Lay<Q, 3>::al(j));
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
// QM: the largest Q a kernel with S slots can meet (k <= S, so Q <= S / 2);
// larger cases are compiled out, which bounds the kernel's register budget by
// the runs it can actually execute.
template <typename T, int R, bool kInter, int NT, int kXg, int QM>
__device__ __forceinline__ void run_dispatch(int4 ph, const int4* __restrict__ E0, const T* __restrict__ table,
                                             const T* __restrict__ gauss, const int (&xb)[R], const int (&ab)[R],
                                             const T* __restrict__ xg, int cs) {
  const int k = ph.x & 0xff, n_run = ph.x >> 16, q = ph.y;
  const int4* E = E0 + ph.z;
  const T* tab = table + ph.w;
  const int words = nodal_path_words(k, q, NT);
  if constexpr (!kInter && GTS_X2 && sizeof(T) == 4 && R <= 2) {
    // fp32: paired-node FFMA2 runs (Q >= 2); Q = 1 has nothing to pair
    switch (q) {
      case 1: shap_run<T, 1, R, NT, kXg>(k, n_run, E, tab, xb, ab, xg, cs); break;
#define GTS_RUN(QQ) case QQ: if constexpr (QQ <= QM) shap_run_x2<QQ, R, NT, kXg>(k, n_run, E, reinterpret_cast<const float*>(tab), xb, ab, \
                                                         reinterpret_cast<const float*>(xg), cs); break;
      GTS_RUN(2) GTS_RUN(3) GTS_RUN(4)
#if GTS_X2_R2_QMAX >= 5
      GTS_RUN(5)
#endif
#if GTS_X2_R2_QMAX >= 6
      GTS_RUN(6)
#endif
#undef GTS_RUN
      default:
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
          const int xb1[1] = {xb[r]}, ab1[1] = {ab[r]};
          switch (q) {
#define GTS_RUN1(QQ) case QQ: if constexpr (QQ <= QM) shap_run_x2<QQ, 1, NT, kXg>(k, n_run, E, reinterpret_cast<const float*>(tab), xb1, ab1, \
                                                           reinterpret_cast<const float*>(xg), cs); break;
            GTS_RUN1(5) GTS_RUN1(6) GTS_RUN1(7) GTS_RUN1(8)
#undef GTS_RUN1
            default:
              for (int p = 0; p < n_run; ++p) {
                switch (q) {
#define GTS_DYN(QQ) case QQ: if constexpr (QQ <= QM) shap_path_dyn<T, QQ, 1, NT, kXg>(k, E, tab + p * words, xb1, ab1, xg, cs); break;
                  GTS_DYN(9) GTS_DYN(10) GTS_DYN(11) GTS_DYN(12) GTS_DYN(13) GTS_DYN(14) GTS_DYN(15) GTS_DYN(16)
#undef GTS_DYN
                  default: break;
                }
              }
          }
        }
    }
  } else if constexpr (!kInter) {
    switch (q) {
#define GTS_RUN(QQ) case QQ: if constexpr (QQ <= QM) shap_run<T, QQ, R, NT, kXg>(k, n_run, E, tab, xb, ab, xg, cs); break;
      GTS_RUN(1) GTS_RUN(2) GTS_RUN(3) GTS_RUN(4)
#undef GTS_RUN
      default:
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
          const int xb1[1] = {xb[r]}, ab1[1] = {ab[r]};
          switch (q) {
#define GTS_RUN1(QQ) case QQ: if constexpr (QQ <= QM) shap_run<T, QQ, 1, NT, kXg>(k, n_run, E, tab, xb1, ab1, xg, cs); break;
            GTS_RUN1(5) GTS_RUN1(6) GTS_RUN1(7) GTS_RUN1(8)
#undef GTS_RUN1
            default:
              for (int p = 0; p < n_run; ++p) {
                switch (q) {
#define GTS_DYN(QQ) case QQ: if constexpr (QQ <= QM) shap_path_dyn<T, QQ, 1, NT, kXg>(k, E, tab + p * words, xb1, ab1, xg, cs); break;
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
      case 2:
        if constexpr ((GTS_INTER_PAIRED & (1 << 2)) && sizeof(T) == 4 && R == 1) {
          inter_run_q2<2>(k, n_run, E, reinterpret_cast<const float*>(tab), reinterpret_cast<const float*>(gam),
                          xb, ab);
        } else {
          inter_run<T, 2, R, true>(k, n_run, E, tab, gam, xb, ab);
        }
        break;
      default:
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
          const int xb1[1] = {xb[r]}, ab1[1] = {ab[r]};
          switch (q) {
            case 3:
              if constexpr ((GTS_INTER_PAIRED & (1 << 3)) && sizeof(T) == 4) {
                inter_run_q2<3>(k, n_run, E, reinterpret_cast<const float*>(tab),
                                reinterpret_cast<const float*>(gam), xb1, ab1);
              } else {
                inter_run<T, 3, 1, true>(k, n_run, E, tab, gam, xb1, ab1);
              }
              break;
            case 4:
              if constexpr ((GTS_INTER_PAIRED & (1 << 4)) && sizeof(T) == 4) {
                inter_run_q2<4>(k, n_run, E, reinterpret_cast<const float*>(tab),
                                reinterpret_cast<const float*>(gam), xb1, ab1);
              } else {
                inter_run<T, 4, 1, false>(k, n_run, E, tab, gam, xb1, ab1);
              }
              break;
            case 5:
              if constexpr (QM >= 5) inter_run<T, 5, 1, (GTS_INTER_REGACC & (1 << 5)) != 0>(k, n_run, E, tab, gam, xb1, ab1);
              break;
            case 6:
              if constexpr (sizeof(T) == 4 && QM >= 6) {
                inter_run<T, 6, 1, (GTS_INTER_REGACC & (1 << 6)) != 0>(k, n_run, E, tab, gam, xb1, ab1);
                break;
              }
              [[fallthrough]];
            case 7:
              if constexpr (sizeof(T) == 4 && QM >= 7) {
                if (q == 7) { inter_run<T, 7, 1, false>(k, n_run, E, tab, gam, xb1, ab1); break; }
              }
              [[fallthrough]];
            default:
              for (int p = 0; p < n_run; ++p) {
                switch (q) {
#define GTS_IP(QQ) case QQ: if constexpr (QQ <= QM) inter_path<T, QQ, 1, false>(k, E, tab + p * words, gam, xb1, ab1); break;
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
  int64_t n_rows;
  int64_t row_stride, col_stride;  // X[r][f] at X[r * row_stride + f * col_stride]
  void* out;
  void* out_phi;  // interaction kernel only: if set, the phi_i cells are also added to phi (fused call)
  int upper_only;  // interaction kernel only: write cells (i, j) with i < j only; mirror_kernel fills (j, i)
  int n_splits;
  // Work items (taken by persistent blocks): item = ((batch * n_bgroups + g) * n_splits + split) * tiles_per_batch + tile.
  // n_bgroups = 1: a block walks the chunks of every group (its split of them);
  // n_bgroups = G: a block walks group g's chunks only, so the blocks resident
  // at one time share one group's phi rows and the rows of one batch (L2 reuse).
  int n_bgroups;
  int64_t tiles_per_batch;
  int64_t n_batches;  // work items = n_batches * n_bgroups * n_splits * tiles_per_batch (persistent grid)
  int tile_minor;     // 1: item = ((batch * n_bgroups + g) * n_splits + split) * tiles_per_batch + tile;
                      // 0: item = ((batch * n_bgroups + g) * tiles_per_batch + tile) * n_splits + split
  int tile_w;  // SHAP: row stride of the X / phi tiles = widest slot map + 1 (odd)
  int M, G;
  int64_t n_chunks;
  int max_chunk_bytes;
};

template <bool kInter>
__host__ __device__ constexpr int acc_width(int S) { return kInter ? S * (S + 1) / 2 : S; }

template <typename T, int S, int R, bool kInter>
__host__ __device__ constexpr int tile_words_per_warp() {
  return R * 32 * ((S + 1) + (acc_width<kInter>(S) | 1));
}

// Row stride (words) of the X and phi tiles.  Interaction tiles are sized by
// the slot width S (upper triangle of S x S); SHAP tiles by the blob's widest
// slot map (tile_w = max slots + 1, odd: lanes = rows hit distinct banks), so
// identity maps of M features cost M + 1 words per row, not S + 1.
#ifndef GTS_XG_FIXED_STRIDE
#define GTS_XG_FIXED_STRIDE 0  // global-X SHAP kernels: phi tile row stride S + 1 (compile time) or the blob's widest map + 1
#endif
#ifndef GTS_TMEM_X
#define GTS_TMEM_X 3  // bit 0: fp32 SHAP kernels with identity maps of <= 64 features keep X in TMEM (XG = 2);
                      // bit 1: the 32-slot fp32 SHAP kernel keeps each slot map's X in TMEM (XG = 3)
#endif
#ifndef GTS_XG_MIN_S
#define GTS_XG_MIN_S 32  // SHAP kernels with >= this many slots read X from feature-major global memory
                         // (measured in lost sessions, see profiles/README.md: with 2 rows per lane fashion 5.06e5 -> 6.14e5 rows/s,
                         // the per-chunk X gathers are gone; covtype 1.40e4 -> 1.43e4)
#endif
// kXg kernels keep no X tile: every run reads its x values straight from a
// feature-major copy of X (L1-resident for the rows in flight), which halves
// the shared memory per row and lets twice the warps share an SM.
template <bool kInter, int S>
__host__ __device__ constexpr bool xg_enabled() { return !kInter && S >= GTS_XG_MIN_S; }
template <bool kInter, int S>
__host__ __device__ constexpr int x_stride(int tile_w) { return kInter ? S + 1 : (xg_enabled<kInter, S>() ? 0 : tile_w); }
template <bool kInter, int S>
__host__ __device__ constexpr int acc_stride(int tile_w) {
  // kXg kernels: a compile-time row stride S + 1 (odd), so the R rows of a lane sit at immediate offsets
  return kInter ? (acc_width<kInter>(S) | 1) : (xg_enabled<kInter, S>() && GTS_XG_FIXED_STRIDE ? S + 1 : tile_w);
}

// Launch shape per (dtype, kernel, slot width): R rows per lane and W warps
// per block.  Interactions and narrow SHAP tiles: two blocks (tiles + chunk
// staging) share an SM.  Wide SHAP tiles (identity maps up to 64 features,
// per-chunk maps of 32) trade warps for rows per lane: the per-path tables
// are read from shared memory once per lane and used for R rows, which is
// what bounds these kernels (LSU pipe, profiles/r01g).
#ifndef GTS_INTER8_W
#define GTS_INTER8_W 8  // warps per block of the 8-slot fp32 interaction kernel
#endif
#ifndef GTS_INTER8_MINB
#define GTS_INTER8_MINB 2  // resident blocks per SM the 8-slot fp32 interaction kernel's registers are sized for
#endif
#ifndef GTS_SHAP_R32
#define GTS_SHAP_R32 2  // measured with global X (lost session): fashion R 2 / W 4 6.14e5 rows/s, R 1 / W 8 4.44e5
#endif
#ifndef GTS_SHAP_W32
#define GTS_SHAP_W32 4
#endif
#ifndef GTS_SHAP_B32
#define GTS_SHAP_B32 2  // resident blocks per SM the register budget is sized for
#endif
#ifndef GTS_SHAP_R64
#define GTS_SHAP_R64 2  // measured with global X (lost session): covtype R 2 / W 4 1.43e4 rows/s, R 1 / W 8 1.38e4
#endif
#ifndef GTS_SHAP_W64
#define GTS_SHAP_W64 4  // no X tile (kXg): 4 warps x 64 rows x 2 blocks fit the phi tiles
#endif
#ifndef GTS_SHAP_B64
#define GTS_SHAP_B64 3  // 3 blocks x 4 warps x 64 rows per SM (168 registers, runtime tile stride, 8 KB chunks):
                        // covtype 1.44e4 -> 1.64e4 rows/s (lost session; r02e measures the result)
#endif
template <typename T, bool kInter, int S>
struct Cfg {
  static constexpr bool kWide = !kInter && S >= 32;
  static constexpr int R = (sizeof(T) == 4 && !kInter && S == 8) ? GTS_SHAP_R8
                           : (sizeof(T) == 4 && kInter && S == 8) ? GTS_INTER_R8
                           : (sizeof(T) == 4 && !kInter && S <= 16) ? 2
                           : (sizeof(T) == 4 && kWide) ? (S == 32 ? GTS_SHAP_R32 : GTS_SHAP_R64)
                                                       : 1;
  static constexpr int tile_bytes = (int)sizeof(T) * tile_words_per_warp<T, S, R, kInter>();
  static constexpr int W = (sizeof(T) == 4 && kWide) ? (S == 32 ? GTS_SHAP_W32 : GTS_SHAP_W64)
                           : (sizeof(T) == 4 && kInter && S == 8) ? GTS_INTER8_W
                           : tile_bytes * 8 <= 74 * 1024  ? 8
                           : tile_bytes * 4 <= 80 * 1024  ? 4
                           : tile_bytes * 2 <= 160 * 1024 ? 2
                                                          : 1;  // 32-slot interaction tiles (528 pair cells per row)
  static constexpr int kMinBlocks = (sizeof(T) == 4 && kWide) ? (S == 32 ? GTS_SHAP_B32 : GTS_SHAP_B64)
                                   : (sizeof(T) == 4 && kInter && S == 8) ? GTS_INTER8_MINB
                                                                          : (W >= 8 ? 2 : 1);
};

// shared-memory layout: gauss (T) | X tiles (T) | phi tiles (T) | 2 staging buffers | 2 mbarriers
template <typename T, int S, int W, int R, bool kInter>
__host__ __device__ constexpr int staging_byte_offset(int tile_w) {
  return (((kQMax * 3 * kQMax + W * R * 32 * (x_stride<kInter, S>(tile_w) + acc_stride<kInter, S>(tile_w))) *
           (int)sizeof(T)) + 127) & ~127;
}

// ---- TMA bulk copy (global -> shared) completing on an mbarrier (PTX ISA:
//      cp.async.bulk, mbarrier.*); SASS shows UBLKCP / SYNCS.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
#ifndef GTS_PERSIST
#define GTS_PERSIST 0  // 1: persistent blocks (grid = resident blocks) walking the items tile-minor: 3.3x less DRAM
                       // traffic on covtype SHAP but slower (covtype SHAP -3.5 %, fashion interactions -30 %, r02l)
#endif
#ifndef GTS_STAGGER
#define GTS_STAGGER 4  // chunks of start rotation per row tile (persistent blocks, see nodal_kernel)
#endif
#ifndef GTS_TMA_POLICY
#define GTS_TMA_POLICY 0  // L2 policy of the chunk copies: 0 default, 1 evict_normal, 2 evict_last, 3 evict_first
#endif
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  if constexpr (GTS_TMA_POLICY == 0) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
  } else {
    uint64_t pol;
    if constexpr (GTS_TMA_POLICY == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else if constexpr (GTS_TMA_POLICY == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// XG: where runs read x (0: the warp's shared X tile, 1: a feature-major copy
// in global memory, 2: TMEM filled from that copy; see load_x).
template <typename T, int S, int W, int R, bool kInter, int XG>
__global__ void __launch_bounds__(W * 32, (Cfg<T, kInter, S>::kMinBlocks)) nodal_kernel(Args a) {
  static_assert(XG < 2 || (sizeof(T) == 4 && W == 4 && !kInter), "TMEM X: 4 warps = 128 lanes");
  static_assert(XG != 2 || R * 64 <= 128, "TMEM X by feature: 128 columns");
  static_assert(XG != 3 || R * S <= 64, "TMEM X by slot: 64 columns");
  constexpr int kTmCols = XG == 2 ? 128 : 64;
  const int XS = x_stride<kInter, S>(a.tile_w);
  const int AS = acc_stride<kInter, S>(a.tile_w);
  const int AW = kInter ? acc_width<kInter>(S) : a.tile_w - 1;  // cells per row
  constexpr int ROWS = 32 * R;
  constexpr int o_x = kQMax * 3 * kQMax;
  const int o_acc = o_x + W * ROWS * XS;
  const int b_stage = staging_byte_offset<T, S, W, R, kInter>(a.tile_w);
  const int buf_bytes = a.max_chunk_bytes;  // multiple of 128 (host rounding)
  unsigned char* const stage0 = g_smem + b_stage;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(stage0 + 2 * buf_bytes);

  const BlobHeader* hdr = reinterpret_cast<const BlobHeader*>(a.blob);
  const ChunkRec* chunks = reinterpret_cast<const ChunkRec*>(a.blob + hdr->off_units);
  const double* work = reinterpret_cast<const double*>(a.blob + hdr->off_work) + (kInter ? (a.n_chunks + 1) : 0);
  const int32_t* slotmap = reinterpret_cast<const int32_t*>(a.blob + hdr->off_slotmap);
  const T* X = static_cast<const T*>(a.X);
  T* out = static_cast<T*>(a.out);
  T* const sT = reinterpret_cast<T*>(g_smem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // Block b takes work items b, b + gridDim.x, ... -- one item per block by
  // default; with GTS_PERSIST=1 the grid is the resident blocks (kernels.cu).
  // Items (Args::tile_minor): tile-minor within a (batch, group, split), so
  // that the items in flight share a chunk stream, except for SHAP with
  // per-chunk slot maps: split-minor, so that they share rows (kernels.cu,
  // GTS_TILE_MINOR).  Items start their chunk walk at a rotation of
  // GTS_STAGGER chunks per row tile.  (persistent blocks cut the chunk re-reads from HBM
  // 721 -> 219 GB per 65 536-row covtype launch but measured slower.)
  constexpr int64_t rows_per_block = W * ROWS;
  int64_t row0 = 0, c_begin = 0, c_end = 0;
  int split = 0, bgroup = 0;

  auto first_of = [&](int g) -> int64_t {  // first chunk with group >= g (chunks are in group order)
    int64_t lo = 0, hi = a.n_chunks;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (chunks[mid].group < g) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  // the item's chunk range: its split of all chunks, or of group bgroup's
  auto chunk_range = [&]() {
    int64_t g_lo = 0, g_hi = a.n_chunks;
    if (a.n_bgroups > 1) {
      g_lo = first_of(bgroup);
      g_hi = first_of(bgroup + 1);
    }
    const double w_lo = work[g_lo], w_span = work[g_hi] - w_lo;
    auto split_begin = [&](int sp) -> int64_t {
      if (sp >= a.n_splits) return g_hi;
      const double target = w_lo + w_span * (double)sp / (double)a.n_splits;
      int64_t lo = g_lo, hi = g_hi;  // first c with work[c] >= target
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (work[mid] < target) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    c_begin = split_begin(split);
    c_end = split_begin(split + 1);
  };

  // prologue (once per block): barriers, gauss table, TMEM
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  const T* gsrc = reinterpret_cast<const T*>(a.blob + hdr->off_gauss);
  for (int i = tid; i < kQMax * 3 * kQMax; i += blockDim.x) sT[i] = gsrc[i];
  int xb[R], ab[R];
  constexpr int kXg = XG;
  static_assert((XG != 0) == xg_enabled<kInter, S>(), "X source");
  __shared__ uint32_t tm_base;
  uint32_t tm_warp = 0;
  if constexpr (kXg >= 2) {
    // TMEM columns for the row tile's X: kXg = 2: column r * 64 + f of lane (warp, lane),
    // filled once per item; kXg = 3: column r * S + slot, filled at each slot-map change
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tm_base)),
                   "n"(kTmCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tm_warp = tm_base + ((uint32_t)(32 * (warp & 3)) << 16);
  }
  const int M1 = a.M + 1;
  int cur_map = -1, cur_group = -1, cur_slots = 0;
  int64_t cur_map_begin = 0;
  bool dirty = false;

  // Warp-cooperative flush of the warp's tiles: lane = feature slot, rows walked
  // in order, so consecutive lanes issue atomics to consecutive features of one
  // row (coalesced RED) and the loads of the tile are independent (ILP).  One
  // atomic per non-zero (row, group, feature) cell.
  const int tile_row0 = warp * ROWS;
  auto flush = [&]() {
    if (dirty) {
      __syncwarp();
      if constexpr (kInter) {
        // lane = row: every lane walks its own row's upper triangle (cell
        // offsets are compile-time constants, rows have an odd stride, so no
        // bank conflicts), sums the Eq. 6 row sums in registers, zeroes the
        // cells it read and issues one RED per non-zero cell.
        int fm[S];  // slot -> feature (uniform loads)
#pragma unroll
        for (int j = 0; j < S; ++j) fm[j] = j < cur_slots ? __ldg(slotmap + cur_map_begin + j) : 0;
#pragma unroll 1
        for (int r = 0; r < R; ++r) {
          const int64_t rg = row0 + r * 32 + lane;
          const bool ok_r = rg < a.n_rows;
          T* const tile = sT + ab[r];
          T* const base = out + ((size_t)(ok_r ? rg : 0) * a.G + cur_group) * (size_t)M1 * M1;
          T rs[S];
#pragma unroll
          for (int i = 0; i < S; ++i) rs[i] = (T)0;
#pragma unroll
          for (int i = 0; i < S; ++i) {
            if (i < cur_slots) {
#pragma unroll
              for (int j = i + 1; j < S; ++j) {
                if (j < cur_slots) {
                  const int c = i * (2 * S - i - 1) / 2 + j;  // tri_row_base(i, S) + j
                  const T v = tile[c];
                  tile[c] = (T)0;
                  rs[i] += v;
                  rs[j] += v;
                  if (ok_r && v != (T)0) {
                    atomicAdd(base + (size_t)fm[i] * M1 + fm[j], v);
                    if (!a.upper_only) atomicAdd(base + (size_t)fm[j] * M1 + fm[i], v);
                  }
                }
              }
            }
          }
#pragma unroll
          for (int i = 0; i < S; ++i) {
            if (i < cur_slots) {
              const int c = i * (2 * S - i - 1) / 2 + i;
              const T di = tile[c];  // sum of phi_i; Eq. 6: phi_ii = phi_i - sum_{j != i} phi_ij
              tile[c] = (T)0;
              const T d = di - rs[i];
              if (ok_r && d != (T)0) atomicAdd(base + (size_t)fm[i] * (M1 + 1), d);
              // fused call: the diagonal cell before Eq. 6 is the tile's SHAP value phi_i
              if (ok_r && a.out_phi != nullptr && di != (T)0)
                atomicAdd(static_cast<T*>(a.out_phi) + ((size_t)rg * a.G + cur_group) * M1 + fm[i], di);
            }
          }
        }
      } else {
        // lane = slot, rows walked in order: consecutive lanes hit consecutive
        // features of one row (coalesced RED); each lane zeroes the cells it read
        const size_t rstride = (size_t)a.G * M1;
        const int64_t nr = a.n_rows - row0;
        for (int i = lane; i < cur_slots; i += 32) {
          const int fi = slotmap[cur_map_begin + i];
          T* col = sT + o_acc + tile_row0 * AS + i;
          T* dst = out + ((size_t)row0 * a.G + cur_group) * (size_t)M1 + fi;
#pragma unroll 4
          for (int rr = 0; rr < ROWS; ++rr) {
            const T v = col[rr * AS];
            col[rr * AS] = (T)0;
            if (rr < nr && v != (T)0) atomicAdd(dst + rr * rstride, v);
          }
        }
      }
      __syncwarp();
    }
    dirty = false;
  };

  // Warp-cooperative gather of X into slot order: lane = slot, so each load
  // instruction reads one row's features (contiguous for identity maps).
  auto gather = [&](const ChunkRec& c) {
    __syncwarp();
    if (a.col_stride == 1) {
      // row-major X: lane = slot, each load instruction reads one row
      for (int i = lane; i < c.n_slots; i += 32) {
        const int f = slotmap[c.slotmap_begin + i];
#pragma unroll 8
        for (int rr = 0; rr < ROWS; ++rr) {
          const int64_t rg = row0 + rr;
          sT[o_x + (tile_row0 + rr) * XS + i] = rg < a.n_rows ? X[(size_t)rg * a.row_stride + f] : (T)0;
        }
      }
    } else {
      // feature-major X: lane = row, each load instruction reads 32 consecutive rows of one feature
#pragma unroll 4
      for (int i = 0; i < c.n_slots; ++i) {
        const size_t fo = (size_t)slotmap[c.slotmap_begin + i] * a.col_stride;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int64_t rg = row0 + r * 32 + lane;
          sT[o_x + (tile_row0 + r * 32 + lane) * XS + i] = rg < a.n_rows ? X[fo + (size_t)rg * a.row_stride] : (T)0;
        }
      }
    }
    __syncwarp();
  };

  uint32_t phase[2] = {0u, 0u};
  const int64_t n_items = (int64_t)a.n_batches * a.n_bgroups * a.n_splits * a.tiles_per_batch;
  // one item per block unless persistent: a straight-line body (no loop-carried state)
  for (int64_t item = blockIdx.x; item < n_items; item += (GTS_PERSIST ? (int64_t)gridDim.x : n_items)) {
    int64_t tile, bg;
    if (a.tile_minor) {
      tile = item % a.tiles_per_batch;
      const int64_t bs = item / a.tiles_per_batch;  // (batch, group, split)
      split = (int)(bs % a.n_splits);
      bg = bs / a.n_splits;
    } else {
      split = (int)(item % a.n_splits);
      const int64_t bt = item / a.n_splits;  // (batch, group, tile)
      tile = bt % a.tiles_per_batch;
      bg = bt / a.tiles_per_batch;
    }
    const int64_t batch = bg / a.n_bgroups;
    bgroup = (int)(bg % a.n_bgroups);
    const int64_t row_tile = batch * a.tiles_per_batch + tile;
    if (row_tile * rows_per_block >= a.n_rows) continue;  // padding tile of the last batch (block-uniform)
    row0 = row_tile * rows_per_block + (int64_t)warp * ROWS;
    chunk_range();
    // Staggered start: the item walks its chunks from a rotation of GTS_STAGGER
    // chunks per row tile, so the blocks in flight cover a window of ~GTS_STAGGER
    // x grid chunks of the stream (in L2) instead of requesting the same chunk
    // at once (all blocks on one L2 line set).
    const int64_t c_len = c_end - c_begin;
    const int64_t rot = c_len > 0 ? (tile * GTS_STAGGER) % c_len : 0;
    auto chunk_at = [&](int64_t j) -> int64_t {
      const int64_t q = rot + j;
      return c_begin + (q >= c_len ? q - c_len : q);
    };
    __syncthreads();  // the previous item is done with both staging buffers and the tiles
    if (tid == 0 && c_len > 0) {
      const ChunkRec c0 = chunks[chunk_at(0)];
      mbar_expect_tx(&bars[0], (uint32_t)c0.data_bytes);
      tma_bulk_g2s(stage0, a.blob + c0.data_off, (uint32_t)c0.data_bytes, &bars[0]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int lr = warp * ROWS + r * 32 + lane;
      const int64_t rr = row0 + r * 32 + lane;
      // kXg = 1: the row (the feature-major copy is padded to whole tiles); 2, 3: the row's TMEM column base
      xb[r] = kXg == 2 ? r * 64 : kXg == 3 ? r * S : kXg ? (int)rr : o_x + lr * XS;
      ab[r] = o_acc + lr * AS;
      for (int i = 0; i < AW; ++i) sT[ab[r] + i] = (T)0;
    }
    if constexpr (kXg == 2) {
      for (int f = 0; f < a.M; ++f) {
#pragma unroll
        for (int r = 0; r < R; ++r) tm_st(tm_warp + r * 64 + f, X[(size_t)f * a.col_stride + row0 + r * 32 + lane]);
      }
      tm_wait_st();
    }
    cur_map = -1;
    cur_group = -1;
    cur_slots = 0;
    cur_map_begin = 0;
    dirty = false;
    for (int64_t j = 0; j < c_len; ++j) {
      const int b = (int)(j & 1);
      const ChunkRec c = chunks[chunk_at(j)];
      __syncthreads();  // every warp is done with buffer b^1 (the previous chunk)
      if (tid == 0 && j + 1 < c_len) {  // prefetch the next chunk while this one computes
        const ChunkRec cn = chunks[chunk_at(j + 1)];
        mbar_expect_tx(&bars[b ^ 1], (uint32_t)cn.data_bytes);
        tma_bulk_g2s(stage0 + (b ^ 1) * buf_bytes, a.blob + cn.data_off, (uint32_t)cn.data_bytes, &bars[b ^ 1]);
      }
      if (c.map_id != cur_map || c.group != cur_group) {
        flush();
        if (!kXg && c.map_id != cur_map) gather(c);
        if (kXg == 3 && c.map_id != cur_map) {
          // the new slot map's x values of this warp's rows into TMEM (lane = row)
          for (int i = 0; i < c.n_slots; ++i) {
            const size_t fo = (size_t)slotmap[c.slotmap_begin + i] * a.col_stride + row0 + lane;
#pragma unroll
            for (int r = 0; r < R; ++r) tm_st(tm_warp + r * S + i, X[fo + r * 32]);
          }
          tm_wait_st();
        }
        cur_map = c.map_id;
        cur_group = c.group;
        cur_slots = c.n_slots;
        cur_map_begin = c.slotmap_begin;
      }
      mbar_wait(&bars[b], phase[b]);
      phase[b] ^= 1u;
      if (row0 < a.n_rows) {
        const int4* sE = reinterpret_cast<const int4*>(stage0 + b * buf_bytes);
        const int4* sP = sE + c.n_elems;
        const T* tab = reinterpret_cast<const T*>(sP + c.n_paths);
        for (int p = 0; p < c.n_paths;) {
          const int4 ph = sP[p];
          run_dispatch<T, R, kInter, kInter ? 3 : nodal_tables(S), kXg, (S / 2 < kQMax ? S / 2 : kQMax)>(
              ph, sE, tab, sT, xb, ab, X, kXg >= 2 ? (int)tm_warp : (int)a.col_stride);
          p += ph.x >> 16;
        }
        dirty = true;
      }
    }
    flush();
  }
  if constexpr (kXg >= 2) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_base), "n"(kTmCols));
    }
  }
}

}  // namespace nodal
}  // namespace gts
