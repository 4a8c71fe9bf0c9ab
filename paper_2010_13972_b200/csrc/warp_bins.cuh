// warp_bins.cuh -- paper-lineage kernels (GTS_LAYOUT_WARP_BINS).
//
// Lanes = path elements of a packed 32-lane bin (§3.3).  Per row: one-fraction
// (the listing's GetOneFraction), EXTEND via __shfl_up_sync
// (Algorithm 2, reading G4), UNWOUNDSUM via __shfl_sync (Algorithm 3, reading
// G5), phi = U (o - z) v.  Lanes with equal (group, feature) are
// summed with __match_any_sync + shuffles, then one atomic per sum.
// Interactions: swap-to-end conditioning (§3.5).
#pragma once
#include "blob_format.h"

namespace gts {
namespace wb {

constexpr unsigned kFull = 0xffffffffu;

template <typename T>
struct BinLanes {
  const int32_t* feat;
  const int32_t* meta;
  const int32_t* grp;
  const float* lo;
  const float* hi;
  const T* z;
  const T* v;
};

template <typename T>
__device__ __forceinline__ BinLanes<T> bin_lanes(const char* blob) {
  const BlobHeader* hdr = reinterpret_cast<const BlobHeader*>(blob);
  const int64_t lanes = hdr->n_units * kWarp;
  BinLanes<T> b;
  b.feat = reinterpret_cast<const int32_t*>(blob + hdr->off_elems);
  b.meta = b.feat + lanes;
  b.grp = b.meta + lanes;
  b.lo = reinterpret_cast<const float*>(b.grp + lanes);
  b.hi = b.lo + lanes;
  b.z = reinterpret_cast<const T*>(b.hi + lanes);
  b.v = b.z + lanes;
  return b;
}

// Algorithm 2 (reading G4): extend a path group by its elements of ranks 1..K
// (K <= kmax); lane r of the group holds w_r.  Elements are taken from lanes
// base + perm(u).  Lanes outside any group or beyond their K keep w.
template <typename T>
__device__ __forceinline__ T warp_extend(int rank, int K, int base, T zl, T ol, int kmax_steps,
                                         int skip_rank) {
  const int lane = threadIdx.x & 31;
  T w = (rank == 0) ? (T)1 : (T)0;
  for (int u = 1; u <= kmax_steps; ++u) {
    // element of new rank u lives in lane base + u (after the swap done by the caller)
    const int src = min(base + u, 31);
    const T zu = __shfl_sync(kFull, zl, src);
    const T ou = __shfl_sync(kFull, ol, src);
    T left = __shfl_up_sync(kFull, w, 1);
    if (rank == 0 || lane == 0) left = (T)0;  // shuffle(...) of a missing thread returns 0
    if (u <= K && u != skip_rank && rank <= u) {
      const T inv = (T)1 / (T)(u + 1);
      w = zu * w * (T)(u - rank) * inv + ou * left * (T)rank * inv;
    }
  }
  return w;
}

// Algorithm 3 (reading G5): sum of the weights after unwinding this lane's own
// element from a state w_0..w_K held in lanes base..base+K.
template <typename T>
__device__ __forceinline__ T warp_unwound_sum(T w, int base, int K, int kmax_steps, T z, T o) {
  T next = __shfl_sync(kFull, w, min(base + K, 31));
  T tot = 0;
  const T K1 = (T)(K + 1);
  for (int i = kmax_steps - 1; i >= 0; --i) {
    const T wi = __shfl_sync(kFull, w, min(base + i, 31));
    if (i < K) {
      const T tmp = next * K1 / (T)(i + 1);
      tot += o * tmp;
      next = wi - tmp * z * (T)(K - i) / K1;
      tot += ((T)1 - o) * wi * K1 / (z * (T)(K - i));
    }
  }
  return tot;
}

// Segmented sum over lanes with equal key, then one atomic by the group leader.
template <typename T, typename K>
__device__ __forceinline__ void seg_atomic_add(bool active, K key, T val, T* addr) {
  const int lane = threadIdx.x & 31;
  const unsigned peers = __match_any_sync(kFull, active ? key : (K)(-1 - lane));
  if (!active) return;
  T s = 0;
  unsigned m = peers;
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    s += __shfl_sync(peers, val, src);
  }
  if (lane == __ffs(peers) - 1) atomicAdd(addr, s);
}

struct BinArgs {
  const char* blob;
  const void* X;
  int64_t n_rows;
  int64_t row_stride, col_stride;
  void* out;
  int M, G;
  int64_t n_bins;
  int rows_per_item;
};

template <typename T, int W>
__global__ void __launch_bounds__(W * 32) bins_shap_kernel(BinArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bin = (int64_t)blockIdx.x * W + warp;
  if (bin >= a.n_bins) return;
  const BlobHeader* hdr = reinterpret_cast<const BlobHeader*>(a.blob);
  const int32_t kmax = reinterpret_cast<const int32_t*>(a.blob + hdr->off_units)[bin];
  const BinLanes<T> B = bin_lanes<T>(a.blob);
  const int64_t l = bin * kWarp + lane;
  const int feat = B.feat[l], meta = B.meta[l], grp = B.grp[l];
  const int rank = meta & 0xff, K = (meta >> 8) & 0xff, base = (meta >> 16) & 0xff;
  const float lo = B.lo[l], hi = B.hi[l];
  const T z = B.z[l], v = B.v[l];
  const T* X = static_cast<const T*>(a.X);
  T* out = static_cast<T*>(a.out);
  const int64_t r0 = (int64_t)blockIdx.y * a.rows_per_item;
  const int64_t r1 = min(r0 + a.rows_per_item, a.n_rows);
  const int M1 = a.M + 1;
  for (int64_t row = r0; row < r1; ++row) {
    T o = (T)0;
    if (feat == -1) o = (T)1;  // root: irrelevant to every output (reading G6)
    else if (feat >= 0) {
      const T x = X[row * a.row_stride + (int64_t)feat * a.col_stride];
      o = (x >= (T)lo && x < (T)hi) ? (T)1 : (T)0;  // GetOneFraction
    }
    const T w = warp_extend<T>(feat >= -1 ? rank : 99, K, base, z, o, kmax, -1);
    const T U = warp_unwound_sum<T>(w, base, K, kmax, z, o);
    const bool active = feat >= 0;
    const T phi = U * (o - z) * v;
    seg_atomic_add<T, int>(active, grp * M1 + feat, phi, out + ((size_t)row * a.G + grp) * M1 + (active ? feat : 0));
  }
}

template <typename T, int W>
__global__ void __launch_bounds__(W * 32) bins_inter_kernel(BinArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t bin = (int64_t)blockIdx.x * W + warp;
  if (bin >= a.n_bins) return;
  const BlobHeader* hdr = reinterpret_cast<const BlobHeader*>(a.blob);
  const int32_t kmax = reinterpret_cast<const int32_t*>(a.blob + hdr->off_units)[bin];
  const BinLanes<T> B = bin_lanes<T>(a.blob);
  const int64_t l = bin * kWarp + lane;
  const int feat0 = B.feat[l], meta = B.meta[l], grp = B.grp[l];
  const int rank = meta & 0xff, K = (meta >> 8) & 0xff, base = (meta >> 16) & 0xff;
  const float lo = B.lo[l], hi = B.hi[l];
  const T z0 = B.z[l], v = B.v[l];
  const T* X = static_cast<const T*>(a.X);
  T* out = static_cast<T*>(a.out);
  const int64_t r0 = (int64_t)blockIdx.y * a.rows_per_item;
  const int64_t r1 = min(r0 + a.rows_per_item, a.n_rows);
  const int M1 = a.M + 1;
  const bool in_group = feat0 >= -1;
  for (int64_t row = r0; row < r1; ++row) {
    T o0 = (T)0;
    if (feat0 == -1) o0 = (T)1;
    else if (feat0 >= 0) {
      const T x = X[row * a.row_stride + (int64_t)feat0 * a.col_stride];
      o0 = (x >= (T)lo && x < (T)hi) ? (T)1 : (T)0;
    }
    T* rowbase = out + ((size_t)row * a.G + grp) * (size_t)M1 * M1;
    // SHAP pass -> diagonal phi_ii += phi_i
    {
      const T w = warp_extend<T>(in_group ? rank : 99, K, base, z0, o0, kmax, -1);
      const T U = warp_unwound_sum<T>(w, base, K, kmax, z0, o0);
      const bool active = feat0 >= 0;
      seg_atomic_add<T, int>(active, grp * M1 + feat0, U * (o0 - z0) * v,
                             rowbase + (active ? (size_t)feat0 * M1 + feat0 : 0));
    }
    // conditioned rounds (§3.5): swap rank c to the end, extend the others
    for (int c = 1; c <= kmax; ++c) {
      const bool grp_on = in_group && c <= K && K >= 2;
      // new rank of this lane's slot r holds old element perm(r)
      const int src_rank = (rank == c) ? K : ((rank == K) ? c : rank);
      const int src = min(base + src_rank, 31);
      const T zs = __shfl_sync(kFull, z0, src);
      const T os = __shfl_sync(kFull, o0, src);
      const int fs = __shfl_sync(kFull, feat0, src);
      const int cl = min(base + c, 31);
      const T zc = __shfl_sync(kFull, z0, cl);
      const T oc = __shfl_sync(kFull, o0, cl);
      const int fc = __shfl_sync(kFull, feat0, cl);
      const int Kp = grp_on ? K - 1 : 0;
      const T w = warp_extend<T>(grp_on ? rank : 99, Kp, base, zs, os, kmax - 1, -1);
      const T U = warp_unwound_sum<T>(w, base, Kp, kmax - 1, zs, os);
      const bool active = grp_on && rank >= 1 && rank <= K - 1;
      const T val = (T)0.5 * U * (os - zs) * v * (oc - zc);
      const int64_t key_ij = active ? ((int64_t)(grp * M1 + fs) * M1 + fc) : 0;
      seg_atomic_add<T, long long>(active, (long long)key_ij, val,
                                   rowbase + (active ? (size_t)fs * M1 + fc : 0));
      const int64_t key_ii = active ? ((int64_t)(grp * M1 + fs) * M1 + fs) : 0;
      seg_atomic_add<T, long long>(active, (long long)key_ii, -val,
                                   rowbase + (active ? (size_t)fs * M1 + fs : 0));
    }
  }
}


}  // namespace wb
}  // namespace gts
