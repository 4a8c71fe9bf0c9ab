// kernels.cu -- sm_100a device code behind gts_shap / gts_shap_interactions.
//
// Two kernel families read the blob (blob_format.h):
//
// NODAL (default, B200-native).  Lanes = rows.  A warp owns 32
// rows and walks every path of a chunk; each (row, path) evaluates the
// permutation-weight polynomial of Algorithm 1 in the nodal basis:
//   U_i = sum_m m!(k-1-m)!/k! [t^m] prod_{s!=i}(z_s + o_s t)
//       = int_0^1 prod_{s!=i} (z_s + (o_s - z_s) t) dt       (Beta integral)
//       = sum_q w_q P(t_q) / f_i(t_q)                          (Gauss-Legendre,
//                                                               exact for Q = ceil(k/2))
// EXTEND becomes one multiply per node (P(t_q) *= f_s(t_q)), UNWIND a division
// folded into per-element constants staged in shared memory; phi_i = U_i (o_i -
// z_i) v.  Interactions (Eq. 3, §3.5 conditioning on features of
// the path only) use phi_ij = 1/2 v (o_i-z_i)(o_j-z_j) int prod_{s!=i,j}.
// Contributions accumulate in a per-warp shared-memory phi tile (rows x feature
// slots) and are flushed with one atomic per (row, group, feature) per chunk run.
//
// WARP_BINS (paper lineage).  Lanes = path elements of a
// packed bin; per row: one-fraction (listing), EXTEND via
// __shfl_up_sync (Algorithm 2, reading G4), UNWOUNDSUM via __shfl_sync
// (Algorithm 3, reading G5), phi = U (o - z) v; lanes with equal (group,
// feature) are reduced with __match_any_sync + shuffles before one atomic.
// Interactions: swap-to-end conditioning.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "../../include/gts.h"
#include "blob_format.h"

namespace gts {
gts_status fail(gts_status st, const char* fmt, ...);
}

namespace gts {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------ init kernels

// phi[row][g][m] = (m == M) ? bias[g] : 0           (reading G14)
template <typename T>
__global__ void init_phi_kernel(T* __restrict__ phi, int64_t n_rows, int G, int M,
                                const double* __restrict__ bias) {
  const int64_t M1 = M + 1;
  const int64_t total = n_rows * G * M1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i % M1;
    const int64_t g = (i / M1) % G;
    phi[i] = (m == M) ? (T)bias[g] : (T)0;
  }
}

// phi_ij[row][g][a][b] = (a == M && b == M) ? bias[g] : 0
template <typename T>
__global__ void init_phi_ij_kernel(T* __restrict__ phi, int64_t n_rows, int G, int M,
                                   const double* __restrict__ bias) {
  const int64_t M1 = M + 1, MM = M1 * M1;
  const int64_t total = n_rows * G * MM;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = i % MM;
    const int64_t g = (i / MM) % G;
    phi[i] = (cell == MM - 1) ? (T)bias[g] : (T)0;
  }
}

// ------------------------------------------------------------ NODAL family

template <typename T>
struct NodalSmem {
  // carved from dynamic shared memory at kernel start
  T* gauss;      // [kQMax][3][kQMax]
  int4* elem;    // [max_chunk_elems] {slot, lo bits, hi bits, tri row base}
  int4* path;    // [max_chunk_paths] {k, q, elem, table}
  T* table;      // [max_chunk_words]
  T* xt;         // [W][32][S+1]
  T* acc;        // [W][32][ACC]
};

__device__ __forceinline__ int tri_row_base(int a, int S) { return a * (2 * S - a - 1) / 2; }

// Stage one chunk into shared memory; the tables are computed in fp64 from the
// blob's fp64 zero fractions and rounded once to T.
template <typename T, bool kInter>
__device__ void stage_chunk(const ChunkRec& c, const PathRec* __restrict__ gpaths, const ElemRec* __restrict__ gelems,
                            const NodalSmem<T>& sm, int S, int nwarps) {
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int e = tid; e < c.n_elems; e += nth) {
    const ElemRec er = gelems[c.elem_begin + e];
    sm.elem[e] = make_int4(er.slot, __float_as_int(er.lo), __float_as_int(er.hi), tri_row_base(er.slot, S));
  }
  for (int p = tid; p < c.n_paths; p += nth) {
    const PathRec pr = gpaths[c.path_begin + p];
    sm.path[p] = make_int4(pr.k, pr.q, pr.elem, pr.table);
  }
  // tables: one warp per path, lanes over (element, node) pairs
  const int warp = tid >> 5, lane = tid & 31;
  for (int p = warp; p < c.n_paths; p += nwarps) {
    const PathRec pr = gpaths[c.path_begin + p];
    const int k = pr.k, Q = pr.q;
    const ElemRec* el = gelems + c.elem_begin + pr.elem;
    T* tab = sm.table + pr.table;
    const T* g = sm.gauss + (Q - 1) * 3 * kQMax;
    for (int idx = lane; idx < k * Q; idx += 32) {
      const int s = idx / Q, q = idx % Q;
      const double z = el[s].z, t = (double)g[q];
      const double A = z + (1.0 - z) * t;  // f_s(t_q) for o_s = 1
      const double B = z * (1.0 - t);      // f_s(t_q) for o_s = 0
      T* row = tab + 2 * Q + s * 2 * Q;
      row[q] = (T)(B / A);                 // rho
      if (kInter) row[Q + q] = (T)((1.0 - z) / A);                         // alpha = (o-z)/f for o=1
      else row[Q + q] = (T)(pr.v * (double)g[kQMax + q] * (1.0 - z) / A);  // C
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
      if (kInter) tab[Q + q] = (T)(0.5 * pr.v * w);
      else tab[Q + q] = (T)(-pr.v * w / (1.0 - t));
    }
  }
}

// One (row, path) of the SHAP kernel: lane = row.
template <typename T, int Q>
__device__ __forceinline__ void nodal_shap_path(int k, const int4* __restrict__ el, const T* __restrict__ tab,
                                                const T* __restrict__ xrow, T* __restrict__ arow) {
  const T* c = tab;
  const T* d = tab + Q;
  const T* es = tab + 2 * Q;
  T P[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) P[q] = c[q];
  uint32_t omask = 0;
  for (int s = 0; s < k; ++s) {
    const int4 r = el[s];
    const T x = xrow[r.x];
    const bool o = (x >= (T)__int_as_float(r.y)) & (x < (T)__int_as_float(r.z));
    omask |= (uint32_t)o << s;
    const T* rho = es + s * 2 * Q;
#pragma unroll
    for (int q = 0; q < Q; ++q) P[q] = o ? P[q] : P[q] * rho[q];  // EXTEND at node t_q
  }
  T phi0 = 0;
#pragma unroll
  for (int q = 0; q < Q; ++q) phi0 = fma(P[q], d[q], phi0);
  for (int s = 0; s < k; ++s) {
    const T* C = es + s * 2 * Q + Q;
    T a = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) a = fma(P[q], C[q], a);  // UNWIND folded into C
    arow[el[s].x] += ((omask >> s) & 1u) ? a : phi0;
  }
}

// One (row, path) of the interaction kernel: lane = row.
template <typename T, int Q>
__device__ __forceinline__ void nodal_inter_path(int k, const int4* __restrict__ el, const T* __restrict__ tab,
                                                 const T* __restrict__ gam, const T* __restrict__ xrow,
                                                 T* __restrict__ arow) {
  const T* c = tab;
  const T* h = tab + Q;
  const T* es = tab + 2 * Q;
  T P[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) P[q] = c[q];
  uint32_t omask = 0;
  for (int s = 0; s < k; ++s) {
    const int4 r = el[s];
    const T x = xrow[r.x];
    const bool o = (x >= (T)__int_as_float(r.y)) & (x < (T)__int_as_float(r.z));
    omask |= (uint32_t)o << s;
    const T* rho = es + s * 2 * Q;
#pragma unroll
    for (int q = 0; q < Q; ++q) P[q] = o ? P[q] : P[q] * rho[q];
  }
  T W[Q], Ssum[Q], G[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) { W[q] = h[q] * P[q]; Ssum[q] = 0; G[q] = gam[q]; }
  for (int s = 0; s < k; ++s) {
    const T* al = es + s * 2 * Q + Q;
    const bool o = (omask >> s) & 1u;
#pragma unroll
    for (int q = 0; q < Q; ++q) Ssum[q] += o ? al[q] : G[q];
  }
  for (int i = 0; i < k; ++i) {
    const int4 ri = el[i];
    const T* ai = es + i * 2 * Q + Q;
    const bool oi = (omask >> i) & 1u;
    T y[Q];
    T diag = 0, yg = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const T u = oi ? ai[q] : G[q];
      y[q] = W[q] * u;
      diag = fma(y[q], (T)2 - Ssum[q] + u, diag);  // Eq. 6 via sum_j u_j
      yg = fma(y[q], G[q], yg);                   // partner with o_j = 0
    }
    arow[ri.w + ri.x] += diag;
    for (int j = i + 1; j < k; ++j) {
      const T* aj = es + j * 2 * Q + Q;
      T s1 = 0;
#pragma unroll
      for (int q = 0; q < Q; ++q) s1 = fma(y[q], aj[q], s1);
      arow[ri.w + el[j].x] += ((omask >> j) & 1u) ? s1 : yg;
    }
  }
}

template <typename T, int Q, bool kInter>
__device__ __forceinline__ void nodal_path(int k, const int4* el, const T* tab, const T* gam, const T* xrow, T* arow) {
  if constexpr (kInter) nodal_inter_path<T, Q>(k, el, tab, gam, xrow, arow);
  else nodal_shap_path<T, Q>(k, el, tab, xrow, arow);
}

template <typename T, bool kInter>
__device__ __forceinline__ void nodal_dispatch(int4 ph, const int4* el, const T* table, const T* gauss,
                                               const T* xrow, T* arow) {
  const int k = ph.x, q = ph.y;
  const int4* e = el + ph.z;
  const T* tab = table + ph.w;
  const T* gam = gauss + (q - 1) * 3 * kQMax + 2 * kQMax;
  switch (q) {
#define GTS_CASE(QQ) case QQ: nodal_path<T, QQ, kInter>(k, e, tab, gam, xrow, arow); break;
    GTS_CASE(1) GTS_CASE(2) GTS_CASE(3) GTS_CASE(4) GTS_CASE(5) GTS_CASE(6) GTS_CASE(7) GTS_CASE(8)
    GTS_CASE(9) GTS_CASE(10) GTS_CASE(11) GTS_CASE(12) GTS_CASE(13) GTS_CASE(14) GTS_CASE(15) GTS_CASE(16)
#undef GTS_CASE
    default: break;
  }
}

struct NodalArgs {
  const char* blob;
  const void* X;
  int64_t n_rows, ld_x;
  void* out;
  int n_splits;
  int M, G, S;
  int64_t n_chunks;
  int max_elems, max_paths, max_words;
};

// acc tile width per row: SHAP = S slots, interactions = upper triangle S(S+1)/2
template <bool kInter>
__host__ __device__ constexpr int acc_width(int S) { return kInter ? S * (S + 1) / 2 : S; }

template <typename T, int S, int W, bool kInter>
__global__ void __launch_bounds__(W * 32) nodal_kernel(NodalArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const BlobHeader* hdr = reinterpret_cast<const BlobHeader*>(a.blob);
  const ChunkRec* chunks = reinterpret_cast<const ChunkRec*>(a.blob + hdr->off_units);
  const double* work = reinterpret_cast<const double*>(a.blob + hdr->off_work) + (kInter ? (a.n_chunks + 1) : 0);
  const int32_t* slotmap = reinterpret_cast<const int32_t*>(a.blob + hdr->off_slotmap);
  const PathRec* gpaths = reinterpret_cast<const PathRec*>(a.blob + hdr->off_paths);
  const ElemRec* gelems = reinterpret_cast<const ElemRec*>(a.blob + hdr->off_elems);
  const double* bias = reinterpret_cast<const double*>(a.blob + hdr->off_bias);
  (void)bias;
  const T* X = static_cast<const T*>(a.X);
  T* out = static_cast<T*>(a.out);

  constexpr int XS = S + 1;                       // odd stride: conflict-free per-lane rows
  constexpr int AW = acc_width<kInter>(S);
  constexpr int AS = AW | 1;                      // odd stride
  NodalSmem<T> sm;
  unsigned char* p = smem_raw;
  sm.gauss = reinterpret_cast<T*>(p);  p += sizeof(T) * kQMax * 3 * kQMax;
  sm.xt = reinterpret_cast<T*>(p);     p += sizeof(T) * W * 32 * XS;
  sm.acc = reinterpret_cast<T*>(p);    p += sizeof(T) * W * 32 * AS;
  p = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  sm.table = reinterpret_cast<T*>(p);  p += sizeof(T) * ((a.max_words + 3) & ~3);
  sm.elem = reinterpret_cast<int4*>(p); p += sizeof(int4) * a.max_elems;
  sm.path = reinterpret_cast<int4*>(p);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t row_tile = blockIdx.x / a.n_splits;
  const int split = blockIdx.x % a.n_splits;
  const int64_t row0 = row_tile * (W * 32) + warp * 32;
  const int64_t row = row0 + lane;
  const bool row_ok = row < a.n_rows;

  // chunk range of this split: balanced on the prefix work
  const double wtot = work[a.n_chunks];
  auto split_begin = [&](int s) -> int64_t {
    if (s >= a.n_splits) return a.n_chunks;
    const double target = wtot * (double)s / (double)a.n_splits;
    int64_t lo = 0, hi = a.n_chunks;  // first c with work[c] >= target
    while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (work[mid] < target) lo = mid + 1; else hi = mid; }
    return lo;
  };
  const int64_t c_begin = split_begin(split), c_end = split_begin(split + 1);

  const T* gsrc = reinterpret_cast<const T*>(a.blob + hdr->off_gauss);
  for (int i = tid; i < kQMax * 3 * kQMax; i += blockDim.x) sm.gauss[i] = gsrc[i];
  T* xrow = sm.xt + (warp * 32 + lane) * XS;
  T* arow = sm.acc + (warp * 32 + lane) * AS;
  for (int i = 0; i < AW; ++i) arow[i] = (T)0;

  const int M1 = a.M + 1;
  int cur_map = -1, cur_group = -1, cur_slots = 0;
  int64_t cur_map_begin = 0;
  bool dirty = false;

  // flush this lane's accumulator row to phi (one atomic per non-zero cell)
  auto flush = [&]() {
    if (row_ok && dirty) {
      if constexpr (kInter) {
        T* base = out + ((size_t)row * a.G + cur_group) * (size_t)M1 * M1;
        for (int i = 0; i < cur_slots; ++i) {
          const int fi = slotmap[cur_map_begin + i];
          const int rb = tri_row_base(i, S);
          for (int j = i; j < cur_slots; ++j) {
            const T v = arow[rb + j];
            if (v != (T)0) {
              const int fj = slotmap[cur_map_begin + j];
              atomicAdd(base + (size_t)fi * M1 + fj, v);
              if (j != i) atomicAdd(base + (size_t)fj * M1 + fi, v);
              arow[rb + j] = (T)0;
            }
          }
        }
      } else {
        T* base = out + ((size_t)row * a.G + cur_group) * (size_t)M1;
        for (int i = 0; i < cur_slots; ++i) {
          const T v = arow[i];
          if (v != (T)0) {
            atomicAdd(base + slotmap[cur_map_begin + i], v);
            arow[i] = (T)0;
          }
        }
      }
    }
    dirty = false;
  };

  for (int64_t ci = c_begin; ci < c_end; ++ci) {
    const ChunkRec c = chunks[ci];
    __syncthreads();  // previous chunk's tables no longer in use
    stage_chunk<T, kInter>(c, gpaths, gelems, sm, S, W);
    if (c.map_id != cur_map || c.group != cur_group) {
      flush();
      if (c.map_id != cur_map) {
        // gather this lane's row of X into slot order
        for (int i = 0; i < c.n_slots; ++i)
          xrow[i] = row_ok ? X[(size_t)row * a.ld_x + slotmap[c.slotmap_begin + i]] : (T)0;
      }
      cur_map = c.map_id;
      cur_group = c.group;
      cur_slots = c.n_slots;
      cur_map_begin = c.slotmap_begin;
    }
    __syncthreads();  // tables staged
    if (row0 < a.n_rows) {
      for (int pth = 0; pth < c.n_paths; ++pth)
        nodal_dispatch<T, kInter>(sm.path[pth], sm.elem, sm.table, sm.gauss, xrow, arow);
      dirty = true;
    }
  }
  flush();
}

// ------------------------------------------------------- WARP_BINS family

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
  int64_t n_rows, ld_x;
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
      const T x = X[row * a.ld_x + feat];
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
      const T x = X[row * a.ld_x + feat0];
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

// ------------------------------------------------------------- launchers

constexpr int64_t kBiasOffset = 256;  // align256(sizeof(BlobHeader)), host.cpp blob_plan

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

gts_status cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GTS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return GTS_OK;
}

template <typename T>
gts_status launch_init(bool inter, const gts_blob_info* info, const char* d_blob, int64_t n_rows, void* out,
                       cudaStream_t st) {
  const double* bias = reinterpret_cast<const double*>(d_blob + kBiasOffset);
  const int64_t M1 = info->n_features + 1;
  const int64_t total = n_rows * info->n_groups * (inter ? M1 * M1 : M1);
  const int threads = 256;
  const int64_t want = (total + threads - 1) / threads;
  const int blocks = (int)std::min<int64_t>(want, (int64_t)num_sms() * 16);
  if (inter)
    init_phi_ij_kernel<T><<<blocks, threads, 0, st>>>(static_cast<T*>(out), n_rows, info->n_groups,
                                                       info->n_features, bias);
  else
    init_phi_kernel<T><<<blocks, threads, 0, st>>>(static_cast<T*>(out), n_rows, info->n_groups,
                                                    info->n_features, bias);
  return cuda_check("init kernel launch");
}

template <typename T, bool kInter, int S>
constexpr int nodal_warps() {
  constexpr int XS = S + 1;
  constexpr int AS = acc_width<kInter>(S) | 1;
  return (sizeof(T) * 32 * (XS + AS) * 8 <= 160 * 1024) ? 8 : 4;
}

template <typename T, bool kInter, int S>
size_t nodal_smem_bytes(const gts_blob_info* info) {
  constexpr int W = nodal_warps<T, kInter, S>();
  constexpr int XS = S + 1;
  constexpr int AS = acc_width<kInter>(S) | 1;
  size_t b = sizeof(T) * (kQMax * 3 * kQMax + (size_t)W * 32 * XS + (size_t)W * 32 * AS);
  b = (b + 15) & ~size_t(15);
  b += sizeof(T) * (size_t)((info->max_chunk_words + 3) & ~3);
  b += sizeof(int4) * (size_t)info->max_chunk_elems;
  b += sizeof(int4) * (size_t)info->max_chunk_paths;
  return b;
}

template <typename T, bool kInter, int S>
gts_status launch_nodal(const gts_blob_info* info, const char* d_blob, const void* d_X, int64_t n_rows, int64_t ld_x,
                        void* out, cudaStream_t st) {
  constexpr int W = nodal_warps<T, kInter, S>();
  auto kern = nodal_kernel<T, S, W, kInter>;
  const size_t smem = nodal_smem_bytes<T, kInter, S>(info);
  if (smem > 227 * 1024) return fail(GTS_ERR_INVALID_ARGUMENT, "chunk staging needs %zu bytes of shared memory", smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
  per_sm = std::max(per_sm, 1);
  const int64_t row_tiles = (n_rows + W * 32 - 1) / (W * 32);
  const int64_t target = (int64_t)num_sms() * per_sm * 2;
  int64_t splits = (target + row_tiles - 1) / row_tiles;
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, std::min<int64_t>(info->n_units, 1024)));
  NodalArgs a;
  a.blob = d_blob;
  a.X = d_X;
  a.n_rows = n_rows;
  a.ld_x = ld_x;
  a.out = out;
  a.n_splits = (int)splits;
  a.M = info->n_features;
  a.G = info->n_groups;
  a.S = S;
  a.n_chunks = info->n_units;
  a.max_elems = (int)info->max_chunk_elems;
  a.max_paths = (int)info->max_chunk_paths;
  a.max_words = (int)info->max_chunk_words;
  if (info->n_units == 0) return GTS_OK;
  const int64_t blocks = row_tiles * splits;
  if (blocks > INT32_MAX) return fail(GTS_ERR_INVALID_ARGUMENT, "too many rows");
  kern<<<(unsigned)blocks, W * 32, smem, st>>>(a);
  return cuda_check("nodal kernel launch");
}

template <typename T, bool kInter>
gts_status launch_nodal_s(const gts_blob_info* info, const char* d_blob, const void* d_X, int64_t n_rows,
                          int64_t ld_x, void* out, cudaStream_t st) {
  switch (info->max_slots) {
    case 16: return launch_nodal<T, kInter, 16>(info, d_blob, d_X, n_rows, ld_x, out, st);
    case 32:
      if constexpr (kInter) break;
      else return launch_nodal<T, kInter, 32>(info, d_blob, d_X, n_rows, ld_x, out, st);
    case 64:
      if constexpr (kInter) break;
      else return launch_nodal<T, kInter, 64>(info, d_blob, d_X, n_rows, ld_x, out, st);
    default: break;
  }
  return fail(GTS_ERR_INVALID_ARGUMENT,
              kInter ? "interaction kernel needs a NODAL blob with max_slots == 16 (got %d)"
                     : "unsupported max_slots %d",
              info->max_slots);
}

template <typename T, bool kInter>
gts_status launch_bins(const gts_blob_info* info, const char* d_blob, const void* d_X, int64_t n_rows, int64_t ld_x,
                       void* out, cudaStream_t st) {
  constexpr int W = 4;
  if (info->n_units == 0) return GTS_OK;
  BinArgs a;
  a.blob = d_blob;
  a.X = d_X;
  a.n_rows = n_rows;
  a.ld_x = ld_x;
  a.out = out;
  a.M = info->n_features;
  a.G = info->n_groups;
  a.n_bins = info->n_units;
  a.rows_per_item = (int)std::max<int64_t>(kInter ? 8 : 32, (n_rows + 65534) / 65535);
  dim3 grid((unsigned)((info->n_units + W - 1) / W), (unsigned)((n_rows + a.rows_per_item - 1) / a.rows_per_item));
  if (kInter) bins_inter_kernel<T, W><<<grid, W * 32, 0, st>>>(a);
  else bins_shap_kernel<T, W><<<grid, W * 32, 0, st>>>(a);
  return cuda_check("warp-bin kernel launch");
}

gts_status check_call(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows, int64_t ld_x,
                      void* d_out) {
  if (!info) return fail(GTS_ERR_INVALID_ARGUMENT, "info is NULL");
  if (info->magic != kMagic || info->abi_version != GTS_ABI_VERSION)
    return fail(GTS_ERR_INVALID_ARGUMENT, "info is not a gts_blob_info of ABI version %d", GTS_ABI_VERSION);
  if (info->dtype != GTS_F32 && info->dtype != GTS_F64) return fail(GTS_ERR_INVALID_ARGUMENT, "bad dtype");
  if (info->layout != GTS_LAYOUT_NODAL && info->layout != GTS_LAYOUT_WARP_BINS)
    return fail(GTS_ERR_INVALID_ARGUMENT, "bad layout");
  if (n_rows < 0) return fail(GTS_ERR_INVALID_ARGUMENT, "n_rows < 0");
  if (n_rows == 0) return GTS_OK;
  if (!d_blob || !d_X || !d_out) return fail(GTS_ERR_INVALID_ARGUMENT, "NULL device pointer");
  if (ld_x < info->n_features) return fail(GTS_ERR_INVALID_ARGUMENT, "ld_x < n_features");
  const size_t ts = info->dtype == GTS_F32 ? 4 : 8;
  if ((reinterpret_cast<uintptr_t>(d_blob) & 15) != 0) return fail(GTS_ERR_INVALID_ARGUMENT, "blob not 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(d_X) % ts) != 0 || (reinterpret_cast<uintptr_t>(d_out) % ts) != 0)
    return fail(GTS_ERR_INVALID_ARGUMENT, "X / phi not aligned to the element size");
  return GTS_OK;
}

template <bool kInter>
gts_status run(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows, int64_t ld_x,
               void* d_out, void* stream) {
  gts_status s = check_call(info, d_blob, d_X, n_rows, ld_x, d_out);
  if (s != GTS_OK || n_rows == 0) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* blob = static_cast<const char*>(d_blob);
  const bool f32 = info->dtype == GTS_F32;
  s = f32 ? launch_init<float>(kInter, info, blob, n_rows, d_out, st)
          : launch_init<double>(kInter, info, blob, n_rows, d_out, st);
  if (s != GTS_OK) return s;
  if (info->layout == GTS_LAYOUT_NODAL)
    return f32 ? launch_nodal_s<float, kInter>(info, blob, d_X, n_rows, ld_x, d_out, st)
               : launch_nodal_s<double, kInter>(info, blob, d_X, n_rows, ld_x, d_out, st);
  return f32 ? launch_bins<float, kInter>(info, blob, d_X, n_rows, ld_x, d_out, st)
             : launch_bins<double, kInter>(info, blob, d_X, n_rows, ld_x, d_out, st);
}

}  // namespace
}  // namespace gts

extern "C" {

gts_status gts_shap(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows, int64_t ld_x,
                    void* d_phi, void* stream) {
  return gts::run<false>(info, d_blob, d_X, n_rows, ld_x, d_phi, stream);
}

gts_status gts_shap_interactions(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows,
                                 int64_t ld_x, void* d_phi_ij, void* stream) {
  return gts::run<true>(info, d_blob, d_X, n_rows, ld_x, d_phi_ij, stream);
}

int32_t gts_launches_per_call(const gts_blob_info* info, int32_t interactions) {
  (void)interactions;
  if (!info) return 0;
  return info->n_units > 0 ? 2 : 1;  // init + main kernel
}

}  // extern "C"

