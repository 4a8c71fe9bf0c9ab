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
#include <cstdlib>

#include "../../include/gts.h"
#include "blob_format.h"
#include "nodal.cuh"
#include "trace.h"
#include "warp_bins.cuh"

namespace gts {
gts_status fail(gts_status st, const char* fmt, ...);
}

// The library is built from several compilations of this file (_build.py,
// in parallel): GTS_PART = 0 holds everything except the NODAL launches,
// GTS_PART = 1..4 instantiate launch_nodal (and so the nodal kernels) for
// {fp32, fp64} x {SHAP, interactions}.
#ifndef GTS_PART
#define GTS_PART 0
#endif

namespace gts {
namespace {


// ------------------------------------------------------------ init kernels

// The outputs are zeroed with cudaMemsetAsync; this kernel then writes the
// bias cells (reading G14): phi[row][g][M] = bias[g] (stride M + 1, cell M) or
// phi_ij[row][g][M][M] = bias[g] (stride (M + 1)^2, cell (M + 1)^2 - 1).
template <typename T>
__global__ void bias_cells_kernel(T* __restrict__ out, int64_t n_rg, int G, int64_t stride, int64_t cell,
                                  const double* __restrict__ bias) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rg; i += (int64_t)gridDim.x * blockDim.x)
    out[i * stride + cell] = (T)bias[i % G];
}

// phi_ij is symmetric (Eq. 3).  With per-chunk slot maps (wide models) the
// interaction kernel adds each pair once, to (i, j) with feature i < j (slot
// maps are sorted), which halves its atomics; this pass then copies the upper
// triangle of every [M+1][M+1] matrix onto the lower one through 32 x 32
// shared-memory tiles (coalesced reads and writes).
template <typename T>
__global__ void mirror_kernel(T* __restrict__ phi, int64_t n_mats, int M1) {
  __shared__ T tile[32][33];
  const int nt = (M1 + 31) / 32;
  const int64_t tiles_per_mat = (int64_t)nt * (nt + 1) / 2;
  for (int64_t t = blockIdx.x; t < n_mats * tiles_per_mat; t += gridDim.x) {
    const int64_t mat = t / tiles_per_mat;
    const int tt = (int)(t - mat * tiles_per_mat);
    int bi = 0;  // lower-triangle tile (bi, bj), bi >= bj
    while ((bi + 1) * (bi + 2) / 2 <= tt) ++bi;
    const int bj = tt - bi * (bi + 1) / 2;
    T* m = phi + mat * (int64_t)M1 * M1;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
      const int a = bj * 32 + y, b = bi * 32 + threadIdx.x;  // upper source (a, b)
      if (a < M1 && b < M1) tile[y][threadIdx.x] = m[(int64_t)a * M1 + b];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
      const int b = bi * 32 + y, a = bj * 32 + threadIdx.x;  // lower target (b, a) = (a, b)
      if (a < M1 && b < M1 && b > a) m[(int64_t)b * M1 + a] = tile[threadIdx.x][y];
    }
    __syncthreads();
  }
}

#ifndef GTS_TILE_MINOR
#define GTS_TILE_MINOR 4  // item order: 0 split-minor, 1 tile-minor for group-major models, 2 always tile-minor,
                          // 3 tile-minor for identity slot maps, 4 tile-minor except SHAP with per-chunk slot maps
                          // (measured, profiles/r02o: adult both +7 %, fashion SHAP +8 % over mode 1)
#endif
#ifndef GTS_GROUP_MAJOR
#define GTS_GROUP_MAJOR 2  // group-major blocks: 0 never, 1 per-chunk slot maps (wide models), 2 whenever G > 1
                           // (measured, profiles/r02d: fashion SHAP 2.94e5 -> 5.06e5 rows/s, covtype 1.21e4 -> 1.40e4)
#endif
#ifndef GTS_L2_BUDGET_MB
#define GTS_L2_BUDGET_MB 32  // rows in flight keep X + phi (phi_ij) under this many MiB of L2
#endif

#ifndef GTS_INTER_MIRROR
#define GTS_INTER_MIRROR 1  // per-chunk slot maps: upper-triangle atomics + mirror pass
#endif

bool uses_mirror(const gts_blob_info* info) {
  return GTS_INTER_MIRROR && info->layout == GTS_LAYOUT_NODAL && info->n_units > 0 &&
         info->max_slots < info->n_features;
}

// ------------------------------------------------- X validation (reading G17)

// first[0] = smallest linear (row * M + feature) index of a non-finite X entry
template <typename T>
__global__ void nonfinite_kernel(const T* __restrict__ X, int64_t n_rows, int M, int64_t rs, int64_t cs,
                                 unsigned long long* first) {
  const int64_t total = n_rows * M;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / M, f = i - r * M;
    const T v = X[r * rs + f * cs];
    if (!isfinite(v)) atomicMin(first, (unsigned long long)i);
  }
}

// Feature-major copy of X for the kernels that read X from global memory
// (nodal::xg_enabled): xt[f * ld + r] = X[r][f] for r < n.  Row-major X goes
// through 32 x 32 shared tiles (coalesced on both sides); feature-major X is a
// strided column copy.
template <typename T>
__global__ void transpose_x_kernel(const T* __restrict__ X, int64_t n, int M, int64_t rs, T* __restrict__ xt,
                                   int64_t ld) {
  __shared__ T tile[32][33];
  const int64_t tiles_r = (n + 31) / 32;
  const int tiles_f = (M + 31) / 32;
  for (int64_t t = blockIdx.x; t < tiles_r * tiles_f; t += gridDim.x) {
    const int64_t r0 = (t / tiles_f) * 32;
    const int f0 = (int)(t % tiles_f) * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
      const int64_t r = r0 + y;
      const int f = f0 + threadIdx.x;
      if (r < n && f < M) tile[y][threadIdx.x] = X[r * rs + f];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
      const int f = f0 + y;
      const int64_t r = r0 + threadIdx.x;
      if (r < n && f < M) xt[(int64_t)f * ld + r] = tile[threadIdx.x][y];
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void copy_cols_kernel(const T* __restrict__ X, int64_t n, int M, int64_t cs, T* __restrict__ xt,
                                 int64_t ld) {
  const int64_t total = n * M;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i / n, r = i - f * n;
    xt[f * ld + r] = X[f * cs + r];
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
  const int64_t stride = inter ? M1 * M1 : M1;
  const int64_t n_rg = n_rows * info->n_groups;
  if (cudaMemsetAsync(out, 0, (size_t)(n_rg * stride) * sizeof(T), st) != cudaSuccess)
    return cuda_check("output zero fill");
  const int blocks = (int)std::min<int64_t>((n_rg + 255) / 256, (int64_t)num_sms() * 8);
  bias_cells_kernel<T><<<blocks, 256, 0, st>>>(static_cast<T*>(out), n_rg, info->n_groups, stride, stride - 1, bias);
  return cuda_check("bias kernel launch");
}

size_t nodal_buffer_bytes(const gts_blob_info* info) {
  return ((size_t)info->max_chunk_bytes + 127) & ~size_t(127);
}

int shap_tile_w(const gts_blob_info* info) { return (int)((info->max_chunk_slots + 1) | 1); }

template <typename T, bool kInter, int S>
size_t nodal_smem_bytes(const gts_blob_info* info) {
  constexpr int W = nodal::Cfg<T, kInter, S>::W;
  constexpr int R = nodal::Cfg<T, kInter, S>::R;
  // tiles, then two TMA staging buffers (double buffering) and their mbarriers
  return (size_t)nodal::staging_byte_offset<T, S, W, R, kInter>(shap_tile_w(info)) + 2 * nodal_buffer_bytes(info) + 16;
}

}  // namespace
namespace nl {
template <typename T, bool kInter, int S>
gts_status launch_nodal(const gts_blob_info* info, const char* d_blob, const void* d_X, int64_t n_rows, int64_t rs,
                        int64_t cs, void* out, cudaStream_t st, void* out_phi) {
  constexpr int W = nodal::Cfg<T, kInter, S>::W;
  constexpr int R = nodal::Cfg<T, kInter, S>::R;
  constexpr int XG = nodal::xg_enabled<kInter, S>() ? 1 : 0;
  auto kern = nodal::nodal_kernel<T, S, W, R, kInter, XG>;
  if constexpr (XG == 1 && GTS_TMEM_X && sizeof(T) == 4 && S == 64 && W == 4 && R * 64 <= 128) {
    // identity slot map (features = slots < 64): x from TMEM by feature (nodal::load_x)
    if (info->n_features <= 64) kern = nodal::nodal_kernel<T, S, W, R, kInter, 2>;
  }
  if constexpr (XG == 1 && (GTS_TMEM_X & 2) && sizeof(T) == 4 && S == 32 && W == 4 && R * S <= 64) {
    kern = nodal::nodal_kernel<T, S, W, R, kInter, 3>;  // per-chunk maps: x from TMEM by slot
  }
  const size_t smem = nodal_smem_bytes<T, kInter, S>(info);
  if (smem > 227 * 1024) return fail(GTS_ERR_INVALID_ARGUMENT, "chunk staging needs %zu bytes of shared memory", smem);
  void* xt = nullptr;  // padded feature-major scratch copy of X (xg kernels)
  if constexpr (nodal::xg_enabled<kInter, S>()) {
    if (info->n_units > 0) {
      const int M = info->n_features;
      const int64_t rpb = (int64_t)W * 32 * R;
      // element indices feature * ld + row are 32-bit in the kernel: split huge calls
      const int64_t max_rows = std::max<int64_t>(rpb, ((INT32_MAX / std::max(M, 1)) / rpb - 1) * rpb);
      if (n_rows > max_rows) {
        const int64_t out_row = (int64_t)info->n_groups * (info->n_features + 1);
        for (int64_t r0 = 0; r0 < n_rows; r0 += max_rows) {
          const T* xs = static_cast<const T*>(d_X) + r0 * rs;
          T* os = static_cast<T*>(out) + r0 * out_row;
          gts_status s0 = launch_nodal<T, kInter, S>(info, d_blob, xs, std::min(max_rows, n_rows - r0), rs, cs, os, st,
                                                     out_phi);
          if (s0 != GTS_OK) return s0;
        }
        return GTS_OK;
      }
      const int64_t ld = (n_rows + rpb - 1) / rpb * rpb;  // whole row tiles: lanes of the last tile read the pad
      const size_t bytes = (size_t)ld * M * sizeof(T);
      if (cudaMallocAsync(&xt, bytes, st) != cudaSuccess)
        return fail(GTS_ERR_OUT_OF_MEMORY, "cudaMallocAsync of %zu bytes for the feature-major X copy failed", bytes);
      if (ld > n_rows)
        cudaMemset2DAsync(static_cast<T*>(xt) + n_rows, (size_t)ld * sizeof(T), 0, (size_t)(ld - n_rows) * sizeof(T),
                          (size_t)M, st);
      if (rs == 1 && cs != 1) {  // feature-major input
        const int blocks = (int)std::min<int64_t>((n_rows * M + 255) / 256, (int64_t)num_sms() * 16);
        copy_cols_kernel<T><<<blocks, 256, 0, st>>>(static_cast<const T*>(d_X), n_rows, M, cs, static_cast<T*>(xt), ld);
      } else {
        const int64_t tiles = ((n_rows + 31) / 32) * ((M + 31) / 32);
        const int tb = (int)std::min<int64_t>(tiles, (int64_t)num_sms() * 16);
        transpose_x_kernel<T><<<tb, dim3(32, 8), 0, st>>>(static_cast<const T*>(d_X), n_rows, M, rs,
                                                           static_cast<T*>(xt), ld);
      }
      gts_status s0 = cuda_check("X transpose launch");
      if (s0 != GTS_OK) {
        cudaFreeAsync(xt, st);
        return s0;
      }
      d_X = xt;
      rs = 1;
      cs = ld;
    }
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // The occupancy query assumes the kernel's preferred shared-memory carveout;
  // without one it reported 1 block per SM for kernels that run 3 (ncu:
  // occupancy limits 3 / 3, profiles/r02j), which sized the persistent grid at
  // one block per SM.  Ask for the largest carveout first.
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 1;
  }
  per_sm = std::max(per_sm, 1);
  {
    // The query still returned 1 for the 64-slot SHAP kernel that ncu shows
    // running 3 per SM (r02k), so the limits are also computed here from the
    // kernel's registers and shared memory (and TMEM columns for XG >= 2), and
    // the larger count is used.
    cudaFuncAttributes fa{};
    int dev = 0, smem_sm = 0, reserved = 0;
    cudaGetDevice(&dev);
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess &&
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev) == cudaSuccess) {
      const int64_t regs_warp = ((int64_t)std::max(fa.numRegs, 1) * 32 + 255) / 256 * 256;
      int64_t lim = std::min<int64_t>(65536 / (regs_warp * W), 64 / W);
      lim = std::min<int64_t>(lim, smem_sm / ((int64_t)smem + fa.sharedSizeBytes + reserved));
      if (kern != nodal::nodal_kernel<T, S, W, R, kInter, XG>) lim = std::min<int64_t>(lim, 4);  // TMEM X: 128 / 64 columns
      per_sm = std::max<int>(per_sm, (int)std::max<int64_t>(lim, 1));
    }
    cudaGetLastError();
  }
  if (const char* e = getenv("GTS_DEBUG_LAUNCH"))
    if (e[0] == '1') fprintf(stderr, "gts: nodal launch S=%d W=%d R=%d inter=%d smem=%zu per_sm=%d\n", S, W, R, (int)kInter, smem, per_sm);
  const int64_t rows_per_block = (int64_t)W * 32 * R;
  const int64_t row_tiles = (n_rows + rows_per_block - 1) / rows_per_block;
  const int64_t resident = (int64_t)num_sms() * per_sm;
  const int64_t target = resident * 2;
  const int64_t M1 = info->n_features + 1;
  const int64_t l2_budget = (int64_t)GTS_L2_BUDGET_MB << 20;
  const int G = info->n_groups;
  // Group-major blocks (Args::n_bgroups) for per-chunk slot maps: the gathers
  // re-read X and the flush REDs hit phi (phi_ij) once per chunk, so the rows
  // in flight must keep their X rows and phi rows in L2.  Blocks are dispatched
  // in index order, so with (batch, group, tile, split) order the resident
  // blocks share one batch of rows and one group: tiles_per_batch is sized so
  // that a batch's X and one group's outputs fit the L2 budget.
  const bool wide = info->max_slots < info->n_features;
  const int nbg = (G > 1 && (GTS_GROUP_MAJOR == 2 || (GTS_GROUP_MAJOR == 1 && wide))) ? G : 1;
  const bool tile_minor = GTS_TILE_MINOR == 2 || GTS_PERSIST || (GTS_TILE_MINOR == 1 && nbg > 1) ||
                          (GTS_TILE_MINOR == 3 && !wide) || (GTS_TILE_MINOR == 4 && (kInter || !wide));
  int64_t tiles_per_batch = std::max<int64_t>(row_tiles, 1), splits;
  if (nbg > 1) {
    const int64_t bytes_per_row = (int64_t)sizeof(T) * (info->n_features + (kInter ? M1 * M1 : M1));
    tiles_per_batch = std::max<int64_t>(1, std::min<int64_t>(tiles_per_batch,
                                                             l2_budget / (rows_per_block * bytes_per_row)));
    splits = (target + tiles_per_batch - 1) / tiles_per_batch;
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, info->n_units / G));
  } else if (tile_minor) {
    // Persistent blocks take items tile-minor within a (batch, split), so the
    // items in flight are up to tiles_per_batch row tiles of a few splits:
    // batches keep those rows' X and phi (phi_ij) within the L2 budget.
    const int64_t bytes_per_row = (int64_t)sizeof(T) * (info->n_features + (kInter ? M1 * M1 : M1));
    tiles_per_batch = std::max<int64_t>(1, std::min<int64_t>(tiles_per_batch,
                                                             l2_budget / (rows_per_block * bytes_per_row)));
    splits = (target + tiles_per_batch - 1) / tiles_per_batch;
  } else {
    // One block per item, split-minor (Args::tile_minor = 0): the first
    // `resident` blocks cover resident / splits row tiles.  Keep the rows in
    // flight small enough that their X rows and phi (phi_ij) rows stay in L2;
    // splits only add one flush per split boundary.
    splits = (target + row_tiles - 1) / row_tiles;
    const int64_t bytes_per_row = (int64_t)sizeof(T) * (info->n_features + (kInter ? M1 * M1 : M1));
    const int64_t want = (resident * rows_per_block * bytes_per_row + l2_budget - 1) / l2_budget;
    splits = std::max(splits, std::min(want, row_tiles > 0 ? resident : 1));
  }
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, std::min<int64_t>(info->n_units, 1024)));
  const int64_t n_batches = (row_tiles + tiles_per_batch - 1) / tiles_per_batch;
  nodal::Args a;
  a.blob = d_blob;
  a.X = d_X;
  a.n_rows = n_rows;
  a.row_stride = rs;
  a.col_stride = cs;
  a.out = out;
  a.out_phi = out_phi;
  a.upper_only = kInter && uses_mirror(info);
  a.n_splits = (int)splits;
  a.n_bgroups = nbg;
  a.tiles_per_batch = tiles_per_batch;
  a.n_batches = n_batches;
  // item order: tile-minor (the items in flight share a chunk stream) for
  // persistent blocks and group-major models, split-minor (they share rows)
  // for single-group models with one block per item (cal_housing both: +6 %, r02l)
  a.tile_minor = tile_minor ? 1 : 0;
  a.tile_w = shap_tile_w(info);
  a.M = info->n_features;
  a.G = info->n_groups;
  a.n_chunks = info->n_units;
  a.max_chunk_bytes = (int)nodal_buffer_bytes(info);
  if (info->n_units == 0) return GTS_OK;
  const int64_t blocks = n_batches * nbg * tiles_per_batch * splits;
  if (blocks > INT32_MAX) {
    if (xt != nullptr) cudaFreeAsync(xt, st);
    return fail(GTS_ERR_INVALID_ARGUMENT, "too many rows");
  }
  // persistent grid: the resident blocks walk the work items in order (nodal_kernel);
  // GTS_PERSIST=0: one block per item
  const int64_t grid = GTS_PERSIST ? std::min<int64_t>(blocks, resident) : blocks;
  kern<<<(unsigned)grid, W * 32, smem, st>>>(a);
  gts_status s = cuda_check("nodal kernel launch");
  if (xt != nullptr) cudaFreeAsync(xt, st);  // stream-ordered: after the kernel
  if (s != GTS_OK || !a.upper_only) return s;
  const int64_t nt = (M1 + 31) / 32;
  const int64_t tiles = n_rows * info->n_groups * (nt * (nt + 1) / 2);
  const int mblocks = (int)std::min<int64_t>(tiles, (int64_t)num_sms() * 16);
  mirror_kernel<T><<<mblocks, dim3(32, 8), 0, st>>>(static_cast<T*>(out), n_rows * info->n_groups, (int)M1);
  return cuda_check("mirror kernel launch");
}

#define GTS_LN_SIG(T, I, S)                                                                                       \
  gts_status launch_nodal<T, I, S>(const gts_blob_info*, const char*, const void*, int64_t, int64_t, int64_t, void*, \
                                   cudaStream_t, void*)
#if GTS_PART == 0
#define GTS_LN(T, I, S) extern template GTS_LN_SIG(T, I, S);
#else
#define GTS_LN(T, I, S) template GTS_LN_SIG(T, I, S);
#endif
#if GTS_PART == 0 || GTS_PART == 1
GTS_LN(float, false, 8) GTS_LN(float, false, 16) GTS_LN(float, false, 32) GTS_LN(float, false, 64)
#endif
#if GTS_PART == 0 || GTS_PART == 2
GTS_LN(float, true, 8) GTS_LN(float, true, 16) GTS_LN(float, true, 32)
#endif
#if GTS_PART == 0 || GTS_PART == 3
GTS_LN(double, false, 8) GTS_LN(double, false, 16) GTS_LN(double, false, 32) GTS_LN(double, false, 64)
#endif
#if GTS_PART == 0 || GTS_PART == 4
GTS_LN(double, true, 8) GTS_LN(double, true, 16) GTS_LN(double, true, 32)
#endif
#undef GTS_LN
#undef GTS_LN_SIG
}  // namespace nl
#if GTS_PART == 0
namespace {
using nl::launch_nodal;

template <typename T, bool kInter>
gts_status launch_nodal_s(const gts_blob_info* info, const char* d_blob, const void* d_X, int64_t n_rows,
                          int64_t rs, int64_t cs, void* out, cudaStream_t st, void* out_phi = nullptr) {
  switch (info->max_slots) {
    case 8: return launch_nodal<T, kInter, 8>(info, d_blob, d_X, n_rows, rs, cs, out, st, out_phi);
    case 16: return launch_nodal<T, kInter, 16>(info, d_blob, d_X, n_rows, rs, cs, out, st, out_phi);
    case 32: return launch_nodal<T, kInter, 32>(info, d_blob, d_X, n_rows, rs, cs, out, st, out_phi);
    case 64:
      if constexpr (kInter) break;
      else return launch_nodal<T, kInter, 64>(info, d_blob, d_X, n_rows, rs, cs, out, st, nullptr);
    default: break;
  }
  return fail(GTS_ERR_INVALID_ARGUMENT, "unsupported max_slots %d", info->max_slots);
}

// Shared memory of the NODAL launch for this blob (0 = no such kernel).
template <typename T, bool kInter>
size_t nodal_smem_for(const gts_blob_info* info) {
  switch (info->max_slots) {
    case 8: return nodal_smem_bytes<T, kInter, 8>(info);
    case 16: return nodal_smem_bytes<T, kInter, 16>(info);
    case 32: return nodal_smem_bytes<T, kInter, 32>(info);
    case 64: return kInter ? 0 : nodal_smem_bytes<T, kInter, 64>(info);
    default: return 0;
  }
}

// NODAL blob / kernel compatibility, checked before anything is launched
// (the init fills overwrite the caller's outputs).
gts_status check_nodal(const gts_blob_info* info, bool inter) {
  if (info->layout != GTS_LAYOUT_NODAL || info->n_units == 0) return GTS_OK;
  const int S = info->max_slots;
  if (inter) {
    if (!(info->uses & GTS_USE_INTERACTIONS) || info->n_tables != 3 || (S != 8 && S != 16 && S != 32))
      return fail(GTS_ERR_INVALID_ARGUMENT,
                  "the interaction kernel needs a NODAL blob planned for interactions (uses %d, max_slots %d): "
                  "use gts_blob_plan_for(..., GTS_USE_INTERACTIONS, ...)", info->uses, S);
  } else {
    if (!(info->uses & GTS_USE_SHAP) || info->n_tables != nodal_tables(S) ||
        (S != 8 && S != 16 && S != 32 && S != 64))
      return fail(GTS_ERR_INVALID_ARGUMENT,
                  "the SHAP kernel needs a NODAL blob planned for SHAP (uses %d, max_slots %d, %d tables)", info->uses,
                  S, info->n_tables);
  }
  const size_t smem = info->dtype == GTS_F32 ? (inter ? nodal_smem_for<float, true>(info) : nodal_smem_for<float, false>(info))
                                             : (inter ? nodal_smem_for<double, true>(info) : nodal_smem_for<double, false>(info));
  if (smem == 0 || smem > 227 * 1024)
    return fail(GTS_ERR_INVALID_ARGUMENT, "chunk staging needs %zu bytes of shared memory", smem);
  return GTS_OK;
}

template <typename T, bool kInter>
gts_status launch_bins(const gts_blob_info* info, const char* d_blob, const void* d_X, int64_t n_rows, int64_t rs,
                       int64_t cs, void* out, cudaStream_t st) {
  constexpr int W = 4;
  if (info->n_units == 0) return GTS_OK;
  wb::BinArgs a;
  a.blob = d_blob;
  a.X = d_X;
  a.n_rows = n_rows;
  a.row_stride = rs;
  a.col_stride = cs;
  a.out = out;
  a.M = info->n_features;
  a.G = info->n_groups;
  a.n_bins = info->n_units;
  a.rows_per_item = (int)std::max<int64_t>(kInter ? 8 : 32, (n_rows + 65534) / 65535);
  dim3 grid((unsigned)((info->n_units + W - 1) / W), (unsigned)((n_rows + a.rows_per_item - 1) / a.rows_per_item));
  if (kInter) wb::bins_inter_kernel<T, W><<<grid, W * 32, 0, st>>>(a);
  else wb::bins_shap_kernel<T, W><<<grid, W * 32, 0, st>>>(a);
  return cuda_check("warp-bin kernel launch");
}

gts_status check_call(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows, int64_t rs, int64_t cs,
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
  const bool row_major = cs == 1 && rs >= info->n_features;
  const bool feature_major = rs == 1 && cs >= n_rows;
  if (!row_major && !feature_major)
    return fail(GTS_ERR_INVALID_ARGUMENT,
                "X strides (%lld, %lld): need row-major (col_stride 1, row_stride >= n_features) or "
                "feature-major (row_stride 1, col_stride >= n_rows)", (long long)rs, (long long)cs);
  const size_t ts = info->dtype == GTS_F32 ? 4 : 8;
  if ((reinterpret_cast<uintptr_t>(d_blob) & 15) != 0) return fail(GTS_ERR_INVALID_ARGUMENT, "blob not 16-byte aligned");
  if ((reinterpret_cast<uintptr_t>(d_X) % ts) != 0 || (reinterpret_cast<uintptr_t>(d_out) % ts) != 0)
    return fail(GTS_ERR_INVALID_ARGUMENT, "X / phi not aligned to the element size");
  return GTS_OK;
}

template <bool kInter>
gts_status run(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows, int64_t rs, int64_t cs,
               void* d_out, void* stream) {
  gts_status s = check_call(info, d_blob, d_X, n_rows, rs, cs, d_out);
  if (s != GTS_OK || n_rows == 0) return s;
  s = check_nodal(info, kInter);
  if (s != GTS_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* blob = static_cast<const char*>(d_blob);
  const bool f32 = info->dtype == GTS_F32;
  s = f32 ? launch_init<float>(kInter, info, blob, n_rows, d_out, st)
          : launch_init<double>(kInter, info, blob, n_rows, d_out, st);
  if (s != GTS_OK) return s;
  if (info->layout == GTS_LAYOUT_NODAL)
    return f32 ? launch_nodal_s<float, kInter>(info, blob, d_X, n_rows, rs, cs, d_out, st)
               : launch_nodal_s<double, kInter>(info, blob, d_X, n_rows, rs, cs, d_out, st);
  return f32 ? launch_bins<float, kInter>(info, blob, d_X, n_rows, rs, cs, d_out, st)
             : launch_bins<double, kInter>(info, blob, d_X, n_rows, rs, cs, d_out, st);
}

// SHAP and interaction values in one pass (NODAL): the interaction kernel's
// diagonal cells hold each tile's sum of phi_i before Eq. 6 is applied, so the
// flush adds them to phi as well; no SHAP kernel runs.  WARP_BINS blobs run
// their two kernels back to back.
gts_status run_fused(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows, int64_t rs,
                     int64_t cs, void* d_phi, void* d_phi_ij, void* stream) {
  gts_status s = check_call(info, d_blob, d_X, n_rows, rs, cs, d_phi_ij);
  if (s != GTS_OK || n_rows == 0) return s;
  s = check_call(info, d_blob, d_X, n_rows, rs, cs, d_phi);
  if (s != GTS_OK) return s;
  s = check_nodal(info, true);
  if (s != GTS_OK) return s;
  if (info->layout != GTS_LAYOUT_NODAL) {
    s = run<true>(info, d_blob, d_X, n_rows, rs, cs, d_phi_ij, stream);
    return s != GTS_OK ? s : run<false>(info, d_blob, d_X, n_rows, rs, cs, d_phi, stream);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* blob = static_cast<const char*>(d_blob);
  const bool f32 = info->dtype == GTS_F32;
  s = f32 ? launch_init<float>(true, info, blob, n_rows, d_phi_ij, st)
          : launch_init<double>(true, info, blob, n_rows, d_phi_ij, st);
  if (s != GTS_OK) return s;
  s = f32 ? launch_init<float>(false, info, blob, n_rows, d_phi, st)
          : launch_init<double>(false, info, blob, n_rows, d_phi, st);
  if (s != GTS_OK) return s;
  return f32 ? launch_nodal_s<float, true>(info, blob, d_X, n_rows, rs, cs, d_phi_ij, st, d_phi)
             : launch_nodal_s<double, true>(info, blob, d_X, n_rows, rs, cs, d_phi_ij, st, d_phi);
}

}  // namespace
#endif  // GTS_PART == 0
}  // namespace gts

#if GTS_PART == 0
extern "C" {

gts_status gts_shap(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows, int64_t ld_x,
                    void* d_phi, void* stream) {
  GTS_NVTX("gts_shap");
  return gts::run<false>(info, d_blob, d_X, n_rows, ld_x, 1, d_phi, stream);
}

gts_status gts_shap_interactions(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows,
                                 int64_t ld_x, void* d_phi_ij, void* stream) {
  GTS_NVTX("gts_shap_interactions");
  return gts::run<true>(info, d_blob, d_X, n_rows, ld_x, 1, d_phi_ij, stream);
}

gts_status gts_shap_strided(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows,
                            int64_t row_stride, int64_t col_stride, void* d_phi, void* stream) {
  GTS_NVTX("gts_shap_strided");
  return gts::run<false>(info, d_blob, d_X, n_rows, row_stride, col_stride, d_phi, stream);
}

gts_status gts_shap_interactions_strided(const gts_blob_info* info, const void* d_blob, const void* d_X,
                                         int64_t n_rows, int64_t row_stride, int64_t col_stride, void* d_phi_ij,
                                         void* stream) {
  GTS_NVTX("gts_shap_interactions_strided");
  return gts::run<true>(info, d_blob, d_X, n_rows, row_stride, col_stride, d_phi_ij, stream);
}

gts_status gts_shap_and_interactions(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows,
                                     int64_t row_stride, int64_t col_stride, void* d_phi, void* d_phi_ij,
                                     void* stream) {
  GTS_NVTX("gts_shap_and_interactions");
  return gts::run_fused(info, d_blob, d_X, n_rows, row_stride, col_stride, d_phi, d_phi_ij, stream);
}

gts_status gts_validate_x(gts_dtype dtype, const void* d_X, int64_t n_rows, int32_t n_features, int64_t row_stride,
                          int64_t col_stride, void* stream) {
  GTS_NVTX("gts_validate_x");
  if (dtype != GTS_F32 && dtype != GTS_F64) return gts::fail(GTS_ERR_INVALID_ARGUMENT, "bad dtype");
  if (n_rows < 0 || n_features < 1) return gts::fail(GTS_ERR_INVALID_ARGUMENT, "bad sizes");
  if (n_rows == 0) return GTS_OK;
  if (!d_X) return gts::fail(GTS_ERR_INVALID_ARGUMENT, "NULL X");
  const bool row_major = col_stride == 1 && row_stride >= n_features;
  const bool feature_major = row_stride == 1 && col_stride >= n_rows;
  if (!row_major && !feature_major) return gts::fail(GTS_ERR_INVALID_ARGUMENT, "bad X strides");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* d_first = nullptr;
  if (cudaMallocAsync(&d_first, sizeof(unsigned long long), st) != cudaSuccess)
    return gts::fail(GTS_ERR_CUDA, "cudaMallocAsync failed");
  cudaMemsetAsync(d_first, 0xff, sizeof(unsigned long long), st);
  const int64_t total = n_rows * n_features;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)gts::num_sms() * 8);
  if (dtype == GTS_F32)
    gts::nonfinite_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(d_X), n_rows, n_features,
                                                         row_stride, col_stride, d_first);
  else
    gts::nonfinite_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(d_X), n_rows, n_features,
                                                          row_stride, col_stride, d_first);
  unsigned long long first = ~0ull;
  cudaMemcpyAsync(&first, d_first, sizeof(first), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_first, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return gts::fail(GTS_ERR_CUDA, "gts_validate_x: %s", cudaGetErrorString(e));
  if (first != ~0ull)
    return gts::fail(GTS_ERR_NONFINITE, "X[%llu][%llu] is not finite (reading G17: X must be finite)",
                     first / (unsigned long long)n_features, first % (unsigned long long)n_features);
  return GTS_OK;
}

int32_t gts_launches_per_call(const gts_blob_info* info, int32_t interactions) {
  if (!info) return 0;
  const int32_t main = info->n_units > 0 ? 1 : 0;
  const int32_t mirror = gts::uses_mirror(info) ? 1 : 0;
  if (interactions == 2)  // gts_shap_and_interactions
    return info->layout == GTS_LAYOUT_NODAL ? 2 + main + mirror : 2 + 2 * main;
  // SHAP kernels that read X from global memory transpose a row-major X first
  const int32_t xt = (!interactions && info->layout == GTS_LAYOUT_NODAL && main &&
                      info->max_slots >= GTS_XG_MIN_S) ? 1 : 0;
  return 1 + main + (interactions ? mirror : xt);  // init + main kernel (+ mirror pass / X transpose)
}

}  // extern "C"
#endif  // GTS_PART == 0
