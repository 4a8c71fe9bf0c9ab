// blob_format.h -- device layout of the packed path tables.
//
// One contiguous byte blob per (model, dtype, layout), written on the host by
// gts_blob_write (host.cpp) and read by the kernels (kernels.cu).  Offsets are
// bytes from the blob start; every section is 256-byte aligned.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define GTS_HD __host__ __device__
#else
#define GTS_HD
#endif

namespace gts {

constexpr uint32_t kMagic = 0x47545342u;  // 'GTSB'
constexpr int kWarp = 32;                 // bin capacity B = warp size
constexpr int kQMax = 16;                 // Gauss nodes for merged k <= 31 (k = 2Q max)
constexpr int kMaxChunkPaths = 256;
constexpr int kChunkTableBytes = 16 * 1024;  // staged nodal tables per chunk (T words * sizeof(T))

struct BlobHeader {            // 256 bytes at offset 0
  uint32_t magic, version;
  int32_t dtype, layout;
  int32_t n_features, n_groups, max_slots, max_len;
  int64_t n_paths, n_elems, n_units, bytes;
  int64_t off_bias;            // double[G]
  int64_t off_gauss;           // NODAL: T[kQMax][3][kQMax]  (t_q, w_q, gamma_q = -1/(1-t_q)) for Q = 1..16
  int64_t off_units;           // NODAL: ChunkRec[n_units]; WARP_BINS: int32 kmax[n_units]
  int64_t off_work;            // NODAL: double[2][n_units+1] prefix work (shap, interactions)
  int64_t off_slotmap;         // NODAL: int32 slot -> feature
  int64_t off_paths;           // NODAL: PathRec[n_kept_paths]
  int64_t off_elems;           // NODAL: ElemRec[n_kept_elems]; WARP_BINS: lane arrays
  int64_t n_kept_paths;        // NODAL: paths with k >= 1 (k = 0 paths only feed the bias)
  int64_t n_kept_elems;        // NODAL: non-root elements of the kept paths
  int64_t max_chunk_words;     // NODAL: largest staged table (T words) of any chunk
  int64_t max_chunk_elems;     // NODAL: largest element count of any chunk
  int64_t max_chunk_paths;
  int64_t reserved[12];
};
static_assert(sizeof(BlobHeader) == 256, "header size");

// NODAL: a chunk = consecutive paths of one group that touch at most max_slots
// distinct features; a warp walks all of a chunk's paths for its 32 rows.
struct ChunkRec {              // 64 bytes
  int32_t group;
  int32_t n_paths;
  int32_t n_slots;             // features used by the chunk's slot map
  int32_t map_id;              // equal ids <=> identical slot maps
  int64_t path_begin;          // index into PathRec[]
  int64_t elem_begin;          // index into ElemRec[]
  int64_t slotmap_begin;       // index into the int32 slot map
  int32_t n_elems;
  int32_t table_words;         // staged nodal tables (T words)
  int32_t max_q;
  int32_t pad0;
  int64_t pad1;
};
static_assert(sizeof(ChunkRec) == 64, "chunk size");

struct PathRec {               // 24 bytes
  int32_t k;                   // non-root merged elements (1..31) | run length << 16 (run heads only):
                               // a run = consecutive paths of a chunk with one feature set
  int32_t q;                   // Gauss nodes: ceil(k/2)
  int32_t elem;                // first element, relative to the chunk's elem_begin
  int32_t table;               // first word of the path's staged table inside the chunk
  double v;                    // leaf value
};
static_assert(sizeof(PathRec) == 24, "path size");

struct ElemRec {               // 24 bytes
  int32_t slot;                // feature slot within the chunk's slot map
  float lo, hi;                // lo <= x < hi  <=> o = 1
  int32_t pad;
  double z;                    // merged zero fraction
};
static_assert(sizeof(ElemRec) == 24, "elem size");

// Staged nodal table of one path (T words, shared memory); every row is padded
// to QP = round_up(Q, 4) words so it loads with 16-byte vector loads.  SHAP kernel:
//   c[QP]            prod_s A_sq            (A = z + (1-z) t_q)
//   d[QP]            -v w_q / (1 - t_q)     (phi of every o = 0 element)
//   per element s:   rho[QP] = B_sq / A_sq  (B = z (1 - t_q)),  C[QP] = v w_q (1 - z_s) / A_sq
// Interaction kernel:
//   c[QP], h[QP] = v w_q / 2, per element: rho[QP], alpha[QP] = (1 - z_s) / A_sq
GTS_HD inline int nodal_path_words(int k, int q) { return 2 * ((q + 3) & ~3) * (k + 1); }

// WARP_BINS lane arrays (each [n_bins * 32], in this order after off_elems):
//   int32 feature   (-1 root lane, -2 empty lane)
//   int32 meta      rank | (k << 8) | (base_lane << 16)   (rank 0 = root, k = non-root count)
//   int32 group
//   float lo, float hi
//   T z, T v
}  // namespace gts
