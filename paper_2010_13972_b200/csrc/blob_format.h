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
constexpr int kChunkBytes = 16 * 1024;    // NODAL: staged bytes per chunk (one TMA bulk copy)
#ifndef GTS_CHUNK_BYTES_WIDE
#define GTS_CHUNK_BYTES_WIDE (8 * 1024)  // SHAP-only blobs with identity maps of > 16 features: 8 KB staging
                                         // lets three 4-warp blocks share an SM (covtype)
#endif

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
  int64_t off_paths;           // NODAL: start of the staged chunk regions (= off_elems)
  int64_t off_elems;           // NODAL: staged chunk regions; WARP_BINS: lane arrays
  int64_t n_kept_paths;        // NODAL: paths with k >= 1 (k = 0 paths only feed the bias)
  int64_t n_kept_elems;        // NODAL: non-root elements of the kept paths
  int64_t max_chunk_bytes;     // NODAL: largest staged region of any chunk
  int64_t max_chunk_elems;     // NODAL: largest element count of any chunk
  int64_t max_chunk_paths;
  int32_t uses;                // gts_blob_use bits (NODAL: which kernels the tables serve)
  int32_t n_tables;            // NODAL: table rows per record (2: SHAP only; 3: interactions)
  int32_t max_chunk_slots;     // NODAL: widest slot map of any chunk
  int32_t chunk_bytes;         // NODAL: staged-bytes budget per chunk
  int64_t reserved[10];
};
static_assert(sizeof(BlobHeader) == 256, "header size");

// NODAL: a chunk = consecutive paths of one group that touch at most max_slots
// distinct features; a warp walks all of a chunk's paths for its rows.  Its
// staged region (copied to shared memory with one TMA bulk copy) is
//   int4 elem[n_elems]  {lower bits, upper bits, slot, w}: NT = 3 (interaction
//                       tables): slot index, tri-row base of the slot; NT = 2
//                       (SHAP only): slot byte offset (slot * sizeof(T)), feature
//   int4 path[n_paths]  {k | run length << 16, Q, first elem, first table word}
//   T    table[table_words]   (per path, see below)
struct ChunkRec {              // 64 bytes
  int32_t group;
  int32_t n_paths;
  int32_t n_slots;             // features used by the chunk's slot map
  int32_t map_id;              // equal ids <=> identical slot maps
  int64_t path_begin;          // global index of the chunk's first path (bookkeeping)
  int64_t elem_begin;          // global index of the chunk's first element (bookkeeping)
  int64_t slotmap_begin;       // index into the int32 slot map
  int32_t n_elems;
  int32_t table_words;         // T words of tables
  int32_t max_q;
  int32_t data_bytes;          // staged region size (multiple of 16)
  int64_t data_off;            // staged region offset in the blob (16-byte aligned)
};
static_assert(sizeof(ChunkRec) == 64, "chunk size");

// host-side planning record (not stored in the blob)
struct PathRec {
  int32_t k;                   // non-root merged elements (1..31) | run length << 16 (run heads only):
                               // a run = consecutive paths of a chunk with one feature set
  int32_t q;                   // Gauss nodes: ceil(k/2)
  int32_t elem;                // first element, relative to the chunk
  int32_t table;               // first word of the path's table, relative to the chunk's tables
  int64_t src;                 // index of the path in the canonical table (gts_paths)
};

// Nodal table of one path (T words, shared memory; NT rows per record, the
// third row only when NT = 3; interaction blobs always have NT = 3, SHAP-only
// blobs NT = nodal_tables(S)).  Rows are padded to QP = round_up(Q, 4) words
// (16-byte vector loads).  Every path carries its own split bounds (as T), so
// EXTEND needs no element record (those are stored for run heads only): when
// Q mod 4 is 1 or 2 (nodal_inrow) the rho row has room for them after its
// zero-padded node pairs -- RW = nodal_rw(Q) words, lower / upper at BO =
// nodal_bo(Q) -- so they cost no load at all; otherwise (the rows are full)
// they form a block {lower_s, upper_s} x 2Q after the path rows (one 16-byte
// load per two elements in fp32).  With A_sq = z_s + (1-z_s) t_q,
// B_sq = z_s (1 - t_q) (f_s(t_q) for o_s = 1 / 0):
//   c[QP]  prod_s A_sq                  (P(t_q) when every o = 1)
//   d[QP]  -v w_q / (1 - t_q)           (SHAP: phi of every o = 0 element, times P_q)
//   h[QP]  v w_q / 2                    (interactions: W_q = h_q P_q)
//   [bounds block, nodal_bw(Q) words: lower_s, upper_s for s < k]
//   per element s (stride nodal_es(Q, NT) words):
//     rho[RW]   = B_sq / A_sq [, then lower_s, upper_s at BO]  (EXTEND of an o = 0 element; o_s)
//     C'[QP]    = v w_q ((1 - z_s)/A_sq + 1/(1 - t_q))   (SHAP: C_sq - d_q, where
//               C_sq = v w_q (1-z_s)/A_sq gives phi_s = sum_q P_q C_sq when o_s = 1)
//     alpha[QP] = (1 - z_s) / A_sq      (interactions: u_sq when o_s = 1)
GTS_HD constexpr int nodal_qp(int q) { return (q + 3) & ~3; }
// Algorithmic FP operations of one (row, path) with k non-root elements and
// Q = ceil(k/2) nodes (also the split-balancing work).
GTS_HD constexpr double nodal_shap_flops(int k, int q) { return 3.0 * k * q + 3.0 * k + 2.0 * q; }
GTS_HD constexpr double nodal_inter_flops(int k, int q) {
  // EXTEND kQ, W Q, y kQ, phi_i kQ + k, pairs k(k-1)/2 * 2Q, cell adds k(k-1)/2 + k, compares 2k
  return (double)k * (k - 1) * q + 3.0 * k * q + q + 4.0 * k + 0.5 * k * (k - 1);
}
// Blobs with more than 16 slots serve only the SHAP kernel (the interaction
// kernel takes 8 or 16 slots), so they drop h and alpha: NT = 2 tables per
// row ({c, d} and {rho, C'} per element) instead of 3 -- 1.5x more paths per
// 16 KB chunk, hence fewer slot-map gathers and flushes for wide models.
GTS_HD constexpr int nodal_tables(int slots) { return slots > 16 ? 2 : 3; }
GTS_HD constexpr bool nodal_inrow(int q) { return (q & 3) == 1 || (q & 3) == 2; }  // bounds in the rho row's padding
GTS_HD constexpr int nodal_bo(int q) { return (q + 1) & ~1; }  // in-row: bounds offset in the rho row
GTS_HD constexpr int nodal_rw(int q) { return nodal_inrow(q) ? (nodal_bo(q) + 2 + 3) & ~3 : nodal_qp(q); }  // rho row
GTS_HD constexpr int nodal_bw(int q) { return nodal_inrow(q) ? 0 : 4 * q; }  // bounds block: {lo, hi} x (k <= 2Q)
GTS_HD constexpr int nodal_es(int q, int nt = 3) { return nodal_rw(q) + (nt - 1) * nodal_qp(q); }  // element stride
GTS_HD constexpr int nodal_path_words(int k, int q, int nt = 3) {
  return nt * nodal_qp(q) + nodal_bw(q) + k * nodal_es(q, nt);
}

// WARP_BINS lane arrays (each [n_bins * 32], in this order after off_elems):
//   int32 feature   (-1 root lane, -2 empty lane)
//   int32 meta      rank | (k << 8) | (base_lane << 16)   (rank 0 = root, k = non-root count)
//   int32 group
//   float lo, float hi
//   T z, T v
}  // namespace gts
