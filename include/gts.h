/*
 * gts.h -- C ABI of the B200-native GPUTreeShap hot path (arXiv 2010.13972).
 *
 * The four calls named by the method's four steps (§3):
 *
 *   (1) gts_extract_paths      extract one unique path per leaf and merge
 *                              repeated features      (§3.1-3.2)
 *   (2) gts_binpack            pack paths into 32-lane warps, FFD / BFD / NF /
 *                              none, with utilisation (§3.3)
 *   (3) gts_shap               SHAP values phi and bias phi_0 for every row
 *                              (Eq. 1-2, Algorithm 1-3)
 *   (4) gts_shap_interactions  SHAP interaction values (Eq. 3-6, §3.5;
 *                              PAPER.md:120-139, 377-381)
 *
 * plus the device-layout step between (2) and (3): gts_blob_plan /
 * gts_blob_write serialise the packed tables into one contiguous byte blob that
 * the caller copies to device memory it owns (and, multi-GPU, broadcasts).
 *
 * Conventions (all functions):
 *   - Every call returns gts_status; GTS_OK == 0.  On error a message is
 *     available from gts_last_error() (thread-local, valid until the next call
 *     on the same thread).  Argument errors are detected before any launch.
 *   - Ownership: the caller owns every array it passes (model arrays: host;
 *     X, blob, phi: device).  gts_paths and gts_bins are library-owned and must
 *     be released with their _free functions.  The library keeps no global
 *     state besides the thread-local error string.
 *   - Device calls are asynchronous on the caller's stream (a cudaStream_t
 *     passed as void*; NULL = legacy default stream) and write only the given
 *     output buffer.  Kernel launch failures map to GTS_ERR_CUDA.
 *   - Thread safety: calls with distinct output buffers may run concurrently
 *     from several host threads, streams or devices.
 *   - Determinism: path tables, packings and blobs are bit-exact and
 *     reproducible.  fp32/fp64 phi are accumulated with atomics across thread
 *     blocks, so they are reproducible up to summation order.
 */
#ifndef GTS_H_
#define GTS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GTS_ABI_VERSION 4  /* 4: split bounds in the nodal rho rows; 3: blob uses recorded in the info, 32-slot interaction blobs */
#define GTS_WARP_CAPACITY 32 /* lanes per warp = bin capacity B */

typedef enum gts_status {
  GTS_OK = 0,
  GTS_ERR_INVALID_ARGUMENT = 1, /* null pointer, negative size, bad enum, buffer too small */
  GTS_ERR_INVALID_MODEL = 2,    /* cycle / dangling or shared child, feature out of range,
                                   cover <= 0, cover(parent) != cover(l)+cover(r) beyond 1e-6
                                   relative, non-finite threshold / value, bad group */
  GTS_ERR_PATH_TOO_LONG = 3,    /* merged path length (root included) > 32 */
  GTS_ERR_NONFINITE = 4,        /* non-finite X found by gts_validate_x (reading G17) */
  GTS_ERR_CUDA = 5,             /* CUDA launch / runtime error */
  GTS_ERR_OUT_OF_MEMORY = 6     /* host allocation failed */
} gts_status;

/* Bin-packing heuristics (Table 1). */
typedef enum gts_pack_algo {
  GTS_PACK_FFD = 0,  /* first-fit decreasing */
  GTS_PACK_BFD = 1,  /* best-fit decreasing (the paper's recommendation) */
  GTS_PACK_NF = 2,   /* next-fit, arrival order */
  GTS_PACK_NONE = 3  /* one path per warp (the Table 5 "none" baseline) */
} gts_pack_algo;

/* Arithmetic type of X, phi and the kernels. */
typedef enum gts_dtype { GTS_F32 = 0, GTS_F64 = 1 } gts_dtype;

/* Device layout of the blob = which kernel family runs it. */
typedef enum gts_layout {
  /* Row-lane kernels (default, B200-native): lanes = rows, one warp walks a
     chunk of paths; the permutation-weight polynomial of each (row, path) is
     EXTENDed / UNWOUND in the nodal basis. */
  GTS_LAYOUT_NODAL = 0,
  /* Paper-lineage kernels: lanes = path elements of the packed bins, EXTEND
     via __shfl_up_sync and UNWOUNDSUM via __shfl_sync (Algorithms 2-3,
     readings G4/G5), swap-to-end conditioning for interactions (§3.5). */
  GTS_LAYOUT_WARP_BINS = 1
} gts_layout;

/*
 * Tree ensemble: the node lists {v, a, b, t, r, d} of PAPER.md:114 in CSR over
 * trees.  Caller-owned HOST arrays, read only during gts_extract_paths.
 */
typedef struct gts_model {
  int64_t n_trees;              /* T >= 0 */
  const int64_t* node_offset;   /* [T+1]; tree t owns nodes [node_offset[t], node_offset[t+1]);
                                   node_offset[0] == 0; each tree >= 1 node; local node 0 = root */
  const int32_t* left;          /* a_j: local index of the left child, -1 at leaves */
  const int32_t* right;         /* b_j: local index of the right child, -1 at leaves */
  const int32_t* feature;       /* d_j in [0, n_features) at internal nodes (ignored at leaves) */
  const float* threshold;       /* t_j: split rule x[d_j] < t_j -> left (reading G1) */
  const double* cover;          /* r_j > 0, training weight through node j */
  const double* leaf_value;     /* v_j at leaves (ignored at internal nodes) */
  const int32_t* tree_group;    /* [T] output group of each tree, in [0, n_groups) */
  int32_t n_features;           /* M >= 1 */
  int32_t n_groups;             /* G >= 1 (classes for multiclass, 1 for regression) */
  double base_score;            /* added to the bias phi_0 of every group */
} gts_model;

/* ---------------------------------------------------------------- (1) paths */

typedef struct gts_paths gts_paths; /* opaque, library-owned */

/* Read-only view of the canonical path-element table (Listing 1).
   Pointers stay valid until gts_paths_free. */
typedef struct gts_paths_view {
  int64_t n_paths;              /* L = number of leaves */
  int64_t n_elems;              /* E = sum of merged path lengths, root element included */
  int32_t n_features, n_groups;
  int32_t max_len;              /* longest merged path (root included) */
  const int64_t* path_offset;   /* [L+1] element range of each path */
  const int32_t* feature;       /* [E] -1 for the root element, then ascending features */
  const float* lower;           /* [E] bounds: an instance follows the path when */
  const float* upper;           /* [E]   lower <= x[feature] < upper (root: -inf, +inf) */
  const double* zero_fraction;  /* [E] z: product of cover ratios (root: 1) */
  const double* v;              /* [L] leaf value */
  const int32_t* group;         /* [L] output group */
  const int32_t* tree;          /* [L] source tree */
  const double* bias;           /* [G] phi_0 = sum_paths v * prod z + base_score */
} gts_paths_view;

/* Validate the model, extract one path per leaf (trees in input order, leaves in
   DFS left-first order) and merge repeated features (bounds intersect, zero
   fractions multiply in root-to-leaf order, fp64).  Errors: INVALID_ARGUMENT,
   INVALID_MODEL, PATH_TOO_LONG, OUT_OF_MEMORY.  *out is set only on success. */
gts_status gts_extract_paths(const gts_model* model, gts_paths** out);
gts_status gts_paths_view_get(const gts_paths* paths, gts_paths_view* view);
void gts_paths_free(gts_paths* paths);

/* ----------------------------------------------------------------- (2) bins */

typedef struct gts_bins gts_bins; /* opaque, library-owned; keeps its own reference to the paths */

typedef struct gts_bins_view {
  int64_t n_items;              /* = n_paths */
  int64_t n_bins;               /* K */
  int64_t sum_sizes;            /* sum of item sizes = n_elems */
  int32_t capacity;             /* B */
  int32_t algo;                 /* gts_pack_algo */
  double utilisation;           /* sum_sizes / (capacity * K), 1.0 when K == 0 */
  double pack_seconds;          /* wall time of the packing heuristic alone */
  const int32_t* bin_of_path;   /* [L] bin index, bins numbered by creation */
  const uint8_t* lane_of_path;  /* [L] first lane; a path occupies consecutive lanes */
} gts_bins_view;

/* Pack paths (item size = merged length incl. root) into bins of `capacity`
   lanes (1..32; 32 in production).  FFD/BFD: items in non-increasing size,
   ties by path index; FFD picks the lowest-index bin that fits, BFD the bin
   with the smallest sufficient residual (ties: lowest index).  Errors:
   INVALID_ARGUMENT (capacity, algo), PATH_TOO_LONG (an item > capacity). */
gts_status gts_binpack(const gts_paths* paths, int32_t capacity, gts_pack_algo algo, gts_bins** out);
gts_status gts_bins_view_get(const gts_bins* bins, gts_bins_view* view);
void gts_bins_free(gts_bins* bins);

/* ------------------------------------------------------------ device blob */

/* Host-side description of a blob; plain old data, safe to memcpy / broadcast.
   gts_shap needs it to configure the launch without reading device memory. */
typedef struct gts_blob_info {
  uint32_t magic;               /* 0x47545342 'GTSB' */
  uint32_t abi_version;         /* GTS_ABI_VERSION */
  int32_t dtype;                /* gts_dtype */
  int32_t layout;               /* gts_layout */
  int32_t n_features, n_groups;
  int32_t max_slots;            /* NODAL: feature slots per chunk (16, 32 or 64) */
  int32_t max_len;              /* longest merged path, root included */
  int64_t n_paths, n_elems;
  int64_t n_units;              /* NODAL: chunks; WARP_BINS: bins */
  int64_t bytes;                /* total blob size */
  double shap_flops_per_row;    /* algorithmic flops per row */
  double inter_flops_per_row;
  double paper_shap_flops_per_row;   /* SURVEY.md §8(d) F_shap, for context */
  double paper_inter_flops_per_row;  /* SURVEY.md §8(d) F_int */
  int64_t max_chunk_bytes;      /* NODAL: staged bytes of the largest chunk (shared memory) */
  int64_t max_chunk_elems;
  int64_t max_chunk_paths;
  int32_t uses;                 /* gts_blob_use bits the blob serves (NODAL; WARP_BINS: both) */
  int32_t n_tables;             /* NODAL: nodal table rows per element record (2 or 3) */
  int32_t max_chunk_slots;      /* NODAL: widest slot map of any chunk (SHAP tile row = this + 1) */
  int32_t chunk_bytes;          /* NODAL: staged-bytes budget per chunk the plan used */
  int64_t reserved[3];
} gts_blob_info;

/* What a blob is planned for.  NODAL blobs carry per-path nodal tables
   (blob_format.h); the SHAP kernel needs {rho, C'} per element, the
   interaction kernel {rho, alpha} plus the per-path h row, and its shared
   memory tile holds S(S+1)/2 pair cells per row, so it takes S <= 32 slots. */
typedef enum gts_blob_use {
  GTS_USE_SHAP = 1,
  GTS_USE_INTERACTIONS = 2,
  GTS_USE_BOTH = 3
} gts_blob_use;

/* Describe the blob for (bins, dtype, layout).  max_slots (NODAL only) is the
   number of distinct features a chunk may touch, one of 8, 16, 32, 64, or 0
   for the default (the smallest of them >= n_features, raised to the longest
   merged path; above 64 features, 32 with per-chunk slot maps).  The blob
   serves gts_shap, and the interaction calls too when its slot width is <= 16
   (uses = GTS_USE_BOTH; otherwise GTS_USE_SHAP).  Errors: INVALID_ARGUMENT. */
gts_status gts_blob_plan(const gts_bins* bins, gts_dtype dtype, gts_layout layout, int32_t max_slots,
                         gts_blob_info* info);
/* Same, for an explicit use.  NODAL with GTS_USE_INTERACTIONS (or BOTH):
   max_slots one of 8, 16, 32 or 0 = default (8 when n_features <= 8, else 16,
   raised to 32 when a merged path has more than 16 features -- the paper's
   bound is 31); every such blob serves the interaction
   calls and gts_shap_and_interactions, and gts_shap too when uses is
   GTS_USE_BOTH, which needs a slot width <= 16 (the SHAP kernel reads
   2-row tables above 16 slots).  GTS_USE_SHAP is gts_blob_plan's SHAP
   layout.  WARP_BINS blobs serve every call (uses = BOTH whatever is asked).
   Errors: INVALID_ARGUMENT (bad use, slot width smaller than the longest
   merged path on a per-chunk slot map, interaction slot width > 32, BOTH
   above 16 slots). */
gts_status gts_blob_plan_for(const gts_bins* bins, gts_dtype dtype, gts_layout layout, int32_t max_slots,
                             gts_blob_use uses, gts_blob_info* info);
/* Serialise into caller HOST memory of at least info->bytes (any alignment
   >= 16).  The caller copies the bytes to a device buffer (16-byte aligned). */
gts_status gts_blob_write(const gts_bins* bins, const gts_blob_info* info, void* host_dst, size_t dst_bytes);
/* Bytes [offset, offset + bytes) of the same blob into caller HOST memory
   (host_dst receives exactly `bytes` bytes), so a large blob can be streamed
   host -> device through small pinned buffers while the next range is being
   written.  Writing every range once gives the bytes
   of gts_blob_write.  The plan of the preceding gts_blob_plan* call is kept
   between ranges (gts_blob_write frees it).  Errors: INVALID_ARGUMENT (range
   outside [0, info->bytes), info not of these bins). */
gts_status gts_blob_write_range(const gts_bins* bins, const gts_blob_info* info, int64_t offset, int64_t bytes,
                                void* host_dst);

/* ---------------------------------------------------------- (3)/(4) compute */

/* SHAP values for rows [0, n_rows) of X.
   d_blob:  device copy of the blob described by info.
   d_X:     device, row-major [n_rows][ld_x] of info->dtype, ld_x >= n_features;
            values finite (reading G17).
   d_phi:   device [n_rows][n_groups][n_features+1] of info->dtype, fully
            overwritten; column n_features holds the bias phi_0 (reading G14).
   stream:  cudaStream_t (NULL = default stream).  n_rows == 0 is a no-op.
   Temporary device memory: for NODAL blobs of 32 or 64 slots the kernel
   reads X feature-major, so X is first copied (transposed if row-major) into
   a stream-ordered allocation of about n_rows * n_features elements, padded
   to whole row tiles (cudaMallocAsync, freed after the kernel on the same
   stream; OUT_OF_MEMORY if it fails).                                      */
gts_status gts_shap(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows,
                    int64_t ld_x, void* d_phi, void* stream);

/* SHAP interaction values; d_phi_ij: device
   [n_rows][n_groups][n_features+1][n_features+1] of info->dtype, fully
   overwritten: off-diagonal Eq. 3, diagonal Eq. 6, cell (M,M) = bias,
   cells (i,M) and (M,i) = 0.  NODAL blobs need uses & GTS_USE_INTERACTIONS
   (checked before any launch; gts_shap likewise needs GTS_USE_SHAP). */
gts_status gts_shap_interactions(const gts_blob_info* info, const void* d_blob, const void* d_X,
                                 int64_t n_rows, int64_t ld_x, void* d_phi_ij, void* stream);

/* Same two calls for X in either layout: element (r, f) at
   d_X[r * row_stride + f * col_stride], with row-major (col_stride == 1,
   row_stride >= n_features) or feature-major (row_stride == 1,
   col_stride >= n_rows).  Feature-major X makes the per-chunk gathers of wide
   models (many features per row) coalesced.  gts_shap(..., ld_x, ...) is
   gts_shap_strided(..., ld_x, 1, ...). */
gts_status gts_shap_strided(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows,
                            int64_t row_stride, int64_t col_stride, void* d_phi, void* stream);
gts_status gts_shap_interactions_strided(const gts_blob_info* info, const void* d_blob, const void* d_X,
                                         int64_t n_rows, int64_t row_stride, int64_t col_stride, void* d_phi_ij,
                                         void* stream);

/* SHAP values and SHAP interaction values of the same rows in one pass.
   Outputs are those of gts_shap_strided (d_phi) and
   gts_shap_interactions_strided (d_phi_ij), both fully overwritten; strides as
   above.  info must describe an interaction-capable blob (NODAL with
   max_slots <= 16, or WARP_BINS).  NODAL: phi is not computed by the SHAP
   kernel but read off the interaction pass: per path, the diagonal
   accumulator of the interaction kernel holds phi_i = v (o_i - z_i) U_i
   (Algorithm 1) before Eq. 6 turns it into
   phi_ii, so the tile flush adds it to phi too (one extra atomic per non-zero
   (row, group, feature) per flush).  WARP_BINS: the two kernels back to back.
   Errors as gts_shap_interactions; d_phi and d_phi_ij must not overlap. */
gts_status gts_shap_and_interactions(const gts_blob_info* info, const void* d_blob, const void* d_X, int64_t n_rows,
                                     int64_t row_stride, int64_t col_stride, void* d_phi, void* d_phi_ij,
                                     void* stream);

/* Optional validation of X (reading G17: the method is defined for finite
   inputs only; PAPER.md:50 covers absent features, not NaN).  Checks every
   entry (r, f), f < n_features, of a row- or feature-major X as above on
   `stream` and SYNCHRONISES the stream: GTS_ERR_NONFINITE (message names the
   first offending entry in row-major order) if any is NaN or +-inf, GTS_OK
   otherwise.  The compute calls never check (it costs a pass over X and a
   host sync); callers that cannot vouch for X call this first.  Errors:
   INVALID_ARGUMENT, CUDA, NONFINITE. */
gts_status gts_validate_x(gts_dtype dtype, const void* d_X, int64_t n_rows, int32_t n_features, int64_t row_stride,
                          int64_t col_stride, void* stream);

/* Number of kernel launches one call issues: interactions = 0 for gts_shap,
   1 for gts_shap_interactions, 2 for gts_shap_and_interactions.  NODAL blobs
   with per-chunk slot maps (n_features > max_slots) add one pass to the
   interaction calls: the kernel adds each pair to (i, j), i < j, only, and a
   tiled transpose copies it to (j, i) (phi_ij is symmetric, Eq. 3).  NODAL
   SHAP blobs of 32 or 64 slots add one X copy kernel to gts_shap (the kernel
   reads a padded feature-major copy of X). */
int32_t gts_launches_per_call(const gts_blob_info* info, int32_t interactions);

const char* gts_last_error(void);
const char* gts_status_string(gts_status status);
int32_t gts_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GTS_H_ */
