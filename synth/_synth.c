/*
 * synth/_synth.c -- seeded synthetic INPUT generators shared by the oracle, the
 * tests and bench.py.  This file holds none of the method's arithmetic: it only
 * grows random-split tree ensembles (the {v,a,b,t,r,d} node lists of
 * PAPER.md:114, Algorithm 1 context) and draws feature matrices X.
 *
 * Recipe (after SURVEY.md §8(d)):
 *   - every tree has its own counter-keyed RNG stream (seed, tree), so trees can
 *     be grown in parallel and any subset regenerated bit-identically;
 *   - root cover 2^20, feasible box [0,1)^M;
 *   - repeatedly pick an expandable leaf (depth < D, cover >= 2) with
 *     probability proportional to exp(beta * depth);
 *   - its split feature is Zipf(s) over a per-tree random permutation of the M
 *     features (repeats along a path allowed -> exercises the merge);
 *   - threshold t = fp32 value strictly inside the node's feasible interval on
 *     that feature (x < t -> left, half-open bounds);
 *   - integer covers: c_left = clamp(round(r*C), 1, C-1), r ~ U(0.1, 0.9); or,
 *     with cover_skew = s in (0, 1), r log-uniform on [s, 1] and mirrored to
 *     1 - r with probability 1/2, so per-edge cover ratios (zero fractions)
 *     reach s and 1 - s (the skewed splits of real GBDT models);
 *   - stop at the tree's leaf target or when nothing is expandable;
 *   - leaf values fp32(N(0,1) * 0.01) (lr 0.01 scale).
 *   X[r][c] = U[0,1) fp32 from a counter-based hash of (seed, r, c): any row
 *   shard is reproducible without a scatter.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

typedef struct { uint64_t s[4]; } rng_t;

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t rng_next(rng_t* r) { /* xoshiro256** */
  uint64_t* s = r->s;
  const uint64_t result = rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
  s[2] ^= t; s[3] = rotl(s[3], 45);
  return result;
}

static void rng_seed(rng_t* r, uint64_t seed, uint64_t stream) {
  uint64_t x = splitmix64(seed) ^ splitmix64(stream * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL);
  for (int i = 0; i < 4; ++i) { x = splitmix64(x); r->s[i] = x; }
}

/* uniform double in [0,1) with 53 random bits */
static inline double rng_u01(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_normal(rng_t* r) {
  double u1 = rng_u01(r), u2 = rng_u01(r);
  if (u1 < 1e-300) u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

typedef struct {
  int32_t n_features, max_depth, leaves_floor;
  double leaves_frac;   /* P(tree target = floor+1) */
  double zipf_s, beta;
  double root_cover;
  uint64_t seed;
  double cover_skew;    /* 0: r ~ U(0.1, 0.9); else log-uniform on [cover_skew, 1], mirrored */
} synth_params;

/*
 * Grow tree `tree` into caller arrays sized for max_nodes nodes.
 * Returns the node count (>= 1), or -1 if max_nodes is too small.
 */
static int64_t grow_tree(const synth_params* p, int64_t tree, int64_t max_nodes,
                         int32_t* left, int32_t* right, int32_t* feature, float* threshold,
                         double* cover, double* leaf_value, int32_t* depth, int32_t* parent,
                         int32_t* bucket_store, const double* zipf_cdf, int32_t* perm) {
  rng_t rng;
  rng_seed(&rng, p->seed, (uint64_t)tree);
  const int M = p->n_features, D = p->max_depth;
  for (int i = 0; i < M; ++i) perm[i] = i;
  for (int i = M - 1; i > 0; --i) {
    int j = (int)(rng_next(&rng) % (uint64_t)(i + 1));
    int t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  int64_t target = p->leaves_floor + (rng_u01(&rng) < p->leaves_frac ? 1 : 0);
  if (target < 1) target = 1;
  if (2 * target - 1 > max_nodes) return -1;

  /* buckets of expandable leaves per depth: bucket d occupies
     bucket_store[d*max_nodes ...], with count cnt[d] */
  int64_t cnt[64];
  memset(cnt, 0, sizeof(cnt));
  int64_t n = 1;
  left[0] = right[0] = -1; feature[0] = -1; threshold[0] = 0.0f;
  cover[0] = p->root_cover; leaf_value[0] = 0.0; depth[0] = 0; parent[0] = -1;
  if (D > 0 && cover[0] >= 2.0) bucket_store[0 * max_nodes + cnt[0]++] = 0;
  int64_t leaves = 1;
  double wdepth[64];
  for (int d = 0; d < 64; ++d) wdepth[d] = exp(p->beta * d);

  while (leaves < target) {
    double tot = 0.0;
    for (int d = 0; d < D; ++d) tot += wdepth[d] * (double)cnt[d];
    if (tot <= 0.0) break;
    double u = rng_u01(&rng) * tot;
    int dsel = -1;
    for (int d = 0; d < D; ++d) {
      double w = wdepth[d] * (double)cnt[d];
      if (w <= 0.0) continue;
      dsel = d;
      if (u < w) break;
      u -= w;
    }
    int64_t idx = (int64_t)(rng_next(&rng) % (uint64_t)cnt[dsel]);
    int32_t node = bucket_store[dsel * max_nodes + idx];
    bucket_store[dsel * max_nodes + idx] = bucket_store[dsel * max_nodes + cnt[dsel] - 1];
    cnt[dsel]--;

    /* choose a feature with a non-degenerate feasible interval */
    int ok = 0;
    int f = -1;
    float thr = 0.0f;
    for (int attempt = 0; attempt < 32 && !ok; ++attempt) {
      double uz = rng_u01(&rng);
      int r = 0;
      while (r < M - 1 && uz >= zipf_cdf[r]) ++r;
      f = perm[r];
      /* feasible interval on f from the ancestors */
      float lo = 0.0f, hi = 1.0f;
      int32_t c = node;
      while (parent[c] >= 0) {
        int32_t pa = parent[c];
        if (feature[pa] == f) {
          if (left[pa] == c) { if (threshold[pa] < hi) hi = threshold[pa]; }
          else { if (threshold[pa] > lo) lo = threshold[pa]; }
        }
        c = pa;
      }
      for (int tries = 0; tries < 8; ++tries) {
        double uu = rng_u01(&rng);
        float t = (float)((double)lo + ((double)hi - (double)lo) * uu);
        if (t > lo && t < hi) { thr = t; ok = 1; break; }
      }
    }
    if (!ok) continue; /* node stays a leaf, no longer expandable */

    double C = cover[node];
    double rr;
    if (p->cover_skew > 0.0) {
      rr = exp(log(p->cover_skew) * rng_u01(&rng));
      if (rng_u01(&rng) < 0.5) rr = 1.0 - rr;
    } else {
      rr = 0.1 + 0.8 * rng_u01(&rng);
    }
    double cl = floor(rr * C + 0.5);
    if (cl < 1.0) cl = 1.0;
    if (cl > C - 1.0) cl = C - 1.0;
    double cr = C - cl;

    int32_t a = (int32_t)n, b = (int32_t)(n + 1);
    n += 2;
    feature[node] = f; threshold[node] = thr; left[node] = a; right[node] = b;
    int32_t kids[2] = {a, b};
    double kc[2] = {cl, cr};
    for (int q = 0; q < 2; ++q) {
      int32_t k = kids[q];
      left[k] = right[k] = -1; feature[k] = -1; threshold[k] = 0.0f;
      cover[k] = kc[q]; leaf_value[k] = 0.0; depth[k] = depth[node] + 1; parent[k] = node;
      if (depth[k] < D && cover[k] >= 2.0) bucket_store[depth[k] * max_nodes + cnt[depth[k]]++] = k;
    }
    leaves += 1;
  }
  for (int64_t i = 0; i < n; ++i)
    if (left[i] < 0) leaf_value[i] = (double)(float)(rng_normal(&rng) * 0.01);
  return n;
}

/*
 * Grow T trees.  Arrays are [T * max_nodes] (tree t at offset t*max_nodes);
 * n_nodes[t] receives each tree's node count.  Returns 0, or -1 on overflow.
 */
int synth_grow_ensemble(int64_t n_trees, int32_t n_features, int32_t max_depth,
                        int32_t leaves_floor, double leaves_frac, double zipf_s, double beta,
                        double root_cover, uint64_t seed, double cover_skew, int64_t max_nodes,
                        int32_t* left, int32_t* right, int32_t* feature, float* threshold,
                        double* cover, double* leaf_value, int64_t* n_nodes) {
  synth_params p = {n_features, max_depth, leaves_floor, leaves_frac, zipf_s, beta, root_cover, seed, cover_skew};
  if (max_depth >= 63) return -1;
  double* zipf_cdf = (double*)malloc(sizeof(double) * (size_t)n_features);
  double tot = 0.0;
  for (int r = 0; r < n_features; ++r) tot += 1.0 / pow((double)(r + 1), zipf_s);
  double acc = 0.0;
  for (int r = 0; r < n_features; ++r) { acc += 1.0 / pow((double)(r + 1), zipf_s) / tot; zipf_cdf[r] = acc; }
  int err = 0;
#pragma omp parallel
  {
    int32_t* depth = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_nodes);
    int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_nodes);
    int32_t* buckets = (int32_t*)malloc(sizeof(int32_t) * (size_t)max_nodes * (size_t)(max_depth + 1));
    int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n_features);
#pragma omp for schedule(dynamic, 4)
    for (int64_t t = 0; t < n_trees; ++t) {
      int64_t o = t * max_nodes;
      int64_t nn = grow_tree(&p, t, max_nodes, left + o, right + o, feature + o, threshold + o,
                             cover + o, leaf_value + o, depth, parent, buckets, zipf_cdf, perm);
      n_nodes[t] = nn;
      if (nn < 0) {
#pragma omp atomic write
        err = 1;
      }
    }
    free(depth); free(parent); free(buckets); free(perm);
  }
  free(zipf_cdf);
  return err ? -1 : 0;
}

/* X[r][c] for r in [row0, row0+n_rows), c in [0, n_cols): U[0,1) fp32 keyed on (seed, r, c). */
void synth_fill_x_f32(uint64_t seed, int64_t row0, int64_t n_rows, int32_t n_cols, float* out) {
  const uint64_t k = splitmix64(seed ^ 0xA0761D6478BD642FULL);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n_rows; ++r) {
    uint64_t rowkey = splitmix64(k ^ (uint64_t)(row0 + r) * 0xE7037ED1A0B428DBULL);
    for (int32_t c = 0; c < n_cols; ++c) {
      uint64_t h = splitmix64(rowkey + (uint64_t)c * 0x8EBC6AF09C88C6E3ULL);
      out[r * (int64_t)n_cols + c] = (float)(h >> 40) * 0x1.0p-24f;
    }
  }
}
