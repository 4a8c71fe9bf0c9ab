/*
 * oracle/treeshap.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU oracle for exact TreeShap.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  It shares no code with the product (paper_2010_13972_b200/):
 * it works on the RAW trees (no path extraction, no merging, no packing).
 *
 *   O5  oracle_treeshap      Algorithm 1 exactly as printed:
 *                            RECURSE / EXTEND / UNWIND / FINDFIRST, unwound sums
 *                            at the leaves, with readings
 *                            G1 (x < t -> left), G2 (root d = -1), G3 (UNWIND as
 *                            printed, both branches).  Bias = cover-weighted E[f]
 *                             + base_score, at column M (G13, G14).
 *   O6  oracle_interactions  conditioned recursion: for each
 *                            feature j split on in a tree, RECURSE with j fixed
 *                            present (cond=+1) and absent (cond=-1); j is never
 *                            EXTENDed; phi_ij = (phi_i^on - phi_i^off)/2 for i != j
 *                            (the 1/2 of Eq. 3's 2(M-1)!, reading G15); diagonal
 *                            by Eq. 6; cell (M,M) = bias.
 *   O1  oracle_predict       plain traversal, x < t -> left.
 *
 * OpenMP parallel-for over rows, as the paper's CPU baseline.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t n_trees;
  const int64_t* node_offset;
  const int32_t* left;
  const int32_t* right;
  const int32_t* feature;
  const float* threshold;
  const double* cover;
  const double* leaf_value;
  const int32_t* tree_group;
  int32_t M, G;
  double base_score;
} model_t;

/* one element of the path list m: d, z, o, w */
typedef struct { int32_t d; double z, o, w; } elem_t;

/* EXTEND, in place on m[0..l-1] -> m[0..l] (0-based index i-1). */
static void extend(elem_t* m, int l, double pz, double po, int32_t pi) {
  m[l].d = pi; m[l].z = pz; m[l].o = po; m[l].w = (l == 0) ? 1.0 : 0.0;
  for (int i = l; i >= 1; --i) {           /* 1-based i = l..1 */
    m[i].w += po * m[i - 1].w * (double)i / (double)(l + 1);        /* m_{i+1}.w */
    m[i - 1].w = pz * m[i - 1].w * (double)(l + 1 - i) / (double)(l + 1); /* m_i.w */
  }
}

/* UNWIND: m has length l; removes 1-based element i.
   Writes the result (length l-1) to out. */
static void unwind(const elem_t* m, int l, int i, elem_t* out) {
  double n = m[l - 1].w;
  const double zi = m[i - 1].z, oi = m[i - 1].o;
  for (int j = 0; j < l - 1; ++j) out[j] = m[j];
  for (int j = l - 1; j >= 1; --j) {       /* 1-based j = l-1..1 */
    if (oi != 0.0) {
      double t = out[j - 1].w;
      out[j - 1].w = n * (double)l / ((double)j * oi);
      n = t - out[j - 1].w * zi * (double)(l - j) / (double)l;
    } else {
      out[j - 1].w = (out[j - 1].w * (double)l) / (zi * (double)(l - j));
    }
  }
  for (int j = i; j <= l - 1; ++j) {       /* shift (d,z,o) down */
    out[j - 1].d = m[j].d; out[j - 1].z = m[j].z; out[j - 1].o = m[j].o;
  }
}

typedef struct {
  const model_t* mod;
  int64_t base;          /* global index of local node 0 */
  const double* x;
  double* phi;           /* [M] accumulator for this row and group */
  elem_t* stack;         /* scratch: (max_depth+2) levels x (max_depth+2) elems */
  int stride;
  int32_t cond_feature;  /* -1: unconditioned */
  int cond;              /* +1 present, -1 absent, 0 none */
} rec_ctx;

/* RECURSE with optional conditioning. m is the
   parent's list of length l; this level works on its own copy. */
static void recurse(rec_ctx* c, int level, int32_t j, const elem_t* m_in, int l,
                    double pz, double po, int32_t pi, double cond_frac) {
  if (cond_frac == 0.0) return;
  const model_t* mod = c->mod;
  elem_t* m = c->stack + (size_t)level * c->stride;
  for (int q = 0; q < l; ++q) m[q] = m_in[q];
  if (c->cond == 0 || pi != c->cond_feature) { extend(m, l, pz, po, pi); ++l; }
  const int64_t g = c->base + j;
  if (mod->left[g] < 0) {
    const double v = mod->leaf_value[g];
    elem_t* tmp = c->stack + (size_t)(level + 1) * c->stride;
    for (int i = 2; i <= l; ++i) {
      unwind(m, l, i, tmp);
      double w = 0.0;
      for (int q = 0; q < l - 1; ++q) w += tmp[q].w;
      c->phi[m[i - 1].d] += w * (m[i - 1].o - m[i - 1].z) * v * cond_frac;
    }
    return;
  }
  const int32_t dj = mod->feature[g];
  const int32_t a = mod->left[g], b = mod->right[g];
  const int go_left = c->x[dj] < (double)mod->threshold[g];  /* reading G1 */
  const int32_t h = go_left ? a : b, cc = go_left ? b : a;
  double iz = 1.0, io = 1.0;
  int k = 0;                                  /* FINDFIRST, 1-based; 0 = nothing */
  for (int q = 0; q < l; ++q) if (m[q].d == dj) { k = q + 1; break; }
  const elem_t* mm = m;
  int ll = l;
  if (k != 0) {
    iz = m[k - 1].z; io = m[k - 1].o;
    elem_t* un = c->stack + (size_t)(level + 1) * c->stride;
    unwind(m, l, k, un);
    for (int q = 0; q < l - 1; ++q) m[q] = un[q];
    ll = l - 1;
  }
  const double rj = mod->cover[g];
  const double rh = mod->cover[c->base + h], rc = mod->cover[c->base + cc];
  double hot_cf = cond_frac, cold_cf = cond_frac;
  if (c->cond != 0 && dj == c->cond_feature) {
    if (c->cond > 0) cold_cf = 0.0;
    else { hot_cf *= rh / rj; cold_cf *= rc / rj; }
  }
  recurse(c, level + 1, h, mm, ll, iz * rh / rj, io, dj, hot_cf);
  recurse(c, level + 1, cc, mm, ll, iz * rc / rj, 0.0, dj, cold_cf);
}

static int tree_depth(const model_t* mod, int64_t t) {
  const int64_t base = mod->node_offset[t];
  const int64_t n = mod->node_offset[t + 1] - base;
  int32_t* st = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * n + 2));
  int32_t* dp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(2 * n + 2));
  int sp = 0, maxd = 0;
  st[sp] = 0; dp[sp] = 0; ++sp;
  while (sp > 0) {
    --sp;
    int32_t j = st[sp], d = dp[sp];
    if (d > maxd) maxd = d;
    if (mod->left[base + j] >= 0) {
      st[sp] = mod->left[base + j]; dp[sp] = d + 1; ++sp;
      st[sp] = mod->right[base + j]; dp[sp] = d + 1; ++sp;
    }
  }
  free(st); free(dp);
  return maxd;
}

/* cover-weighted expectation E[f] of one subtree (S = empty) */
static double expect(const model_t* mod, int64_t base, int32_t j) {
  const int64_t g = base + j;
  if (mod->left[g] < 0) return mod->leaf_value[g];
  const int32_t a = mod->left[g], b = mod->right[g];
  return (mod->cover[base + a] * expect(mod, base, a) + mod->cover[base + b] * expect(mod, base, b)) /
         mod->cover[g];
}

static int model_max_depth(const model_t* mod) {
  int d = 0;
  for (int64_t t = 0; t < mod->n_trees; ++t) { int q = tree_depth(mod, t); if (q > d) d = q; }
  return d;
}

static void bias_per_group(const model_t* mod, double* bias) {
  for (int g = 0; g < mod->G; ++g) bias[g] = mod->base_score;
  for (int64_t t = 0; t < mod->n_trees; ++t)
    bias[mod->tree_group[t]] += expect(mod, mod->node_offset[t], 0);
}

#define MODEL_ARGS                                                                               \
  int64_t n_trees, const int64_t *node_offset, const int32_t *left, const int32_t *right,       \
      const int32_t *feature, const float *threshold, const double *cover,                      \
      const double *leaf_value, const int32_t *tree_group, int32_t M, int32_t G, double base_score
#define MODEL_INIT                                                                               \
  model_t mod = {n_trees, node_offset, left, right, feature, threshold, cover, leaf_value,       \
                 tree_group, M, G, base_score}

/* phi: [n_rows][G][M+1], overwritten.  X: [n_rows][ld_x] fp64. */
int oracle_treeshap(MODEL_ARGS, const double* X, int64_t n_rows, int64_t ld_x, double* phi) {
  MODEL_INIT;
  const int D = model_max_depth(&mod);
  const int stride = D + 2;
  double* bias = (double*)malloc(sizeof(double) * (size_t)G);
  bias_per_group(&mod, bias);
#pragma omp parallel
  {
    elem_t* stack = (elem_t*)malloc(sizeof(elem_t) * (size_t)(stride * (D + 3)));
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < n_rows; ++r) {
      double* out = phi + (size_t)r * G * (M + 1);
      memset(out, 0, sizeof(double) * (size_t)G * (M + 1));
      for (int64_t t = 0; t < n_trees; ++t) {
        rec_ctx c = {&mod, node_offset[t], X + (size_t)r * ld_x,
                     out + (size_t)tree_group[t] * (M + 1), stack, stride, -1, 0};
        recurse(&c, 0, 0, NULL, 0, 1.0, 1.0, -1, 1.0);  /* RECURSE(root,[],1,1,-1): reading G2 */
      }
      for (int g = 0; g < G; ++g) out[(size_t)g * (M + 1) + M] = bias[g];
    }
    free(stack);
  }
  free(bias);
  return 0;
}

/* phi_ij: [n_rows][G][M+1][M+1], overwritten. */
int oracle_interactions(MODEL_ARGS, const double* X, int64_t n_rows, int64_t ld_x, double* phi_ij) {
  MODEL_INIT;
  const int D = model_max_depth(&mod);
  const int stride = D + 2;
  const int64_t M1 = M + 1;
  double* bias = (double*)malloc(sizeof(double) * (size_t)G);
  bias_per_group(&mod, bias);
  /* features split on per tree */
  unsigned char* used = (unsigned char*)calloc((size_t)n_trees * (size_t)M, 1);
  for (int64_t t = 0; t < n_trees; ++t)
    for (int64_t q = node_offset[t]; q < node_offset[t + 1]; ++q)
      if (left[q] >= 0) used[(size_t)t * M + feature[q]] = 1;
#pragma omp parallel
  {
    elem_t* stack = (elem_t*)malloc(sizeof(elem_t) * (size_t)(stride * (D + 3)));
    double* phi_plain = (double*)malloc(sizeof(double) * (size_t)M);
    double* on = (double*)malloc(sizeof(double) * (size_t)M);
    double* off = (double*)malloc(sizeof(double) * (size_t)M);
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < n_rows; ++r) {
      double* out = phi_ij + (size_t)r * G * M1 * M1;
      memset(out, 0, sizeof(double) * (size_t)G * M1 * M1);
      const double* x = X + (size_t)r * ld_x;
      for (int g = 0; g < G; ++g) {
        double* mat = out + (size_t)g * M1 * M1;
        memset(phi_plain, 0, sizeof(double) * (size_t)M);
        for (int64_t t = 0; t < n_trees; ++t) {
          if (tree_group[t] != g) continue;
          rec_ctx c = {&mod, node_offset[t], x, phi_plain, stack, stride, -1, 0};
          recurse(&c, 0, 0, NULL, 0, 1.0, 1.0, -1, 1.0);
          for (int32_t jf = 0; jf < M; ++jf) {
            if (!used[(size_t)t * M + jf]) continue;  /* nabla_ij = 0 */
            memset(on, 0, sizeof(double) * (size_t)M);
            memset(off, 0, sizeof(double) * (size_t)M);
            rec_ctx con = {&mod, node_offset[t], x, on, stack, stride, jf, +1};
            recurse(&con, 0, 0, NULL, 0, 1.0, 1.0, -1, 1.0);
            rec_ctx coff = {&mod, node_offset[t], x, off, stack, stride, jf, -1};
            recurse(&coff, 0, 0, NULL, 0, 1.0, 1.0, -1, 1.0);
            for (int32_t i = 0; i < M; ++i)
              if (i != jf) mat[(size_t)i * M1 + jf] += (on[i] - off[i]) / 2.0;
          }
        }
        for (int32_t i = 0; i < M; ++i) {   /* Eq. 6 */
          double s = 0.0;
          for (int32_t jf = 0; jf < M; ++jf) if (jf != i) s += mat[(size_t)i * M1 + jf];
          mat[(size_t)i * M1 + i] = phi_plain[i] - s;
        }
        mat[(size_t)M * M1 + M] = bias[g];
      }
    }
    free(stack); free(phi_plain); free(on); free(off);
  }
  free(used);
  free(bias);
  return 0;
}

/* out: [n_rows][G] = base_score + sum of leaf values reached (x < t -> left). */
int oracle_predict(MODEL_ARGS, const double* X, int64_t n_rows, int64_t ld_x, double* out) {
  MODEL_INIT;
  (void)mod;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n_rows; ++r) {
    const double* x = X + (size_t)r * ld_x;
    for (int g = 0; g < G; ++g) out[r * G + g] = base_score;
    for (int64_t t = 0; t < n_trees; ++t) {
      const int64_t base = node_offset[t];
      int32_t j = 0;
      while (left[base + j] >= 0) j = (x[feature[base + j]] < (double)threshold[base + j]) ? left[base + j] : right[base + j];
      out[r * G + tree_group[t]] += leaf_value[base + j];
    }
  }
  return 0;
}

/* bias[G] = base_score + sum over trees of E[f] (S = empty). */
int oracle_bias(MODEL_ARGS, double* bias) {
  MODEL_INIT;
  bias_per_group(&mod, bias);
  return 0;
}

/* number of OpenMP threads the oracle will use */
int oracle_num_threads(void) {
  int n = 1;
#pragma omp parallel
  {
#pragma omp single
    {
#ifdef _OPENMP
      extern int omp_get_num_threads(void);
      n = omp_get_num_threads();
#endif
    }
  }
  return n;
}

/* ---- primitives exported for the pins (tests/test_oracle_pins.py) ---- */

/* EXTEND a fresh list with (z[q], o[q], d=q) for q = 0..n-1 (the first call is
   the root seed); writes the n weights w[0..n-1]. */
int oracle_extend_chain(int n, const double* z, const double* o, double* w_out) {
  elem_t m[64];
  if (n < 0 || n > 63) return -1;
  for (int q = 0; q < n; ++q) extend(m, q, z[q], o[q], q);
  for (int q = 0; q < n; ++q) w_out[q] = m[q].w;
  return 0;
}

/* UNWIND element i (1-based) from the list built by oracle_extend_chain and
   write the n-1 remaining weights; returns 0. */
int oracle_unwind_after_chain(int n, const double* z, const double* o, int i, double* w_out) {
  elem_t m[64], u[64];
  if (n < 1 || n > 63 || i < 1 || i > n) return -1;
  for (int q = 0; q < n; ++q) extend(m, q, z[q], o[q], q);
  unwind(m, n, i, u);
  for (int q = 0; q < n - 1; ++q) w_out[q] = u[q].w;
  return 0;
}
