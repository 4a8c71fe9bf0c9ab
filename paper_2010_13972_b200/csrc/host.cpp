// host.cpp -- host side of the C ABI (include/gts.h): model validation, path
// extraction + duplicate merge, bin packing, bias, blob serialisation.
//
// SURVEY.md §8(a) rows a1 (ingest + validate), a2 (extract + merge), a3 (bin
// packing), a4 (device layout), a5 (bias).  Parallel over trees with OpenMP,
// deterministic: per-tree results are concatenated in tree order.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <new>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/gts.h"
#include "blob_format.h"
#include "trace.h"

namespace gts {

// ---------------------------------------------------------------- errors

static thread_local std::string g_last_error;

gts_status fail(gts_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

const char* last_error() { return g_last_error.c_str(); }

// ------------------------------------------------------------- path table

// Allocator whose resize() leaves new elements uninitialised: the big table
// arrays are filled by parallel loops (first touch spread over the threads)
// instead of being zeroed by one thread first.
template <class T>
struct NoInitAlloc : std::allocator<T> {
  template <class U>
  struct rebind { using other = NoInitAlloc<U>; };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  template <class U>
  void construct(U* p) noexcept { ::new (static_cast<void*>(p)) U; }
  template <class U, class... A>
  void construct(U* p, A&&... a) { ::new (static_cast<void*>(p)) U(std::forward<A>(a)...); }
};
template <class T>
using big_vector = std::vector<T, NoInitAlloc<T>>;

struct PathTable {
  int32_t n_features = 0, n_groups = 0, max_len = 0;
  double base_score = 0.0;
  big_vector<int64_t> path_offset;
  big_vector<int32_t> feature;
  big_vector<float> lower, upper;
  big_vector<double> zero_fraction;
  big_vector<double> v;
  big_vector<int32_t> group, tree;
  std::vector<double> bias;
  int64_t n_paths() const { return (int64_t)v.size(); }
  int64_t n_elems() const { return (int64_t)feature.size(); }
  int32_t len(int64_t p) const { return (int32_t)(path_offset[p + 1] - path_offset[p]); }
};

}  // namespace gts

struct gts_paths {
  std::shared_ptr<gts::PathTable> tab;
};

namespace gts {
struct PlanCache;
}

struct gts_bins {
  std::shared_ptr<gts::PathTable> tab;
  mutable std::mutex cache_mu;                   // guards cache
  mutable std::shared_ptr<gts::PlanCache> cache;  // last blob plan, taken by gts_blob_write
  int32_t capacity = 32;
  int32_t algo = 0;
  int64_t n_bins = 0;
  int64_t sum_sizes = 0;
  double pack_seconds = 0.0;
  std::vector<int32_t> bin_of_path;
  std::vector<uint8_t> lane_of_path;
};

namespace gts {

// ----------------------------------------------------------- validation (a1)

static gts_status validate_model(const gts_model* m) {
  if (!m) return fail(GTS_ERR_INVALID_ARGUMENT, "model is NULL");
  if (m->n_trees < 0) return fail(GTS_ERR_INVALID_ARGUMENT, "n_trees < 0");
  if (m->n_features < 1) return fail(GTS_ERR_INVALID_ARGUMENT, "n_features < 1");
  if (m->n_groups < 1) return fail(GTS_ERR_INVALID_ARGUMENT, "n_groups < 1");
  if (!std::isfinite(m->base_score)) return fail(GTS_ERR_INVALID_MODEL, "base_score not finite");
  if (m->n_trees == 0) return GTS_OK;
  if (!m->node_offset || !m->left || !m->right || !m->feature || !m->threshold || !m->cover ||
      !m->leaf_value || !m->tree_group)
    return fail(GTS_ERR_INVALID_ARGUMENT, "model array is NULL");
  if (m->node_offset[0] != 0) return fail(GTS_ERR_INVALID_MODEL, "node_offset[0] != 0");
  for (int64_t t = 0; t < m->n_trees; ++t) {
    if (m->node_offset[t + 1] <= m->node_offset[t])
      return fail(GTS_ERR_INVALID_MODEL, "tree %lld has no nodes", (long long)t);
    if (m->node_offset[t + 1] - m->node_offset[t] > (int64_t)INT32_MAX)
      return fail(GTS_ERR_INVALID_MODEL, "tree %lld too large", (long long)t);
    if (m->tree_group[t] < 0 || m->tree_group[t] >= m->n_groups)
      return fail(GTS_ERR_INVALID_MODEL, "tree %lld group %d out of range", (long long)t, m->tree_group[t]);
  }
  const int64_t T = m->n_trees;
  std::vector<int> err_code(T, 0);
  std::vector<std::string> err_msg(T);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t t = 0; t < T; ++t) {
    const int64_t base = m->node_offset[t];
    const int32_t n = (int32_t)(m->node_offset[t + 1] - base);
    std::vector<uint8_t> parents(n, 0);
    char buf[256];
    auto bad = [&](const char* what, int32_t j) {
      snprintf(buf, sizeof(buf), "tree %lld node %d: %s", (long long)t, j, what);
      err_code[t] = 1;
      err_msg[t] = buf;
    };
    for (int32_t j = 0; j < n && !err_code[t]; ++j) {
      const int64_t g = base + j;
      const double c = m->cover[g];
      if (!(c > 0.0) || !std::isfinite(c)) { bad("cover must be finite and > 0", j); break; }
      const int32_t a = m->left[g], b = m->right[g];
      if (a < 0 && b < 0) {
        if (!std::isfinite(m->leaf_value[g])) bad("leaf value not finite", j);
        continue;
      }
      if (a <= 0 || b <= 0 || a >= n || b >= n || a == b) { bad("dangling or invalid child index", j); break; }
      if (m->feature[g] < 0 || m->feature[g] >= m->n_features) { bad("feature out of range", j); break; }
      if (!std::isfinite(m->threshold[g])) { bad("threshold not finite", j); break; }
      if (++parents[a] > 1 || ++parents[b] > 1) { bad("node has more than one parent", j); break; }
      const double sum = m->cover[base + a] + m->cover[base + b];
      if (std::fabs(sum - c) > 1e-6 * c) { bad("cover(parent) != cover(left) + cover(right)", j); break; }
    }
    if (!err_code[t] && parents[0] != 0) bad("root has a parent (cycle)", 0);
    for (int32_t j = 1; j < n && !err_code[t]; ++j)
      if (parents[j] != 1) bad("node unreachable (no parent)", j);
    if (!err_code[t]) {  // exactly-one-parent + all reachable from the root => a tree
      std::vector<int32_t> st{0};
      int32_t seen = 0;
      while (!st.empty() && seen <= n) {
        int32_t j = st.back();
        st.pop_back();
        ++seen;
        if (m->left[base + j] >= 0) { st.push_back(m->left[base + j]); st.push_back(m->right[base + j]); }
      }
      if (seen != n) bad("cycle or unreachable nodes", 0);
    }
  }
  for (int64_t t = 0; t < T; ++t)
    if (err_code[t]) return fail(GTS_ERR_INVALID_MODEL, "%s", err_msg[t].c_str());
  return GTS_OK;
}

// ------------------------------------------------- extraction + merge (a2)

struct Edge {
  int32_t f;
  float lo, hi;
  double z;
};

// Stable insertion sort by feature (paths are short), then merge runs of equal
// features: lower = max, upper = min, z = product in root-to-leaf order
// (reading G11).  Returns the merged count.
static int merge_path(const Edge* raw, int n, Edge* out, Edge* scratch) {
  for (int i = 0; i < n; ++i) {
    Edge e = raw[i];
    int j = i;
    while (j > 0 && scratch[j - 1].f > e.f) { scratch[j] = scratch[j - 1]; --j; }
    scratch[j] = e;
  }
  int m = 0;
  for (int i = 0; i < n; ++i) {
    const Edge& e = scratch[i];
    if (m > 0 && out[m - 1].f == e.f) {
      Edge& p = out[m - 1];
      p.lo = std::max(p.lo, e.lo);
      p.hi = std::min(p.hi, e.hi);
      p.z = p.z * e.z;
    } else {
      out[m++] = e;
    }
  }
  return m;
}

struct TreeOut {
  std::vector<int32_t> len;  // merged length incl. root, per path
  std::vector<Edge> elems;   // non-root merged elements, path after path
  std::vector<double> v;
  int32_t max_len = 0;
};

// One path per leaf, DFS left-first (reading G9).  Edge of the left child:
// [-inf, t); right child: [t, +inf) (x < t -> left, reading G1); z = r_child / r_parent.
static void extract_tree(const gts_model* m, int64_t t, TreeOut& out) {
  const int64_t base = m->node_offset[t];
  struct Item { int32_t node, depth; Edge edge; };
  std::vector<Item> st;
  std::vector<Edge> edges, merged, scratch;
  st.push_back({0, 0, Edge{-1, 0.f, 0.f, 1.0}});
  while (!st.empty()) {
    Item it = st.back();
    st.pop_back();
    if (it.depth > 0) {
      edges.resize(it.depth - 1);
      edges.push_back(it.edge);
    }
    const int64_t g = base + it.node;
    const int32_t a = m->left[g], b = m->right[g];
    if (a < 0) {
      const int d = it.depth;
      merged.resize(d + 1);
      scratch.resize(d + 1);
      const int k = merge_path(edges.data(), d, merged.data(), scratch.data());
      out.len.push_back(k + 1);
      out.max_len = std::max(out.max_len, k + 1);
      out.elems.insert(out.elems.end(), merged.begin(), merged.begin() + k);
      out.v.push_back(m->leaf_value[g]);
      continue;
    }
    const float thr = m->threshold[g];
    const int32_t f = m->feature[g];
    const double rj = m->cover[g];
    const float inf = std::numeric_limits<float>::infinity();
    st.push_back({b, it.depth + 1, Edge{f, thr, inf, m->cover[base + b] / rj}});
    st.push_back({a, it.depth + 1, Edge{f, -inf, thr, m->cover[base + a] / rj}});
  }
}

static gts_status extract(const gts_model* m, std::shared_ptr<PathTable>& out) {
  gts_status st = validate_model(m);
  if (st != GTS_OK) return st;
  auto tab = std::make_shared<PathTable>();
  tab->n_features = m->n_features;
  tab->n_groups = m->n_groups;
  tab->base_score = m->base_score;
  const int64_t T = m->n_trees;
  std::vector<TreeOut> trees(T);
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t t = 0; t < T; ++t) extract_tree(m, t, trees[t]);
  int64_t L = 0, E = 0;
  std::vector<int64_t> path_base(T + 1, 0), elem_base(T + 1, 0);
  for (int64_t t = 0; t < T; ++t) {
    path_base[t + 1] = path_base[t] + (int64_t)trees[t].v.size();
    elem_base[t + 1] = elem_base[t] + (int64_t)trees[t].elems.size() + (int64_t)trees[t].v.size();
    tab->max_len = std::max(tab->max_len, trees[t].max_len);
  }
  L = path_base[T];
  E = elem_base[T];
  if (tab->max_len > kWarp)
    return fail(GTS_ERR_PATH_TOO_LONG, "merged path length %d exceeds the warp size %d (PAPER.md:215)",
                tab->max_len, kWarp);
  tab->path_offset.resize(L + 1);
  tab->feature.resize(E);
  tab->lower.resize(E);
  tab->upper.resize(E);
  tab->zero_fraction.resize(E);
  tab->v.resize(L);
  tab->group.resize(L);
  tab->tree.resize(L);
  const float inf = std::numeric_limits<float>::infinity();
#pragma omp parallel for schedule(dynamic, 8)
  for (int64_t t = 0; t < T; ++t) {
    const TreeOut& tr = trees[t];
    int64_t p = path_base[t], e = elem_base[t];
    size_t src = 0;
    for (size_t q = 0; q < tr.v.size(); ++q, ++p) {
      tab->path_offset[p] = e;
      tab->feature[e] = -1;  // root element (Listing 1: "-1 is root"; reading G2)
      tab->lower[e] = -inf;
      tab->upper[e] = inf;
      tab->zero_fraction[e] = 1.0;
      ++e;
      for (int32_t i = 1; i < tr.len[q]; ++i, ++e, ++src) {
        const Edge& x = tr.elems[src];
        tab->feature[e] = x.f;
        tab->lower[e] = x.lo;
        tab->upper[e] = x.hi;
        tab->zero_fraction[e] = x.z;
      }
      tab->v[p] = tr.v[q];
      tab->group[p] = m->tree_group[t];
      tab->tree[p] = (int32_t)t;
    }
  }
  tab->path_offset[L] = E;
  // bias (a5, reading G13): sum over paths in path order of v * prod z (table
  // order), fp64; base_score added last.
  // The per-path products are independent (computed in parallel, each in
  // table order); the sum runs serially in path order, so the result is the
  // same bit pattern as one serial loop.
  tab->bias.assign(m->n_groups, 0.0);
  std::vector<double> vprod(L);
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < L; ++p) {
    double prod = 1.0;
    for (int64_t e = tab->path_offset[p]; e < tab->path_offset[p + 1]; ++e) prod *= tab->zero_fraction[e];
    vprod[p] = tab->v[p] * prod;
  }
  for (int64_t p = 0; p < L; ++p) tab->bias[tab->group[p]] += vprod[p];
  for (int32_t g = 0; g < m->n_groups; ++g) tab->bias[g] += m->base_score;
  out = std::move(tab);
  return GTS_OK;
}

// -------------------------------------------------------- bin packing (a3)

// Items in non-increasing size, ties by index (counting sort, stable).
static std::vector<int64_t> decreasing_order(const std::vector<int32_t>& size, int32_t cap) {
  std::vector<int64_t> count(cap + 2, 0);
  for (int32_t s : size) count[s]++;
  std::vector<int64_t> start(cap + 2, 0);
  int64_t pos = 0;
  for (int32_t s = cap; s >= 1; --s) { start[s] = pos; pos += count[s]; }
  std::vector<int64_t> order(size.size());
  for (int64_t i = 0; i < (int64_t)size.size(); ++i) order[start[size[i]]++] = i;
  return order;
}

// FFD with a max-segment-tree over bin residuals packed into an array
// (PAPER.md:526).  Unopened bins have residual = capacity and lie after the
// opened ones, so "first leaf with residual >= s" is either the first opened bin
// that fits or the next new bin.
static int64_t pack_ffd(const std::vector<int32_t>& size, int32_t cap, std::vector<int32_t>& bin_of) {
  const int64_t n = (int64_t)size.size();
  int64_t leaves = 1;
  while (leaves < std::max<int64_t>(n, 1)) leaves <<= 1;
  std::vector<int32_t> tree(2 * leaves, cap);
  int64_t n_bins = 0;
  for (int64_t i : decreasing_order(size, cap)) {
    const int32_t s = size[i];
    int64_t node = 1;
    while (node < leaves) node = (tree[2 * node] >= s) ? 2 * node : 2 * node + 1;
    const int64_t b = node - leaves;
    if (b >= n_bins) n_bins = b + 1;
    bin_of[i] = (int32_t)b;
    tree[node] -= s;
    for (node >>= 1; node >= 1; node >>= 1) tree[node] = std::max(tree[2 * node], tree[2 * node + 1]);
  }
  return n_bins;
}

// Set of bin ids with lowest-member lookup: a three-level 64-ary bitset
// (level 2 scanned from a cursor below which it is known to be empty).
class IdBitset {
 public:
  explicit IdBitset(int64_t n)
      : l0_((n + 63) / 64, 0), l1_((l0_.size() + 63) / 64, 0), l2_((l1_.size() + 63) / 64, 0) {}
  bool empty() const { return count_ == 0; }
  void insert(int64_t b) {
    ++count_;
    l0_[b >> 6] |= 1ull << (b & 63);
    l1_[b >> 12] |= 1ull << ((b >> 6) & 63);
    l2_[b >> 18] |= 1ull << ((b >> 12) & 63);
    if ((b >> 18) < lo_) lo_ = b >> 18;
  }
  void erase(int64_t b) {
    --count_;
    if ((l0_[b >> 6] &= ~(1ull << (b & 63))) != 0) return;
    if ((l1_[b >> 12] &= ~(1ull << ((b >> 6) & 63))) != 0) return;
    l2_[b >> 18] &= ~(1ull << ((b >> 12) & 63));
  }
  int64_t lowest() {  // precondition: !empty()
    while (l2_[lo_] == 0) ++lo_;
    const int64_t w2 = lo_, w1 = (w2 << 6) + __builtin_ctzll(l2_[w2]);
    const int64_t w0 = (w1 << 6) + __builtin_ctzll(l1_[w1]);
    return (w0 << 6) + __builtin_ctzll(l0_[w0]);
  }

 private:
  std::vector<uint64_t> l0_, l1_, l2_;
  int64_t lo_ = 0, count_ = 0;
};

// BFD: the open bin with the smallest residual >= s, ties to the
// lowest bin id.  Residuals are 1..cap (<= 32), so the open bins are kept in one
// id set per residual plus a bit mask of the non-empty residuals: the best bin
// is the lowest id of residual ctz(mask >> s) + s.  (The paper's std::set of
// (residual, bin) pairs gives the same packing, 5-10x slower at 6.6M items.)
static int64_t pack_bfd(const std::vector<int32_t>& size, int32_t cap, std::vector<int32_t>& bin_of) {
  const int64_t n = (int64_t)size.size();
  std::vector<IdBitset> open;
  open.reserve(cap + 1);
  for (int32_t r = 0; r <= cap; ++r) open.emplace_back(std::max<int64_t>(n, 1));
  uint64_t nonempty = 0;  // bit r: some open bin has residual r
  int64_t n_bins = 0;
  for (int64_t i : decreasing_order(size, cap)) {
    const int32_t s = size[i];
    const uint64_t fit = nonempty >> s;
    int64_t b;
    int32_t res;
    if (fit == 0) {
      b = n_bins++;
      res = cap - s;
    } else {
      const int32_t r = s + __builtin_ctzll(fit);
      b = open[r].lowest();
      open[r].erase(b);
      if (open[r].empty()) nonempty &= ~(1ull << r);
      res = r - s;
    }
    if (res > 0) {
      open[res].insert(b);
      nonempty |= 1ull << res;
    }
    bin_of[i] = (int32_t)b;
  }
  return n_bins;
}

static int64_t pack_nf(const std::vector<int32_t>& size, int32_t cap, std::vector<int32_t>& bin_of) {
  int64_t n_bins = 0;
  int32_t fill = cap + 1;
  for (size_t i = 0; i < size.size(); ++i) {
    if (fill + size[i] > cap) { ++n_bins; fill = 0; }
    bin_of[i] = (int32_t)(n_bins - 1);
    fill += size[i];
  }
  return n_bins;
}

static gts_status binpack(const std::shared_ptr<PathTable>& tab, int32_t cap, int32_t algo, gts_bins& out) {
  if (cap < 1 || cap > kWarp) return fail(GTS_ERR_INVALID_ARGUMENT, "capacity %d not in [1, %d]", cap, kWarp);
  if (algo < GTS_PACK_FFD || algo > GTS_PACK_NONE) return fail(GTS_ERR_INVALID_ARGUMENT, "bad pack algo %d", algo);
  const int64_t L = tab->n_paths();
  std::vector<int32_t> size(L);
  for (int64_t p = 0; p < L; ++p) {
    size[p] = tab->len(p);
    if (size[p] > cap)
      return fail(GTS_ERR_PATH_TOO_LONG, "path %lld of length %d exceeds capacity %d", (long long)p, size[p], cap);
  }
  out.tab = tab;
  out.capacity = cap;
  out.algo = algo;
  out.bin_of_path.assign(L, 0);
  out.lane_of_path.assign(L, 0);
  auto t0 = std::chrono::steady_clock::now();
  int64_t K = 0;
  switch (algo) {
    case GTS_PACK_FFD: K = pack_ffd(size, cap, out.bin_of_path); break;
    case GTS_PACK_BFD: K = pack_bfd(size, cap, out.bin_of_path); break;
    case GTS_PACK_NF: K = pack_nf(size, cap, out.bin_of_path); break;
    default:
      for (int64_t p = 0; p < L; ++p) out.bin_of_path[p] = (int32_t)p;
      K = L;
  }
  auto t1 = std::chrono::steady_clock::now();
  out.pack_seconds = std::chrono::duration<double>(t1 - t0).count();
  out.n_bins = K;
  // lanes: consecutive, in insertion order (FFD/BFD: decreasing order; NF/none: path order)
  std::vector<int32_t> fill(K, 0);
  if (algo == GTS_PACK_FFD || algo == GTS_PACK_BFD) {
    for (int64_t i : decreasing_order(size, cap)) {
      out.lane_of_path[i] = (uint8_t)fill[out.bin_of_path[i]];
      fill[out.bin_of_path[i]] += size[i];
    }
  } else {
    for (int64_t i = 0; i < L; ++i) {
      out.lane_of_path[i] = (uint8_t)fill[out.bin_of_path[i]];
      fill[out.bin_of_path[i]] += size[i];
    }
  }
  out.sum_sizes = tab->n_elems();
  return GTS_OK;
}

// --------------------------------------------------------- Gauss-Legendre

// Nodes t_q in (0,1) ascending and weights w_q (sum 1) of the Q-point
// Gauss-Legendre rule on [0,1]; exact for polynomials of degree <= 2Q-1.
// Newton iteration on P_Q in long double.
static void gauss_legendre01(int Q, long double* t, long double* w) {
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < Q; ++i) {
    long double x = std::cos(pi * (i + 0.75L) / (Q + 0.5L));
    long double dp = 0;
    for (int it = 0; it < 100; ++it) {
      long double p0 = 1, p1 = x;
      for (int n = 2; n <= Q; ++n) {
        long double p2 = ((2 * n - 1) * x * p1 - (n - 1) * p0) / n;
        p0 = p1;
        p1 = p2;
      }
      if (Q == 1) { p1 = x; p0 = 1; }
      dp = Q * (x * p1 - p0) / (x * x - 1);
      long double dx = p1 / dp;
      x -= dx;
      if (std::fabs((double)dx) < 1e-19) break;
    }
    {  // recompute derivative at the converged root
      long double p0 = 1, p1 = x;
      for (int n = 2; n <= Q; ++n) {
        long double p2 = ((2 * n - 1) * x * p1 - (n - 1) * p0) / n;
        p0 = p1;
        p1 = p2;
      }
      dp = Q * (x * p1 - p0) / (x * x - 1);
    }
    // x descending in i -> t = (1 - x)/2 ascending
    t[i] = (1 - x) / 2;
    w[i] = 1 / ((1 - x * x) * dp * dp);  // (2 / ((1-x^2) P'^2)) / 2
  }
}

// ------------------------------------------------------------ blobs (a4)

static int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

struct NodalPlan {
  std::vector<ChunkRec> chunks;
  std::vector<int32_t> slotmap;
  std::vector<PathRec> paths;
  std::vector<uint8_t> slots;  // slot of every planned element, chunk after chunk
  std::vector<double> work_shap, work_inter;
  int64_t max_words = 0, max_elems = 0, max_paths = 0;
  int32_t max_slots_used = 0, chunk_bytes = kChunkBytes;
};

// Default slot width of a SHAP-only blob: identity slot map up to 64 features.
static int pick_slots(int32_t requested, int32_t M) {
  if (requested != 0) return requested;
  if (M <= 8) return 8;
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  return 32;  // wide models: per-chunk slot maps
}

// nodal op counts per (row, path), DESIGN.md §6
static double paper_shap_flops(int k) { return 5.5 * k * k + 7.5 * k; }
static double paper_inter_flops(int k) { return paper_shap_flops(k) + (double)k * (k - 1) * (5.5 * k + 1) + 2.0 * k; }

// Chunking (blob_format.h): consecutive paths of one group, at most kChunkBytes
// of staged records + tables, at most S distinct features.  With an identity
// slot map (M <= S) the paths of a group are first ordered by (Q descending,
// length descending, feature set, index) so that paths sharing a feature set
// form runs; the feature set of a path is its bit mask (M <= 64).  Per-chunk
// slot maps (wide models) keep the input (DFS) order, which keeps the features
// of consecutive paths local.
static void plan_nodal(const PathTable& tab, int S, int nt, size_t tsize, NodalPlan& np) {
  const int32_t M = tab.n_features;
  const bool identity = M <= S;
  // wide identity tiles (SHAP only) leave less shared memory for staging
  const int chunk_bytes = (identity && S >= 32 && nt == 2) ? GTS_CHUNK_BYTES_WIDE : kChunkBytes;
  np.chunk_bytes = chunk_bytes;
  const int64_t L = tab.n_paths();
  std::vector<uint64_t> mask;
  if (identity) {
    mask.assign(L, 0);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < L; ++p) {
      uint64_t m = 0;
      for (int64_t e = tab.path_offset[p] + 1; e < tab.path_offset[p + 1]; ++e) m |= 1ull << tab.feature[e];
      mask[p] = m;
    }
  }
  auto fs_less = [&](int64_t a, int64_t b) {
    const int la = tab.len(a), lb = tab.len(b);
    const int qa = la / 2, qb = lb / 2;
    if (qa != qb) return qa > qb;
    if (la != lb) return la > lb;
    if (identity) {
      if (mask[a] != mask[b]) return mask[a] < mask[b];
    } else {
      for (int i = 1; i < la; ++i) {
        const int32_t fa = tab.feature[tab.path_offset[a] + i], fb = tab.feature[tab.path_offset[b] + i];
        if (fa != fb) return fa < fb;
      }
    }
    return a < b;
  };
  auto same_set = [&](int64_t a, int64_t b) {
    if (tab.len(a) != tab.len(b)) return false;
    if (identity) return mask[a] == mask[b];
    for (int i = 1; i < tab.len(a); ++i)
      if (tab.feature[tab.path_offset[a] + i] != tab.feature[tab.path_offset[b] + i]) return false;
    return true;
  };
  const int32_t G = tab.n_groups;
  std::vector<std::vector<int64_t>> by_group(G);
  for (int64_t p = 0; p < L; ++p)
    if (tab.len(p) > 1) by_group[tab.group[p]].push_back(p);
  // (Cutting small models into ~one chunk per SM lowered the 1-row latency of
  // cal_housing-small from 23 to 18 us but cost 30 % at 2^20 rows, since runs
  // and staging get shorter; profiles/r01h.  Not adopted.)
  // staged bytes of a chunk: element records (run heads only) + path headers (16 B each) + tables
  auto path_bytes = [&](int k, int q, bool head) {
    return (int64_t)16 * ((head ? k : 0) + 1) + (int64_t)tsize * nodal_path_words(k, q, nt);
  };

  // Chunks never span groups, so every group is planned on its own (in
  // parallel) with group-local offsets; the pieces are then concatenated in
  // group order, which gives the same plan as one pass over all groups.
  struct Part {
    std::vector<ChunkRec> chunks;    // path_begin / elem_begin local; slotmap_begin local to `maps`
    std::vector<int32_t> maps;       // this group's slot maps (one per local map id)
    std::vector<PathRec> paths;
    std::vector<uint8_t> slots;
    std::vector<double> ws, wi;
  };
  std::vector<Part> parts(G);
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t g = 0; g < G; ++g) {
    std::vector<int64_t>& order = by_group[g];
    if (identity) std::sort(order.begin(), order.end(), fs_less);
    Part& pt = parts[g];
    int32_t map_id = -1, n_cur = 0;
    int32_t cur_map[64], feats[64], u[128];
    int nf = 0;
    std::vector<int64_t> members;
    size_t i = 0;
    while (i < order.size()) {
      ChunkRec c{};
      c.group = g;
      c.path_begin = (int64_t)pt.paths.size();
      c.elem_begin = (int64_t)pt.slots.size();
      nf = 0;
      members.clear();
      int64_t bytes = 0, nel = 0;
      size_t j = i;
      while (j < order.size() && (int)members.size() < kMaxChunkPaths) {
        const int64_t p = order[j];
        const int k = tab.len(p) - 1, q = (k + 1) / 2;
        // a path repeating its predecessor's feature set joins its run (no element
        // records); sorting the chunk below only merges runs further, so this
        // count bounds the staged bytes
        const bool head = members.empty() || !same_set(members.back(), p);
        const int64_t w = path_bytes(k, q, head);
        if (!members.empty() && bytes + w > chunk_bytes) break;
        if (!identity) {  // union of two sorted feature lists
          const int32_t* pf = &tab.feature[tab.path_offset[p] + 1];
          int a = 0, b = 0, n = 0;
          while (a < nf || b < k) {
            int32_t x;
            if (b >= k || (a < nf && feats[a] < pf[b])) x = feats[a++];
            else if (a >= nf || pf[b] < feats[a]) x = pf[b++];
            else { x = feats[a++]; ++b; }
            u[n++] = x;
          }
          if (!members.empty() && n > S) break;
          std::memcpy(feats, u, sizeof(int32_t) * n);
          nf = n;
        }
        members.push_back(p);
        bytes += w;
        ++j;
      }
      if (identity) {
        nf = M;
        for (int32_t f = 0; f < M; ++f) feats[f] = f;
      }
      // inside the chunk: Q descending (template locality), then feature set (runs)
      std::sort(members.begin(), members.end(), fs_less);
      if (map_id < 0 || nf != n_cur || std::memcmp(feats, cur_map, sizeof(int32_t) * nf) != 0) {
        ++map_id;
        n_cur = nf;
        std::memcpy(cur_map, feats, sizeof(int32_t) * nf);
        c.slotmap_begin = (int64_t)pt.maps.size();
        pt.maps.insert(pt.maps.end(), feats, feats + nf);
      } else {
        c.slotmap_begin = pt.chunks.back().slotmap_begin;
      }
      c.map_id = map_id;
      c.n_slots = (int32_t)nf;
      c.n_paths = (int32_t)members.size();
      int32_t table = 0, rel = 0, maxq = 0;
      double ws = 0, wi = 0;
      size_t run_head = 0;
      for (size_t mi = 0; mi < members.size(); ++mi) {
        const int64_t p = members[mi];
        const int k = tab.len(p) - 1, q = (k + 1) / 2;
        if (mi == 0 || !same_set(members[run_head], p)) run_head = mi;
        const size_t head_index = pt.paths.size() - (mi - run_head);
        PathRec pr{};
        pr.k = k;
        if (run_head == mi) pr.k |= 1 << 16;
        else pt.paths[head_index].k += 1 << 16;
        pr.q = q;
        // element records: run heads only; the run's other paths share them
        // (same features, so the same x values and tile slots; each path's
        // split bounds are in its own rho rows)
        pr.elem = run_head == mi ? rel : pt.paths[head_index].elem;
        pr.table = table;
        pr.src = p;
        pt.paths.push_back(pr);
        if (run_head == mi) {
          for (int64_t e = tab.path_offset[p] + 1; e < tab.path_offset[p + 1]; ++e) {
            const int32_t f = tab.feature[e];
            pt.slots.push_back((uint8_t)(identity ? f : (std::lower_bound(feats, feats + nf, f) - feats)));
          }
          rel += k;
        }
        table += nodal_path_words(k, q, nt);
        maxq = std::max(maxq, q);
        ws += nodal_shap_flops(k, q);
        wi += nodal_inter_flops(k, q);
      }
      nel = rel;
      c.n_elems = (int32_t)nel;
      c.table_words = table;
      c.max_q = maxq;
      c.data_bytes = (int32_t)(16 * ((int64_t)nel + c.n_paths) + (int64_t)tsize * table);
      c.data_bytes = (c.data_bytes + 15) & ~15;
      pt.chunks.push_back(c);
      pt.ws.push_back(ws);
      pt.wi.push_back(wi);
      i = j;
    }
    std::vector<int64_t>().swap(order);
  }
  // concatenate: global offsets, and map ids that (as in one pass) continue
  // the previous chunk's id when its slot map is identical
  size_t n_chunks = 0, n_paths = 0, n_slots = 0;
  for (const Part& pt : parts) {
    n_chunks += pt.chunks.size();
    n_paths += pt.paths.size();
    n_slots += pt.slots.size();
  }
  np.chunks.reserve(n_chunks);
  np.work_shap.reserve(n_chunks);
  np.work_inter.reserve(n_chunks);
  np.paths.reserve(n_paths);
  np.slots.reserve(n_slots);
  int32_t gmap = -1;
  const int32_t* gmap_ptr = nullptr;
  int32_t gmap_n = 0;
  for (Part& pt : parts) {
    const int64_t path0 = (int64_t)np.paths.size(), elem0 = (int64_t)np.slots.size();
    int32_t last_local = -1;
    for (size_t ci = 0; ci < pt.chunks.size(); ++ci) {
      ChunkRec c = pt.chunks[ci];
      c.path_begin += path0;
      c.elem_begin += elem0;
      if (c.map_id != last_local) {
        last_local = c.map_id;
        const int32_t* mp = pt.maps.data() + c.slotmap_begin;
        if (gmap < 0 || c.n_slots != gmap_n || std::memcmp(mp, gmap_ptr, sizeof(int32_t) * c.n_slots) != 0) {
          ++gmap;
          gmap_n = c.n_slots;
          c.slotmap_begin = (int64_t)np.slotmap.size();
          np.slotmap.insert(np.slotmap.end(), mp, mp + c.n_slots);
        } else {
          c.slotmap_begin = np.chunks.back().slotmap_begin;
        }
        gmap_ptr = np.slotmap.data() + c.slotmap_begin;
      } else {
        c.slotmap_begin = np.chunks.back().slotmap_begin;
      }
      c.map_id = gmap;
      np.max_words = std::max<int64_t>(np.max_words, c.data_bytes);
      np.max_elems = std::max<int64_t>(np.max_elems, c.n_elems);
      np.max_paths = std::max<int64_t>(np.max_paths, c.n_paths);
      np.max_slots_used = std::max<int32_t>(np.max_slots_used, c.n_slots);
      np.chunks.push_back(c);
    }
    np.work_shap.insert(np.work_shap.end(), pt.ws.begin(), pt.ws.end());
    np.work_inter.insert(np.work_inter.end(), pt.wi.begin(), pt.wi.end());
    np.paths.insert(np.paths.end(), pt.paths.begin(), pt.paths.end());
    np.slots.insert(np.slots.end(), pt.slots.begin(), pt.slots.end());
    Part().chunks.swap(pt.chunks);
    std::vector<PathRec>().swap(pt.paths);
    std::vector<uint8_t>().swap(pt.slots);
  }
}

struct BinsPlan {
  std::vector<int64_t> bin_order;  // device bin -> packer bin, k_max descending
  std::vector<int32_t> kmax;
};

static void plan_bins(const gts_bins& b, BinsPlan& bp) {
  const PathTable& tab = *b.tab;
  std::vector<int32_t> km(b.n_bins, 0);
  for (int64_t p = 0; p < tab.n_paths(); ++p)
    km[b.bin_of_path[p]] = std::max(km[b.bin_of_path[p]], tab.len(p) - 1);
  bp.bin_order.resize(b.n_bins);
  for (int64_t i = 0; i < b.n_bins; ++i) bp.bin_order[i] = i;
  std::stable_sort(bp.bin_order.begin(), bp.bin_order.end(), [&](int64_t x, int64_t y) { return km[x] > km[y]; });
  bp.kmax.resize(b.n_bins);
  for (int64_t i = 0; i < b.n_bins; ++i) bp.kmax[i] = km[bp.bin_order[i]];
}

// Slot width and table rows of a NODAL blob for the requested uses.
// uses == 0: gts_blob_plan's default (SHAP layout; interactions too when S <= 16).
static gts_status nodal_shape(const PathTable& tab, int32_t max_slots, int32_t uses, int* S_out, int* nt_out,
                              int32_t* uses_out) {
  const int max_k = std::max(tab.max_len - 1, 0);
  const int32_t M = tab.n_features;
  int S;
  if (uses == 0 || uses == GTS_USE_SHAP) {
    if (max_slots != 0 && max_slots != 8 && max_slots != 16 && max_slots != 32 && max_slots != 64)
      return fail(GTS_ERR_INVALID_ARGUMENT, "max_slots must be 0, 8, 16, 32 or 64");
    S = pick_slots(max_slots, M);
    if (max_slots == 0) {
      while (S < max_k && S < 64) S *= 2;
    } else if (S < max_k && S < M) {
      return fail(GTS_ERR_INVALID_ARGUMENT,
                  "max_slots %d is smaller than the %d features of the longest path", S, max_k);
    }
    *nt_out = nodal_tables(S);
    *uses_out = uses == 0 ? (S <= 16 ? GTS_USE_BOTH : GTS_USE_SHAP) : GTS_USE_SHAP;
  } else if (uses == GTS_USE_INTERACTIONS || uses == GTS_USE_BOTH) {
    if (max_slots != 0 && max_slots != 8 && max_slots != 16 && max_slots != 32)
      return fail(GTS_ERR_INVALID_ARGUMENT, "interaction blobs take max_slots 0, 8, 16 or 32 (got %d)", max_slots);
    S = max_slots != 0 ? max_slots : (M <= 8 ? 8 : 16);
    if (max_slots == 0) {
      while (S < max_k) S *= 2;  // merged paths of 17..31 features: 32 slots
    } else if (S < max_k && S < M) {
      return fail(GTS_ERR_INVALID_ARGUMENT,
                  "max_slots %d is smaller than the %d features of the longest path", S, max_k);
    }
    if (uses == GTS_USE_BOTH && S > 16)
      return fail(GTS_ERR_INVALID_ARGUMENT,
                  "GTS_USE_BOTH needs a slot width <= 16 (this model needs %d): plan a SHAP blob and an "
                  "interaction blob", S);
    *nt_out = 3;
    *uses_out = uses;
  } else {
    return fail(GTS_ERR_INVALID_ARGUMENT, "bad blob uses %d", uses);
  }
  *S_out = S;
  return GTS_OK;
}

static gts_status blob_plan(const gts_bins* b, int32_t dtype, int32_t layout, int32_t max_slots, int32_t uses,
                            gts_blob_info* info, BlobHeader* hdr, NodalPlan* np, BinsPlan* bp) {
  if (!b || !info) return fail(GTS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (dtype != GTS_F32 && dtype != GTS_F64) return fail(GTS_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  if (layout != GTS_LAYOUT_NODAL && layout != GTS_LAYOUT_WARP_BINS)
    return fail(GTS_ERR_INVALID_ARGUMENT, "bad layout %d", layout);
  if (uses < 0 || uses > GTS_USE_BOTH) return fail(GTS_ERR_INVALID_ARGUMENT, "bad blob uses %d", uses);
  const PathTable& tab = *b->tab;
  const size_t tsize = dtype == GTS_F32 ? 4 : 8;
  BlobHeader h{};
  h.magic = kMagic;
  h.version = GTS_ABI_VERSION;
  h.dtype = dtype;
  h.layout = layout;
  h.n_features = tab.n_features;
  h.n_groups = tab.n_groups;
  h.max_len = tab.max_len;
  h.n_paths = tab.n_paths();
  h.n_elems = tab.n_elems();
  int64_t off = align256(sizeof(BlobHeader));
  h.off_bias = off;
  off = align256(off + 8 * (int64_t)tab.n_groups);
  double fs = 0, fi = 0, ps = 0, pi = 0;
  for (int64_t p = 0; p < tab.n_paths(); ++p) {
    const int k = tab.len(p) - 1, q = (k + 1) / 2;
    if (k == 0) continue;
    fs += nodal_shap_flops(k, q);
    fi += nodal_inter_flops(k, q);
    ps += paper_shap_flops(k);
    pi += paper_inter_flops(k);
  }
  if (layout == GTS_LAYOUT_NODAL) {
    int S = 0, nt = 0;
    int32_t u = 0;
    gts_status st = nodal_shape(tab, max_slots, uses, &S, &nt, &u);
    if (st != GTS_OK) return st;
    h.max_slots = S;
    h.uses = u;
    h.n_tables = nt;
    NodalPlan local;
    NodalPlan& P = np ? *np : local;
    plan_nodal(tab, S, nt, tsize, P);
    h.n_units = (int64_t)P.chunks.size();
    h.n_kept_paths = (int64_t)P.paths.size();
    h.n_kept_elems = (int64_t)P.slots.size();
    h.max_chunk_bytes = P.max_words;
    h.max_chunk_elems = P.max_elems;
    h.max_chunk_paths = P.max_paths;
    h.max_chunk_slots = P.max_slots_used;
    h.chunk_bytes = P.chunk_bytes;
    h.off_gauss = off;
    off = align256(off + (int64_t)tsize * kQMax * 3 * kQMax);
    h.off_units = off;
    off = align256(off + (int64_t)sizeof(ChunkRec) * h.n_units);
    h.off_work = off;
    off = align256(off + 8 * 2 * (h.n_units + 1));
    h.off_slotmap = off;
    off = align256(off + 4 * (int64_t)P.slotmap.size());
    h.off_paths = h.off_elems = off;  // staged chunk regions, back to back
    for (ChunkRec& c : P.chunks) {
      c.data_off = off;
      off += c.data_bytes;
    }
    off = align256(off);
  } else {
    h.max_slots = 0;
    h.uses = GTS_USE_BOTH;
    h.n_tables = 0;
    h.n_units = b->n_bins;
    if (b->capacity != kWarp)
      return fail(GTS_ERR_INVALID_ARGUMENT, "WARP_BINS layout needs capacity %d packing", kWarp);
    BinsPlan local;
    BinsPlan& P = bp ? *bp : local;
    plan_bins(*b, P);
    h.off_units = off;
    off = align256(off + 4 * h.n_units);
    h.off_elems = off;
    const int64_t lanes = h.n_units * kWarp;
    off = align256(off + lanes * (4 + 4 + 4 + 4 + 4) + lanes * 2 * (int64_t)tsize);
  }
  h.bytes = off;
  std::memset(info, 0, sizeof(*info));
  info->magic = kMagic;
  info->abi_version = GTS_ABI_VERSION;
  info->dtype = dtype;
  info->layout = layout;
  info->n_features = tab.n_features;
  info->n_groups = tab.n_groups;
  info->max_slots = h.max_slots;
  info->max_len = tab.max_len;
  info->n_paths = h.n_paths;
  info->n_elems = h.n_elems;
  info->n_units = h.n_units;
  info->bytes = h.bytes;
  info->shap_flops_per_row = fs;
  info->inter_flops_per_row = fi;
  info->paper_shap_flops_per_row = ps;
  info->paper_inter_flops_per_row = pi;
  info->max_chunk_bytes = h.max_chunk_bytes;
  info->max_chunk_elems = h.max_chunk_elems;
  info->max_chunk_paths = h.max_chunk_paths;
  info->uses = h.uses;
  info->n_tables = h.n_tables;
  info->max_chunk_slots = h.max_chunk_slots;
  info->chunk_bytes = h.chunk_bytes;
  if (hdr) *hdr = h;
  return GTS_OK;
}

template <typename T>
static void write_gauss(char* dst) {
  T* g = reinterpret_cast<T*>(dst);
  for (int Q = 1; Q <= kQMax; ++Q) {
    long double t[kQMax], w[kQMax];
    gauss_legendre01(Q, t, w);
    T* row = g + (size_t)(Q - 1) * 3 * kQMax;
    for (int q = 0; q < kQMax; ++q) {
      row[q] = q < Q ? (T)t[q] : (T)0;
      row[kQMax + q] = q < Q ? (T)w[q] : (T)0;
      row[2 * kQMax + q] = q < Q ? (T)(-1.0L / (1.0L - t[q])) : (T)0;
    }
  }
}

// Staged chunk regions (blob_format.h): element records, path headers, and the
// nodal tables, computed in fp64 from the fp64 zero fractions and leaf values
// and rounded once to T (reading G11: one rounding in fp32 mode).  Per node the
// reciprocals 1/A_sq and 1/(1 - t_q) are formed once and multiplied.
struct GaussTab {  // Q-point rules on [0, 1] for Q = 1..kQMax, in fp64
  double tq[kQMax + 1][kQMax], wq[kQMax + 1][kQMax], rq[kQMax + 1][kQMax];
  GaussTab() {
    for (int Q = 1; Q <= kQMax; ++Q) {
      long double t[kQMax], w[kQMax];
      gauss_legendre01(Q, t, w);
      for (int q = 0; q < Q; ++q) {
        tq[Q][q] = (double)t[q];
        wq[Q][q] = (double)w[q];
        rq[Q][q] = (double)(1.0L / (1.0L - t[q]));
      }
    }
  }
};

// The staged region of chunk ci, written at `region` (c.data_bytes bytes;
// table pads q >= Q and the tail stay zero).
template <typename T>
static void write_region(const PathTable& tab, const NodalPlan& np, const GaussTab& gt, int64_t ci, int S, int nt,
                         char* region) {
  const ChunkRec& c = np.chunks[ci];
  std::memset(region, 0, (size_t)c.data_bytes);
  int32_t* E = reinterpret_cast<int32_t*>(region);
  int32_t* Pp = E + 4 * (int64_t)c.n_elems;
  T* tab_out = reinterpret_cast<T*>(Pp + 4 * (int64_t)c.n_paths);
  for (int32_t p = 0; p < c.n_paths; ++p) {
    const PathRec& pr = np.paths[c.path_begin + p];
    Pp[4 * p + 0] = pr.k;
    Pp[4 * p + 1] = pr.q;
    Pp[4 * p + 2] = pr.elem;
    Pp[4 * p + 3] = pr.table;
    const int k = pr.k & 0xff, Q = pr.q, QP = nodal_qp(Q), RW = nodal_rw(Q), ES = nodal_es(Q, nt), BO = nodal_bo(Q),
              BW = nodal_bw(Q);
    const int64_t e0 = tab.path_offset[pr.src] + 1;  // first non-root element
    const uint8_t* sl = &np.slots[c.elem_begin + pr.elem];
    for (int s = 0; s < ((pr.k >> 16) != 0 ? k : 0); ++s) {  // run heads write the run's records
      int32_t* rec = E + 4 * (int64_t)(pr.elem + s);
      std::memcpy(&rec[0], &tab.lower[e0 + s], 4);
      std::memcpy(&rec[1], &tab.upper[e0 + s], 4);
      // interaction tables (nt = 3): the slot and the upper-triangle row base of
      // the slot; SHAP-only tables (nt = 2): the slot's byte offset in a tile row
      // and the feature itself (kernels that read X from global memory)
      rec[2] = nt == 3 ? sl[s] : sl[s] * (int32_t)sizeof(T);
      rec[3] = nt == 3 ? sl[s] * (2 * S - sl[s] - 1) / 2 : tab.feature[e0 + s];
    }
    const double* z = &tab.zero_fraction[e0];
    const double v = tab.v[pr.src];
    T* t = tab_out + pr.table;
    for (int q = 0; q < Q; ++q) {
      const double tt = gt.tq[Q][q], w = gt.wq[Q][q], r1 = gt.rq[Q][q];
      double cq = 1.0;
      for (int s = 0; s < k; ++s) cq *= z[s] + (1.0 - z[s]) * tt;
      t[q] = (T)cq;
      t[QP + q] = (T)(-v * w * r1);
      if (nt == 3) t[2 * QP + q] = (T)(0.5 * v * w);
      for (int s = 0; s < k; ++s) {
        const double zs = z[s];
        const double A = zs + (1.0 - zs) * tt, iA = 1.0 / A;
        T* row = t + nt * QP + BW + s * ES;
        row[q] = (T)(zs * (1.0 - tt) * iA);                 // rho = B / A
        row[RW + q] = (T)(v * w * ((1.0 - zs) * iA + r1));  // C' = C - d
        if (nt == 3) row[RW + QP + q] = (T)((1.0 - zs) * iA);
      }
    }
    for (int s = 0; s < k; ++s) {  // split bounds (exact in T: they are fp32 values)
      T* b = nodal_inrow(Q) ? t + nt * QP + s * ES + BO : t + nt * QP + 2 * s;
      b[0] = (T)tab.lower[e0 + s];
      b[1] = (T)tab.upper[e0 + s];
    }
  }
}

template <typename T>
static void write_bins(const gts_bins& b, const BinsPlan& bp, const BlobHeader& h, char* dst) {
  const PathTable& tab = *b.tab;
  const int64_t K = h.n_units, lanes = K * kWarp;
  std::memcpy(dst + h.off_units, bp.kmax.data(), 4 * K);
  char* base = dst + h.off_elems;
  int32_t* feat = reinterpret_cast<int32_t*>(base);
  int32_t* meta = feat + lanes;
  int32_t* grp = meta + lanes;
  float* lo = reinterpret_cast<float*>(grp + lanes);
  float* hi = lo + lanes;
  T* z = reinterpret_cast<T*>(hi + lanes);
  T* v = z + lanes;
  std::vector<int64_t> dev_of(K);
  for (int64_t i = 0; i < K; ++i) dev_of[bp.bin_order[i]] = i;
  const float inf = std::numeric_limits<float>::infinity();
  for (int64_t l = 0; l < lanes; ++l) {
    feat[l] = -2;
    meta[l] = 0;
    grp[l] = 0;
    lo[l] = -inf;
    hi[l] = inf;
    z[l] = (T)1;
    v[l] = (T)0;
  }
  for (int64_t p = 0; p < tab.n_paths(); ++p) {
    const int64_t db = dev_of[b.bin_of_path[p]];
    const int32_t lane0 = b.lane_of_path[p];
    const int32_t len = tab.len(p);
    for (int32_t r = 0; r < len; ++r) {
      const int64_t e = tab.path_offset[p] + r;
      const int64_t l = db * kWarp + lane0 + r;
      feat[l] = tab.feature[e];
      meta[l] = r | ((len - 1) << 8) | (lane0 << 16);
      grp[l] = tab.group[p];
      lo[l] = tab.lower[e];
      hi[l] = tab.upper[e];
      z[l] = (T)tab.zero_fraction[e];
      v[l] = (T)tab.v[p];
    }
  }
}

// The plan of the last gts_blob_plan* call on these bins is kept (keyed by its
// arguments) for the gts_blob_write that normally follows, which takes it.
struct PlanCache {
  int32_t dtype = -1, layout = -1, max_slots = -1, uses = -1;
  gts_blob_info info{};
  BlobHeader hdr{};
  NodalPlan np;
  BinsPlan bp;
};

static gts_status blob_plan_cached(const gts_bins* b, int32_t dtype, int32_t layout, int32_t max_slots, int32_t uses,
                                   gts_blob_info* info) {
  if (!b || !info) return fail(GTS_ERR_INVALID_ARGUMENT, "NULL argument");
  auto pc = std::make_shared<PlanCache>();
  gts_status st = blob_plan(b, dtype, layout, max_slots, uses, info, &pc->hdr, &pc->np, &pc->bp);
  if (st != GTS_OK) return st;
  pc->dtype = dtype;
  pc->layout = layout;
  pc->max_slots = max_slots;
  pc->uses = uses;
  pc->info = *info;
  std::lock_guard<std::mutex> lock(b->cache_mu);
  b->cache = std::move(pc);
  return GTS_OK;
}

// Bytes [offset, offset + len) of the blob into dst.  The plan of the last
// gts_blob_plan* call on these bins is used when it matches `info` (taken when
// `take`, i.e. by a whole-blob gts_blob_write; kept for the next range
// otherwise), else the plan is rebuilt (a pure function of the bins and the
// info's dtype / layout / slots / uses).
static gts_status blob_write_range(const gts_bins* b, const gts_blob_info* info, int64_t offset, int64_t len,
                                   void* dst, bool take) {
  if (!b || !info || (!dst && len > 0)) return fail(GTS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (info->magic != kMagic || info->abi_version != GTS_ABI_VERSION)
    return fail(GTS_ERR_INVALID_ARGUMENT, "info is not a gts_blob_info of ABI version %d", GTS_ABI_VERSION);
  if (offset < 0 || len < 0 || offset + len > info->bytes)
    return fail(GTS_ERR_INVALID_ARGUMENT, "range [%lld, %lld) outside the %lld-byte blob", (long long)offset,
                (long long)(offset + len), (long long)info->bytes);
  std::shared_ptr<PlanCache> pc;
  {
    std::lock_guard<std::mutex> lock(b->cache_mu);
    if (b->cache && std::memcmp(&b->cache->info, info, sizeof(*info)) == 0) {
      pc = b->cache;
      if (take) b->cache.reset();
    }
  }
  if (!pc) {
    pc = std::make_shared<PlanCache>();
    const int32_t req_uses = info->layout == GTS_LAYOUT_NODAL ? info->uses : 0;
    gts_status st = blob_plan(b, info->dtype, info->layout, info->max_slots, req_uses, &pc->info, &pc->hdr, &pc->np,
                              &pc->bp);
    if (st != GTS_OK) return st;
    if (pc->info.bytes != info->bytes || pc->info.n_units != info->n_units || pc->info.n_tables != info->n_tables)
      return fail(GTS_ERR_INVALID_ARGUMENT, "blob info does not match these bins");
    pc->dtype = info->dtype;
    pc->layout = info->layout;
    pc->max_slots = info->max_slots;
    pc->uses = req_uses;
    if (!take) {
      std::lock_guard<std::mutex> lock(b->cache_mu);
      b->cache = pc;
    }
  }
  const BlobHeader& h = pc->hdr;
  char* out = static_cast<char*>(dst);
  const int64_t end = offset + len;
  if (h.layout != GTS_LAYOUT_NODAL) {  // WARP_BINS: the whole blob, then the range
    std::vector<char> full;
    char* w = out;
    if (offset != 0 || len != h.bytes) {
      full.assign((size_t)h.bytes, 0);
      w = full.data();
    } else {
      std::memset(w, 0, (size_t)h.bytes);
    }
    std::memcpy(w, &h, sizeof(h));
    std::memcpy(w + h.off_bias, b->tab->bias.data(), 8 * b->tab->bias.size());
    if (h.dtype == GTS_F32) write_bins<float>(*b, pc->bp, h, w);
    else write_bins<double>(*b, pc->bp, h, w);
    if (w != out) std::memcpy(out, w + offset, (size_t)len);
    return GTS_OK;
  }
  const NodalPlan& np = pc->np;
  // head: header, bias, Gauss table, chunk records, prefix work, slot maps
  if (offset < h.off_elems) {
    std::vector<char> head((size_t)h.off_elems, 0);
    char* w = head.data();
    std::memcpy(w, &h, sizeof(h));
    std::memcpy(w + h.off_bias, b->tab->bias.data(), 8 * b->tab->bias.size());
    if (h.dtype == GTS_F32) write_gauss<float>(w + h.off_gauss);
    else write_gauss<double>(w + h.off_gauss);
    std::memcpy(w + h.off_units, np.chunks.data(), sizeof(ChunkRec) * np.chunks.size());
    double* ws = reinterpret_cast<double*>(w + h.off_work);
    double* wi = ws + (h.n_units + 1);
    ws[0] = wi[0] = 0;
    for (int64_t c = 0; c < h.n_units; ++c) {
      ws[c + 1] = ws[c] + np.work_shap[c];
      wi[c + 1] = wi[c] + np.work_inter[c];
    }
    std::memcpy(w + h.off_slotmap, np.slotmap.data(), 4 * np.slotmap.size());
    const int64_t e = std::min<int64_t>(end, h.off_elems);
    std::memcpy(out, w + offset, (size_t)(e - offset));
  }
  // staged chunk regions (back to back from off_elems), then zero padding to h.bytes
  const int64_t C = (int64_t)np.chunks.size();
  int64_t c0 = 0, c1 = C;
  {
    int64_t lo = 0, hi = C;  // first chunk ending after offset
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (np.chunks[mid].data_off + np.chunks[mid].data_bytes <= offset) lo = mid + 1; else hi = mid;
    }
    c0 = lo;
    lo = c0, hi = C;  // first chunk starting at or after end
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (np.chunks[mid].data_off < end) lo = mid + 1; else hi = mid;
    }
    c1 = lo;
  }
  const GaussTab gt;
  const int S = h.max_slots, nt = h.n_tables;
#pragma omp parallel
  {
    std::vector<char> tmp;
#pragma omp for schedule(dynamic, 16)
    for (int64_t ci = c0; ci < c1; ++ci) {
      const ChunkRec& c = np.chunks[ci];
      const int64_t a = c.data_off, z = c.data_off + c.data_bytes;
      char* reg;
      if (a >= offset && z <= end) {
        reg = out + (a - offset);
      } else {
        tmp.resize((size_t)c.data_bytes);
        reg = tmp.data();
      }
      if (h.dtype == GTS_F32) write_region<float>(*b->tab, np, gt, ci, S, nt, reg);
      else write_region<double>(*b->tab, np, gt, ci, S, nt, reg);
      if (reg != out + (a - offset)) {
        const int64_t s0 = std::max(a, offset), s1 = std::min(z, end);
        std::memcpy(out + (s0 - offset), reg + (s0 - a), (size_t)(s1 - s0));
      }
    }
  }
  const int64_t regions_end = C > 0 ? np.chunks[C - 1].data_off + np.chunks[C - 1].data_bytes : h.off_elems;
  const int64_t p0 = std::max(offset, regions_end);
  if (end > p0) std::memset(out + (p0 - offset), 0, (size_t)(end - p0));
  return GTS_OK;
}

static gts_status blob_write(const gts_bins* b, const gts_blob_info* info, void* dst, size_t dst_bytes) {
  if (!b || !info || !dst) return fail(GTS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (info->magic != kMagic || info->abi_version != GTS_ABI_VERSION)
    return fail(GTS_ERR_INVALID_ARGUMENT, "info is not a gts_blob_info of ABI version %d", GTS_ABI_VERSION);
  if (dst_bytes < (size_t)info->bytes)
    return fail(GTS_ERR_INVALID_ARGUMENT, "destination too small: %zu < %lld", dst_bytes, (long long)info->bytes);
  return blob_write_range(b, info, 0, info->bytes, dst, true);
}

}  // namespace gts

// ================================================================ C ABI

extern "C" {

gts_status gts_extract_paths(const gts_model* model, gts_paths** out) {
  if (!out) return gts::fail(GTS_ERR_INVALID_ARGUMENT, "out is NULL");
  GTS_NVTX("gts_extract_paths");
  try {
    std::shared_ptr<gts::PathTable> tab;
    gts_status st = gts::extract(model, tab);
    if (st != GTS_OK) return st;
    *out = new gts_paths{std::move(tab)};
    return GTS_OK;
  } catch (const std::bad_alloc&) {
    return gts::fail(GTS_ERR_OUT_OF_MEMORY, "out of host memory");
  }
}

gts_status gts_paths_view_get(const gts_paths* paths, gts_paths_view* v) {
  if (!paths || !v) return gts::fail(GTS_ERR_INVALID_ARGUMENT, "NULL argument");
  const gts::PathTable& t = *paths->tab;
  v->n_paths = t.n_paths();
  v->n_elems = t.n_elems();
  v->n_features = t.n_features;
  v->n_groups = t.n_groups;
  v->max_len = t.max_len;
  v->path_offset = t.path_offset.data();
  v->feature = t.feature.data();
  v->lower = t.lower.data();
  v->upper = t.upper.data();
  v->zero_fraction = t.zero_fraction.data();
  v->v = t.v.data();
  v->group = t.group.data();
  v->tree = t.tree.data();
  v->bias = t.bias.data();
  return GTS_OK;
}

void gts_paths_free(gts_paths* paths) { delete paths; }

gts_status gts_binpack(const gts_paths* paths, int32_t capacity, gts_pack_algo algo, gts_bins** out) {
  if (!paths || !out) return gts::fail(GTS_ERR_INVALID_ARGUMENT, "NULL argument");
  GTS_NVTX("gts_binpack");
  try {
    auto b = std::make_unique<gts_bins>();
    gts_status st = gts::binpack(paths->tab, capacity, (int32_t)algo, *b);
    if (st != GTS_OK) return st;
    *out = b.release();
    return GTS_OK;
  } catch (const std::bad_alloc&) {
    return gts::fail(GTS_ERR_OUT_OF_MEMORY, "out of host memory");
  }
}

gts_status gts_bins_view_get(const gts_bins* b, gts_bins_view* v) {
  if (!b || !v) return gts::fail(GTS_ERR_INVALID_ARGUMENT, "NULL argument");
  v->n_items = (int64_t)b->bin_of_path.size();
  v->n_bins = b->n_bins;
  v->sum_sizes = b->sum_sizes;
  v->capacity = b->capacity;
  v->algo = b->algo;
  v->utilisation = b->n_bins == 0 ? 1.0 : (double)b->sum_sizes / ((double)b->capacity * (double)b->n_bins);
  v->pack_seconds = b->pack_seconds;
  v->bin_of_path = b->bin_of_path.data();
  v->lane_of_path = b->lane_of_path.data();
  return GTS_OK;
}

void gts_bins_free(gts_bins* b) { delete b; }

gts_status gts_blob_plan(const gts_bins* bins, gts_dtype dtype, gts_layout layout, int32_t max_slots,
                         gts_blob_info* info) {
  GTS_NVTX("gts_blob_plan");
  try {
    return gts::blob_plan_cached(bins, (int32_t)dtype, (int32_t)layout, max_slots, 0, info);
  } catch (const std::bad_alloc&) {
    return gts::fail(GTS_ERR_OUT_OF_MEMORY, "out of host memory");
  }
}

gts_status gts_blob_plan_for(const gts_bins* bins, gts_dtype dtype, gts_layout layout, int32_t max_slots,
                             gts_blob_use uses, gts_blob_info* info) {
  if ((int32_t)uses < GTS_USE_SHAP || (int32_t)uses > GTS_USE_BOTH)
    return gts::fail(GTS_ERR_INVALID_ARGUMENT, "bad blob uses %d", (int)uses);
  GTS_NVTX("gts_blob_plan_for");
  try {
    return gts::blob_plan_cached(bins, (int32_t)dtype, (int32_t)layout, max_slots, (int32_t)uses, info);
  } catch (const std::bad_alloc&) {
    return gts::fail(GTS_ERR_OUT_OF_MEMORY, "out of host memory");
  }
}

gts_status gts_blob_write(const gts_bins* bins, const gts_blob_info* info, void* host_dst, size_t dst_bytes) {
  GTS_NVTX("gts_blob_write");
  try {
    return gts::blob_write(bins, info, host_dst, dst_bytes);
  } catch (const std::bad_alloc&) {
    return gts::fail(GTS_ERR_OUT_OF_MEMORY, "out of host memory");
  }
}

gts_status gts_blob_write_range(const gts_bins* bins, const gts_blob_info* info, int64_t offset, int64_t bytes,
                                void* host_dst) {
  GTS_NVTX("gts_blob_write_range");
  try {
    return gts::blob_write_range(bins, info, offset, bytes, host_dst, false);
  } catch (const std::bad_alloc&) {
    return gts::fail(GTS_ERR_OUT_OF_MEMORY, "out of host memory");
  }
}

const char* gts_last_error(void) { return gts::last_error(); }

const char* gts_status_string(gts_status s) {
  switch (s) {
    case GTS_OK: return "GTS_OK";
    case GTS_ERR_INVALID_ARGUMENT: return "GTS_ERR_INVALID_ARGUMENT";
    case GTS_ERR_INVALID_MODEL: return "GTS_ERR_INVALID_MODEL";
    case GTS_ERR_PATH_TOO_LONG: return "GTS_ERR_PATH_TOO_LONG";
    case GTS_ERR_NONFINITE: return "GTS_ERR_NONFINITE";
    case GTS_ERR_CUDA: return "GTS_ERR_CUDA";
    case GTS_ERR_OUT_OF_MEMORY: return "GTS_ERR_OUT_OF_MEMORY";
  }
  return "GTS_UNKNOWN_STATUS";
}

int32_t gts_abi_version(void) { return GTS_ABI_VERSION; }

}  // extern "C"
