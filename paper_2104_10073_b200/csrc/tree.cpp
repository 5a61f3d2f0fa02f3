// tree.cpp — lock-step host driver of tree_refine (ref src/estimator.cpp:
// 184-318) over many trees; see tree.hpp.  Every floating-point step of the
// selection (mean / sd of the leaf std_errors, threshold), the split
// (longest edge, midpoint low + 0.5*(high-low)) and the final combine_cells
// (src/estimator.cpp:145-159) is the reference's, in its order, built with
// -ffp-contract=off.  Only the cell estimates come from the GPU.
#include "tree.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

namespace mcb::tree {

namespace {

uint64_t chunk_count(uint64_t n) { return (n + MCB_CHUNK_SIZE - 1) / MCB_CHUNK_SIZE; }

// cell_grid_size, src/estimator.cpp:94-105 (false = CellBudgetExceeded)
bool cell_grid_size(uint32_t k, uint32_t d, uint64_t cap, uint64_t& cells) {
  if (k == 0) return false;
  cells = 1;
  for (uint32_t i = 0; i < d; ++i) {
    if (cells > cap / k + 1) return false;
    cells *= k;
  }
  return cells <= cap;
}

// auto_cells_per_dim, src/estimator.cpp:107-122
uint32_t auto_cells_per_dim(uint32_t d, uint64_t limit) {
  uint32_t k = 1;
  for (;;) {
    uint64_t cells = 1;
    for (uint32_t i = 0; i < d; ++i) {
      cells *= uint64_t(k) + 1;
      if (cells > limit) return k;
    }
    ++k;
  }
}

// Trees are independent, so the per-round host work (selection + splits,
// result scatter, first pass, combine) is spread over a small pool of host
// threads; each tree is touched by one thread at a time, in its reference
// order, so results do not depend on the thread count.
class Pool {
 public:
  explicit Pool(unsigned n_threads) {
    for (unsigned i = 1; i < n_threads; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  // fn(i) for i in [0, n), dynamic chunks; returns when all are done.
  void run(size_t n, const std::function<void(size_t)>& fn) {
    if (workers_.empty() || n < 2 * kChunk) {
      for (size_t i = 0; i < n; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      busy_ = workers_.size();
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return busy_ == 0; });
    fn_ = nullptr;
  }

 private:
  static constexpr size_t kChunk = 8;
  void drain() {
    for (;;) {
      const size_t b = next_.fetch_add(kChunk);
      if (b >= n_) return;
      const size_t e = std::min(n_, b + kChunk);
      for (size_t i = b; i < e; ++i) (*fn_)(i);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      drain();
      std::lock_guard<std::mutex> lk(mu_);
      if (--busy_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* fn_ = nullptr;
  size_t n_ = 0;
  std::atomic<size_t> next_{0};
  size_t busy_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

unsigned host_threads(size_t n_trees) {
  if (n_trees < 64) return 1;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  return std::min(hw, 16u);
}

// Leaves are kept structure-of-arrays: the per-round selection scans only
// the std_errors and depths (12 B per leaf), not the rectangles.
struct Tree {
  TreeTask* task;
  Config cfg;
  uint32_t dim;
  uint32_t spc;
  uint64_t cpc;
  std::vector<double> rect;          // leaf i: rect[2*dim*i ..] = {low[dim], high[dim]}
  std::vector<double> se;            // leaf std_error (the selection statistic)
  std::vector<uint32_t> depth;
  std::vector<mcb_trial_stats> est;  // leaf McEstimate
  uint64_t next_chunk;
  uint64_t used = 0;
  bool exhausted = false;
  bool active = true;
  uint32_t fail = MCB_TRIAL_OK;  // CELL_BUDGET / CHUNK_RANGE: the tree threw
  // this round's cells: leaf index, rectangle, estimate; chunk of the first
  std::vector<uint32_t> r_leaf;
  std::vector<double> r_rects;
  std::vector<CellEst> r_est;
  uint64_t r_chunk0 = 0;

  size_t size() const { return se.size(); }
  double* lo(size_t i) { return rect.data() + 2 * dim * i; }
  double* hi(size_t i) { return rect.data() + 2 * dim * i + dim; }
  void add_leaf(uint32_t d) {
    rect.resize(rect.size() + 2 * dim);
    se.push_back(0.0);
    depth.push_back(d);
    est.emplace_back();
  }
};

// estimate_cell (src/estimator.cpp:238-253): key chunk next_chunk, then
// next_chunk += chunks_per_cell and used += spc.  The estimate is deferred
// to the round's launch.
void estimate_cell(Tree& t, size_t leaf) {
  if (t.next_chunk + t.cpc - 1 > 0xFFFFFFFFull) {  // UniformStream throws (src/sampling.cpp:80-81)
    t.fail = MCB_TRIAL_CHUNK_RANGE;
    t.active = false;
    return;
  }
  if (t.r_leaf.empty()) t.r_chunk0 = t.next_chunk;
  t.r_leaf.push_back(uint32_t(leaf));
  const double* r = t.lo(leaf);
  t.r_rects.insert(t.r_rects.end(), r, r + 2 * t.dim);
  t.next_chunk += t.cpc;
  t.used += t.spc;
}

// The AllSamplesNonFinite catch of estimate_cell: a dead leaf.
mcb_trial_stats dead_leaf(uint32_t spc) {
  mcb_trial_stats s;
  std::memset(&s, 0, sizeof s);
  s.status = MCB_TRIAL_ALL_NONFINITE;
  s.n_samples = spc;
  s.n_nonfinite = spc;
  s.nonfinite_warning = 1;
  return s;
}

// MCB_TREE_TRACE=1: per-round cell counts and times on stderr.
bool trace_on() {
  static const bool on = [] {
    const char* e = std::getenv("MCB_TREE_TRACE");
    return e && *e && *e != '0';
  }();
  return on;
}

// One launch set for every tree's pending cells, then the results land in
// the leaves.
mcb_status run_round(std::vector<Tree>& trees, const CellRunner& run, Pool& pool) {
  std::vector<CellBatch> batches;
  std::vector<Tree*> owner;
  size_t cells = 0;
  for (Tree& t : trees) {
    if (t.r_leaf.empty()) continue;
    if (t.fail != MCB_TRIAL_OK) {
      t.r_leaf.clear();
      t.r_rects.clear();
      continue;
    }
    t.r_est.resize(t.r_leaf.size());
    batches.push_back(CellBatch{t.task->fn, t.task->trial, t.r_chunk0, t.spc, uint32_t(t.r_leaf.size()),
                                t.r_rects.data(), t.r_est.data()});
    owner.push_back(&t);
    cells += t.r_leaf.size();
  }
  if (batches.empty()) return MCB_OK;
  const auto t0 = std::chrono::steady_clock::now();
  const mcb_status st = run(batches);
  if (trace_on())
    std::fprintf(stderr, "[mcb tree] round: %zu trees, %zu cells, %.3f ms\n", batches.size(), cells,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  if (st != MCB_OK) return st;
  pool.run(owner.size(), [&](size_t k) {
    Tree* t = owner[k];
    for (size_t i = 0; i < t->r_leaf.size(); ++i) {
      const uint32_t l = t->r_leaf[i];
      mcb_trial_stats& e = t->est[l];
      const CellEst& r = t->r_est[i];
      if (r.status == MCB_TRIAL_OK) {
        std::memset(&e, 0, sizeof e);
        e.value = r.value;
        e.std_error = r.std_error;
        e.n_samples = t->spc;
        e.n_nonfinite = r.n_nonfinite;
        e.nonfinite_warning = double(r.n_nonfinite) > MCB_NONFINITE_WARN_FRACTION * double(t->spc) ? 1u : 0u;
        e.n_cells = 1;
      } else {
        e = dead_leaf(t->spc);
      }
      t->se[l] = e.std_error;
    }
    t->r_leaf.clear();
    t->r_rects.clear();
  });
  return MCB_OK;
}

// split_longest_edge, src/estimator.cpp:192-210: first axis of maximal
// width; the lower half replaces leaf `idx` in place, the upper half is
// appended as leaf `hi_idx`.
void split_longest_edge(Tree& t, size_t idx, size_t hi_idx) {
  const uint32_t d = t.dim;
  uint32_t axis = 0;
  double best = -1.0;
  const double* lo = t.lo(idx);
  const double* hi = t.hi(idx);
  for (uint32_t j = 0; j < d; ++j) {
    const double w = hi[j] - lo[j];
    if (w > best) {
      best = w;
      axis = j;
    }
  }
  const double mid = lo[axis] + 0.5 * (hi[axis] - lo[axis]);
  std::memcpy(t.lo(hi_idx), t.lo(idx), sizeof(double) * 2 * d);
  t.hi(idx)[axis] = mid;
  t.lo(hi_idx)[axis] = mid;
}

// One refinement step of the `while (!exhausted)` loop, src/estimator.cpp:265-297.
void refine_step(Tree& t, std::vector<uint32_t>& selected) {
  const size_t n = t.size();
  const double* se = t.se.data();
  double mean_err = 0.0;
  for (size_t i = 0; i < n; ++i) mean_err += se[i];
  mean_err /= double(n);
  double ss = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double dlt = se[i] - mean_err;
    ss += dlt * dlt;
  }
  const double sd = n > 1 ? std::sqrt(ss / double(n - 1)) : 0.0;
  const double threshold = mean_err + t.cfg.sigma_multiplier * sd;

  selected.clear();
  for (size_t i = 0; i < n; ++i)
    if (t.depth[i] < t.cfg.max_depth && se[i] > 0 && se[i] > threshold) selected.push_back(uint32_t(i));
  if (selected.empty()) {
    t.active = false;
    return;
  }
  for (uint32_t idx : selected) {
    if (t.used + 2ull * t.spc > t.cfg.total_budget) {
      t.exhausted = true;
      break;
    }
    const uint32_t child_depth = t.depth[idx] + 1;
    t.add_leaf(child_depth);
    const size_t hi_idx = t.size() - 1;
    split_longest_edge(t, idx, hi_idx);
    t.depth[idx] = child_depth;
    estimate_cell(t, idx);
    if (t.fail != MCB_TRIAL_OK) return;
    estimate_cell(t, hi_idx);
    if (t.fail != MCB_TRIAL_OK) return;
  }
  if (t.exhausted) t.active = false;  // the while condition
}

void finish(Tree& t) {
  mcb_trial_stats& o = *t.task->out;
  std::memset(&o, 0, sizeof o);
  if (t.fail != MCB_TRIAL_OK) {
    o.status = t.fail;
    return;
  }
  // combine_cells (src/estimator.cpp:145-159) over the leaves in order
  double value = 0.0, var = 0.0;
  uint64_t n_samples = 0, n_nonfinite = 0, total_finite = 0;
  uint32_t depth = 0;
  for (size_t i = 0; i < t.size(); ++i) {
    const mcb_trial_stats& e = t.est[i];
    value += e.value;
    var += e.std_error * e.std_error;
    n_samples += e.n_samples;
    n_nonfinite += e.n_nonfinite;
    total_finite += e.n_samples - e.n_nonfinite;
    depth = std::max(depth, t.depth[i]);
  }
  o.n_samples = n_samples;
  o.n_nonfinite = n_nonfinite;
  o.n_cells = uint32_t(t.size());
  o.max_depth = depth;
  o.budget_exhausted = t.exhausted ? 1u : 0u;
  if (total_finite == 0) {  // AllSamplesNonFinite, src/estimator.cpp:299-306
    o.status = MCB_TRIAL_ALL_NONFINITE;
  } else {
    o.status = MCB_TRIAL_OK;
    o.value = value;
    o.std_error = std::sqrt(var);
    o.nonfinite_warning = double(n_nonfinite) > MCB_NONFINITE_WARN_FRACTION * double(n_samples) ? 1u : 0u;
  }
  if (t.task->leaves) {  // leaves_out is written only when tree_refine returns
    t.task->leaves->clear();
    if (o.status != MCB_TRIAL_OK) return;
    t.task->leaves->reserve(t.size());
    for (size_t i = 0; i < t.size(); ++i) {
      mcb_leaf m;
      std::memset(&m, 0, sizeof m);
      std::memcpy(m.low, t.lo(i), sizeof(double) * t.dim);
      std::memcpy(m.high, t.hi(i), sizeof(double) * t.dim);
      m.estimate = t.est[i];
      m.depth = t.depth[i];
      t.task->leaves->push_back(m);
    }
  }
}

}  // namespace

Config config_of(const mcb_integrand& f) {
  Config c;
  c.init_cells_per_dim = f.cells_per_dim;
  if (f.flags & MCB_FLAG_REFINE_CONFIG) {
    c.samples_per_cell = f.samples_per_cell;
    c.max_depth = f.max_depth;
    c.sigma_multiplier = f.sigma_multiplier;
  }
  c.total_budget = f.n_samples;  // run_batch: rc.total_budget = spec.n_samples
  if (f.cell_cap) c.cell_cap = f.cell_cap;
  return c;
}

namespace {

// All rounds of one group of trees (tasks[0, n)).
mcb_status run_group(TreeTask* tasks, size_t n, const CellRunner& run, unsigned threads) {
  std::vector<Tree> trees(n);
  Pool pool(threads);
  // First pass (src/estimator.cpp:215-263): grid size, then every grid cell.
  pool.run(n, [&](size_t i) {
    Tree& t = trees[i];
    t.task = &tasks[i];
    t.cfg = config_of(*tasks[i].fn);
    t.dim = tasks[i].fn->dim;
    t.spc = std::max<uint32_t>(t.cfg.samples_per_cell, 2);
    t.cpc = chunk_count(t.spc);
    t.next_chunk = tasks[i].chunk_base;
    uint32_t k = t.cfg.init_cells_per_dim;
    uint64_t n_cells = 0;
    bool ok = true;
    if (k == 0) {
      k = auto_cells_per_dim(t.dim, 4096);
      while (k > 1) {  // keep the first pass cheap relative to the budget
        uint64_t cells;
        if (!cell_grid_size(k, t.dim, t.cfg.cell_cap, cells)) {
          ok = false;
          break;
        }
        if (cells * t.spc <= t.cfg.total_budget / 2) break;
        --k;
      }
    }
    if (!ok || !cell_grid_size(k, t.dim, t.cfg.cell_cap, n_cells)) {
      t.fail = MCB_TRIAL_CELL_BUDGET;
      t.active = false;
      return;
    }
    // leaves never exceed the first pass plus two per affordable split
    const uint64_t cap_leaves =
        std::min<uint64_t>(n_cells + 2 * (t.cfg.total_budget / (2ull * t.spc)) + 1, uint64_t(1) << 20);
    t.rect.reserve(cap_leaves * 2 * t.dim);
    t.se.reserve(cap_leaves);
    t.depth.reserve(cap_leaves);
    t.est.reserve(cap_leaves);
    t.rect.resize(n_cells * 2 * t.dim);
    t.se.assign(n_cells, 0.0);
    t.depth.assign(n_cells, 0u);
    t.est.resize(n_cells);
    const mcb_integrand& f = *tasks[i].fn;
    for (uint64_t c = 0; c < n_cells; ++c) {
      double* lo = t.lo(c);
      double* hi = t.hi(c);
      // grid_cell, src/estimator.cpp:124-143 (axis 0 most significant)
      uint64_t rem = c;
      for (uint32_t j = t.dim; j-- > 0;) {
        const uint32_t digit = uint32_t(rem % k);
        rem /= k;
        const double width = f.high[j] - f.low[j];
        lo[j] = digit == 0 ? f.low[j] : f.low[j] + width * (double(digit) / k);
        hi[j] = digit + 1 == k ? f.high[j] : f.low[j] + width * (double(digit + 1) / k);
      }
    }
    t.r_leaf.reserve(n_cells);
    t.r_rects.reserve(n_cells * 2 * t.dim);
    for (uint64_t c = 0; c < n_cells && t.fail == MCB_TRIAL_OK; ++c) estimate_cell(t, c);
  });
  mcb_status st = run_round(trees, run, pool);
  if (st != MCB_OK) return st;
  std::vector<uint32_t> active;
  for (;;) {
    active.clear();
    for (size_t i = 0; i < trees.size(); ++i)
      if (trees[i].active) active.push_back(uint32_t(i));
    if (active.empty()) break;
    pool.run(active.size(), [&](size_t k) {
      thread_local std::vector<uint32_t> selected;
      refine_step(trees[active[k]], selected);
    });
    if ((st = run_round(trees, run, pool)) != MCB_OK) return st;
  }
  pool.run(trees.size(), [&](size_t i) { finish(trees[i]); });
  return MCB_OK;
}

}  // namespace

// Large batches run as a few groups of trees on their own host threads:
// while one group's cells are on the GPU (the runner serialises device work
// per device), the others do their host work (selection, splits, results),
// so host and device time overlap.  Each tree is computed exactly as alone.
#ifndef MCB_TREE_GROUPS
#define MCB_TREE_GROUPS 4
#endif
constexpr size_t kTreeGroups = MCB_TREE_GROUPS;
mcb_status run_trees(std::vector<TreeTask>& tasks, const CellRunner& run) {
  const size_t n = tasks.size();
  const unsigned threads = host_threads(n);
  const size_t groups = std::min<size_t>(kTreeGroups, std::max<size_t>(1, n / 256));
  if (groups == 1) return run_group(tasks.data(), n, run, threads);
  std::vector<mcb_status> st(groups, MCB_OK);
  std::vector<std::thread> pool;
  for (size_t g = 0; g < groups; ++g) {
    const size_t b = n * g / groups, e = n * (g + 1) / groups;
    const unsigned t = std::max(1u, unsigned(threads / groups));
    pool.emplace_back([&, g, b, e, t] { st[g] = run_group(tasks.data() + b, e - b, run, t); });
  }
  for (auto& th : pool) th.join();
  for (mcb_status s : st)
    if (s != MCB_OK) return s;
  return MCB_OK;
}

}  // namespace mcb::tree
