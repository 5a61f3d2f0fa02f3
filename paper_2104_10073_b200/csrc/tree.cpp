// tree.cpp — lock-step host driver of tree_refine (ref src/estimator.cpp:
// 184-318) over many trees; see tree.hpp.  Every floating-point step of the
// selection (mean / sd of the leaf std_errors, threshold), the split
// (longest edge, midpoint low + 0.5*(high-low)) and the final combine_cells
// (src/estimator.cpp:145-159) is the reference's, in its order, built with
// -ffp-contract=off.  Only the cell estimates come from the GPU.
#include "tree.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

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

struct Leaf {
  double low[MCB_MAX_DIM];
  double high[MCB_MAX_DIM];
  mcb_trial_stats est;
  uint32_t depth;
};

struct Tree {
  TreeTask* task;
  Config cfg;
  uint32_t dim;
  uint32_t spc;
  uint64_t cpc;
  std::vector<Leaf> leaves;
  uint64_t next_chunk;
  uint64_t used = 0;
  bool exhausted = false;
  bool active = true;
  uint32_t fail = MCB_TRIAL_OK;  // CELL_BUDGET / CHUNK_RANGE: the tree threw
  // this round's cells: leaf index, rectangle, estimate; chunk of the first
  std::vector<size_t> r_leaf;
  std::vector<double> r_rects;
  std::vector<mcb_trial_stats> r_est;
  uint64_t r_chunk0 = 0;
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
  t.r_leaf.push_back(leaf);
  const Leaf& l = t.leaves[leaf];
  t.r_rects.insert(t.r_rects.end(), l.low, l.low + t.dim);
  t.r_rects.insert(t.r_rects.end(), l.high, l.high + t.dim);
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
mcb_status run_round(std::vector<Tree>& trees, const CellRunner& run) {
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
    t.r_est.assign(t.r_leaf.size(), mcb_trial_stats{});
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
  for (Tree* t : owner) {
    for (size_t i = 0; i < t->r_leaf.size(); ++i) {
      mcb_trial_stats& e = t->leaves[t->r_leaf[i]].est;
      if (t->r_est[i].status == MCB_TRIAL_OK) {
        e = t->r_est[i];
        e.n_cells = 1;
        e.budget_exhausted = 0;
        e.max_depth = 0;
      } else {
        e = dead_leaf(t->spc);
      }
    }
    t->r_leaf.clear();
    t->r_rects.clear();
  }
  return MCB_OK;
}

// split_longest_edge, src/estimator.cpp:192-210: first axis of maximal width.
void split_longest_edge(const Leaf& cell, uint32_t d, Leaf& lo, Leaf& hi) {
  uint32_t axis = 0;
  double best = -1.0;
  for (uint32_t j = 0; j < d; ++j) {
    const double w = cell.high[j] - cell.low[j];
    if (w > best) {
      best = w;
      axis = j;
    }
  }
  const double mid = cell.low[axis] + 0.5 * (cell.high[axis] - cell.low[axis]);
  lo = cell;
  hi = cell;
  lo.high[axis] = mid;
  hi.low[axis] = mid;
}

// One refinement step of the `while (!exhausted)` loop, src/estimator.cpp:265-297.
void refine_step(Tree& t) {
  const size_t n = t.leaves.size();
  double mean_err = 0.0;
  for (const Leaf& l : t.leaves) mean_err += l.est.std_error;
  mean_err /= double(n);
  double ss = 0.0;
  for (const Leaf& l : t.leaves) {
    const double dlt = l.est.std_error - mean_err;
    ss += dlt * dlt;
  }
  const double sd = n > 1 ? std::sqrt(ss / double(n - 1)) : 0.0;
  const double threshold = mean_err + t.cfg.sigma_multiplier * sd;

  std::vector<size_t> selected;
  for (size_t i = 0; i < n; ++i)
    if (t.leaves[i].depth < t.cfg.max_depth && t.leaves[i].est.std_error > 0 &&
        t.leaves[i].est.std_error > threshold)
      selected.push_back(i);
  if (selected.empty()) {
    t.active = false;
    return;
  }
  for (size_t idx : selected) {
    if (t.used + 2ull * t.spc > t.cfg.total_budget) {
      t.exhausted = true;
      break;
    }
    Leaf lo, hi;
    split_longest_edge(t.leaves[idx], t.dim, lo, hi);
    lo.depth = hi.depth = t.leaves[idx].depth + 1;
    t.leaves[idx] = lo;  // the lower half replaces the parent in place
    t.leaves.push_back(hi);
    const size_t hi_idx = t.leaves.size() - 1;
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
  for (const Leaf& l : t.leaves) {
    value += l.est.value;
    var += l.est.std_error * l.est.std_error;
    n_samples += l.est.n_samples;
    n_nonfinite += l.est.n_nonfinite;
    total_finite += l.est.n_samples - l.est.n_nonfinite;
    depth = std::max(depth, l.depth);
  }
  o.n_samples = n_samples;
  o.n_nonfinite = n_nonfinite;
  o.n_cells = uint32_t(t.leaves.size());
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
    t.task->leaves->reserve(t.leaves.size());
    for (const Leaf& l : t.leaves) {
      mcb_leaf m;
      std::memset(&m, 0, sizeof m);
      std::memcpy(m.low, l.low, sizeof m.low);
      std::memcpy(m.high, l.high, sizeof m.high);
      m.estimate = l.est;
      m.depth = l.depth;
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

mcb_status run_trees(std::vector<TreeTask>& tasks, const CellRunner& run) {
  std::vector<Tree> trees(tasks.size());
  // First pass (src/estimator.cpp:215-263): grid size, then every grid cell.
  for (size_t i = 0; i < tasks.size(); ++i) {
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
      continue;
    }
    t.leaves.resize(n_cells);
    const mcb_integrand& f = *tasks[i].fn;
    for (uint64_t c = 0; c < n_cells; ++c) {
      Leaf& l = t.leaves[c];
      std::memset(&l, 0, sizeof l);
      // grid_cell, src/estimator.cpp:124-143 (axis 0 most significant)
      uint64_t rem = c;
      for (uint32_t j = t.dim; j-- > 0;) {
        const uint32_t digit = uint32_t(rem % k);
        rem /= k;
        const double width = f.high[j] - f.low[j];
        l.low[j] = digit == 0 ? f.low[j] : f.low[j] + width * (double(digit) / k);
        l.high[j] = digit + 1 == k ? f.high[j] : f.low[j] + width * (double(digit + 1) / k);
      }
    }
    t.r_leaf.reserve(n_cells);
    t.r_rects.reserve(n_cells * 2 * t.dim);
    for (uint64_t c = 0; c < n_cells && t.fail == MCB_TRIAL_OK; ++c) estimate_cell(t, c);
  }
  mcb_status st = run_round(trees, run);
  if (st != MCB_OK) return st;
  for (;;) {
    bool any = false;
    for (Tree& t : trees)
      if (t.active) {
        refine_step(t);
        any = true;
      }
    if (!any) break;
    if ((st = run_round(trees, run)) != MCB_OK) return st;
  }
  for (Tree& t : trees) finish(t);
  return MCB_OK;
}

}  // namespace mcb::tree
