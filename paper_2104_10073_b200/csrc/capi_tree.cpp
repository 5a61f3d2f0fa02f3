// capi_tree.cpp — the tree method's runners: device-resident rounds
// (tree_device.cuh, the default), the cell-batch runner of the host driver
// (tree.cpp) and the dispatcher between them; stratified_mc and
// tree_refine of the C-ABI run through here.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <thread>
#include <tuple>

#include "capi_internal.hpp"

namespace mcb {
namespace capi {

// One device's share of a tree round: a cell-list descriptor per batch
// (prepared as the tree's integrand, cells from the rectangle table), the
// fused kernels in cell-list mode, per-cell estimates back to the batches.
mcb_status run_cell_shard(const std::vector<const mcb::tree::CellBatch*>& batches, uint64_t seed,
                          int device) {
  const size_t n = batches.size();
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  HostPlan hp;
  std::vector<Prepared> prep(n);
  size_t n_rects = 0, n_cells = 0;
  std::map<const mcb_integrand*, Prepared> base;  // one prepare per integrand (its trials share it)
  for (size_t i = 0; i < n; ++i) {
    const mcb::tree::CellBatch& b = *batches[i];
    auto it = base.find(b.fn);
    if (it == base.end()) it = base.emplace(b.fn, prepare(*b.fn, seed, 0, 0, true)).first;
    prep[i] = it->second;
    prep[i].d.chunk_base = uint32_t(b.chunk_base);
    prep[i].d.trial_base = b.trial;
    if (b.spc <= mcb::detail::kWarpTileMaxSpc) prep[i].variant |= mcb::detail::kWarpTile;
    n_rects += size_t(b.n_cells) * 2 * b.fn->dim;
    n_cells += b.n_cells;
  }
  std::vector<size_t> order(n);
  std::iota(order.begin(), order.end(), size_t(0));
  auto prog_key = [&](size_t i) {
    return batches[i]->fn->family == MCB_FAMILY_PROGRAM ? reinterpret_cast<uintptr_t>(batches[i]->fn->program)
                                                        : uintptr_t(0);
  };
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
    return std::make_tuple(batches[x]->fn->family, batches[x]->fn->dim, prep[x].variant, prog_key(x)) <
           std::make_tuple(batches[y]->fn->family, batches[y]->fn->dim, prep[y].variant, prog_key(y));
  });
  uint64_t tiles = 0;  // upper bound incl. warp-tile padding and alignment
  for (size_t i = 0; i < n; ++i)
    tiles += uint64_t(batches[i]->n_cells) * chunk_count(batches[i]->spc) + 2 * mcb::detail::kTileAlign;

  DeviceCtx& c = device_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  DeviceGuard guard(device);
  cudaError_t e;
  if (!c.ready) {
    if ((e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
    c.ready = true;
  }
  // program tables first (sizes), then buffers, then descriptors with device addresses
  std::map<const mcb_program*, std::pair<uint32_t, uint32_t>> prog_at;
  for (size_t i = 0; i < n; ++i) {
    const mcb_program* pg = batches[i]->fn->program;
    if (batches[i]->fn->family != MCB_FAMILY_PROGRAM || prog_at.count(pg)) continue;
    prog_at.emplace(pg, std::make_pair(uint32_t(hp.code.size()), uint32_t(hp.consts.size())));
    hp.code.insert(hp.code.end(), pg->words.begin(), pg->words.end());
    hp.consts.insert(hp.consts.end(), pg->p.consts.begin(), pg->p.consts.end());
  }
  if ((e = c.buf.reserve(n, tiles, n, hp.code.size(), hp.consts.size())) != cudaSuccess ||
      (e = DevBuf::grow(c.buf.rects, c.buf.cap_rects, n_rects)) != cudaSuccess ||
      (e = DevBuf::grow(c.buf.cell_est, c.buf.cap_cell_est, n_cells)) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc");
  if ((e = grow_pinned(c.h_descs, c.h_descs_cap, n)) != cudaSuccess ||
      (e = grow_pinned(c.h_rects, c.h_rects_cap, n_rects)) != cudaSuccess ||
      (e = grow_pinned(c.h_cell_est, c.h_cell_est_cap, n_cells)) != cudaSuccess)
    return cuda_fail(e, "cudaMallocHost");
  hp.descs.resize(n);
  std::vector<size_t> est_at(n);
  uint64_t tile = 0;
  size_t rect_at = 0, cell_at = 0;
  for (size_t r = 0; r < n; ++r) {
    const size_t i = order[r];
    const mcb::tree::CellBatch& b = *batches[i];
    FnDesc d = prep[i].d;
    d.strat_k = 0;
    d.n_cells = b.n_cells;
    d.spc = b.spc;
    d.cpc = uint32_t(chunk_count(b.spc));
    d.n_chunks = d.n_cells * d.cpc;
    d.n_samples = uint64_t(b.n_cells) * b.spc;
    if (prep[i].variant & mcb::detail::kWarpTile) {
      d.n_chunks = round_up<uint32_t>(d.n_chunks, mcb::detail::kTileAlign);
      tile = round_up<uint64_t>(tile, mcb::detail::kTileAlign);
    }
    d.tile_base = tile;
    d.out_slot = r;
    d.cell_rects = c.buf.rects + rect_at;
    d.cell_est = c.buf.cell_est + cell_at;
    const size_t nr = size_t(b.n_cells) * 2 * b.fn->dim;
    std::memcpy(c.h_rects + rect_at, b.rects, sizeof(double) * nr);
    est_at[i] = cell_at;
    rect_at += nr;
    cell_at += b.n_cells;
    const int fam = int(b.fn->family), dim = int(b.fn->dim), var = prep[i].variant;
    uint32_t slots = 0;
    if (fam == MCB_FAMILY_PROGRAM) {
      const auto& at = prog_at.at(b.fn->program);
      d.prog_off = at.first;
      d.prog_len = uint32_t(b.fn->program->p.code.size());
      d.const_off = at.second;
      d.n_consts = uint32_t(b.fn->program->p.consts.size());
      slots = b.fn->program->p.depth;
    }
    const mcb::prog::Program* gp = fam == MCB_FAMILY_PROGRAM ? &b.fn->program->p : nullptr;
    if (hp.groups.empty() || hp.groups.back().family != fam || hp.groups.back().dim != dim ||
        hp.groups.back().variant != var || hp.groups.back().prog != gp) {
      hp.groups.push_back(GroupLaunch{fam, dim, var, tile, 0, 0, gp});
      hp.groups.back().tile_samples = 0;
    }
    hp.groups.back().tile_samples = std::max(hp.groups.back().tile_samples, std::min<uint32_t>(b.spc, MCB_CHUNK_SIZE));
    hp.groups.back().n_tiles += d.n_chunks;
    hp.groups.back().slots = std::max(hp.groups.back().slots, slots);
    tile += d.n_chunks;
    hp.descs[r] = d;
  }
  hp.n_tiles = tile;
  for (const auto& g : hp.groups)
    if (g.family != MCB_FAMILY_PROGRAM && !mcb::detail::variant_supported(g.family, g.dim, g.variant))
      return fail(MCB_ERR_INVALID_ARGUMENT, "unsupported (family, dim) combination");
  std::memcpy(c.h_descs, hp.descs.data(), sizeof(FnDesc) * n);
  const auto t_host = clk::now();
  if (n_rects &&
      (e = cudaMemcpyAsync(c.buf.rects, c.h_rects, sizeof(double) * n_rects, cudaMemcpyHostToDevice,
                           c.stream)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(cells)");
  mcb_status st = enqueue_run(hp, c.buf, 1, c.h_descs, true, c.stream);
  if (st != MCB_OK) return st;
  if ((e = cudaMemcpyAsync(c.h_cell_est, c.buf.cell_est, sizeof(mcb::CellEst) * n_cells,
                           cudaMemcpyDeviceToHost, c.stream)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(cell estimates)");
  if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  const auto t_gpu = clk::now();
  for (size_t i = 0; i < n; ++i)
    std::memcpy(batches[i]->est, c.h_cell_est + est_at[i], sizeof(mcb::CellEst) * batches[i]->n_cells);
  static const bool trace = [] {
    const char* env = std::getenv("MCB_TREE_TRACE");
    return env && *env && *env != '0';
  }();
  if (trace) {
    auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[mcb cells] dev %d: %zu batches, %zu cells: host %.3f ms, H2D+kernels+D2H %.3f ms, scatter %.3f ms\n",
                 device, n, n_cells, ms(t_start, t_host), ms(t_host, t_gpu), ms(t_gpu, clk::now()));
  }
  return MCB_OK;
}

// tree_refine's first-pass grid (src/estimator.cpp:219-231): cells per dim
// and cell count; false = CellBudgetExceeded.
bool tree_first_pass(const mcb_integrand& f, const mcb::tree::Config& cfg, uint32_t spc, uint32_t& k,
                     uint64_t& n0) {
  k = cfg.init_cells_per_dim;
  if (k == 0) {
    // the reference steps k down from the automatic size until the grid
    // takes at most half the budget (stopping at 1), every step through the
    // cell cap; k^d falls with k, so only the first step can hit the cap and
    // the stop is the largest k with k^d <= (budget/2)/spc
    k = auto_cells_per_dim(f.dim, 4096);
    if (k > 1) {
      uint64_t cells;
      if (!cell_grid_size(k, f.dim, cfg.cell_cap, cells)) return false;
      k = std::min(k, int_root_floor(cfg.total_budget / 2 / spc, f.dim));
    }
  }
  return cell_grid_size(k, f.dim, cfg.cell_cap, n0);
}

// Most leaves a tree can reach: one per split the budget allows past the
// first pass, and at most 2^max_depth per first-pass cell.
uint64_t tree_leaf_bound(uint64_t n0, uint32_t spc, const mcb::tree::Config& cfg) {
  const uint64_t first = n0 * spc;
  const uint64_t splits = cfg.total_budget >= first ? (cfg.total_budget - first) / (2ull * spc) : 0;
  const uint64_t by_depth = cfg.max_depth >= 40 ? ~0ull : n0 << cfg.max_depth;
  return std::min(n0 + splits, std::max(n0, by_depth));
}

// Device-resident tree_refine for `tasks` on one device (tree_device.cuh):
// the host builds each tree's first-pass grid and constants once; every
// round then runs on the GPU with one small read-back (the launch groups'
// tile ranges).  Results are those of the host driver (tree.cpp).
mcb_status run_trees_device(std::vector<mcb::tree::TreeTask*>& tasks, uint64_t seed, int device) {
  using namespace mcb::detail;
  using tclk = std::chrono::steady_clock;
  const auto t_start = tclk::now();
  static const bool trace = [] {
    const char* v = std::getenv("MCB_TREE_TRACE");
    return v && *v && *v != '0';
  }();
  using mcb::tdev::TreeConst;
  using mcb::tdev::TreeState;
  const size_t T = tasks.size();
  if (T == 0) return MCB_OK;
  // ---- host: configs, first-pass grids, descriptors, launch groups ----
  struct HostTree {  // per distinct integrand: its trials share config, grid and descriptor
    mcb::tree::Config cfg;
    uint32_t k = 0, spc = 0, cpc = 0, fail = 0;
    uint64_t n0 = 0, cap = 0;
    Prepared prep;
  };
  struct TrialOf {  // per tree: its integrand's HostTree and its own first-pass outcome
    size_t base;
    uint32_t fail;
    uint64_t n0, cap;
  };
  std::vector<HostTree> ht;
  std::vector<TrialOf> tr(T);
  std::map<const mcb_integrand*, size_t> first_of;
  for (size_t i = 0; i < T; ++i) {
    const mcb_integrand& f = *tasks[i]->fn;
    // an integrand's trials are usually adjacent: skip the map look-up for them
    size_t seen_base = i > 0 && tasks[i - 1]->fn == tasks[i]->fn ? tr[i - 1].base : SIZE_MAX;
    if (seen_base == SIZE_MAX) {
      auto seen = first_of.find(tasks[i]->fn);
      if (seen != first_of.end()) seen_base = seen->second;
    }
    if (seen_base != SIZE_MAX) {
      const HostTree& h = ht[seen_base];
      tr[i] = TrialOf{seen_base, h.fail, h.n0, h.cap};
      if (!h.fail && tasks[i]->chunk_base + h.n0 * h.cpc - 1 > 0xFFFFFFFFull)
        tr[i] = TrialOf{seen_base, MCB_TRIAL_CHUNK_RANGE, 0, tree_leaf_bound(0, h.spc, h.cfg) + 1};
      continue;
    }
    first_of.emplace(tasks[i]->fn, ht.size());
    ht.emplace_back();
    HostTree& h = ht.back();
    h.cfg = mcb::tree::config_of(f);
    h.spc = std::max<uint32_t>(h.cfg.samples_per_cell, 2);
    h.cpc = uint32_t(chunk_count(h.spc));
    uint32_t k = 0;
    if (!tree_first_pass(f, h.cfg, h.spc, k, h.n0)) {
      h.fail = MCB_TRIAL_CELL_BUDGET;
      h.n0 = 0;
    } else if (tasks[i]->chunk_base + h.n0 * h.cpc - 1 > 0xFFFFFFFFull) {
      h.fail = MCB_TRIAL_CHUNK_RANGE;
      h.n0 = 0;
    }
    h.k = k;
    h.cap = tree_leaf_bound(h.n0, h.spc, h.cfg) + 1;
    if (h.cap > 0xFFFFFFFFull) return fail(MCB_ERR_INVALID_ARGUMENT, "tree budget too large for one device run");
    h.prep = prepare(f, seed, 0, tasks[i]->trial, true);
    if (h.spc <= kWarpTileMaxSpc) h.prep.variant |= kWarpTile;
    tr[i] = TrialOf{ht.size() - 1, h.fail, h.n0, h.cap};
  }
  const auto t_cfg = tclk::now();
  std::vector<size_t> order(T);  // launch groups: (family, dim, variant, program)
  std::iota(order.begin(), order.end(), size_t(0));
  using Key = std::tuple<uint32_t, uint32_t, int, uintptr_t>;
  std::vector<Key> keys(T);
  for (size_t i = 0; i < T; ++i) {
    const mcb_integrand& f = *tasks[i]->fn;
    keys[i] = Key(f.family, f.dim, ht[tr[i].base].prep.variant,
                  f.family == MCB_FAMILY_PROGRAM ? reinterpret_cast<uintptr_t>(f.program) : uintptr_t(0));
  }
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return keys[a] < keys[b]; });
  // per-thread scratch reused across calls: fresh vectors of this size are
  // mmap'ed and page-faulted in on every call
  thread_local HostPlan hp;
  thread_local std::vector<TreeConst> tc;
  thread_local std::vector<TreeState> tst;
  hp.groups.clear();
  hp.code.clear();
  hp.consts.clear();
  tc.resize(T);
  tst.resize(T);
  std::map<const mcb_program*, std::pair<uint32_t, uint32_t>> prog_at;
  const mcb_program* last_prog = nullptr;
  std::pair<uint32_t, uint32_t> last_at{0, 0};
  uint64_t leaves = 0, rect_doubles = 0, max_tiles = 0;
  hp.descs.resize(T);
  for (size_t r = 0; r < T; ++r) {
    const size_t i = order[r];
    const mcb_integrand& f = *tasks[i]->fn;
    const HostTree& h = ht[tr[i].base];
    const TrialOf& t = tr[i];
    const int fam = int(f.family), dim = int(f.dim), var = h.prep.variant;
    const mcb::prog::Program* gp = fam == MCB_FAMILY_PROGRAM ? &f.program->p : nullptr;
    if (hp.groups.empty() || hp.groups.back().family != fam || hp.groups.back().dim != dim ||
        hp.groups.back().variant != var || hp.groups.back().prog != gp) {
      hp.groups.push_back(GroupLaunch{fam, dim, var, 0, 0, 0, gp});
      hp.groups.back().tile_samples = 0;
    }
    hp.groups.back().tile_samples = std::max(hp.groups.back().tile_samples, std::min<uint32_t>(h.spc, MCB_CHUNK_SIZE));
    FnDesc& d = hp.descs[r];
    d = h.prep.d;
    d.trial_base = tasks[i]->trial;
    d.strat_k = 0;
    d.spc = h.spc;
    d.cpc = h.cpc;
    d.out_slot = r;
    if (fam == MCB_FAMILY_PROGRAM) {
      if (f.program != last_prog) {  // trees of one program are adjacent after the sort
        auto it = prog_at.find(f.program);
        if (it == prog_at.end()) {
          it = prog_at.emplace(f.program, std::make_pair(uint32_t(hp.code.size()), uint32_t(hp.consts.size()))).first;
          hp.code.insert(hp.code.end(), f.program->words.begin(), f.program->words.end());
          hp.consts.insert(hp.consts.end(), f.program->p.consts.begin(), f.program->p.consts.end());
        }
        last_prog = f.program;
        last_at = it->second;
      }
      d.prog_off = last_at.first;
      d.prog_len = uint32_t(f.program->p.code.size());
      d.const_off = last_at.second;
      d.n_consts = uint32_t(f.program->p.consts.size());
      hp.groups.back().slots = std::max(hp.groups.back().slots, f.program->p.depth);
    }
    TreeConst& c = tc[r];
    c.leaf_off = leaves;
    c.rect_off = rect_doubles;
    c.budget = h.cfg.total_budget;
    c.sigma = h.cfg.sigma_multiplier;
    c.leaf_cap = uint32_t(t.cap);
    c.dim = f.dim;
    c.spc = h.spc;
    c.cpc = h.cpc;
    c.max_depth = h.cfg.max_depth;
    c.warp_tiles = (var & kWarpTile) ? 1u : 0u;
    c.group = uint32_t(hp.groups.size() - 1);
    c.reserved = 0;
    TreeState& st = tst[r];
    std::memset(&st, 0, sizeof st);
    st.fail = t.fail;
    st.n_leaves = uint32_t(t.n0);
    st.n_new = uint32_t(t.n0);
    st.active = t.fail ? 0u : 1u;
    st.chunk0 = tasks[i]->chunk_base;
    st.next_chunk = tasks[i]->chunk_base + t.n0 * h.cpc;
    st.used = t.n0 * h.spc;
    leaves += t.cap;
    rect_doubles += t.cap * 2 * f.dim;
    max_tiles += (t.cap * h.cpc + kTileAlign - 1) / kTileAlign * kTileAlign;
  }
  max_tiles += kTileAlign * hp.groups.size();
  if (hp.groups.size() > 256) return fail(MCB_ERR_INVALID_ARGUMENT, "too many distinct tree kernels in one run");
  for (const auto& g : hp.groups)
    if (g.family != MCB_FAMILY_PROGRAM && !variant_supported(g.family, g.dim, g.variant))
      return fail(MCB_ERR_INVALID_ARGUMENT, "unsupported (family, dim) combination");
  // first-pass grids (grid_cell, src/estimator.cpp:124-143) = the initial
  // leaves and round-0 cells: one packed grid per integrand (its trials share
  // it), k_tree_init spreads them into every tree's storage
  uint64_t packed_doubles = 0;
  std::map<const mcb_integrand*, uint64_t> grid_at;  // packed offset of an integrand's grid
  std::vector<size_t> grid_rows;                      // one tree per distinct grid
  const mcb_integrand* last_fn = nullptr;
  uint64_t last_off = 0;
  for (size_t r = 0; r < T; ++r) {
    tc[r].init_off = 0;
    if (tst[r].n_leaves == 0) continue;  // failed before the first pass
    const mcb_integrand* fn = tasks[order[r]]->fn;
    if (fn != last_fn) {  // trials of one integrand are adjacent after the (stable) sort
      auto it = grid_at.find(fn);
      if (it == grid_at.end()) {
        it = grid_at.emplace(fn, packed_doubles).first;
        packed_doubles += uint64_t(tst[r].n_leaves) * 2 * tc[r].dim;
        grid_rows.push_back(r);
      }
      last_fn = fn;
      last_off = it->second;
    }
    tc[r].init_off = last_off;
  }
  const auto t_desc = tclk::now();
  DeviceCtx& c = device_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  DeviceGuard guard(device);
  cudaError_t e;
  if ((e = grow_pinned(c.h_rects, c.h_rects_cap, packed_doubles)) != cudaSuccess)
    return cuda_fail(e, "cudaMallocHost");
  for (size_t r : grid_rows) {
    const size_t i = order[r];
    const mcb_integrand& f = *tasks[i]->fn;
    const uint32_t k = ht[tr[i].base].k, D = f.dim;
    for (uint64_t cell = 0; cell < tst[r].n_leaves; ++cell) {
      double* lo = c.h_rects + tc[r].init_off + 2 * D * cell;
      double* hi = lo + D;
      uint64_t rem = cell;
      for (uint32_t j = D; j-- > 0;) {
        const uint32_t digit = uint32_t(rem % k);
        rem /= k;
        const double width = f.high[j] - f.low[j];
        lo[j] = digit == 0 ? f.low[j] : f.low[j] + width * (double(digit) / k);
        hi[j] = digit + 1 == k ? f.high[j] : f.low[j] + width * (double(digit + 1) / k);
      }
    }
  }
  const auto t_grid = tclk::now();
  // ---- device ----
  if (!c.ready) {
    if ((e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
    c.ready = true;
  }
  const cudaStream_t s = c.stream;
  if ((e = c.buf.reserve(T, max_tiles, T, hp.code.size(), hp.consts.size())) != cudaSuccess ||
      (e = DevBuf::grow(c.t_const, c.cap_trees, T)) != cudaSuccess ||
      (e = DevBuf::grow(c.t_state, c.cap_tstate, T)) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc");
  if ((e = DevBuf::grow(c.t_groups, c.cap_tgroups, 2 * hp.groups.size())) != cudaSuccess ||
      (e = DevBuf::grow(c.l_rect, c.cap_rect, rect_doubles)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_new_rect, c.cap_new_rect, rect_doubles)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_se, c.cap_se, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_val, c.cap_val, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_nn, c.cap_nn, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_depth, c.cap_depth, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_dead, c.cap_dead, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_new_leaf, c.cap_new_leaf, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_est, c.cap_est, leaves)) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc");
  mcb::tdev::Leaves L{c.l_rect, c.l_se, c.l_val, c.l_nn, c.l_depth, c.l_dead, c.l_new_leaf, c.l_new_rect, c.l_est};
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
  };
  // descriptors through the context's pinned staging (a pageable copy is a
  // synchronous bounce-buffer transfer)
  if ((e = grow_pinned(c.h_descs, c.h_descs_cap, T)) != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
  std::memcpy(c.h_descs, hp.descs.data(), sizeof(FnDesc) * T);
  if ((e = up(c.t_const, tc.data(), sizeof(TreeConst) * T)) != cudaSuccess ||
      (e = up(c.t_state, tst.data(), sizeof(TreeState) * T)) != cudaSuccess ||
      (e = up(c.buf.fns, c.h_descs, sizeof(FnDesc) * T)) != cudaSuccess ||
      (e = DevBuf::grow(c.buf.rects, c.buf.cap_rects, packed_doubles)) != cudaSuccess ||
      (e = up(c.buf.rects, c.h_rects, sizeof(double) * packed_doubles)) != cudaSuccess ||
      (e = launch_tree_init(c.t_const, c.t_state, L, c.buf.rects, uint32_t(T), s)) != cudaSuccess ||
      (!hp.code.empty() && (e = up(c.buf.code, hp.code.data(), sizeof(uint32_t) * hp.code.size())) != cudaSuccess) ||
      (!hp.consts.empty() && (e = up(c.buf.consts, hp.consts.data(), sizeof(double) * hp.consts.size())) != cudaSuccess))
    return cuda_fail(e, "cudaMemcpyAsync(tree setup)");
  prepare_programs(hp, false);
  const auto t_setup = tclk::now();
  int rounds = 0;
  std::vector<uint64_t> gt(2 * hp.groups.size());
  for (int round = 0;; ++round) {
    if (round > 0 && (e = launch_tree_select(c.t_const, c.t_state, L, uint32_t(T), s)) != cudaSuccess)
      return cuda_fail(e, "launch k_tree_select");
    if ((e = launch_tree_layout(c.t_const, c.t_state, c.buf.fns, L, uint32_t(T), c.t_groups,
                                uint32_t(hp.groups.size()), s)) != cudaSuccess)
      return cuda_fail(e, "launch k_tree_layout");
    if ((e = cudaMemcpyAsync(gt.data(), c.t_groups, sizeof(uint64_t) * gt.size(), cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
      return cuda_fail(e, "tree round read-back");
    uint64_t tiles = 0;
    for (size_t g = 0; g < hp.groups.size(); ++g) tiles += gt[2 * g + 1];
    if (tiles == 0) break;
    ++rounds;
    if ((e = launch_expand_tiles(c.buf.fns, uint32_t(T), 1, c.buf.tile_fn, s)) != cudaSuccess)
      return cuda_fail(e, "launch k_expand_tiles");
    for (size_t g = 0; g < hp.groups.size(); ++g) {
      if (gt[2 * g + 1] == 0) continue;
      GroupLaunch gl = hp.groups[g];
      gl.tile0 = gt[2 * g];
      gl.n_tiles = gt[2 * g + 1];
      e = gl.family == MCB_FAMILY_PROGRAM
              ? launch_program_group(gl, c.buf.fns, c.buf.tile_fn, c.buf.part, c.buf.code, c.buf.consts, s)
              : launch_direct_group(gl, c.buf.fns, c.buf.tile_fn, c.buf.part, s);
      if (e != cudaSuccess) return cuda_fail(e, "launch tree cells");
    }
    if ((e = launch_combine(c.buf.fns, uint32_t(T), 1, c.buf.part, c.buf.out, s)) != cudaSuccess ||
        (e = launch_tree_scatter(c.t_const, c.t_state, L, uint32_t(T), s)) != cudaSuccess)
      return cuda_fail(e, "launch tree combine/scatter");
  }
  if (trace) {
    auto ms = [](tclk::time_point a, tclk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr,
                 "[mcb tree/dev %d] %zu trees: host setup %.3f ms (configs %.3f, descriptors %.3f, grids %.3f, "
                 "uploads %.3f), %d rounds %.3f ms\n",
                 device, T, ms(t_start, t_setup), ms(t_start, t_cfg), ms(t_cfg, t_desc), ms(t_desc, t_grid),
                 ms(t_grid, t_setup), rounds, ms(t_setup, tclk::now()));
  }
  if ((e = launch_tree_finish(c.t_const, c.t_state, L, uint32_t(T), c.buf.out, s)) != cudaSuccess)
    return cuda_fail(e, "launch k_tree_finish");
  std::vector<mcb_trial_stats> out(T);
  if ((e = cudaMemcpyAsync(out.data(), c.buf.out, sizeof(mcb_trial_stats) * T, cudaMemcpyDeviceToHost, s)) !=
      cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(tree results)");
  bool want_leaves = false;
  for (auto* t : tasks) want_leaves = want_leaves || t->leaves;
  std::vector<double> h_rect, h_se, h_val;
  std::vector<uint32_t> h_nn, h_depth, h_dead;
  if (want_leaves) {
    h_rect.resize(rect_doubles);
    h_se.resize(leaves);
    h_val.resize(leaves);
    h_nn.resize(leaves);
    h_depth.resize(leaves);
    h_dead.resize(leaves);
    if ((e = cudaMemcpyAsync(h_rect.data(), c.l_rect, sizeof(double) * rect_doubles, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h_se.data(), c.l_se, sizeof(double) * leaves, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(h_val.data(), c.l_val, sizeof(double) * leaves, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h_nn.data(), c.l_nn, sizeof(uint32_t) * leaves, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h_depth.data(), c.l_depth, sizeof(uint32_t) * leaves, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h_dead.data(), c.l_dead, sizeof(uint32_t) * leaves, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync(leaves)");
  }
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  for (size_t r = 0; r < T; ++r) {
    mcb::tree::TreeTask& task = *tasks[order[r]];
    *task.out = out[r];
    if (!task.leaves) continue;
    task.leaves->clear();
    if (out[r].status != MCB_TRIAL_OK) continue;  // leaves_out is written only when tree_refine returns
    const uint32_t D = task.fn->dim, spc = tc[r].spc;
    for (uint32_t i = 0; i < out[r].n_cells; ++i) {
      const uint64_t l = tc[r].leaf_off + i;
      mcb_leaf m;
      std::memset(&m, 0, sizeof m);
      std::memcpy(m.low, h_rect.data() + tc[r].rect_off + 2 * D * i, sizeof(double) * D);
      std::memcpy(m.high, h_rect.data() + tc[r].rect_off + 2 * D * i + D, sizeof(double) * D);
      m.depth = h_depth[l];
      mcb_trial_stats& est = m.estimate;
      est.n_samples = spc;
      est.n_nonfinite = h_nn[l];
      est.n_cells = 1;
      if (h_dead[l]) {
        est.status = MCB_TRIAL_ALL_NONFINITE;
        est.nonfinite_warning = 1;
      } else {
        est.value = h_val[l];
        est.std_error = h_se[l];
        est.nonfinite_warning = double(h_nn[l]) > MCB_NONFINITE_WARN_FRACTION * double(spc) ? 1u : 0u;
      }
      task.leaves->push_back(m);
    }
  }
  return MCB_OK;
}


// One tree round: batches sharded over `devs` by LPT on their sample cost.
mcb_status run_cells(const std::vector<mcb::tree::CellBatch>& batches, uint64_t seed,
                     const std::vector<int>& devs) {
  const size_t n = batches.size();
  std::vector<std::vector<const mcb::tree::CellBatch*>> shard(devs.size());
  if (devs.size() == 1) {
    for (const auto& b : batches) shard[0].push_back(&b);
  } else {
    std::vector<size_t> order(n);
    std::iota(order.begin(), order.end(), size_t(0));
    std::vector<double> cost(n);
    for (size_t i = 0; i < n; ++i)
      cost[i] = double(batches[i].n_cells) * double(batches[i].spc) * sample_cost(*batches[i].fn);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return cost[a] > cost[b]; });
    std::vector<double> load(devs.size(), 0.0);
    for (size_t i : order) {
      size_t best = 0;
      for (size_t w = 1; w < load.size(); ++w)
        if (load[w] < load[best]) best = w;
      shard[best].push_back(&batches[i]);
      load[best] += cost[i];
    }
  }
  std::vector<mcb_status> status(devs.size(), MCB_OK);
  std::vector<std::string> errors(devs.size());
  auto work = [&](size_t w) {
    if (shard[w].empty()) return;
    status[w] = run_cell_shard(shard[w], seed, devs[w]);
    if (status[w] != MCB_OK) errors[w] = g_last_error;
  };
  if (devs.size() == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (size_t w = 0; w < devs.size(); ++w) pool.emplace_back(work, w);
    for (auto& th : pool) th.join();
  }
  for (size_t w = 0; w < devs.size(); ++w)
    if (status[w] != MCB_OK) return fail(status[w], "device " + std::to_string(devs[w]) + ": " + errors[w]);
  return MCB_OK;
}

// Every tree of `tasks`, on `devs`: device-resident rounds (default; trees
// sharded over the devices by budget, each device independent), or the host
// driver over batched cell launches (MCB_TREE_DEVICE=0, kept as the
// cross-check of the device rounds: both give identical trees).
mcb_status run_trees_on(std::vector<mcb::tree::TreeTask>& tasks, uint64_t seed, const std::vector<int>& devs) {
  static const bool host_driven = [] {
    const char* e = std::getenv("MCB_TREE_DEVICE");
    return e && e[0] == '0';
  }();
  if (host_driven) {
    std::mutex err_mu;
    std::string err;
    const mcb_status st = mcb::tree::run_trees(tasks, [&](const std::vector<mcb::tree::CellBatch>& batches) {
      const mcb_status r = run_cells(batches, seed, devs);
      if (r != MCB_OK) {
        std::lock_guard<std::mutex> lk(err_mu);
        err = g_last_error;
      }
      return r;
    });
    return st == MCB_OK ? st : fail(st, err);
  }
  // leaf storage is reserved up front on the device: very large trees (a
  // budget / depth allowing > 64 Mi leaves in one call) take the host driver
  uint64_t bound = 0, last = 0;
  const mcb_integrand* last_fn = nullptr;
  for (auto& t : tasks) {  // the trials of an integrand are adjacent: one bound each
    if (t.fn != last_fn) {
      const mcb::tree::Config cfg = mcb::tree::config_of(*t.fn);
      const uint32_t spc = std::max<uint32_t>(cfg.samples_per_cell, 2);
      uint32_t k;
      uint64_t n0;
      last = tree_first_pass(*t.fn, cfg, spc, k, n0) ? tree_leaf_bound(n0, spc, cfg) : 0;
      last_fn = t.fn;
    }
    bound += last;
  }
  if (bound > (uint64_t(1) << 26)) {
    std::mutex err_mu;
    std::string err;
    const mcb_status st = mcb::tree::run_trees(tasks, [&](const std::vector<mcb::tree::CellBatch>& batches) {
      const mcb_status r = run_cells(batches, seed, devs);
      if (r != MCB_OK) {
        std::lock_guard<std::mutex> lk(err_mu);
        err = g_last_error;
      }
      return r;
    });
    return st == MCB_OK ? st : fail(st, err);
  }
  std::vector<std::vector<mcb::tree::TreeTask*>> shard(devs.size());
  std::vector<double> load(devs.size(), 0.0);
  for (auto& t : tasks) {  // greedy by budget (the trees' work bound)
    size_t best = 0;
    for (size_t w = 1; w < devs.size(); ++w)
      if (load[w] < load[best]) best = w;
    shard[best].push_back(&t);
    load[best] += double(t.fn->n_samples) * sample_cost(*t.fn);
  }
  std::vector<mcb_status> status(devs.size(), MCB_OK);
  std::vector<std::string> errors(devs.size());
  auto work = [&](size_t w) {
    status[w] = run_trees_device(shard[w], seed, devs[w]);
    if (status[w] != MCB_OK) errors[w] = g_last_error;
  };
  if (devs.size() == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (size_t w = 0; w < devs.size(); ++w) pool.emplace_back(work, w);
    for (auto& th : pool) th.join();
  }
  for (size_t w = 0; w < devs.size(); ++w)
    if (status[w] != MCB_OK) return fail(status[w], "device " + std::to_string(devs[w]) + ": " + errors[w]);
  return MCB_OK;
}


}  // namespace capi
}  // namespace mcb
