// capi.cpp — the C-ABI entry points (include/mcb/mcb.h), device plans and
// the multi-GPU host scheduler; descriptor lowering and validation live in
// capi_plan.cpp, the tree runners in capi_tree.cpp.
//
// Reference correspondence (file:line under /root/reference/proj):
//   mcb_validate        validate                 src/batch.cpp:62-120
//   mcb_run_direct      run_batch                src/batch.cpp:195-333
//   mcb_direct_mc       direct_mc                src/estimator.cpp:75-92
//   mcb_tree_refine     tree_refine              src/estimator.cpp:212-318 (capi_tree.cpp)
//   mcb_stratified_mc   stratified_mc            src/estimator.cpp:161-182
//   mcb_summarize_trials summarize_trials        src/estimator.cpp:320-337
//   mcb_stream_key      UniformStream key        src/sampling.cpp:84-87
//   mcb_volume          HyperRect::volume        src/sampling.cpp:16-20
//   mcb_debug_points    sample_uniform           src/sampling.cpp:102-112
// There is no CPU fallback: every numeric result comes from the sm_100a
// kernels; without a device the compute entry points return
// MCB_ERR_NO_DEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "mcb/mcb.h"
#include "capi_internal.hpp"
#include "mcb_internal.hpp"
#include "jit.hpp"
#include "program.hpp"

using namespace mcb::capi;


struct mcb_plan {
  int device = 0;
  uint64_t n_fns = 0;
  uint32_t trials = 0;
  HostPlan hp;
  DevBuf buf;
};

namespace mcb::capi {

mcb_status plan_create_impl(const mcb_integrand* fns, size_t n_fns, uint64_t seed,
                            uint32_t trials, int device, uint32_t chunk_base,
                            uint32_t trial_base, mcb_plan** out) {
  mcb_status st = validate_for_run(fns, n_fns, trials);
  if (st != MCB_OK) return st;
  for (size_t i = 0; i < n_fns; ++i)
    if (fns[i].method == MCB_METHOD_TREE)
      return fail(MCB_ERR_INVALID_ARGUMENT,
                  "method tree has no static plan (use mcb_run_direct or mcb_tree_refine)");
  if (chunk_base) {
    for (size_t i = 0; i < n_fns; ++i)
      if (uint64_t(chunk_base) + chunk_count(fns[i].n_samples) - 1 > 0xFFFFFFFFull)
        return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  }
  if ((st = check_device(device)) != MCB_OK) return st;
  auto plan = new mcb_plan();
  plan->device = device;
  plan->n_fns = n_fns;
  plan->trials = trials;
  if ((st = build_host_plan(fns, n_fns, seed, trials, chunk_base, trial_base, plan->hp)) != MCB_OK) {
    delete plan;
    return st;
  }
  DeviceGuard guard(device);
  cudaError_t e = plan->buf.reserve(n_fns, plan->hp.n_tiles, n_fns * trials, plan->hp.code.size(),
                                    plan->hp.consts.size());
  if (e == cudaSuccess) e = DevBuf::grow(plan->buf.bounds, plan->buf.cap_bounds, plan->hp.bounds.size());
  if (e == cudaSuccess && !plan->hp.bounds.empty())
    e = cudaMemcpy(plan->buf.bounds, plan->hp.bounds.data(), sizeof(double) * plan->hp.bounds.size(),
                   cudaMemcpyHostToDevice);
  for (size_t r = 0; r < n_fns; ++r)
    if (plan->hp.bounds_off[r] >= 0) plan->hp.descs[r].grid_bounds = plan->buf.bounds + plan->hp.bounds_off[r];
  if (e == cudaSuccess)
    e = cudaMemcpy(plan->buf.fns, plan->hp.descs.data(), sizeof(FnDesc) * n_fns, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !plan->hp.code.empty())
    e = cudaMemcpy(plan->buf.code, plan->hp.code.data(), sizeof(uint32_t) * plan->hp.code.size(),
                   cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !plan->hp.consts.empty())
    e = cudaMemcpy(plan->buf.consts, plan->hp.consts.data(), sizeof(double) * plan->hp.consts.size(),
                   cudaMemcpyHostToDevice);
  if (e == cudaSuccess) prepare_programs(plan->hp, true);
  if (e == cudaSuccess)
    e = mcb::detail::launch_expand_tiles(plan->buf.fns, uint32_t(n_fns), trials, plan->buf.tile_fn, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    mcb_plan_destroy(plan);
    return cuda_fail(e, "plan setup");
  }
  *out = plan;
  return MCB_OK;
}

mcb_status plan_launch_impl(mcb_plan* plan, cudaStream_t s) {
  DeviceGuard guard(plan->device);
  return enqueue_run(plan->hp, plan->buf, plan->trials, nullptr, false, s);
}

mcb_status plan_download_impl(mcb_plan* plan, mcb_trial_stats* out, cudaStream_t s) {
  DeviceGuard guard(plan->device);
  MCB_CUDA(cudaMemcpyAsync(out, plan->buf.out, sizeof(mcb_trial_stats) * plan->n_fns * plan->trials,
                           cudaMemcpyDeviceToHost, s));
  MCB_CUDA(cudaStreamSynchronize(s));
  return MCB_OK;
}

// LPT: integrands by decreasing cost onto the least-loaded shard.
void lpt(const mcb_integrand* fns, size_t n, uint32_t trials, int shards, uint32_t* shard_of) {
  std::vector<size_t> order(n);
  std::iota(order.begin(), order.end(), size_t(0));
  std::vector<double> cost(n);
  for (size_t i = 0; i < n; ++i)
    cost[i] = double(trial_samples(fns[i])) * double(trials) * sample_cost(fns[i]);
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return cost[a] > cost[b]; });
  std::vector<double> load(size_t(shards), 0.0);
  for (size_t i : order) {
    size_t best = 0;
    for (size_t s = 1; s < load.size(); ++s)
      if (load[s] < load[best]) best = s;
    shard_of[i] = uint32_t(best);
    load[best] += cost[i];
  }
}

// Multi-device form of run_sharded: the units are (integrand, trial) pairs,
// not whole integrands, so a job of a few integrands still fills every device
// (C1 = 100 integrands on 8 GPUs: 125 pairs each instead of 13 vs 12
// integrands).  A pair runs as a one-trial sub-integrand whose trial_base is
// its trial, so its key, counters and tile structure — and hence its
// McEstimate — are exactly those of the single-device plan (SURVEY.md §8(e):
// a (fn, trial, chunk) unit depends only on (seed, integrand_index, trial,
// chunk, spec), ref tests/test_batch.cpp:137-158).  LPT over the pairs by
// cost, ties in (integrand, trial) order; one host thread per device.
mcb_status run_sharded_trials(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                              const std::vector<int>& devs, mcb_trial_stats* out) {
  const size_t n_units = n_fns * size_t(trials);
  std::vector<double> cost(n_fns);
  for (size_t i = 0; i < n_fns; ++i) cost[i] = double(trial_samples(fns[i])) * sample_cost(fns[i]);
  std::vector<size_t> order(n_units);
  std::iota(order.begin(), order.end(), size_t(0));
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return cost[a / trials] > cost[b / trials]; });
  std::vector<std::vector<size_t>> mine(devs.size());
  std::vector<double> load(devs.size(), 0.0);
  for (size_t u : order) {
    size_t best = 0;
    for (size_t s = 1; s < load.size(); ++s)
      if (load[s] < load[best]) best = s;
    mine[best].push_back(u);
    load[best] += cost[u / trials];
  }
  std::vector<mcb_status> status(devs.size(), MCB_OK);
  std::vector<std::string> errors(devs.size());
  auto work = [&](size_t w) {
    std::vector<size_t>& units = mine[w];
    if (units.empty()) return;
    std::sort(units.begin(), units.end());  // job order within the device
    std::vector<mcb_integrand> sub(units.size());
    std::vector<uint32_t> tb(units.size()), cb(units.size(), 0);
    for (size_t r = 0; r < units.size(); ++r) {
      sub[r] = fns[units[r] / trials];
      tb[r] = uint32_t(units[r] % trials);
    }
    std::vector<mcb_trial_stats> res(units.size());
    const mcb_status s = run_shard(sub.data(), sub.size(), seed, 1, devs[w], res.data(), cb.data(), tb.data());
    status[w] = s;
    if (s != MCB_OK) {
      errors[w] = g_last_error;
      return;
    }
    for (size_t r = 0; r < units.size(); ++r) out[units[r]] = res[r];
  };
  std::vector<std::thread> pool;
  for (size_t w = 0; w < devs.size(); ++w) pool.emplace_back(work, w);
  for (auto& th : pool) th.join();
  for (size_t w = 0; w < devs.size(); ++w)
    if (status[w] != MCB_OK) return fail(status[w], "device " + std::to_string(devs[w]) + ": " + errors[w]);
  return MCB_OK;
}

// Shards integrands over `devs` by LPT, one host thread per device; results
// land in `out` (n_fns * trials) by integrand.  Byte-identical for any list.
mcb_status run_sharded(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                       const std::vector<int>& devs, mcb_trial_stats* out, const uint32_t* chunk_bases,
                       const uint32_t* trial_bases) {
  if (devs.size() > 1 && trials > 1 && !chunk_bases && !trial_bases)
    return run_sharded_trials(fns, n_fns, seed, trials, devs, out);
  if (devs.size() == 1) {  // one shard: the caller's arrays as they are
    const mcb_status s = run_shard(fns, n_fns, seed, trials, devs[0], out, chunk_bases, trial_bases);
    return s == MCB_OK ? s : fail(s, "device " + std::to_string(devs[0]) + ": " + std::string(g_last_error));
  }
  std::vector<uint32_t> shard(n_fns, 0);
  lpt(fns, n_fns, trials, int(devs.size()), shard.data());
  std::vector<mcb_status> status(devs.size(), MCB_OK);
  std::vector<std::string> errors(devs.size());
  auto work = [&](size_t w) {
    std::vector<size_t> mine;
    for (size_t i = 0; i < n_fns; ++i)
      if (shard[i] == w) mine.push_back(i);
    if (mine.empty()) return;
    std::vector<mcb_integrand> sub(mine.size());
    std::vector<uint32_t> cb, tb;
    for (size_t r = 0; r < mine.size(); ++r) sub[r] = fns[mine[r]];
    if (chunk_bases)
      for (size_t i : mine) cb.push_back(chunk_bases[i]);
    if (trial_bases)
      for (size_t i : mine) tb.push_back(trial_bases[i]);
    std::vector<mcb_trial_stats> res(sub.size() * trials);
    const mcb_status s = run_shard(sub.data(), sub.size(), seed, trials, devs[w], res.data(),
                                   chunk_bases ? cb.data() : nullptr, trial_bases ? tb.data() : nullptr);
    status[w] = s;
    if (s != MCB_OK) {
      errors[w] = g_last_error;
      return;
    }
    for (size_t r = 0; r < mine.size(); ++r)
      std::memcpy(out + mine[r] * trials, res.data() + r * trials, sizeof(mcb_trial_stats) * trials);
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

}  // namespace mcb::capi

extern "C" {

uint32_t mcb_abi_version(void) { return MCB_ABI_VERSION; }

const char* mcb_last_error(void) { return g_last_error.c_str(); }

int mcb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void mcb_stream_key(uint64_t global_seed, uint32_t integrand_index, uint32_t key_out[2]) {
  uint64_t h = splitmix64(global_seed);
  h = splitmix64(h ^ (0x9E3779B97F4A7C15ull * (uint64_t(integrand_index) + 1)));
  key_out[0] = uint32_t(h);
  key_out[1] = uint32_t(h >> 32);
}

double mcb_volume(const mcb_integrand* fn) { return fn ? volume(*fn) : 0.0; }

size_t mcb_to_dsl(const mcb_integrand* fn, char* buf, size_t cap) {
  if (!fn) return 0;
  const std::string s = to_dsl(*fn);
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return s.size() + 1;
}

mcb_status mcb_validate(const mcb_integrand* fns, size_t n_fns, const char* const* names,
                        uint32_t trials, mcb_violation* out, size_t cap, size_t* n_out) {
  std::vector<std::pair<int64_t, std::string>> v;
  if (trials < 1) v.push_back({-1, "trials must be >= 1"});
  if (n_fns == 0) v.push_back({-1, "integrand list is empty"});
  if (n_fns && !fns) return fail(MCB_ERR_INVALID_ARGUMENT, "fns is NULL");
  std::map<std::string, int> name_count;
  if (names)
    for (size_t i = 0; i < n_fns; ++i) ++name_count[names[i] ? names[i] : ""];
  for (size_t i = 0; i < n_fns; ++i) {
    std::vector<std::string> msgs;
    if (names && (!names[i] || !names[i][0])) msgs.push_back("integrand name is empty");
    violations_of(fns[i], trials, msgs);
    for (auto& m : msgs) v.push_back({int64_t(i), m});
  }
  if (names)  // duplicate names, once per offending name (src/batch.cpp:113-118)
    for (const auto& [name, count] : name_count)
      if (count > 1) {
        int64_t first = -1;
        for (size_t i = 0; i < n_fns; ++i)
          if (names[i] && name == names[i]) { first = int64_t(i); break; }
        v.push_back({first, "duplicate integrand name (" + std::to_string(count) + " occurrences)"});
      }
  if (n_out) *n_out = v.size();
  for (size_t i = 0; i < v.size() && i < cap && out; ++i) {
    out[i].integrand = v[i].first;
    std::snprintf(out[i].message, sizeof out[i].message, "%s", v[i].second.c_str());
  }
  return MCB_OK;
}

mcb_status mcb_stratified_plan(const mcb_integrand* fn, uint32_t* cells_per_dim, uint64_t* n_cells,
                               uint32_t* samples_per_cell) {
  if (!fn) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL integrand");
  if (fn->dim < 1 || fn->dim > MCB_MAX_DIM) return fail(MCB_ERR_INVALID_ARGUMENT, "bad dim");
  const StratPlan p = stratified_plan(*fn);
  if (!p.ok) return fail(MCB_ERR_VALIDATION, "cell grid exceeds configured cap");
  if (cells_per_dim) *cells_per_dim = p.k;
  if (n_cells) *n_cells = p.n_cells;
  if (samples_per_cell) *samples_per_cell = p.spc;
  return MCB_OK;
}

mcb_status mcb_partition(const mcb_integrand* fns, size_t n_fns, uint32_t trials, int n_shards,
                         uint32_t* shard_of_fn) {
  if (n_shards < 1) return fail(MCB_ERR_INVALID_ARGUMENT, "n_shards must be >= 1");
  if (n_fns && (!fns || !shard_of_fn)) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL buffer");
  lpt(fns, n_fns, trials, n_shards, shard_of_fn);
  return MCB_OK;
}

mcb_status mcb_summarize_trials(const mcb_trial_stats* per_trial, uint32_t n_trials, double* mean,
                                double* trial_stddev, uint32_t* n_ok) {
  if (!per_trial || !mean || !trial_stddev) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL buffer");
  double sum = 0.0;
  uint32_t r = 0;
  for (uint32_t t = 0; t < n_trials; ++t)
    if (per_trial[t].status == MCB_TRIAL_OK) {
      sum += per_trial[t].value;
      ++r;
    }
  if (n_ok) *n_ok = r;
  if (r == 0) return fail(MCB_ERR_INVALID_ARGUMENT, "no successful trials");  // InsufficientTrials
  *mean = sum / double(r);
  *trial_stddev = 0.0;
  if (r >= 2) {
    double ss = 0.0;
    for (uint32_t t = 0; t < n_trials; ++t)
      if (per_trial[t].status == MCB_TRIAL_OK) {
        const double d = per_trial[t].value - *mean;
        ss += d * d;
      }
    *trial_stddev = std::sqrt(ss / double(r - 1));
  }
  return MCB_OK;
}

mcb_status mcb_plan_create(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                           int device, mcb_plan** plan_out) {
  if (!plan_out) return fail(MCB_ERR_INVALID_ARGUMENT, "plan_out is NULL");
  *plan_out = nullptr;
  return plan_create_impl(fns, n_fns, seed, trials, device, 0, 0, plan_out);
}

mcb_status mcb_plan_launch(mcb_plan* plan, void* stream) {
  if (!plan) return fail(MCB_ERR_INVALID_ARGUMENT, "plan is NULL");
  return plan_launch_impl(plan, static_cast<cudaStream_t>(stream));
}

mcb_status mcb_plan_download(mcb_plan* plan, mcb_trial_stats* out, void* stream) {
  if (!plan || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  return plan_download_impl(plan, out, static_cast<cudaStream_t>(stream));
}

mcb_status mcb_plan_get_info(const mcb_plan* plan, mcb_plan_info* info) {
  if (!plan || !info) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  std::memset(info, 0, sizeof *info);
  info->n_fns = plan->n_fns;
  info->trials = plan->trials;
  info->n_groups = uint32_t(plan->hp.groups.size());
  info->n_tiles = plan->hp.n_tiles;
  info->total_samples = plan->hp.total_samples;
  info->philox_blocks = plan->hp.philox_blocks;
  uint32_t launches = 1;  // k_combine
  for (const auto& g : plan->hp.groups) {
    const uint64_t ctas = g.n_tiles / mcb::detail::tiles_per_cta(g.variant, g.family == MCB_FAMILY_PROGRAM);
    launches += uint32_t((ctas + 0x7FFFFFF7ull) / 0x7FFFFFF8ull);
  }
  info->launches_per_run = launches;
  return MCB_OK;
}

void mcb_plan_destroy(mcb_plan* plan) {
  if (!plan) return;
  {
    DeviceGuard guard(plan->device);
    plan->buf.release();
  }
  delete plan;
}

mcb_status mcb_run_direct(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                          const int* devices, int n_devices, mcb_trial_stats* out,
                          double* seconds) {
  static const bool trace = [] {
    const char* e = std::getenv("MCB_TREE_TRACE");
    return e && *e && *e != '0';
  }();
  const auto tv0 = std::chrono::steady_clock::now();
  mcb_status st = validate_for_run(fns, n_fns, trials);
  if (st != MCB_OK) return st;
  if (trace)
    std::fprintf(stderr, "[mcb run] validate %.3f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tv0).count());
  if (!out) return fail(MCB_ERR_INVALID_ARGUMENT, "out is NULL");
  std::vector<int> devs;
  if (!devices || n_devices <= 0) devs.push_back(0);
  else devs.assign(devices, devices + n_devices);
  for (int d : devs)
    if ((st = check_device(d)) != MCB_OK) return st;

  const auto t0 = std::chrono::steady_clock::now();
  std::vector<size_t> plain, trees;
  for (size_t i = 0; i < n_fns; ++i) (fns[i].method == MCB_METHOD_TREE ? trees : plain).push_back(i);
  if (trees.empty()) {  // the common case: no regrouping copies of the job or the results
    if ((st = run_sharded(fns, n_fns, seed, trials, devs, out, nullptr, nullptr)) != MCB_OK) return st;
  } else if (!plain.empty()) {  // direct + stratified: one sharded launch set
    std::vector<mcb_integrand> sub(plain.size());
    for (size_t r = 0; r < plain.size(); ++r) sub[r] = fns[plain[r]];
    std::vector<mcb_trial_stats> res(sub.size() * trials);
    if ((st = run_sharded(sub.data(), sub.size(), seed, trials, devs, res.data(), nullptr, nullptr)) != MCB_OK)
      return st;
    for (size_t r = 0; r < plain.size(); ++r)
      std::memcpy(out + plain[r] * trials, res.data() + r * trials, sizeof(mcb_trial_stats) * trials);
  }
  if (!trees.empty()) {  // tree: lock-step rounds over every (integrand, trial) tree
    std::vector<mcb::tree::TreeTask> tasks;
    tasks.reserve(trees.size() * trials);
    for (size_t i : trees)
      for (uint32_t t = 0; t < trials; ++t)
        tasks.push_back(mcb::tree::TreeTask{&fns[i], t, 0, out + i * trials + t, nullptr});
    if ((st = run_trees_on(tasks, seed, devs)) != MCB_OK) return st;
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (trace)
    std::fprintf(stderr, "[mcb run] run %.3f ms\n", std::chrono::duration<double, std::milli>(t1 - t0).count());
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  return MCB_OK;
}

mcb_status mcb_tree_refine(const mcb_integrand* fn, uint64_t seed, uint32_t trial, uint64_t chunk_base,
                           int device, mcb_trial_stats* out, mcb_leaf* leaves, size_t leaf_cap,
                           size_t* n_leaves) {
  if (!fn || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  // tree_refine itself has no validation step: a grid past the cap is a
  // CellBudgetExceeded result (MCB_TRIAL_CELL_BUDGET), not a job error.
  mcb_integrand f = *fn;
  f.method = MCB_METHOD_DIRECT;
  mcb_status st = validate_for_run(&f, 1, 1);
  if (st != MCB_OK) return st;
  f.method = MCB_METHOD_TREE;
  if ((st = check_device(device)) != MCB_OK) return st;
  std::vector<mcb_leaf> lv;
  std::vector<mcb::tree::TreeTask> tasks{mcb::tree::TreeTask{&f, trial, chunk_base, out, &lv}};
  const std::vector<int> devs{device};
  st = run_trees_on(tasks, seed, devs);
  if (st != MCB_OK) return st;
  if (n_leaves) *n_leaves = lv.size();
  if (leaves)
    std::memcpy(leaves, lv.data(), sizeof(mcb_leaf) * std::min(leaf_cap, lv.size()));
  return MCB_OK;
}

mcb_status mcb_stratified_mc(const mcb_integrand* fn, uint32_t cells_per_dim, uint32_t samples_per_cell,
                             uint64_t cell_cap, uint64_t seed, uint32_t trial, uint64_t chunk_base, int device,
                             mcb_trial_stats* out, mcb_leaf* leaves, size_t leaf_cap, size_t* n_leaves) {
  if (!fn || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (cells_per_dim == 0) return fail(MCB_ERR_INVALID_ARGUMENT, "cells_per_dim must be >= 1");
  if (samples_per_cell < 2) return fail(MCB_ERR_INVALID_ARGUMENT, "n_samples must be >= 2");
  mcb_integrand f = *fn;
  f.method = MCB_METHOD_DIRECT;
  mcb_status st = validate_for_run(&f, 1, 1);
  if (st != MCB_OK) return st;
  if ((st = check_device(device)) != MCB_OK) return st;
  // = the first pass of tree_refine with the grid given and no refinement
  f.method = MCB_METHOD_TREE;
  f.flags |= MCB_FLAG_REFINE_CONFIG;
  f.cells_per_dim = cells_per_dim;
  f.samples_per_cell = samples_per_cell;
  f.max_depth = 0;
  f.cell_cap = cell_cap;
  std::vector<mcb_leaf> lv;
  std::vector<mcb::tree::TreeTask> tasks{mcb::tree::TreeTask{&f, trial, chunk_base, out, &lv}};
  const std::vector<int> devs{device};
  st = run_trees_on(tasks, seed, devs);
  if (st != MCB_OK) return st;
  if (out->status == MCB_TRIAL_ALL_NONFINITE) {  // every cell dead: the first one throws
    out->status = MCB_TRIAL_DEAD_CELL;
    out->detail = 0;
  } else if (out->status == MCB_TRIAL_OK) {
    for (size_t i = 0; i < lv.size(); ++i)
      if (lv[i].estimate.status != MCB_TRIAL_OK) {  // direct_mc of cell i threw
        out->status = MCB_TRIAL_DEAD_CELL;
        out->detail = uint32_t(i);
        out->value = out->std_error = 0.0;
        lv.clear();
        break;
      }
  }
  if (n_leaves) *n_leaves = lv.size();
  if (leaves) std::memcpy(leaves, lv.data(), sizeof(mcb_leaf) * std::min(leaf_cap, lv.size()));
  return MCB_OK;
}

mcb_status mcb_direct_mc(const mcb_integrand* fn, uint64_t seed, uint32_t trial, uint64_t chunk_base,
                         int device, mcb_trial_stats* out) {
  if (!fn || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (fn->n_samples < 2) return fail(MCB_ERR_INVALID_ARGUMENT, "n_samples must be >= 2");
  if (chunk_base + chunk_count(fn->n_samples) - 1 > 0xFFFFFFFFull)
    return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  // One (integrand, trial) unit whose key base is {seed, integrand_index,
  // trial, chunk_base}, on the device's persistent context (no per-call
  // allocations: a call costs H2D + kernels + D2H).
  mcb_integrand f = *fn;  // direct_mc ignores the spec's method
  f.method = MCB_METHOD_DIRECT;
  mcb_status st = validate_for_run(&f, 1, 1);
  if (st != MCB_OK) return st;
  if ((st = check_device(device)) != MCB_OK) return st;
  const uint32_t cb = uint32_t(chunk_base), tb = trial;
  return run_shard(&f, 1, seed, 1, device, out, &cb, &tb);
}

mcb_status mcb_accumulate_chunk(const mcb_integrand* fn, uint64_t seed, uint32_t trial, uint64_t chunk,
                                uint32_t count, int device, mcb_chunk_accum* out) {
  if (!fn || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (count > MCB_CHUNK_SIZE) return fail(MCB_ERR_INVALID_ARGUMENT, "count exceeds the chunk size 65536");
  if (chunk > 0xFFFFFFFFull) return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  mcb_integrand f = *fn;  // one chunk of the direct method
  f.method = MCB_METHOD_DIRECT;
  f.n_samples = count < 2 ? 2 : count;  // the job rules (n_samples >= 2) are not accumulate_chunk's
  mcb_status st = validate_for_run(&f, 1, 1);
  if (st != MCB_OK) return st;
  *out = mcb_chunk_accum{0, 0, 0.0, 0.0};
  if (count == 0) return MCB_OK;
  if ((st = check_device(device)) != MCB_OK) return st;
  f.n_samples = count;
  const uint32_t cb = uint32_t(chunk), tb = trial;
  mcb_trial_stats stats;
  TilePartial p;
  if ((st = run_shard(&f, 1, seed, 1, device, &stats, &cb, &tb, &p, 1)) != MCB_OK) return st;
  // the tile's sums about its shift c -> (mean, m2), as k_combine's merge_tile
  out->n = p.n_finite;
  out->n_nonfinite = p.n_nonfinite;
  if (p.n_finite) {
    const double n = double(p.n_finite), dev = p.s1 / n;
    const double m2 = p.s2 - p.s1 * dev;
    out->mean = p.shift + dev;
    out->m2 = m2 > 0.0 ? m2 : (m2 == m2 ? 0.0 : HUGE_VAL);
  }
  return MCB_OK;
}

mcb_status mcb_debug_points(uint64_t seed, uint32_t integrand_index, uint32_t trial, uint64_t chunk,
                            uint64_t first_point, uint64_t count, uint32_t dim, const double* low,
                            const double* high, int device, double* out) {
  if (dim < 1 || dim > MCB_MAX_DIM || !low || !high || (count && !out))
    return fail(MCB_ERR_INVALID_ARGUMENT, "bad arguments");
  if (chunk > 0xFFFFFFFFull) return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  if ((first_point + count) * dim / 2 > 0xFFFFFFFFull)
    return fail(MCB_ERR_OUT_OF_RANGE, "block index exceeds 32 bits");
  mcb_status st = check_device(device);
  if (st != MCB_OK) return st;
  if (count == 0) return MCB_OK;
  DeviceGuard guard(device);
  uint32_t key[2];
  mcb_stream_key(seed, integrand_index, key);
  double hw[2 * MCB_MAX_DIM];
  for (uint32_t j = 0; j < dim; ++j) {
    hw[j] = low[j];
    hw[MCB_MAX_DIM + j] = high[j] - low[j];
  }
  double* d_lw = nullptr;
  double* d_out = nullptr;
  MCB_CUDA(cudaMalloc(&d_lw, sizeof hw));
  cudaError_t e = cudaMalloc(&d_out, sizeof(double) * count * dim);
  if (e == cudaSuccess) e = cudaMemcpy(d_lw, hw, sizeof hw, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = mcb::detail::launch_debug_points(key[0], key[1], trial, uint32_t(chunk), first_point, count,
                                         dim, d_lw, d_lw + MCB_MAX_DIM, d_out, nullptr);
  if (e == cudaSuccess)
    e = cudaMemcpy(out, d_out, sizeof(double) * count * dim, cudaMemcpyDeviceToHost);
  cudaFree(d_lw);
  if (d_out) cudaFree(d_out);
  if (e != cudaSuccess) return cuda_fail(e, "debug_points");
  return MCB_OK;
}

mcb_status mcb_debug_eval(const mcb_integrand* fn, uint64_t seed, uint32_t trial, uint64_t chunk,
                          uint64_t first_point, uint64_t count, int device, double* out) {
  if (!fn || (count && !out)) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  std::vector<std::string> msgs;
  violations_of(*fn, 1, msgs);
  if (!msgs.empty()) return fail(MCB_ERR_VALIDATION, msgs.front());
  if (chunk > 0xFFFFFFFFull) return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  if (first_point + count > MCB_CHUNK_SIZE)
    return fail(MCB_ERR_OUT_OF_RANGE, "points must lie inside one chunk");
  mcb_status st = check_device(device);
  if (st != MCB_OK) return st;
  if (count == 0) return MCB_OK;
  DeviceGuard guard(device);
  mcb_integrand direct = *fn;  // per-sample values on the integrand's own domain
  direct.method = MCB_METHOD_DIRECT;
  Prepared p = prepare(direct, seed, 0, 0);
  const uint64_t first_pair = first_point / 2;
  const uint64_t n_pairs = (first_point + count - 1) / 2 - first_pair + 1;
  const bool is_prog = fn->family == MCB_FAMILY_PROGRAM;
  FnDesc* d_fn = nullptr;
  double* d_out = nullptr;
  uint32_t* d_code = nullptr;
  double* d_consts = nullptr;
  if (is_prog) {
    p.d.prog_off = 0;
    p.d.prog_len = uint32_t(fn->program->p.code.size());
    p.d.const_off = 0;
    p.d.n_consts = uint32_t(fn->program->p.consts.size());
  }
  MCB_CUDA(cudaMalloc(&d_fn, sizeof(FnDesc)));
  cudaError_t e = cudaMalloc(&d_out, sizeof(double) * 2 * n_pairs);
  if (e == cudaSuccess) e = cudaMemcpy(d_fn, &p.d, sizeof(FnDesc), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && is_prog) {
    const auto& w = fn->program->words;
    const auto& c = fn->program->p.consts;
    e = cudaMalloc(&d_code, sizeof(uint32_t) * std::max<size_t>(w.size(), 1));
    if (e == cudaSuccess) e = cudaMalloc(&d_consts, sizeof(double) * std::max<size_t>(c.size(), 1));
    if (e == cudaSuccess) e = cudaMemcpy(d_code, w.data(), sizeof(uint32_t) * w.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !c.empty())
      e = cudaMemcpy(d_consts, c.data(), sizeof(double) * c.size(), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) {
    if (is_prog)
      e = mcb::detail::launch_program_eval(int(fn->dim), p.variant, d_fn, d_code, d_consts,
                                           fn->program->p.depth, trial, uint32_t(chunk),
                                           uint32_t(first_pair), uint32_t(n_pairs), d_out, nullptr);
    else
      e = mcb::detail::launch_debug_eval_impl(int(fn->family), int(fn->dim), p.variant, d_fn, trial,
                                              uint32_t(chunk), uint32_t(first_pair),
                                              uint32_t(n_pairs), d_out, nullptr);
  }
  std::vector<double> tmp(2 * n_pairs);
  if (e == cudaSuccess)
    e = cudaMemcpy(tmp.data(), d_out, sizeof(double) * 2 * n_pairs, cudaMemcpyDeviceToHost);
  cudaFree(d_fn);
  if (d_out) cudaFree(d_out);
  if (d_code) cudaFree(d_code);
  if (d_consts) cudaFree(d_consts);
  if (e != cudaSuccess) return cuda_fail(e, "debug_eval");
  std::memcpy(out, tmp.data() + (first_point - 2 * first_pair), sizeof(double) * count);
  return MCB_OK;
}

mcb_status mcb_program_eval_points(const mcb_program* program, const double* params, size_t n_params,
                                   const double* points, uint64_t n_points, int device, double* out) {
  if (!program || (n_points && (!points || !out)) || (n_params && !params))
    return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (n_params != program->p.param_names.size())
    return fail(MCB_ERR_INVALID_ARGUMENT, "program binds " + std::to_string(program->p.param_names.size()) +
                                              " parameter(s), got " + std::to_string(n_params));
  mcb_status st = check_device(device);
  if (st != MCB_OK) return st;
  if (n_points == 0) return MCB_OK;
  DeviceGuard guard(device);
  FnDesc d;
  std::memset(&d, 0, sizeof d);
  d.dim = program->p.dim;
  d.prog_len = uint32_t(program->p.code.size());
  d.n_consts = uint32_t(program->p.consts.size());
  for (size_t i = 0; i < n_params; ++i) d.k[i] = params[i];
  const auto& w = program->words;
  const auto& c = program->p.consts;
  const size_t n_coord = size_t(n_points) * program->p.dim;
  FnDesc* d_fn = nullptr;
  uint32_t* d_code = nullptr;
  double *d_consts = nullptr, *d_pts = nullptr, *d_out = nullptr;
  cudaError_t e = cudaMalloc(&d_fn, sizeof(FnDesc));
  if (e == cudaSuccess) e = cudaMalloc(&d_code, sizeof(uint32_t) * std::max<size_t>(w.size(), 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_consts, sizeof(double) * std::max<size_t>(c.size(), 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_pts, sizeof(double) * std::max<size_t>(n_coord, 1));
  if (e == cudaSuccess) e = cudaMalloc(&d_out, sizeof(double) * n_points);
  if (e == cudaSuccess) e = cudaMemcpy(d_fn, &d, sizeof d, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !w.empty())
    e = cudaMemcpy(d_code, w.data(), sizeof(uint32_t) * w.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !c.empty())
    e = cudaMemcpy(d_consts, c.data(), sizeof(double) * c.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && n_coord)
    e = cudaMemcpy(d_pts, points, sizeof(double) * n_coord, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = mcb::detail::launch_program_points(int(program->p.dim), d_fn, d_code, d_consts, program->p.depth,
                                           d_pts, n_points, d_out, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(out, d_out, sizeof(double) * n_points, cudaMemcpyDeviceToHost);
  cudaFree(d_fn);
  cudaFree(d_code);
  cudaFree(d_consts);
  cudaFree(d_pts);
  cudaFree(d_out);
  if (e != cudaSuccess) return cuda_fail(e, "program_eval_points");
  return MCB_OK;
}

int mcb_program_jit(int mode) {
  if (mode >= 0) mcb::jit::set_mode(mode);
  return mcb::jit::mode();
}

uint64_t mcb_program_jit_compiles(void) { return mcb::jit::compile_count(); }

mcb_status mcb_program_jit_build(const mcb_program* program) {
  if (!program) return fail(MCB_ERR_INVALID_ARGUMENT, "program is NULL");
  std::string err;
  if (!mcb::jit::compile_only(program->p, &err)) return fail(MCB_ERR_INVALID_ARGUMENT, "JIT build failed: " + err);
  return MCB_OK;
}

size_t mcb_program_jit_error(char* buf, size_t cap) {
  const std::string s = mcb::jit::last_error();
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return s.size() + 1;
}

mcb_status mcb_probe_philox_peak(int device, double ms, double* blocks_per_s) {
  if (!blocks_per_s) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  mcb_status st = check_device(device);
  if (st != MCB_OK) return st;
  DeviceGuard guard(device);
  int sms = 0;
  MCB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int ctas = sms * 8;
  uint32_t* buf = nullptr;
  MCB_CUDA(cudaMalloc(&buf, sizeof(uint32_t) * (ctas + 2)));
  const uint32_t key[2] = {0x37BA30CAu, 0xCCC782D2u};  // (seed 20200814, integrand 0)
  cudaError_t e = cudaMemcpy(buf, key, sizeof key, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 256;
  float elapsed = 0.f;
  for (int round = 0; round < 14 && e == cudaSuccess; ++round) {  // grow until ~ms
    cudaEventRecord(a);
    e = mcb::detail::launch_philox_probe(buf, buf + 2, ctas, iters, nullptr);
    cudaEventRecord(b);
    if (e == cudaSuccess) e = cudaEventSynchronize(b);
    if (e != cudaSuccess) break;
    cudaEventElapsedTime(&elapsed, a, b);
    if (elapsed >= ms) break;
    iters *= 2;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  if (e != cudaSuccess) return cuda_fail(e, "philox_probe");
  *blocks_per_s = double(ctas) * 256.0 * 4.0 * double(iters) / (double(elapsed) * 1e-3);
  return MCB_OK;
}

mcb_status mcb_program_compile(const char* source, uint32_t dim, const char* const* param_names,
                               size_t n_params, mcb_program** out) {
  if (!source || !out || (n_params && !param_names))
    return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  std::vector<std::string> names;
  for (size_t i = 0; i < n_params; ++i) {
    if (!param_names[i]) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL parameter name");
    names.emplace_back(param_names[i]);
  }
  std::sort(names.begin(), names.end());
  names.erase(std::unique(names.begin(), names.end()), names.end());
  try {
    auto* p = new mcb_program();
    try {
      p->p = mcb::prog::compile(source, dim, names);
    } catch (...) {
      delete p;
      throw;
    }
    p->words = p->p.words();
    *out = p;
    return MCB_OK;
  } catch (const mcb::prog::ParseError& e) {
    return fail(MCB_ERR_VALIDATION, std::string("expression does not parse: ") + e.what());
  } catch (const mcb::prog::CompileError& e) {
    return fail(MCB_ERR_VALIDATION, e.what());
  } catch (const std::exception& e) {
    return fail(MCB_ERR_INVALID_ARGUMENT, e.what());
  }
}

void mcb_program_destroy(mcb_program* program) { delete program; }

mcb_status mcb_program_info(const mcb_program* program, uint32_t* n_instr, uint32_t* depth,
                            uint32_t* n_params) {
  if (!program) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL program");
  if (n_instr) *n_instr = uint32_t(program->p.code.size());
  if (depth) *depth = program->p.depth;
  if (n_params) *n_params = uint32_t(program->p.param_names.size());
  return MCB_OK;
}

size_t mcb_program_param_name(const mcb_program* program, uint32_t i, char* buf, size_t cap) {
  if (!program || i >= program->p.param_names.size()) return 0;
  const std::string& s = program->p.param_names[i];
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return s.size() + 1;
}

}  // extern "C"
