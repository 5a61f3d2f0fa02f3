/*
 * mcb_oracle.c — CPU restatement of the reference direct Monte Carlo path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker.  The product path (paper_2104_10073_b200/libmcb.so)
 * never links, loads or calls it, and has no CPU fallback.
 *
 * Every function restates one reference function; citations are
 * file:line into /root/reference/proj.  Parity of this restatement is pinned
 * (tests/test_oracle.py) against
 *   - Random123 Philox4x32-10 known-answer vectors,
 *   - golden vectors produced by the reference itself, compiled from its own
 *     sources by oracle/Makefile (oracle/_ref) — tests/golden/*.json, made by
 *     tests/golden/make_golden.py,
 *   - the known-answer values in the reference's own tests
 *     (tests/test_estimator.cpp:44-62, tests/test_job_io.cpp:140-171).
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared (see oracle/Makefile).
 * -ffp-contract=off matters: the reference computes low + (high-low)*u and
 * a*cos(t) + b*sin(t) with separately rounded operations (x86-64, no FMA).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "mcb/mcb.h"

#define ORC_EXPORT __attribute__((visibility("default")))

/* ---- sampling: src/sampling.cpp -------------------------------------- */

/* src/sampling.cpp:39-42 */
static const uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
static const uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;

/* src/sampling.cpp:44-49 */
ORC_EXPORT uint64_t orc_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Key derivation inside UniformStream::UniformStream, src/sampling.cpp:84-87 */
ORC_EXPORT void orc_stream_key(uint64_t seed, uint32_t integrand, uint32_t key[2]) {
  uint64_t h = orc_splitmix64(seed);
  h = orc_splitmix64(h ^ (0x9E3779B97F4A7C15ull * ((uint64_t)integrand + 1)));
  key[0] = (uint32_t)h;
  key[1] = (uint32_t)(h >> 32);
}

/* philox_block, src/sampling.cpp:51-70 (Philox4x32-10, Random123 layout) */
ORC_EXPORT void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                                  uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)kM0 * c0;
    uint64_t p1 = (uint64_t)kM1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += kW0;
    k1 += kW1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* to_unit_double, src/sampling.cpp:72-75 */
ORC_EXPORT double orc_to_unit_double(uint32_t hi, uint32_t lo) {
  uint64_t u = ((uint64_t)hi << 32) | lo;
  return (double)(u >> 11) * 0x1.0p-53;
}

/* UniformStream draw `t` of stream (key, chunk, trial):
 * refill() src/sampling.cpp:92-100 makes block b = t/2 with counter
 * {b lo, b hi, chunk, trial}; next() (include/mcbatch/sampling.hpp:52-55) pops
 * buf_[1] = u(out0,out1) first, then buf_[0] = u(out2,out3). */
static double draw_at(const uint32_t key[2], uint32_t chunk, uint32_t trial, uint64_t t) {
  uint64_t b = t >> 1;
  uint32_t ctr[4] = {(uint32_t)b, (uint32_t)(b >> 32), chunk, trial};
  uint32_t o[4];
  orc_philox4x32_10(ctr, key, o);
  return (t & 1) ? orc_to_unit_double(o[2], o[3]) : orc_to_unit_double(o[0], o[1]);
}

/* sample_uniform, src/sampling.cpp:102-112, generalized to start at point
 * `first_point` of the chunk (same draws as the reference's sequential stream).
 * Returns 0, or -1 for an invalid rect / chunk > 2^32-1 (src/sampling.cpp:80-81). */
ORC_EXPORT int orc_sample_uniform(uint32_t dim, const double* low, const double* high,
                                  uint64_t seed, uint32_t integrand, uint32_t trial,
                                  uint64_t chunk, uint64_t first_point, uint64_t count,
                                  double* out) {
  if (dim < 1 || chunk > 0xFFFFFFFFull) return -1;
  for (uint32_t j = 0; j < dim; ++j)
    if (!(low[j] < high[j]) || !isfinite(low[j]) || !isfinite(high[j])) return -1;
  uint32_t key[2];
  orc_stream_key(seed, integrand, key);
  uint64_t t = first_point * dim;
  /* sequential refill as in UniformStream: one block per two draws */
  uint64_t cur_block = UINT64_MAX;
  uint32_t o[4] = {0, 0, 0, 0};
  for (uint64_t p = 0; p < count; ++p)
    for (uint32_t j = 0; j < dim; ++j, ++t) {
      uint64_t b = t >> 1;
      if (b != cur_block) {
        uint32_t ctr[4] = {(uint32_t)b, (uint32_t)(b >> 32), (uint32_t)chunk, trial};
        orc_philox4x32_10(ctr, key, o);
        cur_block = b;
      }
      double u = (t & 1) ? orc_to_unit_double(o[2], o[3]) : orc_to_unit_double(o[0], o[1]);
      double w = high[j] - low[j];
      double prod = w * u;
      out[p * dim + j] = low[j] + prod;
    }
  return 0;
}

/* ---- integrand families: CompiledProgram::evaluate on the lowered DSL --
 * src/expr.cpp:520-553 interprets the postfix program of the mcb_to_dsl
 * source; binary ops apply left-to-right with one rounding each, and
 * Cos/Sin/Abs call std::cos/std::sin/std::fabs (src/expr.cpp:90-99). */
ORC_EXPORT double orc_eval(const mcb_integrand* fn, const double* x) {
  const uint32_t d = fn->dim;
  switch (fn->family) {
    case MCB_FAMILY_HARMONIC: {
      /* "a*cos(k*(x1+...+xd)) + b*sin(k*(x1+...+xd))": ((x1+x2)+x3)+... */
      double s = x[0];
      for (uint32_t j = 1; j < d; ++j) s = s + x[j];
      double t = fn->k[0] * s;
      if (fn->flags & MCB_FLAG_UNIT_COEFFS) return cos(t) + sin(t); /* job_io.cpp:367 */
      double c = fn->a * cos(t);
      double sn = fn->b * sin(t);
      return c + sn;
    }
    case MCB_FAMILY_HARMONIC_VEC: {
      /* "a*cos(k1*x1+...+kd*xd) + ...": ((k1*x1 + k2*x2) + k3*x3) + ... */
      double t = fn->k[0] * x[0];
      for (uint32_t j = 1; j < d; ++j) {
        double p = fn->k[j] * x[j];
        t = t + p;
      }
      double c = fn->a * cos(t);
      double sn = fn->b * sin(t);
      return c + sn;
    }
    case MCB_FAMILY_ABS2: {
      double s = x[0] + x[1];
      return fn->a * fabs(s);
    }
    case MCB_FAMILY_ABS3: {
      double s = x[0] + x[1];
      s = s - x[2];
      return fn->a * fabs(s);
    }
  }
  return NAN;
}

/* ---- estimator: src/estimator.cpp ------------------------------------- */

typedef struct orc_chunk_accum {
  uint64_t n, n_nonfinite;
  double mean, m2;
} orc_chunk_accum;

/* ChunkAccum::add, src/estimator.cpp:9-18 (Welford, non-finite skipped) */
ORC_EXPORT void orc_accum_add(orc_chunk_accum* a, double x) {
  if (!isfinite(x)) { ++a->n_nonfinite; return; }
  ++a->n;
  double delta = x - a->mean;
  a->mean += delta / (double)a->n;
  a->m2 += delta * (x - a->mean);
}

/* ChunkAccum::merge, src/estimator.cpp:20-34 (Chan) */
ORC_EXPORT void orc_accum_merge(orc_chunk_accum* a, const orc_chunk_accum* o) {
  a->n_nonfinite += o->n_nonfinite;
  if (o->n == 0) return;
  if (a->n == 0) { a->n = o->n; a->mean = o->mean; a->m2 = o->m2; return; }
  double delta = o->mean - a->mean;
  uint64_t total = a->n + o->n;
  a->mean += delta * ((double)o->n / (double)total);
  a->m2 += o->m2 + delta * delta * ((double)a->n * (double)o->n / (double)total);
  a->n = total;
}

/* accumulate_chunk, src/estimator.cpp:36-49 */
ORC_EXPORT int orc_accumulate_chunk(const mcb_integrand* fn, uint64_t seed, uint32_t trial,
                                    uint64_t chunk, uint64_t count, orc_chunk_accum* out) {
  orc_chunk_accum acc = {0, 0, 0.0, 0.0};
  double pt[MCB_MAX_DIM];
  const uint64_t step = 4096;
  double* buf = (double*)malloc(sizeof(double) * step * fn->dim);
  if (!buf) return -1;
  for (uint64_t p0 = 0; p0 < count; p0 += step) {
    uint64_t m = count - p0 < step ? count - p0 : step;
    if (orc_sample_uniform(fn->dim, fn->low, fn->high, seed, fn->integrand_index, trial,
                           chunk, p0, m, buf) != 0) {
      free(buf);
      return -1;
    }
    for (uint64_t i = 0; i < m; ++i) {
      memcpy(pt, buf + i * fn->dim, sizeof(double) * fn->dim);
      orc_accum_add(&acc, orc_eval(fn, pt));
    }
  }
  free(buf);
  *out = acc;
  return 0;
}

/* HyperRect::volume, src/sampling.cpp:16-20 */
ORC_EXPORT double orc_volume(const mcb_integrand* fn) {
  double v = 1.0;
  for (uint32_t j = 0; j < fn->dim; ++j) v *= fn->high[j] - fn->low[j];
  return v;
}

/* reduce_chunks, src/estimator.cpp:55-73.  status ALL_NONFINITE replaces the
 * AllSamplesNonFinite exception. */
static void reduce_to_stats(double volume, const orc_chunk_accum* total, mcb_trial_stats* st) {
  memset(st, 0, sizeof *st);
  st->n_samples = total->n + total->n_nonfinite;
  st->n_nonfinite = total->n_nonfinite;
  if (total->n == 0) { st->status = MCB_TRIAL_ALL_NONFINITE; return; }
  st->status = MCB_TRIAL_OK;
  st->n_cells = 1;
  st->value = volume * total->mean;
  if (total->n >= 2) {
    double var = total->m2 / (double)(total->n - 1);
    st->std_error = volume * sqrt(var / (double)total->n);
  } else {
    st->std_error = INFINITY;
  }
  st->nonfinite_warning =
      (double)total->n_nonfinite > MCB_NONFINITE_WARN_FRACTION * (double)st->n_samples;
}

/* chunk_count, src/estimator.cpp:51-53 */
ORC_EXPORT uint64_t orc_chunk_count(uint64_t n) { return (n + MCB_CHUNK_SIZE - 1) / MCB_CHUNK_SIZE; }

/* direct_mc, src/estimator.cpp:75-92: chunk c uses key chunk_base + c and
 * count min(65536, remaining); chunks merge in ascending order. */
ORC_EXPORT int orc_direct_mc(const mcb_integrand* fn, uint64_t seed, uint32_t trial,
                             uint64_t chunk_base, mcb_trial_stats* out) {
  if (fn->n_samples < 2) return -1;
  uint64_t n_chunks = orc_chunk_count(fn->n_samples);
  uint64_t remaining = fn->n_samples;
  orc_chunk_accum total = {0, 0, 0.0, 0.0};
  for (uint64_t c = 0; c < n_chunks; ++c) {
    uint64_t count = remaining < MCB_CHUNK_SIZE ? remaining : MCB_CHUNK_SIZE;
    remaining -= count;
    orc_chunk_accum a;
    if (orc_accumulate_chunk(fn, seed, trial, chunk_base + c, count, &a) != 0) return -1;
    orc_accum_merge(&total, &a);
  }
  reduce_to_stats(orc_volume(fn), &total, out);
  return 0;
}

/* ---- stratified: src/batch.cpp:41-54, src/estimator.cpp:94-182 ---------- */

/* cell_grid_size, src/estimator.cpp:94-105 (returns 0 past the cap) */
static uint64_t cell_grid_size(uint32_t k, uint32_t d, uint64_t cap) {
  if (k == 0) return 0;
  uint64_t cells = 1;
  for (uint32_t i = 0; i < d; ++i) {
    if (cells > cap / k + 1) return 0;
    cells *= k;
  }
  return cells > cap ? 0 : cells;
}

/* auto_cells_per_dim, src/estimator.cpp:107-122 */
static uint32_t auto_cells_per_dim(uint32_t d, uint64_t limit) {
  uint32_t k = 1;
  for (;;) {
    uint64_t cells = 1;
    for (uint32_t i = 0; i < d; ++i) {
      cells *= (uint64_t)k + 1;
      if (cells > limit) return k;
    }
    ++k;
  }
}

/* stratified_plan, src/batch.cpp:41-54 */
ORC_EXPORT int orc_stratified_plan(const mcb_integrand* fn, uint32_t* k, uint64_t* n_cells,
                                   uint32_t* spc) {
  const uint64_t cap = fn->cell_cap ? fn->cell_cap : 1000000ull;
  if (fn->cells_per_dim > 0) {
    *k = fn->cells_per_dim;
  } else {
    uint64_t limit = fn->n_samples / 2 < 4096 ? fn->n_samples / 2 : 4096;
    *k = auto_cells_per_dim(fn->dim, limit > 1 ? limit : 1);
  }
  *n_cells = cell_grid_size(*k, fn->dim, cap);
  if (*n_cells == 0) return -1;
  uint64_t per = fn->n_samples / *n_cells;
  *spc = (uint32_t)(per > 2 ? per : 2);
  return 0;
}

/* grid_cell, src/estimator.cpp:124-143 (axis 0 most significant) */
ORC_EXPORT void orc_grid_cell(const mcb_integrand* fn, uint32_t k, uint64_t index, double* lo,
                              double* hi) {
  uint64_t rem = index;
  for (int j = (int)fn->dim - 1; j >= 0; --j) {
    uint32_t digit = (uint32_t)(rem % k);
    rem /= k;
    double width = fn->high[j] - fn->low[j];
    lo[j] = digit == 0 ? fn->low[j] : fn->low[j] + width * ((double)digit / k);
    hi[j] = digit + 1 == k ? fn->high[j] : fn->low[j] + width * ((double)(digit + 1) / k);
  }
}

/* run_batch Stratified branch for one trial (src/batch.cpp:255-275 tasks,
 * :172-186 assemble) = stratified_mc (src/estimator.cpp:161-182): direct_mc
 * per cell with chunk keys c * chunks_per_cell, combine_cells
 * (src/estimator.cpp:145-159).  status DEAD_CELL (detail = first dead cell)
 * replaces "cell c produced no finite sample". */
ORC_EXPORT int orc_stratified_mc(const mcb_integrand* fn, uint64_t seed, uint32_t trial,
                                 uint64_t chunk_base, mcb_trial_stats* out) {
  uint32_t k, spc;
  uint64_t n_cells;
  if (orc_stratified_plan(fn, &k, &n_cells, &spc) != 0) return -1;
  const uint64_t cpc = orc_chunk_count(spc);
  mcb_integrand cell = *fn;
  cell.method = 0;
  cell.n_samples = spc;
  double value = 0.0, var = 0.0;
  uint64_t n_all = 0, nn_all = 0;
  int64_t dead = -1;
  for (uint64_t c = 0; c < n_cells; ++c) {
    orc_grid_cell(fn, k, c, cell.low, cell.high);
    mcb_trial_stats st;
    if (orc_direct_mc(&cell, seed, trial, chunk_base + c * cpc, &st) != 0) return -1;
    n_all += st.n_samples;
    nn_all += st.n_nonfinite;
    if (st.status != MCB_TRIAL_OK) {
      if (dead < 0) dead = (int64_t)c;
      continue;
    }
    value += st.value;
    var += st.std_error * st.std_error;
  }
  memset(out, 0, sizeof *out);
  out->n_samples = n_all;
  out->n_nonfinite = nn_all;
  out->n_cells = (uint32_t)n_cells;
  out->nonfinite_warning = (double)nn_all > MCB_NONFINITE_WARN_FRACTION * (double)n_all;
  if (dead >= 0) {
    out->status = MCB_TRIAL_DEAD_CELL;
    out->detail = (uint32_t)dead;
    return 0;
  }
  out->status = MCB_TRIAL_OK;
  out->value = value;
  out->std_error = sqrt(var);
  return 0;
}

/* ---- tree: src/estimator.cpp:184-318, src/batch.cpp:276-289 ------------- */

typedef struct {
  double low[MCB_MAX_DIM], high[MCB_MAX_DIM];
  mcb_trial_stats est;
  uint32_t depth;
} orc_leaf;

/* estimate_cell lambda, src/estimator.cpp:238-253: direct_mc of the cell with
 * key chunk next_chunk; AllSamplesNonFinite becomes a dead leaf.  Returns -1
 * when the chunk index leaves 32 bits (UniformStream throws). */
static int orc_estimate_cell(const mcb_integrand* fn, orc_leaf* l, uint32_t spc, uint64_t cpc,
                             uint64_t seed, uint32_t trial, uint64_t* next_chunk, uint64_t* used) {
  if (*next_chunk + cpc - 1 > 0xFFFFFFFFull) return -1;
  mcb_integrand cell = *fn;
  cell.method = MCB_METHOD_DIRECT;
  cell.n_samples = spc;
  memcpy(cell.low, l->low, sizeof cell.low);
  memcpy(cell.high, l->high, sizeof cell.high);
  uint64_t key_chunk = *next_chunk;
  *next_chunk += cpc;
  *used += spc;
  if (orc_direct_mc(&cell, seed, trial, key_chunk, &l->est) != 0) return -1;
  if (l->est.status != MCB_TRIAL_OK) {
    memset(&l->est, 0, sizeof l->est);
    l->est.status = MCB_TRIAL_ALL_NONFINITE;
    l->est.n_samples = spc;
    l->est.n_nonfinite = spc;
    l->est.nonfinite_warning = 1;
  }
  return 0;
}

/* tree_refine, src/estimator.cpp:212-318, with RefineConfig from the
 * descriptor (MCB_FLAG_REFINE_CONFIG; total_budget = n_samples as run_batch
 * sets it, src/batch.cpp:278).  Leaves (may be NULL) in the reference's order. */
ORC_EXPORT int orc_tree_refine(const mcb_integrand* fn, uint64_t seed, uint32_t trial,
                               uint64_t chunk_base, mcb_trial_stats* out, mcb_leaf* leaves_out,
                               size_t cap, size_t* n_leaves) {
  const uint32_t d = fn->dim;
  uint32_t spc_cfg = 2048, max_depth = 6;
  double sigma = 1.0;
  if (fn->flags & MCB_FLAG_REFINE_CONFIG) {
    spc_cfg = fn->samples_per_cell;
    max_depth = fn->max_depth;
    sigma = fn->sigma_multiplier;
  }
  const uint64_t budget = fn->n_samples;
  const uint64_t cell_cap = fn->cell_cap ? fn->cell_cap : 1000000ull;
  const uint32_t spc = spc_cfg > 2 ? spc_cfg : 2;
  memset(out, 0, sizeof *out);
  uint32_t k = fn->cells_per_dim;
  if (k == 0) {
    k = auto_cells_per_dim(d, 4096);
    while (k > 1) {
      uint64_t cells = cell_grid_size(k, d, cell_cap);
      if (cells == 0) { out->status = MCB_TRIAL_CELL_BUDGET; return 0; }
      if (cells * spc <= budget / 2) break;
      --k;
    }
  }
  const uint64_t n_cells = cell_grid_size(k, d, cell_cap);
  if (n_cells == 0) { out->status = MCB_TRIAL_CELL_BUDGET; return 0; }
  const uint64_t cpc = orc_chunk_count(spc);
  uint64_t next_chunk = chunk_base, used = 0;
  int exhausted = 0;
  size_t n = 0, capl = (size_t)n_cells + 16;
  orc_leaf* lv = (orc_leaf*)malloc(sizeof(orc_leaf) * capl);
  size_t* sel = NULL;
  if (!lv) return -1;
  mcb_integrand rect = *fn;
  for (uint64_t c = 0; c < n_cells; ++c, ++n) {
    memset(&lv[n], 0, sizeof lv[n]);
    orc_grid_cell(&rect, k, c, lv[n].low, lv[n].high);
    if (orc_estimate_cell(fn, &lv[n], spc, cpc, seed, trial, &next_chunk, &used) != 0) {
      free(lv);
      out->status = MCB_TRIAL_CHUNK_RANGE;
      return 0;
    }
  }
  while (!exhausted) {
    double mean_err = 0.0;
    for (size_t i = 0; i < n; ++i) mean_err += lv[i].est.std_error;
    mean_err /= (double)n;
    double ss = 0.0;
    for (size_t i = 0; i < n; ++i) {
      double dlt = lv[i].est.std_error - mean_err;
      ss += dlt * dlt;
    }
    double sd = n > 1 ? sqrt(ss / (double)(n - 1)) : 0.0;
    double threshold = mean_err + sigma * sd;
    size_t n_sel = 0;
    free(sel);
    sel = (size_t*)malloc(sizeof(size_t) * n);
    for (size_t i = 0; i < n; ++i)
      if (lv[i].depth < max_depth && lv[i].est.std_error > 0 && lv[i].est.std_error > threshold)
        sel[n_sel++] = i;
    if (n_sel == 0) break;
    for (size_t s = 0; s < n_sel; ++s) {
      size_t idx = sel[s];
      if (used + 2ull * spc > budget) { exhausted = 1; break; }
      if (n + 1 > capl) {
        capl *= 2;
        lv = (orc_leaf*)realloc(lv, sizeof(orc_leaf) * capl);
      }
      /* split_longest_edge, src/estimator.cpp:192-210 */
      orc_leaf lo = lv[idx], hi = lv[idx];
      uint32_t axis = 0;
      double best = -1.0;
      for (uint32_t j = 0; j < d; ++j) {
        double w = lv[idx].high[j] - lv[idx].low[j];
        if (w > best) { best = w; axis = j; }
      }
      double mid = lv[idx].low[axis] + 0.5 * (lv[idx].high[axis] - lv[idx].low[axis]);
      lo.high[axis] = mid;
      hi.low[axis] = mid;
      lo.depth = hi.depth = lv[idx].depth + 1;
      if (orc_estimate_cell(fn, &lo, spc, cpc, seed, trial, &next_chunk, &used) != 0 ||
          orc_estimate_cell(fn, &hi, spc, cpc, seed, trial, &next_chunk, &used) != 0) {
        free(lv); free(sel);
        out->status = MCB_TRIAL_CHUNK_RANGE;
        return 0;
      }
      lv[idx] = lo;
      lv[n++] = hi;
    }
  }
  free(sel);
  /* combine_cells over the leaves, src/estimator.cpp:145-159 and :299-306 */
  double value = 0.0, var = 0.0;
  uint64_t ns = 0, nn = 0, finite = 0;
  uint32_t depth = 0;
  for (size_t i = 0; i < n; ++i) {
    value += lv[i].est.value;
    var += lv[i].est.std_error * lv[i].est.std_error;
    ns += lv[i].est.n_samples;
    nn += lv[i].est.n_nonfinite;
    finite += lv[i].est.n_samples - lv[i].est.n_nonfinite;
    if (lv[i].depth > depth) depth = lv[i].depth;
  }
  out->n_samples = ns;
  out->n_nonfinite = nn;
  out->n_cells = (uint32_t)n;
  out->max_depth = depth;
  out->budget_exhausted = (uint32_t)exhausted;
  if (finite == 0) {
    out->status = MCB_TRIAL_ALL_NONFINITE;
  } else {
    out->status = MCB_TRIAL_OK;
    out->value = value;
    out->std_error = sqrt(var);
    out->nonfinite_warning = (double)nn > MCB_NONFINITE_WARN_FRACTION * (double)ns;
  }
  if (out->status != MCB_TRIAL_OK) n = 0; /* leaves_out is written only on return */
  if (n_leaves) *n_leaves = n;
  for (size_t i = 0; leaves_out && i < n && i < cap; ++i) {
    memset(&leaves_out[i], 0, sizeof leaves_out[i]);
    memcpy(leaves_out[i].low, lv[i].low, sizeof lv[i].low);
    memcpy(leaves_out[i].high, lv[i].high, sizeof lv[i].high);
    leaves_out[i].estimate = lv[i].est;
    leaves_out[i].depth = lv[i].depth;
  }
  free(lv);
  return 0;
}

/* summarize_trials, src/estimator.cpp:320-337, over the OK trials only
 * (run_batch collects the successful ones, src/batch.cpp:309-318). */
ORC_EXPORT int orc_summarize_trials(const mcb_trial_stats* per_trial, uint32_t n,
                                    double* mean, double* stddev, uint32_t* n_ok) {
  double sum = 0.0;
  uint32_t r = 0;
  for (uint32_t t = 0; t < n; ++t)
    if (per_trial[t].status == MCB_TRIAL_OK) { sum += per_trial[t].value; ++r; }
  *n_ok = r;
  if (r == 0) return -1;
  *mean = sum / (double)r;
  *stddev = 0.0;
  if (r >= 2) {
    double ss = 0.0;
    for (uint32_t t = 0; t < n; ++t)
      if (per_trial[t].status == MCB_TRIAL_OK) {
        double dd = per_trial[t].value - *mean;
        ss += dd * dd;
      }
    *stddev = sqrt(ss / (double)(r - 1));
  }
  return 0;
}

/* run_batch, src/batch.cpp:195-333, every method: (integrand, trial) units
 * with StreamKey {seed, integrand_index, trial, 0} drained by a thread pool
 * (src/batch.cpp:150-168).  Results do not depend on n_threads. */
typedef struct {
  const mcb_integrand* fns;
  size_t n_fns;
  uint64_t seed;
  uint32_t trials;
  mcb_trial_stats* out;
  size_t next;
  int failed;
  pthread_mutex_t mu;
} orc_pool;

static void* orc_worker(void* arg) {
  orc_pool* p = (orc_pool*)arg;
  for (;;) {
    pthread_mutex_lock(&p->mu);
    size_t u = p->next++;
    pthread_mutex_unlock(&p->mu);
    if (u >= p->n_fns * p->trials) break;
    size_t i = u / p->trials;
    uint32_t t = (uint32_t)(u % p->trials);
    int rc = p->fns[i].method == MCB_METHOD_STRATIFIED
                 ? orc_stratified_mc(&p->fns[i], p->seed, t, 0, &p->out[u])
                 : p->fns[i].method == MCB_METHOD_TREE
                       ? orc_tree_refine(&p->fns[i], p->seed, t, 0, &p->out[u], NULL, 0, NULL)
                       : orc_direct_mc(&p->fns[i], p->seed, t, 0, &p->out[u]);
    if (rc != 0) p->failed = 1;
  }
  return NULL;
}

ORC_EXPORT int orc_run_direct(const mcb_integrand* fns, size_t n_fns, uint64_t seed,
                              uint32_t trials, int n_threads, mcb_trial_stats* out) {
  orc_pool p = {fns, n_fns, seed, trials, out, 0, 0, PTHREAD_MUTEX_INITIALIZER};
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
  for (int w = 1; w < n_threads; ++w) pthread_create(&th[w], NULL, orc_worker, &p);
  orc_worker(&p);
  for (int w = 1; w < n_threads; ++w) pthread_join(th[w], NULL);
  free(th);
  return p.failed ? -1 : 0;
}

/* ---- harmonic benchmark helpers: src/job_io.cpp ------------------------ */

/* harmonic_k, src/job_io.cpp:336-338 */
ORC_EXPORT double orc_harmonic_k(uint32_t n) { return ((double)n + 50.0) / (2.0 * M_PI); }

/* harmonic_closed_form, src/job_io.cpp:340-348, generalized to [0,1]^d:
 * integral of cos(k*sum x) + sin(k*sum x) = Re(phi^d) + Im(phi^d),
 * phi = (e^{ik} - 1)/(ik) = (sin k + i(1 - cos k))/k. */
ORC_EXPORT double orc_harmonic_closed_form(double k, uint32_t d) {
  if (k == 0.0) return 1.0;
  double pr = sin(k) / k, pi = (1.0 - cos(k)) / k;
  double zr = 1.0, zi = 0.0;
  for (uint32_t j = 0; j < d; ++j) {
    double nr = zr * pr - zi * pi;
    double ni = zr * pi + zi * pr;
    zr = nr; zi = ni;
  }
  return zr + zi;
}
