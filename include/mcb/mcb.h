/*
 * mcb.h — C-ABI drop-in boundary for the direct Monte Carlo multi-function
 * integration path (arXiv 2104.10073, ZMCintegral-v5.1 "multifunctions"),
 * B200-native (sm_100a).
 *
 * The reference (`/root/reference/proj`, library `mcbatch`) exposes this path
 * only as a C++ header API; there is no FFI.  Each entry point below names the
 * reference interface it replaces (file:line, relative to
 * /root/reference/proj).  Plain pointers and sizes, caller-allocated buffers,
 * status codes instead of exceptions; no torch or CUDA types in signatures
 * (streams are passed as `void*` = cudaStream_t).
 *
 * Integrands are *family descriptors* instead of free DSL strings; every
 * descriptor lowers (mcb_to_dsl) to the exact DSL source the reference would
 * parse, and the device evaluator follows the same left-to-right operation
 * order as the reference's compiled postfix program (src/expr.cpp:520-553).
 */
#ifndef MCB_MCB_H_
#define MCB_MCB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCB_ABI_VERSION 2u

#if defined(__GNUC__)
#define MCB_API __attribute__((visibility("default")))
#else
#define MCB_API
#endif

/* Samples per (key, chunk): include/mcbatch/sampling.hpp:11 (kChunkSize). */
#define MCB_CHUNK_SIZE 65536u
/* Largest supported dimension of a family descriptor. */
#define MCB_MAX_DIM 8u
/* Non-finite warning fraction: include/mcbatch/estimator.hpp:16. */
#define MCB_NONFINITE_WARN_FRACTION 0.01

typedef enum mcb_status {
  MCB_OK = 0,
  MCB_ERR_INVALID_ARGUMENT = 1, /* bad pointer/size/descriptor; see mcb_last_error */
  MCB_ERR_VALIDATION = 2,       /* job failed validation (reference ValidationError) */
  MCB_ERR_CUDA = 3,             /* CUDA runtime / launch failure */
  MCB_ERR_NO_DEVICE = 4,        /* no usable sm_100 device */
  MCB_ERR_OUT_OF_RANGE = 5,     /* chunk index > 2^32-1 (src/sampling.cpp:80-81) */
  MCB_ERR_BUFFER_TOO_SMALL = 6
} mcb_status;

/* Built-in integrand families (BASELINE.json north_star; Eq.1/Eq.2).
 * DSL lowering (mcb_to_dsl), with x1..xd the coordinates:
 *   HARMONIC      "a*cos(k*(x1+...+xd)) + b*sin(k*(x1+...+xd))"
 *                 or, when flags has MCB_FLAG_UNIT_COEFFS (a = b = 1),
 *                 "cos(k*(x1+...+xd)) + sin(k*(x1+...+xd))"   (src/job_io.cpp:367)
 *   HARMONIC_VEC  "a*cos(k1*x1+...+kd*xd) + b*sin(k1*x1+...+kd*xd)"
 *   ABS2          "a*abs(x1+x2)"   ("abs(x1+x2)" when a == 1), dim >= 2
 *   ABS3          "a*abs(x1+x2-x3)" ("abs(x1+x2-x3)" when a == 1), dim >= 3
 */
typedef enum mcb_family {
  MCB_FAMILY_HARMONIC = 0,
  MCB_FAMILY_HARMONIC_VEC = 1,
  MCB_FAMILY_ABS2 = 2,
  MCB_FAMILY_ABS3 = 3,
  MCB_FAMILY_PROGRAM = 4 /* any DSL source: compiled by mcb_program_compile, run by
                            the GPU interpreter (ref/src/expr.cpp:520-553 semantics) */
} mcb_family;

/* Maximum number of parameters a PROGRAM integrand binds (values in k[]). */
#define MCB_MAX_PARAMS 8u

/* A compiled DSL program (opaque; immutable, shareable across threads). */
typedef struct mcb_program mcb_program;

#define MCB_FLAG_UNIT_COEFFS 0x1u
/* TREE: samples_per_cell, max_depth and sigma_multiplier are taken as given;
 * without the flag they are the RefineConfig defaults 2048, 6, 1.0
 * (include/mcbatch/estimator.hpp:40-47), so a zeroed descriptor is valid. */
#define MCB_FLAG_REFINE_CONFIG 0x2u

/* One integrand = one reference IntegrandSpec (include/mcbatch/batch.hpp:22-31)
 * restricted to Method::Direct and a family descriptor.  `integrand_index` is
 * the StreamKey integrand index (= the job-list position in the reference,
 * src/batch.cpp:221); it is explicit so that shards of a job keep the global
 * stream identity. */
typedef struct mcb_integrand {
  uint32_t family;          /* mcb_family */
  uint32_t dim;             /* 1..MCB_MAX_DIM */
  uint32_t integrand_index; /* StreamKey.integrand_index */
  uint32_t flags;           /* MCB_FLAG_* */
  uint64_t n_samples;       /* per trial, >= 2 */
  double a, b;              /* coefficients (ABS families use `a`) */
  double k[MCB_MAX_DIM];    /* HARMONIC: k[0]; HARMONIC_VEC: k[0..dim-1];
                               PROGRAM: parameter values in sorted-name order */
  double low[MCB_MAX_DIM];  /* HyperRect low  (include/mcbatch/sampling.hpp:14-24) */
  double high[MCB_MAX_DIM]; /* HyperRect high */
  const mcb_program* program; /* PROGRAM family only (not owned) */
  uint32_t method;          /* mcb_method (reference Method, include/mcbatch/batch.hpp:18) */
  uint32_t cells_per_dim;   /* STRATIFIED: k (0 = auto, ref src/batch.cpp:41-54);
                               TREE: RefineConfig::init_cells_per_dim (0 = auto) */
  uint64_t cell_cap;        /* STRATIFIED/TREE: max k^d cells (0 = 1e6, RefineConfig::cell_cap) */
  /* TREE only (RefineConfig, include/mcbatch/estimator.hpp:40-47; the
   * refinement budget total_budget is n_samples, as run_batch sets it,
   * src/batch.cpp:278-279).  Read only with MCB_FLAG_REFINE_CONFIG. */
  uint32_t samples_per_cell;
  uint32_t max_depth;
  double sigma_multiplier;
} mcb_integrand;

typedef enum mcb_method {
  MCB_METHOD_DIRECT = 0,     /* direct_mc, ref src/estimator.cpp:75-92 */
  MCB_METHOD_STRATIFIED = 1, /* k^d grid cells, direct_mc per cell, combine_cells
                                (ref src/estimator.cpp:94-182, src/batch.cpp:255-275) */
  MCB_METHOD_TREE = 2        /* adaptive longest-edge refinement, tree_refine
                                (ref src/estimator.cpp:184-318, src/batch.cpp:276-289):
                                host-driven rounds, each round's cells batched
                                across every tree (integrand, trial) onto the GPU */
} mcb_method;

enum {
  MCB_TRIAL_OK = 0,
  MCB_TRIAL_ALL_NONFINITE = 1, /* every sample non-finite (AllSamplesNonFinite) */
  MCB_TRIAL_DEAD_CELL = 2,     /* stratified: cell `detail` had no finite sample
                                  (ref src/batch.cpp:176-180) */
  MCB_TRIAL_CELL_BUDGET = 3,   /* tree: auto initial grid exceeds cell_cap
                                  (CellBudgetExceeded, src/estimator.cpp:94-105) */
  MCB_TRIAL_CHUNK_RANGE = 4    /* tree: a cell's chunk index passed 2^32-1
                                  (std::out_of_range, src/sampling.cpp:80-81) */
};

/* Per-(integrand, trial) result = reference McEstimate
 * (include/mcbatch/estimator.hpp:18-25) plus a status replacing the
 * AllSamplesNonFinite exception (src/estimator.cpp:58-59). */
typedef struct mcb_trial_stats {
  double value;       /* volume * mean */
  double std_error;   /* volume * sqrt((m2/(n-1))/n); +inf when n < 2 */
  uint64_t n_samples; /* finite + non-finite */
  uint64_t n_nonfinite;
  uint32_t status;    /* MCB_TRIAL_* */
  uint32_t nonfinite_warning;
  uint32_t detail;    /* MCB_TRIAL_DEAD_CELL: index of the first dead cell */
  uint32_t n_cells;   /* stratified: cells combined; tree: leaves (1 for direct) */
  uint32_t budget_exhausted; /* tree: McEstimate::budget_exhausted */
  uint32_t max_depth;        /* tree: deepest leaf (0 otherwise) */
} mcb_trial_stats;

/* One leaf of a refined tree (reference StratumNode,
 * include/mcbatch/estimator.hpp:33-38). */
typedef struct mcb_leaf {
  double low[MCB_MAX_DIM];
  double high[MCB_MAX_DIM];
  mcb_trial_stats estimate; /* status ALL_NONFINITE for a dead leaf */
  uint32_t depth;
  uint32_t reserved;
} mcb_leaf;

/* One validation problem (reference Violation, include/mcbatch/batch.hpp:40-44).
 * integrand = -1 for job-level problems. */
typedef struct mcb_violation {
  int64_t integrand;
  char message[120];
} mcb_violation;

/* ---- introspection ------------------------------------------------------ */
MCB_API uint32_t mcb_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
MCB_API const char* mcb_last_error(void);
/* Number of visible CUDA devices (0 when none or the driver is absent). */
MCB_API int mcb_device_count(void);

/* ---- host-side helpers (no GPU needed) ---------------------------------- */
/* Cipher key of (seed, integrand): src/sampling.cpp:84-87. */
MCB_API void mcb_stream_key(uint64_t global_seed, uint32_t integrand_index, uint32_t key_out[2]);
/* HyperRect::volume, left-to-right product from 1.0: src/sampling.cpp:16-20. */
MCB_API double mcb_volume(const mcb_integrand* fn);
/* Exact reference DSL source for a descriptor; returns bytes needed incl. NUL. */
MCB_API size_t mcb_to_dsl(const mcb_integrand* fn, char* buf, size_t cap);
/* Reference validate() (src/batch.cpp:62-120) for a direct family job.
 * Writes up to `cap` violations, sets *n_out to the total found.
 * `names` may be NULL (then integrands are named by position, and the
 * duplicate-name check is skipped). Returns MCB_OK even if violations exist. */
MCB_API mcb_status mcb_validate(const mcb_integrand* fns, size_t n_fns, const char* const* names,
                        uint32_t trials, mcb_violation* out, size_t cap, size_t* n_out);
/* stratified_plan (ref src/batch.cpp:41-54): cells per dim, cells and
 * samples per cell of a STRATIFIED integrand.  MCB_ERR_VALIDATION when the
 * grid exceeds the cell cap ("cell grid exceeds configured cap"). */
MCB_API mcb_status mcb_stratified_plan(const mcb_integrand* fn, uint32_t* cells_per_dim,
                                       uint64_t* n_cells, uint32_t* samples_per_cell);
/* LPT shard assignment of integrands to `n_shards` devices by estimated cost
 * n_samples * trials * per-sample cost(family, dim).  Deterministic. */
MCB_API mcb_status mcb_partition(const mcb_integrand* fns, size_t n_fns, uint32_t trials,
                         int n_shards, uint32_t* shard_of_fn);
/* summarize_trials (src/estimator.cpp:320-337) over the OK trials in order. */
MCB_API mcb_status mcb_summarize_trials(const mcb_trial_stats* per_trial, uint32_t n_trials,
                                double* mean, double* trial_stddev, uint32_t* n_ok);

/* ---- DSL programs (MCB_FAMILY_PROGRAM) ------------------------------------- */
/* parse + compile (ref/src/expr.cpp:302-309 parse, :507-518 compile) of
 * `source` for `dim` coordinates and the given parameter names (any order;
 * bound in sorted order as the reference does, src/batch.cpp:129-140).
 * Errors: MCB_ERR_VALIDATION with the reference's wording in mcb_last_error
 * ("expression does not parse: ...", "x3 exceeds dim=2", "unbound parameter
 * 'q'"), or when the program exceeds the interpreter's limits (16 stack
 * slots, 1024 instructions, 512 constants, MCB_MAX_PARAMS parameters). */
MCB_API mcb_status mcb_program_compile(const char* source, uint32_t dim,
                                       const char* const* param_names, size_t n_params,
                                       mcb_program** out);
MCB_API void mcb_program_destroy(mcb_program* program);
/* n_instr, stack depth, n_params (each may be NULL). */
MCB_API mcb_status mcb_program_info(const mcb_program* program, uint32_t* n_instr,
                                    uint32_t* depth, uint32_t* n_params);
/* i-th bound parameter name in binding (sorted) order; returns bytes needed incl. NUL. */
MCB_API size_t mcb_program_param_name(const mcb_program* program, uint32_t i, char* buf,
                                      size_t cap);

/* CompiledProgram::evaluate (ref/src/expr.cpp:520-553) of `program` at
 * caller-given points, on the GPU interpreter the estimators use: `n_points`
 * rows of the program's dim coordinates (row-major), `params` in binding
 * (sorted-name) order, n_params = the program's parameter count.
 * Non-finite values are returned as they are.  Synchronous. */
MCB_API mcb_status mcb_program_eval_points(const mcb_program* program, const double* params,
                                           size_t n_params, const double* points, uint64_t n_points,
                                           int device, double* out);

/* ---- the hot path -------------------------------------------------------- */
/* run_batch (src/batch.cpp:195-333): every integrand, every trial t in
 * [0, trials), StreamKey {seed, integrand_index, t, chunk}, by each
 * integrand's method (DIRECT, STRATIFIED, TREE).
 * `out` is n_fns*trials, row-major by integrand.  Devices: `devices` lists
 * CUDA ordinals (NULL/0 = device 0); one host thread per entry.  With one
 * device every integrand runs there; with several, the (integrand, trial)
 * pairs of direct and stratified integrands are sharded by LPT on cost (tree
 * integrands: whole trees by budget).  Results are byte-identical for any
 * device list.
 * Synchronous.  `seconds` (may be NULL) receives the wall time of the
 * sampling phase (reference BatchResult.total_seconds). */
MCB_API mcb_status mcb_run_direct(const mcb_integrand* fns, size_t n_fns, uint64_t seed,
                          uint32_t trials, const int* devices, int n_devices,
                          mcb_trial_stats* out, double* seconds);

/* direct_mc (src/estimator.cpp:75-92) for one integrand and one key base
 * {seed, fn->integrand_index, trial, chunk_base}, on `device`. */
MCB_API mcb_status mcb_direct_mc(const mcb_integrand* fn, uint64_t seed, uint32_t trial,
                         uint64_t chunk_base, int device, mcb_trial_stats* out);

/* One chunk's accumulator = reference ChunkAccum (include/mcbatch/estimator.hpp:
 * 60-68): finite-sample count, non-finite count, mean and sum of squared
 * deviations of the chunk's f values. */
typedef struct mcb_chunk_accum {
  uint64_t n;
  uint64_t n_nonfinite;
  double mean;
  double m2;
} mcb_chunk_accum;

/* accumulate_chunk (include/mcbatch/estimator.hpp:70-74, src/estimator.cpp:
 * 36-49): the first `count` (<= 65536) points of the stream {seed,
 * fn->integrand_index, trial, chunk} on fn's domain, evaluated and reduced on
 * `device` (one tile of the fused kernel).  n and n_nonfinite are exact;
 * mean and m2 come from the tile's shifted sums (mean = c + S1/n, m2 = S2 -
 * S1*S1/n), within ~1e-15 relative of the reference's Welford recurrence. */
MCB_API mcb_status mcb_accumulate_chunk(const mcb_integrand* fn, uint64_t seed, uint32_t trial,
                                        uint64_t chunk, uint32_t count, int device,
                                        mcb_chunk_accum* out);

/* tree_refine (src/estimator.cpp:212-318) for one integrand (method TREE,
 * n_samples = total_budget) and key base {seed, fn->integrand_index, trial,
 * chunk_base}.  Cells are estimated on `device`.  `leaves` (may be NULL)
 * receives up to `leaf_cap` leaves in the reference's leaf order; *n_leaves
 * (may be NULL) the total.  A dead trial is reported through out->status. */
MCB_API mcb_status mcb_tree_refine(const mcb_integrand* fn, uint64_t seed, uint32_t trial,
                                   uint64_t chunk_base, int device, mcb_trial_stats* out,
                                   mcb_leaf* leaves, size_t leaf_cap, size_t* n_leaves);

/* stratified_mc (src/estimator.cpp:161-182): `cells_per_dim`^d grid cells
 * (at most `cell_cap`; 0 = 1e6), direct_mc of `samples_per_cell` samples per
 * cell with chunk keys chunk_base + c * chunk_count(samples_per_cell),
 * combine_cells.  Leaves as in mcb_tree_refine.  A cell without a finite
 * sample fails the call as in the reference (out->status MCB_TRIAL_DEAD_CELL,
 * detail = the cell); a grid past the cap gives MCB_TRIAL_CELL_BUDGET. */
MCB_API mcb_status mcb_stratified_mc(const mcb_integrand* fn, uint32_t cells_per_dim, uint32_t samples_per_cell,
                                     uint64_t cell_cap, uint64_t seed, uint32_t trial, uint64_t chunk_base,
                                     int device, mcb_trial_stats* out, mcb_leaf* leaves, size_t leaf_cap,
                                     size_t* n_leaves);

/* ---- device-resident plans (descriptors stay in HBM; async on a stream) -- */
typedef struct mcb_plan mcb_plan;
typedef struct mcb_plan_info {
  uint64_t n_fns;
  uint32_t trials;
  uint32_t n_groups;        /* (family, dim) kernel launches per run */
  uint64_t n_tiles;         /* (fn, trial, chunk) work units */
  uint64_t total_samples;   /* sum n_samples * trials */
  uint64_t philox_blocks;   /* sum over tiles of ceil(count*dim/2) */
  uint32_t launches_per_run;/* kernels launched by mcb_plan_launch */
  uint32_t reserved;
} mcb_plan_info;

MCB_API mcb_status mcb_plan_create(const mcb_integrand* fns, size_t n_fns, uint64_t seed,
                           uint32_t trials, int device, mcb_plan** plan_out);
/* Enqueue the fused sample->eval->reduce kernels plus the ordered chunk
 * combine on `stream` (NULL = legacy default stream).  No host sync. */
MCB_API mcb_status mcb_plan_launch(mcb_plan* plan, void* stream);
/* Copy the n_fns*trials results to host (synchronizes `stream`). */
MCB_API mcb_status mcb_plan_download(mcb_plan* plan, mcb_trial_stats* out, void* stream);
MCB_API mcb_status mcb_plan_get_info(const mcb_plan* plan, mcb_plan_info* info);
MCB_API void mcb_plan_destroy(mcb_plan* plan);

/* ---- test / measurement hooks ------------------------------------------- */
/* sample_uniform (src/sampling.cpp:102-112) on the GPU: `count` points of
 * `dim` coordinates starting at point `first_point` of chunk `chunk`,
 * row-major into host `out` (count*dim doubles).  Used for bit-exact tests. */
MCB_API mcb_status mcb_debug_points(uint64_t seed, uint32_t integrand_index, uint32_t trial,
                            uint64_t chunk, uint64_t first_point, uint64_t count,
                            uint32_t dim, const double* low, const double* high,
                            int device, double* out);
/* Per-sample family values f(x) for the same points (device evaluator). */
MCB_API mcb_status mcb_debug_eval(const mcb_integrand* fn, uint64_t seed, uint32_t trial,
                          uint64_t chunk, uint64_t first_point, uint64_t count,
                          int device, double* out);
/* Runtime specialisation of PROGRAM integrands: each program is compiled by
 * NVRTC into straight-line sm_100a code, bit-identical in results to the
 * bytecode interpreter.  mode 0 = off (interpreter), 1 = automatic (default:
 * specialised when the program's cubin is cached in memory or on disk, when
 * a plan (mcb_plan_create) will relaunch it, or when one launch is large
 * enough to repay its ~0.3 s compile), 2 = always (compile before the first
 * launch), < 0 = query; MCB_PROGRAM_JIT=0 / =always select 0 / 2.  Returns
 * the active mode (0 without NVRTC).  Cubins are cached in memory and on
 * disk ($MCB_JIT_CACHE, default ~/.cache/mcb-jit; "0" = off); warm the cache
 * ahead of time with mcb_program_jit_build. */
MCB_API int mcb_program_jit(int mode);
/* Compile a program's specialised kernels without a device (warms the disk
 * cache ahead of time; MCB_ERR_INVALID_ARGUMENT with the NVRTC log if the
 * generated code does not compile or NVRTC is missing). */
MCB_API mcb_status mcb_program_jit_build(const mcb_program* program);
/* NVRTC compilations so far, and the last JIT failure ("" if none). */
MCB_API uint64_t mcb_program_jit_compiles(void);
MCB_API size_t mcb_program_jit_error(char* buf, size_t cap);
/* Roofline probe: Philox4x32-10 blocks per second that `device` can generate
 * with no integrand work at all (same generator code as the fused kernel),
 * timed over ~`ms` milliseconds.  The denominator of bench.py's roofline. */
MCB_API mcb_status mcb_probe_philox_peak(int device, double ms, double* blocks_per_s);

#ifdef __cplusplus
}
#endif

#endif /* MCB_MCB_H_ */
