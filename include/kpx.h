/*
 * kpx.h -- C ABI of the B200-native Kino-PAX planner (libkpx.so).
 *
 * Plain pointers and sizes only; no torch / C++ types cross this boundary.
 * Every entry point returns 0 on success and a nonzero KPX_E_* code on failure
 * (never throws); kpx_last_error() gives the message for the calling thread.
 *
 * Which reference interface each entry point replaces
 * (paths relative to /root/reference/pkg/src/kinopax):
 *
 *   kpx_propagate_batch      _kernel.propagate_batch           _kernel.pyx:299-379
 *                            (called by CompiledBackend,       backend.py:77-89)
 *   kpx_plan_create          KinoPax.__init__                  planner.py:137-172
 *                            (TreeArena planner.py:54-62, Decomposition arrays decomposition.py:66-74)
 *   kpx_plan_reset           init_root + make_available        planner.py:169-172
 *   kpx_plan_run             KinoPax.solve loop                planner.py:271-303
 *                            (propagate_pass :176, update_estimates_pass :206, update_node_sets_pass :212)
 *   kpx_plan_snapshot        TreeArena.snapshot                planner.py:92-102
 *   kpx_plan_regions         Decomposition state / dump_rows   decomposition.py:66-74, 219-234
 *   kpx_plan_solution        extract_trajectory (chain walk)   planner.py:325-336
 *   kpx_trajectory           propagate_ode over the chain       dynamics.py:242-283 (host, float64)
 *   kpx_trajectory_valid     ValidityChecker.segment_valid     validity.py:86-106 (host, float64)
 *   kpx_plan_trace           IterationTrace records            planner.py:121-131, 290-296
 *   kpx_plan_items           the Batch of the last iteration   backend.py:47-61
 *   kpx_plan_load            (no reference equivalent: restores a tree + region state; checkpoint/resume)
 *   kpx_batch_*              run_trials over many seeds/goals  bench.py:106-150, one launch for Q queries
 *
 * Threading: a handle is used by one host thread at a time; different handles
 * are independent.  All work is stream-ordered on the cudaStream_t passed in
 * (0 = default stream); calls that return results synchronise that stream.
 */
#ifndef KPX_H_
#define KPX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KPX_MAX_DIM 48      /* reference kernel: 16 (_kernel.pyx:66) */
#define KPX_MAX_CONTROL 24  /* reference kernel: 8  (_kernel.pyx:67) */
#define KPX_MAX_CHAIN 4096  /* longest root->goal chain kpx_plan_solution returns */

/* model ids 0..2 = _kernel.pyx:88-130; 3 = stacked 3-D double integrators (n = 6k) */
enum { KPX_MODEL_DI6 = 0, KPX_MODEL_DUBINS6 = 1, KPX_MODEL_QUAD12 = 2, KPX_MODEL_STACKED_DI = 3 };
/* random streams: same identity (seed, iteration, slot, extension, phase) and draw index, different generator */
enum { KPX_RNG_SPLITMIX64 = 0, KPX_RNG_PHILOX = 1 };
/* arithmetic of the integration / collision / grid-mapping path */
enum { KPX_F64 = 0, KPX_F32 = 1 };
/* planner status (core.py:86-90) + RUNNING for stepped runs */
enum { KPX_SOLVED = 0, KPX_TIMEOUT = 1, KPX_CAPACITY_EXHAUSTED = 2, KPX_ERROR = 3, KPX_RUNNING = 4, KPX_STOPPED = 5 };
/* node tags (planner.py:31-34) */
enum { KPX_TAG_EMPTY = 0, KPX_TAG_EXPAND = 1, KPX_TAG_OPEN = 2 };
/* error codes */
enum { KPX_OK = 0, KPX_E_ARG = 1, KPX_E_CUDA = 2, KPX_E_LIMIT = 3, KPX_E_STATE = 4 };

/* PlanContext (backend.py:27-44) + PlannerConfig (core.py:142-151), flattened. */
typedef struct kpx_problem {
    int32_t model_id;   /* KPX_MODEL_* */
    int32_t n;          /* state dimension */
    int32_t nu;         /* control dimension */
    int32_t n_obs;      /* number of AABB obstacles */
    int32_t subcells;   /* sub-cells per position dimension */
    int32_t grid_n;     /* grid spans state dims [0, grid_n); reference: grid_n == n */
    int32_t lambda_max; /* PlannerConfig.lambda_max */
    int32_t rng;        /* KPX_RNG_SPLITMIX64: the reference's streams (rng.py:30-54), bit-parity; KPX_RNG_PHILOX: Philox4x32-10 */
    int64_t t_e;        /* tree capacity: nodes the arena is allocated for */
    int64_t t_e_start;  /* adaptive capacity (paper, Remark 1; not in the reference package): capacity in effect at the
                           start, 0 = t_e.  A run that would end CAPACITY_EXHAUSTED multiplies it by t_e_growth (never */
    double t_e_growth;  /* beyond t_e) and carries on; t_e_growth <= 1 keeps the capacity fixed */
    double t_prop, check_res, epsilon, delta;
    double control_lo[KPX_MAX_CONTROL], control_hi[KPX_MAX_CONTROL];
    double state_lo[KPX_MAX_DIM], state_hi[KPX_MAX_DIM];
    double grid_lo[KPX_MAX_DIM], grid_width[KPX_MAX_DIM];
    int64_t grid_cells[KPX_MAX_DIM], grid_strides[KPX_MAX_DIM];
    const double *obs_min; /* host, (n_obs,3) row-major */
    const double *obs_max; /* host, (n_obs,3) row-major */
} kpx_problem;

/* PlanStats (core.py:112-117) + device-side accounting. */
typedef struct kpx_stats {
    int32_t status;          /* KPX_SOLVED ... */
    int32_t iterations;
    int64_t tree_size;
    int64_t solution_slot;   /* -1 if none */
    int64_t chain_len;       /* number of segments root->solution */
    double device_ms;        /* globaltimer: first iteration start -> result written */
    double reset_ms;         /* globaltimer: in-kernel workspace reset */
    uint64_t items;          /* extensions attempted (sum over iterations) */
    uint64_t substeps;       /* RK4 substeps integrated */
    uint64_t points;         /* collision points tested */
    uint64_t boxsteps;       /* substeps whose state-box test ran */
    uint64_t launches;       /* kernel launches issued by this call */
    uint64_t free_items;     /* extensions certified valid and finished from the closed form (float32 double integrators) */
    int64_t capacity;        /* tree capacity in effect when the run ended (> t_e_start after adaptive growth) */
} kpx_stats;

/* IterationTrace (planner.py:121-131). */
typedef struct kpx_trace {
    int32_t iteration, branching;
    int64_t ve_size, vo_size, attempted, valid, staged, appended, tree_size;
    double elapsed_ms;
    double phase_ms[6];  /* device time of this iteration's phases: order/S0, propagate/S1, gate/S2, append+estimates/S3,
                            node sets/S4, epilogue (scan, rescue, trace) */
} kpx_trace;

typedef struct kpx_plan kpx_plan;
typedef struct kpx_batch kpx_batch;

const char *kpx_last_error(void);
int kpx_version(void);
/* sizeof of an ABI struct as compiled: 0 kpx_problem, 1 kpx_stats, 2 kpx_trace, 3 kpx_query_result (binding self-check) */
int kpx_struct_size(int which);
/* SM count / cooperative-residency facts of the current device (for sizing and for bench.py) */
/* FP32 FMA micro-benchmark on `device` (the non-tensor roofline denominator): dense fused multiply-adds
 * on every SM for roughly `ms_target` milliseconds; *tflops counts 2 flops per FMA. */
int kpx_fma_peak(int device, double ms_target, double *tflops, double *tflops_f64);
/*
 * Host-only views of what the collision cull is built from (no CUDA call; used by the CPU test-suite):
 *  - kpx_cull_thresholds: out[k] = largest squared length d2 with fl(sqrt(d2)) <= check_res * 2^k, k = 0..3, in
 *    the arithmetic of `precision` (returned as double) -- the compare-only form of densify_steps
 *    (validity.py:26-31);
 *  - kpx_cull_tables: the 16^3 occupancy-mask table followed by its 2x2x2 dilation (2 * 4096 words), and the
 *    cell lookup's origin / scale per axis (lo[3], inv[3]) so a test can recompute cells.
 */
int kpx_cull_thresholds(const kpx_problem *prob, int32_t precision, double *out4);
int kpx_cull_tables(const kpx_problem *prob, int32_t precision, uint32_t *masks8192, double *lo3, double *inv3);

/*
 * Batched goal sampler of BASELINE.json's config 5 (8192 queries with random goals): goal of query id q = centre
 * uniform in [lo, hi]^3 from the reference's GENERIC stream of seed q (rng.py:57-95, RngStream(q, phase=5)), three
 * draws per try, rejected while closer than min_dist to start3 or inside an obstacle grown by radius + margin;
 * goals (host, n_queries x 4) = centre + radius.  One device thread per query; bit-identical to the host loop
 * batch.goal_for_query.  The reference has no batched sampler: its scenes carry one goal (envgen.py:127-163).
 */
int kpx_sample_goals(int64_t n_queries, const uint64_t *query_ids, int32_t n_obs, const double *obs_min,
                     const double *obs_max, const double *start3, double lo, double hi, double radius,
                     double min_dist, double margin, double *goals, void *stream);

/*
 * Self-test hook of the production generator: Philox4x32-10 of (counter[4], key[2]) computed on the host and by a
 * one-thread kernel on the current device (out_host[4], out_device[4]; either may be NULL) -- for the known-answer
 * vectors of the Random123 distribution.
 */
int kpx_philox4x32(const uint32_t *counter4, const uint32_t *key2, uint32_t *out_host4, uint32_t *out_device4);

int kpx_device_info(int device, int32_t *sm_count, int32_t *max_coop_blocks_f32, int32_t *max_coop_blocks_f64);

/*
 * Drop-in for _kernel.propagate_batch (_kernel.pyx:299): host arrays in, host
 * arrays out, same layouts and dtypes as the reference's Batch (backend.py:47):
 * states (rows,n) f64 row-major, e_slots (m) i64 ascending; outputs for
 * I = m*lam items: valid u8[I] (init 0), region i64[I] (init -1), sub i64[I]
 * (init 0), end f64[I,n], control f64[I,nu], dt f64[I], accept_u f64[I].
 * precision KPX_F64 reproduces the reference bit-for-bit for di6 (<=1e-12 for
 * the trig models); KPX_F32 integrates in float (end within 1e-5 relative).
 * Optional o_substeps/o_points (i64[I], may be NULL): work counters per item.
 * Returns KPX_E_LIMIT if n > KPX_MAX_DIM or nu > KPX_MAX_CONTROL (reference: ValueError).
 */
int kpx_propagate_batch(const kpx_problem *prob, const double *states, int64_t state_rows,
                        const int64_t *e_slots, int64_t m, int32_t lam, uint64_t seed, uint64_t iteration,
                        int32_t precision, uint8_t *o_valid, int64_t *o_region, int64_t *o_sub,
                        double *o_end, double *o_control, double *o_dt, double *o_accept,
                        int64_t *o_substeps, int64_t *o_points, double *o_kernel_ms, void *stream);

/*
 * One planner = one device-resident arena + region state + scratch.
 * team_ctas: CTAs cooperating on the query; 0 = whole GPU (cooperative launch).
 */
int kpx_plan_create(const kpx_problem *prob, int32_t precision, int32_t team_ctas, int32_t device,
                    kpx_plan **out);
void kpx_plan_destroy(kpx_plan *p);
/* new query on the same problem: seed, start state (n), goal (cx,cy,cz,r) */
int kpx_plan_reset(kpx_plan *p, uint64_t seed, const double *start, const double *goal4);
/* replace the obstacle set / goal without reallocating (same n_obs capacity or fewer) */
/* Test hook: overwrite the claim-table epoch the next reset starts from (the table is epoch-tagged and only
 * refilled when the epochs run out, once in 2^(32-bits(t_e)) queries; this lets a test cross that boundary). */
int kpx_plan_set_epoch(kpx_plan *p, uint32_t epoch_used);
int kpx_plan_set_obstacles(kpx_plan *p, int32_t n_obs, const double *obs_min, const double *obs_max);
/*
 * Run the device-resident loop.  t_max seconds (device clock), max_iters <= 0
 * means unlimited; lam_override > 0 forces the branching factor (tests);
 * stop_flag (device pointer to a 32-bit word, may be NULL) is polled once per
 * iteration -- nonzero stops the run with KPX_STOPPED (OR-parallel race);
 * peer_flags/n_peers: device-accessible words this run sets to 1 when it solves.
 */
int kpx_plan_run(kpx_plan *p, double t_max, int32_t max_iters, int32_t lam_override,
                 uint32_t *stop_flag, uint32_t *const *peer_flags, int32_t n_peers,
                 kpx_stats *out, void *stream);
/* tree in the reference's snapshot layout (planner.py:92): host buffers sized by tree_size */
int kpx_plan_snapshot(kpx_plan *p, int64_t rows, double *states, int64_t *parent, double *control,
                      double *dt, uint8_t *tag, int64_t *region);
/* region state, each array of n_regions (visited: n_regions*subcells^3) elements; any pointer may be NULL */
int kpx_plan_regions(kpx_plan *p, int64_t *n_valid, int64_t *n_invalid, int64_t *cov, double *free_vol,
                     double *score, double *p_accept, uint8_t *visited, uint8_t *avail);
/* solution chain: for each of chain_len segments the start state (n), control (nu), dt, and the slot */
int kpx_plan_solution(kpx_plan *p, int64_t max_segments, double *seg_start, double *seg_control,
                      double *seg_dt, int64_t *seg_slot, double *end_state);
/*
 * Host-side float64 rebuild of a solution: segment s integrates seg_control[s] for seg_dt[s] with the
 * reference's fixed-step RK4 (S = max(4, ceil(dt/0.02)) substeps) from seg_start[s] -- or, with
 * chain_from_root, from the previous segment's end (seg_start[0] = root).  sampled receives
 * S+1 rows per segment; seg_offset[n_seg+1] the row offsets.  No device work.
 */
/*
 * extract_trajectory of the solved plan in ONE host call (planner.py:325-341): fetch the device-built chain
 * (already on the host in the result packet of kpx_plan_run), rebuild it in float64 like kpx_trajectory and -- when
 * `start` is given, i.e. the chain is continued from the root (float32 trees) -- check it like kpx_trajectory_valid
 * against `goal4` at resolution `res`.  Outputs: seg_control (n_seg, nu), seg_dt (n_seg), sampled (rows, n),
 * seg_offset (n_seg + 1), *ok / *fail_code as kpx_trajectory_valid (ok = 1 when no check was asked for).
 */
int kpx_plan_trajectory(kpx_plan *p, const double *start, const double *goal4, double res, int64_t max_seg,
                        int64_t max_rows, double *seg_control, double *seg_dt, double *sampled,
                        int64_t *seg_offset, int64_t *n_seg, int32_t *ok, int32_t *fail_code);
int kpx_trajectory(int32_t model_id, int32_t n, int32_t nu, int64_t n_seg, const double *seg_start,
                   const double *seg_control, const double *seg_dt, int32_t chain_from_root,
                   double *sampled, int64_t max_rows, int64_t *seg_offset);
/* Host-side check of a rebuilt trajectory with the reference checker's rules (validity.py:58-106, closed
 * boxes, power-of-two densification at `res`) plus the closed goal ball; *ok = 1/0, *fail_code 3 segment / 4 goal. */
int kpx_trajectory_valid(const kpx_problem *prob, int64_t n_seg, const double *sampled, const int64_t *seg_offset,
                         const double *goal4, double res, int32_t *ok, int32_t *fail_code);
int kpx_plan_trace(kpx_plan *p, int32_t max_records, kpx_trace *out, int32_t *n_records);
/* the last iteration's per-item results in Batch layout + keep flag, parent slot and the kernel's own goal test
 * of the end state (debug/parity; any output may be NULL) */
int kpx_plan_items(kpx_plan *p, int64_t max_items, int64_t *n_items, uint8_t *valid, int64_t *region,
                   int64_t *sub, double *end, uint8_t *keep, int64_t *parent_slot, uint8_t *goal_hit);
/* restore a tree + region state produced elsewhere (checkpoint/resume; parity tests load oracle states) */
int kpx_plan_load(kpx_plan *p, uint64_t seed, const double *goal4, int32_t iteration, int64_t rows,
                  const double *states, const int64_t *parent, const double *control, const double *dt,
                  const uint8_t *tag, const int64_t *region, const int64_t *n_valid,
                  const int64_t *n_invalid, const int64_t *cov, const double *score, const double *p_accept,
                  const uint8_t *visited, const uint8_t *avail);

/*
 * Many independent queries in one persistent launch: n_teams teams of
 * team_ctas CTAs each pull queries from a device-side queue; every team owns
 * one workspace.  Results are written per query.
 */
typedef struct kpx_query_result {
    int32_t status, iterations;
    int64_t tree_size, solution_slot, chain_len;
    double device_ms;
    uint64_t items, substeps, points, boxsteps, free_items;
    int64_t capacity;    /* tree capacity in effect when the query ended */
    int32_t checked;     /* kpx_batch_validate: 1 = solution re-validated in float64, -1 = rejected, 0 = not checked */
    int32_t check_code;  /* 0 ok, 3 a state or interpolant is invalid, 4 goal missed, 5 chain longer than max_chain */
} kpx_query_result;

int kpx_batch_create(const kpx_problem *prob, int32_t precision, int32_t n_teams, int32_t team_ctas,
                     int32_t max_chain, int32_t device, kpx_batch **out);
/* teams / CTAs per team the batch was created with (n_teams = 0 at creation: as many teams as are co-resident;
 * n_teams = -k: min(k, co-resident), for callers that know how many queries they will ever upload;
 * team_ctas = 0: 1, 2, 4, 8 or 16 CTAs per team, the widest that keeps all n_teams teams co-resident -- the
 * trial runner's choice: 100 trials on a device that holds 592 CTAs plan on teams of 4) */
int kpx_batch_info(const kpx_batch *b, int32_t *n_teams, int32_t *team_ctas);
/* Hand-off of a batch's stragglers (default on, batches of >= 16 queries): when the query queue is empty and half of
 * the teams have run out of work, kpx_batch_launch ends its first kernel after the current iteration of the teams still
 * planning and continues those queries in a second one on teams of twice the width, and so on through teams of
 * 2, 4, 8, 16, 64 and finally all co-resident CTAs -- KPX_HANDOFF_STAGES follow-up launches on the caller's stream,
 * no host synchronisation; a stage whose queries already fit the next one passes them straight on.  Results are those
 * of the one-CTA run (a plan does not depend on the team size); only device_ms of the handed-off queries is shorter.
 * No reference counterpart: the reference plans one query per process (bench.py:106-171). */
#define KPX_HANDOFF_STAGES 6
int kpx_batch_set_handoff(kpx_batch *b, int32_t enable);
/* queries the last kpx_batch_launch handed on at the end of its first kernel (counts[0]) and of every follow-up stage
 * (counts[1 .. KPX_HANDOFF_STAGES - 1]); synchronises the device */
int kpx_batch_handoff_counts(kpx_batch *b, int32_t *counts);
void kpx_batch_destroy(kpx_batch *b);
/* seeds[Q], starts[Q,n], goals[Q,4] host arrays; chain buffers (may be NULL) sized Q*max_chain */
int kpx_batch_run(kpx_batch *b, int64_t n_queries, const uint64_t *seeds, const double *starts,
                  const double *goals, double t_max, kpx_query_result *results, double *chain_start,
                  double *chain_control, double *chain_dt, double *o_kernel_ms, void *stream);

/*
 * Obstacle sets a query can name ("scenes"): n_scenes sets of n_obs[s] boxes each, concatenated in obs_min / obs_max
 * ((sum n_obs, 3) row-major).  Every set must fit the obstacle count the batch was created with; scene 0 replaces the
 * problem's own.  The workspace box, the model and the configuration are shared.  The reference plans one
 * Environment per process (envgen.py:127-163, core.py:51-83); this is its batched form.
 */
int kpx_batch_set_scenes(kpx_batch *b, int32_t n_scenes, const int32_t *n_obs, const double *obs_min,
                         const double *obs_max);
/* kpx_batch_upload with the scene of every query (scene_idx[Q], NULL = all scene 0) */
int kpx_batch_upload_scenes(kpx_batch *b, int64_t n_queries, const uint64_t *seeds, const double *starts,
                            const double *goals, const int32_t *scene_idx, int32_t want_chains, void *stream);

/* the same in three stream-ordered pieces, so a caller can keep queries resident and re-launch:
 * upload (H2D, synchronous), launch (asynchronous, one persistent kernel), download (D2H, synchronises) */
int kpx_batch_upload(kpx_batch *b, int64_t n_queries, const uint64_t *seeds, const double *starts,
                     const double *goals, int32_t want_chains, void *stream);
int kpx_batch_launch(kpx_batch *b, double t_max, void *stream);
/*
 * Re-validate every solved query of the last kpx_batch_launch on the device, in float64, with the reference
 * checker's rules (ValidityChecker.trajectory_valid, validity.py:108-125, on the trajectory that
 * propagate_ode, dynamics.py:242-283, rebuilds from the query's start state): fills `checked` / `check_code`
 * of the per-query records that kpx_batch_download returns.  Needs want_chains = 1 at upload.  `res` <= 0
 * selects the problem's check_res.  Asynchronous on `stream`.  Replaces a host loop over
 * extract_trajectory (planner.py:325-341) + trajectory_valid per query.
 */
int kpx_batch_validate(kpx_batch *b, double res, void *stream);

int kpx_batch_download(kpx_batch *b, kpx_query_result *results, double *chain_start, double *chain_control,
                       double *chain_dt, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* KPX_H_ */
