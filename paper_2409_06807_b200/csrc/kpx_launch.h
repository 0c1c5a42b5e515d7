// kpx_launch.h -- host-side seam between the C-ABI (kpx_api.cu) and the two
// precision instantiation units (kpx_inst_f64.cu built with -fmad=false,
// kpx_inst_f32.cu with FMA contraction on).
#pragma once
#include <cuda_runtime.h>

#include "kpx_plan.cuh"

namespace kpx {

struct PlanLaunch {
    const kpx_problem* prob;
    const void* obs_dev;            // boxes [n_obs][8] in the launch precision
    const uint32_t* occ_dev;        // occupancy masks [kOccGrid^3]
    Workspace* ws_dev;
    const QueryIn* queries_dev;
    kpx_query_result* results_dev;
    unsigned int* queue_dev;        // null: single bound query
    int n_queries, n_teams, team_ctas, max_chunks, max_trace, max_chain, stride, claim_shift;
    int resume, max_iters, lam_override;
    double t_max_s;
    const uint32_t* stop_flag;
    uint32_t* const* peer_flags;
    int n_peers;
    double *b_chain_start, *b_chain_control, *b_chain_dt;
    // hand-off of a batch's last queries to wider teams (PlanArgs, kpx_plan.cuh)
    unsigned int* idle;
    int handoff_at, pass_on_below;
    int2* susp_out; unsigned int* n_susp_out;
    const int2* resume_in; const unsigned int* n_resume_in;
    size_t smem;
    bool cooperative;
    bool latency;                   // one query on the whole GPU: the latency build of the float32 kernels
};

struct BatchLaunch {
    const kpx_problem* prob;
    const void* obs_dev;
    const uint32_t* occ_dev;
    const double* states_dev;
    const long long* e_slots_dev;
    long long items;
    int lam;
    unsigned long long seed, iteration;
    uint8_t* o_valid;
    long long *o_region, *o_sub;
    double *o_end, *o_control, *o_dt, *o_accept;
    long long *o_substeps, *o_points;
    int grid;
    size_t smem;
};

struct ValidateLaunch {
    const kpx_problem* prob;
    const double* boxes_dev;        // float64 boxes [n_obs][8]
    const QueryIn* queries_dev;
    kpx_query_result* results_dev;
    const double *chain_control, *chain_dt;
    int n_queries, max_chain;
    double res;
};

// each returns cudaErrorInvalidValue for an unsupported (model_id, n)
cudaError_t launch_validate_f64(const ValidateLaunch& L, cudaStream_t st);
cudaError_t launch_plan_f64(const PlanLaunch& L, cudaStream_t st);
cudaError_t launch_plan_f32(const PlanLaunch& L, cudaStream_t st);       // forwards L.latency launches to ...
cudaError_t launch_plan_f32lat(const PlanLaunch& L, cudaStream_t st);    // the LATENCY build (own translation unit)
cudaError_t launch_batch_f64(const BatchLaunch& L, cudaStream_t st);
cudaError_t launch_batch_f32(const BatchLaunch& L, cudaStream_t st);
// the same kernels drawing from Philox4x32-10 (kpx_problem.rng = KPX_RNG_PHILOX): own translation units
cudaError_t launch_plan_f64p(const PlanLaunch& L, cudaStream_t st);
cudaError_t launch_plan_f32p(const PlanLaunch& L, cudaStream_t st);
cudaError_t launch_plan_f32latp(const PlanLaunch& L, cudaStream_t st);
cudaError_t launch_batch_f64p(const BatchLaunch& L, cudaStream_t st);
cudaError_t launch_batch_f32p(const BatchLaunch& L, cudaStream_t st);
int plan_blocks_per_sm_f64p(int model_id, int n, size_t smem, bool latency);
int plan_blocks_per_sm_f32p(int model_id, int n, size_t smem, bool latency);
int plan_blocks_per_sm_f32latp(int model_id, int n, size_t smem, bool latency);
// host: occupancy masks (kOccGrid^3 words) computed with the launch precision's own cell arithmetic
void occupancy_masks_f64(const kpx_problem& pr, int n_obs, const double* omin, const double* omax, uint32_t* masks);
void occupancy_masks_f32(const kpx_problem& pr, int n_obs, const double* omin, const double* omax, uint32_t* masks);
// host: Params<R>::d2_thr and the occupancy lookup constants, as doubles
void cull_constants_f64(const kpx_problem& pr, double* thr4, double* lo3, double* inv3);
void cull_constants_f32(const kpx_problem& pr, double* thr4, double* lo3, double* inv3);
// co-resident CTAs per SM of the plan kernel for this model (0 if unsupported)
int plan_blocks_per_sm_f64(int model_id, int n, size_t smem, bool latency);
int plan_blocks_per_sm_f32(int model_id, int n, size_t smem, bool latency);
int plan_blocks_per_sm_f32lat(int model_id, int n, size_t smem, bool latency);

}  // namespace kpx
