// kpx_inst.inl -- included by the instantiation units with KPX_REAL and KPX_SUFFIX set:
//   kpx_inst_f64.cu     double, one build of every kernel (-fmad=false)
//   kpx_inst_f32.cu     float, THROUGHPUT build of the plan kernels + everything else; forwards single-query
//                       launches to ...
//   kpx_inst_f32lat.cu  float, LATENCY build of the plan kernels only (KPX_PLAN_ONLY; its own translation unit so
//                       that the two float32 builds compile in parallel)
//   kpx_inst_*p.cu      the same three with KPX_INST_RNG = KPX_RNG_PHILOX: the kernels of the "-philox" backends
#include "kpx_launch.h"

#ifndef KPX_VARIANT
#define KPX_VARIANT KPX_THROUGHPUT
#endif

namespace kpx {
namespace {

using Real = KPX_REAL;

template <class M>
cudaError_t do_launch_plan(const PlanLaunch& L, cudaStream_t st) {
    PlanArgs<Real> A;
    fill_params<Real>(A.P, *L.prob);
    A.obs = (const Real*)L.obs_dev; A.occ = L.occ_dev; A.ws = L.ws_dev; A.queries = L.queries_dev; A.results = L.results_dev;
    A.queue = L.queue_dev; A.n_queries = L.n_queries; A.n_teams = L.n_teams; A.team_ctas = L.team_ctas;
    A.max_chunks = L.max_chunks; A.stride = L.stride;
    A.claim_shift = L.claim_shift; A.max_trace = L.max_trace; A.max_chain = L.max_chain; A.resume = L.resume;
    A.max_iters = L.max_iters; A.lam_override = L.lam_override; A.t_max_s = L.t_max_s;
    A.stop_flag = L.stop_flag; A.peer_flags = L.peer_flags; A.n_peers = L.n_peers;
    A.b_chain_start = L.b_chain_start; A.b_chain_control = L.b_chain_control; A.b_chain_dt = L.b_chain_dt;
    A.idle = L.idle; A.handoff_at = L.handoff_at; A.pass_on_below = L.pass_on_below; A.susp_out = L.susp_out; A.n_susp_out = L.n_susp_out;
    A.resume_in = L.resume_in; A.n_resume_in = L.n_resume_in;
    auto kern = plan_kernel<M, Real, KPX_VARIANT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)(L.n_teams * L.team_ctas)), block(kBlock);
    if (L.cooperative) {
        void* args[] = {(void*)&A};
        return cudaLaunchCooperativeKernel((const void*)kern, grid, block, args, L.smem, st);
    }
    kern<<<grid, block, L.smem, st>>>(A);
    return cudaGetLastError();
}

#ifndef KPX_PLAN_ONLY
template <class M>
cudaError_t do_launch_batch(const BatchLaunch& L, cudaStream_t st) {
    BatchArgs<Real> A;
    fill_params<Real>(A.P, *L.prob);
    A.obs = (const Real*)L.obs_dev; A.occ = L.occ_dev; A.states = L.states_dev; A.e_slots = L.e_slots_dev; A.items = L.items;
    A.lam = L.lam; A.seed = L.seed; A.iteration = L.iteration; A.o_valid = L.o_valid; A.o_region = L.o_region;
    A.o_sub = L.o_sub; A.o_end = L.o_end; A.o_control = L.o_control; A.o_dt = L.o_dt; A.o_accept = L.o_accept;
    A.o_substeps = L.o_substeps; A.o_points = L.o_points;
    auto kern = batch_kernel<M, Real>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
    if (e != cudaSuccess) return e;
    kern<<<L.grid, kBlock, L.smem, st>>>(A);
    return cudaGetLastError();
}

#endif  // !KPX_PLAN_ONLY

template <class M>
int do_occupancy(size_t smem) {
    auto kern = plan_kernel<M, Real, KPX_VARIANT>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kBlock, smem) != cudaSuccess) return 0;
    return nb;
}

// every kernel of this unit draws from ONE generator (KPX_INST_RNG): the stream is a template property of the model
#ifndef KPX_INST_RNG
#define KPX_INST_RNG KPX_RNG_SPLITMIX64
#endif
#define KPX_MODEL(...) WithRng<__VA_ARGS__, KPX_INST_RNG>
#define KPX_DISPATCH(CALL)                                                                   \
    switch (model_id) {                                                                      \
        case KPX_MODEL_DI6: if (n == 6) { CALL(KPX_MODEL(ModelDI6)); } break;                \
        case KPX_MODEL_DUBINS6: if (n == 6) { CALL(KPX_MODEL(ModelDubins6)); } break;        \
        case KPX_MODEL_QUAD12: if (n == 12) { CALL(KPX_MODEL(ModelQuad12)); } break;         \
        case KPX_MODEL_STACKED_DI:                                                           \
            if (n == 6) { CALL(KPX_MODEL(ModelStackedDI<1>)); }                              \
            else if (n == 12) { CALL(KPX_MODEL(ModelStackedDI<2>)); }                        \
            else if (n == 24) { CALL(KPX_MODEL(ModelStackedDI<4>)); }                        \
            else if (n == 48) { CALL(KPX_MODEL(ModelStackedDI<8>)); }                        \
            break;                                                                           \
        default: break;                                                                      \
    }

}  // namespace

#define KPX_CAT2(a, b) a##b
#define KPX_CAT(a, b) KPX_CAT2(a, b)

cudaError_t KPX_CAT(launch_plan_, KPX_SUFFIX)(const PlanLaunch& L, cudaStream_t st) {
#ifdef KPX_FORWARD_LATENCY
    if (L.latency) return KPX_CAT(launch_plan_, KPX_FORWARD_LATENCY)(L, st);
#endif
    const int model_id = L.prob->model_id, n = L.prob->n;
#define CALL(M) return do_launch_plan<M>(L, st)
    KPX_DISPATCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}

#ifndef KPX_PLAN_ONLY
cudaError_t KPX_CAT(launch_batch_, KPX_SUFFIX)(const BatchLaunch& L, cudaStream_t st) {
    const int model_id = L.prob->model_id, n = L.prob->n;
#define CALL(M) return do_launch_batch<M>(L, st)
    KPX_DISPATCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}

#if KPX_INST_RNG == KPX_RNG_SPLITMIX64     // host helpers: once per precision
void KPX_CAT(occupancy_masks_, KPX_SUFFIX)(const kpx_problem& pr, int n_obs, const double* omin, const double* omax,
                                           uint32_t* masks) {
    Params<Real> P;
    fill_params<Real>(P, pr);
    build_occupancy_masks<Real>(P, n_obs, omin, omax, masks);
}

void KPX_CAT(cull_constants_, KPX_SUFFIX)(const kpx_problem& pr, double* thr4, double* lo3, double* inv3) {
    Params<Real> P;
    fill_params<Real>(P, pr);
    for (int k = 0; k < 4; ++k) thr4[k] = (double)P.d2_thr[k];
    for (int a = 0; a < 3; ++a) { lo3[a] = (double)P.occ_lo[a]; inv3[a] = (double)P.occ_inv[a]; }
}
#endif

#endif  // !KPX_PLAN_ONLY

int KPX_CAT(plan_blocks_per_sm_, KPX_SUFFIX)(int model_id, int n, size_t smem, bool latency) {
#ifdef KPX_FORWARD_LATENCY
    if (latency) return KPX_CAT(plan_blocks_per_sm_, KPX_FORWARD_LATENCY)(model_id, n, smem, true);
#endif
    (void)latency;
#define CALL(M) return do_occupancy<M>(smem)
    KPX_DISPATCH(CALL)
#undef CALL
    return 0;
}

}  // namespace kpx
