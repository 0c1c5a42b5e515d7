// f64 instantiations: bit-parity build, compiled with -fmad=false (reference builds with -ffp-contract=off, pkg/setup.py:21)
#define KPX_REAL double
#define KPX_SUFFIX f64
#include "kpx_inst.inl"

// float64 re-validation of batch solutions (this unit only: it must round like the reference)
#include "kpx_validate.cuh"
namespace kpx {
namespace {
template <class M>
cudaError_t do_launch_validate(const ValidateLaunch& L, cudaStream_t st) {
    ValidateArgs A;
    fill_params<double>(A.P, *L.prob);
    A.boxes = L.boxes_dev; A.queries = L.queries_dev; A.results = L.results_dev; A.chain_control = L.chain_control;
    A.chain_dt = L.chain_dt; A.n_queries = L.n_queries; A.max_chain = L.max_chain; A.res = L.res;
    validate_kernel<M><<<(L.n_queries + 127) / 128, 128, 0, st>>>(A);
    return cudaGetLastError();
}
}  // namespace
cudaError_t launch_validate_f64(const ValidateLaunch& L, cudaStream_t st) {
    const int model_id = L.prob->model_id, n = L.prob->n;
#define CALL(M) return do_launch_validate<M>(L, st)
    KPX_DISPATCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}
}  // namespace kpx
