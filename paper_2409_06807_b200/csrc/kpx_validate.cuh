// kpx_validate.cuh -- float64 re-validation of batch solutions on the device.
//
// One thread per query: re-propagate the solution chain from the query's start state in float64 with the
// reference's integrator (propagate_ode, dynamics.py:242-283: S = max(4, ceil(dt/0.02)) RK4 substeps per
// segment, angle wrap after every substep) and apply the reference checker to it
// (ValidityChecker.trajectory_valid, validity.py:58-125): every sampled state finite, inside the closed state
// box and outside every closed obstacle box; between consecutive samples the full state is interpolated at the
// power-of-two densification of `res` and tested the same way; the final state lies in the closed goal ball.
// The chain is always continued from the root (validity.py:116-120 demands chaining within 1e-9, which a
// float32 tree cannot give from its stored node states), so the same kernel serves both tree precisions.
// This is the device twin of kpx_trajectory + kpx_trajectory_valid (host, kpx_api.cu); a test holds the two
// to identical verdicts.  Included by the float64 instantiation unit only (-fmad=false).
#pragma once
#include "kpx_plan.cuh"

namespace kpx {

struct ValidateArgs {
    Params<double> P;
    const double* boxes;            // device [n_scenes][n_obs][8] float64: min xyz, -, max xyz, -  (scene of a query: QueryIn::scene)
    const QueryIn* queries;
    kpx_query_result* results;
    const double* chain_control;    // [n_queries][max_chain][nu]
    const double* chain_dt;         // [n_queries][max_chain]
    int n_queries, max_chain;
    double res;
};

template <int N>
__device__ __forceinline__ bool state_ok_f64(const Params<double>& P, const double* __restrict__ boxes, const double* x) {
    bool okf = true;
#pragma unroll
    for (int d = 0; d < N; ++d) okf = okf && isfinite(x[d]);
    if (!okf) return false;
#pragma unroll
    for (int d = 0; d < N; ++d) if (x[d] < P.state_lo[d] || x[d] > P.state_hi[d]) return false;
    for (int k = 0; k < P.n_obs; ++k) {
        const double* b = boxes + 8 * k;
        if (x[0] >= b[0] && x[0] <= b[4] && x[1] >= b[1] && x[1] <= b[5] && x[2] >= b[2] && x[2] <= b[6]) return false;
    }
    return true;
}

template <class M>
__global__ void __launch_bounds__(128) validate_kernel(const __grid_constant__ ValidateArgs A) {
    constexpr int N = M::N, NU = M::NU;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= A.n_queries) return;
    kpx_query_result* r = A.results + q;
    r->checked = 0; r->check_code = 0;
    if (r->status != KPX_SOLVED) return;
    const long long L = r->chain_len;
    if (L < 0 || L > A.max_chain) { r->checked = -1; r->check_code = 5; return; }     // chain did not fit the buffer
    const QueryIn& Q = A.queries[q];
    const double* const boxes = A.boxes + (size_t)Q.scene * 8 * (size_t)A.P.n_obs;
    double cur[N], prev[N], st[N], comp[1] = {0.0};
#pragma unroll
    for (int d = 0; d < N; ++d) cur[d] = Q.start[d];
    bool ok = state_ok_f64<N>(A.P, boxes, cur);
    for (long long s = 0; s < L && ok; ++s) {
        double u[NU];
#pragma unroll
        for (int j = 0; j < NU; ++j) u[j] = A.chain_control[((size_t)q * A.max_chain + s) * NU + j];
        const double dt = A.chain_dt[(size_t)q * A.max_chain + s];
        if (!(dt > 0.0)) { ok = false; break; }
        int S = (int)ceil(dt / 0.02);                                  // dynamics.py:237-239
        if (S < 4) S = 4;
        const double h = dt / S, h6 = h / 6.0;
        for (int i = 0; i < S && ok; ++i) {
#pragma unroll
            for (int d = 0; d < N; ++d) prev[d] = cur[d];
            Stepper<typename M::Base, double>::step(cur, comp, u, h, h6);
            if (!state_ok_f64<N>(A.P, boxes, cur)) { ok = false; break; }
            const double d0 = cur[0] - prev[0], d1 = cur[1] - prev[1], d2 = cur[2] - prev[2];
            const double dist = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            long long m = 1;
            while ((double)m * A.res < dist) m <<= 1;
            for (long long j = 1; j < m && ok; ++j) {
                const double t = (double)j / (double)m;
#pragma unroll
                for (int d = 0; d < N; ++d) st[d] = prev[d] + t * (cur[d] - prev[d]);
                if (!state_ok_f64<N>(A.P, boxes, st)) ok = false;
            }
        }
    }
    if (!ok) { r->checked = -1; r->check_code = 3; return; }
    const double g0 = cur[0] - Q.goal[0], g1 = cur[1] - Q.goal[1], g2 = cur[2] - Q.goal[2];
    if (!(sqrt(g0 * g0 + g1 * g1 + g2 * g2) <= Q.goal[3])) { r->checked = -1; r->check_code = 4; return; }
    r->checked = 1;
}

}  // namespace kpx
