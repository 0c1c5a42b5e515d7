// kpx_device.cuh -- device building blocks of the B200 Kino-PAX planner.
//
//  * counter RNG (SplitMix64 chain, bit-identical to reference rng.py:30-54)
//  * robot models as compile-time traits (vector fields of _kernel.pyx:84-130)
//  * propagate_item<M,R>: one tree extension = sample (u,dt), RK4 in registers,
//    per-substep finite/box/AABB walk against obstacles staged in shared memory,
//    clamped grid mapping.  Semantics follow _kernel.pyx:157-296 line by line
//    (SURVEY.md section 9 lists the rules); R=double built with -fmad=false is
//    bit-exact for the double integrator, R=float is the throughput path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

#include "../../include/kpx.h"

namespace kpx {

constexpr int kBlock = 256;          // threads per CTA of every kernel here
constexpr int kChunk = 4 * kBlock;   // slots / items per ordered-compaction chunk
constexpr int kOccGrid = 16;         // occupancy-mask grid resolution per axis (16 KB of shared memory)
constexpr uint32_t kUnclaimed = 0xFFFFFFFFu;
constexpr uint32_t kVisited = 0xFFFFFFFEu;
constexpr uint32_t kItemInvalid = 0xFFFFFFFFu;
constexpr uint32_t kItemGoalBit = 0x80000000u;

enum : int { PH_SAMPLE = 1, PH_ACCEPT = 2, PH_DEMOTE = 3, PH_PROMOTE = 4 };

// ------------------------------------------------------------------ RNG ----
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// key = mix(mix(mix(h0 ^ slot) ^ ext) ^ phase), h0 = mix(mix(seed) ^ iteration)  (rng.py:38-44)
__host__ __device__ __forceinline__ uint64_t iter_hash(uint64_t seed, uint64_t it) { return mix64(mix64(seed) ^ it); }
__host__ __device__ __forceinline__ uint64_t slot_ext_hash(uint64_t h0, uint64_t slot, uint64_t ext) {
    return mix64(mix64(h0 ^ slot) ^ ext);
}
__host__ __device__ __forceinline__ uint64_t draw_u64(uint64_t key, uint64_t i) {
    return mix64(key ^ ((i + 1) * 0x9E3779B97F4A7C15ULL));
}
__host__ __device__ __forceinline__ double unit53(uint64_t x) {
    return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}
// one keyed uniform: phase stream of (slot, ext), draw 0
__device__ __forceinline__ double keyed_uniform(uint64_t h0, uint64_t slot, uint64_t ext, int phase) {
    return unit53(draw_u64(mix64(slot_ext_hash(h0, slot, ext) ^ (uint64_t)phase), 0));
}

// ------------------------------------------------------- typed parameters ----
template <class R>
struct Params {
    int n, nu, n_obs, subcells, grid_n, lambda_max;
    long long t_e;
    double t_prop, epsilon, delta, vol;   // RNG / estimates always in f64
    double control_lo[KPX_MAX_CONTROL], control_span[KPX_MAX_CONTROL];  // span = hi - lo (f64, as reference)
    R check_res;
    R state_lo[KPX_MAX_DIM], state_hi[KPX_MAX_DIM];
    R grid_lo[KPX_MAX_DIM], grid_width[KPX_MAX_DIM];
    R grid_cmax[KPX_MAX_DIM];             // (R)(cells-1)
    int grid_strides[KPX_MAX_DIM];
    int n_regions, subs_per_region;
    // occupancy-mask grid over the position box (0 = disabled -> every obstacle is tested)
    int occ_g;
    R occ_lo[3], occ_inv[3];
};

template <class R>
inline void fill_params(Params<R>& P, const kpx_problem& pr) {
    P.n = pr.n; P.nu = pr.nu; P.n_obs = pr.n_obs; P.subcells = pr.subcells; P.grid_n = pr.grid_n;
    P.lambda_max = pr.lambda_max; P.t_e = pr.t_e;
    P.t_prop = pr.t_prop; P.epsilon = pr.epsilon; P.delta = pr.delta;
    P.vol = pr.grid_width[0] * pr.grid_width[1] * pr.grid_width[2];  // decomposition.py:64
    for (int j = 0; j < KPX_MAX_CONTROL; ++j) {
        P.control_lo[j] = j < pr.nu ? pr.control_lo[j] : 0.0;
        P.control_span[j] = j < pr.nu ? pr.control_hi[j] - pr.control_lo[j] : 0.0;
    }
    P.check_res = (R)pr.check_res;
    long long regions = 1;
    for (int d = 0; d < KPX_MAX_DIM; ++d) {
        bool in = d < pr.n, ing = d < pr.grid_n;
        P.state_lo[d] = in ? (R)pr.state_lo[d] : (R)0; P.state_hi[d] = in ? (R)pr.state_hi[d] : (R)0;
        P.grid_lo[d] = ing ? (R)pr.grid_lo[d] : (R)0; P.grid_width[d] = ing ? (R)pr.grid_width[d] : (R)1;
        P.grid_cmax[d] = ing ? (R)(pr.grid_cells[d] - 1) : (R)0;
        P.grid_strides[d] = ing ? (int)pr.grid_strides[d] : 0;
        if (ing) regions *= pr.grid_cells[d];
    }
    P.n_regions = (int)regions;
    P.subs_per_region = pr.subcells * pr.subcells * pr.subcells;
    P.occ_g = (pr.n_obs > 0 && pr.n_obs <= 32) ? kOccGrid : 0;
    for (int a = 0; a < 3; ++a) {
        P.occ_lo[a] = (R)pr.state_lo[a];
        P.occ_inv[a] = (R)((double)kOccGrid / (pr.state_hi[a] - pr.state_lo[a]));
    }
}

// Cell of a coordinate along one axis.  Both operations round monotonically, so p in [omin, omax] implies
// cell(omin) <= cell(p) <= cell(omax): computing an obstacle's cell range with this very function (same
// precision, same constants) yields masks that are exactly conservative without any safety margin.
template <class R>
__host__ __device__ __forceinline__ int occ_cell(R p, R lo, R inv) {
    int c = (int)((p - lo) * inv);
    return c < 0 ? 0 : (c > kOccGrid - 1 ? kOccGrid - 1 : c);
}

// Host: cell -> bitmask of the obstacles whose closed box (as rounded to R) can contain a point of that cell.
template <class R>
inline void build_occupancy_masks(const Params<R>& P, int n_obs, const double* omin, const double* omax,
                                  uint32_t* masks /* kOccGrid^3 */) {
    const int G = kOccGrid;
    for (int i = 0; i < G * G * G; ++i) masks[i] = 0u;
    for (int k = 0; k < n_obs && k < 32; ++k) {
        int lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = occ_cell<R>((R)omin[3 * k + a], P.occ_lo[a], P.occ_inv[a]);
            hi[a] = occ_cell<R>((R)omax[3 * k + a], P.occ_lo[a], P.occ_inv[a]);
        }
        for (int x = lo[0]; x <= hi[0]; ++x)
            for (int y = lo[1]; y <= hi[1]; ++y)
                for (int z = lo[2]; z <= hi[2]; ++z) masks[(x * G + y) * G + z] |= 1u << k;
    }
}

// ----------------------------------------------------------------- models ----
template <class R> struct MathK;
template <> struct MathK<double> {
    static constexpr double PI = 3.14159265358979323846, TWO_PI = 2.0 * 3.14159265358979323846;
    __device__ static __forceinline__ void sc(double x, double* s, double* c) { *s = sin(x); *c = cos(x); }
    __device__ static __forceinline__ double mod(double a, double b) { return fmod(a, b); }
    __device__ static __forceinline__ double sq(double x) { return sqrt(x); }
    __device__ static __forceinline__ double fl(double x) { return floor(x); }
};
template <> struct MathK<float> {
    static constexpr float PI = 3.14159265358979323846f, TWO_PI = 2.0f * 3.14159265358979323846f;
    // sin and cos together for the wrapped angles of the models (|x| is a few radians): Cody-Waite quadrant
    // reduction with the magic-number round (no int<->float conversions) and the Cephes minimax polynomials
    // on [-pi/4, pi/4]; max error 9e-8 absolute (1.4 ulp), ~22 instructions for the pair versus ~50 for
    // sincosf, whose general-range reduction these arguments never need.
    __device__ static __forceinline__ void sc(float x, float* s, float* c) {
        if (!(fabsf(x) < 512.0f)) { sincosf(x, s, c); return; }        // diverged states: library path
        const float t = __fmaf_rn(x, 0.636619772f, 12582912.0f);
        const int q = __float_as_int(t);
        const float qf = t - 12582912.0f;
        float r = __fmaf_rn(qf, -1.57079637f, x);
        r = __fmaf_rn(qf, 4.37113883e-8f, r);
        const float z = r * r;
        float sp = __fmaf_rn(z, -1.9515295891e-4f, 8.3321608736e-3f);
        sp = __fmaf_rn(z, sp, -1.6666654611e-1f);
        const float sv = __fmaf_rn(z * r, sp, r);
        float cp = __fmaf_rn(z, 2.443315711809948e-5f, -1.388731625493765e-3f);
        cp = __fmaf_rn(z, cp, 4.166664568298827e-2f);
        const float cv = __fmaf_rn(z * z, cp, __fmaf_rn(z, -0.5f, 1.0f));
        const bool swap = q & 1;
        float so = swap ? cv : sv, co = swap ? sv : cv;
        if (q & 2) so = -so;
        if ((q + 1) & 2) co = -co;
        *s = so; *c = co;
    }
    __device__ static __forceinline__ float mod(float a, float b) { return fmodf(a, b); }
    __device__ static __forceinline__ float sq(float x) { return sqrtf(x); }
    __device__ static __forceinline__ float fl(float x) { return floorf(x); }
};

// wrap to (-pi, pi]  (_kernel.pyx:77-81).  fmod only changes t outside [0, 2pi);
// the in-range fast path returns the identical value.
template <class R>
__device__ __forceinline__ R wrap_angle(R a) {
    R t = a + MathK<R>::PI;
    if (!(t >= (R)0 && t < MathK<R>::TWO_PI)) t = MathK<R>::mod(t, MathK<R>::TWO_PI);
    if (t <= (R)0) t += MathK<R>::TWO_PI;
    return t - MathK<R>::PI;
}

struct ModelDI6 {
    static constexpr int ID = KPX_MODEL_DI6, N = 6, NU = 3;
    template <class R> __device__ static __forceinline__ void deriv(const R* x, const R* u, R* o) {
        o[0] = x[3]; o[1] = x[4]; o[2] = x[5]; o[3] = u[0]; o[4] = u[1]; o[5] = u[2];
    }
    template <class R> __device__ static __forceinline__ void wrap(R*) {}
};

struct ModelDubins6 {
    static constexpr int ID = KPX_MODEL_DUBINS6, N = 6, NU = 3;
    template <class R> __device__ static __forceinline__ void deriv(const R* x, const R* u, R* o) {
        R st, ct, sg, cg;
        MathK<R>::sc(x[4], &st, &ct);
        MathK<R>::sc(x[5], &sg, &cg);
        R v = x[3];
        o[0] = v * ct * cg; o[1] = v * st * cg; o[2] = v * sg;
        o[3] = u[0]; o[4] = u[1]; o[5] = u[2];
    }
    template <class R> __device__ static __forceinline__ void wrap(R* x) { x[4] = wrap_angle(x[4]); }
};

struct ModelQuad12 {
    static constexpr int ID = KPX_MODEL_QUAD12, N = 12, NU = 4;
    template <class R> __device__ static __forceinline__ void deriv(const R* x, const R* u, R* o) {
        R sphi, cphi, sth, cth, spsi, cpsi;
        MathK<R>::sc(x[6], &sphi, &cphi);
        MathK<R>::sc(x[7], &sth, &cth);
        MathK<R>::sc(x[8], &spsi, &cpsi);
        R p = x[9], q = x[10], r = x[11];
        o[0] = x[3]; o[1] = x[4]; o[2] = x[5];
        if constexpr (std::is_same<R, double>::value) {
            // expression shapes of _kernel.pyx:117-130 (m=1, J=diag(.01,.01,.02), g=9.81)
            R acc = u[0] / 1.0;
            o[3] = acc * (cphi * sth * cpsi + sphi * spsi);
            o[4] = acc * (cphi * sth * spsi - sphi * cpsi);
            o[5] = acc * (cphi * cth) - 9.81;
            R sw = q * sphi + r * cphi;
            o[6] = p + sw * (sth / cth);
            o[7] = q * cphi - r * sphi;
            o[8] = sw / cth;
            o[9] = (u[1] - (0.02 - 0.01) * q * r) / 0.01;
            o[10] = (u[2] - (0.01 - 0.02) * p * r) / 0.01;
            o[11] = (u[3] - (0.01 - 0.01) * p * q) / 0.02;
        } else {
            R acc = u[0];
            o[3] = acc * (cphi * sth * cpsi + sphi * spsi);
            o[4] = acc * (cphi * sth * spsi - sphi * cpsi);
            o[5] = acc * (cphi * cth) - 9.81f;
            R sw = q * sphi + r * cphi;
            R icth = 1.0f / cth;
            o[6] = p + sw * (sth * icth);
            o[7] = q * cphi - r * sphi;
            o[8] = sw * icth;
            o[9] = (u[1] - 0.01f * q * r) * 100.0f;
            o[10] = (u[2] + 0.01f * p * r) * 100.0f;
            o[11] = u[3] * 50.0f;
        }
    }
    template <class R> __device__ static __forceinline__ void wrap(R* x) {
        x[6] = wrap_angle(x[6]); x[7] = wrap_angle(x[7]); x[8] = wrap_angle(x[8]);
    }
};

// B stacked 3-D double integrators, state [p1 v1 p2 v2 ...]; only block 1 is workspace position.
template <int B>
struct ModelStackedDI {
    static constexpr int ID = KPX_MODEL_STACKED_DI, N = 6 * B, NU = 3 * B;
    template <class R> __device__ static __forceinline__ void deriv(const R* x, const R* u, R* o) {
#pragma unroll
        for (int b = 0; b < B; ++b) {
            o[6 * b + 0] = x[6 * b + 3]; o[6 * b + 1] = x[6 * b + 4]; o[6 * b + 2] = x[6 * b + 5];
            o[6 * b + 3] = u[3 * b + 0]; o[6 * b + 4] = u[3 * b + 1]; o[6 * b + 5] = u[3 * b + 2];
        }
    }
    template <class R> __device__ static __forceinline__ void wrap(R*) {}
};

// One RK4 substep with zero-order hold.  Accumulating k1 + 2k2 + 2k3 + k4 left to
// right keeps the reference's rounding order (_kernel.pyx:223) with 3 live vectors.
// float32 only: the state update is Kahan-compensated (`comp` carries the running
// rounding error across substeps), which keeps ~50 chained substeps within a few
// float32 ulps of the float64 trajectory; float64 uses the plain reference expression.
template <class M, class R>
__device__ __forceinline__ void rk4_step(R* cur, R* comp, const R* u, R h, R half_h, R h6) {
    R k[M::N], acc[M::N], tmp[M::N];
    M::template deriv<R>(cur, u, k);
#pragma unroll
    for (int i = 0; i < M::N; ++i) { acc[i] = k[i]; tmp[i] = cur[i] + half_h * k[i]; }
    M::template deriv<R>(tmp, u, k);
#pragma unroll
    for (int i = 0; i < M::N; ++i) { acc[i] = acc[i] + (R)2 * k[i]; tmp[i] = cur[i] + half_h * k[i]; }
    M::template deriv<R>(tmp, u, k);
#pragma unroll
    for (int i = 0; i < M::N; ++i) { acc[i] = acc[i] + (R)2 * k[i]; tmp[i] = cur[i] + h * k[i]; }
    M::template deriv<R>(tmp, u, k);
#pragma unroll
    for (int i = 0; i < M::N; ++i) {
        if constexpr (std::is_same<R, float>::value) {
            const float y = __fmaf_rn(h6, acc[i] + k[i], -comp[i]);
            const float t = __fadd_rn(cur[i], y);
            comp[i] = __fsub_rn(__fsub_rn(t, cur[i]), y);
            cur[i] = t;
        } else {
            cur[i] = cur[i] + h6 * (acc[i] + k[i]);
        }
    }
    M::template wrap<R>(cur);
}

// Stacked double integrators: the blocks do not couple, so stepping them one 6-D block
// at a time performs exactly the same operations per dimension while keeping only a
// 6-D set of RK4 temporaries live (N = 48 would otherwise need ~200 registers).
template <int B, class R>
__device__ __forceinline__ void rk4_step_blocks(R* cur, R* comp, const R* u, R h, R half_h, R h6) {
#pragma unroll
    for (int b = 0; b < B; ++b) rk4_step<ModelDI6, R>(cur + 6 * b, comp + 6 * b, u + 3 * b, h, half_h, h6);
}
template <class M, class R>
struct Stepper {
    __device__ static __forceinline__ void step(R* cur, R* comp, const R* u, R h, R half_h, R h6) {
        rk4_step<M, R>(cur, comp, u, h, half_h, h6);
    }
};
template <int B, class R>
struct Stepper<ModelStackedDI<B>, R> {
    __device__ static __forceinline__ void step(R* cur, R* comp, const R* u, R h, R half_h, R h6) {
        rk4_step_blocks<B, R>(cur, comp, u, h, half_h, h6);
    }
};

// closed-box point test against obstacles staged in shared memory as SoA
// [minx | miny | minz | maxx | maxy | maxz], each n_obs long (all lanes read the
// same k -> broadcast).  _kernel.pyx:142-154.
template <class R>
__device__ __forceinline__ bool point_hits(R px, R py, R pz, const R* __restrict__ s_obs, int n_obs) {
    bool h = false;
    for (int k = 0; k < n_obs; ++k) {
        bool in = px >= s_obs[k] && px <= s_obs[3 * n_obs + k] && py >= s_obs[n_obs + k] &&
                  py <= s_obs[4 * n_obs + k] && pz >= s_obs[2 * n_obs + k] && pz <= s_obs[5 * n_obs + k];
        h = h || in;
    }
    return h;
}

// Same verdict through the occupancy grid: look up the point's cell, test only the flagged obstacles.
template <class R>
__device__ __forceinline__ bool point_hits_grid(const Params<R>& P, R px, R py, R pz, const R* __restrict__ s_obs,
                                                const uint32_t* __restrict__ s_occ, int n_obs) {
    if (P.occ_g == 0) return point_hits<R>(px, py, pz, s_obs, n_obs);
    const int ix = occ_cell<R>(px, P.occ_lo[0], P.occ_inv[0]);
    const int iy = occ_cell<R>(py, P.occ_lo[1], P.occ_inv[1]);
    const int iz = occ_cell<R>(pz, P.occ_lo[2], P.occ_inv[2]);
    uint32_t m = s_occ[(ix * kOccGrid + iy) * kOccGrid + iz];
    bool h = false;
    while (m) {
        const int k = __ffs(m) - 1;
        m &= m - 1;
        h = h || (px >= s_obs[k] && px <= s_obs[3 * n_obs + k] && py >= s_obs[n_obs + k] && py <= s_obs[4 * n_obs + k] &&
                  pz >= s_obs[2 * n_obs + k] && pz <= s_obs[5 * n_obs + k]);
    }
    return h;
}

template <class R, int N>
struct ItemOut {
    R end[N];
    double accept_u;   // not filled by propagate_item (cheap to regenerate from the key)
    int region;        // -1 if the integration went non-finite
    int sub;
    int substeps;      // RK4 substeps actually integrated
    int points;        // collision points tested
    int boxsteps;      // substeps whose state-box test ran (the segment was still valid)
    bool valid;
};

// The extension itself.  `u` and `dt` are the sampled control / duration already
// rounded to R; x0 is the parent state.
template <class M, class R>
__device__ __forceinline__ void integrate_and_map(const Params<R>& P, const R* __restrict__ s_obs,
                                                  const uint32_t* __restrict__ s_occ, const R* x0,
                                                  const R* u, R dt, int substeps, ItemOut<R, M::N>& out) {
    constexpr int N = M::N;
    R h = dt / (R)substeps, half_h = (R)0.5 * h, h6 = h / (R)6;
    R cur[N];
    R comp[std::is_same<R, float>::value ? N : 1];   // Kahan carry (float32 only)
#pragma unroll
    for (int i = 0; i < N; ++i) { cur[i] = x0[i]; if constexpr (std::is_same<R, float>::value) comp[i] = 0.0f; }
    R prev0 = cur[0], prev1 = cur[1], prev2 = cur[2];
    bool ok = true, alive = true;
    int done = 0, points = 0, boxsteps = 0;
    const int n_obs = P.n_obs;
    for (int s = 0; s < substeps; ++s) {
        Stepper<M, R>::step(cur, comp, u, h, half_h, h6);
        ++done;
        bool fin = true;
#pragma unroll
        for (int i = 0; i < N; ++i) fin = fin && isfinite(cur[i]);
        if (!fin) { alive = false; ok = false; break; }
        if (ok) {
            ++boxsteps;
            bool inb = true;
#pragma unroll
            for (int i = 0; i < N; ++i) inb = inb && !(cur[i] < P.state_lo[i] || cur[i] > P.state_hi[i]);
            ok = inb;
            if (ok && n_obs > 0) {
                R dx = cur[0] - prev0, dy = cur[1] - prev1, dz = cur[2] - prev2;
                R dist = MathK<R>::sq(dx * dx + dy * dy + dz * dz);
                // smallest power of two with steps * res >= dist (validity.py:26-31).  res * 2^k and 2^-k are
                // exact, so doubling the threshold / halving the fraction reproduces steps * res and j / steps
                // bit for bit without integer->float conversions.
                int steps = 1;
                R thr = P.check_res, inv_steps = (R)1;
                while (thr < dist) { thr += thr; inv_steps *= (R)0.5; steps <<= 1; }
                R t = (R)0;
                for (int j = 1; j < steps; ++j) {
                    t += inv_steps;
                    ++points;
                    if (point_hits_grid<R>(P, prev0 + t * dx, prev1 + t * dy, prev2 + t * dz, s_obs, s_occ, n_obs)) { ok = false; break; }
                }
                if (ok) { ++points; if (point_hits_grid<R>(P, cur[0], cur[1], cur[2], s_obs, s_occ, n_obs)) ok = false; }
            }
        }
        prev0 = cur[0]; prev1 = cur[1]; prev2 = cur[2];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) out.end[i] = cur[i];
    out.substeps = done; out.points = points; out.boxsteps = boxsteps;
    out.region = -1; out.sub = 0; out.valid = false;
    if (alive) {
        int reg = 0;
        R rel3[3], cell3[3];
#pragma unroll
        for (int d = 0; d < N; ++d) {
            if (d < P.grid_n) {
                R rel = (cur[d] - P.grid_lo[d]) / P.grid_width[d];
                R cl = rel < (R)0 ? (R)0 : (rel > P.grid_cmax[d] ? P.grid_cmax[d] : rel);
                R fl = MathK<R>::fl(cl);
                reg += (int)fl * P.grid_strides[d];
                if (d < 3) { rel3[d] = rel; cell3[d] = fl; }
            }
        }
        out.region = reg;
        if (ok) {
            int sub = 0;
            R smax = (R)(P.subcells - 1);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                R fr = (rel3[d] - cell3[d]) * (R)P.subcells;
                fr = fr < (R)0 ? (R)0 : (fr > smax ? smax : fr);
                sub = sub * P.subcells + (int)MathK<R>::fl(fr);
            }
            out.sub = sub;
            out.valid = true;
        }
    }
}

// Sample (u, dt) for item (slot, ext) of the iteration hashed into h0.  Controls and
// duration are drawn in f64 exactly as the reference does (_kernel.pyx:190-194) and
// then rounded once to R; the substep count is taken from the rounded dt so that a
// host re-propagation of the stored (control, dt) uses the same step size.
template <class M, class R>
__device__ __forceinline__ void sample_control(const Params<R>& P, uint64_t h0, int slot, int ext, R* u, R* dt,
                                               int* substeps, double* u64v, double* dt64) {
    uint64_t key = mix64(slot_ext_hash(h0, (uint64_t)slot, (uint64_t)ext) ^ (uint64_t)PH_SAMPLE);
#pragma unroll
    for (int j = 0; j < M::NU; ++j) {
        double v = __dadd_rn(P.control_lo[j], __dmul_rn(unit53(draw_u64(key, (uint64_t)j)), P.control_span[j]));
        if (u64v) u64v[j] = v;
        u[j] = (R)v;
    }
    double d = __dmul_rn(__dsub_rn(1.0, unit53(draw_u64(key, (uint64_t)M::NU))), P.t_prop);
    if (dt64) *dt64 = d;
    *dt = (R)d;
    int s = (int)ceil(__ddiv_rn((double)(*dt), 0.02));
    *substeps = s < 4 ? 4 : s;
}

// substep count of item (slot, ext) alone: the duration draw and the same rounding as sample_control
template <class M, class R>
__device__ __forceinline__ int substeps_of(const Params<R>& P, uint64_t h0, int slot, int ext) {
    const uint64_t key = mix64(slot_ext_hash(h0, (uint64_t)slot, (uint64_t)ext) ^ (uint64_t)PH_SAMPLE);
    const double d = __dmul_rn(__dsub_rn(1.0, unit53(draw_u64(key, (uint64_t)M::NU))), P.t_prop);
    const R dt = (R)d;
    const int s = (int)ceil(__ddiv_rn((double)dt, 0.02));
    return s < 4 ? 4 : s;
}

}  // namespace kpx
