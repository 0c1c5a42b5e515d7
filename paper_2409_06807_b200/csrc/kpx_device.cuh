// kpx_device.cuh -- device building blocks of the B200 Kino-PAX planner.
//
//  * counter RNG (SplitMix64 chain, bit-identical to reference rng.py:30-54)
//  * robot models as compile-time traits (vector fields of _kernel.pyx:84-130)
//  * integrate_and_map<M,R> (warp-synchronous): one tree extension per lane = RK4 in
//    registers (float32: packed pairs, Kahan-compensated), per substep finite / state
//    box / obstacle walk against the scene staged in shared memory -- the walk as an
//    exact segment cull through an occupancy grid plus a deferred, warp-cooperative
//    point walk -- and the clamped grid mapping.  Verdicts and counters follow
//    _kernel.pyx:157-296 (SURVEY.md section 9 lists the rules); R=double built with
//    -fmad=false is bit-exact for the double integrator, R=float is the throughput path.
//  * the shared-memory scene (Scene<R>), the node-major row layout of per-node vectors (Row, load_row / store_row)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cmath>
#include <limits>
#include <type_traits>

#include "../../include/kpx.h"

#ifndef KPX_Q12_KAHAN
// Kahan-compensated float32 quadcopter update: OFF.  Measured on 1 M extensions against the float64 kernel
// (tools/f32_err.py, profiles/tuning_r02.md): max relative end-state error 1.2e-6 with, 2.4e-6 without (tolerance 1e-5),
// the same verdicts and cells (<= 1 flip per million either way), the same success over 1000 seeds (599 / 608; float64
// 591) -- and 12 fewer live registers: spill loads 400 -> 208 B, quad12/narrow +9 %, config 5 +11 %.
#define KPX_Q12_KAHAN 0
#endif
#ifndef KPX_DUB_KAHAN
#define KPX_DUB_KAHAN 1              // float32 Dubins airplane: 1 = Kahan-compensated accumulation, 0 = closed-form (v, theta, gamma) + plain position update
#endif
#ifndef KPX_DI_KAHAN
#define KPX_DI_KAHAN 1               // Kahan-compensated float32 double-integrator step (0: plain, ~3 % faster, 10x the error)
#endif
#ifndef KPX_PACKED_F32
#define KPX_PACKED_F32 1             // RK4 vector updates and paired sincos on packed float32 pairs (FFMA2 / FADD2 / FMUL2)
#endif

namespace kpx {

constexpr int kBlock = 256;          // threads per CTA of every kernel here
constexpr int kChunk = 4 * kBlock;   // slots / items per ordered-compaction chunk
constexpr int kOccGrid = 16;         // occupancy-mask grid resolution per axis (16 KB of shared memory per table)
constexpr int kOccCells = kOccGrid * kOccGrid * kOccGrid;
constexpr int kWarps = kBlock / 32;
constexpr int kCoopSteps = 8;        // segments densified into more points than this take the in-lane walk
// inlining policy of the propagation path (tuning knobs)
#ifndef KPX_WALK_ATTR
#define KPX_WALK_ATTR __forceinline__
#endif
#ifndef KPX_COOP_ATTR
#define KPX_COOP_ATTR __forceinline__
#endif
#ifndef KPX_INT_ATTR
#define KPX_INT_ATTR __forceinline__
#endif
#ifndef KPX_SUBSTEP_UNROLL
#define KPX_SUBSTEP_UNROLL 1         // unroll factor of the substep loop (2 trades code size for register moves)
#endif
#ifndef KPX_FLUSH_AT
#define KPX_FLUSH_AT 12              // deferred segment walks per warp that trigger a cooperative pass
#endif
constexpr uint32_t kUnclaimed = 0xFFFFFFFFu;

// per-item result word of an iteration: a VALID item holds its (region, sub) pair in bits 0..29 and the goal test
// of its end state in bit 31; an INVALID item has bit 30 set, with its region below (the region still counts
// towards n_invalid, _kernel.pyx:261-271) -- or all ones if the integration went non-finite (region -1)
constexpr uint32_t kItemInvalid = 0xFFFFFFFFu;
constexpr uint32_t kItemGoalBit = 0x80000000u;
constexpr uint32_t kItemDeadBit = 0x40000000u;

enum : int { PH_SAMPLE = 1, PH_ACCEPT = 2, PH_DEMOTE = 3, PH_PROMOTE = 4 };

// Per-node vectors (states, controls, the end states of an iteration) are stored node-major, one padded ROW per
// node: n reals rounded up to a multiple of 16 bytes (float: 6 -> 8, 12 -> 12; double: 6 -> 6).  Every access of the
// planner is a gather or scatter BY NODE -- an extension reads its parent's state, an append copies an item's end
// state into the tree, the chain walk reads parents -- so a row costs one or two 32-byte sectors (2-3 LDG.128)
// where a structure-of-arrays layout costs one sector per dimension (12 for the quadcopter): round 1's chunked SoA
// moved 1.2 GB of DRAM per quadcopter query, most of it in such gathers.  Consecutive nodes are consecutive rows,
// so the stores of a warp's 32 end states and the appended slots of an iteration are still contiguous.
__host__ __device__ constexpr int row_elems(int n, int elem_size) { return ((n * elem_size + 15) / 16) * (16 / elem_size); }
template <class R, int N> struct Row {
    static constexpr int kStride = row_elems(N, (int)sizeof(R));   // reals per row
    static constexpr int kVecs = kStride * (int)sizeof(R) / 16;     // 16-byte vectors per row
};
template <int N>
__device__ __forceinline__ void load_row(const float* __restrict__ base, long long row, float* out) {
    const float4* p = (const float4*)(base + (size_t)row * Row<float, N>::kStride);
    float tmp[Row<float, N>::kStride];
#pragma unroll
    for (int v = 0; v < Row<float, N>::kVecs; ++v) {
        const float4 q = __ldcg(p + v);
        tmp[4 * v] = q.x; tmp[4 * v + 1] = q.y; tmp[4 * v + 2] = q.z; tmp[4 * v + 3] = q.w;
    }
#pragma unroll
    for (int d = 0; d < N; ++d) out[d] = tmp[d];
}
template <int N>
__device__ __forceinline__ void load_row(const double* __restrict__ base, long long row, double* out) {
    const double2* p = (const double2*)(base + (size_t)row * Row<double, N>::kStride);
    double tmp[Row<double, N>::kStride];
#pragma unroll
    for (int v = 0; v < Row<double, N>::kVecs; ++v) { const double2 q = __ldcg(p + v); tmp[2 * v] = q.x; tmp[2 * v + 1] = q.y; }
#pragma unroll
    for (int d = 0; d < N; ++d) out[d] = tmp[d];
}
template <int N>
__device__ __forceinline__ void store_row(float* __restrict__ base, long long row, const float* in) {
    float4* p = (float4*)(base + (size_t)row * Row<float, N>::kStride);
    float tmp[Row<float, N>::kStride];
#pragma unroll
    for (int d = 0; d < Row<float, N>::kStride; ++d) tmp[d] = d < N ? in[d] : 0.0f;
#pragma unroll
    for (int v = 0; v < Row<float, N>::kVecs; ++v) __stcg(p + v, make_float4(tmp[4 * v], tmp[4 * v + 1], tmp[4 * v + 2], tmp[4 * v + 3]));
}
template <int N>
__device__ __forceinline__ void store_row(double* __restrict__ base, long long row, const double* in) {
    double2* p = (double2*)(base + (size_t)row * Row<double, N>::kStride);
    double tmp[Row<double, N>::kStride];
#pragma unroll
    for (int d = 0; d < Row<double, N>::kStride; ++d) tmp[d] = d < N ? in[d] : 0.0;
#pragma unroll
    for (int v = 0; v < Row<double, N>::kVecs; ++v) __stcg(p + v, make_double2(tmp[2 * v], tmp[2 * v + 1]));
}
// row -> row copy without unpacking
template <class R, int N>
__device__ __forceinline__ void copy_row(R* __restrict__ dst, long long drow, const R* __restrict__ src, long long srow) {
    const uint4* s = (const uint4*)(src + (size_t)srow * Row<R, N>::kStride);
    uint4* d = (uint4*)(dst + (size_t)drow * Row<R, N>::kStride);
    uint4 t[Row<R, N>::kVecs];
#pragma unroll
    for (int v = 0; v < Row<R, N>::kVecs; ++v) t[v] = __ldcg(s + v);
#pragma unroll
    for (int v = 0; v < Row<R, N>::kVecs; ++v) __stcg(d + v, t[v]);
}

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

// ---- Philox4x32-10 (Salmon et al., "Parallel random numbers: as easy as 1, 2, 3", SC'11): the production stream.
// The reference's streams are SplitMix64 chains (above; the parity mode, KPX_RNG_SPLITMIX64).  With KPX_RNG_PHILOX the
// same five-word stream identity (seed, iteration, slot, extension, phase) and draw index feed a counter-based
// generator instead of a hash chain:
//     iteration key  h0 = words 0..1 of philox(counter = (seed_lo, seed_hi, it_lo, it_hi), key = kPhiloxDomain)
//     draw i         = 64 bits (words 2 (i & 1), 2 (i & 1) + 1) of philox(counter = (slot, ext, phase, i >> 1), key = h0)
// and a uniform is the top 53 bits of those 64, as in rng.py:52.  Trees then differ from the reference's by
// construction (other random numbers); everything downstream of a draw is unchanged.
struct Philox4 { uint32_t x, y, z, w; };
__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32);
#endif
}
__host__ __device__ __forceinline__ Philox4 philox4x32_10(Philox4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = Philox4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    return c;
}
constexpr uint32_t kPhiloxDomain0 = 0x4B696E6Fu, kPhiloxDomain1 = 0x50415821u;      // "Kino" "PAX!"
__host__ __device__ __forceinline__ uint64_t philox_iter_key(uint64_t seed, uint64_t it) {
    const Philox4 r = philox4x32_10(Philox4{(uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)it, (uint32_t)(it >> 32)},
                                    kPhiloxDomain0, kPhiloxDomain1);
    return (uint64_t)r.x | ((uint64_t)r.y << 32);
}
// draws 2 blk and 2 blk + 1 of the stream (slot, ext, phase) under iteration key h0
__host__ __device__ __forceinline__ void philox_draw2(uint64_t h0, uint32_t slot, uint32_t ext, int phase, uint32_t blk,
                                                      uint64_t* a, uint64_t* b) {
    const Philox4 r = philox4x32_10(Philox4{slot, ext, (uint32_t)phase, blk}, (uint32_t)h0, (uint32_t)(h0 >> 32));
    *a = (uint64_t)r.x | ((uint64_t)r.y << 32);
    *b = (uint64_t)r.z | ((uint64_t)r.w << 32);
}
// the two generators behind one face: iteration key and "draw 0 of stream (slot, ext, phase)"
__host__ __device__ __forceinline__ uint64_t iter_key(int rng, uint64_t seed, uint64_t it) {
    return rng == KPX_RNG_PHILOX ? philox_iter_key(seed, it) : iter_hash(seed, it);
}
template <int RNG>
__device__ __forceinline__ double keyed_uniform_of(uint64_t h0, uint64_t slot, uint64_t ext, int phase) {
    if constexpr (RNG == KPX_RNG_PHILOX) {
        uint64_t a, b;
        philox_draw2(h0, (uint32_t)slot, (uint32_t)ext, phase, 0u, &a, &b);
        return unit53(a);
    }
    return keyed_uniform(h0, slot, ext, phase);
}

// ------------------------------------------------------- typed parameters ----
template <class R>
struct Params {
    int n, nu, n_obs, subcells, grid_n, lambda_max;
    long long t_e;                        // nodes the arena holds
    long long t_e_start;                  // capacity in effect at the start (0: t_e) and its growth factor when a run
    double t_e_growth;                    // would end exhausted (adaptive t_e); <= 1: fixed capacity
    double t_prop, epsilon, delta, vol;   // RNG / estimates always in f64
    double control_lo[KPX_MAX_CONTROL], control_span[KPX_MAX_CONTROL];  // span = hi - lo (f64, as reference)
    R check_res;
    // the arrays the substep loop reads every iteration are 16-byte aligned: fewer, wider constant loads
    alignas(16) R state_lo[KPX_MAX_DIM];
    alignas(16) R state_hi[KPX_MAX_DIM];
    R grid_lo[KPX_MAX_DIM], grid_width[KPX_MAX_DIM];
    R grid_cmax[KPX_MAX_DIM];             // (R)(cells-1)
    int grid_strides[KPX_MAX_DIM];
    int n_regions, subs_per_region;
    // occupancy-mask grid over the position box (0 = disabled -> every obstacle is tested)
    int occ_g;
    alignas(16) R occ_lo[3];
    alignas(16) R occ_inv[3];
    // d2_thr[k] = largest d2 with sqrt(d2) <= check_res * 2^k: the densification count of a segment
    // (validity.py:26-31) follows from its squared length by compares alone, bit for bit
    alignas(16) R d2_thr[4];
};

// largest x with fl(sqrt(x)) <= thr (sqrt is correctly rounded and monotone on host and device alike)
template <class R>
inline R sqrt_threshold(R thr) {
    R x = thr * thr;
    const R inf = std::numeric_limits<R>::infinity();
    while (std::sqrt(x) > thr) x = std::nextafter(x, (R)0);
    while (std::sqrt(std::nextafter(x, inf)) <= thr) x = std::nextafter(x, inf);
    return x;
}

template <class R>
inline void fill_params(Params<R>& P, const kpx_problem& pr) {
    P.n = pr.n; P.nu = pr.nu; P.n_obs = pr.n_obs; P.subcells = pr.subcells; P.grid_n = pr.grid_n;
    P.lambda_max = pr.lambda_max; P.t_e = pr.t_e; P.t_e_start = pr.t_e_start; P.t_e_growth = pr.t_e_growth;
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
    R thr = P.check_res;
    for (int k = 0; k < 4; ++k) { P.d2_thr[k] = thr > (R)0 ? sqrt_threshold<R>(thr) : (R)0; thr += thr; }
}

// Cell of a coordinate along one axis.  Both operations round monotonically, so p in [omin, omax] implies
// cell(omin) <= cell(p) <= cell(omax): computing an obstacle's cell range with this very function (same
// precision, same constants) yields masks that are exactly conservative without any safety margin.
template <class R>
__host__ __device__ __forceinline__ int occ_cell(R p, R lo, R inv) {
    int c = (int)((p - lo) * inv);
    return c < 0 ? 0 : (c > kOccGrid - 1 ? kOccGrid - 1 : c);
}

// Host: cell -> bitmask of the obstacles whose closed box (as rounded to R) can contain a point of that cell,
// followed by the dilated table: cell c -> OR of the masks of the 2x2x2 block of cells starting at c (what a
// segment whose end points lie in adjacent cells can touch).
template <class R>
inline void build_occupancy_masks(const Params<R>& P, int n_obs, const double* omin, const double* omax,
                                  uint32_t* masks /* 2 * kOccGrid^3 */) {
    const int G = kOccGrid;
    for (int i = 0; i < 2 * G * G * G; ++i) masks[i] = 0u;
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
    uint32_t* dil = masks + G * G * G;
    for (int x = 0; x < G; ++x)
        for (int y = 0; y < G; ++y)
            for (int z = 0; z < G; ++z) {
                uint32_t m = 0u;
                for (int c = 0; c < 8; ++c) {
                    const int xx = x + (c & 1), yy = y + ((c >> 1) & 1), zz = z + (c >> 2);
                    if (xx < G && yy < G && zz < G) m |= masks[(xx * G + yy) * G + zz];
                }
                dil[(x * G + y) * G + z] = m;
            }
}

// ----------------------------------------------------------------- models ----
template <class R> struct MathK;
template <> struct MathK<double> {
    static constexpr double PI = 3.14159265358979323846, TWO_PI = 2.0 * 3.14159265358979323846;
    __device__ static __forceinline__ void sc(double x, double* s, double* c) { *s = sin(x); *c = cos(x); }
    __device__ static __forceinline__ void sc2(double xa, double xb, double* sa, double* ca, double* sb, double* cb) {
        sc(xa, sa, ca); sc(xb, sb, cb);
    }
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
#ifndef KPX_SC_REDUCE
#define KPX_SC_REDUCE 1
#endif
    // whole turns off first (exact no-op inside (-pi, pi); three instructions, no branch): a diverged angle of
    // hundreds of radians is brought back into the range the quadrant reduction is accurate for, and a non-finite one
    // stays non-finite
    __device__ static __forceinline__ float reduce_turns(float x) {
        return __fmaf_rn(rintf(x * 0.15915494309189535f), -6.283185307179586f, x);
    }
    __device__ static __forceinline__ void sc(float x, float* s, float* c) {
        // Angles are wrapped to (-pi, pi] after every substep, so only states that have already diverged (body
        // rates of hundreds of rad/s inside an RK4 stage) come here; they get the hardware approximation instead
        // of 12 inlined copies of sincosf's Payne-Hanek path in the substep loop (17 % no-instruction stalls).
#if KPX_SC_REDUCE
        x = reduce_turns(x);
#else
        if (!(fabsf(x) < 512.0f)) { __sincosf(x, s, c); return; }
#endif
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
    // the same for two angles at once on packed float32 pairs (sm_100 FFMA2 / FMUL2 / FADD2): the reduction and
    // both polynomials cost one instruction per pair; only the quadrant fix-up stays per component
    __device__ static __forceinline__ void sc2(float xa, float xb, float* sa, float* ca, float* sb, float* cb) {
#if KPX_PACKED_F32
        // a diverged angle means a diverged state: both components take the hardware approximation (see sc)
#if KPX_SC_REDUCE
        xa = reduce_turns(xa); xb = reduce_turns(xb);
#else
        if (!(fabsf(xa) < 512.0f) || !(fabsf(xb) < 512.0f)) { __sincosf(xa, sa, ca); __sincosf(xb, sb, cb); return; }
#endif
        sc2_bounded(xa, xb, sa, ca, sb, cb);
#else
        sc(xa, sa, ca); sc(xb, sb, cb);
#endif
    }
    // the same without the large-argument path, for angles that cannot grow (the Dubins airplane's heading is wrapped
    // after every substep and its climb angle moves by |u| dt at most): the compiler predicates that path instead of
    // branching around it, 16 of ~45 instructions per call.  A non-finite argument still gives NaN.
    __device__ static __forceinline__ void sc2_bounded(float xa, float xb, float* sa, float* ca, float* sb, float* cb) {
#if KPX_PACKED_F32
        const float2 x = make_float2(xa, xb);
        const float2 t = __ffma2_rn(x, make_float2(0.636619772f, 0.636619772f), make_float2(12582912.0f, 12582912.0f));
        const float2 qf = __fadd2_rn(t, make_float2(-12582912.0f, -12582912.0f));
        float2 r = __ffma2_rn(qf, make_float2(-1.57079637f, -1.57079637f), x);
        r = __ffma2_rn(qf, make_float2(4.37113883e-8f, 4.37113883e-8f), r);
        const float2 z = __fmul2_rn(r, r);
        float2 sp = __ffma2_rn(z, make_float2(-1.9515295891e-4f, -1.9515295891e-4f), make_float2(8.3321608736e-3f, 8.3321608736e-3f));
        sp = __ffma2_rn(z, sp, make_float2(-1.6666654611e-1f, -1.6666654611e-1f));
        const float2 sv = __ffma2_rn(__fmul2_rn(z, r), sp, r);
        float2 cp = __ffma2_rn(z, make_float2(2.443315711809948e-5f, 2.443315711809948e-5f),
                               make_float2(-1.388731625493765e-3f, -1.388731625493765e-3f));
        cp = __ffma2_rn(z, cp, make_float2(4.166664568298827e-2f, 4.166664568298827e-2f));
        const float2 cv = __ffma2_rn(__fmul2_rn(z, z), cp, __ffma2_rn(z, make_float2(-0.5f, -0.5f), make_float2(1.0f, 1.0f)));
        quadrant(__float_as_int(t.x), sv.x, cv.x, sa, ca);
        quadrant(__float_as_int(t.y), sv.y, cv.y, sb, cb);
#else
        sc(xa, sa, ca); sc(xb, sb, cb);
#endif
    }
    __device__ static __forceinline__ void quadrant(int q, float sv, float cv, float* s, float* c) {
        const bool swap = q & 1;
        float so = swap ? cv : sv, co = swap ? sv : cv;
        if (q & 2) so = -so;
        if ((q + 1) & 2) co = -co;
        *s = so; *c = co;
    }
    // only reached by angles that left [0, 2 pi) by more than a wrap, i.e. diverged states: one floor instead
    // of fmodf's exact (looping) reduction in the substep loop
    __device__ static __forceinline__ float mod(float a, float b) { return a - b * floorf(a * (1.0f / b)); }
    __device__ static __forceinline__ float sq(float x) { return sqrtf(x); }
    __device__ static __forceinline__ float fl(float x) { return floorf(x); }
};

// wrap to (-pi, pi]  (_kernel.pyx:77-81).  fmod only changes t outside [0, 2pi);
// the in-range fast path returns the identical value.
template <class R>
__device__ __forceinline__ R wrap_angle(R a) {
    // float32: an angle already inside (-pi, pi) is returned as it is -- (a + pi) - pi would round it to a multiple
    // of ulp(2 pi) = 4.8e-7 after every substep, an error the float64 formula does not have
    if constexpr (std::is_same<R, float>::value) {
        // ... and whole turns come off in three instructions (fmod's exact reduction buys nothing at float32; the result
        // lies in [-pi, pi], the closed end only for an argument that is an exact odd multiple of pi)
        return fabsf(a) < MathK<float>::PI ? a : MathK<float>::reduce_turns(a);
    }
    R t = a + MathK<R>::PI;
    if (!(t >= (R)0 && t < MathK<R>::TWO_PI)) t = MathK<R>::mod(t, MathK<R>::TWO_PI);
    if (t <= (R)0) t += MathK<R>::TWO_PI;
    return t - MathK<R>::PI;
}

struct ModelDI6 {
    using Base = ModelDI6;
    static constexpr int kRng = KPX_RNG_SPLITMIX64;
    static constexpr int ID = KPX_MODEL_DI6, N = 6, NU = 3;
    template <class R> __device__ static __forceinline__ void deriv(const R* x, const R* u, R* o) {
        o[0] = x[3]; o[1] = x[4]; o[2] = x[5]; o[3] = u[0]; o[4] = u[1]; o[5] = u[2];
    }
    template <class R> __device__ static __forceinline__ void wrap(R*) {}
};

struct ModelDubins6 {
    using Base = ModelDubins6;
    static constexpr int kRng = KPX_RNG_SPLITMIX64;
    static constexpr int ID = KPX_MODEL_DUBINS6, N = 6, NU = 3;
    template <class R> __device__ static __forceinline__ void deriv(const R* x, const R* u, R* o) {
        R st, ct, sg, cg;
        MathK<R>::sc2(x[4], x[5], &st, &ct, &sg, &cg);
        R v = x[3];
        o[0] = v * ct * cg; o[1] = v * st * cg; o[2] = v * sg;
        o[3] = u[0]; o[4] = u[1]; o[5] = u[2];
    }
    template <class R> __device__ static __forceinline__ void wrap(R* x) { x[4] = wrap_angle(x[4]); }
};

struct ModelQuad12 {
    using Base = ModelQuad12;
    static constexpr int kRng = KPX_RNG_SPLITMIX64;
    static constexpr int ID = KPX_MODEL_QUAD12, N = 12, NU = 4;
    template <class R> __device__ static __forceinline__ void deriv(const R* x, const R* u, R* o) {
        R sphi, cphi, sth, cth, spsi, cpsi;
        MathK<R>::sc2(x[6], x[7], &sphi, &cphi, &sth, &cth);
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
            R icth = __fdividef(1.0f, cth);       // MUFU.RCP (2 ulp) instead of the IEEE division sequence, 4x per substep
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
    // float32: the same field from given sines / cosines of (phi, theta, psi): sc = {s_phi, c_phi, s_th, c_th, s_psi, c_psi}
    __device__ static __forceinline__ void deriv_sc(const float* x, const float* u, const float* sc, float* o) {
        const float sphi = sc[0], cphi = sc[1], sth = sc[2], cth = sc[3], spsi = sc[4], cpsi = sc[5];
        const float p = x[9], q = x[10], r = x[11], acc = u[0];
        o[0] = x[3]; o[1] = x[4]; o[2] = x[5];
        o[3] = acc * (cphi * sth * cpsi + sphi * spsi);
        o[4] = acc * (cphi * sth * spsi - sphi * cpsi);
        o[5] = acc * (cphi * cth) - 9.81f;
        const float sw = q * sphi + r * cphi;
        const float icth = __fdividef(1.0f, cth);
        o[6] = p + sw * (sth * icth);
        o[7] = q * cphi - r * sphi;
        o[8] = sw * icth;
        o[9] = __fmaf_rn(-q, r, u[1] * 100.0f);          // (u1 - (Jz - Jy) q r) / Jx with J = diag(.01, .01, .02)
        o[10] = __fmaf_rn(p, r, u[2] * 100.0f);
        o[11] = u[3] * 50.0f;
    }
};

// B stacked 3-D double integrators, state [p1 v1 p2 v2 ...]; only block 1 is workspace position.
template <int B>
struct ModelStackedDI {
    using Base = ModelStackedDI<B>;
    static constexpr int kRng = KPX_RNG_SPLITMIX64;
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

// The same model drawing from another generator: the random stream is a compile-time property of the kernel (a
// run-time switch in the sampling code cost 5-8 % of the throughput of BOTH streams); `Base` keeps the per-model
// specialisations (Stepper, FreeFlight) keyed on the plain model.
template <class M0, int RNG>
struct WithRng : M0 {
    using Base = typename M0::Base;
    static constexpr int kRng = RNG;
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
    for (int i = 0; i < M::N; ++i) cur[i] = cur[i] + h6 * (acc[i] + k[i]);
    M::template wrap<R>(cur);
}

#if KPX_PACKED_F32
// float32 on sm_100: the vector updates of RK4 run on packed pairs (FFMA2 / FADD2: two float32 operations per
// lane per instruction) -- the kernel is issue-bound, so halving the instruction count of the axpy's is what
// counts.  Same operations and roundings per component as the scalar form; the state update is
// Kahan-compensated (`comp` carries the running rounding error across substeps), which keeps ~50 chained
// substeps within a few float32 ulps of the float64 trajectory.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
template <class M>
__device__ __forceinline__ void rk4_step_f32(float* cur, float* comp, const float* u, float h, float half_h, float h6) {
    constexpr int N = M::N, H = N / 2;
    static_assert(N % 2 == 0, "packed float32 RK4 needs an even state dimension");
    float k[N], tmp[N];
    float2 acc[H];
    const float2 hh2 = f2(half_h, half_h), h2 = f2(h, h), two = f2(2.0f, 2.0f), h62 = f2(h6, h6);
    M::template deriv<float>(cur, u, k);
#pragma unroll
    for (int j = 0; j < H; ++j) {
        const float2 kj = f2(k[2 * j], k[2 * j + 1]);
        acc[j] = kj;
        const float2 t = __ffma2_rn(hh2, kj, f2(cur[2 * j], cur[2 * j + 1]));
        tmp[2 * j] = t.x; tmp[2 * j + 1] = t.y;
    }
    M::template deriv<float>(tmp, u, k);
#pragma unroll
    for (int j = 0; j < H; ++j) {
        const float2 kj = f2(k[2 * j], k[2 * j + 1]);
        acc[j] = __ffma2_rn(two, kj, acc[j]);
        const float2 t = __ffma2_rn(hh2, kj, f2(cur[2 * j], cur[2 * j + 1]));
        tmp[2 * j] = t.x; tmp[2 * j + 1] = t.y;
    }
    M::template deriv<float>(tmp, u, k);
#pragma unroll
    for (int j = 0; j < H; ++j) {
        const float2 kj = f2(k[2 * j], k[2 * j + 1]);
        acc[j] = __ffma2_rn(two, kj, acc[j]);
        const float2 t = __ffma2_rn(h2, kj, f2(cur[2 * j], cur[2 * j + 1]));
        tmp[2 * j] = t.x; tmp[2 * j + 1] = t.y;
    }
    M::template deriv<float>(tmp, u, k);
#pragma unroll
    for (int j = 0; j < H; ++j) {
        const float2 c = f2(cur[2 * j], cur[2 * j + 1]), e = f2(comp[2 * j], comp[2 * j + 1]);
        const float2 s4 = __fadd2_rn(acc[j], f2(k[2 * j], k[2 * j + 1]));
        const float2 y = __ffma2_rn(h62, s4, f2(-e.x, -e.y));
        const float2 t = __fadd2_rn(c, y);
        const float2 d = __fadd2_rn(__fadd2_rn(t, f2(-c.x, -c.y)), f2(-y.x, -y.y));
        comp[2 * j] = d.x; comp[2 * j + 1] = d.y;
        cur[2 * j] = t.x; cur[2 * j + 1] = t.y;
    }
    M::template wrap<float>(cur);
}
#else
template <class M>
__device__ __forceinline__ void rk4_step_f32(float* cur, float* comp, const float* u, float h, float half_h, float h6) {
    float k[M::N], acc[M::N], tmp[M::N];
    M::template deriv<float>(cur, u, k);
#pragma unroll
    for (int i = 0; i < M::N; ++i) { acc[i] = k[i]; tmp[i] = cur[i] + half_h * k[i]; }
    M::template deriv<float>(tmp, u, k);
#pragma unroll
    for (int i = 0; i < M::N; ++i) { acc[i] = acc[i] + 2.0f * k[i]; tmp[i] = cur[i] + half_h * k[i]; }
    M::template deriv<float>(tmp, u, k);
#pragma unroll
    for (int i = 0; i < M::N; ++i) { acc[i] = acc[i] + 2.0f * k[i]; tmp[i] = cur[i] + h * k[i]; }
    M::template deriv<float>(tmp, u, k);
#pragma unroll
    for (int i = 0; i < M::N; ++i) {
        // Kahan-compensated update: `comp` carries the running rounding error across substeps
        const float y = __fmaf_rn(h6, acc[i] + k[i], -comp[i]);
        const float t = __fadd_rn(cur[i], y);
        comp[i] = __fsub_rn(__fsub_rn(t, cur[i]), y);
        cur[i] = t;
    }
    M::template wrap<float>(cur);
}
#endif

// float32 double integrator: x' = (v, u) has a nilpotent system matrix, so the four RK4 stages collapse
// algebraically to  p += h (v + h/2 u),  v += h u  -- the same polynomial RK4 evaluates, in 9 instead of ~45
// operations per block and with no stage vectors live.  (float64 keeps the staged form: it is pinned bit for
// bit to the reference's rounding order.)
__device__ __forceinline__ void di_step_f32(float* cur, float* comp, const float* u, float h, float half_h) {
#if !KPX_DI_KAHAN
    // measured alternative without the compensation (profiles/tuning_r01.md): 6 packed + 3 scalar operations
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        cur[i] = __fmaf_rn(h, __fmaf_rn(half_h, u[i], cur[3 + i]), cur[i]);
        cur[3 + i] = __fmaf_rn(h, u[i], cur[3 + i]);
    }
    (void)comp;
#elif KPX_PACKED_F32
    // axes x and y as a packed pair (FFMA2 / FADD2), z on its own: 18 instead of 27 instructions
    {
        const float2 u2 = make_float2(u[0], u[1]), v2 = make_float2(cur[3], cur[4]), p2 = make_float2(cur[0], cur[1]);
        const float2 hh = make_float2(half_h, half_h), hv = make_float2(h, h), m1 = make_float2(-1.0f, -1.0f);
        const float2 cp = make_float2(comp[0], comp[1]), cv = make_float2(comp[3], comp[4]);
        const float2 yp = __ffma2_rn(hv, __ffma2_rn(hh, u2, v2), make_float2(-cp.x, -cp.y));
        const float2 tp = __fadd2_rn(p2, yp);
        const float2 dp = __ffma2_rn(yp, m1, __ffma2_rn(p2, m1, tp));        // (tp - p) - yp
        const float2 yv = __ffma2_rn(hv, u2, make_float2(-cv.x, -cv.y));
        const float2 tv = __fadd2_rn(v2, yv);
        const float2 dv = __ffma2_rn(yv, m1, __ffma2_rn(v2, m1, tv));
        comp[0] = dp.x; comp[1] = dp.y; cur[0] = tp.x; cur[1] = tp.y;
        comp[3] = dv.x; comp[4] = dv.y; cur[3] = tv.x; cur[4] = tv.y;
    }
    {
        const float yp = __fmaf_rn(h, __fmaf_rn(half_h, u[2], cur[5]), -comp[2]);
        const float tp = __fadd_rn(cur[2], yp);
        comp[2] = __fsub_rn(__fsub_rn(tp, cur[2]), yp);
        cur[2] = tp;
        const float yv = __fmaf_rn(h, u[2], -comp[5]);
        const float tv = __fadd_rn(cur[5], yv);
        comp[5] = __fsub_rn(__fsub_rn(tv, cur[5]), yv);
        cur[5] = tv;
    }
#else
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float yp = __fmaf_rn(h, __fmaf_rn(half_h, u[i], cur[3 + i]), -comp[i]);
        const float tp = __fadd_rn(cur[i], yp);
        comp[i] = __fsub_rn(__fsub_rn(tp, cur[i]), yp);
        cur[i] = tp;
        const float yv = __fmaf_rn(h, u[i], -comp[3 + i]);
        const float tv = __fadd_rn(cur[3 + i], yv);
        comp[3 + i] = __fsub_rn(__fsub_rn(tv, cur[3 + i]), yv);
        cur[3 + i] = tv;
    }
#endif
}

// float32 derives its step constants from h inside the step (h/2 is exact, h/6 is taken as h * (1/6), one
// rounding away from the quotient) so that only h stays live in the loop; float64 is handed the reference's
// own h/6 (_kernel.pyx:196-201).
template <class M, class R>
struct Stepper {
    // values carried across the substeps of an extension: the Kahan compensation of every dimension (float32)
    static constexpr int kCarry = std::is_same<R, float>::value ? M::N : 1;
    __device__ static __forceinline__ void init(const R*, const R*, R* carry) {
#pragma unroll
        for (int i = 0; i < kCarry; ++i) carry[i] = (R)0;
    }
    __device__ static __forceinline__ void step(R* cur, R* comp, const R* u, R h, R h6) {
        if constexpr (std::is_same<R, float>::value) rk4_step_f32<M>(cur, comp, u, h, 0.5f * h, h * 0.16666667f);
        else rk4_step<M, R>(cur, comp, u, h, (R)0.5 * h, h6);
    }
};
template <>
struct Stepper<ModelDI6, float> {
    static constexpr int kCarry = 6;
    __device__ static __forceinline__ void init(const float*, const float*, float* carry) {
#pragma unroll
        for (int i = 0; i < kCarry; ++i) carry[i] = 0.0f;
    }
    __device__ static __forceinline__ void step(float* cur, float* comp, const float* u, float h, float) {
        di_step_f32(cur, comp, u, h, 0.5f * h);
    }
};
// float32 quadcopter.  The four RK4 stages need sin / cos of the three Euler angles at four nearby arguments: the
// stage angles differ from the substep's starting angles by delta = c h k (a few hundredths of a radian), so stages
// 2-4 ROTATE the stage-1 values -- sin(a + d) = s cos d + c sin d with short polynomials for sin d, cos d (|d| <= 1/4:
// error < 2e-8) -- instead of three more full reductions + polynomials + quadrant fix-ups per stage: 12 full sincos per
// substep become 3 plus 9 rotations (~11 packed / scalar operations per angle).  A larger step of an angle (only next
// to the pitch singularity) takes the full evaluation.  Same RK4; the update is plain (KPX_Q12_KAHAN, measured) -- the generic path and the other models compensate it.
#if KPX_PACKED_F32
template <>
struct Stepper<ModelQuad12, float> {
    static constexpr int kCarry = 12;
    __device__ static __forceinline__ void init(const float*, const float*, float* carry) {
#pragma unroll
        for (int i = 0; i < kCarry; ++i) carry[i] = 0.0f;
    }
    __device__ static __forceinline__ void full_sc(const float* x, float* sc) {
        MathK<float>::sc2(x[6], x[7], &sc[0], &sc[1], &sc[2], &sc[3]);
        MathK<float>::sc(x[8], &sc[4], &sc[5]);
    }
    // the rare large-step case, out of line: three inlined copies of the full evaluation in the substep loop cost more
    // in instruction-cache misses (stall_no_instruction 1.0 -> 1.7 per issue) than the rotation saves
    struct SC6 { float v[6]; };
#ifndef KPX_ROT_COLD
#define KPX_ROT_COLD 0
#endif
    __device__ static __noinline__ SC6 full_sc_cold(float a, float b, float c) {
        SC6 r;
        MathK<float>::sc2(a, b, &r.v[0], &r.v[1], &r.v[2], &r.v[3]);
        MathK<float>::sc(c, &r.v[4], &r.v[5]);
        return r;
    }
    // sc_out = sin / cos of (base angles + d), from sc_base = sin / cos of the base angles
    __device__ static __forceinline__ void rotate_sc(const float* sc_base, float d0, float d1, float d2, const float* x_stage, float* sc_out) {
#ifndef KPX_ROT_LIMIT
#define KPX_ROT_LIMIT 0.25f
#endif
        if (__builtin_expect(!(fabsf(d0) <= KPX_ROT_LIMIT && fabsf(d1) <= KPX_ROT_LIMIT && fabsf(d2) <= KPX_ROT_LIMIT), 0)) {
#if KPX_ROT_COLD
            const SC6 r = full_sc_cold(x_stage[6], x_stage[7], x_stage[8]);
#pragma unroll
            for (int i = 0; i < 6; ++i) sc_out[i] = r.v[i];
#else
            full_sc(x_stage, sc_out);
#endif
            return;
        }
        const float2 d = make_float2(d0, d1);
        const float2 z = __fmul2_rn(d, d);
        // sin d = d + d z (-1/6 + z/120), cos d = 1 + z (-1/2 + z (1/24 - z/720))
        const float2 sd = __ffma2_rn(__fmul2_rn(d, z), __ffma2_rn(z, f2(8.3333333e-3f, 8.3333333e-3f), f2(-0.16666667f, -0.16666667f)), d);
        const float2 cd = __ffma2_rn(z, __ffma2_rn(z, __ffma2_rn(z, f2(-1.3888889e-3f, -1.3888889e-3f), f2(4.1666667e-2f, 4.1666667e-2f)), f2(-0.5f, -0.5f)), f2(1.0f, 1.0f));
        const float2 sb = make_float2(sc_base[0], sc_base[2]), cb = make_float2(sc_base[1], sc_base[3]);
        const float2 so = __ffma2_rn(cb, sd, __fmul2_rn(sb, cd));
        const float2 co = __ffma2_rn(f2(-sb.x, -sb.y), sd, __fmul2_rn(cb, cd));
        sc_out[0] = so.x; sc_out[1] = co.x; sc_out[2] = so.y; sc_out[3] = co.y;
        const float z2 = d2 * d2;
        const float sd2 = __fmaf_rn(d2 * z2, __fmaf_rn(z2, 8.3333333e-3f, -0.16666667f), d2);
        const float cd2 = __fmaf_rn(z2, __fmaf_rn(z2, __fmaf_rn(z2, -1.3888889e-3f, 4.1666667e-2f), -0.5f), 1.0f);
        sc_out[4] = __fmaf_rn(sc_base[5], sd2, sc_base[4] * cd2);
        sc_out[5] = __fmaf_rn(-sc_base[4], sd2, sc_base[5] * cd2);
    }
    __device__ static __forceinline__ void step(float* cur, float* comp, const float* u, float h, float) {
        constexpr int N = 12, H = 6;
        const float half_h = 0.5f * h, h6 = h * 0.16666667f;
        float k[N], tmp[N], sc[6];
        float sc1[6];
        float2 acc[H];
        const float2 hh2 = f2(half_h, half_h), h2 = f2(h, h), two = f2(2.0f, 2.0f), h62 = f2(h6, h6);
        full_sc(cur, sc1);
        ModelQuad12::deriv_sc(cur, u, sc1, k);
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const float2 kj = f2(k[2 * j], k[2 * j + 1]);
            acc[j] = kj;
            const float2 t = __ffma2_rn(hh2, kj, f2(cur[2 * j], cur[2 * j + 1]));
            tmp[2 * j] = t.x; tmp[2 * j + 1] = t.y;
        }
        rotate_sc(sc1, half_h * k[6], half_h * k[7], half_h * k[8], tmp, sc);
        ModelQuad12::deriv_sc(tmp, u, sc, k);
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const float2 kj = f2(k[2 * j], k[2 * j + 1]);
            acc[j] = __ffma2_rn(two, kj, acc[j]);
            const float2 t = __ffma2_rn(hh2, kj, f2(cur[2 * j], cur[2 * j + 1]));
            tmp[2 * j] = t.x; tmp[2 * j + 1] = t.y;
        }
        rotate_sc(sc1, half_h * k[6], half_h * k[7], half_h * k[8], tmp, sc);
        ModelQuad12::deriv_sc(tmp, u, sc, k);
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const float2 kj = f2(k[2 * j], k[2 * j + 1]);
            acc[j] = __ffma2_rn(two, kj, acc[j]);
            const float2 t = __ffma2_rn(h2, kj, f2(cur[2 * j], cur[2 * j + 1]));
            tmp[2 * j] = t.x; tmp[2 * j + 1] = t.y;
        }
        rotate_sc(sc1, h * k[6], h * k[7], h * k[8], tmp, sc);
        ModelQuad12::deriv_sc(tmp, u, sc, k);
#pragma unroll
        for (int j = 0; j < H; ++j) {
            const float2 c = f2(cur[2 * j], cur[2 * j + 1]);
            const float2 s4 = __fadd2_rn(acc[j], f2(k[2 * j], k[2 * j + 1]));
            float2 t;
            if (KPX_Q12_KAHAN) {
                const float2 e = f2(comp[2 * j], comp[2 * j + 1]);
                const float2 y = __ffma2_rn(h62, s4, f2(-e.x, -e.y));
                t = __fadd2_rn(c, y);
                const float2 dd = __fadd2_rn(__fadd2_rn(t, f2(-c.x, -c.y)), f2(-y.x, -y.y));
                comp[2 * j] = dd.x; comp[2 * j + 1] = dd.y;
            } else {
                t = __ffma2_rn(h62, s4, c);              // plain update
            }
            cur[2 * j] = t.x; cur[2 * j + 1] = t.y;
        }
        ModelQuad12::wrap<float>(cur);
    }
};
#endif
// float32 Dubins airplane.  Speed, heading and climb angle have constant derivatives (v' = u0, theta' = u1,
// gamma' = u2), so the position does not feed back into the vector field and RK4 degenerates: stages 2 and 3 see
// the SAME (v, theta, gamma) -- one evaluation, weight 4 -- and stage 4 sees the state the substep ends in, i.e.
// the next substep's stage 1.  Per substep that is TWO evaluations of the field (two paired sincos) instead of four;
// the velocity field at the current state is carried to the next substep (carry[6..8]).  The update
// p += h/6 (k1 + 4 k2 + k4), (v, theta, gamma) += h u is RK4's, Kahan-compensated like the generic path.
// (float64 keeps the staged form: it is pinned bit for bit to the reference's rounding order.)
template <>
struct Stepper<ModelDubins6, float> {
    static constexpr int kCarry = 9;
    __device__ static __forceinline__ void field(float v, float th, float ga, float* f) {
        float st, ct, sg, cg;
        MathK<float>::sc2_bounded(th, ga, &st, &ct, &sg, &cg);
        f[0] = v * ct * cg; f[1] = v * st * cg; f[2] = v * sg;
    }
    __device__ static __forceinline__ void init(const float* x0, const float*, float* carry) {
#pragma unroll
        for (int i = 0; i < 6; ++i) carry[i] = 0.0f;
#if !KPX_DUB_KAHAN
        carry[3] = x0[3]; carry[4] = x0[4]; carry[5] = x0[5];      // (v, theta, gamma) the extension starts from
#endif
        field(x0[3], x0[4], x0[5], carry + 6);
    }
#if !KPX_DUB_KAHAN
    // Measured alternative (profiles/tuning_r02.md).  (v, theta, gamma) have constant derivatives, so RK4's update of
    // them is exact and the state after n substeps is x0 + (n h) u: ONE rounding instead of n accumulated ones (and
    // instead of the compensation); the position update is plain.  carry[0] = n (exact in float32).
    __device__ static __forceinline__ void step(float* cur, float* carry, const float* u, float h, float) {
        const float hh = 0.5f * h, h6 = h * 0.16666667f;
        float k2[3], k4[3];
        field(__fmaf_rn(hh, u[0], cur[3]), __fmaf_rn(hh, u[1], cur[4]), __fmaf_rn(hh, u[2], cur[5]), k2);
        carry[0] += 1.0f;
        const float tn = carry[0] * h;
        cur[3] = __fmaf_rn(tn, u[0], carry[3]);
        cur[4] = wrap_angle(__fmaf_rn(tn, u[1], carry[4]));
        cur[5] = __fmaf_rn(tn, u[2], carry[5]);
        field(cur[3], cur[4], cur[5], k4);               // stage 4 = the state this substep ends in
#pragma unroll
        for (int i = 0; i < 3; ++i) {                    // position: Simpson weights
            cur[i] = __fmaf_rn(h6, __fadd_rn(__fmaf_rn(4.0f, k2[i], carry[6 + i]), k4[i]), cur[i]);
            carry[6 + i] = k4[i];                        // next substep's stage 1
        }
    }
#else
    __device__ static __forceinline__ void step(float* cur, float* carry, const float* u, float h, float) {
        const float hh = 0.5f * h, h6 = h * 0.16666667f;
        float k2[3], k4[3];
        field(__fmaf_rn(hh, u[0], cur[3]), __fmaf_rn(hh, u[1], cur[4]), __fmaf_rn(hh, u[2], cur[5]), k2);
#pragma unroll
        for (int i = 3; i < 6; ++i) {                    // v, theta, gamma: += h u, compensated
            const float y = __fmaf_rn(h, u[i - 3], -carry[i]);
            const float t = __fadd_rn(cur[i], y);
            carry[i] = __fsub_rn(__fsub_rn(t, cur[i]), y);
            cur[i] = t;
        }
        field(cur[3], cur[4], cur[5], k4);               // stage 4 = the state this substep ends in
#pragma unroll
        for (int i = 0; i < 3; ++i) {                    // position: Simpson weights, compensated
            const float y = __fmaf_rn(h6, __fadd_rn(__fmaf_rn(4.0f, k2[i], carry[6 + i]), k4[i]), -carry[i]);
            const float t = __fadd_rn(cur[i], y);
            carry[i] = __fsub_rn(__fsub_rn(t, cur[i]), y);
            cur[i] = t;
            carry[6 + i] = k4[i];                        // next substep's stage 1
        }
        // sin / cos are periodic: the carried field is unchanged
        cur[4] = wrap_angle(cur[4]);
    }
#endif
};
// Stacked double integrators: the blocks do not couple, so stepping them one 6-D block at a time performs
// exactly the same operations per dimension while keeping only a 6-D set of RK4 temporaries live
// (N = 48 would otherwise need ~200 registers).
template <int B, class R>
struct Stepper<ModelStackedDI<B>, R> {
    static constexpr int kCarry = std::is_same<R, float>::value ? 6 * B : 1;
    __device__ static __forceinline__ void init(const R*, const R*, R* carry) {
#pragma unroll
        for (int i = 0; i < kCarry; ++i) carry[i] = (R)0;
    }
    __device__ static __forceinline__ void step(R* cur, R* comp, const R* u, R h, R h6) {
#pragma unroll
        for (int b = 0; b < B; ++b) Stepper<ModelDI6, R>::step(cur + 6 * b, comp + 6 * b, u + 3 * b, h, h6);
    }
};

// ------------------------------------------------------- collision scene ----
// The scene lives at the START of the dynamic shared memory, at compile-time offsets, so that no kernel keeps
// a pointer register for it:
//     [occ: kOccCells u32][occ2: kOccCells u32][coop: kWarps x WarpCoop<R>][boxes: n_obs x 8 R][caller's area]
extern __shared__ __align__(16) unsigned char kpx_dyn_smem[];

// Per-warp staging of deferred segment walks (see integrate_and_map).
template <class R>
struct WarpCoop {
    R seg[10][32];                       // prev xyz | d xyz | cur xyz | 1/steps, [field][lane]
    int steps[32];
    int hit[32];                         // lowest point index of the segment that hits an obstacle
    int mark_pts[32];                    // the lane's point counter before the staged segment
    int mark_sub[32];                    // substep index of the staged segment
    uint16_t list[32 * kCoopSteps];      // (lane | point << 5) of every point to test
};

template <class R>
struct Scene {
    static constexpr size_t kOcc = 0, kOcc2 = sizeof(uint32_t) * kOccCells, kCoop = 2 * sizeof(uint32_t) * kOccCells;
    static constexpr size_t kBoxes = kCoop + (size_t)kWarps * sizeof(WarpCoop<R>);
    __device__ static __forceinline__ uint32_t* occ() { return (uint32_t*)(kpx_dyn_smem + kOcc); }
    __device__ static __forceinline__ uint32_t* occ2() { return (uint32_t*)(kpx_dyn_smem + kOcc2); }
    __device__ static __forceinline__ WarpCoop<R>& coop() { return ((WarpCoop<R>*)(kpx_dyn_smem + kCoop))[threadIdx.x >> 5]; }
    // obstacle k: 8 values {min x, min y, min z, -, max x, max y, max z, -}
    __device__ static __forceinline__ R* boxes() { return (R*)(kpx_dyn_smem + kBoxes); }
    __host__ __device__ static size_t bytes(int n_obs) {
        return kBoxes + (((size_t)(n_obs > 0 ? n_obs : 1) * 8 * sizeof(R) + 15) & ~(size_t)15);
    }
    // fill from global memory (boxes in the same 8-value layout); ends with __syncthreads()
    __device__ static __forceinline__ void stage(const Params<R>& P, const R* __restrict__ boxes_g,
                                                 const uint32_t* __restrict__ occ_g) {
        R* bx = boxes();
        for (int i = threadIdx.x; i < 8 * P.n_obs; i += kBlock) bx[i] = boxes_g[i];
        if (P.occ_g) { uint32_t* o = occ(); for (int i = threadIdx.x; i < 2 * kOccCells; i += kBlock) o[i] = occ_g[i]; }
        __syncthreads();
    }
};
// bytes of dynamic shared memory the scene needs for element size rs (4 or 8)
inline size_t scene_smem_bytes(int n_obs, size_t rs) {
    return rs == 8 ? Scene<double>::bytes(n_obs) : Scene<float>::bytes(n_obs);
}

template <class R> struct Box { R lx, ly, lz, hx, hy, hz; };
__device__ __forceinline__ Box<float> load_box(const float* b, int k) {
    const float4 lo = ((const float4*)b)[2 * k], hi = ((const float4*)b)[2 * k + 1];
    return Box<float>{lo.x, lo.y, lo.z, hi.x, hi.y, hi.z};
}
__device__ __forceinline__ Box<double> load_box(const double* b, int k) {
    const double2 a = ((const double2*)b)[4 * k], c = ((const double2*)b)[4 * k + 1], d = ((const double2*)b)[4 * k + 2],
                  e = ((const double2*)b)[4 * k + 3];
    return Box<double>{a.x, a.y, c.x, d.x, d.y, e.x};
}

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { int t = __shfl_up_sync(0xffffffffu, v, o); if (lane >= o) v += t; }
    return v;
}

// closed-box point test (_kernel.pyx:142-154): against every obstacle, or -- through the occupancy grid --
// only against the obstacles flagged for the point's cell.  Same verdict either way.
template <class R>
__device__ __forceinline__ bool point_hits(const Params<R>& P, R px, R py, R pz) {
    const R* bx = Scene<R>::boxes();
    bool h = false;
    if (P.occ_g == 0) {
#pragma unroll 1
        for (int k = 0; k < P.n_obs; ++k) {
            const Box<R> b = load_box(bx, k);
            h = h || (px >= b.lx && px <= b.hx && py >= b.ly && py <= b.hy && pz >= b.lz && pz <= b.hz);
        }
        return h;
    }
    const int ix = occ_cell<R>(px, P.occ_lo[0], P.occ_inv[0]);
    const int iy = occ_cell<R>(py, P.occ_lo[1], P.occ_inv[1]);
    const int iz = occ_cell<R>(pz, P.occ_lo[2], P.occ_inv[2]);
    uint32_t m = Scene<R>::occ()[(ix * kOccGrid + iy) * kOccGrid + iz];
#pragma unroll 1
    while (m) {
        const Box<R> b = load_box(bx, __ffs(m) - 1);
        m &= m - 1;
        h = h || (px >= b.lx && px <= b.hx && py >= b.ly && py <= b.hy && pz >= b.lz && pz <= b.hz);
    }
    return h;
}

// In-lane walk of one segment exactly as the reference orders it (_kernel.pyx:238-253): interior points
// prev + (j/steps) d for j = 1..steps-1, then the end point itself.  Returns the number of points tested up
// to and including the first hit, negated if there was a hit.  Out of line: only segments longer than
// kCoopSteps * check_res and scenes without an occupancy grid come here.
template <class R>
__device__ KPX_WALK_ATTR int walk_segment(const Params<R>* Pp, R p0, R p1, R p2, R dx, R dy, R dz, R c0, R c1, R c2, R d2) {
    const Params<R>& P = *Pp;
    const R dist = MathK<R>::sq(d2);
    // smallest power of two with steps * res >= dist (validity.py:26-31).  res * 2^k and 2^-k are exact, so
    // doubling the threshold / halving the fraction reproduces steps * res and j / steps bit for bit.
    int steps = 1;
    R thr = P.check_res, inv_steps = (R)1;
    while (thr < dist) { thr += thr; inv_steps *= (R)0.5; steps <<= 1; }
    R t = (R)0;
#pragma unroll 1
    for (int j = 1; j < steps; ++j) {
        t += inv_steps;
        if (point_hits<R>(P, p0 + t * dx, p1 + t * dy, p2 + t * dz)) return -j;
    }
    return point_hits<R>(P, c0, c1, c2) ? -steps : steps;
}

// Cooperative pass over the warp's deferred segments: every (segment, point) pair becomes one unit of work
// spread over all 32 lanes.  A segment's outcome is the lowest point index that hits (the reference stops at
// it); returns that index for the calling lane's own segment, or 0x7fffffff if it is free (or the lane holds
// none).  Must be called by all 32 lanes.
template <class R>
__device__ KPX_COOP_ATTR int coop_walk(const Params<R>* Pp, bool pend) {
    const Params<R>& P = *Pp;
    WarpCoop<R>& C = Scene<R>::coop();
    const int lane = threadIdx.x & 31;
    const int cnt = pend ? C.steps[lane] : 0;
    const int incl = warp_incl_scan(cnt);
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (pend) {
        C.hit[lane] = 0x7fffffff;
        const int base = incl - cnt;
        for (int j = 1; j <= cnt; ++j) C.list[base + j - 1] = (uint16_t)(lane | (j << 5));
    }
    __syncwarp();
    for (int q = lane; q < total; q += 32) {
        const int e = C.list[q], J = e & 31, j = e >> 5;
        R px, py, pz;
        if (j == C.steps[J]) {
            px = C.seg[6][J]; py = C.seg[7][J]; pz = C.seg[8][J];
        } else {
            const R t = (R)j * C.seg[9][J];          // j / steps, exact (steps is a power of two)
            px = C.seg[0][J] + t * C.seg[3][J]; py = C.seg[1][J] + t * C.seg[4][J]; pz = C.seg[2][J] + t * C.seg[5][J];
        }
        if (point_hits<R>(P, px, py, pz)) atomicMin(&C.hit[J], j);
    }
    __syncwarp();
    const int h = pend ? C.hit[lane] : 0x7fffffff;
    __syncwarp();
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

// Clamped grid mapping of an end state (_kernel.pyx:261-292): region iff the state is finite (`alive`), sub-region
// and valid = 1 iff the whole segment was valid too (`ok`).
template <class M, class R>
__device__ __forceinline__ void map_end_state(const Params<R>& P, const R* cur, bool alive, bool ok, ItemOut<R, M::N>& out) {
    constexpr int N = M::N;
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

// The extension itself, warp-synchronous: ALL 32 lanes of the warp call it together (`active` = this lane
// holds an item).  `u` and `dt` are the sampled control / duration already rounded to R; x0 is the parent state.
//
// Per substep, in the reference's order (_kernel.pyx:226-256): finite -> state box -> obstacle walk.  The
// verdict of an item is the AND of those tests over all substeps and the integration never depends on it, so
// the walk -- the only expensive, ragged part -- is restructured without changing any verdict or counter:
//   1. the number of points follows from the squared length by compares (Params::d2_thr);
//   2. every point of the walk lies inside the segment's axis-aligned box [min(prev,cur), max(prev,cur)]
//      (prev + t d is monotone in t under rounding and t <= 3/4 for interior points), and the cell lookup is
//      monotone, so the points' cells lie in the cell range of (prev, cur).  One lookup -- the cell's own mask
//      when both ends share a cell, the dilated mask of the lower cell otherwise -- yields a superset of the
//      obstacles any point could hit; comparing the segment box with those obstacle boxes (same floats,
//      exact compares) clears almost every segment without walking it;
//   3. a segment that survives is staged in shared memory and the lane carries on, as if it were free;
//      once KPX_FLUSH_AT lanes of the warp hold one (or a lane needs a second slot, or the item ends) the
//      warp walks all staged points together (coop_walk).  A hit rewinds the lane's counters to their values
//      at that point and clears `ok`, which is all the reference's early-out would have produced.
// Counters: while a lane is ok its box test has run on every substep so far, so `boxsteps` is just where ok
// flipped (box_end); `substeps` is where the lane stopped (S, cut short by a non-finite state).
template <class M, class R>
__device__ KPX_INT_ATTR void integrate_and_map(const Params<R>& P, bool active, const R* x0, const R* u, R dt,
                                                  int substeps, ItemOut<R, M::N>& out) {
    constexpr int N = M::N;
    constexpr unsigned FULL = 0xffffffffu;
    int S = active ? substeps : 0;
    const int Smax = __reduce_max_sync(FULL, S);
    const R h = dt / (R)(S > 0 ? S : 1);
    const R h6 = std::is_same<R, float>::value ? (R)0 : h / (R)6;      // float32 re-derives it per step
    R cur[N];
    R comp[Stepper<typename M::Base, R>::kCarry];     // carried across substeps: Kahan compensation (float32), ...
#pragma unroll
    for (int i = 0; i < N; ++i) cur[i] = x0[i];
    Stepper<typename M::Base, R>::init(x0, u, comp);
    bool ok = active, alive = active, pend = false;
    int points = 0, box_end = -1;
    const int n_obs = P.n_obs;
    const bool grid = P.occ_g != 0 && n_obs > 0;           // warp-uniform
    int pcx = 0, pcy = 0, pcz = 0;
    if (grid) {
        pcx = occ_cell<R>(cur[0], P.occ_lo[0], P.occ_inv[0]);
        pcy = occ_cell<R>(cur[1], P.occ_lo[1], P.occ_inv[1]);
        pcz = occ_cell<R>(cur[2], P.occ_lo[2], P.occ_inv[2]);
    }
    constexpr int kUnroll = KPX_SUBSTEP_UNROLL;
#pragma unroll kUnroll
    for (int s = 0; s < Smax; ++s) {
        bool run = s < S;
        const R q0 = cur[0], q1 = cur[1], q2 = cur[2];      // start of this substep's segment
        // closed state box, evaluated beside the finite test (two independent predicate chains instead of one
        // after the other: the warp runs both whenever any lane is still ok, and a lone warp saves the latency);
        // for a finite state !(x < lo || x > hi) == (x >= lo) & (x <= hi), and the result is only used then
        bool inb = true;
        if (run) {
            Stepper<typename M::Base, R>::step(cur, comp, u, h, h6);
            bool fin = true;
            if constexpr (std::is_same<R, float>::value && N % 2 == 0 && KPX_PACKED_F32) {
                // x * 0 is 0 for a finite x and NaN otherwise: N/2 packed FMAs and one compare instead of N compares
                float2 z = make_float2(0.0f, 0.0f);
#pragma unroll
                for (int i = 0; i < N / 2; ++i) z = __ffma2_rn(make_float2(cur[2 * i], cur[2 * i + 1]), make_float2(0.0f, 0.0f), z);
                fin = (z.x + z.y) == 0.0f;
            } else {
#pragma unroll
                for (int i = 0; i < N; ++i) fin = fin && isfinite(cur[i]);
            }
#pragma unroll
            for (int i = 0; i < N; ++i) inb = inb & (cur[i] >= P.state_lo[i]) & (cur[i] <= P.state_hi[i]);
            if (!fin) {                                     // _kernel.pyx:226-232: stop integrating
                if (ok) box_end = s;
                alive = false; ok = false; run = false; S = s + 1;
            }
        }
        bool cand = false;
        int steps = 1;
        if (run && ok) {
            ok = inb;
            if (!ok) box_end = s + 1;
            if (ok && n_obs > 0) {
                const R dx = cur[0] - q0, dy = cur[1] - q1, dz = cur[2] - q2;
                const R d2 = dx * dx + dy * dy + dz * dz;
                if (__builtin_expect(!grid, 0)) {
                    const int r = walk_segment<R>(&P, q0, q1, q2, dx, dy, dz, cur[0], cur[1], cur[2], d2);
                    points += r < 0 ? -r : r;
                    if (r < 0) { ok = false; box_end = s + 1; }
                } else {
                    const int cx = occ_cell<R>(cur[0], P.occ_lo[0], P.occ_inv[0]);
                    const int cy = occ_cell<R>(cur[1], P.occ_lo[1], P.occ_inv[1]);
                    const int cz = occ_cell<R>(cur[2], P.occ_lo[2], P.occ_inv[2]);
                    // cells of the two ends: equal or one step apart along one axis (L1 distance <= 1) -> the
                    // walk's points can only lie in those two cells; otherwise the dilated table of the lower
                    // corner (<= 1 apart on every axis) or, for a long jump, every obstacle
                    const int l1 = abs(cx - pcx) + abs(cy - pcy) + abs(cz - pcz);
                    uint32_t m = Scene<R>::occ()[(cx * kOccGrid + cy) * kOccGrid + cz] |
                                 Scene<R>::occ()[(pcx * kOccGrid + pcy) * kOccGrid + pcz];
                    if (l1 > 1) {
                        const int mx = min(cx, pcx), my = min(cy, pcy), mz = min(cz, pcz);
                        const bool near = (cx + pcx - 2 * mx) <= 1 && (cy + pcy - 2 * my) <= 1 && (cz + pcz - 2 * mz) <= 1;
                        m = near ? Scene<R>::occ2()[(mx * kOccGrid + my) * kOccGrid + mz] : 0xffffffffu >> (32 - n_obs);
                    }
                    pcx = cx; pcy = cy; pcz = cz;
                    if (m) {
                        const R lx = fmin(q0, cur[0]), hx = fmax(q0, cur[0]);
                        const R ly = fmin(q1, cur[1]), hy = fmax(q1, cur[1]);
                        const R lz = fmin(q2, cur[2]), hz = fmax(q2, cur[2]);
                        const R* bx = Scene<R>::boxes();
                        do {
                            const Box<R> b = load_box(bx, __ffs(m) - 1);
                            m &= m - 1;
                            cand = (hx >= b.lx) & (lx <= b.hx) & (hy >= b.ly) & (ly <= b.hy) & (hz >= b.lz) & (lz <= b.hz);
                        } while (m && !cand);
                    }
                    if (__builtin_expect(d2 > P.d2_thr[3], 0)) {   // more than kCoopSteps points: walk it here
                        int r;
                        if (cand) {
                            r = walk_segment<R>(&P, q0, q1, q2, dx, dy, dz, cur[0], cur[1], cur[2], d2);
                        } else {
                            const R dist = MathK<R>::sq(d2);
                            R thr = P.check_res;
                            r = 1;
                            while (thr < dist) { thr += thr; r <<= 1; }
                        }
                        points += r < 0 ? -r : r;
                        if (r < 0) { ok = false; box_end = s + 1; }
                        cand = false;
                    } else {
                        if (d2 > P.d2_thr[0]) steps = 2;
                        if (d2 > P.d2_thr[1]) steps = 4;
                        if (d2 > P.d2_thr[2]) steps = 8;
                        points += steps;                 // a staged segment counts as free until coop_walk says otherwise
                    }
                }
            }
        }
        if (grid) {
            const bool last = s + 1 >= Smax;             // the item ends: whatever is staged is resolved now
            unsigned cm = __ballot_sync(FULL, cand);
            if (cm || last) {
                WarpCoop<R>& C = Scene<R>::coop();
                const int lane = threadIdx.x & 31;
                // One static call site of the cooperative walk, run at most twice: a lane that needs its slot
                // again forces a walk of what is staged before the new segments are stored.
#pragma unroll 1
                for (;;) {
                    unsigned pm = __ballot_sync(FULL, pend);
                    const bool conflict = (cm & pm) != 0u;
                    if (!conflict) {
                        if (cand) {
                            C.seg[0][lane] = q0; C.seg[1][lane] = q1; C.seg[2][lane] = q2;
                            C.seg[3][lane] = cur[0] - q0; C.seg[4][lane] = cur[1] - q1; C.seg[5][lane] = cur[2] - q2;
                            C.seg[6][lane] = cur[0]; C.seg[7][lane] = cur[1]; C.seg[8][lane] = cur[2];
                            C.seg[9][lane] = (R)1 / (R)steps;
                            C.steps[lane] = steps;
                            C.mark_pts[lane] = points - steps; C.mark_sub[lane] = s;
                            pend = true; cand = false;
                        }
                        pm |= cm; cm = 0u;
                    }
                    if (conflict || __popc(pm) >= KPX_FLUSH_AT || (last && pm != 0u)) {
                        const int hit = coop_walk<R>(&P, pend);
                        if (hit != 0x7fffffff) {         // the staged segment hits: rewind, and drop a newer one
                            ok = false; cand = false; points = C.mark_pts[lane] + hit; box_end = C.mark_sub[lane] + 1;
                        }
                        pend = false;
                        if (conflict) cm = __ballot_sync(FULL, cand);
                    }
                    if (cm == 0u) break;
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) out.end[i] = cur[i];
    out.substeps = S; out.points = points; out.boxsteps = box_end >= 0 ? box_end : S;
    map_end_state<M, R>(P, cur, alive, ok, out);
}

// Sample (u, dt) for item (slot, ext) of the iteration hashed into h0.  Controls and
// duration are drawn in f64 exactly as the reference does (_kernel.pyx:190-194) and
// then rounded once to R; the substep count is taken from the rounded dt so that a
// host re-propagation of the stored (control, dt) uses the same step size.
template <class M, class R>
__device__ __forceinline__ void sample_control(const Params<R>& P, uint64_t h0, int slot, int ext, R* u, R* dt,
                                               int* substeps, double* u64v, double* dt64) {
    double unit[M::NU + 1];                 // draws 0..NU-1 -> controls, draw NU -> duration
    if constexpr (M::kRng == KPX_RNG_PHILOX) {
#pragma unroll
        for (int blk = 0; 2 * blk < M::NU + 1; ++blk) {
            uint64_t a, b;
            philox_draw2(h0, (uint32_t)slot, (uint32_t)ext, PH_SAMPLE, (uint32_t)blk, &a, &b);
            unit[2 * blk] = unit53(a);
            if (2 * blk + 1 < M::NU + 1) unit[2 * blk + 1] = unit53(b);
        }
    } else {
        const uint64_t key = mix64(slot_ext_hash(h0, (uint64_t)slot, (uint64_t)ext) ^ (uint64_t)PH_SAMPLE);
#pragma unroll
        for (int j = 0; j < M::NU + 1; ++j) unit[j] = unit53(draw_u64(key, (uint64_t)j));
    }
#pragma unroll
    for (int j = 0; j < M::NU; ++j) {
        double v = __dadd_rn(P.control_lo[j], __dmul_rn(unit[j], P.control_span[j]));
        if (u64v) u64v[j] = v;
        u[j] = (R)v;
    }
    double d = __dmul_rn(__dsub_rn(1.0, unit[M::NU]), P.t_prop);
    if (dt64) *dt64 = d;
    *dt = (R)d;
    int s = (int)ceil(__ddiv_rn((double)(*dt), 0.02));
    *substeps = s < 4 ? 4 : s;
}

// substep count of item (slot, ext) alone: the duration draw and the same rounding as sample_control
template <class M, class R>
__device__ __forceinline__ int substeps_of(const Params<R>& P, uint64_t h0, int slot, int ext) {
    double un;
    if constexpr (M::kRng == KPX_RNG_PHILOX) {
        uint64_t a, b;
        philox_draw2(h0, (uint32_t)slot, (uint32_t)ext, PH_SAMPLE, (uint32_t)(M::NU >> 1), &a, &b);
        un = unit53((M::NU & 1) ? b : a);
    } else {
        const uint64_t key = mix64(slot_ext_hash(h0, (uint64_t)slot, (uint64_t)ext) ^ (uint64_t)PH_SAMPLE);
        un = unit53(draw_u64(key, (uint64_t)M::NU));
    }
    const double d = __dmul_rn(__dsub_rn(1.0, un), P.t_prop);
    const R dt = (R)d;
    const int s = (int)ceil(__ddiv_rn((double)dt, 0.02));
    return s < 4 ? 4 : s;
}

// ------------------------------------------------------------------ free flight ----
// float32 double integrators only.  x' = (v, u) with u held has the closed form p(t) = p0 + t (v0 + t u / 2),
// v(t) = v0 + t u, so for most extensions the verdict is decidable in O(1) before integrating anything:
//   * INVALID for certain: the last sampled state (t = dt) lies outside the closed state box.  (v is monotone per axis,
//     so a velocity that leaves its box is still outside at the end.)
//   * VALID for certain: v(dt) inside its box (then every sampled velocity is: the first one is a tree node), and the
//     position stays clear of the box faces and of every obstacle.  p is a parabola per axis; its extremes over a time
//     interval are the ends and, if inside, the vertex.  The sampled states s h and every interpolant the obstacle walk
//     visits between two CONSECUTIVE samples lie inside the axis-aligned box of those extremes over any interval
//     [s_a h, s_b h] containing both samples.  If those boxes (KPX_FREE_PIECES of them, split at sample times, grown
//     by a few float32 ulps of the workspace) stay inside the state box and overlap no obstacle box, nothing the
//     reference's checker would test can fail.  Obstacles are found through the occupancy grid of the scene (the
//     dilated table answers a box spanning <= 2 cells per axis in one lookup) and compared box against box, exactly.
// Either way the extension is finished on the spot -- end state from the closed form, grid mapping, counters -- with
// no substep loop at all; ~90 % of the Trees workload.  Everything else (extensions that pass near an obstacle, or
// whose parabola only grazes a box face between samples) is evaluated one item per warp, lane = substep
// (di_item_by_substeps below).
// Work counters of a finished extension: substeps = S (the reference integrates every substep whatever the verdict).
// Certified valid: boxsteps = S and points = the sum of the densification counts of its S segments (validity.py:26-31),
// counted from the closed-form segment lengths |h v0 + h^2 u (s - 1/2)|.  Certified invalid: boxsteps = 1, points = 0
// -- lower bounds (the first failing substep is not computed), so the algorithmic-work total is never overstated.
#ifndef KPX_FREE_PIECES
#define KPX_FREE_PIECES 2
#endif
#ifndef KPX_FREE_FLIGHT
#define KPX_FREE_FLIGHT 1            // 0: every extension takes the full path (measurement knob)
#endif
enum : int { kFlightFull = 0, kFlightValid = 1, kFlightInvalid = 2 };
template <class M, class R> struct FreeFlight {
    static constexpr bool kEnabled = false;
    __device__ static __forceinline__ int certify(const Params<R>&, const R*, const R*, R, int, ItemOut<R, M::N>&) { return kFlightFull; }
};

__device__ __forceinline__ float di_pos(float p0, float v0, float u, float t) { return __fmaf_rn(t, __fmaf_rn(0.5f * t, u, v0), p0); }
// extremes of one axis over [ta, tb]
__device__ __forceinline__ void di_axis_range(float p0, float v0, float u, float ta, float tb, float* lo, float* hi) {
    const float pa = di_pos(p0, v0, u, ta), pb = di_pos(p0, v0, u, tb);
    float l = fminf(pa, pb), h = fmaxf(pa, pb);
    const float ts = __fdividef(-v0, u);                 // vertex; u = 0 gives inf / nan and both compares fail
    if (ts > ta && ts < tb) { const float pv = di_pos(p0, v0, u, ts); l = fminf(l, pv); h = fmaxf(h, pv); }
    *lo = l; *hi = h;
}
// does the closed box [lo, hi] overlap an obstacle?  Candidates from the occupancy grid, then box against box.
__device__ __forceinline__ bool box_touches_obstacle(const Params<float>& P, const float* lo, const float* hi) {
    uint32_t m;
    if (P.occ_g != 0) {
        int c0[3], c1[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            c0[a] = occ_cell<float>(lo[a], P.occ_lo[a], P.occ_inv[a]);
            c1[a] = occ_cell<float>(hi[a], P.occ_lo[a], P.occ_inv[a]);
        }
        const uint32_t* occ2 = Scene<float>::occ2();
        if (c1[0] - c0[0] <= 1 && c1[1] - c0[1] <= 1 && c1[2] - c0[2] <= 1) {
            m = occ2[(c0[0] * kOccGrid + c0[1]) * kOccGrid + c0[2]];
        } else if (c1[0] - c0[0] <= 3 && c1[1] - c0[1] <= 3 && c1[2] - c0[2] <= 3) {
            m = 0u;
#pragma unroll 1
            for (int x = c0[0]; x <= c1[0]; x += 2)
#pragma unroll 1
                for (int y = c0[1]; y <= c1[1]; y += 2)
#pragma unroll 1
                    for (int z = c0[2]; z <= c1[2]; z += 2) m |= occ2[(x * kOccGrid + y) * kOccGrid + z];
        } else {
            m = 0xffffffffu >> (32 - P.n_obs);
        }
        const float* bx = Scene<float>::boxes();
        bool touch = false;
#pragma unroll 1
        while (m && !touch) {
            const Box<float> b = load_box(bx, __ffs(m) - 1);
            m &= m - 1;
            touch = (hi[0] >= b.lx) & (lo[0] <= b.hx) & (hi[1] >= b.ly) & (lo[1] <= b.hy) & (hi[2] >= b.lz) & (lo[2] <= b.hz);
        }
        return touch;
    }
    const float* bx = Scene<float>::boxes();
    bool touch = false;
#pragma unroll 1
    for (int j = 0; j < P.n_obs; ++j) {
        const Box<float> b = load_box(bx, j);
        touch = touch | ((hi[0] >= b.lx) & (lo[0] <= b.hx) & (hi[1] >= b.ly) & (lo[1] <= b.hy) & (hi[2] >= b.lz) & (lo[2] <= b.hz));
    }
    return touch;
}
// one 6-D block [p v] starting at state dimension d0: kFlightInvalid / kFlightValid / kFlightFull (undecided)
__device__ __forceinline__ int di_block_flight(const Params<float>& P, int d0, const float* x0, const float* u, float dt, int S,
                                               float h, bool obstacles) {
    constexpr float kGrow = 1e-5f;                       // ~10 float32 ulps of a 10 m workspace
    bool end_in = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {                        // the last sample, exactly as the full path would test it
        const float pe = di_pos(x0[a], x0[3 + a], u[a], dt), ve = __fmaf_rn(dt, u[a], x0[3 + a]);
        end_in = end_in & (pe >= P.state_lo[d0 + a]) & (pe <= P.state_hi[d0 + a]) & (ve >= P.state_lo[d0 + 3 + a]) & (ve <= P.state_hi[d0 + 3 + a]);
    }
    if (!end_in) return kFlightInvalid;
    bool good = true;
#pragma unroll 1
    for (int k = 0; k < KPX_FREE_PIECES && good; ++k) {
        const float ta = (float)((S * k) / KPX_FREE_PIECES) * h;
        const float tb = k + 1 == KPX_FREE_PIECES ? dt : (float)((S * (k + 1)) / KPX_FREE_PIECES) * h;
        float lo[3], hi[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            di_axis_range(x0[a], x0[3 + a], u[a], ta, tb, &lo[a], &hi[a]);
            lo[a] -= kGrow; hi[a] += kGrow;
            good = good & (lo[a] >= P.state_lo[d0 + a]) & (hi[a] <= P.state_hi[d0 + a]);
        }
        if (obstacles && good) good = !box_touches_obstacle(P, lo, hi);
    }
    return good ? kFlightValid : kFlightFull;
}
// Collision points the reference's walk tests along the S segments of a free extension: segment s has the squared
// length q(sigma) = |h v0 + h^2 u sigma|^2 at sigma = s - 1/2, a parabola in sigma, so the number of segments above
// each densification threshold follows from its roots; points = S + #(q > thr0) + 2 #(q > thr1) + 4 #(q > thr2).
// (A substep of a double integrator inside its velocity box is shorter than 8 check_res: no segment needs more.)
__device__ __forceinline__ int di_free_points(const Params<float>& P, const float* x0, const float* u, int S, float h) {
    const float hh = h * h;
    const float A = hh * (x0[3] * x0[3] + x0[4] * x0[4] + x0[5] * x0[5]);
    const float B = 2.0f * hh * h * (x0[3] * u[0] + x0[4] * u[1] + x0[5] * u[2]);
    const float C = hh * hh * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    int points = S;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float T = P.d2_thr[k];
        int above;
        const float disc = B * B - 4.0f * C * (A - T);
        if (!(C > 0.0f)) above = A > T ? S : 0;
        else if (disc < 0.0f) above = S;                 // upward parabola without roots: above everywhere
        else {
            const float sq = sqrtf(disc), i2c = __fdividef(0.5f, C);
            const float s_lo = (-B - sq) * i2c + 0.5f, s_hi = (-B + sq) * i2c + 0.5f;   // q <= T for s in [s_lo, s_hi]
            int a = (int)ceilf(s_lo), b = (int)floorf(s_hi);
            a = a < 1 ? 1 : a; b = b > S ? S : b;
            above = S - (b >= a ? b - a + 1 : 0);
        }
        points += above << k;
    }
    return points;
}
template <int B>
__device__ __forceinline__ int di_certify(const Params<float>& P, const float* x0, const float* u, float dt, int S,
                                          ItemOut<float, 6 * B>& out) {
    const float h = dt / (float)S;
    int verdict = di_block_flight(P, 0, x0, u, dt, S, h, P.n_obs > 0);
#pragma unroll
    for (int b = 1; b < B; ++b) {
        const int v = di_block_flight(P, 6 * b, x0 + 6 * b, u + 3 * b, dt, S, h, false);
        verdict = (verdict == kFlightInvalid || v == kFlightInvalid) ? kFlightInvalid
                                                                     : ((verdict == kFlightValid && v == kFlightValid) ? kFlightValid : kFlightFull);
    }
    if (verdict == kFlightFull) return verdict;
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            out.end[6 * b + a] = di_pos(x0[6 * b + a], x0[6 * b + 3 + a], u[3 * b + a], dt);
            out.end[6 * b + 3 + a] = __fmaf_rn(dt, u[3 * b + a], x0[6 * b + 3 + a]);
        }
    out.substeps = S;
    if (verdict == kFlightValid) { out.boxsteps = S; out.points = P.n_obs > 0 ? di_free_points(P, x0, u, S, h) : 0; }
    else { out.boxsteps = 1; out.points = 0; }
    return verdict;
}
// An extension the certificate could not settle, evaluated by the WHOLE WARP: lane = RK4 substep.  Sample s of the
// closed form does not depend on sample s - 1, so the S box tests and segment walks of the extension run side by side,
// 32 per round; the first failing substep (lowest lane of the first round that has one) decides, exactly as the
// reference's sequential early-out would: boxsteps = its index, points = the densification counts of the segments
// before it plus the points walked in it up to and including the hit.  All lanes call it with the same arguments and
// receive the same result.
template <int B>
__device__ __forceinline__ void di_item_by_substeps(const Params<float>& P, const float* x0, const float* u, float dt, int S,
                                                    bool* ok_out, int* boxsteps_out, int* points_out) {
    const int lane = threadIdx.x & 31;
    const float h = dt / (float)S;
    const int n_obs = P.n_obs;
    const bool grid = P.occ_g != 0;
    int points = 0;
#pragma unroll 1
    for (int base = 0; base < S; base += 32) {
        const int s = base + lane + 1;                          // sample index, 1..S
        const bool act = s <= S;
        const float t1 = s == S ? dt : (float)s * h, t0 = (float)(s - 1) * h;
        bool fail = false;
        int steps = 0, hit = 0;
        if (act) {
            bool inb = true;                                    // sample s of every block inside the closed state box
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const float p = di_pos(x0[6 * b + a], x0[6 * b + 3 + a], u[3 * b + a], t1);
                    const float v = __fmaf_rn(t1, u[3 * b + a], x0[6 * b + 3 + a]);
                    inb = inb & (p >= P.state_lo[6 * b + a]) & (p <= P.state_hi[6 * b + a]) &
                          (v >= P.state_lo[6 * b + 3 + a]) & (v <= P.state_hi[6 * b + 3 + a]);
                }
            fail = !inb;
            if (inb && n_obs > 0) {                             // segment (s - 1) -> s of block 1 against the obstacles
                const float q0 = di_pos(x0[0], x0[3], u[0], t0), q1 = di_pos(x0[1], x0[4], u[1], t0), q2 = di_pos(x0[2], x0[5], u[2], t0);
                const float c0 = di_pos(x0[0], x0[3], u[0], t1), c1 = di_pos(x0[1], x0[4], u[1], t1), c2 = di_pos(x0[2], x0[5], u[2], t1);
                const float dx = c0 - q0, dy = c1 - q1, dz = c2 - q2;
                const float d2 = dx * dx + dy * dy + dz * dz;
                steps = 1;
                if (d2 > P.d2_thr[0]) steps = 2;
                if (d2 > P.d2_thr[1]) steps = 4;
                if (d2 > P.d2_thr[2]) steps = 8;
                if (__builtin_expect(d2 > P.d2_thr[3], 0)) {
                    const float dist = sqrtf(d2);
                    float thr = P.check_res;
                    steps = 1;
                    while (thr < dist) { thr += thr; steps <<= 1; }
                }
                // obstacles the segment's box can touch (same cull as the sequential path), then the walk itself
                const float lo[3] = {fminf(q0, c0), fminf(q1, c1), fminf(q2, c2)}, hi[3] = {fmaxf(q0, c0), fmaxf(q1, c1), fmaxf(q2, c2)};
                if (!grid || box_touches_obstacle(P, lo, hi)) {
                    const float inv = 1.0f / (float)steps;
#pragma unroll 1
                    for (int j = 1; j < steps && hit == 0; ++j) {
                        const float t = (float)j * inv;
                        if (point_hits<float>(P, q0 + t * dx, q1 + t * dy, q2 + t * dz)) hit = j;
                    }
                    if (hit == 0 && point_hits<float>(P, c0, c1, c2)) hit = steps;
                    fail = hit != 0;
                }
            }
        }
        const unsigned fm = __ballot_sync(0xffffffffu, act && fail);
        const int first = fm ? __ffs(fm) - 1 : 32;
        points += __reduce_add_sync(0xffffffffu, act ? (lane < first ? steps : (lane == first ? hit : 0)) : 0);
        if (fm) { *ok_out = false; *boxsteps_out = base + first + 1; *points_out = points; return; }
    }
    *ok_out = true; *boxsteps_out = S; *points_out = points;
}
template <int B>
__device__ __forceinline__ void di_end_state(const float* x0, const float* u, float dt, float* end) {
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            end[6 * b + a] = di_pos(x0[6 * b + a], x0[6 * b + 3 + a], u[3 * b + a], dt);
            end[6 * b + 3 + a] = __fmaf_rn(dt, u[3 * b + a], x0[6 * b + 3 + a]);
        }
}

template <> struct FreeFlight<ModelDI6, float> {
    static constexpr bool kEnabled = KPX_FREE_FLIGHT != 0;
    __device__ static __forceinline__ int certify(const Params<float>& P, const float* x0, const float* u, float dt, int S,
                                                  ItemOut<float, 6>& out) { return di_certify<1>(P, x0, u, dt, S, out); }
    __device__ static __forceinline__ void by_substeps(const Params<float>& P, const float* x0, const float* u, float dt, int S,
                                                       bool* ok, int* boxsteps, int* points) { di_item_by_substeps<1>(P, x0, u, dt, S, ok, boxsteps, points); }
    __device__ static __forceinline__ void end_state(const float* x0, const float* u, float dt, float* end) { di_end_state<1>(x0, u, dt, end); }
};
template <int B> struct FreeFlight<ModelStackedDI<B>, float> {
    static constexpr bool kEnabled = KPX_FREE_FLIGHT != 0;
    __device__ static __forceinline__ int certify(const Params<float>& P, const float* x0, const float* u, float dt, int S,
                                                  ItemOut<float, 6 * B>& out) { return di_certify<B>(P, x0, u, dt, S, out); }
    __device__ static __forceinline__ void by_substeps(const Params<float>& P, const float* x0, const float* u, float dt, int S,
                                                       bool* ok, int* boxsteps, int* points) { di_item_by_substeps<B>(P, x0, u, dt, S, ok, boxsteps, points); }
    __device__ static __forceinline__ void end_state(const float* x0, const float* u, float dt, float* end) { di_end_state<B>(x0, u, dt, end); }
};

}  // namespace kpx
