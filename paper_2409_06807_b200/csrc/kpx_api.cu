// kpx_api.cu -- the C ABI declared in include/kpx.h.
//
// Owns device memory (one slab per handle, carved into the node-major arena, the region
// state and the per-iteration scratch), stages the few host inputs, launches the
// persistent planner kernel and copies results back.  No CPU fallback exists:
// every entry point either runs the CUDA path or returns an error code.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <vector>

#include "kpx_launch.h"

using namespace kpx;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e__ = (call);                                                                  \
        if (e__ != cudaSuccess) return fail(KPX_E_CUDA, "%s: %s", #call, cudaGetErrorString(e__)); \
    } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int check_problem(const kpx_problem* pr) {
    if (!pr) return fail(KPX_E_ARG, "problem is null");
    if (pr->n > KPX_MAX_DIM || pr->nu > KPX_MAX_CONTROL)
        return fail(KPX_E_LIMIT, "state/control dimension exceeds kernel limits");
    if (pr->n < 3 || pr->nu < 1 || pr->grid_n < 3 || pr->grid_n > pr->n) return fail(KPX_E_ARG, "bad dimensions");
    if (pr->model_id < 0 || pr->model_id > KPX_MODEL_STACKED_DI) return fail(KPX_E_ARG, "unknown model id");
    if (pr->rng != KPX_RNG_SPLITMIX64 && pr->rng != KPX_RNG_PHILOX) return fail(KPX_E_ARG, "unknown rng");
    if (pr->n_obs < 0 || (pr->n_obs > 0 && (!pr->obs_min || !pr->obs_max))) return fail(KPX_E_ARG, "bad obstacles");
    if (pr->subcells < 1 || pr->lambda_max < 1 || pr->t_e < 1) return fail(KPX_E_ARG, "bad configuration");
    if (pr->t_e_start < 0 || pr->t_e_start > pr->t_e || (pr->t_e_start > 0 && !(pr->t_e_growth >= 1.0)))
        return fail(KPX_E_ARG, "adaptive capacity needs 1 <= t_e_start <= t_e and t_e_growth >= 1");
    double regions = 1.0;
    for (int d = 0; d < pr->grid_n; ++d) regions *= (double)pr->grid_cells[d];
    if (regions * pr->subcells * pr->subcells * pr->subcells >= 1073741824.0)
        return fail(KPX_E_LIMIT, "regions x sub-cells must stay below 2^30");
    if (pr->t_e >= (1ll << 30)) return fail(KPX_E_LIMIT, "t_e too large");
    return KPX_OK;
}

// obstacles -> device boxes [n_obs][8] = {min xyz, -, max xyz, -} in the launch precision
int upload_obstacles(const kpx_problem& pr, int precision, int n_obs, const double* omin, const double* omax, void* dev,
                     uint32_t* occ_dev, cudaStream_t st) {
    if (n_obs == 0) return KPX_OK;
    {
        std::vector<uint32_t> masks(2 * (size_t)kOccCells);      // exact table | dilated table
        if (precision == KPX_F64) occupancy_masks_f64(pr, n_obs, omin, omax, masks.data());
        else occupancy_masks_f32(pr, n_obs, omin, omax, masks.data());
        CU(cudaMemcpyAsync(occ_dev, masks.data(), masks.size() * 4, cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
    }
    if (precision == KPX_F64) {
        std::vector<double> h(8 * (size_t)n_obs, 0.0);
        for (int k = 0; k < n_obs; ++k)
            for (int a = 0; a < 3; ++a) { h[8 * k + a] = omin[3 * k + a]; h[8 * k + 4 + a] = omax[3 * k + a]; }
        CU(cudaMemcpyAsync(dev, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
    } else {
        std::vector<float> h(8 * (size_t)n_obs, 0.0f);
        for (int k = 0; k < n_obs; ++k)
            for (int a = 0; a < 3; ++a) {
                h[8 * k + a] = (float)omin[3 * k + a];
                h[8 * k + 4 + a] = (float)omax[3 * k + a];
            }
        CU(cudaMemcpyAsync(dev, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st));
        CU(cudaStreamSynchronize(st));
    }
    return KPX_OK;
}

// a pair of timing events that is destroyed on every return path
struct EventPair {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaError_t create() { cudaError_t e = cudaEventCreate(&e0); return e != cudaSuccess ? e : cudaEventCreate(&e1); }
    ~EventPair() { if (e0) cudaEventDestroy(e0); if (e1) cudaEventDestroy(e1); }
};

struct Carver {
    size_t off = 0;
    size_t take(size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; }
};

}  // namespace

constexpr int kHandoffLevels = KPX_HANDOFF_STAGES;   // hand-off stages at most; kpx_batch::hand_width holds the ones in use

struct kpx_batch {
    kpx_problem prob;
    std::vector<double> obs_min, obs_max;
    int precision = KPX_F64, n_teams = 1, team_ctas = 1, device = 0;
    int max_chunks = 0, max_trace = 4096, max_chain = KPX_MAX_CHAIN;
    int obs_cap = 0;                   // obstacles the device buffers (and the shared-memory scene) were sized for
    // obstacle sets ("scenes") a query can name: n_scenes x scene_obs boxes, each set padded to scene_obs boxes with
    // boxes nothing can hit; scene 0 is the problem's own.  prob.n_obs == scene_obs.
    int n_scenes = 1, scene_obs = 0, scenes_alloc = 0;
    std::vector<double> sc_min, sc_max;
    bool cooperative = false, latency = false;
    size_t rs = 8, smem = 0;
    int cap = 0, cap_pad = 0, regions = 0, subs = 0, claim_shift = 30;
    char* slab = nullptr;
    size_t ws_bytes = 0;
    std::vector<Workspace> ws_host;
    Workspace* ws_dev = nullptr;
    void* obs_dev = nullptr;
    double* boxes64_dev = nullptr;     // float64 boxes for kpx_batch_validate (whatever the tree precision)
    uint32_t* occ_dev = nullptr;
    unsigned int* queue_dev = nullptr;
    QueryIn* q_dev = nullptr;
    kpx_query_result* r_dev = nullptr;
    long long q_cap = 0;
    double *bc_start = nullptr, *bc_ctrl = nullptr, *bc_dt = nullptr;
    long long bc_cap = 0, n_uploaded = 0;
    double *bp_start = nullptr, *bp_ctrl = nullptr, *bp_dt = nullptr;   // packed copies of the chains (download)
    long long* bp_off = nullptr;
    double* bp_host = nullptr;         // pinned staging of the packed chains
    size_t bp_host_cap = 0;
    size_t d2h_chain_bytes = 0;        // chain bytes the last download moved
    bool want_chains = false;
    std::vector<QueryIn> q_stage;
    uint32_t** peers_dev = nullptr;
    int peers_cap = 0;
    // single-plan state
    bool fresh = false;      // reset requested, not yet consumed by a run
    bool loaded = false;
    QueryIn q_host;
    unsigned long long launches = 0;
    ResultPacket* pk_host = nullptr;   // pinned
    QueryIn* q_pinned = nullptr;       // pinned
    bool pk_valid = false;
    // hand-off of a batch's last queries to wider teams (kpx_batch_launch)
    int max_resident = 0;              // CTAs of the plan kernel the device holds at once
    bool handoff = true;
    bool auto_width = false;           // kpx_batch_create(team_ctas = 0): teams as wide as the team count leaves room for
    unsigned int* hand_dev = nullptr;  // [0..7] idle teams per stage, [8..15] suspended queries per stage
    int2* susp_dev = nullptr;          // [kHandoffLevels][n_teams] (workspace, query)
    int hand_levels = 6, hand_width[kHandoffLevels] = {2, 4, 8, 16, 64, 512};   // CTAs per team of the follow-up stages (clamped to the device)
};

struct kpx_plan { kpx_batch b; };

namespace {

void destroy_batch(kpx_batch& b) {
    cudaSetDevice(b.device);
    cudaFree(b.slab); cudaFree(b.ws_dev); cudaFree(b.obs_dev); cudaFree(b.boxes64_dev); cudaFree(b.occ_dev); cudaFree(b.queue_dev); cudaFree(b.hand_dev); cudaFree(b.susp_dev); cudaFree(b.q_dev);
    cudaFree(b.r_dev); cudaFree(b.bc_start); cudaFree(b.bc_ctrl); cudaFree(b.bc_dt); cudaFree(b.peers_dev);
    cudaFree(b.bp_start); cudaFree(b.bp_ctrl); cudaFree(b.bp_dt); cudaFree(b.bp_off); cudaFreeHost(b.bp_host);
    cudaFreeHost(b.pk_host); cudaFreeHost(b.q_pinned);
}

int blocks_per_sm(const kpx_batch& b) {
    if (b.prob.rng == KPX_RNG_PHILOX)
        return b.precision == KPX_F64 ? plan_blocks_per_sm_f64p(b.prob.model_id, b.prob.n, b.smem, b.latency)
                                      : plan_blocks_per_sm_f32p(b.prob.model_id, b.prob.n, b.smem, b.latency);
    return b.precision == KPX_F64 ? plan_blocks_per_sm_f64(b.prob.model_id, b.prob.n, b.smem, b.latency)
                                  : plan_blocks_per_sm_f32(b.prob.model_id, b.prob.n, b.smem, b.latency);
}

// (re)build the device copies of every obstacle set: boxes in the launch precision + occupancy tables per scene
int upload_scenes(kpx_batch& b) {
    const int k = b.scene_obs;
    if (b.n_scenes > b.scenes_alloc) {
        cudaFree(b.obs_dev); cudaFree(b.occ_dev);
        b.obs_dev = nullptr; b.occ_dev = nullptr;
        CU(cudaMalloc(&b.obs_dev, 8 * (size_t)std::max(b.obs_cap, 1) * b.rs * (size_t)b.n_scenes));
        CU(cudaMalloc(&b.occ_dev, 2 * sizeof(uint32_t) * (size_t)kOccCells * (size_t)b.n_scenes));
        b.scenes_alloc = b.n_scenes;
    }
    b.prob.n_obs = k;
    b.obs_min.assign(b.sc_min.begin(), b.sc_min.begin() + 3 * (size_t)k);      // scene 0: what prob.obs_min points at
    b.obs_max.assign(b.sc_max.begin(), b.sc_max.begin() + 3 * (size_t)k);
    b.prob.obs_min = b.obs_min.data(); b.prob.obs_max = b.obs_max.data();
    cudaFree(b.boxes64_dev); b.boxes64_dev = nullptr;                           // rebuilt on the next validation
    for (int sc = 0; sc < b.n_scenes; ++sc) {
        int rc = upload_obstacles(b.prob, b.precision, k, b.sc_min.data() + 3 * (size_t)sc * k, b.sc_max.data() + 3 * (size_t)sc * k,
                                  (char*)b.obs_dev + 8 * (size_t)k * b.rs * sc, b.occ_dev + 2 * (size_t)kOccCells * sc, 0);
        if (rc) return rc;
    }
    return KPX_OK;
}

// allocate everything a batch of n_teams workspaces needs
int init_batch(kpx_batch& b, const kpx_problem* prob, int precision, int n_teams, int team_ctas, int max_chain,
               int device) {
    int rc = check_problem(prob);
    if (rc) return rc;
    if (precision != KPX_F64 && precision != KPX_F32) return fail(KPX_E_ARG, "precision must be KPX_F64 or KPX_F32");
    CU(cudaSetDevice(device));
    b.device = device;
    b.prob = *prob;
    b.obs_min.assign(prob->obs_min, prob->obs_min + 3 * (size_t)prob->n_obs);
    b.obs_max.assign(prob->obs_max, prob->obs_max + 3 * (size_t)prob->n_obs);
    b.prob.obs_min = b.obs_min.data(); b.prob.obs_max = b.obs_max.data();
    b.precision = precision; b.rs = precision == KPX_F64 ? 8 : 4;
    b.cap = (int)prob->t_e;
    b.cap_pad = (int)align_up((size_t)b.cap, kChunk) + kChunk;
    b.max_chunks = b.cap_pad / kChunk + 1;
    b.max_chain = max_chain > 0 ? max_chain : KPX_MAX_CHAIN;
    long long regions = 1;
    for (int d = 0; d < prob->grid_n; ++d) regions *= prob->grid_cells[d];
    b.regions = (int)regions;
    b.subs = prob->subcells * prob->subcells * prob->subcells;
    // after the scene: one int array shared by the chunk prefixes (max_chunks + 1) and the block prefix of the
    // estimate list (one entry per 1024 regions + 1)
    const size_t n_blocks = ((size_t)b.regions + 1023) / 1024;
    b.smem = scene_smem_bytes(prob->n_obs, b.rs) + align_up((std::max((size_t)b.max_chunks, n_blocks) + 2) * sizeof(int), 16);
    if (b.smem > 200 * 1024) return fail(KPX_E_LIMIT, "t_e / obstacle count need more shared memory than one SM has");

    cudaDeviceProp dp;
    CU(cudaGetDeviceProperties(&dp, device));
    b.latency = team_ctas <= 0;     // whole GPU on one query
    const int bps = blocks_per_sm(b);
    if (bps < 1) return fail(KPX_E_ARG, "no kernel for model_id=%d n=%d", prob->model_id, prob->n);
    const int max_resident = bps * dp.multiProcessorCount;
    if (team_ctas <= 0) {
        n_teams = 1;
        team_ctas = max_resident;
    }
    b.max_resident = max_resident;
    if (const char* e = getenv("KPX_HANDOFF")) b.handoff = atoi(e) != 0;     // measurement knobs
    if (const char* e = getenv("KPX_HANDOFF_WIDTHS")) {
        b.hand_levels = 0;
        for (const char* p = e; *p && b.hand_levels < kHandoffLevels;) {
            b.hand_width[b.hand_levels++] = std::max(2, atoi(p));
            while (*p && *p != ',') ++p;
            if (*p == ',') ++p;
        }
    }
    if (n_teams < 0) n_teams = std::max(1, std::min(-n_teams, max_resident / team_ctas));   // at most -n_teams, never beyond what is co-resident
    if (n_teams == 0) n_teams = std::max(1, max_resident / team_ctas);     // as many teams as fit the device
    if (n_teams < 1) return fail(KPX_E_ARG, "n_teams must be >= 1");
    if (b.auto_width) {                // few queries on a big device: 2, 4, 8 or 16 CTAs per team from the start
        team_ctas = 1;
        while (team_ctas < 16 && (long long)n_teams * team_ctas * 2 <= max_resident) team_ctas *= 2;
    }
    b.cooperative = team_ctas > 1;
    if (b.cooperative && (long long)n_teams * team_ctas > max_resident)
        return fail(KPX_E_LIMIT, "teams of %d CTAs x %d exceed the %d co-resident CTAs of this device", team_ctas,
                    n_teams, max_resident);
    b.n_teams = n_teams; b.team_ctas = team_ctas;

    const int n = prob->n, nu = prob->nu;
    const size_t cp = (size_t)b.cap_pad, R = (size_t)b.regions, pairs = R * (size_t)b.subs;
    Carver c;
    struct Off { size_t states, control, dt, parent, region, tag, n_valid, n_invalid, cov, score, claim, bits, dregions, it_end,
                        it_code, it_rank, it_parent, it_bin, order, pos_of, bin_cursor, e_local, cnt_e, cnt_k, est_ids, leaf_sum, bar, ctl, trace, ch_start, ch_ctrl,
                        ch_dt, ch_slot, ch_end, packet; } o;
    const size_t row_n = (size_t)row_elems(n, (int)b.rs), row_nu = (size_t)row_elems(nu, (int)b.rs);   // padded rows
    o.states = c.take(b.rs * row_n * cp); o.control = c.take(b.rs * row_nu * cp); o.dt = c.take(b.rs * cp);
    o.parent = c.take(4 * cp); o.region = c.take(4 * cp); o.tag = c.take(cp);
    o.n_valid = c.take(4 * R); o.n_invalid = c.take(4 * R); o.cov = c.take(4 * R);
    o.score = c.take(8 * R); o.claim = c.take(4 * (pairs + 4));
    b.claim_shift = 1;
    while ((1ll << b.claim_shift) <= (long long)b.cap) ++b.claim_shift;      // 2^shift > t_e >= item index + 1
    o.bits = c.take(4 * ((R + 31) / 32 + 1));
    o.dregions = c.take(4 * ((R + 31) / 32 + 1));
    o.it_end = c.take(b.rs * row_n * cp); o.it_code = c.take(4 * cp); o.it_rank = c.take(4 * cp); o.it_parent = c.take(4 * cp);
    o.it_bin = c.take(cp); o.order = c.take(8 * cp); o.pos_of = c.take(4 * cp); o.bin_cursor = c.take(4 * (size_t)kBins);
    o.e_local = c.take(4 * cp); o.cnt_e = c.take(4 * (size_t)b.max_chunks); o.cnt_k = c.take(4 * (size_t)b.max_chunks);
    o.est_ids = c.take(4 * (R + 32)); o.leaf_sum = c.take(8 * (R / 64 + 2)); o.bar = c.take(256); o.ctl = c.take(sizeof(Ctl));
    o.trace = c.take(sizeof(kpx_trace) * (size_t)b.max_trace);
    o.ch_start = c.take(8 * (size_t)b.max_chain * n); o.ch_ctrl = c.take(8 * (size_t)b.max_chain * nu);
    o.ch_dt = c.take(8 * (size_t)b.max_chain); o.ch_slot = c.take(8 * (size_t)b.max_chain); o.ch_end = c.take(8 * n);
    o.packet = c.take(sizeof(ResultPacket));
    b.ws_bytes = align_up(c.off, 4096);
    if (cudaMalloc(&b.slab, b.ws_bytes * (size_t)n_teams) != cudaSuccess) {
        cudaGetLastError();
        return fail(KPX_E_CUDA, "cudaMalloc of %.1f MB for %d workspace(s) failed",
                    (double)b.ws_bytes * n_teams / 1e6, n_teams);
    }
    CU(cudaMemset(b.slab, 0, b.ws_bytes * (size_t)n_teams));
    b.ws_host.resize(n_teams);
    for (int t = 0; t < n_teams; ++t) {
        char* s = b.slab + (size_t)t * b.ws_bytes;
        Workspace& w = b.ws_host[t];
        w.states = s + o.states; w.control = s + o.control; w.dt = s + o.dt;
        w.parent = (int*)(s + o.parent); w.region = (int*)(s + o.region); w.tag = (uint8_t*)(s + o.tag);
        w.n_valid = (int*)(s + o.n_valid); w.n_invalid = (int*)(s + o.n_invalid); w.cov = (int*)(s + o.cov);
        w.score = (double*)(s + o.score); w.claim = (uint32_t*)(s + o.claim);
        w.avail_bits = (uint32_t*)(s + o.bits); w.touched_bits = (uint32_t*)(s + o.dregions);
        w.it_end = s + o.it_end; w.it_code = (uint32_t*)(s + o.it_code); w.it_rank = (int*)(s + o.it_rank);
        w.it_parent = (int*)(s + o.it_parent); w.e_local = (int*)(s + o.e_local);
        w.it_bin = (uint8_t*)(s + o.it_bin); w.order = (int2*)(s + o.order); w.pos_of = (int*)(s + o.pos_of); w.bin_cursor = (unsigned int*)(s + o.bin_cursor);
        w.cnt_expand = (int*)(s + o.cnt_e); w.cnt_keep = (int*)(s + o.cnt_k); w.est_ids = (int*)(s + o.est_ids); w.leaf_sum = (double*)(s + o.leaf_sum);
        w.bar = (unsigned int*)(s + o.bar); w.ctl = (Ctl*)(s + o.ctl); w.trace = (kpx_trace*)(s + o.trace);
        w.chain_start = (double*)(s + o.ch_start); w.chain_control = (double*)(s + o.ch_ctrl);
        w.chain_dt = (double*)(s + o.ch_dt); w.chain_slot = (long long*)(s + o.ch_slot);
        w.chain_end = (double*)(s + o.ch_end);
        w.packet = (ResultPacket*)(s + o.packet);
    }
    for (int t = 0; t < n_teams; ++t) {      // a fresh workspace is clean: no pair ever claimed, every epoch left
        CU(cudaMemset(b.ws_host[t].claim, 0xFF, 4 * pairs));
        CU(cudaMemset(b.ws_host[t].score, 0xFF, 8 * R));                     // all ones = NaN = "never estimated"
        Ctl c0;
        memset(&c0, 0, sizeof c0);
        c0.epoch_valid = 1;
        c0.epoch_used = (1u << (32 - b.claim_shift)) - 1u;                   // the first query takes e_max
        CU(cudaMemcpy(b.ws_host[t].ctl, &c0, sizeof c0, cudaMemcpyHostToDevice));
    }
    CU(cudaMalloc(&b.ws_dev, sizeof(Workspace) * (size_t)n_teams));
    CU(cudaMemcpy(b.ws_dev, b.ws_host.data(), sizeof(Workspace) * (size_t)n_teams, cudaMemcpyHostToDevice));
    b.obs_cap = prob->n_obs;
    b.n_scenes = 1; b.scene_obs = prob->n_obs; b.sc_min = b.obs_min; b.sc_max = b.obs_max;
    rc = upload_scenes(b);
    if (rc) return rc;
    CU(cudaMalloc(&b.queue_dev, 256));
    CU(cudaMemset(b.queue_dev, 0, 256));
    CU(cudaMalloc(&b.hand_dev, 64));
    CU(cudaMemset(b.hand_dev, 0, 64));
    CU(cudaMalloc(&b.susp_dev, sizeof(int2) * (size_t)kHandoffLevels * (size_t)n_teams));
    CU(cudaMallocHost(&b.pk_host, sizeof(ResultPacket)));
    CU(cudaMallocHost(&b.q_pinned, sizeof(QueryIn)));
    return KPX_OK;
}

int ensure_queries(kpx_batch& b, long long q) {
    if (q <= b.q_cap) return KPX_OK;
    cudaFree(b.q_dev); cudaFree(b.r_dev);
    b.q_dev = nullptr; b.r_dev = nullptr;
    CU(cudaMalloc(&b.q_dev, sizeof(QueryIn) * (size_t)q));
    CU(cudaMalloc(&b.r_dev, sizeof(kpx_query_result) * (size_t)q));
    b.q_cap = q;
    return KPX_OK;
}

int launch(kpx_batch& b, const PlanLaunch& L, cudaStream_t st) {
    cudaError_t e;
    if (b.prob.rng == KPX_RNG_PHILOX) e = b.precision == KPX_F64 ? launch_plan_f64p(L, st) : launch_plan_f32p(L, st);
    else e = b.precision == KPX_F64 ? launch_plan_f64(L, st) : launch_plan_f32(L, st);
    if (e != cudaSuccess) return fail(KPX_E_CUDA, "planner kernel launch: %s", cudaGetErrorString(e));
    ++b.launches;
    return KPX_OK;
}

PlanLaunch base_launch(kpx_batch& b) {
    PlanLaunch L{};
    L.prob = &b.prob; L.obs_dev = b.obs_dev; L.occ_dev = b.occ_dev; L.ws_dev = b.ws_dev; L.n_teams = b.n_teams; L.team_ctas = b.team_ctas;
    L.max_chunks = b.max_chunks; L.stride = b.cap_pad; L.claim_shift = b.claim_shift; L.max_trace = b.max_trace; L.max_chain = b.max_chain; L.smem = b.smem;
    L.cooperative = b.cooperative; L.latency = b.latency;
    return L;
}

template <class T>
int d2h(std::vector<T>& dst, const void* src, size_t count) {
    dst.resize(count);
    CU(cudaMemcpy(dst.data(), src, count * sizeof(T), cudaMemcpyDeviceToHost));
    return KPX_OK;
}

// node-major device rows (Row<R, N>, kpx_device.cuh) of `rows` x `dims` reals -> dense f64 host rows
int rows_to_host(const kpx_batch& b, const void* dev, int dims, long long rows, double* out, bool padded = true) {
    if (rows == 0) return KPX_OK;
    const size_t stride = padded ? (size_t)row_elems(dims, (int)b.rs) : (size_t)dims;
    std::vector<char> h((size_t)rows * stride * b.rs);
    CU(cudaMemcpy(h.data(), dev, h.size(), cudaMemcpyDeviceToHost));
    for (long long i = 0; i < rows; ++i)
        for (int d = 0; d < dims; ++d) {
            const size_t k = (size_t)i * stride + (size_t)d;
            out[i * dims + d] = b.rs == 8 ? ((const double*)h.data())[k] : (double)((const float*)h.data())[k];
        }
    return KPX_OK;
}

int rows_from_host(const kpx_batch& b, void* dev, int dims, long long rows, const double* in, bool padded = true) {
    if (rows == 0) return KPX_OK;
    const size_t stride = padded ? (size_t)row_elems(dims, (int)b.rs) : (size_t)dims;
    std::vector<char> h((size_t)rows * stride * b.rs, 0);
    for (long long i = 0; i < rows; ++i)
        for (int d = 0; d < dims; ++d) {
            const size_t k = (size_t)i * stride + (size_t)d;
            if (b.rs == 8) ((double*)h.data())[k] = in[i * dims + d];
            else ((float*)h.data())[k] = (float)in[i * dims + d];
        }
    CU(cudaMemcpy(dev, h.data(), h.size(), cudaMemcpyHostToDevice));
    return KPX_OK;
}

// NumPy's pairwise float64 sum (the order combine_leaves / estimate_leaves follow on the device)
double pairwise_total(const double* a, long long n) {
    if (n < 8) { double r = 0.0; for (long long i = 0; i < n; ++i) r += a[i]; return r; }
    if (n <= 128) {
        double r[8];
        long long i;
        for (i = 0; i < 8; ++i) r[i] = a[i];
        for (i = 8; i < n - (n % 8); i += 8) for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_total(a, n2) + pairwise_total(a + n2, n - n2);
}

int read_ctl(const kpx_batch& b, Ctl* out) {
    CU(cudaMemcpy(out, b.ws_host[0].ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    return KPX_OK;
}

}  // namespace

namespace {
template <class T>
__global__ void fma_peak_kernel(T* out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (T)(threadIdx.x + i) * (T)1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = x[i] * a + b;
        }
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == (T)123.456) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class T>
int measure_fma(int sms, double ms_target, double* tflops) {
    T* d = nullptr;
    const int blocks = sms * 8, threads = 256;
    CU(cudaMalloc(&d, sizeof(T) * (size_t)blocks * threads));
    EventPair ev;
    CU(ev.create());
    const cudaEvent_t e0 = ev.e0, e1 = ev.e1;
    int iters = 2000;
    double best = 0.0;
    for (int rep = 0; rep < 6; ++rep) {
        CU(cudaEventRecord(e0));
        fma_peak_kernel<T><<<blocks, threads>>>(d, iters, (T)1.000001, (T)1e-7);
        CU(cudaEventRecord(e1));
        CU(cudaEventSynchronize(e1));
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, e0, e1));
        const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
        if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
        if (ms < ms_target) iters = (int)std::min(2.0e6, iters * std::max(1.5, ms_target / std::max(ms, 1e-3f)));
    }
    cudaFree(d);
    *tflops = best;
    return KPX_OK;
}
}  // namespace

namespace {
// Solution chains leave the device packed: off[q] = rows of the solved queries before q (one block scans the
// chain lengths), then one block per query copies its rows.  A query's chain is chain_len rows of n + nu + 1
// doubles out of a max_chain-row slot, typically 6 of 64: the packed copy is a tenth of the dense one.
// a suspended query's workspace still holds the stop word that suspended it: cleared between the launches (inside
// the resumed kernel one CTA of a team could clear it after another has already read it)
__global__ void clear_stop_kernel(Workspace* ws, const int2* __restrict__ list, const unsigned int* __restrict__ n_list) {
    const unsigned int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < *n_list) ws[list[i].x].ctl->stop = 0;
}

__global__ void chain_offsets_kernel(int n_q, const kpx_query_result* __restrict__ res, long long* __restrict__ off) {
    __shared__ long long s_part[32];
    __shared__ long long s_carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < n_q; base += blockDim.x) {
        const int q = base + threadIdx.x;
        long long v = 0;
        if (q < n_q && res[q].status == KPX_SOLVED && res[q].chain_len > 0) v = res[q].chain_len;
        long long inc = v;
        for (int o = 1; o < 32; o <<= 1) { const long long t = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += t; }
        if (lane == 31) s_part[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            long long x = lane < nw ? s_part[lane] : 0, xi = x;
            for (int o = 1; o < 32; o <<= 1) { const long long t = __shfl_up_sync(0xffffffffu, xi, o); if (lane >= o) xi += t; }
            if (lane < nw) s_part[lane] = xi - x;
        }
        __syncthreads();
        const long long carry = s_carry;
        if (q < n_q) off[q] = carry + s_part[wid] + inc - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = carry + s_part[wid] + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) off[n_q] = s_carry;
}
__global__ void chain_pack_kernel(int n_q, const kpx_query_result* __restrict__ res, const long long* __restrict__ off,
                                  int max_chain, int n, int nu, const double* __restrict__ cs, const double* __restrict__ cc,
                                  const double* __restrict__ cd, double* __restrict__ ps, double* __restrict__ pc,
                                  double* __restrict__ pd) {
    const int q = blockIdx.x;
    if (q >= n_q) return;
    const long long rows = off[q + 1] - off[q], o = off[q];
    const size_t src = (size_t)q * max_chain;
    for (long long i = threadIdx.x; i < rows * n; i += blockDim.x) ps[o * n + i] = cs[src * n + i];
    for (long long i = threadIdx.x; i < rows * nu; i += blockDim.x) pc[o * nu + i] = cc[src * nu + i];
    for (long long i = threadIdx.x; i < rows; i += blockDim.x) pd[o + i] = cd[src + i];
}

__global__ void philox_kernel(Philox4 c, uint32_t k0, uint32_t k1, uint32_t* out) {
    const Philox4 r = philox4x32_10(c, k0, k1);
    out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}

// Goal of query q (BASELINE.json config 5): centre uniform in [lo, hi]^3 drawn from the GENERIC stream of
// seed q (rng.py:57-95: key(seed = q, 0, 0, 0, phase 5), draws 0, 1, 2, ...), three draws per try; a try is rejected
// if the centre is closer than min_dist to the start or inside an obstacle grown by `grow` on every side.  One thread
// per query, the same float64 operations in the same order as batch.goal_for_query (no FMA contraction).
__global__ void sample_goals_kernel(int n, const unsigned long long* __restrict__ ids, const double* __restrict__ obs /* [k][6] */,
                                    int n_obs, double sx, double sy, double sz, double lo, double hi, double radius,
                                    double min_dist, double grow, int max_tries, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t key = mix64(ids[i]);
    key = mix64(key ^ 0ull); key = mix64(key ^ 0ull); key = mix64(key ^ 0ull); key = mix64(key ^ 5ull);
    const double span = __dsub_rn(hi, lo);
    uint64_t idx = 0;
    double c[3] = {0.0, 0.0, 0.0};
    bool found = false;
    for (int t = 0; t < max_tries && !found; ++t) {
        for (int a = 0; a < 3; ++a) c[a] = __dadd_rn(lo, __dmul_rn(unit53(draw_u64(key, idx++)), span));
        const double d0 = __dsub_rn(c[0], sx), d1 = __dsub_rn(c[1], sy), d2 = __dsub_rn(c[2], sz);
        const double dist = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
        if (dist < min_dist) continue;
        bool inside = false;
        for (int k = 0; k < n_obs && !inside; ++k) {
            bool in = true;
            for (int a = 0; a < 3; ++a)
                in = in && c[a] >= __dsub_rn(obs[6 * k + a], grow) && c[a] <= __dadd_rn(obs[6 * k + 3 + a], grow);
            inside = in;
        }
        found = !inside;
    }
    out[4 * i + 0] = found ? c[0] : nan(""); out[4 * i + 1] = found ? c[1] : nan(""); out[4 * i + 2] = found ? c[2] : nan("");
    out[4 * i + 3] = radius;
}
}  // namespace

extern "C" {

int kpx_philox4x32(const uint32_t* counter4, const uint32_t* key2, uint32_t* out_host4, uint32_t* out_device4) {
    if (!counter4 || !key2) return fail(KPX_E_ARG, "null argument");
    const Philox4 c{counter4[0], counter4[1], counter4[2], counter4[3]};
    if (out_host4) {
        const Philox4 r = philox4x32_10(c, key2[0], key2[1]);
        out_host4[0] = r.x; out_host4[1] = r.y; out_host4[2] = r.z; out_host4[3] = r.w;
    }
    if (out_device4) {
        uint32_t* d = nullptr;
        CU(cudaMalloc(&d, 16));
        philox_kernel<<<1, 1>>>(c, key2[0], key2[1], d);
        cudaError_t e = cudaMemcpy(out_device4, d, 16, cudaMemcpyDeviceToHost);
        cudaFree(d);
        if (e != cudaSuccess) return fail(KPX_E_CUDA, "philox self-test: %s", cudaGetErrorString(e));
    }
    return KPX_OK;
}

int kpx_sample_goals(int64_t n_queries, const uint64_t* query_ids, int32_t n_obs, const double* obs_min,
                     const double* obs_max, const double* start3, double lo, double hi, double radius, double min_dist,
                     double margin, double* goals, void* stream) {
    if (n_queries < 0 || !query_ids || !start3 || !goals || n_obs < 0 || (n_obs && (!obs_min || !obs_max)))
        return fail(KPX_E_ARG, "bad goal-sampler arguments");
    if (n_queries == 0) return KPX_OK;
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<double> boxes(6 * (size_t)std::max(n_obs, 1), 0.0);
    for (int k = 0; k < n_obs; ++k)
        for (int a = 0; a < 3; ++a) { boxes[6 * k + a] = obs_min[3 * k + a]; boxes[6 * k + 3 + a] = obs_max[3 * k + a]; }
    char* dev = nullptr;
    const size_t o_ids = 0, o_box = align_up(8 * (size_t)n_queries, 256), o_out = o_box + align_up(8 * boxes.size(), 256);
    if (cudaMalloc(&dev, o_out + 32 * (size_t)n_queries) != cudaSuccess) { cudaGetLastError(); return fail(KPX_E_CUDA, "cudaMalloc failed"); }
    struct Free { char* p; ~Free() { cudaFree(p); } } guard{dev};
    CU(cudaMemcpyAsync(dev + o_ids, query_ids, 8 * (size_t)n_queries, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dev + o_box, boxes.data(), 8 * boxes.size(), cudaMemcpyHostToDevice, st));
    sample_goals_kernel<<<(unsigned)((n_queries + 127) / 128), 128, 0, st>>>(
        (int)n_queries, (const unsigned long long*)(dev + o_ids), (const double*)(dev + o_box), n_obs, start3[0], start3[1],
        start3[2], lo, hi, radius, min_dist, radius + margin, 1000, (double*)(dev + o_out));
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(goals, dev + o_out, 32 * (size_t)n_queries, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < n_queries; ++i)
        if (std::isnan(goals[4 * i])) return fail(KPX_E_STATE, "no admissible goal for query id %llu in 1000 tries", (unsigned long long)query_ids[i]);
    return KPX_OK;
}

int kpx_fma_peak(int device, double ms_target, double* tflops, double* tflops_f64) {
    cudaDeviceProp dp;
    CU(cudaGetDeviceProperties(&dp, device));
    CU(cudaSetDevice(device));
    int rc = KPX_OK;
    if (tflops && (rc = measure_fma<float>(dp.multiProcessorCount, ms_target, tflops))) return rc;
    if (tflops_f64 && (rc = measure_fma<double>(dp.multiProcessorCount, ms_target, tflops_f64))) return rc;
    return KPX_OK;
}

const char* kpx_last_error(void) { return g_err.c_str(); }
int kpx_version(void) { return 100; }
int kpx_struct_size(int which) {
    switch (which) {
        case 0: return (int)sizeof(kpx_problem);
        case 1: return (int)sizeof(kpx_stats);
        case 2: return (int)sizeof(kpx_trace);
        case 3: return (int)sizeof(kpx_query_result);
        default: return -1;
    }
}

int kpx_cull_thresholds(const kpx_problem* prob, int32_t precision, double* out4) {
    int rc = check_problem(prob);
    if (rc) return rc;
    if (!out4) return fail(KPX_E_ARG, "null output");
    double lo[3], inv[3];
    if (precision == KPX_F64) cull_constants_f64(*prob, out4, lo, inv); else cull_constants_f32(*prob, out4, lo, inv);
    return KPX_OK;
}

int kpx_cull_tables(const kpx_problem* prob, int32_t precision, uint32_t* masks, double* lo3, double* inv3) {
    int rc = check_problem(prob);
    if (rc) return rc;
    if (!masks || !lo3 || !inv3) return fail(KPX_E_ARG, "null output");
    double thr[4];
    if (precision == KPX_F64) {
        cull_constants_f64(*prob, thr, lo3, inv3);
        occupancy_masks_f64(*prob, std::min(prob->n_obs, 32), prob->obs_min, prob->obs_max, masks);
    } else {
        cull_constants_f32(*prob, thr, lo3, inv3);
        occupancy_masks_f32(*prob, std::min(prob->n_obs, 32), prob->obs_min, prob->obs_max, masks);
    }
    return KPX_OK;
}

int kpx_device_info(int device, int32_t* sm_count, int32_t* f32_blocks, int32_t* f64_blocks) {
    cudaDeviceProp dp;
    CU(cudaGetDeviceProperties(&dp, device));
    CU(cudaSetDevice(device));
    if (sm_count) *sm_count = dp.multiProcessorCount;
    if (f32_blocks) *f32_blocks = plan_blocks_per_sm_f32(KPX_MODEL_DI6, 6, 4096, false) * dp.multiProcessorCount;
    if (f64_blocks) *f64_blocks = plan_blocks_per_sm_f64(KPX_MODEL_DI6, 6, 4096, false) * dp.multiProcessorCount;
    return KPX_OK;
}

int kpx_propagate_batch(const kpx_problem* prob, const double* states, int64_t state_rows, const int64_t* e_slots,
                        int64_t m, int32_t lam, uint64_t seed, uint64_t iteration, int32_t precision,
                        uint8_t* o_valid, int64_t* o_region, int64_t* o_sub, double* o_end, double* o_control,
                        double* o_dt, double* o_accept, int64_t* o_substeps, int64_t* o_points, double* o_kernel_ms,
                        void* stream) {
    int rc = check_problem(prob);
    if (rc) return rc;
    if (m < 0 || lam < 1 || state_rows < 0) return fail(KPX_E_ARG, "bad batch shape");
    if (precision != KPX_F64 && precision != KPX_F32) return fail(KPX_E_ARG, "bad precision");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t items = m * lam;
    if (o_kernel_ms) *o_kernel_ms = 0.0;
    if (items == 0) return KPX_OK;
    for (int64_t i = 0; i < m; ++i)
        if (e_slots[i] < 0 || e_slots[i] >= state_rows) return fail(KPX_E_ARG, "e_slots[%lld] out of range", (long long)i);
    const int n = prob->n, nu = prob->nu;
    const size_t rs = precision == KPX_F64 ? 8 : 4;
    char* slab = nullptr;
    Carver c;
    const size_t o_states = c.take(8 * (size_t)state_rows * n), o_slots = c.take(8 * (size_t)m),
                 o_obs = c.take(8 * (size_t)std::max(prob->n_obs, 1) * rs),
                 o_occ = c.take(2 * sizeof(uint32_t) * (size_t)kOccCells), o_v = c.take((size_t)items),
                 o_r = c.take(8 * (size_t)items), o_s = c.take(8 * (size_t)items), o_e = c.take(8 * (size_t)items * n),
                 o_c = c.take(8 * (size_t)items * nu), o_d = c.take(8 * (size_t)items), o_a = c.take(8 * (size_t)items),
                 o_ss = c.take(8 * (size_t)items), o_pp = c.take(8 * (size_t)items);
    // device scratch of the seam call: one grow-only slab per device, kept between calls (the call itself stays
    // stateless for the caller: nothing in it survives but capacity); serialised by a mutex like the reference's GIL
    static std::mutex slab_mutex;
    static std::map<int, std::pair<char*, size_t>> slabs;
    std::lock_guard<std::mutex> lock(slab_mutex);
    int dev_id = 0;
    CU(cudaGetDevice(&dev_id));
    auto& cached = slabs[dev_id];
    if (cached.second < c.off) {
        if (cached.first) cudaFree(cached.first);
        cached = {nullptr, 0};
        const size_t want = c.off + c.off / 4;
        if (cudaMalloc(&cached.first, want) != cudaSuccess) { cudaGetLastError(); return fail(KPX_E_CUDA, "cudaMalloc failed"); }
        cached.second = want;
    }
    slab = cached.first;
    CU(cudaMemcpyAsync(slab + o_states, states, 8 * (size_t)state_rows * n, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(slab + o_slots, e_slots, 8 * (size_t)m, cudaMemcpyHostToDevice, st));
    rc = upload_obstacles(*prob, precision, prob->n_obs, prob->obs_min, prob->obs_max, slab + o_obs, (uint32_t*)(slab + o_occ), st);
    if (rc) return rc;
    BatchLaunch L{};
    L.prob = prob; L.obs_dev = slab + o_obs; L.occ_dev = (const uint32_t*)(slab + o_occ); L.states_dev = (const double*)(slab + o_states);
    L.e_slots_dev = (const long long*)(slab + o_slots); L.items = items; L.lam = lam; L.seed = seed;
    L.iteration = iteration; L.o_valid = (uint8_t*)(slab + o_v); L.o_region = (long long*)(slab + o_r);
    L.o_sub = (long long*)(slab + o_s); L.o_end = (double*)(slab + o_e); L.o_control = (double*)(slab + o_c);
    L.o_dt = (double*)(slab + o_d); L.o_accept = (double*)(slab + o_a);
    L.o_substeps = (long long*)(slab + o_ss); L.o_points = (long long*)(slab + o_pp);
    L.grid = (int)std::min<int64_t>((items + kBlock - 1) / kBlock, 148 * 16);
    L.smem = scene_smem_bytes(prob->n_obs, rs);
    EventPair ev;
    CU(ev.create());
    const cudaEvent_t e0 = ev.e0, e1 = ev.e1;
    CU(cudaEventRecord(e0, st));
    cudaError_t e;
    if (prob->rng == KPX_RNG_PHILOX) e = precision == KPX_F64 ? launch_batch_f64p(L, st) : launch_batch_f32p(L, st);
    else e = precision == KPX_F64 ? launch_batch_f64(L, st) : launch_batch_f32(L, st);
    if (e != cudaSuccess) return fail(e == cudaErrorInvalidValue ? KPX_E_ARG : KPX_E_CUDA,
                                      "propagate kernel launch (model_id=%d n=%d): %s", prob->model_id, n,
                                      cudaGetErrorString(e));
    CU(cudaEventRecord(e1, st));
    CU(cudaMemcpyAsync(o_valid, slab + o_v, (size_t)items, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(o_region, slab + o_r, 8 * (size_t)items, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(o_sub, slab + o_s, 8 * (size_t)items, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(o_end, slab + o_e, 8 * (size_t)items * n, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(o_control, slab + o_c, 8 * (size_t)items * nu, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(o_dt, slab + o_d, 8 * (size_t)items, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(o_accept, slab + o_a, 8 * (size_t)items, cudaMemcpyDeviceToHost, st));
    if (o_substeps) CU(cudaMemcpyAsync(o_substeps, slab + o_ss, 8 * (size_t)items, cudaMemcpyDeviceToHost, st));
    if (o_points) CU(cudaMemcpyAsync(o_points, slab + o_pp, 8 * (size_t)items, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (o_kernel_ms) { float ms = 0; CU(cudaEventElapsedTime(&ms, e0, e1)); *o_kernel_ms = ms; }
    return KPX_OK;
}

// ------------------------------------------------------------------ single plan
int kpx_plan_create(const kpx_problem* prob, int32_t precision, int32_t team_ctas, int32_t device, kpx_plan** out) {
    if (!out) return fail(KPX_E_ARG, "out is null");
    *out = nullptr;
    kpx_plan* p = new kpx_plan();
    int rc = init_batch(p->b, prob, precision, 1, team_ctas, KPX_MAX_CHAIN, device);
    if (rc) { destroy_batch(p->b); delete p; return rc; }
    rc = ensure_queries(p->b, 1);
    if (rc) { destroy_batch(p->b); delete p; return rc; }
    *out = p;
    return KPX_OK;
}

void kpx_plan_destroy(kpx_plan* p) {
    if (!p) return;
    destroy_batch(p->b);
    delete p;
}

int kpx_plan_reset(kpx_plan* p, uint64_t seed, const double* start, const double* goal4) {
    if (!p || !start || !goal4) return fail(KPX_E_ARG, "null argument");
    kpx_batch& b = p->b;
    memset(&b.q_host, 0, sizeof b.q_host);
    b.q_host.seed = seed;
    memcpy(b.q_host.start, start, sizeof(double) * b.prob.n);
    memcpy(b.q_host.goal, goal4, sizeof(double) * 4);
    b.fresh = true; b.loaded = false; b.pk_valid = false;
    return KPX_OK;
}

int kpx_plan_set_epoch(kpx_plan* p, uint32_t epoch_used) {
    if (!p) return fail(KPX_E_ARG, "null plan");
    kpx_batch& b = p->b;
    CU(cudaSetDevice(b.device));
    Ctl c;
    int rc = read_ctl(b, &c);
    if (rc) return rc;
    c.epoch_used = epoch_used;
    CU(cudaMemcpy(b.ws_host[0].ctl, &c, sizeof c, cudaMemcpyHostToDevice));
    return KPX_OK;
}

int kpx_plan_set_obstacles(kpx_plan* p, int32_t n_obs, const double* omin, const double* omax) {
    if (!p) return fail(KPX_E_ARG, "null plan");
    kpx_batch& b = p->b;
    if (n_obs < 0 || (n_obs && (!omin || !omax))) return fail(KPX_E_ARG, "bad obstacle arguments");
    if (n_obs > b.obs_cap)
        return fail(KPX_E_ARG, "obstacle count %d exceeds the capacity (%d) the plan was created with", n_obs, b.obs_cap);
    CU(cudaSetDevice(b.device));
    b.n_scenes = 1; b.scene_obs = n_obs;
    b.sc_min.assign(omin, omin + 3 * (size_t)n_obs);
    b.sc_max.assign(omax, omax + 3 * (size_t)n_obs);
    return upload_scenes(b);
}

int kpx_batch_set_scenes(kpx_batch* bp, int32_t n_scenes, const int32_t* n_obs, const double* omin, const double* omax) {
    if (!bp || n_scenes < 1 || !n_obs) return fail(KPX_E_ARG, "bad scene arguments");
    kpx_batch& b = *bp;
    int k = 0;
    size_t total = 0;
    for (int sc = 0; sc < n_scenes; ++sc) {
        if (n_obs[sc] < 0) return fail(KPX_E_ARG, "scene %d: negative obstacle count", sc);
        if (n_obs[sc] > b.obs_cap)
            return fail(KPX_E_ARG, "scene %d has %d obstacles, the batch was created with room for %d", sc, n_obs[sc], b.obs_cap);
        k = std::max(k, (int)n_obs[sc]);
        total += (size_t)n_obs[sc];
    }
    if (total && (!omin || !omax)) return fail(KPX_E_ARG, "null obstacle arrays");
    CU(cudaSetDevice(b.device));
    // pad every set to k boxes with boxes that lie outside the state box and are empty (min > max): no cell of the
    // occupancy grid gets their bit and no point or box can overlap them
    b.sc_min.assign(3 * (size_t)k * n_scenes, 0.0);
    b.sc_max.assign(3 * (size_t)k * n_scenes, 0.0);
    size_t src = 0;
    for (int sc = 0; sc < n_scenes; ++sc)
        for (int j = 0; j < k; ++j)
            for (int a = 0; a < 3; ++a) {
                const size_t dst = 3 * ((size_t)sc * k + j) + a;
                if (j < n_obs[sc]) { b.sc_min[dst] = omin[3 * (src + j) + a]; b.sc_max[dst] = omax[3 * (src + j) + a]; }
                else { b.sc_min[dst] = b.prob.state_hi[a] + 1.0; b.sc_max[dst] = b.prob.state_lo[a] - 1.0; }
                if (a == 2 && j + 1 == k) src += (size_t)n_obs[sc];
            }
    b.n_scenes = n_scenes; b.scene_obs = k;
    return upload_scenes(b);
}

int kpx_plan_run(kpx_plan* p, double t_max, int32_t max_iters, int32_t lam_override, uint32_t* stop_flag,
                 uint32_t* const* peer_flags, int32_t n_peers, kpx_stats* out, void* stream) {
    if (!p || !out) return fail(KPX_E_ARG, "null argument");
    kpx_batch& b = p->b;
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(b.device));
    if (!b.fresh && !b.loaded && b.launches == 0) return fail(KPX_E_STATE, "kpx_plan_reset or kpx_plan_load first");
    PlanLaunch L = base_launch(b);
    L.n_queries = 1; L.queries_dev = b.q_dev; L.results_dev = nullptr; L.queue_dev = nullptr;
    L.resume = b.fresh ? 0 : 1;
    L.max_iters = max_iters; L.lam_override = lam_override; L.t_max_s = t_max; L.stop_flag = stop_flag;
    if (n_peers > 0) {
        if (n_peers > b.peers_cap) {
            cudaFree(b.peers_dev);
            CU(cudaMalloc(&b.peers_dev, sizeof(uint32_t*) * (size_t)n_peers));
            b.peers_cap = n_peers;
        }
        CU(cudaMemcpyAsync(b.peers_dev, peer_flags, sizeof(uint32_t*) * (size_t)n_peers, cudaMemcpyHostToDevice, st));
        L.peer_flags = b.peers_dev; L.n_peers = n_peers;
    }
    const unsigned long long l0 = b.launches;
    if (!b.fresh)   // a continued run starts with a clear stop word (its status word says why the last launch ended)
        CU(cudaMemsetAsync((char*)b.ws_host[0].ctl + offsetof(Ctl, stop), 0, sizeof(int), st));
    if (b.fresh) {
        *b.q_pinned = b.q_host;
        CU(cudaMemcpyAsync(b.q_dev, b.q_pinned, sizeof(QueryIn), cudaMemcpyHostToDevice, st));
    }
    int rc = launch(b, L, st);
    if (rc) return rc;
    b.fresh = false;
    b.pk_valid = false;
    CU(cudaMemcpyAsync(b.pk_host, b.ws_host[0].packet, sizeof(ResultPacket), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    b.pk_valid = true;
    const Ctl& c = b.pk_host->ctl;
    out->status = c.status; out->iterations = c.iteration; out->tree_size = c.size;
    out->solution_slot = c.solution_slot; out->chain_len = c.chain_len;
    out->device_ms = (double)c.elapsed_ns * 1e-6;      // run clock: summed over the launches since the reset
    out->reset_ms = (double)(c.t_reset_done - c.t_begin) * 1e-6;
    out->items = c.sum_items; out->substeps = c.sum_substeps; out->points = c.sum_points;
    out->boxsteps = c.sum_boxsteps; out->free_items = c.sum_free; out->capacity = c.cap;
    out->launches = b.launches - l0;
    return KPX_OK;
}

int kpx_plan_snapshot(kpx_plan* p, int64_t rows, double* states, int64_t* parent, double* control, double* dt,
                      uint8_t* tag, int64_t* region) {
    if (!p) return fail(KPX_E_ARG, "null plan");
    kpx_batch& b = p->b;
    CU(cudaSetDevice(b.device));
    Ctl c;
    int rc = read_ctl(b, &c);
    if (rc) return rc;
    if (rows > c.size) return fail(KPX_E_ARG, "rows exceeds tree size %d", c.size);
    const Workspace& w = b.ws_host[0];
    if (states && (rc = rows_to_host(b, w.states, b.prob.n, rows, states))) return rc;
    if (control && (rc = rows_to_host(b, w.control, b.prob.nu, rows, control))) return rc;
    if (dt && (rc = rows_to_host(b, w.dt, 1, rows, dt, false))) return rc;      // one real per node, dense
    std::vector<int> tmp;
    if (parent) { if ((rc = d2h(tmp, w.parent, (size_t)rows))) return rc; for (int64_t i = 0; i < rows; ++i) parent[i] = tmp[i]; }
    if (region) { if ((rc = d2h(tmp, w.region, (size_t)rows))) return rc; for (int64_t i = 0; i < rows; ++i) region[i] = tmp[i]; }
    if (tag && rows) CU(cudaMemcpy(tag, w.tag, (size_t)rows, cudaMemcpyDeviceToHost));
    return KPX_OK;
}

int kpx_plan_regions(kpx_plan* p, int64_t* n_valid, int64_t* n_invalid, int64_t* cov, double* free_vol, double* score,
                     double* p_accept, uint8_t* visited, uint8_t* avail) {
    if (!p) return fail(KPX_E_ARG, "null plan");
    kpx_batch& b = p->b;
    CU(cudaSetDevice(b.device));
    Ctl c;
    int rc = read_ctl(b, &c);
    if (rc) return rc;
    const Workspace& w = b.ws_host[0];
    const size_t R = (size_t)b.regions;
    std::vector<int> nv, ni, cv;
    std::vector<uint32_t> av;
    std::vector<double> sc;
    if ((rc = d2h(nv, w.n_valid, R)) || (rc = d2h(ni, w.n_invalid, R)) || (rc = d2h(cv, w.cov, R)) ||
        (rc = d2h(av, w.avail_bits, (R + 31) / 32)) || (rc = d2h(sc, w.score, R))) return rc;
    const double vol = b.prob.grid_width[0] * b.prob.grid_width[1] * b.prob.grid_width[2];
    const double eps = b.prob.epsilon, delta = b.prob.delta, total = c.total_prev;
    for (size_t r = 0; r < R; ++r) {
        const bool is_avail = (av[r >> 5] >> (r & 31)) & 1u;
        const bool est = is_avail && sc[r] >= 0.0;            // covered by an estimate pass
        if (n_valid) n_valid[r] = nv[r];
        if (n_invalid) n_invalid[r] = ni[r];
        if (cov) cov[r] = cv[r];
        if (avail) avail[r] = is_avail;
        if (score) score[r] = est ? sc[r] : 0.0;
        if (free_vol) free_vol[r] = est ? (delta + nv[r]) * vol / (delta + nv[r] + ni[r]) : 0.0;
        if (p_accept) {
            double pa = 1.0;
            if (est) pa = total <= 0.0 ? std::min(1.0, eps) : std::min(1.0, sc[r] / total + eps);
            p_accept[r] = pa;
        }
    }
    if (visited) {
        std::vector<uint32_t> cl;
        if ((rc = d2h(cl, w.claim, R * (size_t)b.subs))) return rc;
        Ctl c;
        if ((rc = read_ctl(b, &c))) return rc;
        const uint32_t tag = c.epoch_used << b.claim_shift;                   // "visited" of the current query's epoch
        for (size_t i = 0; i < cl.size(); ++i) visited[i] = cl[i] == tag;
    }
    return KPX_OK;
}

int kpx_plan_solution(kpx_plan* p, int64_t max_segments, double* seg_start, double* seg_control, double* seg_dt,
                      int64_t* seg_slot, double* end_state) {
    if (!p) return fail(KPX_E_ARG, "null plan");
    kpx_batch& b = p->b;
    CU(cudaSetDevice(b.device));
    Ctl c;
    int rc = KPX_OK;
    if (b.pk_valid) c = b.pk_host->ctl;                  // the result packet of the last run is on the host
    else if ((rc = read_ctl(b, &c))) return rc;
    if (c.status != KPX_SOLVED) return fail(KPX_E_STATE, "plan is not solved");
    if (c.chain_len < 0) return fail(KPX_E_LIMIT, "solution chain longer than KPX_MAX_CHAIN");
    if (c.chain_len > max_segments) return fail(KPX_E_ARG, "need room for %d segments", c.chain_len);
    const Workspace& w = b.ws_host[0];
    const size_t L = (size_t)c.chain_len;
    if (L && b.pk_valid && L <= (size_t)kPacketSegs) {       // already on the host: no further copies
        const ResultPacket& pk = *b.pk_host;
        for (size_t i = 0; i < L; ++i) {
            if (seg_start) memcpy(seg_start + i * b.prob.n, pk.seg_start[i], 8 * (size_t)b.prob.n);
            if (seg_control) memcpy(seg_control + i * b.prob.nu, pk.seg_control[i], 8 * (size_t)b.prob.nu);
            if (seg_dt) seg_dt[i] = pk.seg_dt[i];
            if (seg_slot) seg_slot[i] = pk.seg_slot[i];
        }
        if (end_state) memcpy(end_state, pk.end_state, 8 * (size_t)b.prob.n);
        return KPX_OK;
    }
    if (L) {
        if (seg_start) CU(cudaMemcpy(seg_start, w.chain_start, 8 * L * b.prob.n, cudaMemcpyDeviceToHost));
        if (seg_control) CU(cudaMemcpy(seg_control, w.chain_control, 8 * L * b.prob.nu, cudaMemcpyDeviceToHost));
        if (seg_dt) CU(cudaMemcpy(seg_dt, w.chain_dt, 8 * L, cudaMemcpyDeviceToHost));
        if (seg_slot) CU(cudaMemcpy(seg_slot, w.chain_slot, 8 * L, cudaMemcpyDeviceToHost));
        if (end_state) CU(cudaMemcpy(end_state, w.chain_end, 8 * (size_t)b.prob.n, cudaMemcpyDeviceToHost));
    }
    return KPX_OK;
}

int kpx_plan_trace(kpx_plan* p, int32_t max_records, kpx_trace* out, int32_t* n_records) {
    if (!p || !n_records) return fail(KPX_E_ARG, "null argument");
    kpx_batch& b = p->b;
    CU(cudaSetDevice(b.device));
    Ctl c;
    int rc = read_ctl(b, &c);
    if (rc) return rc;
    const int n = std::min(c.n_trace, max_records);
    if (n > 0 && out) CU(cudaMemcpy(out, b.ws_host[0].trace, sizeof(kpx_trace) * (size_t)n, cudaMemcpyDeviceToHost));
    *n_records = n;
    return KPX_OK;
}

int kpx_plan_items(kpx_plan* p, int64_t max_items, int64_t* n_items, uint8_t* valid, int64_t* region, int64_t* sub,
                   double* end, uint8_t* keep, int64_t* parent_slot, uint8_t* goal_hit) {
    if (!p || !n_items) return fail(KPX_E_ARG, "null argument");
    kpx_batch& b = p->b;
    CU(cudaSetDevice(b.device));
    Ctl c;
    int rc = read_ctl(b, &c);
    if (rc) return rc;
    const int64_t I = c.n_items_last;
    *n_items = I;
    if (I > max_items) return fail(KPX_E_ARG, "need room for %lld items", (long long)I);
    if (I == 0) return KPX_OK;
    const Workspace& w = b.ws_host[0];
    std::vector<uint32_t> code;
    std::vector<int> rank, par;
    if ((rc = d2h(code, w.it_code, (size_t)I)) || (rc = d2h(rank, w.it_rank, (size_t)I)) ||
        (rc = d2h(par, w.it_parent, (size_t)I))) return rc;
    std::vector<double> e;
    if (end) { e.resize((size_t)I * b.prob.n); if ((rc = rows_to_host(b, w.it_end, b.prob.n, I, e.data()))) return rc; }
    std::vector<int> pos;      // sorted iterations keep per-item results at the item's sorted position
    if (c.last_sorted && (rc = d2h(pos, w.pos_of, (size_t)I))) return rc;
    for (int64_t i = 0; i < I; ++i) {
        const int64_t ip = c.last_sorted ? pos[i] : i;
        const bool v = !(code[ip] & kItemDeadBit);
        const uint32_t pair = code[ip] & ~kItemGoalBit;
        if (valid) valid[i] = v;
        if (region) region[i] = v ? (int64_t)(pair / (uint32_t)b.subs)
                                  : (code[ip] == kItemInvalid ? -1 : (int64_t)(code[ip] & (kItemDeadBit - 1u)));
        if (sub) sub[i] = v ? (int64_t)(pair % (uint32_t)b.subs) : 0;
        if (keep) keep[i] = v && rank[i] >= 0;
        if (goal_hit) goal_hit[i] = v && (code[ip] & kItemGoalBit) != 0;
        if (parent_slot) parent_slot[i] = par[i];
        if (end) for (int d = 0; d < b.prob.n; ++d) end[i * b.prob.n + d] = v ? e[(size_t)ip * b.prob.n + d] : 0.0;
    }
    return KPX_OK;
}

int kpx_plan_load(kpx_plan* p, uint64_t seed, const double* goal4, int32_t iteration, int64_t rows, const double* states,
                  const int64_t* parent, const double* control, const double* dt, const uint8_t* tag,
                  const int64_t* region, const int64_t* n_valid, const int64_t* n_invalid, const int64_t* cov,
                  const double* score, const double* p_accept, const uint8_t* visited, const uint8_t* avail) {
    if (!p || !goal4 || !states || !parent || !control || !dt || !tag || !region || !n_valid || !n_invalid || !cov ||
        !score || !p_accept || !visited || !avail) return fail(KPX_E_ARG, "null argument");
    kpx_batch& b = p->b;
    if (rows < 1 || rows > b.cap) return fail(KPX_E_ARG, "rows out of range");
    CU(cudaSetDevice(b.device));
    const Workspace& w = b.ws_host[0];
    int rc;
    if ((rc = rows_from_host(b, w.states, b.prob.n, rows, states)) || (rc = rows_from_host(b, w.control, b.prob.nu, rows, control)) ||
        (rc = rows_from_host(b, w.dt, 1, rows, dt, false))) return rc;
    std::vector<int> tmp((size_t)rows);
    for (int64_t i = 0; i < rows; ++i) tmp[i] = (int)parent[i];
    CU(cudaMemcpy(w.parent, tmp.data(), 4 * (size_t)rows, cudaMemcpyHostToDevice));
    for (int64_t i = 0; i < rows; ++i) tmp[i] = (int)region[i];
    CU(cudaMemcpy(w.region, tmp.data(), 4 * (size_t)rows, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(w.tag, tag, (size_t)rows, cudaMemcpyHostToDevice));
    const size_t R = (size_t)b.regions;
    std::vector<int> x(R);
    std::vector<double> sc_dev(R);
    std::vector<double> est_scores;
    for (size_t r = 0; r < R; ++r) {
        // score > 0 <=> the region has been through an estimate pass; regions made available by the
        // most recent append are estimated from the next iteration on (planner.py:246)
        const bool est = avail[r] && score[r] > 0.0;
        sc_dev[r] = est ? score[r] : -1.0;
        if (est) est_scores.push_back(score[r]);
    }
    const double total = pairwise_total(est_scores.data(), (long long)est_scores.size());   // as the device sums it
    {
        std::vector<uint32_t> bits((R + 31) / 32 + 1, 0u);
        for (size_t r = 0; r < R; ++r) if (avail[r]) bits[r >> 5] |= 1u << (r & 31);
        CU(cudaMemcpy(w.avail_bits, bits.data(), 4 * bits.size(), cudaMemcpyHostToDevice));
    }
    for (size_t r = 0; r < R; ++r) x[r] = (int)n_valid[r];
    CU(cudaMemcpy(w.n_valid, x.data(), 4 * R, cudaMemcpyHostToDevice));
    for (size_t r = 0; r < R; ++r) x[r] = (int)n_invalid[r];
    CU(cudaMemcpy(w.n_invalid, x.data(), 4 * R, cudaMemcpyHostToDevice));
    for (size_t r = 0; r < R; ++r) x[r] = (int)cov[r];
    CU(cudaMemcpy(w.cov, x.data(), 4 * R, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(w.score, sc_dev.data(), 8 * R, cudaMemcpyHostToDevice));
    std::vector<uint32_t> cl(R * (size_t)b.subs);
    const uint32_t load_epoch = (1u << (32 - b.claim_shift)) - 2u;           // e_max
    for (size_t i = 0; i < cl.size(); ++i) cl[i] = visited[i] ? load_epoch << b.claim_shift : kUnclaimed;
    CU(cudaMemcpy(w.claim, cl.data(), 4 * cl.size(), cudaMemcpyHostToDevice));
    // EXPAND lists per chunk
    std::vector<int> e_local((size_t)b.cap_pad, 0), cnt((size_t)b.max_chunks, 0);
    int ve = 0;
    for (int64_t s = 0; s < rows; ++s)
        if (tag[s] == KPX_TAG_EXPAND) { const int c = (int)(s / kChunk); e_local[(size_t)c * kChunk + cnt[c]++] = (int)s; ++ve; }
    CU(cudaMemcpy(w.e_local, e_local.data(), 4 * e_local.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(w.cnt_expand, cnt.data(), 4 * cnt.size(), cudaMemcpyHostToDevice));
    Ctl c;
    memset(&c, 0, sizeof c);
    c.size = (int)rows; c.iteration = iteration; c.status = KPX_RUNNING; c.solution_slot = -1; c.total_prev = total;
    c.ve = ve; c.first_hit_w = 0x7fffffff; c.rescue_slot = 0x7fffffff;
    c.cap = (int)(b.prob.t_e_start > 0 ? std::max<int64_t>(b.prob.t_e_start, rows) : b.prob.t_e);
    c.epoch_used = load_epoch; c.epoch_valid = 0;      // resumed with this epoch; the next reset is dense
    CU(cudaMemcpy(w.ctl, &c, sizeof c, cudaMemcpyHostToDevice));
    // t_reset_done stays 0: the first resumed launch stamps the start of the run clock itself
    memset(&b.q_host, 0, sizeof b.q_host);
    b.q_host.seed = seed;
    memcpy(b.q_host.goal, goal4, 4 * sizeof(double));
    CU(cudaMemcpy(b.q_dev, &b.q_host, sizeof(QueryIn), cudaMemcpyHostToDevice));
    b.loaded = true; b.fresh = false; b.pk_valid = false;
    return KPX_OK;
}

// ------------------------------------------------------------------ host-side trajectory rebuild
namespace {
double wrap_pi(double a) {
    const double PI = 3.14159265358979323846;
    double t = fmod(a + PI, 2.0 * PI);
    if (t <= 0.0) t += 2.0 * PI;
    return t - PI;
}
// vector fields in float64 with the reference's expression shapes (dynamics.py:105-159)
void host_deriv(int model_id, int n, const double* x, const double* u, double* o) {
    if (model_id == KPX_MODEL_DI6 || model_id == KPX_MODEL_STACKED_DI) {
        for (int b = 0; b < n / 6; ++b)
            for (int a = 0; a < 3; ++a) { o[6 * b + a] = x[6 * b + 3 + a]; o[6 * b + 3 + a] = u[3 * b + a]; }
    } else if (model_id == KPX_MODEL_DUBINS6) {
        const double v = x[3], ct = cos(x[4]), st = sin(x[4]), cg = cos(x[5]), sg = sin(x[5]);
        o[0] = v * ct * cg; o[1] = v * st * cg; o[2] = v * sg; o[3] = u[0]; o[4] = u[1]; o[5] = u[2];
    } else {
        const double cphi = cos(x[6]), sphi = sin(x[6]), cth = cos(x[7]), sth = sin(x[7]), cpsi = cos(x[8]), spsi = sin(x[8]);
        const double p = x[9], q = x[10], r = x[11], acc = u[0] / 1.0;
        o[0] = x[3]; o[1] = x[4]; o[2] = x[5];
        o[3] = acc * (cphi * sth * cpsi + sphi * spsi);
        o[4] = acc * (cphi * sth * spsi - sphi * cpsi);
        o[5] = acc * (cphi * cth) - 9.81;
        const double sw = q * sphi + r * cphi;
        o[6] = p + sw * (sth / cth);
        o[7] = q * cphi - r * sphi;
        o[8] = sw / cth;
        o[9] = (u[1] - (0.02 - 0.01) * q * r) / 0.01;
        o[10] = (u[2] - (0.01 - 0.02) * p * r) / 0.01;
        o[11] = (u[3] - (0.01 - 0.01) * p * q) / 0.02;
    }
}
}  // namespace

int kpx_trajectory(int32_t model_id, int32_t n, int32_t nu, int64_t n_seg, const double* seg_start,
                   const double* seg_control, const double* seg_dt, int32_t chain_from_root, double* sampled,
                   int64_t max_rows, int64_t* seg_offset) {
    if (n > KPX_MAX_DIM || nu > KPX_MAX_CONTROL || n < 6 || !seg_start || !seg_control || !seg_dt || !sampled || !seg_offset)
        return fail(KPX_E_ARG, "bad trajectory arguments");
    if ((model_id == KPX_MODEL_DUBINS6 && n != 6) || (model_id == KPX_MODEL_QUAD12 && n != 12) || model_id < 0 ||
        model_id > KPX_MODEL_STACKED_DI) return fail(KPX_E_ARG, "bad model");
    int64_t row = 0;
    double cur[KPX_MAX_DIM], tmp[KPX_MAX_DIM], k1[KPX_MAX_DIM], k2[KPX_MAX_DIM], k3[KPX_MAX_DIM], k4[KPX_MAX_DIM];
    for (int64_t s = 0; s < n_seg; ++s) {
        const double dt = seg_dt[s];
        if (!(dt > 0.0)) return fail(KPX_E_ARG, "dt must be positive");
        int S = (int)ceil(dt / 0.02);                                  // dynamics.py:237-239
        if (S < 4) S = 4;
        if (row + S + 1 > max_rows) return fail(KPX_E_ARG, "sampled buffer too small");
        const double h = dt / S, hh = 0.5 * h, h6 = h / 6.0;
        const double* u = seg_control + s * nu;
        if (!(chain_from_root && s > 0)) memcpy(cur, seg_start + s * n, sizeof(double) * n);
        seg_offset[s] = row;
        memcpy(sampled + row * n, cur, sizeof(double) * n); ++row;
        for (int i = 0; i < S; ++i) {                                  // dynamics.py:270-282
            host_deriv(model_id, n, cur, u, k1);
            for (int d = 0; d < n; ++d) tmp[d] = cur[d] + hh * k1[d];
            host_deriv(model_id, n, tmp, u, k2);
            for (int d = 0; d < n; ++d) tmp[d] = cur[d] + hh * k2[d];
            host_deriv(model_id, n, tmp, u, k3);
            for (int d = 0; d < n; ++d) tmp[d] = cur[d] + h * k3[d];
            host_deriv(model_id, n, tmp, u, k4);
            for (int d = 0; d < n; ++d) cur[d] = cur[d] + h6 * (k1[d] + 2.0 * k2[d] + 2.0 * k3[d] + k4[d]);
            if (model_id == KPX_MODEL_DUBINS6) cur[4] = wrap_pi(cur[4]);
            else if (model_id == KPX_MODEL_QUAD12) { cur[6] = wrap_pi(cur[6]); cur[7] = wrap_pi(cur[7]); cur[8] = wrap_pi(cur[8]); }
            memcpy(sampled + row * n, cur, sizeof(double) * n); ++row;
        }
    }
    seg_offset[n_seg] = row;
    return KPX_OK;
}

// validity.py:58-106 + in_goal on a rebuilt trajectory (host, float64): every sampled state finite, inside
// the state box and outside every closed obstacle box; interpolants at the power-of-two densification of
// `res`; last state inside the closed goal ball.  *fail_code: 0 ok, 3 segment invalid, 4 goal missed.
int kpx_trajectory_valid(const kpx_problem* prob, int64_t n_seg, const double* sampled, const int64_t* seg_offset,
                         const double* goal4, double res, int32_t* ok, int32_t* fail_code) {
    if (!prob || !sampled || !seg_offset || !goal4 || !ok || !(res > 0.0)) return fail(KPX_E_ARG, "bad arguments");
    const int n = prob->n, k = prob->n_obs;
    auto state_ok = [&](const double* x) {
        for (int d = 0; d < n; ++d) if (!std::isfinite(x[d])) return false;
        for (int d = 0; d < n; ++d) if (x[d] < prob->state_lo[d] || x[d] > prob->state_hi[d]) return false;
        for (int j = 0; j < k; ++j) {
            const double *a = prob->obs_min + 3 * j, *b = prob->obs_max + 3 * j;
            if (x[0] >= a[0] && x[0] <= b[0] && x[1] >= a[1] && x[1] <= b[1] && x[2] >= a[2] && x[2] <= b[2]) return false;
        }
        return true;
    };
    *ok = 1;
    if (fail_code) *fail_code = 0;
    double st[KPX_MAX_DIM];
    for (int64_t s = 0; s < n_seg && *ok; ++s) {
        for (int64_t r = seg_offset[s]; r < seg_offset[s + 1] && *ok; ++r) {
            const double* b = sampled + r * n;
            if (!state_ok(b)) { *ok = 0; break; }
            if (r == seg_offset[s]) continue;
            const double* a = b - n;
            const double d0 = b[0] - a[0], d1 = b[1] - a[1], d2 = b[2] - a[2];
            const double dist = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            int64_t m = 1;
            while ((double)m * res < dist) m <<= 1;
            for (int64_t j = 1; j < m && *ok; ++j) {
                const double t = (double)j / (double)m;
                for (int d = 0; d < n; ++d) st[d] = a[d] + t * (b[d] - a[d]);
                if (!state_ok(st)) *ok = 0;
            }
        }
    }
    if (!*ok) { if (fail_code) *fail_code = 3; return KPX_OK; }
    if (n_seg > 0) {
        const double* e = sampled + (seg_offset[n_seg] - 1) * n;
        const double d0 = e[0] - goal4[0], d1 = e[1] - goal4[1], d2 = e[2] - goal4[2];
        if (!(sqrt(d0 * d0 + d1 * d1 + d2 * d2) <= goal4[3])) { *ok = 0; if (fail_code) *fail_code = 4; }
    }
    return KPX_OK;
}

int kpx_plan_trajectory(kpx_plan* p, const double* start, const double* goal4, double res, int64_t max_seg,
                        int64_t max_rows, double* seg_control, double* seg_dt, double* sampled, int64_t* seg_offset,
                        int64_t* n_seg, int32_t* ok, int32_t* fail_code) {
    if (!p || !seg_control || !seg_dt || !sampled || !seg_offset || !n_seg || !ok) return fail(KPX_E_ARG, "null argument");
    kpx_batch& b = p->b;
    const int n = b.prob.n, nu = b.prob.nu;
    int status, chain_len;
    if (b.pk_valid) { status = b.pk_host->ctl.status; chain_len = b.pk_host->ctl.chain_len; }
    else {
        CU(cudaSetDevice(b.device));
        Ctl c;
        int rc = read_ctl(b, &c);
        if (rc) return rc;
        status = c.status; chain_len = c.chain_len;
    }
    if (status != KPX_SOLVED) return fail(KPX_E_STATE, "plan is not solved");
    if (chain_len < 0) return fail(KPX_E_LIMIT, "solution chain longer than KPX_MAX_CHAIN");
    if (chain_len > max_seg) return fail(KPX_E_ARG, "need room for %d segments", chain_len);
    const int64_t L = chain_len;
    *n_seg = L; *ok = 1;
    if (fail_code) *fail_code = 0;
    seg_offset[0] = 0;
    if (L == 0) return KPX_OK;
    std::vector<double> seg_start((size_t)L * n);
    int rc = kpx_plan_solution(p, L, seg_start.data(), seg_control, seg_dt, nullptr, nullptr);
    if (rc) return rc;
    if (start) memcpy(seg_start.data(), start, sizeof(double) * n);
    rc = kpx_trajectory(b.prob.model_id, n, nu, L, seg_start.data(), seg_control, seg_dt, start ? 1 : 0, sampled, max_rows,
                        seg_offset);
    if (rc) return rc;
    if (start) {
        if (!goal4) return fail(KPX_E_ARG, "goal4 is needed to check a chain continued from the root");
        rc = kpx_trajectory_valid(&b.prob, L, sampled, seg_offset, goal4, res > 0.0 ? res : b.prob.check_res, ok, fail_code);
    }
    return rc;
}

// ------------------------------------------------------------------ batches
int kpx_batch_create(const kpx_problem* prob, int32_t precision, int32_t n_teams, int32_t team_ctas, int32_t max_chain,
                     int32_t device, kpx_batch** out) {
    if (!out) return fail(KPX_E_ARG, "out is null");
    *out = nullptr;
    if (team_ctas < 0) return fail(KPX_E_ARG, "team_ctas must be >= 0 for batches (0: as wide as n_teams leaves room for)");
    kpx_batch* b = new kpx_batch();
    b->auto_width = team_ctas == 0;
    int rc = init_batch(*b, prob, precision, n_teams, std::max(team_ctas, 1), max_chain > 0 ? max_chain : 64, device);
    if (rc) { destroy_batch(*b); delete b; return rc; }
    *out = b;
    return KPX_OK;
}

int kpx_batch_set_handoff(kpx_batch* b, int32_t enable) {
    if (!b) return fail(KPX_E_ARG, "null batch");
    b->handoff = enable != 0;
    return KPX_OK;
}

int kpx_batch_handoff_counts(kpx_batch* b, int32_t* counts) {
    if (!b || !counts) return fail(KPX_E_ARG, "null argument");
    unsigned int h[KPX_HANDOFF_STAGES];
    CU(cudaSetDevice(b->device));
    CU(cudaMemcpy(h, b->hand_dev + 8, sizeof h, cudaMemcpyDeviceToHost));
    for (int i = 0; i < KPX_HANDOFF_STAGES; ++i) counts[i] = (int32_t)h[i];
    return KPX_OK;
}

int kpx_batch_info(const kpx_batch* b, int32_t* n_teams, int32_t* team_ctas) {
    if (!b) return fail(KPX_E_ARG, "null batch");
    if (n_teams) *n_teams = b->n_teams;
    if (team_ctas) *team_ctas = b->team_ctas;
    return KPX_OK;
}

void kpx_batch_destroy(kpx_batch* b) {
    if (!b) return;
    destroy_batch(*b);
    delete b;
}

int kpx_batch_upload(kpx_batch* bp, int64_t n_queries, const uint64_t* seeds, const double* starts,
                     const double* goals, int32_t want_chains, void* stream) {
    return kpx_batch_upload_scenes(bp, n_queries, seeds, starts, goals, nullptr, want_chains, stream);
}

int kpx_batch_upload_scenes(kpx_batch* bp, int64_t n_queries, const uint64_t* seeds, const double* starts,
                            const double* goals, const int32_t* scene_idx, int32_t want_chains, void* stream) {
    if (!bp || !seeds || !starts || !goals) return fail(KPX_E_ARG, "null argument");
    if (n_queries < 1) return fail(KPX_E_ARG, "n_queries must be >= 1");
    kpx_batch& b = *bp;
    if (scene_idx)
        for (int64_t i = 0; i < n_queries; ++i)
            if (scene_idx[i] < 0 || scene_idx[i] >= b.n_scenes)
                return fail(KPX_E_ARG, "query %lld names scene %d, the batch holds %d", (long long)i, scene_idx[i], b.n_scenes);
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(b.device));
    int rc = ensure_queries(b, n_queries);
    if (rc) return rc;
    const int n = b.prob.n, nu = b.prob.nu;
    b.q_stage.resize((size_t)n_queries);
    for (int64_t i = 0; i < n_queries; ++i) {
        memset(&b.q_stage[i], 0, sizeof(QueryIn));
        b.q_stage[i].seed = seeds[i];
        memcpy(b.q_stage[i].start, starts + i * n, sizeof(double) * n);
        memcpy(b.q_stage[i].goal, goals + i * 4, sizeof(double) * 4);
        b.q_stage[i].scene = scene_idx ? scene_idx[i] : 0;
    }
    if (want_chains && (!b.bc_start || b.bc_cap < b.q_cap)) {
        cudaFree(b.bc_start); cudaFree(b.bc_ctrl); cudaFree(b.bc_dt);
        b.bc_start = b.bc_ctrl = b.bc_dt = nullptr;
        CU(cudaMalloc(&b.bc_start, 8 * (size_t)b.q_cap * b.max_chain * n));
        CU(cudaMalloc(&b.bc_ctrl, 8 * (size_t)b.q_cap * b.max_chain * nu));
        CU(cudaMalloc(&b.bc_dt, 8 * (size_t)b.q_cap * b.max_chain));
        cudaFree(b.bp_start); cudaFree(b.bp_ctrl); cudaFree(b.bp_dt); cudaFree(b.bp_off);
        b.bp_start = b.bp_ctrl = b.bp_dt = nullptr; b.bp_off = nullptr;
        CU(cudaMalloc(&b.bp_start, 8 * (size_t)b.q_cap * b.max_chain * n));
        CU(cudaMalloc(&b.bp_ctrl, 8 * (size_t)b.q_cap * b.max_chain * nu));
        CU(cudaMalloc(&b.bp_dt, 8 * (size_t)b.q_cap * b.max_chain));
        CU(cudaMalloc(&b.bp_off, 8 * ((size_t)b.q_cap + 1)));
        b.bc_cap = b.q_cap;
    }
    b.want_chains = want_chains != 0;
    b.n_uploaded = n_queries;
    CU(cudaMemcpyAsync(b.q_dev, b.q_stage.data(), sizeof(QueryIn) * (size_t)n_queries, cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
    return KPX_OK;
}

/* asynchronous: one persistent launch over the uploaded queries; no host synchronisation */
int kpx_batch_launch(kpx_batch* bp, double t_max, void* stream) {
    if (!bp) return fail(KPX_E_ARG, "null batch");
    kpx_batch& b = *bp;
    if (b.n_uploaded < 1) return fail(KPX_E_STATE, "kpx_batch_upload first");
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(b.device));
    CU(cudaMemsetAsync(b.queue_dev, 0, 4, st));
    PlanLaunch L = base_launch(b);
    L.n_queries = (int)b.n_uploaded; L.queries_dev = b.q_dev; L.results_dev = b.r_dev; L.queue_dev = b.queue_dev;
    L.resume = 0; L.max_iters = 0; L.lam_override = 0; L.t_max_s = t_max;
    if (b.want_chains) { L.b_chain_start = b.bc_start; L.b_chain_control = b.bc_ctrl; L.b_chain_dt = b.bc_dt; }
    // Hand-off: the launch ends when the queue is empty and only a few teams are still planning; those queries carry
    // on in the next launch on teams of 8 CTAs, the last of them on teams of 64 -- instead of one CTA each while the
    // rest of the device idles.  Results do not depend on the team size, so nothing else changes.  Everything is
    // stream-ordered: a stage that finds nothing suspended costs one empty launch.
    int levels = 0, keep[kHandoffLevels] = {}, width[kHandoffLevels] = {};
    if (b.handoff && !b.latency && b.n_uploaded >= 16)
        for (int i = 0; i < b.hand_levels; ++i) {          // the stages wider than the teams the batch starts with
            const int w = std::min(b.hand_width[i], b.max_resident);
            if (w > (levels ? width[levels - 1] : b.team_ctas)) {
                width[levels] = w;
                keep[levels] = b.max_resident / w;
                ++levels;
            }
        }
    if (levels) {
        CU(cudaMemsetAsync(b.hand_dev, 0, 64, st));
        L.idle = b.hand_dev; L.handoff_at = std::max(1, b.n_teams - keep[0]);
        L.susp_out = b.susp_dev; L.n_susp_out = b.hand_dev + 8;
    }
    int rc = launch(b, L, st);
    for (int s = 1; s <= levels && rc == KPX_OK; ++s) {
        const int2* list = b.susp_dev + (size_t)(s - 1) * (size_t)b.n_teams;
        const unsigned int* n_list = b.hand_dev + 8 + (s - 1);
        const int teams = std::min(keep[s - 1], b.n_teams);          // at most that many were suspended
        clear_stop_kernel<<<(teams + 255) / 256, 256, 0, st>>>(b.ws_dev, list, n_list);
        PlanLaunch H = L;
        H.queue_dev = nullptr; H.resume = 1; H.n_teams = teams; H.team_ctas = width[s - 1]; H.cooperative = true;
        H.resume_in = list; H.n_resume_in = n_list; H.idle = b.hand_dev + s;
        H.handoff_at = s < levels ? std::max(1, teams - keep[s]) : 0;
        H.pass_on_below = s < levels ? keep[s] : 0;
        H.susp_out = b.susp_dev + (size_t)s * (size_t)b.n_teams; H.n_susp_out = b.hand_dev + 8 + s;
        rc = launch(b, H, st);
    }
    return rc;
}

int kpx_batch_validate(kpx_batch* bp, double res, void* stream) {
    if (!bp) return fail(KPX_E_ARG, "null batch");
    kpx_batch& b = *bp;
    if (b.n_uploaded < 1) return fail(KPX_E_STATE, "kpx_batch_upload first");
    if (!b.want_chains || !b.bc_ctrl || !b.bc_dt) return fail(KPX_E_STATE, "validation needs want_chains = 1 at upload");
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(b.device));
    if (!b.boxes64_dev) {
        const size_t k = (size_t)b.scene_obs, tot = k * (size_t)b.n_scenes;
        std::vector<double> h(8 * std::max<size_t>(tot, 1), 0.0);
        for (size_t j = 0; j < tot; ++j)
            for (int a = 0; a < 3; ++a) { h[8 * j + a] = b.sc_min[3 * j + a]; h[8 * j + 4 + a] = b.sc_max[3 * j + a]; }
        CU(cudaMalloc(&b.boxes64_dev, h.size() * 8));
        CU(cudaMemcpy(b.boxes64_dev, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    }
    ValidateLaunch L{};
    L.prob = &b.prob; L.boxes_dev = b.boxes64_dev; L.queries_dev = b.q_dev; L.results_dev = b.r_dev;
    L.chain_control = b.bc_ctrl; L.chain_dt = b.bc_dt; L.n_queries = (int)b.n_uploaded; L.max_chain = b.max_chain;
    L.res = res > 0.0 ? res : b.prob.check_res;
    cudaError_t e = launch_validate_f64(L, st);
    if (e != cudaSuccess) return fail(KPX_E_CUDA, "validate kernel launch: %s", cudaGetErrorString(e));
    return KPX_OK;
}

int kpx_batch_download(kpx_batch* bp, kpx_query_result* results, double* chain_start, double* chain_control,
                       double* chain_dt, void* stream) {
    if (!bp || !results) return fail(KPX_E_ARG, "null argument");
    kpx_batch& b = *bp;
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(b.device));
    const size_t q = (size_t)b.n_uploaded;
    const int n = b.prob.n, nu = b.prob.nu;
    const bool chains = b.want_chains && chain_start && chain_control && chain_dt;
    if (chains) {       // pack on the device while the records travel
        chain_offsets_kernel<<<1, 1024, 0, st>>>((int)q, b.r_dev, b.bp_off);
        chain_pack_kernel<<<(unsigned)q, 64, 0, st>>>((int)q, b.r_dev, b.bp_off, b.max_chain, n, nu, b.bc_start, b.bc_ctrl,
                                                       b.bc_dt, b.bp_start, b.bp_ctrl, b.bp_dt);
        CU(cudaGetLastError());
    }
    CU(cudaMemcpyAsync(results, b.r_dev, sizeof(kpx_query_result) * q, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (chains) {
        // the caller's arrays keep the dense (Q, max_chain, .) layout; only the rows that exist cross the bus
        size_t rows = 0;
        for (size_t i = 0; i < q; ++i) if (results[i].status == KPX_SOLVED && results[i].chain_len > 0) rows += (size_t)results[i].chain_len;
        b.d2h_chain_bytes = 8 * rows * (size_t)(n + nu + 1);
        if (rows) {
            const size_t need = rows * (size_t)(n + nu + 1);
            if (need > b.bp_host_cap) {
                cudaFreeHost(b.bp_host); b.bp_host = nullptr; b.bp_host_cap = 0;
                CU(cudaMallocHost(&b.bp_host, 8 * (need + need / 4)));
                b.bp_host_cap = need + need / 4;
            }
            double *hs = b.bp_host, *hc = hs + rows * n, *hd = hc + rows * nu;
            CU(cudaMemcpyAsync(hs, b.bp_start, 8 * rows * n, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(hc, b.bp_ctrl, 8 * rows * nu, cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(hd, b.bp_dt, 8 * rows, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            size_t o = 0;
            for (size_t i = 0; i < q; ++i) {
                if (!(results[i].status == KPX_SOLVED && results[i].chain_len > 0)) continue;
                const size_t L = (size_t)results[i].chain_len, dst = i * (size_t)b.max_chain;
                memcpy(chain_start + dst * n, hs + o * n, 8 * L * n);
                memcpy(chain_control + dst * nu, hc + o * nu, 8 * L * nu);
                memcpy(chain_dt + dst, hd + o, 8 * L);
                o += L;
            }
        }
    }
    return KPX_OK;
}

int kpx_batch_run(kpx_batch* bp, int64_t n_queries, const uint64_t* seeds, const double* starts, const double* goals,
                  double t_max, kpx_query_result* results, double* chain_start, double* chain_control,
                  double* chain_dt, double* o_kernel_ms, void* stream) {
    if (!bp || !results) return fail(KPX_E_ARG, "null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int want = chain_start && chain_control && chain_dt;
    int rc = kpx_batch_upload(bp, n_queries, seeds, starts, goals, want, stream);
    if (rc) return rc;
    EventPair ev;
    CU(ev.create());
    const cudaEvent_t e0 = ev.e0, e1 = ev.e1;
    CU(cudaEventRecord(e0, st));
    rc = kpx_batch_launch(bp, t_max, stream);
    if (rc) return rc;
    if (want) { rc = kpx_batch_validate(bp, 0.0, stream); if (rc) return rc; }    // every solution is re-checked in float64
    CU(cudaEventRecord(e1, st));
    rc = kpx_batch_download(bp, results, chain_start, chain_control, chain_dt, stream);
    if (rc) return rc;
    if (o_kernel_ms) { float ms = 0; CU(cudaEventElapsedTime(&ms, e0, e1)); *o_kernel_ms = ms; }
    return KPX_OK;
}

}  // extern "C"
