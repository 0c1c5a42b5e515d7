// kpx_plan.cuh -- the device-resident Kino-PAX loop as ONE persistent kernel.
//
// A "team" of CTAs owns one planning query at a time: the whole grid for a
// single query (cooperative launch), or 1..k CTAs per query when many
// independent queries share the GPU.  Team members meet at a
// sense-reversing barrier in global memory; with one CTA per team it degrades
// to __syncthreads().  Per iteration (reference planner.py:283-303):
//
//   S0  order the items by RK4 substep count (known from the RNG draw alone) so that a warp's 32 items are
//       equally long: a global counting sort for many-CTA teams, tile by tile in shared memory and fused
//       with S1 for one-CTA teams; skipped when one round of the team's threads covers the iteration, and
//       absent for the float32 double integrators (nothing there is longer than anything else, see S1)
//   S1  propagate every (EXPAND slot x extension) item, count outcomes per region
//       (warp-aggregated atomics), claim fresh (region,sub) pairs with atomicMin on the epoch-tagged table.
//       float32 double integrators: every lane first settles its item from the closed form (certified valid or
//       invalid, ~90 %); the undecided rest goes to a list and is evaluated one item per warp, lane = substep
//   --- team barrier ---
//   S2  resolve first-visit winners (lowest item index), acceptance gate against
//       LAST iteration's p_accept, per-chunk keep counts + chunk-local ranks,
//       first goal hit (atomicMin over item index)
//   --- team barrier ---
//   S3  ordered append: slot = size + rank (capacity clamp, cut at first goal hit),
//       mark regions available from the NEXT iteration; estimate pass over the available regions: one warp
//       per leaf of NumPy's pairwise-sum tree computes the leaf's scores and their sum in NumPy's order
//   --- team barrier ---
//   S4  every CTA combines the leaf sums up the tree -> total (bit-identical to ndarray.sum, for any team size);
//       p_accept on the fly from (score, total); demote / promote every live slot
//       from its keyed uniforms; per-chunk compaction of the next EXPAND set
//   --- team barrier ---
//       list of available regions for the next estimate pass; scan chunk counts -> |V_E|; rescue rule;
//       termination (goal, capacity -- adaptive capacity grows it in place --, run clock, stop word)
//
// Ordering rules (ascending slot order of V_E, item w = i*lambda + ext, append in
// item order) are kept by construction: compaction is chunk-ordered and ranks are
// chunk prefix + in-chunk rank, so the tree is identical for any team size.
//
// Code structure: run_query = reset_query, then iteration_head / s1_propagate / iteration_tail until the run
// ends, then finish_query.  The phases exchange the CTA-uniform run state through RunState in shared memory
// and re-derive their locals, so nothing but the integrator's own registers is live across S1; everything is
// __forceinline__ (an out-of-line call anywhere on the propagation path costs ~30 % of the throughput).
#pragma once
#include "kpx_device.cuh"

// Resident CTAs per SM the float32 kernels are compiled for (register budget = 65536 / (256 * n)), per use:
// THROUGHPUT (many queries, one CTA each) wants warps to hide latency; LATENCY (one query on the whole GPU)
// wants fewer, fatter CTAs: fewer barrier participants and no spills.  Measured on B200.
#ifndef KPX_MINB_F32_DI
#define KPX_MINB_F32_DI 4        // double integrators (6-D blocks), throughput
#endif
#ifndef KPX_MINS_F32_DI
#define KPX_MINS_F32_DI 2        // ... latency
#endif
#ifndef KPX_MINB_F32_TRIG6
#define KPX_MINB_F32_TRIG6 4     // Dubins airplane, throughput
#endif
#ifndef KPX_MINS_F32_TRIG6
#define KPX_MINS_F32_TRIG6 2
#endif
#ifndef KPX_MINB_F32_MID
#define KPX_MINB_F32_MID 3       // 12-D models (quadcopter, 2 stacked integrators), throughput
#endif
#ifndef KPX_MINS_F32_MID
#define KPX_MINS_F32_MID 2
#endif
#ifndef KPX_MINB_F32_DI12
#define KPX_MINB_F32_DI12 3      // 12-D stacked integrators, throughput
#endif
#ifndef KPX_MINB_F32_BIG
#define KPX_MINB_F32_BIG 2       // 24-D / 48-D stacked integrators, throughput (1: di24 -21 %, di48 -44 %)
#endif

// Everything on the propagation path is inlined into the kernel: measured on B200, any out-of-line call on
// it (the S1 phase, the integrator, or even the rare cooperative walk) costs 30 % of the batch throughput.
#ifndef KPX_S1_ATTR
#define KPX_S1_ATTR __forceinline__
#endif
#ifndef KPX_RQ_ATTR
#define KPX_RQ_ATTR __forceinline__
#endif

namespace kpx {

struct Ctl {                      // one per workspace, global memory
    // persistent run state (valid between launches: stepped runs, resume)
    int size, iteration, status, solution_slot;
    double total_prev;            // sum of scores of the last estimate pass
    double total_pub;             // exchange word for the total when one CTA combines it for the team
    int ve;                       // |V_E| for the next iteration
    int lam_last;
    // per-iteration exchange words
    int first_hit_w;              // lowest kept item index that ends in the goal
    int stop;                     // set by the timekeeper thread
    unsigned long long rescue_key;
    int rescue_slot;
    int n_items_last, n_keep_last;
    int cnt_valid[2], cnt_open[2];  // by iteration parity (trace only)
    // cumulative work
    unsigned long long sum_items, sum_substeps, sum_points, sum_boxsteps;
    unsigned long long sum_free;  // extensions finished from the closed form (FreeFlight), a subset of sum_items
    // timing (globaltimer ns)
    unsigned long long t_begin, t_reset_done, t_end;
    int n_trace;
    int chain_len;
    int cur_query;                // batch mode: query index broadcast to the team
    unsigned int unit_next;       // S1: next 32-item unit of the length-sorted order / of the undecided-item list
    unsigned int n_todo;          // S1 (float32 double integrators): undecided items in the list (Workspace::order)
    int last_sorted;              // 1 if the last iteration's it_* arrays are in sorted-position order
    // claim-table epoch (see Workspace::claim): the epoch the last query used; epoch_valid = 0 forces a dense
    // reset of the claim table and the region arrays (fresh state loaded from the host)
    int epoch_valid;
    unsigned int epoch_used;
    // run clock: device time the loop has been running over all launches since the reset (stepped / resumed runs
    // do not count the host's idle time between launches; planner.py:282 compares against t_max)
    unsigned long long elapsed_ns;
    int n_est;                    // regions in Workspace::est_ids (those the next estimate pass covers)
    int cap, growths;             // capacity in effect and how often it was raised (adaptive t_e)
};

constexpr int kBins = 64;          // substep-count bins of the S0 counting sort (S >= 63 share the last bin)
constexpr int kPacketSegs = 64;    // solution segments carried inline in the result packet
struct ResultPacket {             // everything the host needs after a run, one D2H copy
    Ctl ctl;
    double end_state[KPX_MAX_DIM];
    double seg_dt[kPacketSegs];
    long long seg_slot[kPacketSegs];
    double seg_control[kPacketSegs][KPX_MAX_CONTROL];
    double seg_start[kPacketSegs][KPX_MAX_DIM];
};

struct RunState {                 // CTA-uniform state of the running query, shared memory (one copy per CTA)
    int size, it, status, solution_slot, ve, iters;
    int cap;                      // tree capacity in effect (t_e, or what adaptive growth has made of t_e_start)
    double total_prev;
    unsigned long long t_start;   // keeper only
    // header of the current iteration
    int lam, items, n_sch_old, par, sorted;
    int n_est;                    // available regions, i.e. entries of Workspace::est_ids, for this iteration's estimate pass
    uint32_t claim_tag;           // epoch of this query << claim_shift
    unsigned long long h0;
    unsigned long long tp[7];     // keeper only: phase boundary timestamps
    // S1 work of this CTA in the current iteration (substeps, points, boxsteps, valid items, closed-form items): summed
    // here and flushed to Ctl once per CTA -- thousands of units adding to the same global words serialise in L2
    unsigned long long work[5];
};

struct Workspace {                // device pointers of one team's state
    void *states, *control, *dt;  // R[cap][row(n)], R[cap][row(nu)], R[cap]   (tree arena, node-major padded rows: Row<R, N>)
    int *parent, *region;         // [cap]
    uint8_t* tag;                 // [cap]
    int *n_valid, *n_invalid, *cov;   // [R]
    // [R] score of the last estimate pass that covered the region; NEGATIVE (or NaN) = never estimated, which is
    // exactly "p_accept is still 1.0" (decomposition.py:66-74: p_accept starts at 1; planner.py:246: a region joins the
    // estimate pass one iteration after its first node) -- so one 8-byte gather answers p_accept for a node
    double* score;
    uint32_t* avail_bits;         // [ceil(R/32)] bit r set once region r has been made available
    uint32_t* touched_bits;       // [ceil(R/32)] regions whose counters the current query has touched (lazy reset)
    // [R * subs] first-visit claims, epoch-tagged so that a new query needs no reset: with E the query's epoch
    // (counting DOWN from query to query) and s = PlanArgs::claim_shift, a word is  E << s        visited,
    //                                                                              E << s | w+1  claimed by item w
    // and any word whose upper bits differ from E (older epochs are LARGER, 0xFFFFFFFF = never) is free, which is
    // exactly the order atomicMin needs: a fresh claim beats stale words, the lowest item beats other items, and
    // nothing beats "visited".  The table is refilled with 0xFF only when the epochs run out (2^(32-s) - 1 queries).
    uint32_t* claim;
    void* it_end;                 // rows like `states`: end states of this iteration's valid items, by sorted position
    uint32_t* it_code;            // [cap] per-item result word (kItemGoalBit / kItemDeadBit, kpx_device.cuh)
    int *it_rank, *it_parent;     // [cap]
    uint8_t* it_bin;              // [cap] substep-count bin of each item
    int2* order;                  // [cap] (item number, parent slot) sorted by substep count, longest first
    int* pos_of;                  // [cap] inverse of `order`: where item w's results live in the it_* arrays
    unsigned int* bin_cursor;     // [kBins] per-bin fill cursor / histogram of the current iteration
    int *e_local;                 // [cap]  chunk-major compacted EXPAND slots
    int *cnt_expand, *cnt_keep;   // [max_chunks]
    int* est_ids;                 // [R] available regions in ascending order: the reference's avail_ids (decomposition.py:175)
    double* leaf_sum;             // [R/64 + 2] leaf sums of the pairwise score total (see estimate_leaves)
    unsigned int* bar;            // {count, generation}
    Ctl* ctl;
    kpx_trace* trace;             // [max_trace]
    // solution chain written on success
    double *chain_start, *chain_control, *chain_dt; long long* chain_slot; double* chain_end;
    ResultPacket* packet;         // packed copy of ctl + the first kPacketSegs chain segments
};

struct QueryIn {
    unsigned long long seed;
    double start[KPX_MAX_DIM];
    double goal[4];
    int scene;                    // obstacle set of this query (kpx_batch_set_scenes); 0 = the problem's own
    int pad;
};

template <class R>
struct PlanArgs {
    Params<R> P;
    const R* obs;                 // device boxes [n_scenes][n_obs][8]: min xyz, -, max xyz, -
    const uint32_t* occ;          // device occupancy masks [n_scenes][2][kOccGrid^3] (exact | dilated)
    Workspace* ws;                // [n_teams]
    const QueryIn* queries;       // [n_queries]
    kpx_query_result* results;    // [n_queries] (may be null)
    unsigned int* queue;          // next query index (batch mode)
    int n_queries, n_teams, team_ctas, max_chunks, max_trace, max_chain;
    int claim_shift;              // bits of a claim word that hold the item index + 1 (2^shift > t_e)
    int stride;                   // rows every per-node array is allocated for: capacity padded to a chunk multiple
    int resume;                   // 1: continue from Ctl (no reset), single query
    int max_iters, lam_override;
    double t_max_s;
    const uint32_t* stop_flag;    // polled once per iteration (may be null)
    uint32_t* const* peer_flags;  // set to 1 on success (may be null)
    int n_peers;
    // batch-mode chain outputs, [n_queries][max_chain][...] (may be null)
    double *b_chain_start, *b_chain_control, *b_chain_dt;
    // Hand-off of the last queries of a batch to wider teams (kpx_batch_launch).  Every team that runs out of work
    // adds 1 to *idle; once handoff_at teams are idle the teams still planning stop after their iteration with the
    // run state in Ctl (exactly the state a stepped single plan keeps between launches) and list (workspace, query)
    // in susp_out.  The next launch -- teams of more CTAs, resume = 1 -- continues entry j of resume_in on team j.
    unsigned int* idle;           // may be null
    int handoff_at;               // 0: never suspend
    int pass_on_below;            // a resumed stage handed this many queries or fewer passes them straight on (they
                                  // already fit the next, wider stage)
    int2* susp_out; unsigned int* n_susp_out;
    const int2* resume_in; const unsigned int* n_resume_in;
};
constexpr int KPX_HANDOFF = 6;    // internal stop code: never reaches a result (the resumed launch overwrites it)

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct Team {
    int ctas, rank;
    unsigned int* bar;
    int ws_index;                 // which workspace of PlanArgs::ws this team plans on
};

// Barrier over the team's CTAs (all co-resident: cooperative launch).  One atomic per CTA: rank 0 adds
// 2^31 - (ctas-1), everyone else 1, so the word's top bit flips exactly when the last CTA arrives and the
// low bits return to their old value; each CTA spins until the top bit differs from what its own add saw.
__device__ __forceinline__ void team_sync(const Team& T) {
    __syncthreads();
    if (T.ctas > 1) {
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned int inc = T.rank == 0 ? 0x80000000u - (unsigned)(T.ctas - 1) : 1u;
            const unsigned int old = atomicAdd(T.bar, inc);
            volatile unsigned int* w = T.bar;
            while (((old ^ *w) & 0x80000000u) == 0u) {}
            __threadfence();
        }
        __syncthreads();
    }
}

// ---- block-level helpers (kBlock threads) ----------------------------------
// exclusive prefix of one value per thread; *total = block sum.  s_w: >= kBlock/32 + 1 ints.
__device__ __forceinline__ int block_excl_scan(int v, int* s_w, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = warp_incl_scan(v);
    __syncthreads();                       // protect s_w reuse
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int x = lane < kBlock / 32 ? s_w[lane] : 0;
        int xi = warp_incl_scan(x);
        if (lane < kBlock / 32) s_w[lane] = xi - x;
        if (lane == kBlock / 32 - 1) s_w[kBlock / 32] = xi;
    }
    __syncthreads();
    *total = s_w[kBlock / 32];
    return s_w[wid] + inc - v;
}
// exclusive scan of a global int array (n <= max_chunks) into shared memory; s_out[n] = total
__device__ __forceinline__ int scan_counts(const int* __restrict__ g, int n, int* s_out, int* s_w) {
    int carry = 0;
    for (int base = 0; base < n; base += kBlock) {
        int i = base + threadIdx.x;
        int v = i < n ? __ldcg(g + i) : 0;
        int tot;
        int ex = block_excl_scan(v, s_w, &tot);
        if (i < n) s_out[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) s_out[n] = carry;
    __syncthreads();
    return carry;
}
__device__ __forceinline__ double block_sum_f64(double v, double* s_d) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) s_d[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (wid == 0) {
        t = lane < kBlock / 32 ? s_d[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) s_d[0] = t;
    }
    __syncthreads();
    return s_d[0];
}

// acceptance probability of region r as of the last estimate pass (decomposition.py:189-203); regions no pass
// has covered yet keep 1.0 (their score word is still the "never" sentinel).
__device__ __forceinline__ double p_accept_of(int r, const double* __restrict__ score, double total, double eps) {
    const double sc = __ldcg(score + r);
    if (!(sc >= 0.0)) return 1.0;
    if (total <= 0.0) return eps < 1.0 ? eps : 1.0;
    const double v = __dadd_rn(__ddiv_rn(sc, total), eps);
    return v < 1.0 ? v : 1.0;
}

// warp-aggregated region counters (decomposition.py:117-125): one fire-and-forget atomic per distinct key per
// warp, plus the region's bit in the touched-bitmap that drives the lazy reset of the next query.
__device__ __forceinline__ void count_outcome(int* __restrict__ n_valid, int* __restrict__ n_invalid, int region,
                                              bool valid, bool active, uint32_t* __restrict__ touched_bits) {
    unsigned mask = __ballot_sync(0xffffffffu, active && region >= 0);
    if (active && region >= 0) {
        int key = region * 2 + (valid ? 1 : 0);
        unsigned peers = __match_any_sync(mask, key);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) {
            atomicAdd((valid ? n_valid : n_invalid) + region, __popc(peers));
            atomicOr(touched_bits + (region >> 5), 1u << (region & 31));
        }
    }
}


// ---- estimate total in NumPy's pairwise order (decomposition.py:199: score[avail_ids].sum()) ---------------
// np.sum over a contiguous float64 array of n elements is a fixed recursion: n > 128 splits at
// n2 = n/2 - (n/2) % 8 into sum(a[0:n2]) + sum(a[n2:n]); a block of 8 <= n <= 128 elements keeps 8 strided
// accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and then adds the n % 8 tail in order; n < 8 is a
// plain left-to-right sum.  Every node of n > 128 elements has children of >= 64 elements, so the leaves are
// 64..128 elements long and the compact indices 0, 64, 128, ... ("probes") each fall into one leaf, every leaf
// containing one or two of them: the leaf that starts at compact index lo belongs to probe ceil(lo / 64).
// The tree therefore needs no list: each probe finds its node by descending from the root (<= ~20 steps).
__device__ __forceinline__ int pw_left(int n) { int n2 = n >> 1; return n2 - (n2 & 7); }
// node of depth <= max_depth that contains compact index i: returns its depth, (*lo, *n) its range
__device__ __forceinline__ int pw_descend(int na, int i, int max_depth, int* lo, int* n) {
    int l = 0, m = na, d = 0;
    while (m > 128 && d < max_depth) {
        const int n2 = pw_left(m);
        if (i < l + n2) m = n2; else { l += n2; m -= n2; }
        ++d;
    }
    *lo = l; *n = m;
    return d;
}

// S3: one warp per leaf computes the scores of its <= 128 regions (Eq. 3-4, decomposition.py:175-187), stores
// them, and sums them in NumPy's order into leaf_sum[probe].  Leaves are spread over the team's warps.
// `buf`: 128 doubles of shared memory per warp.
template <class R>
__device__ __forceinline__ void estimate_leaves(const Params<R>& P, const Workspace& W, const Team& T, int na, double* buf) {
    const int lane = threadIdx.x & 31;
    const int n_probe = (na + 63) >> 6;
    const int team_warps = T.ctas * kWarps;
    for (int k = T.rank * kWarps + (threadIdx.x >> 5); k < n_probe; k += team_warps) {
        int lo, n;
        pw_descend(na, k << 6, 0x7fffffff, &lo, &n);
        if (k != ((lo + 63) >> 6)) continue;                 // the leaf's other probe (warp-uniform)
        for (int e = lane; e < n; e += 32) {
            const int r = __ldcg(W.est_ids + lo + e);
            const double nv = (double)__ldcg(W.n_valid + r), ni = (double)__ldcg(W.n_invalid + r);
            // rn intrinsics: never contracted to FMA, so both precision builds agree bit for bit
            const double dn = __dadd_rn(P.delta, nv);
            const double fv = __ddiv_rn(__dmul_rn(dn, P.vol), __dadd_rn(dn, ni));
            const double tt = __dadd_rn(nv, ni);
            const double f2 = __dmul_rn(fv, fv);
            const double sc = __ddiv_rn(__dmul_rn(f2, f2), __dmul_rn(__dadd_rn(1.0, (double)__ldcg(W.cov + r)),
                                                                      __dadd_rn(1.0, __dmul_rn(tt, tt))));
            __stcg(W.score + r, sc);
            buf[e] = sc;
        }
        __syncwarp();
        double res = 0.0;
        if (n < 8) {
            if (lane == 0) for (int i = 0; i < n; ++i) res = __dadd_rn(res, buf[i]);
        } else {
            const int body = n - (n & 7);
            double acc = buf[lane & 7];
            for (int i = 8 + (lane & 7); i < body; i += 8) acc = __dadd_rn(acc, buf[i]);
            acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));       // r0+r1 | r2+r3 | r4+r5 | r6+r7
            acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));       // (r0+r1)+(r2+r3) | (r4+r5)+(r6+r7)
            acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
            res = acc;
            if (lane == 0) for (int i = body; i < n; ++i) res = __dadd_rn(res, buf[i]);
        }
        if (lane == 0) __stcg(W.leaf_sum + k, res);
        __syncwarp();
    }
}

// S4: the tree above the leaves, level by level from the deepest, in place: the result of the node that
// starts at compact index lo lives in slot ceil(lo / 64) (the slot of its leftmost leaf).  GLOBAL = false: `v` is
// n_probe doubles of shared memory private to the CTA, filled from leaf_sum here (every CTA of a team combines
// for itself); GLOBAL = true: one CTA combines in leaf_sum itself.  Returns the total to every calling thread.
template <bool GLOBAL>
__device__ __forceinline__ double combine_leaves(double* leaf_sum, int na, double* v) {
    if (na <= 0) return 0.0;
    const int n_probe = (na + 63) >> 6;
    if (GLOBAL) v = leaf_sum;
    else for (int k = threadIdx.x; k < n_probe; k += kBlock) v[k] = __ldcg(leaf_sum + k);   // non-owner slots are never read
    int depth = 0;
    for (int m = na; m > 128; m -= pw_left(m)) ++depth;      // the right child is the larger one
    __syncthreads();
    for (int d = depth - 1; d >= 0; --d) {
        for (int k = threadIdx.x; k < n_probe; k += kBlock) {
            int lo, n;
            const int dd = pw_descend(na, k << 6, d, &lo, &n);
            if (dd == d && n > 128 && k == ((lo + 63) >> 6)) {
                const int kr = (lo + pw_left(n) + 63) >> 6;
                if (GLOBAL) __stcg(v + k, __dadd_rn(__ldcg(v + k), __ldcg(v + kr)));
                else v[k] = __dadd_rn(v[k], v[kr]);
            }
        }
        __syncthreads();
    }
    const double total = GLOBAL ? __ldcg(v) : v[0];
    __syncthreads();
    return total;
}
constexpr int kMaxProbes = 2048;   // leaf slots a CTA can combine in shared memory: up to 131 072 available regions

// Ascending list of the available regions (= the regions the NEXT estimate pass covers) out of the availability
// bitmap: every CTA counts the 1024-region blocks into shared memory (s_pre[n_blocks + 1], exclusive prefix),
// then the team's warps expand the blocks.  Readers are separated from this by at least one team barrier.
// Returns the number of available regions (the same value in every thread of the team).
__device__ __forceinline__ int build_est_list(const Workspace& W, const Team& T, int n_regions, int* s_pre, int* s_w) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n_words = (n_regions + 31) >> 5, n_blocks = (n_words + 31) >> 5;
    __syncthreads();
    for (int b = wid; b < n_blocks; b += kWarps) {
        const int wi = b * 32 + lane;
        const int c = __reduce_add_sync(0xffffffffu, wi < n_words ? __popc(__ldcg(W.avail_bits + wi)) : 0);
        if (lane == 0) s_pre[b] = c;
    }
    __syncthreads();
    int carry = 0;
    for (int base = 0; base < n_blocks; base += kBlock) {
        const int i = base + threadIdx.x;
        const int v = i < n_blocks ? s_pre[i] : 0;
        int tot;
        const int ex = block_excl_scan(v, s_w, &tot);
        if (i < n_blocks) s_pre[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) s_pre[n_blocks] = carry;
    __syncthreads();
    const int team_warps = T.ctas * kWarps;
    for (int b = T.rank * kWarps + wid; b < n_blocks; b += team_warps) {
        if (s_pre[b + 1] == s_pre[b]) continue;
        const int wi = b * 32 + lane;
        uint32_t bits = wi < n_words ? __ldcg(W.avail_bits + wi) : 0u;
        const int c = __popc(bits);
        int at = s_pre[b] + warp_incl_scan(c) - c;
        while (bits) { __stcg(W.est_ids + at++, wi * 32 + __ffs(bits) - 1); bits &= bits - 1; }
    }
    __syncthreads();
    return carry;
}

// ---- S1: propagation ---------------------------------------------------------------------------------
#ifndef KPX_TILE_CHUNKS
#define KPX_TILE_CHUNKS 2            // 2 048 items per sorted tile (1: -1 %, 4: -1.4 %, 8: -3 % on quad12/narrow)
#endif

// i-th EXPAND slot: chunk by binary search over the chunk prefix, then the chunk-local compacted list
__device__ __forceinline__ int expand_slot(const Workspace& W, const int* s_prefix, int n_sch_old, int i) {
    int lo = 0, hi = n_sch_old;                    // prefix[lo] <= i < prefix[hi]
    while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (s_prefix[mid] <= i) lo = mid; else hi = mid; }
    return __ldcg(W.e_local + lo * kChunk + (i - s_prefix[lo]));
}

// Results of one item (warp-synchronous: all 32 lanes call it, `active` = this lane holds a finished item):
// the item word + end state at its position, the first-visit claim, the region counters, the work counters.
template <class M, class R>
__device__ __forceinline__ void commit_item(const PlanArgs<R>& A, const Workspace& W, const QueryIn& Q, uint32_t claim_tag,
                                            unsigned long long* work, bool active, int w, int pos, const ItemOut<R, M::N>& o) {
    constexpr int N = M::N;
    const Params<R>& P = A.P;
    int region = -1; bool valid = false;
    if (active) {
        region = o.region; valid = o.valid;
        uint32_t code = region >= 0 ? (kItemDeadBit | (uint32_t)region) : kItemInvalid;
        if (valid) {
            const uint32_t pair = (uint32_t)region * (uint32_t)P.subs_per_region + (uint32_t)o.sub;
            const R d0 = o.end[0] - (R)Q.goal[0], d1 = o.end[1] - (R)Q.goal[1], d2 = o.end[2] - (R)Q.goal[2];
            const bool hit = MathK<R>::sq(d0 * d0 + d1 * d1 + d2 * d2) <= (R)Q.goal[3];
            code = pair | (hit ? kItemGoalBit : 0u);
            store_row<N>((R*)W.it_end, pos, o.end);
            if (__ldcg(W.claim + pair) != claim_tag) atomicMin(W.claim + pair, claim_tag | (uint32_t)(w + 1));
        }
        __stcg(W.it_code + pos, code);
    }
    count_outcome(W.n_valid, W.n_invalid, region, valid, active, W.touched_bits);
    // work counters: one reduction and one shared-memory atomic per unit (RunState::work)
    const int t_sub = __reduce_add_sync(0xffffffffu, active ? o.substeps : 0);
    const int t_pts = __reduce_add_sync(0xffffffffu, active ? o.points : 0);
    const int t_box = __reduce_add_sync(0xffffffffu, active ? o.boxsteps : 0);
    const int t_val = __popc(__ballot_sync(0xffffffffu, valid));
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(work + 0, (unsigned long long)t_sub);
        atomicAdd(work + 1, (unsigned long long)t_pts);
        atomicAdd(work + 2, (unsigned long long)t_box);
        if (t_val) atomicAdd(work + 3, (unsigned long long)t_val);
    }
}

// One 32-item unit (warp-synchronous): lane `lane` handles the item stored at position `pos` (< limit).
// sorted: the item number and its parent slot come from `order` (results stay addressed by item number w
// through pos_of); unsorted: position == item number.
template <class M, class R>
__device__ __forceinline__ void propagate_unit(const PlanArgs<R>& A, const Workspace& W, const QueryIn& Q,
                                               RunState& RS, const int* s_prefix, int pos, int limit, bool sorted) {
    constexpr int N = M::N, NU = M::NU;
    const Params<R>& P = A.P;
    // the iteration header is re-read from shared memory per unit: nothing of it stays in registers
    const int lam = RS.lam;
    const uint64_t h0 = RS.h0;
    const bool active = pos < limit;
    int w = 0, S = 0;
    R u[NU], dt = (R)0, x0[N];
    if (active) {
        int slot;
        if (sorted) {
            const int2 ws = __ldcg(W.order + pos);          // item number and its parent slot in one load
            w = ws.x; slot = ws.y;
        } else {
            w = pos;
            slot = expand_slot(W, s_prefix, RS.n_sch_old, w / lam);
            __stcg(W.it_parent + w, slot);
        }
        sample_control<M, R>(P, h0, slot, w % lam, u, &dt, &S, nullptr, nullptr);
        load_row<N>((const R*)W.states, slot, x0);
    } else {
#pragma unroll
        for (int d = 0; d < N; ++d) x0[d] = (R)0;
#pragma unroll
        for (int j = 0; j < NU; ++j) u[j] = (R)0;
    }
    ItemOut<R, N> o;
    integrate_and_map<M, R>(P, active, x0, u, dt, S, o);     // warp-synchronous
    commit_item<M, R>(A, W, Q, RS.claim_tag, RS.work, active, w, pos, o);
}

// The same for the float32 double integrators (FreeFlight, kpx_device.cuh), in two passes over the iteration.
// Pass 1 (flight_settle_unit): every lane tries to settle its item from the closed form -- certified valid or invalid,
// ~90 % of the Trees workload -- and commits it; an undecided item (it passes near an obstacle) is appended to a list.
// Pass 2 (flight_eval_unit): warps pull 32 list entries at a time, each lane re-derives ITS item's sample, and the
// warp then evaluates them ONE ITEM AT A TIME, lane = RK4 substep (di_item_by_substeps): the closed form makes the
// sampled states independent of each other, so the S segment tests of an extension run side by side and an extension
// costs one or two warp rounds whatever its length.  The list decouples the second pass from where the hard items
// cluster (the lambda children of a node next to an obstacle are all undecided): every warp gets the same load.
// Position == item number throughout: nothing is sorted.
template <class M>
__device__ __forceinline__ void flight_settle_unit(const PlanArgs<float>& A, const Workspace& W, const QueryIn& Q,
                                                   RunState& RS, const int* s_prefix, int pos, int limit) {
    constexpr int N = M::N, NU = M::NU;
    using F = FreeFlight<typename M::Base, float>;
    const Params<float>& P = A.P;
    const int lam = RS.lam, lane = threadIdx.x & 31;
    const bool active = pos < limit;
    const int w = pos;
    int slot = 0, verdict = kFlightInvalid;
    ItemOut<float, N> o;
    if (active) {
        float u[NU], dt, x0[N];
        int S;
        slot = expand_slot(W, s_prefix, RS.n_sch_old, w / lam);
        __stcg(W.it_parent + w, slot);
        sample_control<M, float>(P, RS.h0, slot, w % lam, u, &dt, &S, nullptr, nullptr);
        load_row<N>((const float*)W.states, slot, x0);
        verdict = F::certify(P, x0, u, dt, S, o);
        if (verdict != kFlightFull) map_end_state<M, float>(P, o.end, true, verdict == kFlightValid, o);
    }
    const bool settled = active && verdict != kFlightFull;
    const unsigned sm = __ballot_sync(0xffffffffu, settled), tm = __ballot_sync(0xffffffffu, active && !settled);
    if (tm) {                                       // undecided items: (item, parent slot) into the list, one atomic per warp
        int base = 0;
        if (lane == 0) base = (int)atomicAdd(&W.ctl->n_todo, (unsigned)__popc(tm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (active && !settled) __stcg(W.order + base + __popc(tm & ((1u << lane) - 1u)), make_int2(w, slot));
    }
    if (sm) {
        commit_item<M, float>(A, W, Q, RS.claim_tag, RS.work, settled, w, pos, o);
        if (lane == 0) atomicAdd(RS.work + 4, (unsigned long long)__popc(sm));
    }
}

template <class M>
__device__ __forceinline__ void flight_eval_unit(const PlanArgs<float>& A, const Workspace& W, const QueryIn& Q,
                                                 RunState& RS, int idx, int n_todo) {
    constexpr int N = M::N, NU = M::NU;
    using F = FreeFlight<typename M::Base, float>;
    const Params<float>& P = A.P;
    const int lam = RS.lam, lane = threadIdx.x & 31;
    const bool active = idx < n_todo;
    int w = 0, S = 0;
    float u[NU], dt = 0.0f, x0[N];
    if (active) {
        const int2 ws = __ldcg(W.order + idx);
        w = ws.x;
        sample_control<M, float>(P, RS.h0, ws.y, w % lam, u, &dt, &S, nullptr, nullptr);
        load_row<N>((const float*)W.states, ws.y, x0);
    } else {
#pragma unroll
        for (int d = 0; d < N; ++d) x0[d] = 0.0f;
#pragma unroll
        for (int j = 0; j < NU; ++j) u[j] = 0.0f;
    }
    ItemOut<float, N> o;
    bool valid = false;
    unsigned todo = __ballot_sync(0xffffffffu, active);
#pragma unroll 1
    while (todo) {
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        float bx[N], bu[NU];
#pragma unroll
        for (int d = 0; d < N; ++d) bx[d] = __shfl_sync(0xffffffffu, x0[d], src);
#pragma unroll
        for (int j = 0; j < NU; ++j) bu[j] = __shfl_sync(0xffffffffu, u[j], src);
        const float bdt = __shfl_sync(0xffffffffu, dt, src);
        const int bS = __shfl_sync(0xffffffffu, S, src);
        bool ok; int boxsteps, points;
        F::by_substeps(P, bx, bu, bdt, bS, &ok, &boxsteps, &points);
        if (lane == src) { valid = ok; o.substeps = S; o.boxsteps = boxsteps; o.points = points; }
    }
    if (active) {
        F::end_state(x0, u, dt, o.end);
        map_end_state<M, float>(P, o.end, true, valid, o);
    }
    commit_item<M, float>(A, W, Q, RS.claim_tag, RS.work, active, w, w, o);     // results live at the item's own number
}

// S1 of one iteration: propagate every (EXPAND slot x extension) item, count outcomes per region, claim fresh
// (region, sub) pairs.  Schedules, identical results (everything downstream is addressed by item number):
//   * position == item number, units strided over the team's warps: iterations that fit one round of the team's
//     threads -- and ALWAYS for the float32 double integrators, whose units all cost the same (flight_settle_unit),
//     followed by their second pass over the list of undecided items (flight_eval_unit);
//   * a team of many CTAs: the items were sorted by length over the whole iteration (S0 in iteration_head),
//     warps pull units from a shared cursor, longest first;
//   * a team of ONE CTA (many queries per GPU): tiles of kTileM consecutive items are sorted by length in shared
//     memory and propagated right away.  A warp's 32 items then have nearly equal length AND parents that lie
//     close to each other (a tile spans kTileM / lambda consecutive EXPAND slots), and S0 needs neither global
//     atomics nor team barriers.
template <class M, class R>
__device__ KPX_S1_ATTR void s1_propagate(const PlanArgs<R>& A, const Workspace& W, const QueryIn& Q, RunState& RS,
                                         int team_rank, int team_ctas, const int* s_prefix, int* s_bin) {
    const int lane = threadIdx.x & 31, tid = threadIdx.x;
    const bool sorted = RS.sorted != 0;
    const bool tiled = sorted && team_ctas == 1;
    uint8_t* const s_len = (uint8_t*)(kpx_dyn_smem + Scene<R>::kCoop);   // [kTileM]; the staging area is idle while sorting
    constexpr int kTileM = KPX_TILE_CHUNKS * kChunk;        // items per tile
    static_assert(sizeof(WarpCoop<R>) * kWarps >= kTileM, "tile lengths must fit the staging area");
    int tile = -kTileM, n_units = 0, tile_limit = 0;
    int unit = sorted ? 0x3fffffff : (team_rank * kBlock + tid) >> 5;    // unsorted: this warp's slice of the one round
    // one loop, one copy of the integrator: the three schedules only differ in how the next unit is found
#pragma unroll 1
    for (;;) {
        int pos, limit;
        if (tiled) {
            if (unit >= n_units) {
                // this warp is through with the tile: every warp of the CTA meets here once per tile.
                // Counting sort of the next tile by substep count, longest first.
                tile += kTileM;
                const int items = RS.items;
                if (tile >= items) break;
                const int lam = RS.lam, n_sch_old = RS.n_sch_old;
                const uint64_t h0 = RS.h0;
                const int n_t = items - tile < kTileM ? items - tile : kTileM;
                __syncthreads();                        // the previous tile's walks are done with the staging area
                for (int b = tid; b < 2 * kBins; b += kBlock) s_bin[b] = 0;          // histogram | fill
                if (tid == 0) s_bin[3 * kBins] = 0;                                  // unit cursor of the tile
                __syncthreads();
#pragma unroll 1
                for (int j = tid; j < n_t; j += kBlock) {
                    const int w = tile + j;
                    const int i = w / lam;
                    const int slot = expand_slot(W, s_prefix, n_sch_old, i);
                    int S = substeps_of<M, R>(A.P, h0, slot, w - i * lam);
                    S = S < kBins - 1 ? S : kBins - 1;
                    __stcg(W.it_parent + w, slot);
                    s_len[j] = (uint8_t)S;
                    atomicAdd(&s_bin[S], 1);
                }
                __syncthreads();
                if (tid < 32) {                         // start of every bin, longest first (2 bins per lane)
                    const int b1 = kBins - 1 - 2 * lane, b0 = b1 - 1;
                    const int h1 = s_bin[b1], h0c = s_bin[b0];
                    const int incl = warp_incl_scan(h1 + h0c);
                    s_bin[2 * kBins + b1] = incl - h1 - h0c;
                    s_bin[2 * kBins + b0] = incl - h0c;
                }
                __syncthreads();
#pragma unroll 1
                for (int j = tid; j < n_t; j += kBlock) {
                    const int b = s_len[j];
                    const int p = tile + s_bin[2 * kBins + b] + atomicAdd(&s_bin[kBins + b], 1);
                    __stcg(W.order + p, make_int2(tile + j, __ldcg(W.it_parent + tile + j)));
                    __stcg(W.pos_of + tile + j, p);     // results of item w are stored at its sorted position
                }
                __syncthreads();
                tile_limit = tile + n_t;
                n_units = (n_t + 31) >> 5;
            }
            // warps pull the tile's units from a shared-memory cursor, longest first
            if (lane == 0) unit = atomicAdd(&s_bin[3 * kBins], 1);
            unit = __shfl_sync(0xffffffffu, unit, 0);
            if (unit >= n_units) continue;              // tile exhausted: on to the next one
            pos = tile + unit * 32 + lane;
            limit = tile_limit;
        } else if (sorted) {
            if (lane == 0) unit = (int)atomicAdd(&W.ctl->unit_next, 1u);
            unit = __shfl_sync(0xffffffffu, unit, 0);
            limit = RS.items;
            if ((long long)unit * 32 >= limit) break;
            pos = unit * 32 + lane;
        } else {
            limit = RS.items;
            if ((long long)unit * 32 >= limit) break;
            pos = unit * 32 + lane;
            unit += team_ctas * kWarps;                 // one round, unless nothing is sorted for this model
        }
        if constexpr (FreeFlight<typename M::Base, R>::kEnabled) flight_settle_unit<M>(A, W, Q, RS, s_prefix, pos, limit);
        else propagate_unit<M, R>(A, W, Q, RS, s_prefix, pos, limit, sorted);
    }
    if constexpr (FreeFlight<typename M::Base, R>::kEnabled) {
        // second pass: the undecided items, 32 list entries per pull
        Team T;
        T.ctas = team_ctas; T.rank = team_rank; T.bar = W.bar;
        team_sync(T);                                   // the list is complete
        const int n_todo = (int)__ldcg(&W.ctl->n_todo);
        // entries per pull: a warp's worth when the team is small against the list (many queries per GPU), fewer when
        // one query has the whole GPU -- a warp evaluates its entries one after the other, and the longest warp is S1
        const int team_warps = team_ctas * kWarps;
        int chunk = (n_todo + team_warps - 1) / team_warps;
        chunk = chunk < 1 ? 1 : (chunk > 32 ? 32 : chunk);
#pragma unroll 1
        for (;;) {
            int unit2 = 0;
            if (lane == 0) unit2 = (int)atomicAdd(&W.ctl->unit_next, 1u);
            unit2 = __shfl_sync(0xffffffffu, unit2, 0);
            if ((long long)unit2 * chunk >= n_todo) break;
            const int hi = unit2 * chunk + chunk < n_todo ? unit2 * chunk + chunk : n_todo;
            flight_eval_unit<M>(A, W, Q, RS, unit2 * chunk + lane, lane < chunk ? hi : 0);
        }
    }
    // this CTA's work counters of the iteration: one global atomic each
    __syncthreads();
    if (tid < 5 && RS.work[tid]) {
        Ctl* const c = W.ctl;
        if (tid == 3) atomicAdd(&c->cnt_valid[RS.par], (int)RS.work[3]);
        else atomicAdd(tid == 0 ? &c->sum_substeps : (tid == 1 ? &c->sum_points : (tid == 2 ? &c->sum_boxsteps : &c->sum_free)), RS.work[tid]);
    }
}

// Thread / problem constants every phase re-derives for itself (nothing here is carried between phases).
#define KPX_PHASE_LOCALS                                                                                     \
    constexpr int N = M::N, NU = M::NU;                                                                      \
    const Params<R>& P = A.P;                                                                                \
    const int tid = threadIdx.x;                                                                             \
    const int RG = P.n_regions, SUBS = P.subs_per_region;                                                    \
    const bool keeper = (T.rank == 0 && tid == 0);                                                           \
    const long long tthreads = (long long)T.ctas * kBlock;                                                   \
    const long long ttid = (long long)T.rank * kBlock + tid;                                                 \
    R* const states = (R*)W.states; R* const control = (R*)W.control; R* const dts = (R*)W.dt;               \
    R* const it_end = (R*)W.it_end;                                                                          \
    Ctl* const ctl = W.ctl;                                                                                  \
    (void)N; (void)NU; (void)RG; (void)SUBS; (void)keeper; (void)tthreads; (void)ttid;  \
    (void)states; (void)control; (void)dts; (void)it_end; (void)ctl; (void)P;

// ---- reset of a team's workspace for a new query ---------------------------------------------------------
template <class M, class R>
__device__ __forceinline__ void reset_query(const PlanArgs<R>& A, const Workspace& W, const Team& T, const QueryIn& Q) {
    KPX_PHASE_LOCALS
    // ------------------------------------------------------------------ reset
    {
        if (keeper) ctl->t_begin = gtimer();
        const int n_words = (RG + 31) >> 5;
        // epochs left?  (usable epochs: 2^(32-shift) - 2 down to 0; the all-ones field means "never claimed")
        const unsigned int e_max = (1u << (32 - A.claim_shift)) - 2u;
        const unsigned int e_old = __ldcg(&ctl->epoch_used);
        const bool lazy = __ldcg(&ctl->epoch_valid) != 0 && e_old != 0u && e_old <= e_max + 1u;
        const unsigned int e_new = lazy ? e_old - 1u : e_max;
        if (lazy) {
            // the claim table needs nothing (new epoch); the region arrays are cleared where the previous query
            // touched them: one warp per bitmap word, one lane per region
            // a warp reads 32 bitmap words at once (one coalesced load instead of 32 dependent ones) and then
            // clears the regions of every non-zero word, one lane per region
            const int lane = tid & 31;
            for (long long base = (ttid >> 5) * 32; base < n_words; base += (tthreads >> 5) * 32) {
                const long long wi = base + lane;
                const uint32_t mine = wi < n_words ? __ldcg(W.touched_bits + wi) : 0u;
                unsigned nz = __ballot_sync(0xffffffffu, mine != 0u);
                if (mine) { W.touched_bits[wi] = 0u; W.avail_bits[wi] = 0u; }
                while (nz) {
                    const int src = __ffs(nz) - 1;
                    nz &= nz - 1;
                    const uint32_t bits = __shfl_sync(0xffffffffu, mine, src);
                    if ((bits >> lane) & 1u) {
                        const long long r = (base + src) * 32 + lane;
                        W.n_valid[r] = 0; W.n_invalid[r] = 0; W.cov[r] = 0; W.score[r] = -1.0;
                    }
                }
            }
        } else {   // dense reset: claim table + region arrays, 16-byte stores
            uint4* c4 = (uint4*)W.claim;
            long long n4 = ((long long)RG * SUBS) / 4;
            const uint4 ones = make_uint4(kUnclaimed, kUnclaimed, kUnclaimed, kUnclaimed);
            for (long long i = ttid; i < n4; i += tthreads) c4[i] = ones;
            for (long long i = n4 * 4 + ttid; i < (long long)RG * SUBS; i += tthreads) W.claim[i] = kUnclaimed;
            for (long long i = ttid; i < RG; i += tthreads) {
                W.n_valid[i] = 0; W.n_invalid[i] = 0; W.cov[i] = 0; W.score[i] = -1.0;
            }
            for (long long i = ttid; i < n_words; i += tthreads) { W.avail_bits[i] = 0u; W.touched_bits[i] = 0u; }
        }
        if (keeper) {
            // init_root + make_available (planner.py:169-171)
            int reg = 0;
            bool in_goal0;
            for (int d = 0; d < N; ++d) {
                R x = (R)Q.start[d];
                states[d] = x;                                           // row 0
                if (d < P.grid_n) {
                    R rel = (x - P.grid_lo[d]) / P.grid_width[d];
                    R cl = rel < (R)0 ? (R)0 : (rel > P.grid_cmax[d] ? P.grid_cmax[d] : rel);
                    reg += (int)MathK<R>::fl(cl) * P.grid_strides[d];
                }
            }
            {
                double d0 = Q.start[0] - Q.goal[0], d1 = Q.start[1] - Q.goal[1], d2 = Q.start[2] - Q.goal[2];
                in_goal0 = sqrt(d0 * d0 + d1 * d1 + d2 * d2) <= Q.goal[3];
            }
            for (int j = 0; j < NU; ++j) control[j] = (R)0;
            dts[0] = (R)0;
            W.parent[0] = -1; W.region[0] = reg; W.tag[0] = KPX_TAG_EXPAND;
            W.cnt_expand[0] = 1; W.e_local[0] = 0;
            ctl->size = 1; ctl->iteration = 0; ctl->solution_slot = in_goal0 ? 0 : -1;
            ctl->cap = (int)(P.t_e_start > 0 ? P.t_e_start : P.t_e); ctl->growths = 0;
            ctl->status = in_goal0 ? KPX_SOLVED : KPX_RUNNING;      // planner.py:278-280
            ctl->total_prev = 0.0; ctl->ve = 1; ctl->lam_last = 0;
            ctl->first_hit_w = 0x7fffffff; ctl->stop = 0; ctl->rescue_key = 0ull; ctl->rescue_slot = 0x7fffffff;
            ctl->n_items_last = 0; ctl->n_keep_last = 0;
            ctl->cnt_valid[0] = ctl->cnt_valid[1] = ctl->cnt_open[0] = ctl->cnt_open[1] = 0;
            ctl->sum_items = ctl->sum_substeps = ctl->sum_points = ctl->sum_boxsteps = ctl->sum_free = 0ull;
            ctl->n_trace = 0; ctl->chain_len = 0; ctl->unit_next = 0u; ctl->n_todo = 0u;
            for (int b = 0; b < kBins; ++b) W.bin_cursor[b] = 0u;
        }
        team_sync(T);
        if (keeper) {
            const int reg0 = __ldcg(W.region);
            W.avail_bits[reg0 >> 5] = 1u << (reg0 & 31);
            W.touched_bits[reg0 >> 5] = 1u << (reg0 & 31);   // the root's region is dirty from the start
            ctl->epoch_used = e_new; ctl->epoch_valid = 1;
            ctl->t_reset_done = gtimer();
        }
        team_sync(T);
    }

}

// ---- head of an iteration: termination tests, branching factor, S0.  Returns false when the run is over. ---
template <class M, class R>
__device__ __forceinline__ bool iteration_head(const PlanArgs<R>& A, const Workspace& W, const Team& T, const QueryIn& Q,
                                               RunState& RS, int* s_prefix, int* s_bin) {
    KPX_PHASE_LOCALS
    const int size = RS.size, ve = RS.ve, iters = RS.iters, cap = RS.cap;
    int it = RS.it, status = RS.status;
    __syncthreads();                            // every thread holds the state before thread 0 rewrites it
    bool go = status == KPX_RUNNING;
    if (go && A.max_iters > 0 && iters >= A.max_iters) go = false;
    if (go) { const int st = __ldcg(&ctl->stop); if (st) { status = st; go = false; } }
    int lam = 1;
    long long items_ll = 0;
    if (go) {
        ++it;
        lam = (cap - size) / ve;                                       // planner.py:48
        lam = lam > P.lambda_max ? P.lambda_max : lam;
        lam = lam < 1 ? 1 : lam;
        if (A.lam_override > 0) lam = A.lam_override;
        items_ll = (long long)ve * lam;
        if (items_ll > cap) { status = KPX_ERROR; go = false; }
    }
    if (!go) {
        if (tid == 0) { RS.status = status; RS.it = it; }
        __syncthreads();
        return false;
    }
    const int items = (int)items_ll;
    const int n_sch_old = (size + kChunk - 1) / kChunk;
    const uint64_t h0 = iter_key(M::kRng, Q.seed, (uint64_t)it);
    // float32 double integrators finish ~90 % of their items from the closed form and evaluate the rest one warp per
    // item (propagate_unit_flight): no item is longer than another, so there is nothing to sort
    const bool sorted = items > tthreads && !FreeFlight<typename M::Base, R>::kEnabled;
    if (tid == 0) {
        RS.it = it; RS.iters = iters + 1; RS.lam = lam; RS.items = items; RS.n_sch_old = n_sch_old; RS.par = it & 1;
        RS.sorted = sorted ? 1 : 0; RS.h0 = h0;
        for (int k = 0; k < 5; ++k) RS.work[k] = 0ull;
    }
    if (keeper) RS.tp[0] = gtimer();

        // ================================================================= S0: order items by length
        // The substep count S = max(4, ceil(dt/0.02)) of an item follows from its RNG draw alone.  A counting
        // sort on S (longest first) lets every warp integrate 32 items of nearly equal length, and warps pull
        // 32-item units from a shared cursor, so neither lanes nor warps idle behind one long extension.
        // Results stay indexed by the item number w, so nothing downstream sees the processing order.
        // An iteration that fits in one round (items <= team threads) gains nothing from it and skips S0.
        const bool global_sort = sorted && T.ctas > 1;    // one-CTA teams sort tile by tile inside S1
        if (global_sort) {
            for (int b = tid; b < kBins; b += kBlock) { s_bin[b] = 0; s_bin[2 * kBins + b] = 0; }
            __syncthreads();
#pragma unroll 1
            for (long long w0 = (long long)T.rank * kBlock; w0 < items; w0 += tthreads) {
                const int w = (int)w0 + tid;
                if (w < items) {
                    const int i = w / lam, ext = w - i * lam;
                    const int slot = expand_slot(W, s_prefix, n_sch_old, i);
                    int S = substeps_of<M, R>(P, h0, slot, ext);
                    S = S < kBins - 1 ? S : kBins - 1;
                    __stcg(W.it_parent + w, slot);
                    __stcg(W.it_bin + w, (uint8_t)S);
                    atomicAdd(&s_bin[S], 1);
                }
            }
            __syncthreads();
            // reserve this CTA's range inside every bin; the cursor ends up holding the global histogram
            for (int b = tid; b < kBins; b += kBlock) {
                const int h = s_bin[b];
                s_bin[kBins + b] = h ? (int)atomicAdd(W.bin_cursor + b, (unsigned)h) : 0;
            }
        }
        if (global_sort) team_sync(T);
        if (global_sort) {
            if (tid < kBins) s_bin[3 * kBins + tid] = (int)__ldcg(W.bin_cursor + tid);
            __syncthreads();
            if (tid == 0) {
                int acc = 0;
                for (int b = kBins - 1; b >= 0; --b) { const int h = s_bin[3 * kBins + b]; s_bin[3 * kBins + b] = acc; acc += h; }
            }
            __syncthreads();
#pragma unroll 1
            for (long long w0 = (long long)T.rank * kBlock; w0 < items; w0 += tthreads) {
                const int w = (int)w0 + tid;
                if (w < items) {
                    const int b = (int)__ldcg(W.it_bin + w);
                    const int pos = s_bin[3 * kBins + b] + s_bin[kBins + b] + atomicAdd(&s_bin[2 * kBins + b], 1);
                    __stcg(W.order + pos, make_int2(w, __ldcg(W.it_parent + w)));
                    __stcg(W.pos_of + w, pos);          // results of item w are stored at `pos` (coalesced S1 stores)
                }
            }
        }
        if (global_sort) team_sync(T);
        if (keeper) RS.tp[1] = gtimer();

    __syncthreads();                            // the iteration header is visible to the whole CTA
    return true;
}

// ---- S2..S4 and the epilogue of an iteration -------------------------------------------------------------
template <class M, class R>
__device__ __forceinline__ void iteration_tail(const PlanArgs<R>& A, const Workspace& W, const Team& T, const QueryIn& Q,
                                               RunState& RS, int* s_prefix, int* s_w, double* s_d) {
    KPX_PHASE_LOCALS
    const int size = RS.size, it = RS.it, lam = RS.lam, items = RS.items, par = RS.par, cap = RS.cap;
    const bool sorted = RS.sorted != 0;
    const uint64_t h0 = RS.h0;
    const uint32_t claim_tag = RS.claim_tag;
    const double total_prev = RS.total_prev;
    const int n_ich = (items + kChunk - 1) / kChunk;
    {
        // ================================================================= S2
        for (int c = T.rank; c < n_ich; c += T.ctas) {
            const int base = c * kChunk + tid * 4;
            uint32_t code[4];
            if (sorted) {           // results live at the sorted position of each item: one 4-byte gather per item
                int ps[4] = {0, 0, 0, 0};
                if (base + 3 < items) {
                    const int4 p4 = __ldcg((const int4*)(W.pos_of + base));
                    ps[0] = p4.x; ps[1] = p4.y; ps[2] = p4.z; ps[3] = p4.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) if (base + j < items) ps[j] = __ldcg(W.pos_of + base + j);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) code[j] = base + j < items ? __ldcg(W.it_code + ps[j]) : kItemInvalid;
            } else if (base + 3 < items) {
                const uint4 v = __ldcg((const uint4*)(W.it_code + base));
                code[0] = v.x; code[1] = v.y; code[2] = v.z; code[3] = v.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) code[j] = base + j < items ? __ldcg(W.it_code + base + j) : kItemInvalid;
            }
            bool keep[4];
            int cnt = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                keep[j] = false;
                if (!(code[j] & kItemDeadBit)) {
                    const int w = base + j;
                    const uint32_t pair = code[j] & ~kItemGoalBit;
                    const int region = (int)(pair / (uint32_t)SUBS);
                    const bool first = __ldcg(W.claim + pair) == (claim_tag | (uint32_t)(w + 1));   // lowest item index wins
                    if (first) {
                        __stcg(W.claim + pair, claim_tag);                                           // visited
                        atomicAdd(W.cov + region, 1);
                    }
                    bool kp = first;
                    if (!kp) {
                        const int slot = __ldcg(W.it_parent + w);
                        const double ua = keyed_uniform_of<M::kRng>(h0, (uint64_t)slot, (uint64_t)(w % lam), PH_ACCEPT);
                        kp = ua < p_accept_of(region, W.score, total_prev, P.epsilon);
                    }
                    keep[j] = kp;
                    if (kp) {
                        ++cnt;
                        if (code[j] & kItemGoalBit) atomicMin(&ctl->first_hit_w, w);
                    }
                }
            }
            int tot;
            int ex = block_excl_scan(cnt, s_w, &tot);
            int4 rk;
            rk.x = keep[0] ? ex : -1; ex += keep[0];
            rk.y = keep[1] ? ex : -1; ex += keep[1];
            rk.z = keep[2] ? ex : -1; ex += keep[2];
            rk.w = keep[3] ? ex : -1;
            __stcg((int4*)(W.it_rank + base), rk);        // arrays are padded to a chunk multiple
            if (tid == 0) __stcg(W.cnt_keep + c, tot);
        }
        team_sync(T);
        if (keeper) RS.tp[3] = gtimer();

        // ================================================================= S3
        const int k_keep = scan_counts(W.cnt_keep, n_ich, s_prefix, s_w);
        const int remaining = cap - size;
        const int take = k_keep < remaining ? k_keep : remaining;
        const bool exhausted = k_keep > 0 && take == 0;                     // planner.py:233-235
        const int w_hit = __ldcg(&ctl->first_hit_w);
        bool found = false;
        int n_app = take;
        if (w_hit != 0x7fffffff) {
            const int rank_hit = s_prefix[w_hit / kChunk] + __ldcg(W.it_rank + w_hit);
            if (rank_hit < take) { found = true; n_app = rank_hit + 1; }   // planner.py:237-242
        }
        for (int c = T.rank; c < n_ich; c += T.ctas) {
            const int base = c * kChunk + tid * 4;
            const int cpre = s_prefix[c];
            if (cpre >= n_app) break;                                       // later chunks only hold larger ranks
            const int4 rk = __ldcg((const int4*)(W.it_rank + base));
            const int r4[4] = {rk.x, rk.y, rk.z, rk.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (r4[j] < 0) continue;
                const int rank = cpre + r4[j];
                if (rank >= n_app) continue;
                const int w = base + j, slot = size + rank;
                const int ipos = sorted ? __ldcg(W.pos_of + w) : w;
                const int par_slot = __ldcg(W.it_parent + w);
                const uint32_t pair = __ldcg(W.it_code + ipos) & ~kItemGoalBit;
                const int region = (int)(pair / (uint32_t)SUBS);
                R u[NU], dt; int S;
                sample_control<M, R>(P, h0, par_slot, w % lam, u, &dt, &S, nullptr, nullptr);
                copy_row<R, N>(states, slot, it_end, ipos);
                store_row<NU>(control, slot, u);
                dts[slot] = dt;
                W.parent[slot] = par_slot; W.region[slot] = region; W.tag[slot] = KPX_TAG_EXPAND;
                // planner.py:246: the region is available from now on; the estimate pass covers it from the next
                // iteration (build_est_list in the epilogue), until then its score word says "never"
                if (!((__ldcg(W.avail_bits + (region >> 5)) >> (region & 31)) & 1u))
                    atomicOr(W.avail_bits + (region >> 5), 1u << (region & 31));
            }
        }
        // estimate pass (decomposition.py:175-203) over the regions available before this append (est_ids, built in
        // the previous iteration's epilogue): scores and the leaf sums of NumPy's pairwise total
        estimate_leaves<R>(P, W, T, RS.n_est, (double*)&Scene<R>::coop());
        const int new_size = size + n_app;
        team_sync(T);
        if (keeper) RS.tp[4] = gtimer();

        // ================================================================= S4
        // sum of the scores in NumPy's pairwise order (bit-identical to the reference's `total`, and the same for
        // any team size); every CTA combines the leaf sums for itself
        double total;
        {
            const int na = RS.n_est;
            if (((na + 63) >> 6) <= kMaxProbes) {
                total = combine_leaves<false>(W.leaf_sum, na, (double*)(kpx_dyn_smem + Scene<R>::kCoop));
            } else {            // more leaves than a CTA holds in shared memory: CTA 0 combines in place and publishes
                if (T.rank == 0) {
                    const double t = combine_leaves<true>(W.leaf_sum, na, nullptr);
                    if (tid == 0) __stcg(&ctl->total_pub, t);
                }
                team_sync(T);
                total = __ldcg(&ctl->total_pub);
            }
        }
        {
            const int n_sch = (new_size + kChunk - 1) / kChunk;
            int my_open = 0;
            for (int c = T.rank; c < n_sch; c += T.ctas) {
                const int base = c * kChunk + tid * 4;
                int slots[4]; int cnt = 0;
                uint8_t newtag[4];
                uint8_t tg[4] = {0, 0, 0, 0}; int rg[4] = {0, 0, 0, 0};
                if (base + 3 < new_size) {
                    const uchar4 t4 = __ldcg((const uchar4*)(W.tag + base));
                    const int4 r4 = __ldcg((const int4*)(W.region + base));
                    tg[0] = t4.x; tg[1] = t4.y; tg[2] = t4.z; tg[3] = t4.w;
                    rg[0] = r4.x; rg[1] = r4.y; rg[2] = r4.z; rg[3] = r4.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (base + j < new_size) { tg[j] = __ldcg(W.tag + base + j); rg[j] = __ldcg(W.region + base + j); }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int s = base + j;
                    newtag[j] = KPX_TAG_EMPTY;
                    if (s >= new_size) continue;
                    uint8_t t = tg[j];
                    if (s < size) {
                        const double p = p_accept_of(rg[j], W.score, total, P.epsilon);
                        constexpr bool philox = M::kRng == KPX_RNG_PHILOX;
                        const uint64_t hs = philox ? 0ull : slot_ext_hash(h0, (uint64_t)s, 0ull);
                        if (t == KPX_TAG_EXPAND) {                                     // phase A, planner.py:219-225
                            const double ud = philox ? keyed_uniform_of<KPX_RNG_PHILOX>(h0, (uint64_t)s, 0ull, PH_DEMOTE)
                                                     : unit53(draw_u64(mix64(hs ^ (uint64_t)PH_DEMOTE), 0));
                            if (ud >= p) t = KPX_TAG_OPEN;
                        }
                        if (t == KPX_TAG_OPEN) {                                       // phase C, planner.py:251-257
                            const double up = philox ? keyed_uniform_of<KPX_RNG_PHILOX>(h0, (uint64_t)s, 0ull, PH_PROMOTE)
                                                     : unit53(draw_u64(mix64(hs ^ (uint64_t)PH_PROMOTE), 0));
                            if (up < p) t = KPX_TAG_EXPAND;
                        }
                    } else {
                        t = KPX_TAG_EXPAND;                                            // appended this iteration
                    }
                    newtag[j] = t;
                    if (t == KPX_TAG_EXPAND) slots[cnt++] = s; else ++my_open;
                }
                if (base + 3 < new_size) {
                    __stcg((uchar4*)(W.tag + base), make_uchar4(newtag[0], newtag[1], newtag[2], newtag[3]));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) if (base + j < new_size) __stcg(W.tag + base + j, newtag[j]);
                }
                int tot;
                const int ex = block_excl_scan(cnt, s_w, &tot);
                for (int j = 0; j < cnt; ++j) __stcg(W.e_local + c * kChunk + ex + j, slots[j]);
                if (tid == 0) __stcg(W.cnt_expand + c, tot);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) my_open += __shfl_xor_sync(0xffffffffu, my_open, o);
            if ((tid & 31) == 0 && my_open) atomicAdd(&ctl->cnt_open[par], my_open);
        }
        if (keeper) {
            __stcg(&ctl->first_hit_w, 0x7fffffff);
            __stcg(&ctl->unit_next, 0u);
            __stcg(&ctl->n_todo, 0u);
            for (int b = 0; b < kBins; ++b) __stcg(W.bin_cursor + b, 0u);
            atomicAdd(&ctl->sum_items, (unsigned long long)items);
            const double el = (double)(gtimer() - RS.t_start) * 1e-9;
            int stop = 0;
            if (!(el < A.t_max_s)) stop = KPX_TIMEOUT;                               // planner.py:282
            if (A.stop_flag && *((volatile const uint32_t*)A.stop_flag)) stop = KPX_STOPPED;
            if (!stop && A.handoff_at > 0 && *((volatile const unsigned int*)A.idle) >= (unsigned)A.handoff_at) stop = KPX_HANDOFF;
            if (stop) ctl->stop = stop;
        }
        team_sync(T);
        if (keeper) RS.tp[5] = gtimer();

        // ================================================= epilogue of the iteration
        // regions made available by this append join the estimate pass from the next iteration on (planner.py:246)
        const int n_est_next = build_est_list(W, T, RG, s_prefix, s_w);
        int ve = scan_counts(W.cnt_expand, (new_size + kChunk - 1) / kChunk, s_prefix, s_w);
        if (ve == 0) {
            // rescue rule (planner.py:259-265): OPEN slot with max p_accept, lowest slot on ties
            unsigned long long best = 0ull;
            for (long long s = ttid; s < new_size; s += tthreads) {
                const double p = p_accept_of(__ldcg(W.region + s), W.score, total, P.epsilon);
                const unsigned long long b = (unsigned long long)__double_as_longlong(p);   // p > 0: bits are ordered
                best = b > best ? b : best;
            }
            atomicMax(&ctl->rescue_key, best);
            team_sync(T);
            const unsigned long long kmax = __ldcg(&ctl->rescue_key);
            for (long long s = ttid; s < new_size; s += tthreads) {
                const double p = p_accept_of(__ldcg(W.region + s), W.score, total, P.epsilon);
                if ((unsigned long long)__double_as_longlong(p) == kmax) { atomicMin(&ctl->rescue_slot, (int)s); break; }
            }
            team_sync(T);
            if (keeper) {
                const int s = __ldcg(&ctl->rescue_slot);
                W.tag[s] = KPX_TAG_EXPAND;
                const int c = s / kChunk;
                W.e_local[c * kChunk] = s; W.cnt_expand[c] = 1;
                ctl->rescue_key = 0ull; ctl->rescue_slot = 0x7fffffff;
                atomicAdd(&ctl->cnt_open[par], -1);
            }
            team_sync(T);
            ve = scan_counts(W.cnt_expand, (new_size + kChunk - 1) / kChunk, s_prefix, s_w);
        }
        if (keeper) {   // IterationTrace (planner.py:290-296)
            const int nt = __ldcg(&ctl->n_trace);
            if (nt < A.max_trace) {
                kpx_trace tr;
                tr.iteration = it; tr.branching = lam; tr.ve_size = items / lam; tr.vo_size = __ldcg(&ctl->cnt_open[par]);
                tr.attempted = items; tr.valid = __ldcg(&ctl->cnt_valid[par]); tr.staged = k_keep; tr.appended = n_app;
                RS.tp[6] = gtimer();
                tr.tree_size = new_size; tr.elapsed_ms = (double)(RS.tp[6] - RS.t_start) * 1e-6;
                for (int ph = 0; ph < 6; ++ph) tr.phase_ms[ph] = (double)(RS.tp[ph + 1] - RS.tp[ph]) * 1e-6;
                W.trace[nt] = tr;
                ctl->n_trace = nt + 1;
            }
            ctl->cnt_open[par] = 0; ctl->cnt_valid[par] = 0;
            ctl->n_items_last = items; ctl->n_keep_last = k_keep; ctl->lam_last = lam; ctl->last_sorted = sorted ? 1 : 0;
        }
        __syncthreads();                        // every thread is done with this iteration's state
        if (tid == 0) {
            RS.size = new_size; RS.total_prev = total; RS.ve = ve; RS.n_est = n_est_next;
            if (found) { RS.status = KPX_SOLVED; RS.solution_slot = new_size - 1; }              // planner.py:297-303
            else if (exhausted) {
                // adaptive capacity (Remark 1): the arena was reserved for P.t_e nodes, so raising
                // the capacity in effect by the constant multiple costs nothing -- no reallocation, no copy
                if (P.t_e_growth > 1.0 && cap < (int)P.t_e) {
                    const long long grown = (long long)((double)cap * P.t_e_growth);
                    RS.cap = grown < P.t_e ? (int)grown : (int)P.t_e;
                    ctl->growths = __ldcg(&ctl->growths) + 1;
                } else RS.status = KPX_CAPACITY_EXHAUSTED;
            }
        }
        __syncthreads();
    }
}

// ---- results of a run: chain walk, packet, per-query record (keeper thread) -------------------------------
template <class M, class R>
__device__ __forceinline__ void finish_query(const PlanArgs<R>& A, const Workspace& W, const Team& T, const RunState& RS,
                                             kpx_query_result* res_out, long long query_index) {
    KPX_PHASE_LOCALS
    // ------------------------------------------------------------------ results
    if (keeper) {
        const int size = RS.size, it = RS.it, status = RS.status, solution_slot = RS.solution_slot;
        ctl->size = size; ctl->iteration = it; ctl->status = status; ctl->solution_slot = solution_slot;
        ctl->total_prev = RS.total_prev; ctl->ve = RS.ve; ctl->n_est = RS.n_est; ctl->cap = RS.cap;
        ctl->elapsed_ns = gtimer() - RS.t_start;
        if (status == KPX_HANDOFF && A.susp_out)
            A.susp_out[atomicAdd(A.n_susp_out, 1u)] = make_int2(T.ws_index, (int)query_index);
        int len = 0;
        if (status == KPX_SOLVED) {
            // parent chain (planner.py:325-336), written root-first
            int s = solution_slot;
            while (s != 0 && len < A.max_chain) { s = __ldcg(W.parent + s); ++len; }
            if (s != 0) len = -1;                   // chain longer than the buffer: caller falls back to snapshot
            double* c_start = W.chain_start; double* c_ctrl = W.chain_control; double* c_dt = W.chain_dt;
            if (res_out && A.b_chain_start) {
                c_start = A.b_chain_start + (size_t)query_index * A.max_chain * N;
                c_ctrl = A.b_chain_control + (size_t)query_index * A.max_chain * NU;
                c_dt = A.b_chain_dt + (size_t)query_index * A.max_chain;
            }
            if (len > 0 && c_start) {
                s = solution_slot;
                for (int i = len - 1; i >= 0; --i) {
                    const int par_s = __ldcg(W.parent + s);
                    for (int d = 0; d < N; ++d) c_start[(size_t)i * N + d] = (double)__ldcg(states + (size_t)par_s * Row<R, N>::kStride + d);
                    for (int q = 0; q < NU; ++q) c_ctrl[(size_t)i * NU + q] = (double)__ldcg(control + (size_t)s * Row<R, NU>::kStride + q);
                    c_dt[i] = (double)__ldcg(dts + s);
                    if (!res_out && W.chain_slot) W.chain_slot[i] = s;
                    s = par_s;
                }
                if (!res_out && W.chain_end)
                    for (int d = 0; d < N; ++d) W.chain_end[d] = (double)__ldcg(states + (size_t)solution_slot * Row<R, N>::kStride + d);
            }
            for (int i = 0; i < A.n_peers; ++i) { *((volatile uint32_t*)A.peer_flags[i]) = 1u; }
            if (A.n_peers) __threadfence_system();
        }
        ctl->chain_len = len;
        if (!res_out && W.packet) {       // packed result for the single-plan API
            ResultPacket* pk = W.packet;
            const int m = len < kPacketSegs ? len : kPacketSegs;
            for (int i = 0; i < m; ++i) {
                pk->seg_dt[i] = W.chain_dt[i]; pk->seg_slot[i] = W.chain_slot[i];
                for (int q = 0; q < NU; ++q) pk->seg_control[i][q] = W.chain_control[(size_t)i * NU + q];
                for (int d = 0; d < N; ++d) pk->seg_start[i][d] = W.chain_start[(size_t)i * N + d];
            }
            if (len > 0) for (int d = 0; d < N; ++d) pk->end_state[d] = W.chain_end[d];
        }
        ctl->t_end = gtimer();
        if (!res_out && W.packet) W.packet->ctl = *ctl;
        if (res_out) {
            kpx_query_result r;
            r.status = status; r.iterations = it; r.tree_size = size; r.solution_slot = solution_slot;
            r.chain_len = len; r.device_ms = (double)(ctl->t_end - __ldcg(&ctl->t_begin)) * 1e-6;
            r.checked = 0; r.check_code = 0;        // filled by kpx_batch_validate
            r.items = __ldcg(&ctl->sum_items); r.substeps = __ldcg(&ctl->sum_substeps); r.points = __ldcg(&ctl->sum_points); r.boxsteps = __ldcg(&ctl->sum_boxsteps);
            r.free_items = __ldcg(&ctl->sum_free); r.capacity = RS.cap;
            *res_out = r;
        }
    }
}

// One query on one team.  The CTA-uniform run state lives in shared memory (RunState), each phase re-derives
// its locals from it, and nothing but the propagation loop's own registers is live across S1.
template <class M, class R>
__device__ KPX_RQ_ATTR void run_query(const PlanArgs<R>& A, const Workspace& W, const Team& T, const QueryIn& Q,
                                      kpx_query_result* res_out, long long query_index, RunState& RS, int* s_prefix,
                                      int* s_w, double* s_d, int* s_bin, int* s_scene) {
    if (*s_scene != Q.scene) {      // stage this query's obstacle set (boxes + occupancy tables); CTA-uniform
        __syncthreads();
        Scene<R>::stage(A.P, A.obs + (size_t)Q.scene * 8 * (size_t)A.P.n_obs, A.occ + (size_t)Q.scene * 2 * kOccCells);
        if (threadIdx.x == 0) *s_scene = Q.scene;
        __syncthreads();
    }
    if (!A.resume) reset_query<M, R>(A, W, T, Q);
    {   // run state out of Ctl (valid between launches: stepped runs, resume)
        Ctl* const ctl = W.ctl;
        const int size = __ldcg(&ctl->size);
        const int n_est = build_est_list(W, T, A.P.n_regions, s_prefix, s_w);   // fresh: the root's region
        const int ve = scan_counts(W.cnt_expand, (size + kChunk - 1) / kChunk, s_prefix, s_w);
        // Run clock (planner.py:282): the time this loop has been running, summed over the launches since the
        // reset, so a stepped / resumed run does not count the host's idle time.  A launch that continues a run
        // which a time-out or a race peer stopped carries on (the caller asked for more); a run that has already
        // used up t_max -- t_max = 0 on a fresh query included -- ends before its first iteration, as the
        // reference's `while elapsed < t_max` does.  Every CTA of the team evaluates the same words.
        const unsigned long long elapsed0 = A.resume ? __ldcg(&ctl->elapsed_ns) : 0ull;
        int status = __ldcg(&ctl->status);
        if (A.resume && (status == KPX_TIMEOUT || status == KPX_STOPPED || status == KPX_HANDOFF)) status = KPX_RUNNING;
        if (status == KPX_RUNNING && !((double)elapsed0 * 1e-9 < A.t_max_s)) status = KPX_TIMEOUT;
        if (threadIdx.x == 0) {
            RS.size = size; RS.it = __ldcg(&ctl->iteration); RS.status = status;
            RS.solution_slot = __ldcg(&ctl->solution_slot); RS.total_prev = __ldcg(&ctl->total_prev);
            RS.ve = ve; RS.iters = 0; RS.n_est = n_est; RS.cap = __ldcg(&ctl->cap);
            RS.claim_tag = __ldcg(&ctl->epoch_used) << A.claim_shift;
            unsigned long long t_start = 0;     // run clock origin; only the keeper thread uses it
            if (T.rank == 0) {
                t_start = gtimer() - elapsed0;
                // (a resumed launch finds ctl->stop cleared by the host: kpx_plan_run)
                if (A.resume && __ldcg(&ctl->t_reset_done) == 0) { ctl->t_reset_done = t_start; ctl->t_begin = t_start; }  // loaded state
            }
            RS.t_start = t_start;
        }
        __syncthreads();
    }
    while (iteration_head<M, R>(A, W, T, Q, RS, s_prefix, s_bin)) {
        s1_propagate<M, R>(A, W, Q, RS, T.rank, T.ctas, s_prefix, s_bin);
        team_sync(T);
        if (T.rank == 0 && threadIdx.x == 0) RS.tp[2] = gtimer();
        iteration_tail<M, R>(A, W, T, Q, RS, s_prefix, s_w, s_d);
    }
    finish_query<M, R>(A, W, T, RS, res_out, query_index);
}

enum { KPX_THROUGHPUT = 0, KPX_LATENCY = 1 };
template <class M, class R, int V> struct MinBlocks {
    static constexpr bool kDI = M::ID == KPX_MODEL_DI6 || M::ID == KPX_MODEL_STACKED_DI;
    static constexpr int f32 = M::N <= 6 ? (kDI ? (V == KPX_LATENCY ? KPX_MINS_F32_DI : KPX_MINB_F32_DI)
                                               : (V == KPX_LATENCY ? KPX_MINS_F32_TRIG6 : KPX_MINB_F32_TRIG6))
                                         : (M::N <= 12 ? (V == KPX_LATENCY ? KPX_MINS_F32_MID : (kDI ? KPX_MINB_F32_DI12 : KPX_MINB_F32_MID))
                                                       : (V == KPX_LATENCY ? 1 : KPX_MINB_F32_BIG));
    static constexpr int value = sizeof(R) == 4 ? f32 : (M::N <= 6 ? 2 : 1);
};

template <class M, class R, int V>
__global__ void __launch_bounds__(kBlock, MinBlocks<M, R, V>::value) plan_kernel(const __grid_constant__ PlanArgs<R> A) {
    int* s_prefix = (int*)(kpx_dyn_smem + Scene<R>::bytes(A.P.n_obs));    // [max_chunks + 1], after the scene
    __shared__ int s_w[kBlock / 32 + 1];
    __shared__ double s_d[kBlock / 32];
    __shared__ int s_q;
    __shared__ int s_bin[4 * kBins];      // S0: local histogram | CTA base | local fill | global bin start
    __shared__ int s_scene;               // obstacle set staged in shared memory (queries name theirs: QueryIn::scene)
    if (threadIdx.x == 0) s_scene = -1;
    __syncthreads();

    Team T;
    T.ctas = A.team_ctas;
    const int team_id = blockIdx.x / A.team_ctas;
    T.rank = blockIdx.x - team_id * A.team_ctas;
    if (team_id >= A.n_teams) return;
    __shared__ RunState s_rs;
    __shared__ Workspace s_ws;            // CTA-uniform: one copy in shared memory instead of ~60 registers per thread
    int2 handed = make_int2(team_id, 0);  // hand-off stage: (workspace, query) this team continues
    if (A.resume_in) {
        if ((unsigned)team_id >= __ldcg(A.n_resume_in)) {            // nothing left for this team
            if (T.rank == 0 && threadIdx.x == 0 && A.idle) atomicAdd(A.idle, 1u);
            return;
        }
        handed = __ldcg(A.resume_in + team_id);
        if (A.handoff_at > 0 && __ldcg(A.n_resume_in) <= (unsigned)A.pass_on_below) {
            if (T.rank == 0 && threadIdx.x == 0) A.susp_out[atomicAdd(A.n_susp_out, 1u)] = handed;
            return;
        }
    }
    T.ws_index = handed.x;
    if (threadIdx.x == 0) s_ws = A.ws[handed.x];
    __syncthreads();
    const Workspace& W = s_ws;
    T.bar = W.bar;

    if (A.resume_in) {
        run_query<M, R>(A, W, T, A.queries[handed.y], A.results + handed.y, handed.y, s_rs, s_prefix, s_w, s_d, s_bin, &s_scene);
        if (T.rank == 0 && threadIdx.x == 0 && A.idle) atomicAdd(A.idle, 1u);
        return;
    }

    if (A.queue == nullptr) {       // single query bound to team 0 (plan handle: stepped / resumable)
        run_query<M, R>(A, W, T, A.queries[0], A.results, 0, s_rs, s_prefix, s_w, s_d, s_bin, &s_scene);
        return;
    }
    for (;;) {                      // batch: teams pull queries until the queue is drained
        if (T.ctas == 1) {
            if (threadIdx.x == 0) s_q = (int)atomicAdd(A.queue, 1u);
            __syncthreads();
        } else {
            if (T.rank == 0 && threadIdx.x == 0) __stcg(&W.ctl->cur_query, (int)atomicAdd(A.queue, 1u));
            team_sync(T);
            if (threadIdx.x == 0) s_q = __ldcg(&W.ctl->cur_query);
            __syncthreads();
            team_sync(T);           // everyone has read the slot before reset rewrites it
        }
        const int q = s_q;
        __syncthreads();
        if (q >= A.n_queries) {
            if (T.rank == 0 && threadIdx.x == 0 && A.idle) atomicAdd(A.idle, 1u);
            return;
        }
        run_query<M, R>(A, W, T, A.queries[q], A.results + q, q, s_rs, s_prefix, s_w, s_d, s_bin, &s_scene);
        team_sync(T);
    }
}

// ---- stand-alone propagation batch: the drop-in for _kernel.propagate_batch -------------
template <class R>
struct BatchArgs {
    Params<R> P;
    const R* obs;              // device boxes [n_obs][8]
    const uint32_t* occ;       // device occupancy masks
    const double* states;      // (rows, n) f64 row-major, as the reference passes it
    const long long* e_slots;  // (m)
    long long items; int lam;
    unsigned long long seed, iteration;
    uint8_t* o_valid; long long *o_region, *o_sub; double *o_end, *o_control, *o_dt, *o_accept;
    long long *o_substeps, *o_points;
};

template <class M, class R>
__global__ void __launch_bounds__(kBlock) batch_kernel(const __grid_constant__ BatchArgs<R> A) {
    constexpr int N = M::N, NU = M::NU;
    Scene<R>::stage(A.P, A.obs, A.occ);
    const uint64_t h0 = iter_key(M::kRng, A.seed, A.iteration);
    // whole warps iterate together (integrate_and_map is warp-synchronous); lanes past the end idle
    for (long long base = (long long)blockIdx.x * kBlock; base < A.items; base += (long long)gridDim.x * kBlock) {
        const long long w = base + threadIdx.x;
        const bool active = w < A.items;
        long long slot = 0; int ext = 0, S = 0;
        R u[NU], dt = (R)0, x0[N]; double u64v[NU], dt64 = 0.0;
#pragma unroll
        for (int d = 0; d < N; ++d) x0[d] = (R)0;
#pragma unroll
        for (int j = 0; j < NU; ++j) { u[j] = (R)0; u64v[j] = 0.0; }
        if (active) {
            const long long i = w / A.lam;
            ext = (int)(w - i * A.lam);
            slot = A.e_slots[i];
            // the reference hashes the 64-bit slot; planner slots always fit 31 bits
            sample_control<M, R>(A.P, h0, (int)slot, ext, u, &dt, &S, u64v, &dt64);
#pragma unroll
            for (int d = 0; d < N; ++d) x0[d] = (R)A.states[slot * N + d];
        }
        ItemOut<R, N> o;
        integrate_and_map<M, R>(A.P, active, x0, u, dt, S, o);
        if (!active) continue;
#pragma unroll
        for (int d = 0; d < N; ++d) A.o_end[w * N + d] = (double)o.end[d];
#pragma unroll
        for (int j = 0; j < NU; ++j) A.o_control[w * NU + j] = u64v[j];
        A.o_dt[w] = dt64;
        A.o_valid[w] = o.valid ? 1 : 0;
        A.o_region[w] = o.region;
        A.o_sub[w] = o.sub;
        A.o_accept[w] = keyed_uniform_of<M::kRng>(h0, (uint64_t)slot, (uint64_t)ext, PH_ACCEPT);
        if (A.o_substeps) A.o_substeps[w] = o.substeps;
        if (A.o_points) A.o_points[w] = o.points;
    }
}

}  // namespace kpx
