// kernels_sparse.cuh -- work-efficient refinement loop (default mode).
//
// Same rounds, same Priority winners as the dense loop in kernels.cuh, but a
// round only touches what its splitter C can affect:
//
//   phase A  (mark)   the members of C -- a contiguous range of `members`,
//            the state permutation grouped by block -- mark the slots of
//            their in-edges (reverse CSR).  In-edges are spread over the
//            lanes of a warp (a warp scan of the members' in-degrees), mark
//            bits are fire-and-forget reductions, and each source
//            block is registered once in the touched-block lists.  One warp
//            clears C in the hierarchical unstable set and finds C's
//            successor meanwhile.
//   phase B  (split)  every touched block B (leader l) compares each member's
//            slot vector with l's (bcrp.py:260-265 / rcpp.py:200), elects the
//            minimum split state w (Priority, bcrp.py:269-271), moves split
//            members to the tail of B's range, which becomes block w, and
//            raises l, w (and C for BCRP, bcrp.py:282).  Blocks of <= 32
//            members are finished by one warp; larger ones use a second
//            grid-wide sub-phase for the compaction.
//
// Work per round is O(|C| + in(C) + sum of touched block sizes) instead of
// O(n + m); two grid barriers per round (three when a touched block has
// more than 32 members).
#pragma once

#include "kernels.cuh"

namespace bisim {

// One CTA per SM.  512 threads leave 128 registers per thread (the loop
// spilled at the 64 of 1024-thread CTAs); measured per-round latency on the
// B200 (c1 / c2 / c3 / c4l / c5): 512 beats 1024 by 19 / 15 / 13 / 11 / 7 %,
// 256, 384 and 768 are within a few % or slower on c5.
#ifndef BISIM_SPARSE_THREADS
#define BISIM_SPARSE_THREADS 512
#endif
constexpr int kSparseThreads = BISIM_SPARSE_THREADS;
#ifndef BISIM_SPARSE_PER_SM
#define BISIM_SPARSE_PER_SM 1
#endif
constexpr int kSparsePerSm = BISIM_SPARSE_PER_SM;  // persistent CTAs per SM
constexpr int kMaxShards = 8;         // replicas of the transition-sharded mode

// Grid barrier: one monotonic arrival counter; CTA leaders add with
// acq_rel semantics and spin (ld.acquire) until it reaches this barrier's
// target.  __syncthreads on both sides extends the ordering to the CTA
// (cumulative release/acquire).  Measured at ~1.3 us on the B200
// (tools/barrier_bench.cu), the floor of a grid-wide round trip.
struct GridBarrier {
    unsigned count;
    unsigned pad[31];
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Back-off between two polls of a barrier / arrival record (ns): fewer
// acquire loads queue on the record's L2 line while the arrivals land there
// (A/B: 32 ns c5 -0.5 %, c2 +0.2 %, c1 +0.1 %; 100 ns c5 -0.2 %).
#ifndef BISIM_POLL_NS
#define BISIM_POLL_NS 32
#endif

__device__ __forceinline__ void grid_barrier(GridBarrier* gb, unsigned& gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned target = (gen + 1) * gridDim.x;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&gb->count) : "memory");
        while ((int)(ld_acquire_u32(&gb->count) - target) < 0) {
        }
    }
    ++gen;
    __syncthreads();
}

// Team barrier plus a control snapshot: after the barrier, thread 0 of each
// CTA runs snap() (reading the round's control words once per CTA into
// shared memory) before the CTA is released, so the 1024 threads of a CTA
// never all load the same global words.  solo: the team is this CTA alone.
template <typename F>
__device__ __forceinline__ void team_barrier(bool solo, GridBarrier* gb, unsigned& gen, F&& snap) {
    team_barrier(solo, gb, gen, [] {}, snap);
}

// ... with pre(): run by warp 0 after the CTA has synchronised and before
// the CTA arrives (its writes are released with the arrival).
template <typename G, typename F>
__device__ __forceinline__ void team_barrier(bool solo, GridBarrier* gb, unsigned& gen, G&& pre, F&& snap) {
    __syncthreads();
    if (threadIdx.x < 32) pre();
    if (threadIdx.x == 0) {
        if (!solo) {
            const unsigned target = (gen + 1) * gridDim.x;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&gb->count) : "memory");
            while ((int)(ld_acquire_u32(&gb->count) - target) < 0) {
            }
        }
        snap();
    }
    if (!solo) ++gen;
    __syncthreads();
}

struct SCtrl {
    int32_t C0;                         // entry-time splitter
    int32_t done;
    int32_t error;
    int32_t pad0;
    int64_t round;
    int64_t guard_count;
    int32_t next_min[2];                // min raised label, by round parity
    int32_t succ[2];                    // successor of C in unstable \ {C}
    int2 succ_range[2];                 // brange of that successor, read in phase A
    int32_t n_small[2];                 // touched blocks of <= 32 members
    int32_t pad1[2];
    unsigned long long big_pack[2];     // (#big touched blocks << 32) | #32-member chunks
    unsigned long long big_pack4[2];    // same for the 128-member chunk layout
    unsigned long long work_edges;      // sum of in(C)
    unsigned long long work_members;    // sum of touched-block sizes
    int32_t heavy[2];                   // round touched a block of > 1 member
    int32_t csplit[2];                  // the splitter's own block split this round
    int32_t nontriv[2];                 // skip step: least non-trivial candidate
    int32_t skipcnt[2];                 // skip step: rounds retired
    int32_t skip_next[2];               // skip step: splitter after the window
    unsigned long long skipped_rounds;  // statistics
    // solo stretches (kernels_loop.cuh)
    unsigned wake;                      // hand-overs from CTA 0 back to the grid
    unsigned parked;                    // park acknowledgements of the other CTAs
    int32_t stop;                       // CTA 0 finished during a solo stretch
    int32_t items_last;                 // phase-B work items of the last round
    int32_t pub_try_skip, pub_cooldown, pub_backoff, pad2;
    int64_t pub_skips;
    // End-of-round barrier record of a grid round, by round parity (see
    // end_barrier in kernels_loop.cuh): [0] arrivals; [1] min over the
    // round's raised labels (l << 1) and the successor of C (s << 1 | 1);
    // [2] the successor's member range start | heavy << 31; [3] its size |
    // C-split << 31.  Pollers read all four words with one 16-byte acquire
    // load, so the next splitter comes with the barrier itself.
    alignas(16) unsigned brec[2][4];
    // Mid-round (phase A -> B) barrier record, by parity: [0] arrivals,
    // [1] small touched blocks registered, [2..3] the 64-bit big-block
    // counter (#big blocks << 32 | #32-member chunks) -- the registration
    // atomics work on these words, and one 16-byte acquire load returns
    // them with the last arrival.
    alignas(16) unsigned arec[2][4];
};
constexpr unsigned kRecFlag = 1u << 31;

// Window of unstable labels examined by one skip step (see k_refine_sparse).
constexpr int32_t kSkipSpan = 32768;
constexpr int32_t kSkipMaxEdges = 256;
#ifndef BISIM_KWIDE
#define BISIM_KWIDE 4
#endif
constexpr int kWide = BISIM_KWIDE;  // members per lane in the wide big-block chunk layout (kernels_big.cuh)

// Per-label split record of a big touched block, 16 bytes: the one-pass
// packed arrival word (kernels_big.cuh) and the new-leader minimum
// (red.min).  A one-pass poller reads
// arrival word and minimum with ONE 16-byte acquire load: the arrivals'
// release orders each CTA's red.min before its add, so the load that sees
// the last arrival carries the final minimum (no dependent load after it).
struct alignas(16) SplitRec {
    unsigned long long arr;
    int32_t smin;
    int32_t pad;
};

// A member record carries what the phases read right after the member id,
// so one 16-byte load replaces two dependent ones: (state u, slot base
// off[u] (BCRP; unused for RCPP), in-edge range [e0, e1) of u in the
// reverse CSR).  Records move with their state when a block is compacted.
using MemberRec = int4;

struct SparseParams {
    int32_t n;
    int32_t A;
    int32_t reflag_c;
    int32_t has_guard;
    int64_t max_supersteps;
    int64_t round_limit;
    int64_t splits_cap;
    const int32_t* __restrict__ off;       // BCRP slot offsets (n+1)
    const int32_t* __restrict__ rev_ptr;   // reverse CSR row pointers (n+1)
    const int2* __restrict__ rev;          // BCRP in-edges: (slot, source)
    const int32_t* __restrict__ rev_src;   // RCPP in-edges: source (= slot)
    int32_t* block;
    int4* members;      // member records grouped by block (see MemberRec)
    int2* brange;       // (start, size) of block `label` in members (valid for leaders)
    uint32_t* mark;     // L-bit mark bitmap
    uint32_t* tblock;   // n-bit: block label registered this round
    uint32_t* U0;       // unstable labels, 3-level summary (1 bit per 1024 / 1M)
    uint32_t* U1;
    uint32_t* U2;
    int32_t nw0, nw1, nw2;
    int32_t pad;
    int4* small_list;     // touched blocks of <= 32 members: (label, start, size | nrl << 6, leader slot base)
    int4* big_list;       // larger touched blocks: (label, start, size, first chunk)
    int32_t* big_base;    // first chunk of each big touched block (ascending)
    int4* big_list4;      // the same blocks in the kWide chunk layout
    int32_t* big_base4;
    int2* big_info;       // leader slot base / slot count of each big_list entry
    int2* big_info4;      // same for big_list4
    int4* tmp;            // two-pass records, chunk-major (chunk ci at ci * 32 kWide): x = -1-state if split
    SplitRec* srec;       // per label: arrival word and new-leader minimum (kernels_big.cuh)
    int32_t* scnt;        // per label: two-pass split count (its own line: the pass-1 reductions
                          //   of a block's chunks would otherwise queue behind its minimum's)
    int32_t* kcur;        // per label: two-pass compaction cursors, kept / split members (separate
    int32_t* scur;        //   arrays: a chunk's two returning atomics must not queue on one line)
    int32_t* splits;
    SCtrl* ctrl;
    GridBarrier* bar;
    unsigned long long* trace;  // optional: 4 globaltimer stamps per round (CTA 0)
    int64_t trace_rounds;
    int32_t allow_skip;         // retire runs of no-op rounds in one step
    int32_t cta_minor;          // spread consecutive work items over SMs
    int32_t allow_solo;         // small rounds on CTA 0 alone (kernels_loop.cuh)
    int32_t force_mode_b;       // developer override of the phase-B layout (-1: automatic)
    int32_t solo_max_c;         // solo stretches: splitter size and previous-round work
    int32_t solo_max_items;     //   item limits (kernels_loop.cuh)
    int32_t batch_min_c;        // splitter size from which phase A registers blocks in one wave
    int32_t onepass_major;      // one-pass phase B: CTA-major item placement up to this many chunks per big block
    int32_t wide_major;         // ... and the wide layout when its chunks per big block are at most this
    int32_t prefetch_next;      // prefetch the likely next splitter's member records (1: in phase A) and in-edges (2: + phase B)
    int32_t wide_min;           // one-pass phase B takes the wide layout above this many 32-member chunks per big block
    // ---- transition-sharded mode (kernels_shard.cuh); nshard == 1 otherwise
    int32_t nshard;                       // replicas taking part in every round
    int32_t shard;                        // my index
    int64_t mark_stride;                  // words from the parity-0 to the parity-1 mark buffer
    int64_t bm_stride;                    // same for the tblock bitmap
    uint32_t* peer_mark[kMaxShards];      // every replica's mark buffer (parity 0)
    int32_t* xlist;                       // [2][n] blocks this replica registered first, by parity
    int32_t* peer_xlist[kMaxShards];
    int32_t* peer_xcnt[kMaxShards];       // [2] lengths of those lists
    unsigned* peer_xbar[kMaxShards];      // cross-replica arrival counters
    unsigned* go;                         // release word of the combined barrier (local)
    unsigned long long timeout_ns;        // give up a cross-replica wait after this long
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Developer trace (BISIM_TRACE): kTraceWords words per round, written by
// thread 0 of CTA 0: [0..3] round start / end of phase A / after the A
// barrier / after the B barrier, [4..7] counters, [8..12] phase-B steps of
// the one-pass path (tagged, CTA-synced, arrived, cursors synced, done) or
// [8..10] of the two-pass path (pass 1 done, mid barrier passed, pass 2
// done), [13] the round's phase-B mode, [14..15] batch phase A (warp 0's
// walk done, the CTA's walk done).
constexpr int kTraceWords = 16;
__device__ __forceinline__ void trace_at(const SparseParams& p, int64_t round, int k) {
    if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && round < p.trace_rounds)
        p.trace[round * kTraceWords + k] = globaltimer();
}

// ---- hierarchical unstable set --------------------------------------------

// Phase-B raises are combined per CTA in shared memory and flushed once at
// the end of the phase (raise_flush): the summary levels U1/U2 have few
// words (U2 is one word below 32M states) and next_min / splits[round] are
// single words, so per-raise global reductions from thousands of split
// blocks serialised in L2 on a handful of addresses.
constexpr int kU1Smem = 2048;  // U1 words kept per CTA (n <= 2^26); beyond, U1 raises go to global
__shared__ uint32_t s_u1[kU1Smem];
__shared__ int32_t s_u1_dirty[kU1Smem];  // U1 words that became non-zero this phase
__shared__ int32_t s_ndirty;
__shared__ uint32_t s_u2[32];
__shared__ int32_t s_nmin;
__shared__ int32_t s_nsplit;
__shared__ int32_t s_nmin_round;  // raised minimum of the phase just flushed
__shared__ int32_t s_csplit;       // this CTA split the splitter's own block this phase
__shared__ int32_t s_csplit_round;

// Round control of a solo stretch (CTA 0 alone): the registration counters,
// the successor and its range, the previous round's item count live in
// shared memory, so a solo round's phases hand over without global round
// trips (kernels_loop.cuh).
__shared__ int32_t s_ctr_nsmall;
__shared__ unsigned long long s_ctr_big, s_ctr_big4;
__shared__ int32_t s_ctr_heavy;
__shared__ int32_t s_succ;
__shared__ int2 s_succ_range;
__shared__ int32_t s_items_last;

__device__ __forceinline__ void raise_init() {
    for (int k = threadIdx.x; k < kU1Smem; k += blockDim.x) s_u1[k] = 0u;
    if (threadIdx.x < 32) s_u2[threadIdx.x] = 0u;
    if (threadIdx.x == 0) {
        s_nmin = 0x7fffffff;
        s_nsplit = 0;
        s_ndirty = 0;
        s_nmin_round = 0x7fffffff;
        s_csplit = s_csplit_round = 0;
        s_ctr_nsmall = 0;
        s_ctr_big = s_ctr_big4 = 0ull;
        s_ctr_heavy = 0;
        s_succ = 0x7fffffff;
        s_succ_range = make_int2(0, 0);
        s_items_last = 0x7fffffff;
    }
}

// Raise label x: U0 word in global memory, summary bits in the CTA's copy.
__device__ __forceinline__ void u_set(const SparseParams& p, int32_t x) {
    red_or(&p.U0[x >> 5], 1u << (x & 31));
    if (p.nw1 <= kU1Smem) {
        const int32_t w = x >> 15;
        if (!atomicOr(&s_u1[w], 1u << ((x >> 10) & 31))) s_u1_dirty[atomicAdd(&s_ndirty, 1)] = w;
    } else {
        red_or(&p.U1[x >> 15], 1u << ((x >> 10) & 31));
    }
    atomicOr(&s_u2[x >> 25], 1u << ((x >> 20) & 31));
}

// Warp 0, after a __syncthreads that follows every raise of the phase (the
// start of team_barrier): publish the CTA's summary bits, raised minimum and
// split count, and reset them.  Nothing to do for a CTA without a split.
__device__ __forceinline__ void raise_flush_warp0(const SparseParams& p, int cur, int64_t round) {
    const int lane = threadIdx.x & 31;
    const int32_t ns = s_nsplit;
    if (lane == 0) {
        s_nmin_round = ns ? s_nmin : 0x7fffffff;
        s_csplit_round = s_csplit;
        if (s_csplit) {
            red_or(&p.ctrl->brec[cur][3], kRecFlag);
            s_csplit = 0;
        }
    }
    if (!ns) return;
    const int32_t nd = s_ndirty;
    for (int k = lane; k < nd; k += 32) {
        const int32_t w = s_u1_dirty[k];
        red_or(&p.U1[w], s_u1[w]);
        s_u1[w] = 0u;
    }
    if (lane < p.nw2) {
        const uint32_t v = s_u2[lane];
        if (v) {
            red_or(&p.U2[lane], v);
            s_u2[lane] = 0u;
        }
    }
    __syncwarp();  // every lane has read s_nsplit / s_ndirty before lane 0 resets them
    if (lane == 0) {
        red_min_u32(&p.ctrl->brec[cur][1], (uint32_t)s_nmin << 1);
        if (round < p.splits_cap) red_add(&p.splits[round], ns);
        s_nmin = 0x7fffffff;
        s_nsplit = 0;
        s_ndirty = 0;
    }
    __syncwarp();
}

// Clear C and return its successor: the smallest unstable label > C (kBig
// if none).  One probe of C's 32-word chunk serves both (whole warp
// participates; no raises run concurrently in phase A).
__device__ int32_t u_next_warp(const SparseParams& p, int32_t from);
__device__ __forceinline__ int32_t u_clear_next_warp(const SparseParams& p, int32_t x) {
    const int lane = threadIdx.x & 31;
    const uint32_t bit = 1u << (x & 31);
    if (lane == 0) red_and(&p.U0[x >> 5], ~bit);
    const int32_t c = x >> 10;
    const int32_t wi = (c << 5) + lane;
    uint32_t v = wi < p.nw0 ? p.U0[wi] : 0u;
    if (wi == (x >> 5)) v &= ~bit;
    if (!__ballot_sync(kFull, v != 0u)) {  // the chunk is now empty
        const uint32_t cb = 1u << (c & 31);
        if (lane == 0) red_and(&p.U1[c >> 5], ~cb);
        const int32_t d = x >> 20;
        const int32_t wj = (d << 5) + lane;
        uint32_t v1 = wj < p.nw1 ? p.U1[wj] : 0u;
        if (wj == (c >> 5)) v1 &= ~cb;
        if (!__ballot_sync(kFull, v1 != 0u) && lane == 0) red_and(&p.U2[d >> 5], ~(1u << (d & 31)));
        return u_next_warp(p, (c + 1) << 10);
    }
    // successor inside the chunk: bits above x
    uint32_t sv = v;
    if (wi < (x >> 5)) sv = 0u;
    else if (wi == (x >> 5)) sv = (x & 31) == 31 ? 0u : (v & (~0u << ((x & 31) + 1)));
    const unsigned b = __ballot_sync(kFull, sv != 0u);
    if (b) {
        const int src = __ffs(b) - 1;
        const int32_t r = (wi << 5) + __ffs(sv) - 1;
        return __shfl_sync(kFull, r, src);
    }
    return u_next_warp(p, (c + 1) << 10);
}

// Smallest unstable label >= from (kBig if none); whole warp participates.
// Each probe reads 32 consecutive words of one level (1024 bits).
__device__ int32_t u_next_warp(const SparseParams& p, int32_t from) {
    const int lane = threadIdx.x & 31;
    const int64_t n = p.n;
    int64_t pos = from;
    while (pos < n) {
        {  // level 0: rest of pos's 1024-bit chunk
            const int64_t w_lo = pos >> 5;
            const int64_t wi = ((pos >> 10) << 5) + lane;
            uint32_t v = (wi < p.nw0 && wi >= w_lo) ? p.U0[wi] : 0u;
            if (wi == w_lo) v &= ~0u << (pos & 31);
            const unsigned b = __ballot_sync(kFull, v != 0u);
            if (b) {
                const int src = __ffs(b) - 1;
                const int32_t r = (int32_t)((wi << 5) + __ffs(v) - 1);
                return __shfl_sync(kFull, r, src);
            }
        }
        const int64_t c_from = (pos >> 10) + 1;
        {  // level 1: next non-empty chunk within the same 1M-label window
            const int64_t w_lo = c_from >> 5;
            const int64_t wi = ((c_from >> 10) << 5) + lane;
            uint32_t v = (wi < p.nw1 && wi >= w_lo) ? p.U1[wi] : 0u;
            if (wi == w_lo) v &= ~0u << (c_from & 31);
            const unsigned b = __ballot_sync(kFull, v != 0u);
            if (b) {
                const int src = __ffs(b) - 1;
                const int64_t c = (wi << 5) + __ffs(v) - 1;
                pos = __shfl_sync(kFull, c, src) << 10;
                continue;
            }
        }
        const int64_t d_from = (c_from >> 10) + 1;
        {  // level 2: next non-empty 1M-label window
            const int64_t w_lo = d_from >> 5;
            const int64_t wi = w_lo + lane;
            uint32_t v = wi < p.nw2 ? p.U2[wi] : 0u;
            if (wi == w_lo) v &= ~0u << (d_from & 31);
            const unsigned b = __ballot_sync(kFull, v != 0u);
            if (!b) return kBig;
            const int src = __ffs(b) - 1;
            const int64_t d = (wi << 5) + __ffs(v) - 1;
            pos = __shfl_sync(kFull, d, src) << 20;
        }
    }
    return kBig;
}

// ---- phase A helpers --------------------------------------------------------

// Register block b (first touch this round) in the touched lists; `reg`
// lanes of a warp register at once (warp-uniform call): one counter atomic
// and one `heavy` store per warp instead of one per block -- thousands of
// blocks are registered per round in the big rounds of c2/c1.
// What registration reads about block b: its member range and the leader's
// slot range.  Loaded while the test-and-set is in flight (the arrays only
// change in phase B).
struct BlockInfo {
    int2 r;
    int32_t ob, nb;
};
__device__ __forceinline__ BlockInfo block_info(const SparseParams& p, int32_t b) {
    BlockInfo i;
    i.r = p.brange[b];
    i.ob = p.off ? p.off[b] : b;
    i.nb = p.off ? p.off[b + 1] - i.ob : 1;
    return i;
}

__device__ __forceinline__ void register_blocks_warp(const SparseParams& p, int cur, bool reg, int32_t b,
                                                     BlockInfo bi, bool solo) {
    SCtrl* ctl = p.ctrl;
    // counters: the CTA's shared copies in a solo round, else the global
    // ones (separate code per address space: a generic-pointer atomic costs
    // the grid rounds a few percent)
    const int lane = threadIdx.x & 31;
    int2 r = make_int2(0, 0);
    int32_t ob = 0, nb = 0;
    if (reg) {
        r = bi.r;
        ob = bi.ob;
        nb = bi.nb;
    }
    const unsigned heavy = __ballot_sync(kFull, reg && r.y > 1);
    // the round's "touched a block of > 1 member" flag: per CTA in shared
    // memory, one red per CTA at the mid barrier (a red per registering warp
    // on the end-of-round record word queued thousands deep in c2's rounds,
    // and each CTA's arrival release waited for its own)
    if (heavy && lane == __ffs(heavy) - 1) s_ctr_heavy = 1;
    const unsigned small = __ballot_sync(kFull, reg && r.y <= 32);
    if (small) {
        const int ld = __ffs(small) - 1;
        int32_t base = 0;
        if (lane == ld)
            base = solo ? atomicAdd(&s_ctr_nsmall, __popc(small))
                        : (int32_t)atomicAdd(&ctl->arec[cur][1], (unsigned)__popc(small));
        base = __shfl_sync(kFull, base, ld);
        // (label, start, size | leader slot count << 6, leader slot base)
        if (reg && r.y <= 32)
            p.small_list[base + __popc(small & lanemask_lt())] = make_int4(b, r.x, r.y | (nb << 6), ob);
    }
    if (reg && r.y > 32) {
        const int32_t nch1 = (r.y + 31) >> 5, nch4 = (r.y + 32 * kWide - 1) / (32 * kWide);
        const unsigned long long d1 = (1ull << 32) | (unsigned long long)nch1;
        const unsigned long long d4 = (1ull << 32) | (unsigned long long)nch4;
        unsigned long long pk, pk4;
        if (solo) {
            pk = atomicAdd(&s_ctr_big, d1);
            pk4 = atomicAdd(&s_ctr_big4, d4);
        } else {
            pk = atomicAdd((unsigned long long*)&ctl->arec[cur][2], d1);
            pk4 = atomicAdd(&ctl->big_pack4[cur], d4);
        }
        const int32_t k = (int32_t)(pk >> 32), base = (int32_t)(pk & 0xffffffffu);
        const int32_t k4 = (int32_t)(pk4 >> 32), base4 = (int32_t)(pk4 & 0xffffffffu);
        p.big_list[k] = make_int4(b, r.x, r.y, base);
        p.big_base[k] = base;
        p.big_info[k] = make_int2(ob, nb);
        p.big_list4[k4] = make_int4(b, r.x, r.y, base4);
        p.big_base4[k4] = base4;
        p.big_info4[k4] = make_int2(ob, nb);
        SplitRec z;
        z.arr = 0ull;
        z.smin = kBig;
        z.pad = 0;
        p.srec[b] = z;
        p.scnt[b] = 0;
        p.kcur[b] = 0;
        p.scur[b] = 0;
    }
}

__device__ __forceinline__ void register_blocks_warp(const SparseParams& p, int cur, bool reg, int32_t b,
                                                     bool solo = false) {
    BlockInfo bi{};
    if (reg) bi = block_info(p, b);
    register_blocks_warp(p, cur, reg, b, bi, solo);
}

// Warp-aggregated test-and-set of bit x in bm; returns true in exactly one
// lane grid-wide per distinct x that was clear before this round.
__device__ __forceinline__ bool set_first(uint32_t* bm, int32_t x, bool active) {
    const int lane = threadIdx.x & 31;
    const unsigned same = __match_any_sync(kFull, active ? x : -1 - lane);
    const bool rep = active && lane == __ffs(same) - 1;
    uint32_t old = 0;
    if (rep) {
        const uint32_t bit = 1u << (x & 31);
        const uint32_t cur = ld_vol(&bm[x >> 5]);
        old = (cur & bit) ? cur : atomicOr(&bm[x >> 5], bit);
        return !(old & bit);
    }
    return false;
}

// CTA-level de-duplication of touched-block registrations: many in-edges of
// C usually share few source blocks, and thousands of warps hammering the
// same tblock words serialise in L2.  Only the first inserter of b in a CTA
// goes on to the grid-wide test-and-set.
#ifndef BISIM_SEEN
#define BISIM_SEEN 1024
#endif
constexpr int kSeen = BISIM_SEEN;  // a multiple of the CTA size

// 0: b already seen by this CTA this round; 1: first insertion; 2: table
// crowded (the global test-and-set decides).
__device__ __forceinline__ uint32_t seen_slot(int32_t b) {
    return ((uint32_t)b * 2654435761u) >> 22;  // 10-bit hash
}
__device__ __forceinline__ int cta_first(int32_t* seen, int32_t b) {
    uint32_t h = seen_slot(b);
#pragma unroll 1
    for (int probe = 0; probe < 16; ++probe) {
        const int32_t old = atomicCAS(&seen[h], -1, b);
        if (old == -1) return 1;
        if (old == b) return 0;
        h = (h + 1) & (kSeen - 1);
    }
    return 2;
}

// ---- phase B helpers --------------------------------------------------------

// Split test of member record r against its leader l (slot base ol, nrl
// slots: members share the leader's label set, hence its slot count,
// bcrp.py:16-19).
// tu: u has a marked slot this round; lb: the leader's slot bits (nrl <= 32).
template <bool IDENT>
__device__ __forceinline__ bool member_splits(const SparseParams& p, MemberRec r, int32_t l, bool tl,
                                              uint32_t lb, int32_t ol, int32_t nrl, bool& tu, int32_t& ou,
                                              int32_t& nr) {
    const int32_t u = r.x;
    if (IDENT) {
        tu = get_bit(p.mark, u);
        ou = u;
        nr = 1;
        return u != l && (tu != tl);
    }
    ou = r.y;
    nr = nrl;
    if (nr == 0) {
        tu = false;
        return false;
    }
    if (nr <= 32) {
        const uint32_t ub = get_bits(p.mark, ou, nr);
        tu = ub != 0u;
        return u != l && ub != lb;
    }
    tu = slots_any(p.mark, ou, nr);
    if (u == l || !(tu || tl)) return false;
    return slots_differ(p.mark, ou, ol, nr);
}

// Leader marks of a BCRP block: lb = its slot bits when nrl <= 32, tl = any.
template <bool IDENT>
__device__ __forceinline__ void leader_marks(const SparseParams& p, int32_t l, int32_t ol, int32_t nrl, bool& tl,
                                             uint32_t& lb) {
    if (IDENT) {
        tl = get_bit(p.mark, l);
        lb = tl ? 1u : 0u;
        return;
    }
    lb = (nrl > 0 && nrl <= 32) ? get_bits(p.mark, ol, nrl) : 0u;
    tl = nrl <= 32 ? lb != 0u : slots_any(p.mark, ol, nrl);
}

template <bool IDENT>
__device__ __forceinline__ void clear_member(const SparseParams& p, int32_t u, bool tu, int32_t ou,
                                             int32_t nr) {
    if (!tu) return;
    if (IDENT) {
        red_and(&p.mark[u >> 5], ~(1u << (u & 31)));
        return;
    }
    int32_t pos = ou, left = nr;
    while (left > 0) {
        const int32_t sh = pos & 31, len = min(left, 32 - sh);
        const uint32_t msk = (len == 32 ? ~0u : ((1u << len) - 1u)) << sh;
        red_and(&p.mark[pos >> 5], ~msk);
        pos += len;
        left -= len;
    }
}

__device__ __forceinline__ void raise_split(const SparseParams& p, int cur, int64_t round, int32_t l,
                                            int32_t w, int32_t C) {
    if (l == C) s_csplit = 1;
    u_set(p, l);
    u_set(p, w);
    int32_t lo = min(l, w);
    if (p.reflag_c) {  // BCRP: any split re-destabilises C (bcrp.py:282)
        u_set(p, C);
        lo = min(lo, C);
    }
    atomicMin(&s_nmin, lo);
    atomicAdd(&s_nsplit, 1);
    (void)cur;
    (void)round;
}

// A touched block of <= 32 members, finished by one warp.
template <bool IDENT>
__device__ int32_t process_small(const SparseParams& p, int cur, int64_t round, int32_t C, int4 e) {
    const int lane = threadIdx.x & 31;
    const int32_t l = e.x, bs = e.y, bz = e.z & 63;
    const bool valid = lane < bz;
    const MemberRec rec = valid ? p.members[bs + lane] : make_int4(-1, 0, 0, 0);
    const int32_t u = rec.x;
    // the leader's slot range came with the list entry (register_blocks_warp)
    const int32_t ol = IDENT ? l : e.w, nrl = IDENT ? 1 : (e.z >> 6);
    bool tl;
    uint32_t lb;
    leader_marks<IDENT>(p, l, ol, nrl, tl, lb);
    bool tu = false;
    int32_t ou = 0, nr = 0;
    const bool sp = valid && member_splits<IDENT>(p, rec, l, tl, lb, ol, nrl, tu, ou, nr);
    const unsigned bal = __ballot_sync(kFull, sp);
    if (bal) {
        const int32_t ns = __popc(bal);
        const int32_t keep = bz - ns;
        const int32_t w = __reduce_min_sync(kFull, sp ? u : kBig);
        const unsigned lt = lanemask_lt();
        const unsigned vmask = bz >= 32 ? kFull : ((1u << bz) - 1u);
        if (valid) {
            const int32_t np = sp ? bs + keep + __popc(bal & lt) : bs + __popc(~bal & vmask & lt);
            p.members[np] = rec;
            if (sp) p.block[u] = w;
        }
        if (lane == 0) {
            p.brange[l] = make_int2(bs, keep);
            p.brange[w] = make_int2(bs + keep, ns);
            raise_split(p, cur, round, l, w, C);
        }
    }
    __syncwarp();
    if (valid) clear_member<IDENT>(p, u, tu, ou, nr);
    if (lane == 0) red_and(&p.tblock[l >> 5], ~(1u << (l & 31)));
    return bz;
}

#include "kernels_big.cuh"

// ---- no-op rounds ------------------------------------------------------------

// Is the round whose splitter is c a no-op?  True when every in-edge source
// of c's members lies in a singleton block: singletons never split (a leader
// compares with itself), so the round changes nothing but unstable[c] --
// no split, no raised label, no BCRP re-raise (bcrp.py:267-283).  Answers
// false (the round then runs normally) for splitters of more than 32
// members or more than kSkipMaxEdges in-edges.
#ifndef BISIM_TRIV_G
#define BISIM_TRIV_G 4
#endif
constexpr int kTrivG = BISIM_TRIV_G;
template <bool IDENT>
__device__ __forceinline__ bool round_is_trivial(const SparseParams& p, int32_t c) {
    const int2 r = p.brange[c];
    if (r.y > 32) return false;
    int32_t budget = kSkipMaxEdges;
    for (int32_t i = 0; i < r.y; ++i) {
        const MemberRec mr = p.members[r.x + i];
        const int32_t e0 = mr.z, e1 = mr.w;
        if (e1 - e0 > budget) return false;
        budget -= e1 - e0;
        // kTrivG in-edges per step: their three dependent loads (reverse
        // edge, source block, block size) go out together
        for (int32_t e = e0; e < e1; e += kTrivG) {
            int32_t s[kTrivG], b[kTrivG];
#pragma unroll
            for (int k = 0; k < kTrivG; ++k) s[k] = e + k < e1 ? (IDENT ? p.rev_src[e + k] : p.rev[e + k].y) : -1;
#pragma unroll
            for (int k = 0; k < kTrivG; ++k) b[k] = s[k] >= 0 ? p.block[s[k]] : -1;
            bool single = true;
#pragma unroll
            for (int k = 0; k < kTrivG; ++k) single &= b[k] < 0 || p.brange[b[k]].y == 1;
            if (!single) return false;
        }
    }
    return true;
}

// ---- the persistent kernel ---------------------------------------------------

#include "kernels_shard.cuh"
#include "kernels_loop.cuh"

// ---- setup kernels -----------------------------------------------------------

__global__ void k_block_sizes(int32_t n, const int32_t* __restrict__ block, int32_t* bsize) {
    const int lane = threadIdx.x & 31;
    for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); s0 < n;
         s0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = s0 + lane;
        const int32_t b = s < n ? block[s] : -1 - lane;
        const unsigned g = __match_any_sync(kFull, b);
        if (s < n && lane == __ffs(g) - 1) atomicAdd(&bsize[b], __popc(g));
    }
}

__global__ void k_fill_members(int32_t n, const int32_t* __restrict__ block, int32_t* cursor,
                               const int32_t* __restrict__ off, const int32_t* __restrict__ rev_ptr,
                               MemberRec* members) {
    const int lane = threadIdx.x & 31;
    for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); s0 < n;
         s0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = s0 + lane;
        const int32_t b = s < n ? block[s] : -1 - lane;
        const unsigned g = __match_any_sync(kFull, b);
        const int leader = __ffs(g) - 1;
        int32_t base = 0;
        if (s < n && lane == leader) base = atomicAdd(&cursor[b], __popc(g));
        base = __shfl_sync(kFull, base, leader);
        if (s < n)
            members[base + __popc(g & lanemask_lt())] =
                make_int4((int32_t)s, off ? off[s] : 0, rev_ptr[s], rev_ptr[s + 1]);
    }
}

// brange[b] = (start, size) from the scanned starts and the sizes
__global__ void k_pack_ranges(int32_t n, const int32_t* __restrict__ start,
                              const int32_t* __restrict__ size, int2* brange) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x)
        brange[s] = make_int2(start[s], size[s]);
}

// U1 bit c <=> U0 words [32c, 32c+32) nonzero; U2 likewise over U1.
__global__ void k_summary(const uint32_t* __restrict__ lo, int32_t nlo, uint32_t* hi, int32_t nhi) {
    const int lane = threadIdx.x & 31;
    for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); c0 < (int64_t)nhi * 32;
         c0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = c0 + lane;  // chunk index = bit index in hi
        bool nz = false;
        for (int k = 0; k < 32 && !nz; ++k) {
            const int64_t w = c * 32 + k;
            if (w < nlo && lo[w]) nz = true;
        }
        const unsigned b = __ballot_sync(kFull, nz);
        if (lane == 0) hi[c0 >> 5] = b;
    }
}

// (label mask, slot base) of every state in one 16-byte record, so the
// reverse fill's random lookup by source costs one sector, not two (W == 1).
__global__ void k_pack_sinfo(int32_t n, const unsigned long long* __restrict__ lmask,
                             const int32_t* __restrict__ off, int4* sinfo) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long w = lmask[s];
        sinfo[s] = make_int4((int32_t)(w & 0xffffffffull), (int32_t)(w >> 32), off[s], 0);
    }
}

// |Act| <= 32: (label mask, slot base) in 8 bytes -- half the footprint of
// the random lookups (c5: 80 MB instead of 160 MB, mostly L2 hits).
__global__ void k_pack_sinfo2(int32_t n, const unsigned long long* __restrict__ lmask,
                              const int32_t* __restrict__ off, int2* sinfo2) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
        sinfo2[s] = make_int2((int32_t)(uint32_t)lmask[s], off[s]);
}

// mark slot of (source s, action a) from a packed record (bcrp.py:219)
__device__ __forceinline__ int32_t slot_of(int32_t s, int32_t a, const int4* __restrict__ sinfo,
                                           const int2* __restrict__ sinfo2) {
    if (sinfo2) {
        const int2 q = sinfo2[s];
        return q.y + __popc((uint32_t)q.x & ((1u << (a & 31)) - 1u));
    }
    const int4 q = sinfo[s];
    const unsigned long long w = ((unsigned long long)(uint32_t)q.y << 32) | (uint32_t)q.x;
    return q.z + __popcll(w & ((1ull << (a & 63)) - 1ull));
}

// Pack BCRP reverse edges (slot, source) for one 8-byte load per in-edge.
template <bool BCRP>
__global__ void k_rev_fill2(int32_t n, int64_t m, const int32_t* __restrict__ src,
                            const int32_t* __restrict__ act, const int32_t* __restrict__ dst,
                            const unsigned long long* __restrict__ lmask, const int32_t* __restrict__ off,
                            int32_t* cursor, int2* rev, int32_t* rev_src, int32_t lo, int32_t hi,
                            const int4* __restrict__ sinfo) {
    // only transitions with source in [lo, hi) (the whole range unless sharded)
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < m; i0 += stride) {
        const int64_t i = i0 + lane;
        int32_t t = -1 - lane, slot = 0, s = 0;
        bool in = false;
        if (i < m) {
            s = src[i];
            in = s >= lo && s < hi;
        }
        if (in) {
            t = dst[i];
            if (!BCRP) {
                slot = s;
            } else if (sinfo) {
                const int4 q = sinfo[s];
                const unsigned long long w = ((unsigned long long)(uint32_t)q.y << 32) | (uint32_t)q.x;
                slot = q.z + __popcll(w & ((1ull << (act[i] & 63)) - 1ull));
            } else {
                slot = off[s] + label_rank(lmask, n, s, act[i]);
            }
        }
        const LaneRun run = lane_run(t);
        int32_t base = 0;
        if (in && run.rank == 0) base = atomicAdd(&cursor[t], run.len);
        base = __shfl_sync(kFull, base, run.leader);
        if (in) {
            const int32_t at = base + run.rank;
            if (BCRP) rev[at] = make_int2(slot, s);
            else rev_src[at] = s;
        }
    }
}


// ---- reverse CSR fill in two bucketed passes ----------------------------------
//
// The one-pass fill (k_rev_fill2) scatters 8-byte in-edges to random
// positions of an m-entry array far larger than L2: every 32-byte sector is
// fetched and written back several times (~0.25 KB of DRAM traffic per
// transition).  Here transitions are first grouped by target bucket (a range
// of 2^shift targets) into a staging array laid out like rev itself (bucket
// b starts at rev_ptr[b << shift]), with one global reservation per (tile,
// bucket); the second pass walks the staging array in order, so the
// positions it scatters to lie in the one or two buckets being worked on --
// a few MB that stay in L2 until their sectors are complete.
constexpr int kBucketThreads = 512;
#ifndef BISIM_BUCKET_ITEMS
#define BISIM_BUCKET_ITEMS 8
#endif
constexpr int kBucketItems = BISIM_BUCKET_ITEMS;                        // transitions per thread per tile
constexpr int kBucketTile = kBucketThreads * kBucketItems;
constexpr int kMaxBuckets = 1024;

__global__ void k_bucket_init(int32_t n, int shift, int32_t nb, const int32_t* __restrict__ rev_ptr, int32_t* bcur) {
    for (int32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x)
        bcur[b] = rev_ptr[min((int64_t)b << shift, (int64_t)n)];
}

// Pass 1 over transitions [0, m) of (src, act, dst) -- a chunk of the input
// (the host path runs it per chunk while the next chunk is still being
// copied): stage (target, source, action) by target bucket.  Out-of-range
// targets and sources are skipped (k_indeg_checked / k_label_mask flag
// them, and the caller reads the flag before pass 2 uses anything).
//
// slot_here (the label sets are complete): the mark slot is computed here
// instead of the action, so pass 2 needs no per-source lookup (the random
// label-set read overlaps the tile's other loads better here).
template <typename TA = int32_t>
__global__ void __launch_bounds__(kBucketThreads) k_rev_bucket(
    int64_t m, const int32_t* __restrict__ src, const TA* __restrict__ act,
    const int32_t* __restrict__ dst, int shift, int32_t nb, int32_t* bcur, int4* stage, int32_t lo, int32_t hi,
    bool slot_here = false, int32_t n = 0, const int4* __restrict__ sinfo = nullptr,
    const unsigned long long* __restrict__ lmask = nullptr, const int32_t* __restrict__ off = nullptr,
    const int2* __restrict__ sinfo2 = nullptr) {
    __shared__ int32_t cnt[kMaxBuckets];
    __shared__ int32_t base[kMaxBuckets];
    for (int64_t t0 = (int64_t)blockIdx.x * kBucketTile; t0 < m; t0 += (int64_t)gridDim.x * kBucketTile) {
        for (int b = threadIdx.x; b < nb; b += blockDim.x) cnt[b] = 0;
        __syncthreads();
        int32_t t[kBucketItems], s[kBucketItems], a[kBucketItems], r[kBucketItems];
#pragma unroll
        for (int k = 0; k < kBucketItems; ++k) {
            const int64_t i = t0 + k * kBucketThreads + threadIdx.x;
            t[k] = -1;
            if (i < m) {
                s[k] = src[i];
                if (s[k] >= lo && s[k] < hi) {
                    t[k] = dst[i];
                    // the pipelined input path buckets before the host reads
                    // the validation flag back: an out-of-range target (flagged
                    // by k_indeg_checked) must not index a bucket
                    if ((unsigned)t[k] >= (unsigned)n) t[k] = -1;
                    a[k] = act ? (int32_t)act[i] : 0;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kBucketItems; ++k) {
            if (t[k] < 0) continue;
            if (slot_here) {  // a[k] := the mark slot (bcrp.py:219)
                if (sinfo || sinfo2) {
                    a[k] = slot_of(s[k], a[k], sinfo, sinfo2);
                } else {
                    a[k] = off[s[k]] + label_rank(lmask, n, s[k], a[k]);
                }
            }
            r[k] = atomicAdd(&cnt[t[k] >> shift], 1);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += blockDim.x)
            if (cnt[b]) base[b] = atomicAdd(&bcur[b], cnt[b]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kBucketItems; ++k)
            if (t[k] >= 0) stage[base[t[k] >> shift] + r[k]] = make_int4(t[k], s[k], a[k], 0);
        __syncthreads();
    }
}

// In-degree histogram of the targets in range; an out-of-range target flags
// the input as bad and is not counted (nothing is scattered through it).
__global__ void k_indeg_checked(int32_t n, int64_t m, const int32_t* __restrict__ dst, int32_t* cnt, Ctrl* ctrl) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < m; i0 += stride) {
        const int64_t i = i0 + lane;
        bool in = false;
        int32_t t = -1 - lane;
        if (i < m) {
            t = dst[i];
            in = (unsigned)t < (unsigned)n;
            if (!in) {
                ctrl->bad = 1;
                t = -1 - lane;
            }
        }
        const LaneRun r = lane_run(t);
        if (in && r.rank == 0) red_add(&cnt[t], r.len);
    }
}

// Pass 2: in staging order, each in-edge takes the next position of its
// target; BCRP computes its mark slot off[s] + rank of the action among s's
// labels (bcrp.py:219) here, once every label set is known.
// SLOT: pass 1 already put the mark slot in the action's place.
template <bool BCRP, bool SLOT>
__global__ void k_rev_place(const int32_t* __restrict__ ptotal, const int4* __restrict__ stage, int32_t* cursor,
                            int2* rev, int32_t* rev_src, int32_t n, const unsigned long long* __restrict__ lmask,
                            const int32_t* __restrict__ off, const int4* __restrict__ sinfo,
                            const int2* __restrict__ sinfo2 = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t total = *ptotal;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < total;
         i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + lane;
        int4 q = make_int4(-1 - lane, 0, 0, 0);
        if (i < total) q = __ldcs(&stage[i]);
        const LaneRun run = lane_run(q.x);
        int32_t at = 0;
        if (i < total && run.rank == 0) at = atomicAdd(&cursor[q.x], run.len);
        at = __shfl_sync(kFull, at, run.leader) + run.rank;
        if (i < total) {
            if (BCRP) {
                const int32_t sv = q.y, a = q.z;
                int32_t slot;
                if (SLOT) {
                    slot = a;
                } else if (sinfo || sinfo2) {
                    slot = slot_of(sv, a, sinfo, sinfo2);
                } else {
                    slot = off[sv] + label_rank(lmask, n, sv, a);
                }
                rev[at] = make_int2(slot, sv);
            } else {
                rev_src[at] = q.y;
            }
        }
    }
}

// ---- states grouped by block, with CTA-level aggregation -----------------------
//
// After the label pre-partition a handful of blocks may hold all n states
// (c5: 8): per-warp atomics on their counters serialise in L2.  Each CTA
// counts a tile of states per block in a shared hash table and reserves its
// run of every block with one global atomic; a tile with too many distinct
// blocks for the table falls back to per-warp atomics.
constexpr int kGroupThreads = 512;
constexpr int kGroupTable = 512;       // hash slots (power of two)

__device__ __forceinline__ int group_slot(int32_t* keys, int32_t b) {
    uint32_t h = ((uint32_t)b * 2654435761u) >> 23;  // 9 bits
#pragma unroll 1
    for (int probe = 0; probe < 32; ++probe) {
        const int32_t old = atomicCAS(&keys[h], -1, b);
        if (old == -1 || old == b) return (int)h;
        h = (h + 1) & (kGroupTable - 1);
    }
    return -1;
}

// FILL = false: bsize[b] += members of b.  FILL = true: members of b go to
// cursor[b] ... (cursor advanced), as member records.
template <bool FILL>
__global__ void __launch_bounds__(kGroupThreads) k_group_states(
    int32_t n, const int32_t* __restrict__ block, int32_t* counter, const int32_t* __restrict__ off,
    const int32_t* __restrict__ rev_ptr, MemberRec* members) {
    __shared__ int32_t keys[kGroupTable];
    __shared__ int32_t cnt[kGroupTable];
    __shared__ int32_t base[kGroupTable];
    __shared__ int overflow;
    const int lane = threadIdx.x & 31;
    for (int64_t t0 = (int64_t)blockIdx.x * kGroupThreads; t0 < n; t0 += (int64_t)gridDim.x * kGroupThreads) {
        for (int k = threadIdx.x; k < kGroupTable; k += blockDim.x) {
            keys[k] = -1;
            cnt[k] = 0;
        }
        if (threadIdx.x == 0) overflow = 0;
        __syncthreads();
        const int64_t s = t0 + threadIdx.x;
        const int32_t b = s < n ? block[s] : -1 - lane;
        const unsigned g = __match_any_sync(kFull, b);
        const int leader = __ffs(g) - 1;
        int slot = -1, r = 0;
        if (s < n && lane == leader) {
            slot = group_slot(keys, b);
            if (slot >= 0) r = atomicAdd(&cnt[slot], __popc(g));
            else overflow = 1;
        }
        __syncthreads();
        const bool ovf = overflow != 0;
        if (!ovf) {
            for (int k = threadIdx.x; k < kGroupTable; k += blockDim.x)
                if (cnt[k]) {
                    const int32_t v = atomicAdd(&counter[keys[k]], cnt[k]);
                    if (FILL) base[k] = v;
                }
        } else if (s < n && lane == leader) {  // crowded tile: per-warp runs
            r = atomicAdd(&counter[b], __popc(g));
        }
        __syncthreads();
        if (FILL) {
            int32_t at = 0;
            if (s < n && lane == leader) at = ovf ? r : base[slot] + r;
            at = __shfl_sync(kFull, at, leader);
            if (s < n)
                members[at + __popc(g & lanemask_lt())] =
                    make_int4((int32_t)s, off ? off[s] : 0, rev_ptr[s], rev_ptr[s + 1]);
        }
        __syncthreads();
    }
}

}  // namespace bisim
