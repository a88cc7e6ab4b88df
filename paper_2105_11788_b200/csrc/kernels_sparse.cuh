// kernels_sparse.cuh -- work-efficient refinement loop (default mode).
//
// Same rounds, same Priority winners as the dense loop in kernels.cuh, but a
// round only touches what its splitter C can affect:
//
//   phase A  (mark)   the members of C -- a contiguous range of `members`,
//            the state permutation grouped by block -- mark the slots of
//            their in-edges (reverse CSR).  In-edges are spread over the
//            lanes of a warp (a warp scan of the members' in-degrees), mark
//            and touched bits are fire-and-forget reductions, and each source
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

constexpr int kSparseThreads = 1024;  // one CTA per SM

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

struct SCtrl {
    int32_t C0;                         // entry-time splitter
    int32_t done;
    int32_t error;
    int32_t pad0;
    int64_t round;
    int64_t guard_count;
    int32_t next_min[2];                // min raised label, by round parity
    int32_t succ[2];                    // successor of C in unstable \ {C}
    int32_t n_small[2];                 // touched blocks of <= 32 members
    int32_t pad1[2];
    unsigned long long big_pack[2];     // (#big touched blocks << 32) | #32-member chunks
    unsigned long long big_pack4[2];    // same for the 128-member chunk layout
    unsigned long long work_edges;      // sum of in(C)
    unsigned long long work_members;    // sum of touched-block sizes
    int32_t heavy[2];                   // round touched a block of > 1 member
    int32_t nontriv[2];                 // skip step: least non-trivial candidate
    int32_t skipcnt[2];                 // skip step: rounds retired
    int32_t skip_next[2];               // skip step: splitter after the window
    unsigned long long skipped_rounds;  // statistics
};

// Window of unstable labels examined by one skip step (see k_refine_sparse).
constexpr int32_t kSkipSpan = 32768;
constexpr int32_t kSkipMaxEdges = 256;
constexpr int kWide = 4;  // members per lane in the wide big-block chunk layout (kernels_big.cuh)

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
    int32_t* members;   // states grouped by block
    int2* brange;       // (start, size) of block `label` in members (valid for leaders)
    uint32_t* mark;     // L-bit mark bitmap
    uint32_t* touched;  // n-bit: state has a marked slot this round (BCRP)
    uint32_t* tblock;   // n-bit: block label registered this round
    uint32_t* U0;       // unstable labels, 3-level summary (1 bit per 1024 / 1M)
    uint32_t* U1;
    uint32_t* U2;
    int32_t nw0, nw1, nw2;
    int32_t pad;
    int4* small_list;     // touched blocks of <= 32 members: (label, start, size, -)
    int4* big_list;       // larger touched blocks: (label, start, size, first chunk)
    int32_t* big_base;    // first chunk of each big touched block (ascending)
    int4* big_list4;      // the same blocks in the kWide chunk layout
    int32_t* big_base4;
    int32_t* tmp;         // per member position: member, or -1-member if split
    int32_t* scnt;        // per label: split count / min split / compaction cursors
    int32_t* smin;
    int32_t* kcur;
    int32_t* scur;
    int32_t* sarr;        // per label: chunks of the block that have tagged (one-pass split)
    int32_t* splits;
    SCtrl* ctrl;
    GridBarrier* bar;
    unsigned long long* trace;  // optional: 4 globaltimer stamps per round (CTA 0)
    int64_t trace_rounds;
    int32_t allow_skip;         // retire runs of no-op rounds in one step
    int32_t pad2;
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ---- hierarchical unstable set --------------------------------------------

// Raise label x.  Fire-and-forget reductions on all three levels (a summary
// bit may be set redundantly; it only has to be set whenever its range is
// non-empty).
__device__ __forceinline__ void u_set(const SparseParams& p, int32_t x) {
    atomicOr(&p.U0[x >> 5], 1u << (x & 31));
    atomicOr(&p.U1[x >> 15], 1u << ((x >> 10) & 31));
    atomicOr(&p.U2[x >> 25], 1u << ((x >> 20) & 31));
}

// Clear x (whole warp participates; no concurrent raises in this phase).
__device__ __forceinline__ void u_clear_warp(const SparseParams& p, int32_t x) {
    const int lane = threadIdx.x & 31;
    uint32_t w0 = 0;
    if (lane == 0) w0 = atomicAnd(&p.U0[x >> 5], ~(1u << (x & 31))) & ~(1u << (x & 31));
    w0 = __shfl_sync(kFull, w0, 0);
    if (w0) return;
    const int32_t c = x >> 10;  // 32-word chunk of U0
    const int32_t wi = (c << 5) + lane;
    uint32_t v = wi < p.nw0 ? p.U0[wi] : 0u;
    if (__ballot_sync(kFull, v != 0u)) return;
    uint32_t w1 = 0;
    if (lane == 0) w1 = atomicAnd(&p.U1[c >> 5], ~(1u << (c & 31))) & ~(1u << (c & 31));
    w1 = __shfl_sync(kFull, w1, 0);
    if (w1) return;
    const int32_t d = x >> 20;
    const int32_t wj = (d << 5) + lane;
    v = wj < p.nw1 ? p.U1[wj] : 0u;
    if (__ballot_sync(kFull, v != 0u)) return;
    if (lane == 0) atomicAnd(&p.U2[d >> 5], ~(1u << (d & 31)));
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

// Register block b (first touch this round) in the touched lists.
__device__ __forceinline__ void register_block(const SparseParams& p, int cur, int32_t b) {
    SCtrl* ctl = p.ctrl;
    const int2 r = p.brange[b];
    if (r.y > 1) ctl->heavy[cur] = 1;
    if (r.y <= 32) {
        const int32_t k = atomicAdd(&ctl->n_small[cur], 1);
        p.small_list[k] = make_int4(b, r.x, r.y, 0);
    } else {
        // two chunk layouts (kernels_big.cuh); each list is ordered by its
        // own packed counter, so its first-chunk column ascends
        const int32_t nch1 = (r.y + 31) >> 5, nch4 = (r.y + 32 * kWide - 1) / (32 * kWide);
        const unsigned long long pk =
            atomicAdd(&ctl->big_pack[cur], (1ull << 32) | (unsigned long long)nch1);
        const unsigned long long pk4 =
            atomicAdd(&ctl->big_pack4[cur], (1ull << 32) | (unsigned long long)nch4);
        const int32_t k = (int32_t)(pk >> 32), base = (int32_t)(pk & 0xffffffffu);
        const int32_t k4 = (int32_t)(pk4 >> 32), base4 = (int32_t)(pk4 & 0xffffffffu);
        p.big_list[k] = make_int4(b, r.x, r.y, base);
        p.big_base[k] = base;
        p.big_list4[k4] = make_int4(b, r.x, r.y, base4);
        p.big_base4[k4] = base4;
        p.scnt[b] = 0;
        p.smin[b] = kBig;
        p.kcur[b] = 0;
        p.scur[b] = 0;
        p.sarr[b] = 0;
    }
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
constexpr int kSeen = 1024;

__device__ __forceinline__ bool cta_first(int32_t* seen, int32_t b) {
    uint32_t h = ((uint32_t)b * 2654435761u) >> 22;  // 10-bit hash
#pragma unroll 1
    for (int probe = 0; probe < 16; ++probe) {
        const int32_t old = atomicCAS(&seen[h], -1, b);
        if (old == -1) return true;
        if (old == b) return false;
        h = (h + 1) & (kSeen - 1);
    }
    return true;  // table crowded: let the global test-and-set decide
}

// ---- phase B helpers --------------------------------------------------------

template <bool IDENT>
__device__ __forceinline__ bool member_splits(const SparseParams& p, int32_t u, int32_t l,
                                              bool tl, bool& tu, int32_t& ou, int32_t& nr) {
    if (IDENT) {
        tu = get_bit(p.mark, u);
        ou = u;
        nr = 1;
        return u != l && (tu != tl);
    }
    tu = get_bit(p.touched, u);
    ou = p.off[u];
    nr = p.off[u + 1] - ou;
    if (u == l || !(tu || tl) || nr == 0) return false;
    return slots_differ(p.mark, ou, p.off[l], nr);
}

template <bool IDENT>
__device__ __forceinline__ void clear_member(const SparseParams& p, int32_t u, bool tu, int32_t ou,
                                             int32_t nr) {
    if (!tu) return;
    if (IDENT) {
        atomicAnd(&p.mark[u >> 5], ~(1u << (u & 31)));
        return;
    }
    atomicAnd(&p.touched[u >> 5], ~(1u << (u & 31)));
    int32_t pos = ou, left = nr;
    while (left > 0) {
        const int32_t sh = pos & 31, len = min(left, 32 - sh);
        const uint32_t msk = (len == 32 ? ~0u : ((1u << len) - 1u)) << sh;
        atomicAnd(&p.mark[pos >> 5], ~msk);
        pos += len;
        left -= len;
    }
}

__device__ __forceinline__ void raise_split(const SparseParams& p, int cur, int64_t round, int32_t l,
                                            int32_t w, int32_t C) {
    u_set(p, l);
    u_set(p, w);
    int32_t lo = min(l, w);
    if (p.reflag_c) {  // BCRP: any split re-destabilises C (bcrp.py:282)
        u_set(p, C);
        lo = min(lo, C);
    }
    atomicMin(&p.ctrl->next_min[cur], lo);
    if (round < p.splits_cap) atomicAdd(&p.splits[round], 1);
}

// A touched block of <= 32 members, finished by one warp.
template <bool IDENT>
__device__ int32_t process_small(const SparseParams& p, int cur, int64_t round, int32_t C, int4 e) {
    const int lane = threadIdx.x & 31;
    const int32_t l = e.x, bs = e.y, bz = e.z;
    const bool valid = lane < bz;
    const int32_t u = valid ? p.members[bs + lane] : -1;
    const bool tl = IDENT ? get_bit(p.mark, l) : get_bit(p.touched, l);
    bool tu = false;
    int32_t ou = 0, nr = 0;
    const bool sp = valid && member_splits<IDENT>(p, u, l, tl, tu, ou, nr);
    const unsigned bal = __ballot_sync(kFull, sp);
    if (bal) {
        const int32_t ns = __popc(bal);
        const int32_t keep = bz - ns;
        const int32_t w = __reduce_min_sync(kFull, sp ? u : kBig);
        const unsigned lt = lanemask_lt();
        const unsigned vmask = bz >= 32 ? kFull : ((1u << bz) - 1u);
        if (valid) {
            const int32_t np = sp ? bs + keep + __popc(bal & lt) : bs + __popc(~bal & vmask & lt);
            p.members[np] = u;
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
    if (lane == 0) atomicAnd(&p.tblock[l >> 5], ~(1u << (l & 31)));
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
template <bool IDENT>
__device__ __forceinline__ bool round_is_trivial(const SparseParams& p, int32_t c) {
    const int2 r = p.brange[c];
    if (r.y > 32) return false;
    int32_t budget = kSkipMaxEdges;
    for (int32_t i = 0; i < r.y; ++i) {
        const int32_t t = p.members[r.x + i];
        const int32_t e0 = p.rev_ptr[t], e1 = p.rev_ptr[t + 1];
        if (e1 - e0 > budget) return false;
        budget -= e1 - e0;
        for (int32_t e = e0; e < e1; e += 4) {
            int32_t s[4], b[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) s[k] = e + k < e1 ? (IDENT ? p.rev_src[e + k] : p.rev[e + k].y) : -1;
#pragma unroll
            for (int k = 0; k < 4; ++k) b[k] = s[k] >= 0 ? p.block[s[k]] : -1;
            bool single = true;
#pragma unroll
            for (int k = 0; k < 4; ++k) single &= b[k] < 0 || p.brange[b[k]].y == 1;
            if (!single) return false;
        }
    }
    return true;
}

// ---- the persistent kernel ---------------------------------------------------

template <bool IDENT>
__global__ void __launch_bounds__(kSparseThreads, 1) k_refine_sparse(SparseParams p) {
    SCtrl* ctl = p.ctrl;
    const int lane = threadIdx.x & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // logical warp id, CTA-minor: consecutive work items land on different
    // SMs, so a small round's work is spread over the whole chip
    const int32_t gwarp = (int32_t)((threadIdx.x >> 5) * gridDim.x + blockIdx.x);
    const int32_t nwarps = (int32_t)(((int64_t)gridDim.x * blockDim.x) >> 5);
    const int32_t aux_warp = nwarps - 1;  // keeps the unstable-set bookkeeping off phase A's work
    unsigned gen = 0;
    __shared__ int32_t s_seen[kSeen];
    for (int k = threadIdx.x; k < kSeen; k += blockDim.x) s_seen[k] = -1;

    if (gwarp == aux_warp) {
        const int32_t c = u_next_warp(p, 0);
        if (lane == 0) ctl->C0 = c;
    }
    if (gtid == 0) {
        ctl->nontriv[0] = ctl->nontriv[1] = kBig;
        ctl->skipcnt[0] = ctl->skipcnt[1] = 0;
    }
    grid_barrier(p.bar, gen);
    int32_t C = ld_vol(&ctl->C0);
    int64_t round = ld_vol(&ctl->round);
    unsigned long long my_edges = 0, my_members = 0;
    // no-op-round retirement (only in persistent mode: an observer must see
    // every round): tried after a round that touched singleton blocks only,
    // with exponential back-off when a try retires nothing
    bool try_skip = false;
    int32_t cooldown = 0, backoff = 16;
    int64_t skips = 0;

    for (int64_t done_here = 0;; ++done_here) {
        if (done_here == p.round_limit) break;
        const int64_t steps = (int64_t)p.A + round + 1;
        if (p.has_guard && steps > p.max_supersteps) {
            if (gtid == 0) {
                ctl->error = 2;
                ctl->guard_count = steps;
            }
            break;
        }
        if (C == kBig) {
            if (gtid == 0) ctl->done = 1;
            break;
        }

        // ---- skip step: retire the maximal run of no-op rounds -------------
        // The next rounds' splitters are the unstable labels in increasing
        // order; a no-op round only removes its splitter from the unstable
        // set, so every unstable label below the first non-trivial one in
        // the window [C, C + kSkipSpan) is retired at once (0 splits each).
        if (try_skip && p.round_limit == INT64_MAX &&
            (!p.has_guard || (int64_t)p.A + round + kSkipSpan + 1 <= p.max_supersteps)) {
            const int sp = (int)(skips & 1);
            const int32_t lim = (int64_t)C + kSkipSpan < (int64_t)p.n ? C + kSkipSpan : p.n;
            for (int32_t w = (C >> 5) + gwarp; w <= ((lim - 1) >> 5); w += nwarps) {
                const int32_t c = (w << 5) + lane;
                const bool cand = c >= C && c < lim && ((ld_vol(&p.U0[w]) >> lane) & 1u);
                if (cand && !round_is_trivial<IDENT>(p, c)) atomicMin(&ctl->nontriv[sp], c);
            }
            grid_barrier(p.bar, gen);
            const int32_t nt = ld_vol(&ctl->nontriv[sp]);
            const int32_t end = min(nt, lim);
            int32_t cnt = 0;
            if (end > C) {
                const int32_t wlast = (end - 1) >> 5;
                for (int64_t w = (C >> 5) + gtid; w <= wlast; w += (int64_t)gridDim.x * blockDim.x) {
                    uint32_t v = ld_vol(&p.U0[w]);
                    if (w == (C >> 5)) v &= ~0u << (C & 31);
                    if (w == wlast && (end & 31)) v &= (1u << (end & 31)) - 1u;
                    if (v) {
                        atomicAnd(&p.U0[w], ~v);
                        cnt += __popc(v);
                    }
                }
            }
            cnt = __reduce_add_sync(kFull, cnt);
            if (lane == 0 && cnt) atomicAdd(&ctl->skipcnt[sp], cnt);
            if (gwarp == aux_warp) {
                const int32_t nx = nt < lim ? nt : u_next_warp(p, lim);
                if (lane == 0) {
                    ctl->skip_next[sp] = nx;
                    ctl->nontriv[sp ^ 1] = kBig;
                    ctl->skipcnt[sp ^ 1] = 0;
                }
            }
            grid_barrier(p.bar, gen);
            const int32_t retired = ld_vol(&ctl->skipcnt[sp]);
            round += retired;
            C = ld_vol(&ctl->skip_next[sp]);
            ++skips;
            if (gtid == 0) ctl->skipped_rounds += (unsigned long long)retired;
            if (retired == 0) {
                try_skip = false;
                cooldown = backoff;
                backoff = min(backoff * 2, 4096);
            } else {
                backoff = 16;
            }
            continue;
        }

        const int cur = (int)(round & 1), nxt = cur ^ 1;
        const bool tr = p.trace != nullptr && gtid == 0 && round < p.trace_rounds;
        if (tr) p.trace[round * 8 + 0] = globaltimer();

        // ---- phase A --------------------------------------------------------
        if (gwarp == aux_warp) {
            u_clear_warp(p, C);
            const int32_t sc = u_next_warp(p, C + 1);
            if (lane == 0) {
                ctl->succ[cur] = sc;
                ctl->next_min[cur] = kBig;
            }
        }
        {
            const int2 cr = p.brange[C];
            const int32_t cs = cr.x, cz = cr.y;
            // members per warp: spread small splitters one member per warp so
            // their in-edges are walked by as many warps as possible
            const int32_t g = cz >= nwarps * 32 ? 32 : max(1, (cz + nwarps - 1) / nwarps);
            for (int64_t i0 = (int64_t)gwarp * g; i0 < cz; i0 += (int64_t)nwarps * g) {
                const int64_t i = i0 + lane;
                int32_t e0 = 0, d = 0;
                if (lane < g && i < cz) {
                    const int32_t t = p.members[cs + i];
                    e0 = p.rev_ptr[t];
                    d = p.rev_ptr[t + 1] - e0;
                }
                int32_t incl = d;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                const int32_t total = __shfl_sync(kFull, incl, 31);
                const int32_t excl = incl - d;
                my_edges += (unsigned long long)d;
                for (int32_t k0 = 0; k0 < total; k0 += 32) {
                    const int32_t k = k0 + lane;
                    // owner lane j: the last lane with excl_j <= k
                    int32_t j = 0;
#pragma unroll
                    for (int step = 16; step; step >>= 1) {
                        const int32_t ex = __shfl_sync(kFull, excl, j + step);
                        if (ex <= k) j += step;
                    }
                    const int32_t ej = __shfl_sync(kFull, e0, j);
                    const int32_t xj = __shfl_sync(kFull, excl, j);
                    const bool act = k < total;
                    int32_t s = 0;
                    if (act) {
                        const int32_t e = ej + (k - xj);
                        if (IDENT) {
                            s = p.rev_src[e];
                            atomicOr(&p.mark[s >> 5], 1u << (s & 31));
                        } else {
                            const int2 r = p.rev[e];
                            s = r.y;
                            atomicOr(&p.mark[r.x >> 5], 1u << (r.x & 31));
                            atomicOr(&p.touched[s >> 5], 1u << (s & 31));
                        }
                    }
                    const int32_t b = act ? p.block[s] : 0;
                    const unsigned same = __match_any_sync(kFull, act ? b : -1 - lane);
                    const bool rep = act && lane == __ffs(same) - 1;
                    if (rep && cta_first(s_seen, b)) {
                        const uint32_t bit = 1u << (b & 31);
                        if (!(ld_vol(&p.tblock[b >> 5]) & bit) && !(atomicOr(&p.tblock[b >> 5], bit) & bit))
                            register_block(p, cur, b);
                    }
                }
            }
        }
        if (tr) p.trace[round * 8 + 1] = globaltimer();
        grid_barrier(p.bar, gen);
        if (tr) {
            p.trace[round * 8 + 2] = globaltimer();
            p.trace[round * 8 + 4] = p.brange[C].y;
            p.trace[round * 8 + 5] = my_edges;
            p.trace[round * 8 + 6] = ld_vol(&ctl->n_small[cur]);
            p.trace[round * 8 + 7] = ld_vol(&ctl->big_pack[cur]);
        }

        // ---- phase B --------------------------------------------------------
        if (gtid == 0) {
            ctl->n_small[nxt] = 0;
            ctl->big_pack[nxt] = 0ull;
            ctl->big_pack4[nxt] = 0ull;
            ctl->heavy[nxt] = 0;
        }
        const int32_t nsm = ld_vol(&ctl->n_small[cur]);
        const unsigned long long bp = ld_vol(&ctl->big_pack[cur]);
        const unsigned long long bp4 = ld_vol(&ctl->big_pack4[cur]);
        const int32_t nbig = (int32_t)(bp >> 32), nch1 = (int32_t)(bp & 0xffffffffu);
        const int32_t nch4 = (int32_t)(bp4 & 0xffffffffu);
        // chunk layout and pass count for this round (kernels_big.cuh)
        const int mode_b = nsm + nch1 <= nwarps ? 0 : (nsm + nch4 <= nwarps ? 1 : 2);
        const int32_t nch = mode_b == 0 ? nch1 : nch4;
        for (int32_t it = gwarp; it < nsm + nch; it += nwarps) {
            int32_t cnt;
            if (it < nsm) cnt = process_small<IDENT>(p, cur, round, C, p.small_list[it]);
            else if (mode_b == 0) cnt = big_onepass<IDENT, 1>(p, cur, round, C, nbig, it - nsm);
            else if (mode_b == 1) cnt = big_onepass<IDENT, kWide>(p, cur, round, C, nbig, it - nsm);
            else cnt = big_tag<IDENT, kWide>(p, nbig, it - nsm);
            if (lane == 0) my_members += (unsigned long long)cnt;
        }
        if (mode_b == 2) {
            grid_barrier(p.bar, gen);
            for (int32_t it = gwarp; it < nch; it += nwarps) big_split<IDENT, kWide>(p, cur, round, C, nbig, it);
        }
        for (int k = threadIdx.x; k < kSeen; k += blockDim.x) s_seen[k] = -1;
        grid_barrier(p.bar, gen);
        if (tr) p.trace[round * 8 + 3] = globaltimer();
        C = min(ld_vol(&ctl->next_min[cur]), ld_vol(&ctl->succ[cur]));
        ++round;
        if (cooldown > 0) --cooldown;
        try_skip = p.allow_skip && cooldown == 0 && ld_vol(&ctl->heavy[cur]) == 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        my_edges += __shfl_xor_sync(kFull, my_edges, o);
        my_members += __shfl_xor_sync(kFull, my_members, o);
    }
    if (lane == 0) {
        if (my_edges) atomicAdd(&ctl->work_edges, my_edges);
        if (my_members) atomicAdd(&ctl->work_members, my_members);
    }
    if (gtid == 0) ctl->round = round;
}

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
                               int32_t* members) {
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
        if (s < n) members[base + __popc(g & lanemask_lt())] = (int32_t)s;
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

// Pack BCRP reverse edges (slot, source) for one 8-byte load per in-edge.
template <bool BCRP>
__global__ void k_rev_fill2(int32_t n, int64_t m, const int32_t* __restrict__ src,
                            const int32_t* __restrict__ act, const int32_t* __restrict__ dst,
                            const unsigned long long* __restrict__ lmask, const int32_t* __restrict__ off,
                            int32_t* cursor, int2* rev, int32_t* rev_src) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < m; i0 += stride) {
        const int64_t i = i0 + lane;
        int32_t t = -1 - lane, slot = 0, s = 0;
        if (i < m) {
            t = dst[i];
            s = src[i];
            slot = BCRP ? off[s] + label_rank(lmask, n, s, act[i]) : s;
        }
        const unsigned grp = __match_any_sync(kFull, t);
        const int leader = __ffs(grp) - 1;
        int32_t base = 0;
        if (i < m && lane == leader) base = atomicAdd(&cursor[t], __popc(grp));
        base = __shfl_sync(kFull, base, leader);
        if (i < m) {
            const int32_t at = base + __popc(grp & lanemask_lt());
            if (BCRP) rev[at] = make_int2(slot, s);
            else rev_src[at] = s;
        }
    }
}

}  // namespace bisim
