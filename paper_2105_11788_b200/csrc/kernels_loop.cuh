// kernels_loop.cuh -- the persistent refinement loop (default mode).
//
// Included inside namespace bisim by kernels_sparse.cuh.  One cooperative
// launch runs every round (bcrp.py:286-308 / rcpp.py:240-252).  A round is
// executed by a "team":
//
//   grid team  all 148 CTAs, grid barriers between phases (~1.3 us each);
//   solo team  CTA 0 alone, __syncthreads between phases, while the other
//              CTAs park on a hand-over counter.  Used for small rounds
//              (splitter of <= kSoloMaxC members and a previous round with
//              <= kSoloMaxItems phase-B work items), where the grid barrier
//              round trips dominate.  CTA 0 hands the grid back as soon as a
//              round looks bigger, or a skip step is due.
//
// Both teams run the same phase code; only the work distribution (warp ids,
// warp count) and the phase barrier differ, so rounds are bit-identical.
#pragma once

// measured on c1 / c2 (512-thread CTAs): 16 / 128 beat 64 / 64 by 6 / 3 %;
// after the skip-step change 32 / 256 beat 16 / 128 by 4.3 / 0.5 %
constexpr int32_t kSoloMaxC = 32;
constexpr int32_t kSoloMaxItems = 256;
constexpr int32_t kSoloSkipSpan = 512;   // skip-step window of the solo team: one label per thread
#ifndef BISIM_PARK_NS
#define BISIM_PARK_NS 64
#endif
#ifndef BISIM_KA
#define BISIM_KA 1
#endif
#ifdef BISIM_NO_CSNAP
constexpr bool kNoCsnap = true;
#else
constexpr bool kNoCsnap = false;
#endif
#ifndef BISIM_SKIP_GAIN
#define BISIM_SKIP_GAIN 32
#endif
constexpr int32_t kSkipGain = BISIM_SKIP_GAIN;  // rounds a skip step must retire to be retried at once
// in-edges per lane per phase-A step: 1 since the fat barriers (process-level
// A/B vs 2: c1 -3.2 %, c2 -2.0 %, c4l -1.5 %, c3 -1.1 %, c5 / c4u -0.1 %; 3: slower)
constexpr int kA = BISIM_KA;
#ifndef BISIM_KA_BATCH
#define BISIM_KA_BATCH 4
#endif
constexpr int kABatch = BISIM_KA_BATCH;  // ... for splitters of >= batch_min_c members

// Phase A walk over C's members [cs, cs + cz): g members per warp and
// iteration, their in-edges spread over the lanes (warp scan of in-degrees),
// KA in-edges per lane per step issued together.  Marks every in-edge's slot
// and registers each source block once (see the kernel below).
template <int KA, bool IDENT, bool SH>
__device__ __forceinline__ void walk_members(const SparseParams& p, int cur, int32_t cs, int32_t cz, int32_t tw,
                                             int32_t tnw, int32_t g, bool solo, bool batch, int32_t* s_seen,
                                             unsigned long long& my_edges) {
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = (int64_t)tw * g; i0 < cz; i0 += (int64_t)tnw * g) {
        const int64_t i = i0 + lane;
        int32_t e0 = 0, d = 0;
        if (lane < g && i < cz) {
            const MemberRec r = p.members[cs + i];
            e0 = r.z;
            d = r.w - r.z;
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
        // KA in-edges per lane per step: their loads are issued
        // together (reverse edges, then source blocks), so a warp
        // walking a big splitter keeps KA dependent chains in flight
        for (int32_t k0 = 0; k0 < total; k0 += 32 * KA) {
            int32_t s[KA], b[KA];
            bool act[KA];
#pragma unroll
            for (int u = 0; u < KA; ++u) {
                const int32_t k = k0 + 32 * u + lane;
                if (k0 + 32 * u >= total) {  // warp-uniform: nothing left
                    act[u] = false;
                    s[u] = -1;
                    continue;
                }
                // owner lane j: the last lane with excl_j <= k
                int32_t j = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const int32_t ex = __shfl_sync(kFull, excl, j + step);
                    if (ex <= k) j += step;
                }
                const int32_t ej = __shfl_sync(kFull, e0, j);
                const int32_t xj = __shfl_sync(kFull, excl, j);
                act[u] = k < total;
                s[u] = act[u] ? ej + (k - xj) : -1;  // the in-edge index, for now
            }
            int2 rv[KA];
#pragma unroll
            for (int u = 0; u < KA; ++u) {
                // reverse edges stream through (evict-first), so they do not push
                // the randomly accessed per-state arrays out of L2
                if (IDENT) rv[u] = make_int2(0, act[u] ? __ldcs(&p.rev_src[s[u]]) : 0);
                else rv[u] = act[u] ? __ldcs(&p.rev[s[u]]) : make_int2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < KA; ++u) {
                s[u] = rv[u].y;
                const int32_t slot = IDENT ? s[u] : rv[u].x;
                if (act[u]) {
                    if (SH) shard_mark(p, cur, slot);
                    else red_or(&p.mark[slot >> 5], 1u << (slot & 31));
                }
                b[u] = act[u] ? p.block[s[u]] : 0;
            }
#pragma unroll
            for (int u = 0; u < KA; ++u) {
                if (k0 + 32 * u >= total) break;  // warp-uniform
                // a plain shared load first: a block this CTA already
                // met (the common case) skips the table's atomic; lanes
                // of one warp that miss on the same block race in
                // cta_first, which lets exactly one of them through
                const bool rep = act[u] && ld_vol(&s_seen[seen_slot(b[u])]) != b[u];
                bool reg = false;
                BlockInfo bi{};
                if (rep) {
                    const int f = cta_first(s_seen, b[u]);
                    if (f == 1 && solo) {
                        reg = true;  // the solo team is this CTA: its table is exact
                        bi = block_info(p, b[u]);
                    } else if (f == 2 || (f == 1 && !batch)) {
                        // the block's info loads overlap the test-and-set
#ifndef BISIM_NO_PRE
                        bi = block_info(p, b[u]);
#endif
                        const uint32_t bit = 1u << (b[u] & 31);
                        reg = !(atomicOr(&p.tblock[b[u] >> 5], bit) & bit);
                    }
                }
                if (__any_sync(kFull, reg)) {
#ifdef BISIM_NO_PRE
                    if (reg) bi = block_info(p, b[u]);
#endif
                    register_blocks_warp(p, cur, reg, b[u], bi, solo);
                    if (SH && reg) shard_publish(p, cur, b[u]);
                }
            }
        }
    }
}

template <bool IDENT, bool SH>
__global__ void __launch_bounds__(kSparseThreads, kSparsePerSm) k_refine_sparse(SparseParams pk) {
    // SH (transition-sharded replica, kernels_shard.cuh): the round-parity
    // buffers are selected per round on a local copy of the parameters;
    // otherwise p is the kernel parameter itself
    // (in shared memory: a local copy would live on the stack, 700+ bytes)
    __shared__ SparseParams s_pl;
    SparseParams& pl = s_pl;
    if (SH) {
        if (threadIdx.x == 0) pl = pk;
        __syncthreads();
    }
    const SparseParams& p = SH ? pl : pk;
    SCtrl* ctl = p.ctrl;
    unsigned xgen = 0;  // cross-replica barriers passed (SH)
    const int lane = threadIdx.x & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    // logical warp id, CTA-minor: consecutive work items land on different
    // SMs, so a small round's work is spread over the whole chip
    const int32_t gwarp = p.cta_minor ? (int32_t)((threadIdx.x >> 5) * gridDim.x + blockIdx.x)
                                      : (int32_t)(gtid >> 5);
    const int32_t nwarps = (int32_t)(gsize >> 5);
    unsigned gen = 0;
    __shared__ int32_t s_seen[kSeen];
    __shared__ long long s_snap[8];  // control words of the current barrier (team_barrier)
    __shared__ OnePassSlot s_slot[kSparseThreads / 32];
    int32_t cr_c = -1;               // splitter whose member range cr_v holds
    int2 cr_v = make_int2(0, 0);
    for (int k = threadIdx.x; k < kSeen; k += blockDim.x) s_seen[k] = -1;
    raise_init();

    if (gwarp == nwarps - 1) {
        const int32_t c = u_next_warp(p, 0);
        if (lane == 0) ctl->C0 = c;
    }
    if (gtid == 0) {
        ctl->nontriv[0] = ctl->nontriv[1] = kBig;
        ctl->skipcnt[0] = ctl->skipcnt[1] = 0;
        ctl->items_last = kBig;
        for (int q = 0; q < 2; ++q) {
            ctl->brec[q][0] = 0u;
            ctl->brec[q][1] = ~0u;
            ctl->brec[q][2] = ctl->brec[q][3] = 0u;
            ctl->arec[q][0] = ctl->arec[q][1] = ctl->arec[q][2] = ctl->arec[q][3] = 0u;
            ctl->big_pack4[q] = 0ull;
        }
    }
    unsigned genB0 = 0u, genB1 = 0u;  // end-of-round barriers passed, by parity (uniform)
    unsigned genA0 = 0u, genA1 = 0u;  // mid-round barriers passed, by parity (uniform)
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
    const bool solo_ok = !SH && p.allow_solo && p.round_limit == INT64_MAX && gridDim.x > 1;
    bool solo = false;     // this CTA is in a solo stretch (CTA 0 working, others parked)
    bool fresh = false;    // CTA 0: first solo round of a stretch
    unsigned wakes = 0;    // hand-overs so far; identical on every CTA
    unsigned stretches = 0;

    for (int64_t done_here = 0;; ++done_here) {
        // ---- parked CTAs: wait until CTA 0 hands the grid back or stops ----
        if (solo && blockIdx.x != 0) {
            if (threadIdx.x == 0) {
                // acknowledge: this CTA has read everything the solo decision
                // used, CTA 0 may now modify the partition
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&ctl->parked) : "memory");
                while (ld_acquire_u32(&ctl->wake) == wakes) __nanosleep(BISIM_PARK_NS);
            }
            __syncthreads();
            ++wakes;
            solo = false;
            cr_c = -1;
            if (ld_vol(&ctl->stop)) break;
            C = ld_vol(&ctl->C0);
            round = ld_vol(&ctl->round);
            try_skip = ld_vol(&ctl->pub_try_skip) != 0;
            cooldown = ld_vol(&ctl->pub_cooldown);
            backoff = ld_vol(&ctl->pub_backoff);
            skips = ld_vol(&ctl->pub_skips);
        }
        if (done_here == p.round_limit) break;
        const int64_t steps = (int64_t)p.A + round + 1;
        const bool guard_hit = p.has_guard && steps > p.max_supersteps;
        if (guard_hit || C == kBig) {
            if (gtid == 0) {
                if (guard_hit) {
                    ctl->error = 2;
                    ctl->guard_count = steps;
                } else {
                    ctl->done = 1;
                }
                if (solo) {  // release the parked CTAs
                    ctl->stop = 1;
                    __threadfence();
                    atomicAdd(&ctl->wake, 1u);
                }
            }
            break;
        }

        // ---- CTA 0 in a solo stretch: keep going alone or hand back --------
        if (solo) {
            if (fresh) {  // wait until every other CTA has parked
                if (threadIdx.x == 0) {
                    const unsigned target = stretches * (gridDim.x - 1);
                    while ((int)(ld_acquire_u32(&ctl->parked) - target) < 0) {
                    }
                }
                __syncthreads();
                fresh = false;
            }
            const int32_t csz = cr_c == C ? cr_v.y : p.brange[C].y;
            const bool stay = csz <= p.solo_max_c && s_items_last <= p.solo_max_items;
            if (!stay) {
                if (threadIdx.x == 0) {
                    ctl->C0 = C;
                    ctl->round = round;
                    ctl->pub_try_skip = try_skip ? 1 : 0;
                    ctl->pub_cooldown = cooldown;
                    ctl->pub_backoff = backoff;
                    ctl->pub_skips = skips;
                    __threadfence();
                    atomicAdd(&ctl->wake, 1u);
                }
                ++wakes;
                solo = false;
            }
        }

        // the team running this round
        const int32_t tw = solo ? (int32_t)(threadIdx.x >> 5) : gwarp;
        const int32_t tnw = solo ? (int32_t)(blockDim.x >> 5) : nwarps;
        const int64_t ttid = solo ? (int64_t)threadIdx.x : gtid;
        const int64_t tnt = solo ? (int64_t)blockDim.x : gsize;
        const bool aux = tw == tnw - 1;  // unstable-set bookkeeping, off phase A's critical work

        // ---- skip step: retire the maximal run of no-op rounds -------------
        // The next rounds' splitters are the unstable labels in increasing
        // order; a no-op round only removes its splitter from the unstable
        // set, so every unstable label below the first non-trivial one in
        // the window [C, C + span) is retired at once (0 splits each).  The
        // solo team uses a 1024-label window (one U0 word per warp).
        const int32_t span = solo ? kSoloSkipSpan : kSkipSpan;
        if (!SH && try_skip && p.round_limit == INT64_MAX &&
            (!p.has_guard || (int64_t)p.A + round + span + 1 <= p.max_supersteps)) {
            const int sp = (int)(skips & 1);
            const int32_t lim = (int64_t)C + span < (int64_t)p.n ? C + span : p.n;
            for (int32_t w = (C >> 5) + tw; w <= ((lim - 1) >> 5); w += tnw) {
                const int32_t c = (w << 5) + lane;
                const bool cand = c >= C && c < lim && ((ld_vol(&p.U0[w]) >> lane) & 1u);
                if (cand && !round_is_trivial<IDENT>(p, c)) atomicMin(&ctl->nontriv[sp], c);
            }
            team_barrier(solo, p.bar, gen, [&] { s_snap[0] = ld_vol(&ctl->nontriv[sp]); });
            if (ttid == 0) {  // the round after the skip may have either parity
                for (int q = 0; q < 2; ++q) {
                    ctl->brec[q][1] = ~0u;
                    ctl->brec[q][2] = ctl->brec[q][3] = 0u;
                    ctl->arec[q][1] = ctl->arec[q][2] = ctl->arec[q][3] = 0u;
                    ctl->big_pack4[q] = 0ull;
                }
            }
            const int32_t nt = (int32_t)s_snap[0];
            const int32_t end = min(nt, lim);
            int32_t cnt = 0;
            if (end > C) {
                const int32_t wlast = (end - 1) >> 5;
                for (int64_t w = (C >> 5) + ttid; w <= wlast; w += tnt) {
                    uint32_t v = ld_vol(&p.U0[w]);
                    if (w == (C >> 5)) v &= ~0u << (C & 31);
                    if (w == wlast && (end & 31)) v &= (1u << (end & 31)) - 1u;
                    if (v) {
                        red_and(&p.U0[w], ~v);
                        cnt += __popc(v);
                    }
                }
            }
            cnt = __reduce_add_sync(kFull, cnt);
            if (lane == 0 && cnt) atomicAdd(&ctl->skipcnt[sp], cnt);
            if (aux) {
                const int32_t nx = nt < lim ? nt : u_next_warp(p, lim);
                if (lane == 0) {
                    ctl->skip_next[sp] = nx;
                    ctl->nontriv[sp ^ 1] = kBig;
                    ctl->skipcnt[sp ^ 1] = 0;
                }
            }
            team_barrier(solo, p.bar, gen, [&] {
                s_snap[1] = ld_vol(&ctl->skipcnt[sp]);
                s_snap[2] = ld_vol(&ctl->skip_next[sp]);
            });
            const int32_t retired = (int32_t)s_snap[1];
            round += retired;
            C = (int32_t)s_snap[2];
            cr_c = -1;
            ++skips;
            if (gtid == 0) ctl->skipped_rounds += (unsigned long long)retired;
            if (retired == 0) {
                try_skip = false;
                cooldown = backoff;
                backoff = min(backoff * 2, 4096);
            } else {
                backoff = 16;
                // the window stopped at a non-trivial splitter: that round
                // runs next, so a second try now would retire nothing.  A
                // try that paid (>= kSkipGain rounds) leaves the next try to
                // the round's own outcome; a meagre one waits 16 rounds
                if (nt < lim) {
                    try_skip = false;
                    if (retired < kSkipGain) cooldown = 16;
                }
            }
            continue;
        }

        const int cur = (int)(round & 1), nxt = cur ^ 1;
        if (SH) shard_select_parity(pl, pk, cur);
        const bool tr = p.trace != nullptr && gtid == 0 && round < p.trace_rounds;
        if (tr) p.trace[round * kTraceWords + 0] = globaltimer();

        // ---- phase A: mark the in-edges of C's members ----------------------
        if (aux) {
            const int32_t sc = u_clear_next_warp(p, C);
            int2 sr = make_int2(0, 0);
            if (lane == 0) {
                // the usual next splitter: fetch its member range now (it
                // cannot change this round unless the label is raised again);
                // both go into this round's end-of-round record
                if (sc != kBig) sr = p.brange[sc];
                unsigned* rec = ctl->brec[cur];
                red_or(&rec[2], (unsigned)sr.x);
                red_or(&rec[3], (unsigned)sr.y);
                red_min_u32(&rec[1], ((unsigned)sc << 1) | 1u);
                if (solo) {
                    s_succ = sc;
                    s_succ_range = sr;
                }
            }
            if (p.prefetch_next) {
                // and pull its member records towards L2 for the next phase A
                sr.x = __shfl_sync(kFull, sr.x, 0);
                sr.y = __shfl_sync(kFull, sr.y, 0);
                const int32_t lines = min((sr.y + 7) >> 3, 1024);
                for (int32_t k = lane; k < lines; k += 32)
                    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p.members + sr.x + 8 * k));
            }
        }
        // C's member range this round (also C's range at the end of the
        // round unless C itself splits)
        const int2 cr = cr_c == C ? cr_v : p.brange[C];
        {
            const int32_t cs = cr.x, cz = cr.y;
            const bool batch = !solo && cz >= p.batch_min_c;  // CTA-uniform
            // members per warp and iteration: every warp gets the same number
            // of iterations (the smallest that keeps g <= 32), so no warp
            // walks a second slice while most idle; small splitters get one
            // member per warp, their in-edges walked by as many warps as possible
            int32_t g = max(1, (cz + tnw - 1) / tnw);  // 32-bit: cz < 2^30, tnw < 2^13
            if (g > 32) {
                const int32_t iters = (cz + tnw * 32 - 1) / (tnw * 32);
                g = (cz + iters * tnw - 1) / (iters * tnw);
            }
            // big splitters keep several in-edges per lane in flight; the
            // latency-bound small ones are fastest with one
            if (batch) walk_members<kABatch, IDENT, SH>(p, cur, cs, cz, tw, tnw, g, solo, batch, s_seen, my_edges);
            else walk_members<kA, IDENT, SH>(p, cur, cs, cz, tw, tnw, g, solo, batch, s_seen, my_edges);
            if (batch) {
                // a huge splitter: the CTA's table holds every source block
                // its warps met; one wave of global test-and-sets registers
                // them, instead of a returning atomic inside the walk's steps
                trace_at(p, round, 14);  // warp 0's walk done
                __syncthreads();
                trace_at(p, round, 15);  // the CTA's walk done
                // the same source blocks sit in the same slots of every
                // CTA's table: odd CTAs take the table's second half first, so
                // half of the test-and-sets of a hot word find it set by a
                // plain load instead of queueing on it
                constexpr int kPer = kSeen / kSparseThreads;
                static_assert(kSeen % kSparseThreads == 0, "table entries per thread");
                for (int q = 0; q < kPer; ++q) {
                    const int k = ((q + (int)(blockIdx.x & 1u) * (kPer / 2)) % kPer) * kSparseThreads + threadIdx.x;
                    const int32_t b = s_seen[k];
                    bool reg = false;
                    if (b >= 0) {
                        // most source blocks of a huge splitter are met by
                        // every CTA: a plain load first lets all but the
                        // early CTAs skip the test-and-set on the hot word
                        const uint32_t bit = 1u << (b & 31);
                        if (!(ld_vol(&p.tblock[b >> 5]) & bit))
                            reg = !(atomicOr(&p.tblock[b >> 5], bit) & bit);
                    }
                    if (__any_sync(kFull, reg)) {
                        register_blocks_warp(p, cur, reg, b, solo);
                        if (SH && reg) shard_publish(p, cur, b);
                    }
                }
            }
        }
        if (tr) p.trace[round * kTraceWords + 1] = globaltimer();
        if (SH) {
            // every replica's marks are in place; adopt the blocks the other
            // replicas registered first (kernels_shard.cuh)
            if (!shard_exchange(p, cur, gen, xgen, s_snap)) break;
            shard_merge(p, cur, tw, tnw, s_snap);
        }
        if (solo) {
            team_barrier(true, p.bar, gen, [&] {
                s_snap[0] = s_ctr_nsmall;
                s_snap[1] = (long long)s_ctr_big;
                s_snap[2] = (long long)s_ctr_big4;
                s_ctr_nsmall = 0;  // the phase-A counters of the next solo round
                s_ctr_big = s_ctr_big4 = 0ull;
            });
        } else {
            // mid-round barrier on this parity's record: the poll that sees
            // every arrival also returns the registration counters; the wide
            // layout's chunk count is loaded only when the layout choice
            // below needs it
            __syncthreads();
            if (threadIdx.x == 0) {
                if (s_ctr_heavy) {  // the CTA registered a block of > 1 member
                    red_or(&ctl->brec[cur][2], kRecFlag);
                    s_ctr_heavy = 0;
                }
                unsigned* rec = ctl->arec[cur];
                const unsigned target = ((cur ? genA1 : genA0) + 1u) * gridDim.x;
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(rec) : "memory");
                unsigned w0, w1, w2, w3;
                do {
                    asm volatile(
                        "{\n\t.reg .b128 t;\n\tld.acquire.gpu.global.b128 t, [%4];\n\t"
                        "mov.b128 {%0, %1, %2, %3}, t;\n\t}"
                        : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                        : "l"(rec)
                        : "memory");
#if BISIM_POLL_NS > 0
                    if ((int)(w0 - target) < 0) __nanosleep(BISIM_POLL_NS);
#endif
                } while ((int)(w0 - target) < 0);
                s_snap[0] = (int32_t)w1;
                s_snap[1] = (long long)(((unsigned long long)w3 << 32) | w2);
                const int32_t nb = (int32_t)w3, n1 = (int32_t)w2, tw_all = (int32_t)(blockDim.x >> 5) * gridDim.x;
                const bool need4 = n1 > tw_all || n1 > p.wide_min * nb || p.wide_major > 0 || p.force_mode_b > 0;
                s_snap[2] = need4 ? (long long)ld_vol(&ctl->big_pack4[cur]) : 0ll;
            }
            if (cur) ++genA1;
            else ++genA0;
            __syncthreads();
        }
        if (tr) {
            p.trace[round * kTraceWords + 2] = globaltimer();
            p.trace[round * kTraceWords + 4] = p.brange[C].y;
            p.trace[round * kTraceWords + 5] = solo ? 1 : 0;
            p.trace[round * kTraceWords + 6] = s_snap[0];
            p.trace[round * kTraceWords + 7] = s_snap[1];
        }

        // ---- phase B: split the touched blocks ------------------------------
        const int32_t nsm = (int32_t)s_snap[0];
        const unsigned long long bp = (unsigned long long)s_snap[1];
        const unsigned long long bp4 = (unsigned long long)s_snap[2];
        const int32_t nbig = (int32_t)(bp >> 32), nch1 = (int32_t)(bp & 0xffffffffu);
        const int32_t nch4 = (int32_t)(bp4 & 0xffffffffu);
        if (ttid == 0) {
            ctl->arec[nxt][1] = 0u;
            ctl->arec[nxt][2] = ctl->arec[nxt][3] = 0u;
            ctl->big_pack4[nxt] = 0ull;
            ctl->brec[nxt][1] = ~0u;  // the next round's record (its parity's last
            ctl->brec[nxt][2] = 0u;   // readers passed this round's first barrier)
            ctl->brec[nxt][3] = 0u;
            if (SH) p.peer_xcnt[p.shard][nxt] = 0;
        }
        if (threadIdx.x == 0) s_items_last = nsm + nch1;
        // chunk layout and pass count for this round (kernels_big.cuh)
        // one pass needs a warp per big-block chunk only: small blocks are
        // independent items that any warp takes on the side
        int mode_b = nch1 <= tnw ? 0 : (nch4 <= tnw ? 1 : 2);
        // a few very large blocks (> 16K members each on average): the wide
        // layout keeps a quarter of the warps busy with 4 loads in flight per
        // lane, which measured faster than every warp holding one chunk
        if (mode_b == 0 && nch1 > p.wide_min * nbig) mode_b = 1;
        // blocks of a few wide chunks each: the wide layout with CTA-major
        // placement keeps most blocks inside one CTA, whose chunks combine
        // in shared memory instead of a global arrival
        if (mode_b == 0 && p.wide_major > 0 && nch1 > p.onepass_major * nbig && nch4 <= tnw &&
            nch4 <= p.wide_major * nbig)
            mode_b = 1;
        if (p.force_mode_b > mode_b) mode_b = p.force_mode_b;
        const int32_t nch = mode_b == 0 ? nch1 : nch4;
        if (tr) p.trace[round * kTraceWords + 13] = mode_b;
        if (mode_b == 2) {
            for (int32_t it = tw; it < nsm + nch; it += tnw) {
                int32_t cnt;
                if (it < nsm) cnt = process_small<IDENT>(p, cur, round, C, p.small_list[it]);
                else cnt = big_tag<IDENT, kWide>(p, nbig, it - nsm);
                if (lane == 0) my_members += (unsigned long long)cnt;
            }
            trace_at(p, round, 8);  // CTA 0's warp 0 done with pass 1
            team_barrier(solo, p.bar, gen, [] {});
            trace_at(p, round, 9);
            for (int32_t it = tw; it < nch; it += tnw) big_split<IDENT, kWide>(p, cur, round, C, nbig, it);
            trace_at(p, round, 10);
        } else {
            // one pass: every work item has its own warp; all warps of the
            // CTA take part (the big-chunk path synchronises the CTA)
            // blocks of a few chunks each: items go to warps in CTA-major
            // order, so a block's chunks share a CTA and combine in shared
            // memory without a global arrival (c4l -7 %); larger blocks keep
            // the CTA-minor spread (c5: CTA-major 1.5 % slower)
            const bool major = !solo && p.onepass_major > 0 && nch <= p.onepass_major * max(nbig, 1);
            const int32_t twb = major ? (int32_t)(gtid >> 5) : tw;
            int32_t cnt = 0;
            // small blocks first go to the warps without a chunk (ids nch..)
            int32_t it = twb - nch;
            if (it < 0) it += tnw;
            for (; it < nsm; it += tnw) cnt += process_small<IDENT>(p, cur, round, C, p.small_list[it]);
            // warps without an item pull the in-edges of C's successor (the
            // usual next splitter, its range published in phase A) towards
            // L2, a warp per 32 of its members: phase A of the next round
            // then finds them there instead of in HBM (a hint only: a
            // different next splitter just leaves the lines unused).  Only in
            // rounds without small touched blocks: their splits raise the
            // labels that usually come next instead (c2: no gain)
            if (p.prefetch_next >= 2 && !solo && nsm == 0 && twb >= nch) {
                const unsigned* rec = ctl->brec[cur];
                const int32_t sx = (int32_t)(ld_vol(&rec[2]) & ~kRecFlag), sz = (int32_t)(ld_vol(&rec[3]) & ~kRecFlag);
                const int32_t i = (twb - nch) * 32 + lane;
                if (i < sz) {
                    const MemberRec r = p.members[sx + i];
                    const char* a = IDENT ? (const char*)(p.rev_src + r.z) : (const char*)(p.rev + r.z);
                    const char* e = IDENT ? (const char*)(p.rev_src + r.w) : (const char*)(p.rev + r.w);
                    a = (const char*)((uintptr_t)a & ~(uintptr_t)127);
                    for (int k = 0; k < 4 && a < e; ++k, a += 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
                }
            }
            const int32_t ci = twb < nch ? twb : -1;
            if (mode_b == 0) cnt += big_onepass_cta<IDENT, 1>(p, cur, round, C, nbig, ci, s_slot);
            else cnt += big_onepass_cta<IDENT, kWide>(p, cur, round, C, nbig, ci, s_slot);
            if (lane == 0) my_members += (unsigned long long)cnt;
        }
        for (int k = threadIdx.x; k < kSeen; k += blockDim.x) s_seen[k] = -1;
        if (solo) {
            team_barrier(true, p.bar, gen, [&] { raise_flush_warp0(p, cur, round); }, [&] {
                // everything this round raised or found is in this CTA
                const int32_t nm = s_nmin_round, cs = s_csplit_round, sc = s_succ;
                s_snap[4] = s_ctr_heavy;
                s_ctr_heavy = 0;
                s_snap[5] = s_items_last;
                const int32_t c_next = min(nm, sc);
                s_snap[3] = c_next;
                if (c_next != kBig) {
                    if (nm > sc) {
                        s_snap[6] = ((long long)s_succ_range.y << 32) | (unsigned)s_succ_range.x;
                    } else if (!kNoCsnap && c_next == C && !cs) {
                        s_snap[6] = ((long long)cr.y << 32) | (unsigned)cr.x;
                    } else {
                        const int32_t* r = (const int32_t*)&p.brange[c_next];
                        s_snap[6] = ((long long)ld_vol(r + 1) << 32) | (unsigned)ld_vol(r);
                    }
                }
            });
        } else {
            // end-of-round barrier on this parity's record: the poll that
            // sees every arrival also returns the next splitter (min of the
            // raised labels and C's successor), the successor's range and the
            // round's flags -- no separate load of the control words after it
            __syncthreads();
            if (threadIdx.x < 32) raise_flush_warp0(p, cur, round);
            if (threadIdx.x == 0) {
                unsigned* rec = ctl->brec[cur];
                const unsigned target = ((cur ? genB1 : genB0) + 1u) * gridDim.x;
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(rec) : "memory");
                unsigned w0, w1, w2, w3;
                do {
                    asm volatile(
                        "{\n\t.reg .b128 t;\n\tld.acquire.gpu.global.b128 t, [%4];\n\t"
                        "mov.b128 {%0, %1, %2, %3}, t;\n\t}"
                        : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                        : "l"(rec)
                        : "memory");
#if BISIM_POLL_NS > 0
                    if ((int)(w0 - target) < 0) __nanosleep(BISIM_POLL_NS);
#endif
                } while ((int)(w0 - target) < 0);
                const int32_t c_next = (int32_t)(w1 >> 1);  // ~0u -> kBig
                s_snap[3] = c_next;
                s_snap[4] = (w2 & kRecFlag) ? 1 : 0;
                s_snap[5] = s_items_last;
                if (c_next != kBig) {
                    if (w1 & 1u) {  // the successor, not raised this round
                        s_snap[6] = ((long long)(w3 & ~kRecFlag) << 32) | (w2 & ~kRecFlag);
                    } else if (!kNoCsnap && c_next == C && !(w3 & kRecFlag)) {
                        // C raised again (BCRP re-raise) without splitting: its
                        // range is unchanged, no dependent load
                        s_snap[6] = ((long long)cr.y << 32) | (unsigned)cr.x;
                    } else {
                        const int32_t* r = (const int32_t*)&p.brange[c_next];
                        s_snap[6] = ((long long)ld_vol(r + 1) << 32) | (unsigned)ld_vol(r);
                    }
                }
            }
            if (cur) ++genB1;
            else ++genB0;
            __syncthreads();
        }
        if (tr) p.trace[round * kTraceWords + 3] = globaltimer();
        C = (int32_t)s_snap[3];
        if (C != kBig) {
            cr_c = C;
            cr_v = make_int2((int32_t)(s_snap[6] & 0xffffffffll), (int32_t)(s_snap[6] >> 32));
        }
        ++round;
        if (cooldown > 0) --cooldown;
        try_skip = p.allow_skip && cooldown == 0 && s_snap[4] == 0;

        // ---- grid team: go solo for the next rounds? (uniform decision) ----
        if (!solo && solo_ok && !try_skip && C != kBig && cr_v.y <= p.solo_max_c &&
            (int32_t)s_snap[5] <= p.solo_max_items) {
            solo = true;  // CTA 0 continues alone, the others park at the loop head
            fresh = true;
            ++stretches;
        }
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
