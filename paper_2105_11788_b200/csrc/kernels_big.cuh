// kernels_big.cuh -- phase B for touched blocks of more than 32 members.
//
// Included by kernels_sparse.cuh after SparseParams and the member helpers.
// A big touched block is cut into chunks of 32*K members (K members per
// lane, index ci0 + 32 j + lane).  Every big block is registered in two
// chunk layouts, K = 1 and K = kWide; phase B picks per round:
//
//   * every work item fits on its own warp with K = 1 -> one pass, K = 1
//     (late, latency-bound rounds: most warps, shortest chains);
//   * else, if it fits with K = kWide                 -> one pass, K = kWide;
//   * else                                            -> two passes, K = kWide
//     (heavy rounds: several items per warp, K chains in flight per lane).
//
// One pass: the chunks of a block publish their split count and minimum,
// bump an arrival counter and wait for the last one (all items run
// concurrently, so this cannot deadlock), then compact from registers.
// Two passes: tag + publish, grid barrier, then compact.
#pragma once

// (included inside namespace bisim by kernels_sparse.cuh)

template <int K>
__device__ __forceinline__ const int4* big_list_of(const SparseParams& p) {
    return K == 1 ? p.big_list : p.big_list4;
}
template <int K>
__device__ __forceinline__ const int32_t* big_base_of(const SparseParams& p) {
    return K == 1 ? p.big_base : p.big_base4;
}
template <int K>
__device__ __forceinline__ const int2* big_info_of(const SparseParams& p) {
    return K == 1 ? p.big_info : p.big_info4;
}

// Owner (list index) of chunk ci: the last big block whose first chunk <= ci.
template <int K>
__device__ __forceinline__ int32_t find_owner(const SparseParams& p, int32_t nbig, int32_t ci) {
    const int lane = threadIdx.x & 31;
    const int32_t* base = big_base_of<K>(p);
    int32_t lo = 0, hi = nbig;
    while (hi - lo > 32) {
        const int32_t stride = (hi - lo + 31) >> 5;
        const int32_t idx = lo + lane * stride;
        const int32_t v = idx < hi ? base[idx] : 0x7fffffff;
        const unsigned b = __ballot_sync(kFull, v <= ci);
        const int32_t last = 31 - __clz(b);
        lo = lo + last * stride;
        hi = min(lo + stride, hi);
    }
    const int32_t idx = lo + lane;
    const int32_t v = idx < hi ? base[idx] : 0x7fffffff;
    const unsigned b = __ballot_sync(kFull, v <= ci);
    return lo + 31 - __clz(b);
}

// Owner list entry (and leader slot range) of chunk ci.  Up to 128 big
// blocks the warp loads every entry at once and picks the owner by ballot,
// one round trip instead of a base search followed by the entry load.
#ifndef BISIM_ENTRY_PROBE
#define BISIM_ENTRY_PROBE 4
#endif
constexpr int kEntryProbe = BISIM_ENTRY_PROBE;  // entries per lane
template <int K>
__device__ __forceinline__ int32_t find_entry(const SparseParams& p, int32_t nbig, int32_t ci, int4& e, int2& li) {
    const int lane = threadIdx.x & 31;
    if (nbig > 32 * kEntryProbe) {
        const int32_t k = find_owner<K>(p, nbig, ci);
        e = big_list_of<K>(p)[k];
        li = big_info_of<K>(p)[k];
        return k;
    }
    const int4* L = big_list_of<K>(p);
    const int2* I = big_info_of<K>(p);
    int4 ev[kEntryProbe];
    int2 iv[kEntryProbe];
#pragma unroll
    for (int q = 0; q < kEntryProbe; ++q) {
        const int32_t k = lane + 32 * q;
        ev[q] = k < nbig ? L[k] : make_int4(0, 0, 0, 0x7fffffff);
        iv[q] = k < nbig ? I[k] : make_int2(0, 0);
    }
    // the owner is the last entry whose first chunk <= ci (bases ascend)
    int qs = 0;
    unsigned bq = 0u;
#pragma unroll
    for (int q = 0; q < kEntryProbe; ++q) {
        const unsigned b = __ballot_sync(kFull, ev[q].w <= ci);
        if (b) {
            qs = q;
            bq = b;
        }
    }
    const int src = 31 - __clz(bq);
    int4 mine = ev[0];
    int2 mi = iv[0];
#pragma unroll
    for (int q = 1; q < kEntryProbe; ++q)
        if (q == qs) {
            mine = ev[q];
            mi = iv[q];
        }
    e.x = __shfl_sync(kFull, mine.x, src);
    e.y = __shfl_sync(kFull, mine.y, src);
    e.z = __shfl_sync(kFull, mine.z, src);
    e.w = __shfl_sync(kFull, mine.w, src);
    li.x = __shfl_sync(kFull, mi.x, src);
    li.y = __shfl_sync(kFull, mi.y, src);
    return src + 32 * qs;
}

// A lane's members of a chunk.  Slot base comes with the record; the slot
// count is the leader's (members share the leader's label set, bcrp.py:16-19).
template <int K>
struct ChunkLane {
    MemberRec r[K];
    bool valid[K];
    bool sp[K];
    bool tu[K];
};

// slot base / slot count of member record r (RCPP: one slot per state)
template <bool IDENT>
__device__ __forceinline__ int32_t slot_base(const MemberRec& r) {
    return IDENT ? r.x : r.y;
}

// Tag a chunk's members.  Loads are staged across the lane's members
// (records, then mark words) so the K dependency chains overlap instead of
// running back to back.
template <bool IDENT, int K>
__device__ __forceinline__ void chunk_tag(const SparseParams& p, int32_t l, int32_t bs, int32_t bz,
                                          int32_t ci0, int32_t ol, int32_t nrl, ChunkLane<K>& c) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int32_t i = ci0 + 32 * j + lane;
        c.valid[j] = i < bz;
        c.r[j] = c.valid[j] ? p.members[bs + i] : make_int4(0, 0, 0, 0);
    }
    if (IDENT) {
        const bool tl = get_bit(p.mark, l);
        uint32_t mw[K];
#pragma unroll
        for (int j = 0; j < K; ++j) mw[j] = c.valid[j] ? p.mark[c.r[j].x >> 5] : 0u;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            c.tu[j] = (mw[j] >> (c.r[j].x & 31)) & 1u;
            c.sp[j] = c.valid[j] && c.r[j].x != l && c.tu[j] != tl;
        }
        return;
    }
    bool tl;
    uint32_t lb;
    leader_marks<IDENT>(p, l, ol, nrl, tl, lb);
    uint32_t wa[K], wb[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        // the member's mark words in one wave of loads (they also tell
        // whether it is touched)
        const int32_t ou = c.r[j].y, w0 = ou >> 5, sh = ou & 31;
        const bool small = c.valid[j] && nrl > 0 && nrl <= 32;
        wa[j] = small ? p.mark[w0] : 0u;
        wb[j] = (small && sh + nrl > 32) ? p.mark[w0 + 1] : 0u;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int32_t ou = c.r[j].y, sh = ou & 31;
        bool sp = false, tu = false;
        if (c.valid[j] && nrl > 0) {
            if (nrl <= 32) {
                uint32_t v = wa[j] >> sh;
                if (sh + nrl > 32) v |= wb[j] << (32 - sh);
                if (nrl < 32) v &= (1u << nrl) - 1u;
                tu = v != 0u;
                sp = c.r[j].x != l && v != lb;
            } else {
                tu = slots_any(p.mark, ou, nrl);
                sp = c.r[j].x != l && (tu || tl) && slots_differ(p.mark, ou, ol, nrl);
            }
        }
        c.tu[j] = tu;
        c.sp[j] = sp;
    }
}

template <int K>
__device__ __forceinline__ void chunk_counts(const ChunkLane<K>& c, unsigned* bal, unsigned* kb,
                                             int32_t& nsplit, int32_t& nkeep, int32_t& wmin) {
    nsplit = nkeep = 0;
    int32_t m = kBig;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        bal[j] = __ballot_sync(kFull, c.sp[j]);
        kb[j] = __ballot_sync(kFull, c.valid[j] && !c.sp[j]);
        nsplit += __popc(bal[j]);
        nkeep += __popc(kb[j]);
        if (c.sp[j]) m = min(m, c.r[j].x);
    }
    wmin = __reduce_min_sync(kFull, m);
}

// Move the chunk's member records to their compacted positions (keep part
// first, split part at the tail of the block range); relabel split members.
template <int K>
__device__ __forceinline__ void chunk_compact(const SparseParams& p, int32_t l, int32_t bs, int32_t bz,
                                              int32_t ns, int32_t w, const ChunkLane<K>& c,
                                              const unsigned* bal, const unsigned* kb, int32_t nsplit,
                                              int32_t nkeep) {
    const int lane = threadIdx.x & 31;
    const int32_t keep = bz - ns;
    int32_t sbase = 0, kbase = 0;
    if (lane == 0) {
        if (nsplit) sbase = atomicAdd(&p.scur[l], nsplit);
        if (nkeep) kbase = atomicAdd(&p.kcur[l], nkeep);
    }
    sbase = __shfl_sync(kFull, sbase, 0);
    kbase = __shfl_sync(kFull, kbase, 0);
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (c.valid[j]) {
            const int32_t np = c.sp[j] ? bs + keep + sbase + __popc(bal[j] & lt) : bs + kbase + __popc(kb[j] & lt);
            p.members[np] = c.r[j];
            if (c.sp[j]) p.block[c.r[j].x] = w;
        }
        sbase += __popc(bal[j]);
        kbase += __popc(kb[j]);
    }
}

__device__ __forceinline__ void finish_block(const SparseParams& p, int cur, int64_t round, int32_t C,
                                             int32_t l, int32_t bs, int32_t bz, int32_t ns, int32_t w) {
    p.brange[l] = make_int2(bs, bz - ns);
    p.brange[w] = make_int2(bs + bz - ns, ns);
    raise_split(p, cur, round, l, w, C);
}

template <bool IDENT>
__device__ __forceinline__ void leader_slots(const SparseParams& p, int32_t l, int32_t& ol, int32_t& nrl) {
    if (IDENT) {
        ol = l;
        nrl = 1;
    } else {
        ol = p.off[l];
        nrl = p.off[l + 1] - ol;
    }
}

// two-pass, sub-phase 1: tag split members, accumulate count and minimum
template <bool IDENT, int K>
__device__ int32_t big_tag(const SparseParams& p, int32_t nbig, int32_t ci) {
    const int lane = threadIdx.x & 31;
    const int32_t k = find_owner<K>(p, nbig, ci);
    const int4 e = big_list_of<K>(p)[k];
    const int2 li = big_info_of<K>(p)[k];
    const int32_t l = e.x, bs = e.y, bz = e.z, ci0 = (ci - e.w) * (32 * K);
    const int32_t ol = li.x, nrl = li.y;
    ChunkLane<K> c;
    chunk_tag<IDENT, K>(p, l, bs, bz, ci0, ol, nrl, c);
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (!c.valid[j]) continue;
        MemberRec t = c.r[j];
        if (c.sp[j]) t.x = -1 - t.x;
        if (c.tu[j]) t.y |= (int32_t)0x80000000;  // touched: clear its marks in sub-phase 2
        p.tmp[(int64_t)ci * (32 * K) + 32 * j + lane] = t;  // chunk-major: see big_split
    }
    unsigned bal[K], kb[K];
    int32_t nsplit, nkeep, wmin;
    chunk_counts<K>(c, bal, kb, nsplit, nkeep, wmin);
    if (lane == 0 && nsplit) {
        red_add(&p.scnt[l], nsplit);
        red_min(&p.srec[l].smin, wmin);
    }
    return min(32 * K, bz - ci0);
}

// two-pass, sub-phase 2 (after a grid barrier): compact, relabel, clear
template <bool IDENT, int K>
__device__ void big_split(const SparseParams& p, int cur, int64_t round, int32_t C, int32_t nbig,
                          int32_t ci) {
    const int lane = threadIdx.x & 31;
    const int32_t k = find_owner<K>(p, nbig, ci);
    const int4 e = big_list_of<K>(p)[k];
    const int32_t l = e.x, bs = e.y, bz = e.z, ci0 = (ci - e.w) * (32 * K);
    const int32_t nrl = big_info_of<K>(p)[k].y;
    ChunkLane<K> c;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int32_t i = ci0 + 32 * j + lane;
        c.valid[j] = i < bz;
        // tmp is chunk-major (chunk ci at ci * 32K), so every heavy round
        // reuses the same few MB at the head of the array: its lines stay
        // in L2 from round to round instead of being written back to HBM
        MemberRec t = c.valid[j] ? p.tmp[(int64_t)ci * (32 * K) + 32 * j + lane] : make_int4(0, 0, 0, 0);
        c.sp[j] = c.valid[j] && t.x < 0;
        if (c.sp[j]) t.x = -1 - t.x;
        c.tu[j] = c.valid[j] && t.y < 0;
        t.y &= 0x7fffffff;
        c.r[j] = t;
    }
    const int32_t ns = p.scnt[l];  // final after the grid barrier
    if (ns) {
        unsigned bal[K], kb[K];
        int32_t nsplit, nkeep, wmin;
        chunk_counts<K>(c, bal, kb, nsplit, nkeep, wmin);
        const int32_t w = p.srec[l].smin;
        chunk_compact<K>(p, l, bs, bz, ns, w, c, bal, kb, nsplit, nkeep);
        if (ci0 == 0 && lane == 0) finish_block(p, cur, round, C, l, bs, bz, ns, w);
    }
#pragma unroll
    for (int j = 0; j < K; ++j)
        if (c.valid[j]) clear_member<IDENT>(p, c.r[j].x, c.tu[j], slot_base<IDENT>(c.r[j]), nrl);
    if (ci0 == 0 && lane == 0) red_and(&p.tblock[l >> 5], ~(1u << (l & 31)));
}

// ---- one pass with CTA-level aggregation ----------------------------------
//
// Every warp of the CTA calls this once per round (ci < 0: no big chunk).
// The chunks of one big block that land in the same CTA combine their split
// counts, minima and arrivals in shared memory first, so a block of N chunks
// costs one global arrival / count / cursor atomic per CTA it spans instead
// of one per chunk (N reaches thousands in the latency-bound rounds, where
// those same-address atomics serialise in L2).  Two __syncthreads: after
// tagging (counts published), and after the per-CTA cursor reservation.

// Packed arrival word of a big block (one-pass split): arrived chunks |
// split count | kept count.  One-pass blocks have at most tnw * 32 * kWide
// members (< 2^21 for any grid of up to 16K warps).
constexpr int kCntBits = 21;
constexpr unsigned long long kCntMask = (1ull << kCntBits) - 1ull;
constexpr int kArrShift = 2 * kCntBits;


struct OnePassSlot {
    int32_t key;     // big-list index of the warp's block, -1 if none
    int32_t nsplit;
    int32_t nkeep;
    int32_t wmin;
    int32_t sbase;   // cursor bases reserved by the CTA leader of the block
    int32_t kbase;
    int32_t ns;      // the block's split count and new leader, as the CTA leader saw them
    int32_t w;
};

// Kept members at bs + kbase + rank (from the head of the range), split
// members at bs + bz - 1 - (sbase + rank) (from its tail): together a
// permutation of the range whatever the split count.
template <int K>
__device__ __forceinline__ void chunk_place(const SparseParams& p, int32_t bs, int32_t bz, int32_t w,
                                            const ChunkLane<K>& c, const unsigned* bal, const unsigned* kb,
                                            int32_t sbase, int32_t kbase) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (c.valid[j]) {
            const int32_t np = c.sp[j] ? bs + bz - 1 - (sbase + __popc(bal[j] & lt)) : bs + kbase + __popc(kb[j] & lt);
            p.members[np] = c.r[j];
            if (c.sp[j]) p.block[c.r[j].x] = w;
        }
        sbase += __popc(bal[j]);
        kbase += __popc(kb[j]);
    }
    (void)lane;
}

template <bool IDENT, int K>
__device__ int32_t big_onepass_cta(const SparseParams& p, int cur, int64_t round, int32_t C, int32_t nbig,
                                   int32_t ci, OnePassSlot* slot) {
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const bool has = ci >= 0;
    int32_t k = -1, l = 0, bs = 0, bz = 0, ci0 = 0, ol = 0, nrl = 0;
    ChunkLane<K> c;
    unsigned bal[K], kb[K];
    int32_t nsplit = 0, nkeep = 0, wmin = kBig;
    if (has) {
        int4 e;
        int2 li;
        k = find_entry<K>(p, nbig, ci, e, li);
        l = e.x;
        bs = e.y;
        bz = e.z;
        ci0 = (ci - e.w) * (32 * K);
        ol = li.x;
        nrl = li.y;
        chunk_tag<IDENT, K>(p, l, bs, bz, ci0, ol, nrl, c);
        chunk_counts<K>(c, bal, kb, nsplit, nkeep, wmin);
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j) c.valid[j] = false;
    }
    trace_at(p, round, 8);
    if (lane == 0) {
        OnePassSlot& m = slot[wid];
        m.key = k;
        m.nsplit = nsplit;
        m.nkeep = nkeep;
        m.wmin = wmin;
    }
    __syncthreads();
    trace_at(p, round, 9);
    int32_t leader = wid, cnt_cta = 1, tot_s = nsplit, tot_k = nkeep, pre_s = 0, pre_k = 0, mn = wmin;
    int32_t ns = 0, w = kBig, nch_b = 1;
    if (has) {
        OnePassSlot o;  // one slot per warp of the CTA, one per lane
        if (lane < (int)(blockDim.x >> 5)) o = slot[lane];
        else o.key = -1;
        const bool same = o.key == k;
        const unsigned msk = __ballot_sync(kFull, same);
        leader = __ffs(msk) - 1;
        cnt_cta = __popc(msk);
        tot_s = __reduce_add_sync(kFull, same ? o.nsplit : 0);
        tot_k = __reduce_add_sync(kFull, same ? o.nkeep : 0);
        mn = __reduce_min_sync(kFull, same ? o.wmin : kBig);
        pre_s = __reduce_add_sync(kFull, (same && lane < wid) ? o.nsplit : 0);
        pre_k = __reduce_add_sync(kFull, (same && lane < wid) ? o.nkeep : 0);
        nch_b = (bz + 32 * K - 1) / (32 * K);
        if (nch_b > cnt_cta) {  // the block spans CTAs: combine globally
            if (lane == 0) {
                unsigned long long v = 0ull;
                if (wid == leader) {
                    // one acq_rel add on the block's packed word reserves the
                    // placement bases (kept members fill the range from the
                    // head, split members from the tail, so the bases do not
                    // depend on the block's split count), publishes the counts
                    // and arrives; the released minimum is visible with it
                    if (tot_s) red_min(&p.srec[l].smin, mn);
                    const unsigned long long add = ((unsigned long long)cnt_cta << kArrShift) |
                                                   ((unsigned long long)tot_s << kCntBits) | (unsigned)tot_k;
                    unsigned long long old;
                    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;"
                                 : "=l"(old) : "l"(&p.srec[l].arr), "l"(add) : "memory");
                    slot[wid].sbase = (int32_t)((old >> kCntBits) & kCntMask);
                    slot[wid].kbase = (int32_t)(old & kCntMask);
                }
                // only the CTA leader of the block polls the word; the
                // CTA's other warps of the block read its result after the
                // CTA barrier below
#ifdef BISIM_NO_SPIN1
                if (true) {
#else
                if (wid == leader) {
#endif
                    // the record's arrival word and minimum in one 16-byte
                    // acquire load (the last arriver's first load sees both)
                    int32_t mw = kBig;
                    do {
                        unsigned w0, w1, w2, w3;
                        asm volatile(
                            "{\n\t.reg .b128 t;\n\tld.acquire.gpu.global.b128 t, [%4];\n\t"
                            "mov.b128 {%0, %1, %2, %3}, t;\n\t}"
                            : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3)
                            : "l"(&p.srec[l])
                            : "memory");
                        (void)w3;
                        v = ((unsigned long long)w1 << 32) | w0;
                        mw = (int32_t)w2;
#if BISIM_POLL_NS > 0
                        if ((int32_t)(v >> kArrShift) < nch_b) __nanosleep(BISIM_POLL_NS);
#endif
                    } while ((int32_t)(v >> kArrShift) < nch_b);
                    ns = (int32_t)((v >> kCntBits) & kCntMask);
                    w = ns ? mw : kBig;
                    if (wid == leader) {
                        slot[wid].ns = ns;
                        slot[wid].w = w;
                    }
                }
            }
        } else {
            ns = tot_s;
            w = mn;
            if (wid == leader && lane == 0) {
                slot[wid].sbase = 0;
                slot[wid].kbase = 0;
            }
        }
        trace_at(p, round, 10);
    }
    __syncthreads();
    trace_at(p, round, 11);
    if (has && nch_b > cnt_cta) {
        ns = slot[leader].ns;
        w = slot[leader].w;
    }
    if (has) {
        if (ns) {
            const int32_t sb = slot[leader].sbase + pre_s, kbs = slot[leader].kbase + pre_k;
            chunk_place<K>(p, bs, bz, w, c, bal, kb, sb, kbs);
            if (ci0 == 0 && lane == 0) finish_block(p, cur, round, C, l, bs, bz, ns, w);
        }
        // every chunk of the block has read the leader's marks before anyone
        // clears: the arrivals above are complete (or the block is in this CTA)
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (c.valid[j]) clear_member<IDENT>(p, c.r[j].x, c.tu[j], slot_base<IDENT>(c.r[j]), nrl);
        if (ci0 == 0 && lane == 0) red_and(&p.tblock[l >> 5], ~(1u << (l & 31)));
        trace_at(p, round, 12);
        return min(32 * K, bz - ci0);
    }
    return 0;
}

