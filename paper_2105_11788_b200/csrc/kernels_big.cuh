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

template <int K>
struct ChunkLane {
    int32_t u[K];
    int32_t ou[K];
    int32_t nr[K];
    bool valid[K];
    bool sp[K];
    bool tu[K];
};

// Tag a chunk's members.  Loads are staged across the lane's members
// (member ids, then touched bits and slot offsets, then mark words) so the
// K dependency chains overlap instead of running back to back.
template <bool IDENT, int K>
__device__ __forceinline__ void chunk_tag(const SparseParams& p, int32_t l, int32_t bs, int32_t bz,
                                          int32_t ci0, ChunkLane<K>& c) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int32_t i = ci0 + 32 * j + lane;
        c.valid[j] = i < bz;
        c.u[j] = c.valid[j] ? p.members[bs + i] : 0;
    }
    if (IDENT) {
        const bool tl = get_bit(p.mark, l);
        uint32_t mw[K];
#pragma unroll
        for (int j = 0; j < K; ++j) mw[j] = c.valid[j] ? p.mark[c.u[j] >> 5] : 0u;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            c.tu[j] = (mw[j] >> (c.u[j] & 31)) & 1u;
            c.ou[j] = c.u[j];
            c.nr[j] = 1;
            c.sp[j] = c.valid[j] && c.u[j] != l && c.tu[j] != tl;
        }
        return;
    }
    const int32_t ol = p.off[l], nrl = p.off[l + 1] - ol;
    const bool tl = get_bit(p.touched, l);
    uint32_t tw[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        tw[j] = c.valid[j] ? p.touched[c.u[j] >> 5] : 0u;
        c.ou[j] = c.valid[j] ? p.off[c.u[j]] : 0;
        c.nr[j] = c.valid[j] ? p.off[c.u[j] + 1] - c.ou[j] : 0;
    }
    // members share the leader's label set, hence its slot count (bcrp.py:16-19)
    const uint32_t lb = (nrl > 0 && nrl <= 32) ? get_bits(p.mark, ol, nrl) : 0u;
    uint32_t wa[K], wb[K];
    bool need[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        c.tu[j] = (tw[j] >> (c.u[j] & 31)) & 1u;
        need[j] = c.valid[j] && c.u[j] != l && (c.tu[j] || tl) && c.nr[j] > 0;
        const int32_t w0 = c.ou[j] >> 5, sh = c.ou[j] & 31;
        wa[j] = need[j] ? p.mark[w0] : 0u;
        wb[j] = (need[j] && sh + c.nr[j] > 32) ? p.mark[w0 + 1] : 0u;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
        bool sp = false;
        if (need[j]) {
            const int32_t nr = c.nr[j], sh = c.ou[j] & 31;
            if (nr <= 32) {
                uint32_t v = wa[j] >> sh;
                if (sh + nr > 32) v |= wb[j] << (32 - sh);
                if (nr < 32) v &= (1u << nr) - 1u;
                sp = v != lb;
            } else {
                sp = slots_differ(p.mark, c.ou[j], ol, nr);
            }
        }
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
        if (c.sp[j]) m = min(m, c.u[j]);
    }
    wmin = __reduce_min_sync(kFull, m);
}

// Move the chunk's members to their compacted positions (keep part first,
// split part at the tail of the block range) and relabel split members.
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
            p.members[np] = c.u[j];
            if (c.sp[j]) p.block[c.u[j]] = w;
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

// two-pass, sub-phase 1: tag split members, accumulate count and minimum
template <bool IDENT, int K>
__device__ int32_t big_tag(const SparseParams& p, int32_t nbig, int32_t ci) {
    const int lane = threadIdx.x & 31;
    const int4 e = big_list_of<K>(p)[find_owner<K>(p, nbig, ci)];
    const int32_t l = e.x, bs = e.y, bz = e.z, ci0 = (ci - e.w) * (32 * K);
    ChunkLane<K> c;
    chunk_tag<IDENT, K>(p, l, bs, bz, ci0, c);
#pragma unroll
    for (int j = 0; j < K; ++j)
        if (c.valid[j]) p.tmp[bs + ci0 + 32 * j + lane] = c.sp[j] ? -1 - c.u[j] : c.u[j];
    unsigned bal[K], kb[K];
    int32_t nsplit, nkeep, wmin;
    chunk_counts<K>(c, bal, kb, nsplit, nkeep, wmin);
    if (lane == 0 && nsplit) {
        atomicAdd(&p.scnt[l], nsplit);
        atomicMin(&p.smin[l], wmin);
    }
    return min(32 * K, bz - ci0);
}

// two-pass, sub-phase 2 (after a grid barrier): compact, relabel, clear
template <bool IDENT, int K>
__device__ void big_split(const SparseParams& p, int cur, int64_t round, int32_t C, int32_t nbig,
                          int32_t ci) {
    const int lane = threadIdx.x & 31;
    const int4 e = big_list_of<K>(p)[find_owner<K>(p, nbig, ci)];
    const int32_t l = e.x, bs = e.y, bz = e.z, ci0 = (ci - e.w) * (32 * K);
    ChunkLane<K> c;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int32_t i = ci0 + 32 * j + lane;
        c.valid[j] = i < bz;
        const int32_t code = c.valid[j] ? p.tmp[bs + i] : 0;
        c.sp[j] = c.valid[j] && code < 0;
        c.u[j] = c.sp[j] ? -1 - code : code;
    }
    const int32_t ns = p.scnt[l];
    if (ns) {
        unsigned bal[K], kb[K];
        int32_t nsplit, nkeep, wmin;
        chunk_counts<K>(c, bal, kb, nsplit, nkeep, wmin);
        const int32_t w = p.smin[l];
        chunk_compact<K>(p, l, bs, bz, ns, w, c, bal, kb, nsplit, nkeep);
        if (ci0 == 0 && lane == 0) finish_block(p, cur, round, C, l, bs, bz, ns, w);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (!c.valid[j]) continue;
        const int32_t u = c.u[j];
        bool tu;
        int32_t ou = 0, nr = 0;
        if (IDENT) {
            tu = get_bit(p.mark, u);
            ou = u;
            nr = 1;
        } else {
            tu = get_bit(p.touched, u);
            if (tu) {
                ou = p.off[u];
                nr = p.off[u + 1] - ou;
            }
        }
        clear_member<IDENT>(p, u, tu, ou, nr);
    }
    if (ci0 == 0 && lane == 0) atomicAnd(&p.tblock[l >> 5], ~(1u << (l & 31)));
}

// one pass (every item on its own warp)
template <bool IDENT, int K>
__device__ int32_t big_onepass(const SparseParams& p, int cur, int64_t round, int32_t C, int32_t nbig,
                               int32_t ci) {
    const int lane = threadIdx.x & 31;
    const int4 e = big_list_of<K>(p)[find_owner<K>(p, nbig, ci)];
    const int32_t l = e.x, bs = e.y, bz = e.z, ci0 = (ci - e.w) * (32 * K);
    ChunkLane<K> c;
    chunk_tag<IDENT, K>(p, l, bs, bz, ci0, c);
    unsigned bal[K], kb[K];
    int32_t nsplit, nkeep, wmin;
    chunk_counts<K>(c, bal, kb, nsplit, nkeep, wmin);
    const int32_t nch_b = (bz + 32 * K - 1) / (32 * K);
    int32_t ns = nsplit, w = wmin;
    if (nch_b > 1) {
        if (lane == 0) {
            if (nsplit) {
                atomicAdd(&p.scnt[l], nsplit);
                atomicMin(&p.smin[l], wmin);
            }
            __threadfence();
            atomicAdd(&p.sarr[l], 1);
            while (ld_acquire_u32((const unsigned*)&p.sarr[l]) < (unsigned)nch_b) {
            }
            ns = ld_vol(&p.scnt[l]);
            w = ld_vol(&p.smin[l]);
        }
        ns = __shfl_sync(kFull, ns, 0);
        w = __shfl_sync(kFull, w, 0);
    }
    if (ns) {
        chunk_compact<K>(p, l, bs, bz, ns, w, c, bal, kb, nsplit, nkeep);
        if (ci0 == 0 && lane == 0) finish_block(p, cur, round, C, l, bs, bz, ns, w);
    }
    // every chunk has read the leader's marks before anyone clears: the
    // arrival count above is complete (or the block is a single chunk)
#pragma unroll
    for (int j = 0; j < K; ++j)
        if (c.valid[j]) clear_member<IDENT>(p, c.u[j], c.tu[j], c.ou[j], c.nr[j]);
    if (ci0 == 0 && lane == 0) atomicAnd(&p.tblock[l >> 5], ~(1u << (l & 31)));
    return min(32 * K, bz - ci0);
}

