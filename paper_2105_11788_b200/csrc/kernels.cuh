// kernels.cuh -- device code of libbisim.so (sm_100a).
//
// The refinement path of arXiv 2105.11788 restated for a B200:
//
//   preprocessing      bcrp.py:49-126   label masks, slot ranks, offsets, reverse CSR
//   label partition    bcrp.py:144-184  |Act| mark-and-split rounds (one cooperative kernel)
//   refinement loop    bcrp.py:286-315 / rcpp.py:240-259  one cooperative persistent kernel
//
// Priority writes (pram.py:153-154, "lowest processor wins") become order-
// independent atomics: C = min unstable label via atomicMin, leader
// elections via a 64-bit atomicMax on (epoch << 32 | INT32_MAX - s), so a
// newer round always beats a stale entry (the reference never clears
// new_leader, bcrp.py:225) and within a round the smallest state wins.
#pragma once

#include <cooperative_groups.h>
#include <cstdint>

namespace bisim {
namespace cg = cooperative_groups;

constexpr int32_t kBig = 0x7fffffff;  // "no label" inside min-reductions (NONE_LABEL, rcpp.py:35)
constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 512;  // persistent-kernel CTA size

// Control block shared by the persistent kernel's CTAs (global memory).
struct Ctrl {
    int32_t scan_min;     // entry-time min unstable label
    int32_t done;         // terminal pass reached (C == NONE)
    int32_t error;        // BISIM_GUARD when the superstep guard fires
    int32_t bad;          // invalid input seen by a preprocessing kernel
    int64_t round;        // completed main-loop rounds
    int64_t guard_count;  // engine superstep counter at the guard trip
    int32_t next_min[2];  // min label raised unstable in round r (buffer r & 1)
    int32_t succ[2];      // min label of unstable \ {C} in round r
    int32_t n_split[2];   // split-list length of round r
    int32_t n_cmem[2];    // C-member list length of round r
    int32_t count;        // scratch counter (leader counts)
    int32_t pad;
    unsigned long long work_edges;   // sum over rounds of in-edges of C
    unsigned long long work_splits;  // sum over rounds of split states
};

struct LoopParams {
    int32_t n;
    int32_t A;              // |Act|: label rounds already on the engine counter
    int32_t reflag_c;       // BCRP re-raises C after any split (bcrp.py:282); RCPP does not
    int32_t has_guard;
    int64_t max_supersteps;
    int64_t round_limit;    // rounds this launch may run (stepped mode: 1)
    int64_t splits_cap;
    const int32_t* __restrict__ off;       // n+1 slot offsets (BCRP)
    const int32_t* __restrict__ rev_ptr;   // n+1 reverse-CSR row pointers (by target)
    const int32_t* __restrict__ rev_slot;  // m   mark slot of each in-edge
    int32_t* block;
    unsigned long long* nl;  // election keys, indexed by block label
    uint32_t* mark;          // L-bit mark bitmap (+1 pad word)
    uint32_t* unstable;      // n-bit unstable bitmap
    int32_t* split_list;
    int32_t* cmem;
    int32_t* splits;
    Ctrl* ctrl;
};

__device__ __forceinline__ unsigned long long elect_key(int64_t epoch, int32_t s) {
    return ((unsigned long long)epoch << 32) | (unsigned)(kBig - s);
}
__device__ __forceinline__ int32_t elect_winner(unsigned long long key) {
    return kBig - (int32_t)(unsigned)(key & 0xffffffffull);
}
// Fire-and-forget reductions (REDG): unlike atomicOr/And/Min with an unused
// result, which compile to returning ATOMG, these never hold a scoreboard.
__device__ __forceinline__ void red_or(uint32_t* a, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_and(uint32_t* a, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.and.b32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_min(int32_t* a, int32_t v) {
    asm volatile("red.relaxed.gpu.global.min.s32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_min_u32(uint32_t* a, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add(int32_t* a, int32_t v) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void set_bit(uint32_t* bm, int32_t i) {
    atomicOr(&bm[i >> 5], 1u << (i & 31));
}
__device__ __forceinline__ uint32_t get_bit(const uint32_t* bm, int32_t i) {
    return (bm[i >> 5] >> (i & 31)) & 1u;
}
template <typename T>
__device__ __forceinline__ T ld_vol(const T* p) {
    return *(const volatile T*)p;
}
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

// len (1..32) bits of bm starting at bit pos
__device__ __forceinline__ uint32_t get_bits(const uint32_t* bm, int32_t pos, int32_t len) {
    const int32_t w = pos >> 5, sh = pos & 31;
    uint32_t v = bm[w] >> sh;
    if (sh + len > 32) v |= bm[w + 1] << (32 - sh);
    return len == 32 ? v : (v & ((1u << len) - 1u));
}

// Any mark among the nr slots starting at pos (a state is "touched" this
// round iff one of its slots is marked; no separate bitmap is kept).
__device__ __forceinline__ bool slots_any(const uint32_t* mark, int32_t pos, int32_t nr) {
    for (int32_t k = 0; k < nr; k += 32)
        if (get_bits(mark, pos + k, min(32, nr - k))) return true;
    return false;
}

// BCRP split test (bcrp.py:260-265) restated per state: s differs from its
// leader l on some label slot k < nr (same label set => same slot layout).
__device__ __forceinline__ bool slots_differ(const uint32_t* mark, int32_t os, int32_t ol,
                                             int32_t nr) {
    for (int32_t k = 0; k < nr; k += 32) {
        const int32_t len = min(32, nr - k);
        if (get_bits(mark, os + k, len) != get_bits(mark, ol + k, len)) return true;
    }
    return false;
}

// ---------------------------------------------------------------------------
// Preprocessing (bcrp.py:49-126)
// ---------------------------------------------------------------------------

// Per-state label masks: lmask[w * n + s] bit b <=> s has an outgoing
// transition labelled 64 w + b.  Word-major so each label round reads one
// coalesced plane.  Validates transitions (lts.py:47-52).  Warp-aggregated:
// lanes hitting the same mask word OR their bits together first.
// Runs of equal keys on consecutive lanes.  Transition files are usually
// grouped by source, so such runs collapse to one atomic each; on random
// input this costs a shuffle and a ballot (cheaper than __match_any_sync).
struct LaneRun {
    int leader;  // first lane of my run
    int rank;    // my position in the run
    int len;     // run length
    int next;    // first lane after my run
};

template <typename T>
__device__ __forceinline__ LaneRun lane_run(T key) {
    const int lane = threadIdx.x & 31;
    const T prev = __shfl_up_sync(kFull, key, 1);
    const unsigned starts = __ballot_sync(kFull, lane == 0 || prev != key);
    const unsigned le = (2u << lane) - 1u;  // lanes <= me (wraps to all lanes for lane 31)
    LaneRun r;
    r.leader = 31 - __clz(starts & le);
    r.rank = lane - r.leader;
    const unsigned after = starts & ~le;
    r.next = after ? __ffs(after) - 1 : 32;
    r.len = r.next - r.leader;
    return r;
}

// OR of v over my run, valid in the run's leader lane
__device__ __forceinline__ unsigned long long run_or(unsigned long long v, const LaneRun& r) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_down_sync(kFull, v, d);
        if (lane + d < r.next) v |= o;
    }
    return v;
}

// TA: int32_t, or uint8_t for actions narrowed on the host (|Act| <= 256)
template <typename TA = int32_t>
__global__ void k_label_mask(int32_t n, int64_t m, int32_t A, const int32_t* __restrict__ src,
                             const TA* __restrict__ act, const int32_t* __restrict__ dst,
                             unsigned long long* lmask, Ctrl* ctrl) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < m; i0 += stride) {
        const int64_t i = i0 + lane;
        bool ok = false;
        unsigned long long addr = ~0ull - lane, bits = 0;
        if (i < m) {
            const int32_t s = src[i], a = (int32_t)act[i], t = dst[i];
            ok = (unsigned)s < (unsigned)n && (unsigned)t < (unsigned)n && (unsigned)a < (unsigned)A;
            if (ok) {
                addr = (unsigned long long)(a >> 6) * n + s;
                bits = 1ull << (a & 63);
            } else {
                ctrl->bad = 1;
            }
        }
        const LaneRun r = lane_run(addr);
        bits = run_or(bits, r);
        // fire-and-forget (a 64-bit atomicOr with an unused result still
        // compiles to a returning ATOMG that stalls the warp)
        if (ok && r.rank == 0)
            asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(&lmask[addr]), "l"(bits) : "memory");
    }
}

// RCPP input validation (rcpp.py:49-55) -- edges in range.
__global__ void k_check_edges(int32_t n, int64_t m, const int32_t* __restrict__ src,
                              const int32_t* __restrict__ dst, Ctrl* ctrl) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        if ((unsigned)src[i] >= (unsigned)n || (unsigned)dst[i] >= (unsigned)n) ctrl->bad = 1;
}

// pi0 must be a leader-form partition (lts.py:88-94).
__global__ void k_check_pi0(int32_t n, const int32_t* __restrict__ pi0, Ctrl* ctrl) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = pi0[s];
        if ((unsigned)b >= (unsigned)n || pi0[b] != b) ctrl->bad = 1;
    }
}

// nr_marks[s] = number of distinct outgoing labels (bcrp.py:105-106)
__global__ void k_nr_marks(int32_t n, int32_t W, const unsigned long long* __restrict__ lmask,
                           int32_t* nr) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = 0;
        for (int32_t w = 0; w < W; ++w) c += __popcll(lmask[(int64_t)w * n + s]);
        nr[s] = c;
    }
}

// rank of label a among s's labels = order_i (bcrp.py:99-104)
__device__ __forceinline__ int32_t label_rank(const unsigned long long* __restrict__ lmask,
                                              int32_t n, int32_t s, int32_t a) {
    const int32_t w = a >> 6;
    int32_t r = __popcll(lmask[(int64_t)w * n + s] & ((1ull << (a & 63)) - 1ull));
    for (int32_t u = 0; u < w; ++u) r += __popcll(lmask[(int64_t)u * n + s]);
    return r;
}

__global__ void k_order(int32_t n, int64_t m, const int32_t* __restrict__ src,
                        const int32_t* __restrict__ act, const unsigned long long* __restrict__ lmask,
                        int32_t* order) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        order[i] = label_rank(lmask, n, src[i], act[i]);
}

// preprocess() export: radix-sort keys source * |Act| + action with the
// transition index as payload (a stable sort by (source, action),
// bcrp.py:49-52).
__global__ void k_sort_keys(int64_t m, int32_t A, const int32_t* __restrict__ src,
                            const int32_t* __restrict__ act, unsigned long long* keys, int32_t* idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (unsigned long long)src[i] * (unsigned long long)(A > 0 ? A : 1) + (unsigned)act[i];
        idx[i] = (int32_t)i;
    }
}

// Tables of the sorted transition list (BcrpAux, bcrp.py:116-126): sorted
// columns, action_switch[k] = same source and a different action than
// transition k-1 (bcrp.py:55-65), order[k] = rank of the action among the
// source's labels -- the segmented inclusive scan of action_switch
// (bcrp.py:68-104) restated as a popcount of lower label bits.
__global__ void k_sorted_tables(int32_t n, int64_t m, const int32_t* __restrict__ perm,
                                const int32_t* __restrict__ src, const int32_t* __restrict__ act,
                                const int32_t* __restrict__ dst, const unsigned long long* __restrict__ lmask,
                                int32_t* s_src, int32_t* s_act, int32_t* s_dst, int32_t* s_sw, int32_t* s_ord) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = perm[k];
        const int32_t s = src[i], a = act[i];
        s_src[k] = s;
        s_act[k] = a;
        if (dst) s_dst[k] = dst[i];
        int32_t sw = 0;
        if (k > 0) {
            const int32_t p = perm[k - 1];
            sw = (src[p] == s && act[p] != a) ? 1 : 0;
        }
        s_sw[k] = sw;
        s_ord[k] = label_rank(lmask, n, s, a);
    }
}

// in-degree histogram, warp-aggregated on equal targets
// In-degrees; with src != nullptr only transitions whose source lies in
// [lo, hi) count (one shard of the transition-sharded mode).
__global__ void k_indeg(int64_t m, const int32_t* __restrict__ dst, int32_t* cnt,
                        const int32_t* __restrict__ src = nullptr, int32_t lo = 0, int32_t hi = 0) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < m; i0 += stride) {
        const int64_t i = i0 + lane;
        bool in = i < m;
        if (in && src) {
            const int32_t s = src[i];
            in = s >= lo && s < hi;
        }
        const int32_t t = in ? dst[i] : -1 - lane;
        const LaneRun r = lane_run(t);
        if (in && r.rank == 0) atomicAdd(&cnt[t], r.len);
    }
}

// Reverse CSR fill: rev_slot[pos] = mark slot of in-edge (bcrp.py:219 slot =
// off[src] + order).  RCPP: slot = src (one mark per state, rcpp.py:126).
template <bool BCRP>
__global__ void k_rev_fill(int32_t n, int64_t m, const int32_t* __restrict__ src,
                           const int32_t* __restrict__ act, const int32_t* __restrict__ dst,
                           const unsigned long long* __restrict__ lmask,
                           const int32_t* __restrict__ off, int32_t* cursor, int32_t* rev_slot) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < m; i0 += stride) {
        const int64_t i = i0 + lane;
        int32_t t = -1 - lane, slot = 0;
        if (i < m) {
            t = dst[i];
            const int32_t s = src[i];
            slot = BCRP ? off[s] + label_rank(lmask, n, s, act[i]) : s;
        }
        const unsigned grp = __match_any_sync(kFull, t);
        const int leader = __ffs(grp) - 1;
        int32_t base = 0;
        if (i < m && lane == leader) base = atomicAdd(&cursor[t], __popc(grp));
        base = __shfl_sync(kFull, base, leader);
        if (i < m) rev_slot[base + __popc(grp & lanemask_lt())] = slot;
    }
}

// ---------------------------------------------------------------------------
// Exclusive scan of int32 counts (d[0..N) -> prefix, d[N] = total)
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256, kScanItems = 16, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* total) {
    __shared__ int64_t warp_sums[kScanThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(kFull, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kScanThreads / 32) warp_sums[lane] = w;
    }
    __syncthreads();
    const int64_t before = (wid ? warp_sums[wid - 1] : 0) + x - v;
    *total = warp_sums[kScanThreads / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void k_scan_tiles(const int32_t* __restrict__ d, int64_t N, int64_t* tile_sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < N) s += d[base + k];
    int64_t total;
    block_excl_scan(s, &total);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

__global__ void k_scan_sums(int64_t* tile_sums, int64_t ntiles) {
    // one CTA of kScanThreads: serial chunk per thread + block scan
    const int64_t per = (ntiles + kScanThreads - 1) / kScanThreads;
    const int64_t b = threadIdx.x * per;
    int64_t s = 0;
    for (int64_t k = 0; k < per; ++k)
        if (b + k < ntiles) s += tile_sums[b + k];
    int64_t total;
    int64_t run = block_excl_scan(s, &total);
    for (int64_t k = 0; k < per; ++k)
        if (b + k < ntiles) {
            const int64_t v = tile_sums[b + k];
            tile_sums[b + k] = run;
            run += v;
        }
}

__global__ void k_scan_apply(int32_t* d, int64_t N, const int64_t* __restrict__ tile_sums) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int32_t v[kScanItems];
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < N ? d[base + k] : 0;
        s += v[k];
    }
    int64_t total;
    int64_t run = block_excl_scan(s, &total) + tile_sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < N) {
            d[base + k] = (int32_t)run;
            run += v[k];
        }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) d[N] = (int32_t)(tile_sums[blockIdx.x] + total);
}

// ---------------------------------------------------------------------------
// Partition bookkeeping
// ---------------------------------------------------------------------------
__global__ void k_count_leaders(int32_t n, const int32_t* __restrict__ block, int32_t* count) {
    int32_t c = 0;
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x)
        c += block[s] == s;
    c = __reduce_add_sync(kFull, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// unstable[leader] := true for every initial block (bcrp.py:226-229, rcpp.py:68-70)
__global__ void k_init_unstable(int32_t n, const int32_t* __restrict__ block, uint32_t* unstable) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t s0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); s0 < n; s0 += stride) {
        const int64_t s = s0 + lane;
        const unsigned bal = __ballot_sync(kFull, s < n && block[s] == s);
        if (lane == 0 && bal) unstable[s0 >> 5] = bal;  // s0 is a multiple of 32
    }
}

__global__ void k_ctrl_reset(Ctrl* c) {
    c->scan_min = kBig;
    c->done = 0;
    for (int k = 0; k < 2; ++k) {
        c->next_min[k] = kBig;
        c->succ[k] = kBig;
        c->n_split[k] = 0;
        c->n_cmem[k] = 0;
    }
}

// ---------------------------------------------------------------------------
// Label pre-partition (bcrp.py:144-184): |Act| rounds, each "mark states
// carrying label a, split blocks whose members disagree with their leader,
// min-index new leader".  Marks are read straight from the label masks.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_label_rounds(int32_t n, int32_t A,
                                                           const unsigned long long* __restrict__ lmask,
                                                           int32_t* block, unsigned long long* nl) {
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    for (int32_t a = 0; a < A; ++a) {
        const unsigned long long* plane = lmask + (int64_t)(a >> 6) * n;
        const int sh = a & 63;
        const int64_t epoch = a + 1;
        // elect (bcrp.py:176-182)
        for (int64_t s = gtid; s < n; s += gsize) {
            const int32_t l = block[s];
            if (l != s && (((plane[s] ^ plane[l]) >> sh) & 1ull)) atomicMax(&nl[l], elect_key(epoch, (int32_t)s));
        }
        grid.sync();
        // reassign (bcrp.py:155-160)
        for (int64_t s = gtid; s < n; s += gsize) {
            const int32_t l = block[s];
            if (l != s && (((plane[s] ^ plane[l]) >> sh) & 1ull)) block[s] = elect_winner(nl[l]);
        }
        grid.sync();
    }
}

// The same rounds under the plain Common policy (no Alg. 6 election,
// bcrp.py:176-182 with common_election=False): a round's elect phase is
// illegal as soon as two states of one block disagree with their leader
// (pram.py:147-152).  Until that happens the Priority rounds above are the
// Common rounds, and a block's disagreeing states are exactly the states
// that move to its new leader w -- so the first round in which two states
// move to the same w is the first conflict.  w is a fresh label (a state
// becomes a leader once), so per-w move counters never need a reset.
// conf[0] = first conflicting round (INT32_MAX if none); conf_key = min over
// conflicting blocks of (w << 32 | old leader): the reference raises for
// the address ("new_leader", old leader) of the block whose smallest
// disagreeing state is smallest (first group in processor order).
__global__ void __launch_bounds__(kThreads) k_label_rounds_common(int32_t n, int32_t A,
                                                                  const unsigned long long* __restrict__ lmask,
                                                                  int32_t* block, unsigned long long* nl,
                                                                  int32_t* moved, int32_t* conf,
                                                                  unsigned long long* conf_key) {
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    for (int32_t a = 0; a < A; ++a) {
        const unsigned long long* plane = lmask + (int64_t)(a >> 6) * n;
        const int sh = a & 63;
        const int64_t epoch = a + 1;
        for (int64_t s = gtid; s < n; s += gsize) {
            const int32_t l = block[s];
            if (l != s && (((plane[s] ^ plane[l]) >> sh) & 1ull)) atomicMax(&nl[l], elect_key(epoch, (int32_t)s));
        }
        grid.sync();
        for (int64_t s = gtid; s < n; s += gsize) {
            const int32_t l = block[s];
            if (l != s && (((plane[s] ^ plane[l]) >> sh) & 1ull)) {
                const int32_t w = elect_winner(nl[l]);
                block[s] = w;
                if (atomicAdd(&moved[w], 1) == 1) {  // the second mover: a conflicting block
                    atomicMin(conf, a);
                    atomicMin(conf_key, ((unsigned long long)(uint32_t)w << 32) | (uint32_t)l);
                }
            }
        }
        grid.sync();
        if (ld_vol(conf) <= a) break;
    }
}

// ---------------------------------------------------------------------------
// Refinement loop (Alg. 3 / Alg. 2) as one persistent cooperative kernel.
//
// Round r with splitter C, three grid-wide phases:
//   P1 mark   every state t with block[t] == C marks the slots of its in-edges
//             (bcrp.py:255-258 restated per target via the reverse CSR) and is
//             recorded in the C-member list; concurrently the successor of C
//             in the unstable set is found.
//   P2 tag    every state compares its slots with its leader's (bcrp.py:260-265,
//             rcpp.py:200); split states are listed and elect the min-index new
//             leader (sub_a, bcrp.py:267-272); unstable[C] is cleared.
//   P3 split  split states move to their block's winner and raise old/new
//             labels (sub_b, bcrp.py:274-283); BCRP re-raises C after any split;
//             marks are cleared through the C-member list.
// The next splitter is min(successor of C, min raised label): the Priority
// "lowest unstable label" of the next select phase (bcrp.py:241-242).
// ---------------------------------------------------------------------------
template <bool IDENT>  // IDENT: one mark slot per state (RCPP)
__global__ void __launch_bounds__(kThreads) k_refine(LoopParams p) {
    cg::grid_group grid = cg::this_grid();
    Ctrl* ctl = p.ctrl;
    const int lane = threadIdx.x & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    const int64_t wbase = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    const int32_t n = p.n;
    const int64_t nwords = ((int64_t)n + 31) >> 5;

    for (int64_t w = gtid; w < nwords; w += gsize) {
        const uint32_t v = p.unstable[w];
        if (v) atomicMin(&ctl->scan_min, (int32_t)(w * 32 + __ffs(v) - 1));
    }
    grid.sync();
    int32_t C = ld_vol(&ctl->scan_min);
    int64_t round = ld_vol(&ctl->round);
    unsigned long long my_edges = 0;

    for (int64_t done_here = 0;; ++done_here) {
        if (done_here == p.round_limit) break;
        const int64_t steps = (int64_t)p.A + round + 1;  // PramEngine.begin_superstep
        if (p.has_guard && steps > p.max_supersteps) {
            if (gtid == 0) {
                ctl->error = 2;
                ctl->guard_count = steps;
            }
            break;
        }
        if (C == kBig) {  // select found no unstable block (bcrp.py:293)
            if (gtid == 0) ctl->done = 1;
            break;
        }
        const int cur = (int)(round & 1), nxt = cur ^ 1;
        const int64_t epoch = (int64_t)p.A + round + 1;

        // ---- P1: mark ----------------------------------------------------
        for (int64_t s0 = wbase; s0 < n; s0 += gsize) {
            const int64_t s = s0 + lane;
            const bool inC = s < n && p.block[s] == C;
            const unsigned bal = __ballot_sync(kFull, inC);
            if (bal) {
                int32_t base = 0;
                if (lane == 0) base = atomicAdd(&ctl->n_cmem[cur], __popc(bal));
                base = __shfl_sync(kFull, base, 0);
                if (inC) {
                    p.cmem[base + __popc(bal & lanemask_lt())] = (int32_t)s;
                    const int32_t e0 = p.rev_ptr[s], e1 = p.rev_ptr[s + 1];
                    my_edges += (unsigned long long)(e1 - e0);
                    for (int32_t j = e0; j < e1; ++j) {
                        const int32_t sl = p.rev_slot[j];
                        atomicOr(&p.mark[sl >> 5], 1u << (sl & 31));
                    }
                }
            }
        }
        // successor of C in unstable \ {C}; every label below C is stable
        for (int64_t w = (C >> 5) + gtid; w < nwords; w += gsize) {
            uint32_t v = p.unstable[w];
            if (w == (C >> 5)) v &= ~(1u << (C & 31));
            if (v) atomicMin(&ctl->succ[cur], (int32_t)(w * 32 + __ffs(v) - 1));
        }
        grid.sync();

        // ---- P2: tag + elect ---------------------------------------------
        if (gtid == 0) {
            atomicAnd(&p.unstable[C >> 5], ~(1u << (C & 31)));  // sub_a: unstable[C] := false
            ctl->next_min[nxt] = kBig;
            ctl->succ[nxt] = kBig;
            ctl->n_split[nxt] = 0;
            ctl->n_cmem[nxt] = 0;
        }
        for (int64_t s0 = wbase; s0 < n; s0 += gsize) {
            const int64_t s = s0 + lane;
            bool sp = false;
            int32_t l = 0;
            if (s < n) {
                l = p.block[s];
                if (l != s) {  // a leader compares with itself and never splits
                    if (IDENT) {
                        sp = get_bit(p.mark, (int32_t)s) != get_bit(p.mark, l);
                    } else {
                        const int32_t o = p.off[s], nr = p.off[s + 1] - o;
                        if (nr) sp = slots_differ(p.mark, o, p.off[l], nr);
                    }
                }
            }
            const unsigned bal = __ballot_sync(kFull, sp);
            if (bal) {
                int32_t base = 0;
                if (lane == 0) base = atomicAdd(&ctl->n_split[cur], __popc(bal));
                base = __shfl_sync(kFull, base, 0);
                if (sp) {
                    p.split_list[base + __popc(bal & lanemask_lt())] = (int32_t)s;
                    atomicMax(&p.nl[l], elect_key(epoch, (int32_t)s));
                }
            }
        }
        grid.sync();

        // ---- P3: split ---------------------------------------------------
        const int32_t ns = ld_vol(&ctl->n_split[cur]);
        for (int64_t i = gtid; i < ns; i += gsize) {
            const int32_t s = p.split_list[i];
            const int32_t old = p.block[s];
            const int32_t w = elect_winner(p.nl[old]);
            p.block[s] = w;
            set_bit(p.unstable, old);
            set_bit(p.unstable, w);
            if (s == w && round < p.splits_cap) atomicAdd(&p.splits[round], 1);
            atomicMin(&ctl->next_min[cur], min(old, w));
        }
        if (gtid == 0) {
            if (p.reflag_c && ns > 0) {
                set_bit(p.unstable, C);
                atomicMin(&ctl->next_min[cur], C);
            }
            atomicAdd(&ctl->work_splits, (unsigned long long)ns);
        }
        const int32_t nc = ld_vol(&ctl->n_cmem[cur]);
        for (int64_t i = gtid; i < nc; i += gsize) {
            const int32_t t = p.cmem[i];
            const int32_t e1 = p.rev_ptr[t + 1];
            for (int32_t j = p.rev_ptr[t]; j < e1; ++j) p.mark[p.rev_slot[j] >> 5] = 0u;
        }
        grid.sync();
        C = min(ld_vol(&ctl->next_min[cur]), ld_vol(&ctl->succ[cur]));
        ++round;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) my_edges += __shfl_xor_sync(kFull, my_edges, o);
    if (lane == 0 && my_edges) atomicAdd(&ctl->work_edges, my_edges);
    if (gtid == 0) ctl->round = round;
}

}  // namespace bisim
