// kernels_shard.cuh -- transition-sharded mode of the refinement loop
// (SURVEY.md §8e): one LTS, G replicas (one per GPU), in-edges split by
// SOURCE range.
//
// Every replica holds the whole partition state (block, members, ranges,
// unstable set) and runs the same rounds; only phase A's transition scan is
// divided: replica g walks the in-edges of C whose source lies in its range.
// Mark bits go to EVERY replica's buffers (fire-and-forget
// reductions over NVLink peer memory -- the paper's per-round mark-bitmap
// OR-reduction, done inside the persistent kernel instead of by a
// collective), and the touched blocks each replica registered first are
// published in a per-replica list.  One cross-replica barrier per round
// (arrival counters in peer memory, release/acquire at system scope) makes
// all marks visible; each replica then adopts the blocks the others
// published and runs phase B on its own copy.  Phase B is a deterministic
// function of (partition, marks), so the replicas stay identical.
//
// Round state written by remote replicas (marks, published
// lists) is double-buffered by round parity: a replica cannot reach round
// r + 2 before every replica has finished round r, so buffers of parity r & 1
// are only cleared and reused when nobody reads them.
//
// Included inside namespace bisim by kernels_sparse.cuh, before the loop.
#pragma once

// BISIM error code for a cross-replica wait that timed out (replicas not
// running concurrently); mapped to BISIM_CUDA on the host.
constexpr int32_t kShardTimeout = 5;

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// pl is the CTA's shared copy of the parameters: every thread reads it, so
// thread 0 switches the pointers between two CTA barriers.
__device__ __forceinline__ void shard_select_parity(SparseParams& pl, const SparseParams& pk, int cur) {
    __syncthreads();
    if (threadIdx.x == 0) {
        pl.mark = pk.mark + cur * pk.mark_stride;
        pl.tblock = pk.tblock + cur * pk.bm_stride;
    }
    __syncthreads();
}

// Mark slot `slot` in every replica.  (Combining the bits of lanes that hit
// the same word first -- match_any + reduce_or -- measured slower: BCRP and
// RCPP mark slots of one warp step rarely share a word.)
__device__ __forceinline__ void shard_mark(const SparseParams& p, int cur, int32_t slot) {
    const int64_t mo = cur * p.mark_stride + (slot >> 5);
    const uint32_t mb = 1u << (slot & 31);
    for (int r = 0; r < p.nshard; ++r) red_or(p.peer_mark[r] + mo, mb);
}

// This replica registered block b first (locally): publish it.
__device__ __forceinline__ void shard_publish(const SparseParams& p, int cur, int32_t b) {
    const int32_t k = atomicAdd(&p.peer_xcnt[p.shard][cur], 1);
    p.xlist[(int64_t)cur * p.n + k] = b;
}

// Cross-replica barrier, combined with the local grid barrier: every CTA
// fences its remote writes at system scope and arrives locally; CTA 0 waits
// for the local arrivals, signals every replica and waits for all of them,
// then releases the local CTAs.  Thread 0 of every CTA also snapshots the
// replicas' published-list lengths into s_snap[0 .. nshard).  Returns false
// (on every CTA) when the wait timed out.
__device__ __forceinline__ bool shard_exchange(const SparseParams& p, int cur, unsigned& gen, unsigned& xgen,
                                               long long* s_snap) {
    __shared__ int s_abort;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned target = (gen + 1) * gridDim.x;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&p.bar->count) : "memory");
        int abort = 0;
        if (blockIdx.x == 0) {
            const unsigned long long t0 = globaltimer();
            while ((int)(ld_acquire_u32(&p.bar->count) - target) < 0) {
                if (globaltimer() - t0 > p.timeout_ns) {
                    abort = 1;
                    break;
                }
            }
            __threadfence_system();
            for (int r = 0; r < p.nshard; ++r)
                asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p.peer_xbar[r]) : "memory");
            const unsigned xt = (xgen + 1) * (unsigned)p.nshard;
            while (!abort && (int)(ld_acquire_sys(p.peer_xbar[p.shard]) - xt) < 0) {
                if (globaltimer() - t0 > p.timeout_ns) abort = 1;
            }
            if (abort) p.ctrl->error = kShardTimeout;
            __threadfence_system();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.go), "r"((xgen + 1) * 2 + abort)
                         : "memory");
        }
        unsigned g;
        while ((int)((g = ld_acquire_u32(p.go)) - (xgen + 1) * 2) < 0) {
        }
        abort = g & 1;
        __threadfence_system();
        if (!abort)
            for (int r = 0; r < p.nshard; ++r) s_snap[r] = (long long)ld_vol(&p.peer_xcnt[r][cur]);
        s_abort = abort;
    }
    ++gen;
    ++xgen;
    __syncthreads();
    return s_abort == 0;
}

// Adopt the blocks other replicas published this round: a local
// test-and-set on tblock decides whether this replica already has them.
__device__ __forceinline__ void shard_merge(const SparseParams& p, int cur, int32_t tw, int32_t tnw,
                                            const long long* s_snap) {
    const int lane = threadIdx.x & 31;
    int64_t base = 0;
    for (int r = 0; r < p.nshard; ++r) {
        const int64_t cnt = s_snap[r];
        if (r != p.shard) {
            const int32_t* lst = p.peer_xlist[r] + (int64_t)cur * p.n;
            for (int64_t i0 = (int64_t)tw << 5; i0 < cnt; i0 += (int64_t)tnw << 5) {
                const int64_t i = i0 + lane;
                const int32_t b = i < cnt ? lst[i] : 0;
                const uint32_t bit = 1u << (b & 31);
                const bool reg = i < cnt && !(ld_vol(&p.tblock[b >> 5]) & bit) &&
                                 !(atomicOr(&p.tblock[b >> 5], bit) & bit);
                register_blocks_warp(p, cur, reg, b);
            }
        }
        base += cnt;
    }
    (void)base;
}

// lo[g] = first source s whose out-degree prefix reaches g * m / G (deg holds
// the exclusive prefix sums, deg[n] = m); lo[0] = 0, lo[G] = n.
__global__ void k_shard_cuts(const int32_t* __restrict__ deg, int32_t n, int G, int32_t* lo) {
    const int g = threadIdx.x;
    if (g > G) return;
    if (g == 0) { lo[0] = 0; return; }
    if (g == G) { lo[G] = n; return; }
    const int64_t want = (int64_t)deg[n] * g / G;
    int32_t a = 0, b = n;  // first s in [0, n] with deg[s] >= want
    while (a < b) {
        const int32_t mid = a + (b - a) / 2;
        if (deg[mid] < want) a = mid + 1;
        else b = mid;
    }
    lo[g] = a;
}

