// post.cuh -- the steps either side of the refinement path, on the GPU
// (SURVEY.md §8f ranks 2 and 4).  Included by capi.cu (one translation unit,
// so the scan kernels and the per-device context are shared).
//
//   bisim_quotient     quotient(lts, p)             aut.py:132-152
//   bisim_is_stable    is_stable(lts, p)            oracle.py:128-141
//   bisim_canonical    partition_from_assignment    lts.py:117-128
//
// All three are set/dedup problems over the m transitions (or n states).
// They use one GPU hash-table pattern: a transition's triple is hashed to 64
// bits, the table keeps, per distinct hash, the minimum transition index that
// carries it (atomicMin = Priority "first occurrence"), and a verification
// pass compares every transition's full triple with its slot's
// representative.  Distinct triples sharing a 64-bit hash are therefore
// detected, never merged; the call then retries with another hash seed, so
// results are exact.  Output order is the reference's: first occurrences in
// transition order (an exclusive scan of the keep flags).
#pragma once

namespace bisim {

__device__ __forceinline__ unsigned long long fmix64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

// 64-bit hash of a triple (x, a, y); 0 is reserved for "empty slot".
__device__ __forceinline__ unsigned long long triple_hash(int32_t x, int32_t a, int32_t y,
                                                          unsigned long long seed) {
    unsigned long long h = fmix64(((unsigned long long)(uint32_t)x << 32 | (uint32_t)y) ^ seed);
    h = fmix64(h ^ ((unsigned long long)(uint32_t)a * 0x9e3779b97f4a7c15ull) ^ (seed >> 7));
    return h ? h : 1ull;
}

struct Triples {
    // triple of transition i: (xmap(src[i]), act[i], ymap(dst[i])); a map
    // pointer may be null (identity) -- quotient uses qidx[block[.]], the
    // stability check (src, act, block[dst]).
    const int32_t* src;
    const int32_t* act;
    const int32_t* dst;
    const int32_t* xblock;  // x = xblock ? xblock[src] : src
    const int32_t* xidx;    // then x = xidx ? xidx[x] : x
    const int32_t* yblock;
    const int32_t* yidx;
};

__device__ __forceinline__ int3 triple_of(const Triples& t, int64_t i) {
    int32_t x = t.src[i], y = t.dst[i];
    const int32_t a = t.act ? t.act[i] : 0;
    if (t.xblock) x = t.xblock[x];
    if (t.xidx) x = t.xidx[x];
    if (t.yblock) y = t.yblock[y];
    if (t.yidx) y = t.yidx[y];
    return make_int3(x, a, y);
}

// Find (or claim) the slot of hash h.  Linear probing over a power-of-two table.
__device__ __forceinline__ uint64_t ht_slot(unsigned long long* keys, uint64_t mask, unsigned long long h,
                                            bool insert) {
    uint64_t s = h & mask;
    for (;;) {
        const unsigned long long k = keys[s];
        if (k == h) return s;
        if (k == 0ull) {
            if (!insert) return ~0ull;
            const unsigned long long old = atomicCAS(&keys[s], 0ull, h);
            if (old == 0ull || old == h) return s;
        }
        s = (s + 1) & mask;
    }
}

__global__ void k_ht_insert(Triples t, int64_t m, unsigned long long seed, unsigned long long* keys,
                            int32_t* rep, uint64_t mask) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int3 k = triple_of(t, i);
        const uint64_t s = ht_slot(keys, mask, triple_hash(k.x, k.y, k.z, seed), true);
        if (ld_vol(&rep[s]) > (int32_t)i) atomicMin(&rep[s], (int32_t)i);
    }
}

// keep[i] = 1 iff i is the first transition carrying its triple; flags a
// hash collision (two distinct triples in one slot) in *bad.
__global__ void k_ht_verify(Triples t, int64_t m, unsigned long long seed, const unsigned long long* keys,
                            const int32_t* rep, uint64_t mask, int32_t* keep, int32_t* bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int3 k = triple_of(t, i);
        const uint64_t s = ht_slot(const_cast<unsigned long long*>(keys), mask, triple_hash(k.x, k.y, k.z, seed),
                                   false);
        const int32_t j = rep[s];
        const int3 r = triple_of(t, j);
        if (r.x != k.x || r.y != k.y || r.z != k.z) *bad = 1;
        if (keep) keep[i] = j == (int32_t)i ? 1 : 0;
    }
}

// action ids in range (lts.py:50-52)
__global__ void k_check_actions(int64_t m, int32_t A, const int32_t* __restrict__ act, Ctrl* ctrl) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        if ((unsigned)act[i] >= (unsigned)A) ctrl->bad = 1;
}

// ---- quotient (aut.py:132-152) ------------------------------------------------

// Leader-form check of a partition (lts.py:88-94) and leader flags.
__global__ void k_leader_flags(int32_t n, const int32_t* __restrict__ block, int32_t* flag, int32_t* bad) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = block[s];
        if ((unsigned)b >= (unsigned)n || block[b] != b) {
            *bad = 1;
            continue;
        }
        if (b == (int32_t)s) flag[s] = 1;
    }
}

__global__ void k_quotient_emit(Triples t, int64_t m, const int32_t* __restrict__ pos, int32_t* qs, int32_t* qa,
                                int32_t* qd) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = pos[i];
        if (pos[i + 1] == p) continue;  // not a first occurrence
        const int3 k = triple_of(t, i);
        qs[p] = k.x;
        qa[p] = k.y;
        qd[p] = k.z;
    }
}

// ---- stability (oracle.py:128-141) ----------------------------------------------

// distinct (a, block[t]) pairs per source state
__global__ void k_sig_count(const int32_t* __restrict__ src, int64_t m, const int32_t* __restrict__ keep,
                            int32_t* cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        if (keep[i]) atomicAdd(&cnt[src[i]], 1);
}

// sig(s) == sig(block[s]) for all s  <=>  equal sizes and sig(s) within sig(block[s])
__global__ void k_sig_check(int32_t n, const int32_t* __restrict__ block, const int32_t* __restrict__ cnt,
                            int32_t* unstable) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
        if (cnt[s] != cnt[block[s]]) *unstable = 1;
}

__global__ void k_sig_subset(Triples t, int64_t m, unsigned long long seed, const unsigned long long* keys,
                             const int32_t* rep, uint64_t mask, const int32_t* __restrict__ keep,
                             const int32_t* __restrict__ block, int32_t* unstable) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (!keep[i]) continue;
        const int3 k = triple_of(t, i);
        const int32_t l = block[k.x];
        if (l == k.x) continue;
        const uint64_t s = ht_slot(const_cast<unsigned long long*>(keys), mask, triple_hash(l, k.y, k.z, seed), false);
        bool found = false;
        if (s != ~0ull) {
            const int3 r = triple_of(t, rep[s]);
            found = r.x == l && r.y == k.y && r.z == k.z;
        }
        if (!found) *unstable = 1;
    }
}

// ---- stability under a state set (oracle.py:144-154) -------------------------------

// reach[w * n + s] bit a: s has an a-transition into the set (word-major masks)
__global__ void k_reach_mask(int32_t n, int64_t m, const int32_t* __restrict__ src, const int32_t* __restrict__ act,
                             const int32_t* __restrict__ dst, const uint8_t* __restrict__ in_set,
                             unsigned long long* reach) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        if (!in_set[dst[i]]) continue;
        const int32_t a = act[i];
        asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(&reach[(int64_t)(a >> 6) * n + src[i]]),
                     "l"(1ull << (a & 63))
                     : "memory");
    }
}

__global__ void k_reach_check(int32_t n, int32_t W, const int32_t* __restrict__ block,
                              const unsigned long long* __restrict__ reach, int32_t* unstable) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t l = block[s];
        for (int32_t w = 0; w < W; ++w)
            if (reach[(int64_t)w * n + s] != reach[(int64_t)w * n + l]) {
                *unstable = 1;
                break;
            }
    }
}

__global__ void k_set_flags(int64_t k, const int32_t* __restrict__ states, int32_t n, uint8_t* in_set, int32_t* bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t x = states[i];
        if ((unsigned)x < (unsigned)n) in_set[x] = 1;
    }
}

// ---- canonical leader form (lts.py:117-128) --------------------------------------

__device__ __forceinline__ unsigned long long value_hash(long long v, unsigned long long seed) {
    const unsigned long long h = fmix64((unsigned long long)v ^ seed);  // a bijection of v
    return h ? h : 1ull;
}

__global__ void k_canon_insert(int32_t n, const long long* __restrict__ val, unsigned long long seed,
                               unsigned long long* keys, int32_t* rep, uint64_t mask) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t slot = ht_slot(keys, mask, value_hash(val[s], seed), true);
        if (ld_vol(&rep[slot]) > (int32_t)s) atomicMin(&rep[slot], (int32_t)s);
    }
}

__global__ void k_canon_assign(int32_t n, const long long* __restrict__ val, unsigned long long seed,
                               const unsigned long long* keys, const int32_t* rep, uint64_t mask, int32_t* block,
                               int32_t* bad) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t slot =
            ht_slot(const_cast<unsigned long long*>(keys), mask, value_hash(val[s], seed), false);
        const int32_t j = rep[slot];
        if (val[j] != val[s]) *bad = 1;  // only the remapped zero hash can alias
        block[s] = j;
    }
}

// ---- host side -------------------------------------------------------------------

namespace {

struct HashTable {
    unsigned long long* keys;
    int32_t* rep;
    uint64_t mask;
};

HashTable ht_alloc(Ctx& c, DevBuf& kb, DevBuf& rb, int64_t items) {
    uint64_t T = 1024;
    while (T < 2ull * (uint64_t)std::max<int64_t>(items, 1)) T <<= 1;
    HashTable h;
    h.keys = (unsigned long long*)kb.ensure(T * 8);
    h.rep = (int32_t*)rb.ensure(T * 4);
    h.mask = T - 1;
    CK(cudaMemsetAsync(h.keys, 0, T * 8, c.stream));
    CK(cudaMemsetAsync(h.rep, 0x7f, T * 4, c.stream));
    return h;
}

int32_t read_flag(Ctx& c, const int32_t* d) {
    int32_t v = 0;
    CK(cudaMemcpyAsync(&v, d, 4, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return v;
}

constexpr unsigned long long kSeeds[4] = {0x243f6a8885a308d3ull, 0x13198a2e03707344ull, 0xa4093822299f31d0ull,
                                          0x082efa98ec4e6c89ull};

// Dedup the triples of t: keep[i] (m+1 ints) = first occurrence flag.
HashTable dedup(Ctx& c, const Triples& t, int64_t m, int32_t* keep, int32_t* bad, unsigned long long& seed) {
    const int TB = 256;
    for (unsigned long long s : kSeeds) {
        HashTable h = ht_alloc(c, c.lkeys, c.lmins, m);
        CK(cudaMemsetAsync(bad, 0, 4, c.stream));
        k_ht_insert<<<grid_for(m, TB, c.sms), TB, 0, c.stream>>>(t, m, s, h.keys, h.rep, h.mask);
        k_ht_verify<<<grid_for(m, TB, c.sms), TB, 0, c.stream>>>(t, m, s, h.keys, h.rep, h.mask, keep, bad);
        CK(cudaGetLastError());
        if (!read_flag(c, bad)) {
            seed = s;
            return h;
        }
    }
    throw Error(BISIM_CUDA, "hash collisions under every seed (input of pathological size?)");
}

void post_begin(Ctx& c) { CK(cudaSetDevice(c.device)); }

template <typename F>
int post_guarded(F&& f) {
    try {
        g_last_error.clear();
        return f();
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return BISIM_CUDA;
    }
}

void check_transitions(Ctx& c, int32_t n, int64_t m, int32_t A, const int32_t* src, const int32_t* act,
                       const int32_t* dst) {
    // reuse the preprocessing validation (lts.py:47-52)
    Ctrl* ctrl = (Ctrl*)c.ctrl.ensure(std::max(sizeof(Ctrl), sizeof(SCtrl)));
    CK(cudaMemsetAsync(ctrl, 0, sizeof(Ctrl), c.stream));
    if (m) {
        if (act) {
            // bounds check only: label masks are not needed here
            k_check_edges<<<grid_for(m, 256, c.sms), 256, 0, c.stream>>>(n, m, src, dst, ctrl);
            k_check_actions<<<grid_for(m, 256, c.sms), 256, 0, c.stream>>>(m, A, act, ctrl);
        } else {
            k_check_edges<<<grid_for(m, 256, c.sms), 256, 0, c.stream>>>(n, m, src, dst, ctrl);
        }
    }
    CK(cudaGetLastError());
    if (read_flag(c, &ctrl->bad))
        throw Error(BISIM_BAD_INPUT, "transition mentions a state or action outside range");
}

}  // namespace
}  // namespace bisim

extern "C" {

int bisim_quotient(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                   const int32_t* dst, const int32_t* block, int32_t initial_state, int32_t* q_n, int64_t* q_m,
                   int32_t* q_src, int32_t* q_act, int32_t* q_dst, int32_t* q_initial, int device) {
    using namespace bisim;
    return post_guarded([&]() -> int {
        if (n < 1) throw Error(BISIM_BAD_INPUT, "state count must be at least 1");
        if (m < 0 || m >= (int64_t)INT32_MAX) throw Error(BISIM_BAD_INPUT, "transition count out of range");
        if (initial_state < 0 || initial_state >= n) throw Error(BISIM_BAD_INPUT, "initial state out of range");
        if (!block || !q_n || !q_m || (m && (!src || !act || !dst || !q_src || !q_act || !q_dst)))
            throw Error(BISIM_BAD_INPUT, "null array");
        Ctx& c = *get_ctx(device);
        std::lock_guard<std::mutex> lock(c.mu);
        post_begin(c);
        cudaStream_t st = c.stream;
        const int TB = 256;
        const int64_t mm = std::max<int64_t>(m, 1);
        int32_t* d_src = (int32_t*)c.src.ensure(mm * 4);
        int32_t* d_act = (int32_t*)c.act.ensure(mm * 4);
        int32_t* d_dst = (int32_t*)c.dst.ensure(mm * 4);
        int32_t* d_block = (int32_t*)c.block.ensure((int64_t)n * 4);
        h2d(c, d_src, src, m * 4, st);
        h2d(c, d_act, act, m * 4, st);
        h2d(c, d_dst, dst, m * 4, st);
        h2d(c, d_block, block, (int64_t)n * 4, st);
        check_transitions(c, n, m, num_actions, d_src, d_act, d_dst);
        // leader index: dense numbering of the leaders in increasing order
        int32_t* qidx = (int32_t*)c.bstart.ensure(((int64_t)n + 1) * 4);
        int32_t* bad = (int32_t*)c.counter.ensure(16);
        CK(cudaMemsetAsync(qidx, 0, ((int64_t)n + 1) * 4, st));
        CK(cudaMemsetAsync(bad, 0, 4, st));
        k_leader_flags<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, d_block, qidx, bad);
        CK(cudaGetLastError());
        if (read_flag(c, bad)) throw Error(BISIM_BAD_INPUT, "block array is not a leader-form partition");
        scan_excl(c, qidx, n);
        int32_t nq = 0, qi = 0, lead = 0;
        CK(cudaMemcpyAsync(&nq, qidx + n, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&lead, d_block + initial_state, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaMemcpyAsync(&qi, qidx + lead, 4, cudaMemcpyDeviceToHost, st));
        int64_t qm = 0;
        if (m) {
            Triples t{d_src, d_act, d_dst, d_block, qidx, d_block, qidx};
            int32_t* keep = (int32_t*)c.scnt.ensure((mm + 1) * 4);
            unsigned long long seed = 0;
            dedup(c, t, m, keep, bad, seed);
            scan_excl(c, keep, m);
            int32_t qm32 = 0;
            CK(cudaMemcpyAsync(&qm32, keep + m, 4, cudaMemcpyDeviceToHost, st));
            int32_t* o = (int32_t*)c.tmp.ensure(mm * 12);
            k_quotient_emit<<<grid_for(m, TB, c.sms), TB, 0, st>>>(t, m, keep, o, o + mm, o + 2 * mm);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(st));
            qm = qm32;
            if (qm) {
                CK(cudaMemcpyAsync(q_src, o, qm * 4, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(q_act, o + mm, qm * 4, cudaMemcpyDeviceToHost, st));
                CK(cudaMemcpyAsync(q_dst, o + 2 * mm, qm * 4, cudaMemcpyDeviceToHost, st));
            }
        }
        CK(cudaStreamSynchronize(st));
        *q_n = nq;
        *q_m = qm;
        if (q_initial) *q_initial = qi;
        return BISIM_OK;
    });
}

int bisim_is_stable(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                    const int32_t* dst, const int32_t* block, int32_t* stable_out, int device) {
    using namespace bisim;
    return post_guarded([&]() -> int {
        if (n < 1) throw Error(BISIM_BAD_INPUT, "state count must be at least 1");
        if (m < 0 || m >= (int64_t)INT32_MAX) throw Error(BISIM_BAD_INPUT, "transition count out of range");
        if (!block || !stable_out || (m && (!src || !act || !dst))) throw Error(BISIM_BAD_INPUT, "null array");
        Ctx& c = *get_ctx(device);
        std::lock_guard<std::mutex> lock(c.mu);
        post_begin(c);
        cudaStream_t st = c.stream;
        const int TB = 256;
        const int64_t mm = std::max<int64_t>(m, 1);
        int32_t* d_src = (int32_t*)c.src.ensure(mm * 4);
        int32_t* d_act = (int32_t*)c.act.ensure(mm * 4);
        int32_t* d_dst = (int32_t*)c.dst.ensure(mm * 4);
        int32_t* d_block = (int32_t*)c.block.ensure((int64_t)n * 4);
        h2d(c, d_src, src, m * 4, st);
        h2d(c, d_act, act, m * 4, st);
        h2d(c, d_dst, dst, m * 4, st);
        h2d(c, d_block, block, (int64_t)n * 4, st);
        check_transitions(c, n, m, num_actions, d_src, d_act, d_dst);
        int32_t* bad = (int32_t*)c.counter.ensure(16);
        int32_t* flags = (int32_t*)c.bstart.ensure(((int64_t)n + 1) * 4);
        CK(cudaMemsetAsync(flags, 0, ((int64_t)n + 1) * 4, st));
        CK(cudaMemsetAsync(bad, 0, 8, st));
        k_leader_flags<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, d_block, flags, bad);
        CK(cudaGetLastError());
        if (read_flag(c, bad)) throw Error(BISIM_BAD_INPUT, "block array is not a leader-form partition");
        int32_t* cnt = (int32_t*)c.bsize.ensure((int64_t)n * 4);
        CK(cudaMemsetAsync(cnt, 0, (int64_t)n * 4, st));
        int32_t* unstable = bad + 1;
        if (m) {
            Triples t{d_src, d_act, d_dst, nullptr, nullptr, d_block, nullptr};
            int32_t* keep = (int32_t*)c.scnt.ensure((mm + 1) * 4);
            unsigned long long seed = 0;
            HashTable h = dedup(c, t, m, keep, bad, seed);
            k_sig_count<<<grid_for(m, TB, c.sms), TB, 0, st>>>(d_src, m, keep, cnt);
            k_sig_subset<<<grid_for(m, TB, c.sms), TB, 0, st>>>(t, m, seed, h.keys, h.rep, h.mask, keep, d_block,
                                                               unstable);
        }
        k_sig_check<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, d_block, cnt, unstable);
        CK(cudaGetLastError());
        *stable_out = read_flag(c, unstable) ? 0 : 1;
        return BISIM_OK;
    });
}

int bisim_is_stable_under(int32_t n, int64_t m, int32_t num_actions, const int32_t* src, const int32_t* act,
                          const int32_t* dst, const int32_t* block, const int32_t* states, int64_t num_states,
                          int32_t* stable_out, int device) {
    using namespace bisim;
    return post_guarded([&]() -> int {
        if (n < 1) throw Error(BISIM_BAD_INPUT, "state count must be at least 1");
        if (m < 0 || m >= (int64_t)INT32_MAX) throw Error(BISIM_BAD_INPUT, "transition count out of range");
        if (num_states < 0) throw Error(BISIM_BAD_INPUT, "negative state-set size");
        if (!block || !stable_out || (m && (!src || !act || !dst)) || (num_states && !states))
            throw Error(BISIM_BAD_INPUT, "null array");
        Ctx& c = *get_ctx(device);
        std::lock_guard<std::mutex> lock(c.mu);
        post_begin(c);
        cudaStream_t st = c.stream;
        const int TB = 256;
        const int64_t mm = std::max<int64_t>(m, 1);
        const int32_t W = std::max(1, (num_actions + 63) / 64);
        int32_t* d_src = (int32_t*)c.src.ensure(mm * 4);
        int32_t* d_act = (int32_t*)c.act.ensure(mm * 4);
        int32_t* d_dst = (int32_t*)c.dst.ensure(mm * 4);
        int32_t* d_block = (int32_t*)c.block.ensure((int64_t)n * 4);
        int32_t* d_states = (int32_t*)c.pi0.ensure(std::max<int64_t>(num_states, 1) * 4);
        h2d(c, d_src, src, m * 4, st);
        h2d(c, d_act, act, m * 4, st);
        h2d(c, d_dst, dst, m * 4, st);
        h2d(c, d_block, block, (int64_t)n * 4, st);
        if (num_states) CK(cudaMemcpyAsync(d_states, states, num_states * 4, cudaMemcpyHostToDevice, st));
        check_transitions(c, n, m, num_actions, d_src, d_act, d_dst);
        int32_t* bad = (int32_t*)c.counter.ensure(16);
        int32_t* flags = (int32_t*)c.bstart.ensure(((int64_t)n + 1) * 4);
        CK(cudaMemsetAsync(flags, 0, ((int64_t)n + 1) * 4, st));
        CK(cudaMemsetAsync(bad, 0, 8, st));
        k_leader_flags<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, d_block, flags, bad);
        CK(cudaGetLastError());
        if (read_flag(c, bad)) throw Error(BISIM_BAD_INPUT, "block array is not a leader-form partition");
        uint8_t* in_set = (uint8_t*)c.scnt.ensure((int64_t)n);
        CK(cudaMemsetAsync(in_set, 0, (int64_t)n, st));
        if (num_states) k_set_flags<<<grid_for(num_states, TB, c.sms), TB, 0, st>>>(num_states, d_states, n, in_set, bad);
        auto* reach = (unsigned long long*)c.lmask.ensure((size_t)W * n * 8);
        CK(cudaMemsetAsync(reach, 0, (size_t)W * n * 8, st));
        if (m) k_reach_mask<<<grid_for(m, TB, c.sms), TB, 0, st>>>(n, m, d_src, d_act, d_dst, in_set, reach);
        int32_t* unstable = bad + 1;
        k_reach_check<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, W, d_block, reach, unstable);
        CK(cudaGetLastError());
        *stable_out = read_flag(c, unstable) ? 0 : 1;
        return BISIM_OK;
    });
}

int bisim_canonical(int32_t n, const int64_t* assignment, int32_t* block_out, int device) {
    using namespace bisim;
    return post_guarded([&]() -> int {
        if (n < 1) throw Error(BISIM_BAD_INPUT, "a partition needs at least one state");
        if (!assignment || !block_out) throw Error(BISIM_BAD_INPUT, "null array");
        Ctx& c = *get_ctx(device);
        std::lock_guard<std::mutex> lock(c.mu);
        post_begin(c);
        cudaStream_t st = c.stream;
        const int TB = 256;
        long long* val = (long long*)c.nl.ensure((int64_t)n * 8);
        int32_t* d_block = (int32_t*)c.block.ensure((int64_t)n * 4);
        int32_t* bad = (int32_t*)c.counter.ensure(16);
        CK(cudaMemcpyAsync(val, assignment, (int64_t)n * 8, cudaMemcpyHostToDevice, st));
        for (unsigned long long s : kSeeds) {
            HashTable h = ht_alloc(c, c.lkeys, c.lmins, n);
            CK(cudaMemsetAsync(bad, 0, 4, st));
            k_canon_insert<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, val, s, h.keys, h.rep, h.mask);
            k_canon_assign<<<grid_for(n, TB, c.sms), TB, 0, st>>>(n, val, s, h.keys, h.rep, h.mask, d_block, bad);
            CK(cudaGetLastError());
            if (!read_flag(c, bad)) {
                CK(cudaMemcpyAsync(block_out, d_block, (int64_t)n * 4, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                return BISIM_OK;
            }
        }
        throw Error(BISIM_CUDA, "hash aliasing under every seed");
    });
}

}  // extern "C"
