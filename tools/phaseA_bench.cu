// Phase-A cost breakdown on a c5-shaped heavy round (developer experiment):
// walk the in-edges of an 89K-member splitter (in-degree 10, random sources
// in n = 10M states, ~300 distinct source blocks) the way k_refine_sparse's
// phase A does, with parts switched off, and time each variant.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/phaseA_bench tools/phaseA_bench.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <random>
#include <cstdlib>
#include <algorithm>

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSeen = 1024;

__device__ __forceinline__ void red_or(uint32_t* a, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

__device__ __forceinline__ int cta_first(int32_t* seen, int32_t b) {
    uint32_t h = ((uint32_t)b * 2654435761u) >> 22;
    for (int probe = 0; probe < 16; ++probe) {
        const int32_t old = atomicCAS(&seen[h], -1, b);
        if (old == -1) return 1;
        if (old == b) return 0;
        h = (h + 1) & (kSeen - 1);
    }
    return 2;
}

// flags: 1 mark red.or, 2 block gather, 4 match + cta hash, 8 byte-map mark store instead of bit red.or
__device__ unsigned long long g_t[2][148 * 16];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <int KA, bool PF = false>
__global__ void __launch_bounds__(512, 1) walk(const int4* members, int32_t cz, const int2* rev, const int32_t* block,
                                               uint32_t* mark, uint8_t* markb, int flags, unsigned long long* sink) {
    __shared__ int32_t s_seen[kSeen];
    for (int k = threadIdx.x; k < kSeen; k += blockDim.x) s_seen[k] = -1;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int32_t tw = (int32_t)((threadIdx.x >> 5) * gridDim.x + blockIdx.x);
    if (lane == 0) g_t[0][tw] = gtimer();
    const int32_t tnw = (int32_t)((gridDim.x * blockDim.x) >> 5);
    int32_t g = max(1, (cz + tnw - 1) / tnw);
    if (g > 32) {
        const int32_t iters = (cz + tnw * 32 - 1) / (tnw * 32);
        g = (cz + iters * tnw - 1) / (iters * tnw);
    }
    unsigned long long acc = 0;
    int4 nx = make_int4(0, 0, 0, 0);
    if (PF && lane < g && (int64_t)tw * g + lane < cz) nx = members[(int64_t)tw * g + lane];
    for (int64_t i0 = (int64_t)tw * g; i0 < cz; i0 += (int64_t)tnw * g) {
        const int64_t i = i0 + lane;
        int32_t e0 = 0, d = 0;
        if (PF) {
            e0 = nx.z;
            d = nx.w - nx.z;
            const int64_t i2 = i + (int64_t)tnw * g;
            nx = (lane < g && i2 < cz) ? members[i2] : make_int4(0, 0, 0, 0);
        } else if (lane < g && i < cz) {
            const int4 r = members[i];
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
        for (int32_t k0 = 0; k0 < total; k0 += 32 * KA) {
            int2 rv[KA];
            bool act[KA];
#pragma unroll
            for (int u = 0; u < KA; ++u) {
                const int32_t k = k0 + 32 * u + lane;
                int32_t j = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const int32_t ex = __shfl_sync(kFull, excl, j + step);
                    if (ex <= k) j += step;
                }
                const int32_t ej = __shfl_sync(kFull, e0, j);
                const int32_t xj = __shfl_sync(kFull, excl, j);
                act[u] = k < total;
                rv[u] = act[u] ? __ldcs(&rev[ej + (k - xj)]) : make_int2(0, 0);
            }
            int32_t bb[KA];
#pragma unroll
            for (int u = 0; u < KA; ++u) {
                if (flags & 64) {  // per-state record (block | mark bits << 32): one returning atomic
                    bb[u] = act[u] ? (int32_t)atomicOr((unsigned long long*)markb + rv[u].y,
                                                       1ull << (32 + (rv[u].x & 31)))
                                   : 0;
                    continue;
                }
                if ((flags & 8) && act[u]) markb[rv[u].x] = 1;  // byte map: a plain store, no L2 atomic
                if (!(flags & 32) && act[u] && (flags & 1)) red_or(&mark[rv[u].x >> 5], 1u << (rv[u].x & 31));
                bb[u] = (act[u] && (flags & 2)) ? block[rv[u].y] : rv[u].y;
            }
            if (flags & 32) {  // block gathers first, then the marks
#pragma unroll
                for (int u = 0; u < KA; ++u)
                    if (act[u] && (flags & 1)) red_or(&mark[rv[u].x >> 5], 1u << (rv[u].x & 31));
            }
#pragma unroll
            for (int u = 0; u < KA; ++u) {
                const int32_t b = bb[u];
                if (flags & 16) {
                    if (act[u]) {
                        const uint32_t h = ((uint32_t)b * 2654435761u) >> 22;
                        if (s_seen[h] != b) acc += (unsigned long long)cta_first(s_seen, b);
                    }
                } else if (flags & 4) {
                    const unsigned same = __match_any_sync(kFull, act[u] ? b : -1 - lane);
                    if (act[u] && lane == __ffs(same) - 1) acc += (unsigned long long)cta_first(s_seen, b);
                } else {
                    acc += (unsigned long long)b;
                }
            }
        }
    }
    if (acc == 0x123456789ull) sink[0] = acc;
    if (lane == 0) g_t[1][tw] = gtimer();
}

// lane-per-member walk: every lane walks its own member's in-edges, E at a
// time (loads issued together), instead of a warp scan spreading a group of
// members' in-edges over the lanes
template <int E>
__global__ void __launch_bounds__(512, 1) walk_lane(const int4* members, int32_t cz, const int2* rev,
                                                    const int32_t* block, uint32_t* mark, int flags,
                                                    unsigned long long* sink) {
    __shared__ int32_t s_seen[kSeen];
    for (int k = threadIdx.x; k < kSeen; k += blockDim.x) s_seen[k] = -1;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int32_t tw = (int32_t)((threadIdx.x >> 5) * gridDim.x + blockIdx.x);
    if (lane == 0) g_t[0][tw] = gtimer();
    const int64_t gl = (int64_t)tw * 32 + lane, nl = (int64_t)gridDim.x * blockDim.x;
    unsigned long long acc = 0;
    for (int64_t i = gl; i < cz; i += nl) {
        const int4 r = members[i];
        for (int32_t e = r.z; e < r.w; e += E) {
            int2 rv[E];
            int32_t bb[E];
#pragma unroll
            for (int u = 0; u < E; ++u) rv[u] = e + u < r.w ? __ldcs(&rev[e + u]) : make_int2(0, -1);
#pragma unroll
            for (int u = 0; u < E; ++u) {
                if (rv[u].y >= 0 && (flags & 1)) red_or(&mark[rv[u].x >> 5], 1u << (rv[u].x & 31));
                bb[u] = (rv[u].y >= 0 && (flags & 2)) ? block[rv[u].y] : rv[u].y;
            }
#pragma unroll
            for (int u = 0; u < E; ++u) {
                const int32_t b = bb[u];
                if (rv[u].y < 0) continue;
                if (flags & 16) {
                    const uint32_t h = ((uint32_t)b * 2654435761u) >> 22;
                    if (s_seen[h] != b) acc += (unsigned long long)cta_first(s_seen, b);
                } else {
                    acc += (unsigned long long)b;
                }
            }
        }
    }
    if (acc == 0x123456789ull) sink[0] = acc;
    if (lane == 0) g_t[1][tw] = gtimer();
}

int main() {
    const int32_t n = 10000000, cz = 89000, deg = 10, nblocks = 300;
    std::mt19937_64 rng(1);
    // spread=1: every member's in-edge range at a random place of a c5-sized
    // (100M-entry, 800 MB) reverse CSR, as in the loop, instead of packed
    // into 7 MB that stays in L2 across repetitions
    const bool spread = getenv("SPREAD") != nullptr;
    // (and a different splitter each repetition, so its in-edges are not
    // the ones the previous repetition left in L2)
    const size_t nrev = spread ? (size_t)100000000 : (size_t)cz * deg;
    const int nset = spread ? 50 : 1;
    std::vector<int4> mem((size_t)cz * nset);
    for (size_t i = 0; i < mem.size(); ++i) {
        const int32_t e0 = spread ? (int32_t)(rng() % (nrev / deg)) * deg : (int32_t)i * deg;
        mem[i] = make_int4((int32_t)(i % cz), 0, e0, e0 + deg);
    }
    std::vector<int2> rev(nrev);
    for (auto& r : rev) r = make_int2((int32_t)(rng() % (uint64_t)(5 * (uint64_t)n)), (int32_t)(rng() % n));
    std::vector<int32_t> blk(n);
    std::vector<int32_t> labels(nblocks);
    for (auto& l : labels) l = (int32_t)(rng() % n);
    for (auto& b : blk) b = labels[rng() % nblocks];
    int4* d_mem;
    int2* d_rev;
    int32_t* d_blk;
    uint32_t* d_mark;
    uint8_t* d_markb;
    unsigned long long* d_sink;
    cudaMalloc(&d_mem, mem.size() * 16);
    cudaMalloc(&d_rev, rev.size() * 8);
    cudaMalloc(&d_blk, (size_t)n * 4);
    cudaMalloc(&d_mark, (size_t)5 * n / 8 + 64);
    cudaMalloc(&d_markb, (size_t)8 * n + 64);
    cudaMalloc(&d_sink, 8);
    cudaMemcpy(d_mem, mem.data(), mem.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d_rev, rev.data(), rev.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_blk, blk.data(), (size_t)n * 4, cudaMemcpyHostToDevice);
    cudaMemset(d_mark, 0, (size_t)5 * n / 8 + 64);
    {
        std::vector<unsigned long long> rec(n);
        for (int32_t i = 0; i < n; ++i) rec[i] = (uint32_t)blk[i];
        cudaMemcpy(d_markb, rec.data(), (size_t)8 * n, cudaMemcpyHostToDevice);
    }
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct V { const char* name; int flags, ka; };
    const V vs[] = {{"empty launch (g=0)", -1, 1},
                    {"KA1 plain-load hash (r02)", 1 | 2 | 16, 1},
                    {"KA4 plain-load hash", 1 | 2 | 16, 4},
                    {"KA8 plain-load hash", 1 | 2 | 16, 8},
                    {"KA4 rev only", 0, 4},
                    {"KA4 rev + mark", 1, 4},
                    {"KA4 rev + block", 2, 4},
                    {"KA4 rev + block + mark", 3, 4},
                    {"KA8 rev only", 0, 8},
                    {"KA4 full + member prefetch", 1 | 2 | 16, 104},
                    {"KA8 full + member prefetch", 1 | 2 | 16, 108},
                    {"KA4 full, gathers before marks", 1 | 2 | 16 | 32, 4},
                    {"KA8 full, gathers before marks", 1 | 2 | 16 | 32, 8},
                    {"KA4 rev+block+mark, gathers first", 1 | 2 | 32, 4},
                    {"KA4 full, gathers first + mprefetch", 1 | 2 | 16 | 32, 104},
                    {"lane/member E4 full", 1 | 2 | 16, 204},
                    {"lane/member E8 full", 1 | 2 | 16, 208},
                    {"lane/member E12 full", 1 | 2 | 16, 212},
                    {"lane/member E8 rev only", 0, 208},
                    {"KA4 rec64 atomic + hash", 64 | 16, 4},
                    {"KA4 rec64 atomic, no hash", 64, 4},
                    {"KA8 rec64 atomic + hash", 64 | 16, 8},
                    {"KA4 byte-map store + block + hash", 8 | 2 | 16, 4},
                    {"KA4 byte-map store + block", 8 | 2, 4},
                    {"KA4 rev + mark + hash (no block)", 1 | 16, 4}};
    for (const V& v : vs) {
        int rep = 0;
        auto launch = [&]() {
            const int4* m = d_mem + (size_t)(rep++ % nset) * cz;
            const int32_t z = v.flags < 0 ? 0 : cz;
            const int f = v.flags < 0 ? 0 : v.flags;
            if (v.ka == 1) walk<1><<<sms, 512>>>(m, z, d_rev, d_blk, d_mark, d_markb, f, d_sink);
            else if (v.ka == 4) walk<4><<<sms, 512>>>(m, z, d_rev, d_blk, d_mark, d_markb, f, d_sink);
            else if (v.ka == 8) walk<8><<<sms, 512>>>(m, z, d_rev, d_blk, d_mark, d_markb, f, d_sink);
            else if (v.ka == 204) walk_lane<4><<<sms, 512>>>(m, z, d_rev, d_blk, d_mark, f, d_sink);
            else if (v.ka == 208) walk_lane<8><<<sms, 512>>>(m, z, d_rev, d_blk, d_mark, f, d_sink);
            else if (v.ka == 212) walk_lane<12><<<sms, 512>>>(m, z, d_rev, d_blk, d_mark, f, d_sink);
            else if (v.ka == 104) walk<4, true><<<sms, 512>>>(m, z, d_rev, d_blk, d_mark, d_markb, f, d_sink);
            else walk<8, true><<<sms, 512>>>(m, z, d_rev, d_blk, d_mark, d_markb, f, d_sink);
        };
        for (int w = 0; w < 3; ++w) launch();
        const int R = 50;
        cudaEventRecord(e0);
        for (int r = 0; r < R; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<unsigned long long> t(2 * 148 * 16);
        cudaMemcpyFromSymbol(t.data(), g_t, t.size() * 8);
        const int nw = sms * 16;
        unsigned long long t0 = ~0ull;
        for (int w = 0; w < nw; ++w) t0 = std::min(t0, t[w]);
        std::vector<double> st, en;
        for (int w = 0; w < nw; ++w) {
            st.push_back((t[w] - t0) * 1e-3);
            en.push_back((t[nw + w] - t0) * 1e-3);
        }
        std::sort(st.begin(), st.end());
        std::sort(en.begin(), en.end());
        auto q = [&](std::vector<double>& v, double f) { return v[std::min((size_t)(f * v.size()), v.size() - 1)]; };
        printf("%-40s %7.2f us per walk (%s)  warp start p50/max %.2f/%.2f  end p10/p50/p90/p99/max %.2f/%.2f/%.2f/%.2f/%.2f\n",
               v.name, ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()), q(st, .5), st.back(), q(en, .1), q(en, .5),
               q(en, .9), q(en, .99), en.back());
    }
    return 0;
}
