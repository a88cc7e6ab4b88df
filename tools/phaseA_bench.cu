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
template <int KA>
__global__ void __launch_bounds__(512, 1) walk(const int4* members, int32_t cz, const int2* rev, const int32_t* block,
                                               uint32_t* mark, uint8_t* markb, int flags, unsigned long long* sink) {
    __shared__ int32_t s_seen[kSeen];
    for (int k = threadIdx.x; k < kSeen; k += blockDim.x) s_seen[k] = -1;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int32_t tw = (int32_t)((threadIdx.x >> 5) * gridDim.x + blockIdx.x);
    const int32_t tnw = (int32_t)((gridDim.x * blockDim.x) >> 5);
    int32_t g = max(1, (cz + tnw - 1) / tnw);
    if (g > 32) {
        const int32_t iters = (cz + tnw * 32 - 1) / (tnw * 32);
        g = (cz + iters * tnw - 1) / (iters * tnw);
    }
    unsigned long long acc = 0;
    for (int64_t i0 = (int64_t)tw * g; i0 < cz; i0 += (int64_t)tnw * g) {
        const int64_t i = i0 + lane;
        int32_t e0 = 0, d = 0;
        if (lane < g && i < cz) {
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
                if (act[u] && (flags & 1)) red_or(&mark[rv[u].x >> 5], 1u << (rv[u].x & 31));
                bb[u] = (act[u] && (flags & 2)) ? block[rv[u].y] : rv[u].y;
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
    cudaMalloc(&d_markb, (size_t)5 * n + 64);
    cudaMalloc(&d_sink, 8);
    cudaMemcpy(d_mem, mem.data(), mem.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(d_rev, rev.data(), rev.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d_blk, blk.data(), (size_t)n * 4, cudaMemcpyHostToDevice);
    cudaMemset(d_mark, 0, (size_t)5 * n / 8 + 64);
    cudaMemset(d_markb, 0, (size_t)5 * n + 64);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[] = {"KA1 match/hash (r01)", "KA1 plain-load hash (r02)", "KA2 plain-load hash",
                           "KA4 plain-load hash", "KA1 no hash", "KA2 no hash"};
    const int fl[] = {7, 1 | 2 | 16, 1 | 2 | 16, 1 | 2 | 16, 3, 3};
    const int ka[] = {1, 1, 2, 4, 1, 2};
    for (int v = 0; v < 6; ++v) {
        int rep = 0;
        auto launch = [&]() {
            const int4* m = d_mem + (size_t)(rep++ % nset) * cz;
            if (ka[v] == 1) walk<1><<<sms, 512>>>(m, cz, d_rev, d_blk, d_mark, d_markb, fl[v], d_sink);
            else if (ka[v] == 2) walk<2><<<sms, 512>>>(m, cz, d_rev, d_blk, d_mark, d_markb, fl[v], d_sink);
            else walk<4><<<sms, 512>>>(m, cz, d_rev, d_blk, d_mark, d_markb, fl[v], d_sink);
        };
        for (int w = 0; w < 3; ++w) launch();
        const int R = 50;
        cudaEventRecord(e0);
        for (int r = 0; r < R; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %7.2f us per walk (%s)\n", names[v], ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
