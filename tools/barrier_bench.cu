// Grid-barrier latency on the B200: K back-to-back barriers in one
// persistent cooperative kernel, for several implementations.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/barrier_bench tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

struct Bar {
    unsigned gen;
    unsigned pad0[31];
    unsigned long long top;
    unsigned long long pad1[15];
    unsigned long long sub[64 * 16];
    unsigned flat;
};

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long atom_add_rel64(unsigned long long* p, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned atom_add_rel32(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_rel32(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// 0: cooperative groups
// 1: hierarchical, __threadfence around (current libbisim)
// 2: hierarchical, acq_rel atomics, no extra fences
// 3: flat counter: atom.acq_rel on one word, spin ld.acquire on gen
// 4: flat counter with generation in the same word (count up to nblocks*k)
__global__ void bench(Bar* b, int variant, int K, unsigned long long* out) {
    cg::grid_group grid = cg::this_grid();
    unsigned gen = 0;
    long long t0 = clock64();
    for (int k = 0; k < K; ++k) {
        if (variant == 0) {
            grid.sync();
        } else if (variant == 1 || variant == 2) {
            __syncthreads();
            if (threadIdx.x == 0) {
                const unsigned grp = blockIdx.x >> 4;
                const unsigned ngrp = (gridDim.x + 15) >> 4;
                const unsigned in_grp = min(16u, gridDim.x - (grp << 4));
                if (variant == 1) __threadfence();
                unsigned long long old = variant == 1 ? atomicAdd(&b->sub[grp << 4], 1ull)
                                                      : atom_add_rel64(&b->sub[grp << 4], 1ull);
                if ((old + 1) % in_grp == 0) {
                    unsigned long long t = variant == 1 ? atomicAdd(&b->top, 1ull) : atom_add_rel64(&b->top, 1ull);
                    if ((t + 1) % ngrp == 0) {
                        if (variant == 1) {
                            __threadfence();
                            atomicAdd(&b->gen, 1u);
                        } else {
                            red_rel32(&b->gen, 1u);
                        }
                    }
                }
                while (ld_acq(&b->gen) == gen) {
                }
                if (variant == 1) __threadfence();
            }
            ++gen;
            __syncthreads();
        } else if (variant == 3) {
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned old = atom_add_rel32(&b->flat, 1u);
                if ((old + 1) % gridDim.x == 0) red_rel32(&b->gen, 1u);
                while (ld_acq(&b->gen) == gen) {
                }
            }
            ++gen;
            __syncthreads();
        } else {
            __syncthreads();
            if (threadIdx.x == 0) {
                const unsigned target = (gen + 1) * gridDim.x;
                atom_add_rel32(&b->flat, 1u);
                while ((int)(ld_acq(&b->flat) - target) < 0) {
                }
            }
            ++gen;
            __syncthreads();
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}

int main() {
    Bar* b;
    unsigned long long* out;
    cudaMalloc(&b, sizeof(Bar));
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int K = 20000;
    for (int threads : {1024, 512}) {
        for (int per_sm : {1, 2}) {
            if (threads * per_sm > 2048) continue;
            int grid = sms * per_sm;
            for (int v = 0; v < 5; ++v) {
                cudaMemset(b, 0, sizeof(Bar));
                int vv = v, KK = K;
                void* args[] = {&b, &vv, &KK, &out};
                cudaLaunchCooperativeKernel((void*)bench, grid, threads, args, 0, 0);  // warm
                cudaMemset(b, 0, sizeof(Bar));
                cudaEventRecord(e0);
                cudaLaunchCooperativeKernel((void*)bench, grid, threads, args, 0, 0);
                cudaEventRecord(e1);
                cudaError_t err = cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("threads=%d grid=%d variant=%d  %.3f us/barrier  (%s)\n", threads, grid, v,
                       ms * 1e3 / K, cudaGetErrorString(err));
            }
        }
    }
    return 0;
}
