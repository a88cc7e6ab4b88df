// Grid-barrier latency with thread-block clusters on the B200: is a
// hierarchical barrier (hardware cluster barrier + one global arrival per
// cluster) cheaper than the flat 148-arrival counter of kernels_sparse.cuh?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/cbb tools/cluster_barrier_bench.cu
// Each variant runs K barriers back to back in one cooperative (+cluster)
// launch; with `work`, every thread stores to its own global word between
// barriers so the release side has something to flush.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

struct Bar {
    unsigned flat;
    unsigned pad[31];
};

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel32(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_n() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// variant 0: flat counter (libbisim's grid_barrier)
// variant 1: cluster barrier, rank-0 CTA arrives globally and spins, cluster barrier
// variant 2: cluster barrier, rank-0 arrives, every CTA's thread 0 spins on the counter
// variant 3: the first cluster alone syncs with the hardware cluster barrier (team = 1 cluster)
__global__ void bench(Bar* b, int variant, int K, int work, unsigned* sink, unsigned long long* out) {
    unsigned gen = 0;
    const unsigned ncl = gridDim.x / (variant ? cluster_n() : 1u);
    long long t0 = clock64();
    for (int k = 0; k < K; ++k) {
        if (work) sink[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = k;
        if (variant == 0) {
            __syncthreads();
            if (threadIdx.x == 0) {
                const unsigned target = (gen + 1) * gridDim.x;
                red_rel32(&b->flat, 1u);
                while ((int)(ld_acq(&b->flat) - target) < 0) {
                }
            }
            ++gen;
            __syncthreads();
        } else if (variant == 1) {
            cluster_sync_all();
            if (cluster_rank() == 0 && threadIdx.x == 0) {
                const unsigned target = (gen + 1) * ncl;
                red_rel32(&b->flat, 1u);
                while ((int)(ld_acq(&b->flat) - target) < 0) {
                }
            }
            ++gen;
            cluster_sync_all();
        } else if (variant == 3) {
            // the cluster alone (a cluster-sized team): hardware cluster barrier only
            if (blockIdx.x < cluster_n()) cluster_sync_all();
        } else {
            cluster_sync_all();
            if (threadIdx.x == 0) {
                const unsigned target = (gen + 1) * ncl;
                if (cluster_rank() == 0) red_rel32(&b->flat, 1u);
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
    unsigned* sink;
    cudaMalloc(&b, sizeof(Bar));
    cudaMalloc(&out, 8);
    cudaMalloc(&sink, 148 * 1024 * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int K = 20000;
    const int threads = 512;
    cudaFuncSetAttribute((void*)bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int work : {0, 1}) {
        for (int cl : {1, 2, 4, 8, 16}) {
            for (int v = 0; v < 4; ++v) {
                if ((cl == 1) != (v == 0)) continue;
                // largest grid of whole clusters that is co-resident
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute at[2];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cl;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                at[1].id = cudaLaunchAttributeCooperative;
                at[1].val.cooperative = 1;
                cfg.blockDim = dim3(threads);
                cfg.gridDim = dim3(sms / cl * cl);
                cfg.attrs = at;
                cfg.numAttrs = 2;
                int ncl = 0;
                cudaError_t qe = cudaOccupancyMaxActiveClusters(&ncl, (void*)bench, &cfg);
                int grid = std::min(sms / cl, ncl) * cl;
                if (qe != cudaSuccess || grid == 0) {
                    printf("cluster=%d: occupancy query %s (ncl=%d)\n", cl, cudaGetErrorString(qe), ncl);
                    cudaGetLastError();
                    continue;
                }
                cfg.gridDim = dim3(grid);
                int vv = v, KK = K, ww = work;
                cudaMemset(b, 0, sizeof(Bar));
                cudaError_t le = cudaLaunchKernelEx(&cfg, bench, b, vv, 100, ww, sink, out);  // warm
                cudaDeviceSynchronize();
                cudaMemset(b, 0, sizeof(Bar));
                cudaEventRecord(e0);
                le = cudaLaunchKernelEx(&cfg, bench, b, vv, KK, ww, sink, out);
                cudaEventRecord(e1);
                cudaError_t err = cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("work=%d cluster=%2d grid=%3d (max clusters %3d) variant=%d  %.3f us/barrier  (%s / %s)\n", work,
                       cl, grid, ncl, v, ms * 1e3 / K, cudaGetErrorString(le), cudaGetErrorString(err));
            }
        }
    }
    return 0;
}
