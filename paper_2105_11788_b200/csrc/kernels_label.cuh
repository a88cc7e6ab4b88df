// kernels_label.cuh -- label pre-partition by grouping equal label sets.
//
// bcrp.py:144-184 refines the trivial partition by "has an outgoing a-edge"
// for every action a in turn, electing minimum-index leaders; its result is
// the canonical partition of states by outgoing label SET (leader = smallest
// state of the set class).  Instead of |Act| grid-wide
// mark-and-split rounds, every state hashes its label mask, the minimum
// state per distinct mask is found in a hash table (shared-memory
// aggregation per CTA first, so a few popular label sets do not serialise
// on one global cell), and each state takes its group's minimum as leader.
// A final pass compares each state's mask with its leader's; any 64-bit hash
// collision makes the host fall back to the literal rounds (k_label_rounds).
#pragma once

#include "kernels.cuh"

namespace bisim {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// h[s] = nonzero 64-bit hash of s's label mask
__global__ void k_label_hash(int32_t n, int32_t W, const unsigned long long* __restrict__ lmask,
                             unsigned long long* h) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long x = 0x243F6A8885A308D3ull;
        for (int32_t w = 0; w < W; ++w) x = mix64(x ^ lmask[(int64_t)w * n + s]);
        h[s] = x | 1ull;
    }
}

__device__ __forceinline__ void table_insert(unsigned long long* keys, int32_t* mins, uint64_t mask,
                                             unsigned long long key, int32_t s) {
    uint64_t slot = (key >> 11) & mask;
    for (;;) {
        const unsigned long long k = atomicCAS(&keys[slot], 0ull, key);
        if (k == 0ull || k == key) {
            atomicMin(&mins[slot], s);
            return;
        }
        slot = (slot + 1) & mask;
    }
}

constexpr int kLocalKeys = 1024;

__global__ void k_label_insert(int32_t n, const unsigned long long* __restrict__ h,
                               unsigned long long* keys, int32_t* mins, uint64_t mask) {
    __shared__ unsigned long long skey[kLocalKeys];
    __shared__ int32_t smin[kLocalKeys];
    for (int k = threadIdx.x; k < kLocalKeys; k += blockDim.x) {
        skey[k] = 0ull;
        smin[k] = kBig;
    }
    __syncthreads();
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = h[s];
        uint32_t slot = (uint32_t)key & (kLocalKeys - 1);
        bool done = false;
        for (int probe = 0; probe < 8 && !done; ++probe) {
            const unsigned long long k = atomicCAS(&skey[slot], 0ull, key);
            if (k == 0ull || k == key) {
                atomicMin(&smin[slot], (int32_t)s);
                done = true;
            }
            slot = (slot + 1) & (kLocalKeys - 1);
        }
        if (!done) table_insert(keys, mins, mask, key, (int32_t)s);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kLocalKeys; k += blockDim.x)
        if (skey[k]) table_insert(keys, mins, mask, skey[k], smin[k]);
}

__global__ void k_label_assign(int32_t n, int32_t W, const unsigned long long* __restrict__ h,
                               const unsigned long long* __restrict__ keys, const int32_t* __restrict__ mins,
                               uint64_t mask, const unsigned long long* __restrict__ lmask, int32_t* block,
                               int32_t* mismatch) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n;
         s += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = h[s];
        uint64_t slot = (key >> 11) & mask;
        while (keys[slot] != key) slot = (slot + 1) & mask;
        const int32_t l = mins[slot];
        block[s] = l;
        for (int32_t w = 0; w < W; ++w)
            if (lmask[(int64_t)w * n + s] != lmask[(int64_t)w * n + l]) *mismatch = 1;
    }
}

}  // namespace bisim
