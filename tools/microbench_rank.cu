// Microbenchmark: warp ranking primitives on sm_100a (match.any vs 8-ballot multisplit vs smem atomics).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ uint32_t peers_ballot(uint32_t d) {
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const uint32_t m = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? m : ~m;
    }
    return peers;
}
template <int MODE>
__global__ void k(const uint32_t *keys, uint32_t *out, int iters) {
    __shared__ uint32_t h[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t key = keys[blockIdx.x * blockDim.x + threadIdx.x];
    uint32_t acc = 0;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int it = 0; it < iters; it++) {
        key = key * 1664525u + 1013904223u;
        const uint32_t d = key >> 24;
        if (MODE == 0) {
            const uint32_t p = __match_any_sync(0xffffffffu, d);
            acc += __popc(p);
            if ((__ffs(p) - 1) == lane) h[w][d] += __popc(p);
        } else if (MODE == 1) {
            const uint32_t p = peers_ballot(d);
            acc += __popc(p);
            if ((__ffs(p) - 1) == lane) h[w][d] += __popc(p);
        } else {
            atomicAdd(&h[w][d], 1u);
        }
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + h[w][lane];
}
int main() {
    const int blocks = 148 * 8, threads = 256, iters = 2048;
    uint32_t *keys, *out;
    cudaMalloc(&keys, blocks * threads * 4);
    cudaMalloc(&out, blocks * threads * 4);
    { uint32_t *h = (uint32_t *)malloc(blocks * threads * 4); for (int i = 0; i < blocks * threads; i++) h[i] = (uint32_t)i * 2654435761u; cudaMemcpy(keys, h, blocks * threads * 4, cudaMemcpyHostToDevice); free(h); }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char *names[3] = {"match_any", "8-ballot multisplit", "smem atomicAdd"};
    for (int mode = 0; mode < 3; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, threads>>>(keys, out, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(keys, out, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(keys, out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double elems = (double)blocks * threads * iters;
            if (rep) printf("%-22s %8.3f ms  %7.1f G elem/s  %.3f ns/elem/SM\n", names[mode], ms, elems / ms / 1e6,
                            ms * 1e6 / (elems / 148));
        }
    }
    return 0;
}
