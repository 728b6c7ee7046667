// Dependent-chain latency of warp collectives on sm_100a (one warp, clock64 deltas):
// CREDUX (__reduce_min_sync), VOTE (__ballot_sync) + FLO, SHFL, LDS, IADD3, and the
// REDUX -> vector move.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 lat.cu -o lat
#include <cstdio>
#include <cuda_runtime.h>
#define N 256
__global__ void k(unsigned *out, long long *t, unsigned seed) {
    __shared__ unsigned sm[64];
    const unsigned lane = threadIdx.x;
    sm[lane] = lane * seed; sm[lane + 32] = lane;
    __syncwarp();
    unsigned x = lane ^ seed;
    long long t0, t1;
    // 1. REDUX min chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) x = __reduce_min_sync(0xffffffffu, x + lane) ^ i;
    t1 = clock64(); if (lane == 0) t[0] = t1 - t0;
    // 2. ballot + ffs chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) x = __ffs(__ballot_sync(0xffffffffu, ((x + lane) & 7) == 0)) + i;
    t1 = clock64(); if (lane == 0) t[1] = t1 - t0;
    // 3. shfl chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (x + i) & 31);
    t1 = clock64(); if (lane == 0) t[2] = t1 - t0;
    // 4. lds chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) x = sm[(x + i) & 63];
    t1 = clock64(); if (lane == 0) t[3] = t1 - t0;
    // 5. alu chain (iadd/lop)
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) x = (x * 3u + i) ^ (x >> 3);
    t1 = clock64(); if (lane == 0) t[4] = t1 - t0;
    // 6. empty loop
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) x = x + i;
    t1 = clock64(); if (lane == 0) t[5] = t1 - t0;
    // 7. any_sync chain
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) x = __any_sync(0xffffffffu, ((x + lane + i) & 15) == 0) + x + i;
    t1 = clock64(); if (lane == 0) t[6] = t1 - t0;
    // 8. REDUX + data-dependent branch
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < N; ++i) { unsigned r = __reduce_min_sync(0xffffffffu, x + lane); if (r & 1) x += 3; else x ^= 5; }
    t1 = clock64(); if (lane == 0) t[7] = t1 - t0;
    out[lane] = x;
}
int main() {
    unsigned *o; long long *t, h[8];
    cudaMalloc(&o, 128); cudaMalloc(&t, 64);
    for (int r = 0; r < 3; ++r) k<<<1, 32>>>(o, t, 7 + r);
    cudaMemcpy(h, t, 64, cudaMemcpyDeviceToHost);
    const char *nm[8] = {"redux.min", "ballot+ffs", "shfl.idx", "lds", "alu(imad+lop+shf)", "loop only", "vote.any", "redux+branch"};
    for (int i = 0; i < 8; ++i) printf("%-20s %6.1f cycles/iter\n", nm[i], (double)h[i] / N);
    return 0;
}
