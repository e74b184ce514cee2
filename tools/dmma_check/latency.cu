// Dependent-chain latency microbenchmarks (single warp, clock64) for the ops on the
// pivot-step critical path of the sweep kernels.
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters) {
    const int lane = threadIdx.x;
    double x = 1.0 + lane * 1e-3;
    unsigned u = lane * 7 + 1;
    __shared__ double sm[64];
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-9);
    t1 = clock64(); if (lane == 0) cyc[0] = (t1 - t0) / iters;
    // double SHFL chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) + 1e-9;
    t1 = clock64(); if (lane == 0) cyc[1] = (t1 - t0) / iters;
    // redux max + ballot + ffs + shfl (pivot selection)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        unsigned m = __reduce_max_sync(0xffffffffu, u);
        unsigned b = __ballot_sync(0xffffffffu, u == m);
        int src = __ffs(b) - 1;
        u = __shfl_sync(0xffffffffu, u, src) + lane;
    }
    t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0) / iters;
    // FP64 division chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = 1.0 / (x + 1.5);
    t1 = clock64(); if (lane == 0) cyc[3] = (t1 - t0) / iters;
    // SMEM store -> syncwarp -> load round trip
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (lane == (i & 31)) sm[lane] = x;
        __syncwarp();
        x = sm[i & 31] + 1e-9;
        __syncwarp();
    }
    t1 = clock64(); if (lane == 0) cyc[4] = (t1 - t0) / iters;
    // DMMA dependent chain
    double c0 = x, c1 = x;
    t0 = clock64();
    for (int i = 0; i < iters; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(x), "d"(x));
    t1 = clock64(); if (lane == 0) cyc[5] = (t1 - t0) / iters;
    out[lane] = x + u + c0 + c1;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    k<<<1, 32>>>(o, c, 16); k<<<1, 32>>>(o, c, 1024);
    long long h[8]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op: DFMA %lld | SHFL(f64)+DADD %lld | REDUX+BALLOT+FFS+SHFL %lld | DDIV %lld | STS-syncwarp-LDS %lld | DMMA %lld\n",
           h[0], h[1], h[2], h[3], h[4], h[5]);
    return 0;
}
