// Single-warp and per-SM DMMA (m8n8k4 f64) issue rate with independent accumulators.
#include <cstdio>
template <int NACC>
__global__ void k(double* out, long long* cyc, int iters) {
    double c[NACC][2];
    const double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    long long t1 = clock64();
    double s = 0; for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x % 32 == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = (t1 - t0);
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 1 << 20);
    const int iters = 4096;
    for (int warps : {1, 2, 4, 8, 16}) {
        k<16><<<1, 32 * warps>>>(o, c, 16);
        k<16><<<1, 32 * warps>>>(o, c, iters);
        long long h[16]; cudaMemcpy(h, c, 8 * warps, cudaMemcpyDeviceToHost);
        double cyc = 0; for (int w = 0; w < warps; ++w) cyc = h[w] > cyc ? h[w] : cyc;
        printf("warps/SM %2d: %.2f cycles per DMMA per warp, SM rate %.2f cycles/DMMA\n", warps, cyc / (iters * 16.0),
               cyc / (iters * 16.0 * warps));
    }
    return 0;
}
