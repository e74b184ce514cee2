// LDG.128 stream rate of a 128 KiB element tensor into one SM's registers for two lane->address
// patterns: (0) 512 contiguous bytes per warp instruction; (1) the sweep kernel's planar DMMA-fragment
// pattern (lane (g,q): 8 rows x 16 B = one 128-byte line per q, four lines 2 KiB apart per instruction).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int WARPS = 12, BLK = 131072;
template <int MODE>
__global__ void __launch_bounds__(32 * WARPS, 1) k(const double2* T, int nblk, int iters, double* out, long long* cyc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    double s = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double2* b = T + (size_t)((blockIdx.x * WARPS + warp + it * 977) % nblk) * (BLK / 16);
#pragma unroll 1
        for (int i = 0; i < 16; ++i) {   // 16 groups of 16 loads: (tile-column tc = i / 2, row half h = i % 2)
            double2 v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                size_t idx;
                if (MODE == 0) idx = (size_t)(i * 16 + u) * 32 + lane;
                else {
                    const int tc = i >> 1, tr = 4 * (i & 1) + (u >> 2), sl = (u >> 1) & 1, p = u & 1;
                    const int c = 8 * tc + 2 * q + sl, r = 8 * tr + g;
                    idx = (size_t)(2 * c + p) * 64 + r;
                }
                v[u] = __ldg(b + idx);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) s += v[u].x + v[u].y;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nblk = 512;
    double2* T; cudaMalloc(&T, (size_t)nblk * BLK); cudaMemset(T, 0, (size_t)nblk * BLK);
    double* out; cudaMalloc(&out, sms * 32 * WARPS * 8); long long* cyc; cudaMalloc(&cyc, sms * 8);
    long long* h = new long long[sms]; const int iters = 40;
    for (int mode = 0; mode < 2; ++mode) {
        for (int r = 0; r < 2; ++r) { if (mode == 0) k<0><<<sms, 32 * WARPS>>>(T, nblk, iters, out, cyc); else k<1><<<sms, 32 * WARPS>>>(T, nblk, iters, out, cyc); }
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
        double m = 0; for (int i = 0; i < sms; ++i) m += h[i]; m /= sms;
        printf("%s: %.0f cycles per 128 KiB per warp (12 warps), %.1f B/clk/SM\n", mode ? "fragment pattern (4 lines per LDG.128)" : "contiguous 512 B per LDG.128", m / iters, (double)WARPS * iters * BLK / m);
    }
    return 0;
}
