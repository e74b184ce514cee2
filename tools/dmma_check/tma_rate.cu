// Stream rate of per-warp 128 KiB blocks into one SM: (0) LDG.128 from L2 into registers (the
// sweep kernel's element-tensor pass), (1) cp.async.bulk (TMA) 256-byte segments into a per-warp
// shared-memory ring + LDS.128.  12 warps per CTA, one CTA per SM, L2-resident working set.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int WARPS = 12, BLK = 131072, SEG = 256, CHUNK = 4096, SLOTS = 4;
__global__ void __launch_bounds__(32 * WARPS, 1) k_ldg(const double2* T, int nblk, int iters, double* out, long long* cyc) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double s = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double2* b = T + (size_t)((blockIdx.x * WARPS + warp + it * 977) % nblk) * (BLK / 16);
#pragma unroll 1
        for (int i = 0; i < BLK / 16 / 32; i += 16) {
            double2 v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = __ldg(b + (size_t)(i + u) * 32 + lane);
#pragma unroll
            for (int u = 0; u < 16; ++u) s += v[u].x + v[u].y;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32 * WARPS, 1) k_tma(const double2* T, int nblk, int iters, double* out, long long* cyc, int seg) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* ring = sm + (size_t)warp * SLOTS * CHUNK;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)WARPS * SLOTS * CHUNK) + warp * SLOTS;
    if (lane < SLOTS) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bars + lane)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const int nseg = CHUNK / seg;           // segments per chunk (one per lane)
    const int nch = BLK / CHUNK;
    double s = 0.0;
    long long t0 = clock64();
    int issued = 0, used = 0;
    const int total = iters * nch;
    auto issue = [&](int n) {
        const int it = n / nch, c = n % nch, slot = n % SLOTS;
        const char* b = reinterpret_cast<const char*>(T) + (size_t)((blockIdx.x * WARPS + warp + it * 977) % nblk) * BLK + (size_t)c * CHUNK;
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bars + slot)), "r"(CHUNK) : "memory");
        __syncwarp();
        if (lane < nseg)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             sa(ring + slot * CHUNK + lane * seg)), "l"(b + lane * seg), "r"(seg), "r"(sa(bars + slot)) : "memory");
    };
    for (; issued < SLOTS - 1 && issued < total; ++issued) issue(issued);
    for (; used < total; ++used) {
        if (issued < total) { issue(issued); ++issued; }
        const int slot = used % SLOTS; const unsigned par = (used / SLOTS) & 1;
        unsigned ok = 0;
        while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sa(bars + slot)), "r"(par) : "memory");
        const double2* c = reinterpret_cast<const double2*>(ring + slot * CHUNK);
#pragma unroll
        for (int u = 0; u < CHUNK / 16 / 32; ++u) { double2 v = c[u * 32 + lane]; s += v.x + v.y; }
        __syncwarp();
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nblk = 512;  // 64 MiB: L2-resident
    double2* T; cudaMalloc(&T, (size_t)nblk * BLK); cudaMemset(T, 0, (size_t)nblk * BLK);
    double* out; cudaMalloc(&out, sms * 32 * WARPS * 8); long long* cyc; cudaMalloc(&cyc, sms * 8);
    const int iters = 40;
    long long* h = new long long[sms];
    auto rep = [&](const char* name) {
        cudaDeviceSynchronize(); cudaError_t e = cudaGetLastError(); if (e) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
        cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
        double m = 0; for (int i = 0; i < sms; ++i) m += h[i]; m /= sms;
        printf("%s: %.0f cycles per 128 KiB block per warp (12 warps), %.1f B/clk/SM\n", name, m / iters, (double)WARPS * iters * BLK / m);
    };
    for (int r = 0; r < 2; ++r) { k_ldg<<<sms, 32 * WARPS>>>(T, nblk, iters, out, cyc); } rep("LDG.128 -> registers");
    const size_t smem = (size_t)WARPS * SLOTS * CHUNK + WARPS * SLOTS * 8;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int seg : {256, 512, 1024, 4096}) {
        for (int r = 0; r < 2; ++r) k_tma<<<sms, 32 * WARPS, smem>>>(T, nblk, iters, out, cyc, seg);
        char nm[64]; snprintf(nm, 64, "TMA bulk %d B segments + LDS.128", seg); rep(nm);
    }
    return 0;
}
