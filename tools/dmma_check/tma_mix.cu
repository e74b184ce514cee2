// Does a global->SM stream take shared-memory (LSU data pipe) bandwidth away from other warps?
// 6 "stream" warps per SM move 128 KiB blocks (mode 0: LDG.128 into registers; mode 1: cp.async.bulk
// (TMA) 512-byte segments into a shared ring + LDS.128; mode 2: idle) while 6 "smem" warps run a
// fixed number of conflict-free LDS.128/STS.128 round trips; reports the smem warps' cycles.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int WARPS = 12, SW = 6, BLK = 131072, CHUNK = 8192, SLOTS = 2, SEG = 512;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(32 * WARPS, 1) k(const double2* T, int nblk, int iters, int mode, int smem_iters, double* out, long long* cyc) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ int stop;
    if (threadIdx.x == 0) stop = 0;
    unsigned char* ring = sm + (size_t)warp * SLOTS * CHUNK;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)WARPS * SLOTS * CHUNK) + warp * SLOTS;
    if (lane < SLOTS) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(bars + lane)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    double s = 0.0;
    if (warp >= SW) {   // shared-memory warps: fixed work, timed
        volatile double2* p = reinterpret_cast<volatile double2*>(ring) + lane;
        long long t0 = clock64();
        double2 v = make_double2(lane, 1.0);
        for (int i = 0; i < smem_iters; ++i) {
#pragma unroll
            for (int u = 0; u < 8; ++u) { p[u * 32].x = v.x; p[u * 32].y = v.y; }
#pragma unroll
            for (int u = 0; u < 8; ++u) { v.x += p[u * 32].y; v.y += p[u * 32].x; }
        }
        long long t1 = clock64();
        s = v.x + v.y;
        if (lane == 0) cyc[blockIdx.x * WARPS + warp] = t1 - t0;
        __syncwarp();
        if (lane == 0) atomicAdd(&stop, 1);
    } else if (mode == 0) {
        int it = 0;
        while (*(volatile int*)&stop < WARPS - SW) {
            const double2* b = T + (size_t)((blockIdx.x * WARPS + warp + (it++) * 977) % nblk) * (BLK / 16);
#pragma unroll 1
            for (int i = 0; i < BLK / 16 / 32; i += 16) {
                double2 v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = __ldg(b + (size_t)(i + u) * 32 + lane);
#pragma unroll
                for (int u = 0; u < 16; ++u) s += v[u].x + v[u].y;
            }
        }
        if (lane == 0) cyc[blockIdx.x * WARPS + warp] = it;
    } else if (mode == 1) {
        const int nch = BLK / CHUNK;
        int issued = 0, used = 0;
        auto issue = [&](int n) {
            const int it = n / nch, c = n % nch, slot = n % SLOTS;
            const char* b = reinterpret_cast<const char*>(T) + (size_t)((blockIdx.x * WARPS + warp + it * 977) % nblk) * BLK + (size_t)c * CHUNK;
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bars + slot)), "r"(CHUNK) : "memory");
            __syncwarp();
            if (lane < CHUNK / SEG)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 sa(ring + slot * CHUNK + lane * SEG)), "l"(b + lane * SEG), "r"(SEG), "r"(sa(bars + slot)) : "memory");
        };
        issue(issued++);
        while (*(volatile int*)&stop < WARPS - SW) {
            issue(issued); ++issued;
            const int slot = used % SLOTS; const unsigned par = (used / SLOTS) & 1;
            unsigned ok = 0;
            while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sa(bars + slot)), "r"(par) : "memory");
            const double2* c = reinterpret_cast<const double2*>(ring + slot * CHUNK);
#pragma unroll
            for (int u = 0; u < CHUNK / 16 / 32; ++u) { double2 v = c[u * 32 + lane]; s += v.x + v.y; }
            __syncwarp();
            ++used;
        }
        {   // drain the copy in flight before exit
            const int slot = used % SLOTS; const unsigned par = (used / SLOTS) & 1;
            unsigned ok = 0;
            while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sa(bars + slot)), "r"(par) : "memory");
        }
        if (lane == 0) cyc[blockIdx.x * WARPS + warp] = used * (long long)CHUNK / BLK;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nblk = 512;
    double2* T; cudaMalloc(&T, (size_t)nblk * BLK); cudaMemset(T, 0, (size_t)nblk * BLK);
    double* out; cudaMalloc(&out, sms * 32 * WARPS * 8); long long* cyc; cudaMalloc(&cyc, sms * WARPS * 8);
    long long* h = new long long[sms * WARPS];
    const size_t smem = (size_t)WARPS * SLOTS * CHUNK + WARPS * SLOTS * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int smem_iters = 20000;
    const char* names[3] = {"LDG.128 stream", "TMA 512 B segments + LDS.128", "no stream"};
    for (int mode : {2, 0, 1, 2}) {
        for (int r = 0; r < 2; ++r) k<<<sms, 32 * WARPS, smem>>>(T, nblk, 0, mode, smem_iters, out, cyc);
        cudaDeviceSynchronize(); cudaError_t e = cudaGetLastError(); if (e) { printf("%s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, cyc, sms * WARPS * 8, cudaMemcpyDeviceToHost);
        double c = 0, b = 0; for (int i = 0; i < sms; ++i) for (int w = 0; w < WARPS; ++w) (w >= SW ? c : b) += h[i * WARPS + w];
        c /= sms * (WARPS - SW); b /= sms;
        // per smem-warp iteration: 16 STS.64 + 16 LDS.64 (volatile), 2 wavefronts each = 64 wavefronts
        printf("%-32s smem warps: %.0f cycles (%.2f wavefronts/clk/SM); streamed %.0f blocks/SM = %.1f B/clk/SM\n", names[mode], c,
               (double)(WARPS - SW) * smem_iters * 64 / c, b, b * BLK / c);
    }
    return 0;
}
