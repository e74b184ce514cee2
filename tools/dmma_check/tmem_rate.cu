// TMEM (tcgen05.ld/st 32x32b) latency and throughput on B200, 1 CTA per SM.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void tld4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void tld32(uint32_t addr, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(addr));
}
__device__ __forceinline__ void tst4(uint32_t addr, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3]));
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__global__ void k(long long* cyc, unsigned* sink, int iters) {
    __shared__ uint32_t base_sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = base_sh;
    const int nw = blockDim.x / 32;
    const int per_q = (nw + 3) / 4;                          // warps sharing a lane quarter
    const uint32_t col0 = (uint32_t)((warp / 4) * (512 / per_q));
    const uint32_t addr = base + ((uint32_t)(32 * (warp % 4)) << 16) + col0;
    uint32_t r[4] = {(uint32_t)lane, 1u, 2u, 3u};
    tst4(addr, r);
    twait_st();
    // 1) dependent load latency (x4): address depends on the previous value
    long long t0 = clock64();
    uint32_t a = addr;
    for (int i = 0; i < iters; ++i) {
        uint32_t v[4];
        tld4(a, v);
        twait_ld();
        a = addr + (v[0] & 0u);
    }
    long long t1 = clock64();
    // 2) load throughput: x32 loads back to back, one wait per 4
    uint32_t acc = 0;
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t v0[32], v1[32];
        tld32(addr, v0);
        tld32(addr + 32, v1);
        twait_ld();
        acc += v0[0] + v1[31];
    }
    long long t3 = clock64();
    // 3) store + load round trip (update pattern): st x4 then ld x4 of the same columns
    long long t4 = clock64();
    uint32_t w[4] = {1u, 2u, 3u, 4u};
    for (int i = 0; i < iters; ++i) {
        tst4(addr + 4 * (i & 7), w);
        twait_st();
        uint32_t v[4];
        tld4(addr + 4 * (i & 7), v);
        twait_ld();
        w[0] = v[0] + 1;
    }
    long long t5 = clock64();
    if (lane == 0) {
        cyc[(blockIdx.x * nw + warp) * 3 + 0] = (t1 - t0) / iters;
        cyc[(blockIdx.x * nw + warp) * 3 + 1] = (t3 - t2);
        cyc[(blockIdx.x * nw + warp) * 3 + 2] = (t5 - t4) / iters;
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + w[0];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
    long long* c; unsigned* s;
    cudaMalloc(&c, 1 << 20); cudaMalloc(&s, 1 << 22);
    const int iters = 2048;
    for (int nw : {1, 4, 8, 12, 16}) {
        k<<<148, 32 * nw>>>(c, s, 16);
        k<<<148, 32 * nw>>>(c, s, iters);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        long long h[48];
        cudaMemcpy(h, c, sizeof(long long) * 3 * nw, cudaMemcpyDeviceToHost);
        long long mx = 0; for (int w = 0; w < nw; ++w) mx = h[3 * w + 1] > mx ? h[3 * w + 1] : mx;
        const double bytes = (double)nw * iters * 2 * 32 * 32 * 4;   // per SM
        printf("warps %2d: ld x4 dependent latency %lld cyc | ld throughput %.1f B/cyc/SM | st->ld round trip %lld cyc\n",
               nw, h[0], bytes / mx, h[2]);
    }
    return 0;
}
