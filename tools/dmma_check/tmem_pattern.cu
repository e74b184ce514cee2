// Single-warp latency of the TMEM access patterns of the dmma1 sweep kernel (development aid).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void tld4(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void tld16(uint32_t a, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(a));
}
__device__ __forceinline__ void tst16(uint32_t a, const uint32_t (&r)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void wld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wst() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
template <int K> __device__ __forceinline__ void pin(uint32_t (&r)[K]) {
#pragma unroll
    for (int i = 0; i < K; ++i) asm volatile("" : "+r"(r[i]));
}
__device__ __forceinline__ void mma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k(long long* cyc, double* sink, int iters) {
    __shared__ uint32_t base_sh;
    __shared__ double ur[1024];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&base_sh)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = base_sh + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t z[16];
    for (int i = 0; i < 16; ++i) z[i] = __float_as_uint(1.0f) * 0u + i;
    for (int c = 0; c < 160; c += 16) tst16(base + c, z);
    wst();
    double acc = 0;
    long long t0, t1;
    // A) gather pattern: wait::st; 5 x ld4 at a runtime tile-row; wait::ld; STS from holder lanes
    t0 = clock64();
    int p = lane & 7;
    for (int it = 0; it < iters; ++it) {
        uint32_t rv[5][4];
        const int ptr = (p + it) & 7;
#pragma unroll
        for (int tt = 0; tt < 5; ++tt) tld4(base + (uint32_t)((tt * 8 + ptr) * 4), rv[tt]);
        wld();
#pragma unroll
        for (int tt = 0; tt < 5; ++tt) {
            pin(rv[tt]);
            if ((lane >> 2) == (ptr & 7)) ur[tt * 8 + (lane & 3) * 2] = __uint_as_float(rv[tt][0]);
        }
        __syncwarp();
        p += (int)ur[lane & 7] & 1;
    }
    t1 = clock64();
    if (lane == 0) cyc[0] = (t1 - t0) / iters;
    // B) update group: wait::st; ld16; wait::ld; 4 DMMA; st16 (dependent chain over groups)
    double a = 1.0 + lane, b = 0.5;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t col = base + (uint32_t)((it % 10) * 16);
        uint32_t r[16];
        wst();
        tld16(col, r);
        wld();
        pin(r);
        double v[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) { v[j][0] = __hiloint2double(r[4*j+1], r[4*j]); v[j][1] = __hiloint2double(r[4*j+3], r[4*j+2]); }
#pragma unroll
        for (int j = 0; j < 4; ++j) mma(v[j][0], v[j][1], a, b);
#pragma unroll
        for (int j = 0; j < 4; ++j) { r[4*j] = __double2loint(v[j][0]); r[4*j+1] = __double2hiint(v[j][0]); r[4*j+2] = __double2loint(v[j][1]); r[4*j+3] = __double2hiint(v[j][1]); }
        tst16(col, r);
    }
    wst();
    t1 = clock64();
    if (lane == 0) cyc[1] = (t1 - t0) / iters;
    // C) same without wait::st inside
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t col = base + (uint32_t)((it % 10) * 16);
        uint32_t r[16];
        tld16(col, r);
        wld();
        pin(r);
        double v[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) { v[j][0] = __hiloint2double(r[4*j+1], r[4*j]); v[j][1] = __hiloint2double(r[4*j+3], r[4*j+2]); }
#pragma unroll
        for (int j = 0; j < 4; ++j) mma(v[j][0], v[j][1], a, b);
#pragma unroll
        for (int j = 0; j < 4; ++j) { r[4*j] = __double2loint(v[j][0]); r[4*j+1] = __double2hiint(v[j][0]); r[4*j+2] = __double2loint(v[j][1]); r[4*j+3] = __double2hiint(v[j][1]); }
        tst16(col, r);
    }
    wst();
    t1 = clock64();
    if (lane == 0) cyc[2] = (t1 - t0) / iters;
    // D) just ld16 + wait::ld
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[16];
        tld16(base + (uint32_t)((it % 10) * 16), r);
        wld();
        pin(r);
        acc += __uint_as_float(r[it & 15]);
    }
    t1 = clock64();
    if (lane == 0) cyc[3] = (t1 - t0) / iters;
    // E) 4 independent DMMA
    t0 = clock64();
    double v[4][2] = {{1, 2}, {3, 4}, {5, 6}, {7, 8}};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j) mma(v[j][0], v[j][1], a, b);
    }
    t1 = clock64();
    if (lane == 0) cyc[4] = (t1 - t0) / iters;
    // F) STS by 4 holder lanes + syncwarp + LDS by all (UR round trip)
    t0 = clock64();
    double x = lane;
    for (int it = 0; it < iters; ++it) {
        if ((lane >> 2) == (it & 7)) ur[(lane & 3) * 2] = x;
        __syncwarp();
        x = ur[lane & 7] + 1.0;
        __syncwarp();
    }
    t1 = clock64();
    if (lane == 0) cyc[5] = (t1 - t0) / iters;
    sink[threadIdx.x] = acc + p + v[0][0] + v[3][1] + x;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base_sh));
}
int main() {
    long long* c; double* s;
    cudaMalloc(&c, 1024); cudaMalloc(&s, 1 << 16);
    k<<<1, 32>>>(c, s, 16);
    k<<<1, 32>>>(c, s, 4096);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[6];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    printf("single warp, cycles per iteration:\n A gather t (5 ld4 + wait + STS + syncwarp + LDS) %lld\n B update group (wait::st ld16 wait 4 DMMA st16) %lld\n"
           " C update group without wait::st %lld\n D ld16 + wait::ld %lld\n E 4 independent DMMA %lld\n F STS-syncwarp-LDS-syncwarp %lld\n",
           h[0], h[1], h[2], h[3], h[4], h[5]);
    return 0;
}
