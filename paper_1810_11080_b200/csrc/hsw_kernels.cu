// CUDA kernels of the B200 transport sweep (sm_100a).
//
//   K1s scatter_source      rhs base s_e = q_vol + (1/4pi) sigma_s M phi_e (solver.hpp:105-108)
//   K2/K3 phi_norms         phi = sum_d w_d psi_d in ascending d (solver.hpp:157-158),
//                           max_d ||dpsi||_inf (solver.hpp:150-156), ||dphi||_2, ||phi||_2;
//                           fixed-shape tree reductions, atomic-free, deterministic.
#include "hsw_internal.hpp"

#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <string>

namespace hsw {

#define KCHECK(x)                                                                              \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess)                                                                 \
            throw Error(-8, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x);       \
    } while (0)

// ------------------------------------------------------------ scatter source
__global__ void scatter_source_kernel(const DevProblem pr, const double* __restrict__ phi, double* __restrict__ src) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int nb = pr.nb;
    if (i >= (int64_t)pr.nel * nb) return;
    const int e = (int)(i / nb), m = (int)(i - (i / nb) * nb);
    const double* ph = phi + (size_t)e * nb;
    double s = 0.0;
    for (int n = 0; n < nb; ++n) s += pr.T[t_idx(e, nb, m, n, 0)] * ph[n];   // M[m][n]
    const double c4pi = 1.0 / (4.0 * 3.14159265358979323846);
    src[i] = pr.qvol[i] + c4pi * (pr.sig_s[e] * s);
}

void dev_scatter_source(const DevProblem& P, const double* phi, double* src, void* stream) {
    const int64_t n = (int64_t)P.nel * P.nb;
    scatter_source_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(P, phi, src);
    KCHECK(cudaGetLastError());
}

// --------------------------------------------------- phi reduction and norms
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 1024;

__global__ void __launch_bounds__(kRedThreads)
phi_norms_kernel(const DevProblem pr, const double* __restrict__ psi_new, const double* __restrict__ psi_old,
                 const double* __restrict__ phi_old, double* __restrict__ phi_new, double* __restrict__ part) {
    const int64_t N = (int64_t)pr.nel * pr.nb;
    double mx = 0.0, num = 0.0, den = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < N; i += (int64_t)gridDim.x * kRedThreads) {
        double ph = 0.0;
        for (int d = 0; d < pr.nd; ++d) {
            const double a = psi_new[(size_t)d * N + i];
            ph = fma(pr.weight[d], a, ph);   // explicit: hsw_shard_phi_partial chains the same FMAs
            mx = fmax(mx, fabs(a - psi_old[(size_t)d * N + i]));
        }
        phi_new[i] = ph;
        const double df = ph - phi_old[i];
        num = fma(df, df, num);
        den = fma(ph, ph, den);
    }
    __shared__ double s0[kRedThreads], s1[kRedThreads], s2[kRedThreads];
    s0[threadIdx.x] = mx; s1[threadIdx.x] = num; s2[threadIdx.x] = den;
    __syncthreads();
    for (int off = kRedThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s0[threadIdx.x] = fmax(s0[threadIdx.x], s0[threadIdx.x + off]);
            s1[threadIdx.x] += s1[threadIdx.x + off];
            s2[threadIdx.x] += s2[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = s0[0];
        part[gridDim.x + blockIdx.x] = s1[0];
        part[2 * gridDim.x + blockIdx.x] = s2[0];
    }
}

// out = {max part0, sum part1, part2 summed (max2: maxed)}
__global__ void __launch_bounds__(kRedThreads) finish3_kernel(const double* __restrict__ part, int nblk, double* out,
                                                              int max2 = 0) {
    __shared__ double s0[kRedThreads], s1[kRedThreads], s2[kRedThreads];
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < nblk; i += kRedThreads) {
        a = fmax(a, part[i]);
        b += part[nblk + i];
        c = max2 ? fmax(c, part[2 * nblk + i]) : c + part[2 * nblk + i];
    }
    s0[threadIdx.x] = a; s1[threadIdx.x] = b; s2[threadIdx.x] = c;
    __syncthreads();
    for (int off = kRedThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s0[threadIdx.x] = fmax(s0[threadIdx.x], s0[threadIdx.x + off]);
            s1[threadIdx.x] += s1[threadIdx.x + off];
            s2[threadIdx.x] = max2 ? fmax(s2[threadIdx.x], s2[threadIdx.x + off]) : s2[threadIdx.x] + s2[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) { out[0] = s0[0]; out[1] = s1[0]; out[2] = s2[0]; }
}

void dev_phi_and_norms(const DevProblem& P, const double* psi_new, const double* psi_old, const double* phi_old,
                       double* phi_new, double* scratch, double* out3, void* stream) {
    const int64_t N = (int64_t)P.nel * P.nb;
    const int nblk = (int)std::min<int64_t>(kRedBlocks, (N + kRedThreads - 1) / kRedThreads);
    cudaStream_t st = (cudaStream_t)stream;
    phi_norms_kernel<<<nblk, kRedThreads, 0, st>>>(P, psi_new, psi_old, phi_old, phi_new, scratch);
    KCHECK(cudaGetLastError());
    finish3_kernel<<<1, kRedThreads, 0, st>>>(scratch, nblk, out3);
    KCHECK(cudaGetLastError());
}

__global__ void __launch_bounds__(kRedThreads)
maxdiff_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* part) {
    double mx = 0.0, ma = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedThreads) {
        mx = fmax(mx, fabs(a[i] - b[i]));
        ma = fmax(ma, fabs(a[i]));
    }
    __shared__ double s0[kRedThreads], s2[kRedThreads];
    s0[threadIdx.x] = mx;
    s2[threadIdx.x] = ma;
    __syncthreads();
    for (int off = kRedThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s0[threadIdx.x] = fmax(s0[threadIdx.x], s0[threadIdx.x + off]);
            s2[threadIdx.x] = fmax(s2[threadIdx.x], s2[threadIdx.x + off]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = s0[0];
        part[gridDim.x + blockIdx.x] = 0.0;
        part[2 * gridDim.x + blockIdx.x] = s2[0];
    }
}

// ------------------------------------------------ FP64 peak microbenchmark
// 8 independent DFMA chains per thread, all SMs busy: the measured FP64
// roofline denominator (the sweep's FLOPs are FP64 FMAs on the CUDA cores).
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double s) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double m = 0.999999999;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(a0, m, s); a1 = fma(a1, m, s); a2 = fma(a2, m, s); a3 = fma(a3, m, s);
            a4 = fma(a4, m, s); a5 = fma(a5, m, s); a6 = fma(a6, m, s); a7 = fma(a7, m, s);
        }
    }
    const double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 12345.678) out[0] = r;  // keep the chains alive
}

// FP64 tensor-core (DMMA m8n8k4) throughput: 8 independent accumulator tiles per warp
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = threadIdx.x * 1e-9 + i; c[i][1] = 0.0; }
    const double a = 1e-3 + threadIdx.x * 1e-12, b = 0.999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += c[i][0] + c[i][1];
    if (r == 12345.678) out[0] = r;
}

double dev_dmma_peak_tflops(int device) {
    KCHECK(cudaSetDevice(device));
    int sms = 0;
    KCHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* out = nullptr;
    KCHECK(cudaMalloc(&out, sizeof(double)));
    const int blocks = sms * 8, threads = 256, iters = 2048;
    dmma_peak_kernel<<<blocks, threads>>>(out, 16);
    KCHECK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    KCHECK(cudaEventCreate(&e0));
    KCHECK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        KCHECK(cudaEventRecord(e0));
        dmma_peak_kernel<<<blocks, threads>>>(out, iters);
        KCHECK(cudaEventRecord(e1));
        KCHECK(cudaEventSynchronize(e1));
        float ms = 0.f;
        KCHECK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    // 8 DMMA (8x8x4 = 256 FMA = 512 FLOP) per warp per iteration
    const double flops = 512.0 * 8.0 * (double)iters * (double)blocks * (threads / 32);
    return flops / (best * 1e-3) * 1e-12;
}

double dev_fp64_peak_tflops(int device) {
    KCHECK(cudaSetDevice(device));
    int sms = 0;
    KCHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* out = nullptr;
    KCHECK(cudaMalloc(&out, sizeof(double)));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    fp64_peak_kernel<<<blocks, threads>>>(out, 16, 1e-3);  // warm-up
    KCHECK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    KCHECK(cudaEventCreate(&e0));
    KCHECK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        KCHECK(cudaEventRecord(e0));
        fp64_peak_kernel<<<blocks, threads>>>(out, iters, 1e-3);
        KCHECK(cudaEventRecord(e1));
        KCHECK(cudaEventSynchronize(e1));
        float ms = 0.f;
        KCHECK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * 8.0 * 16.0 * (double)iters * (double)blocks * threads;
    return flops / (best * 1e-3) * 1e-12;
}

// ----------------------------------------------- direction-sharded SI (§8e)
// out = prefix + sum_{d0 <= d < d1} w_d psi_new_d with the FMA chain of
// phi_norms_kernel: chaining the blocks of all ranks in order gives its bits.
__global__ void phi_partial_kernel(const DevProblem pr, const double* __restrict__ psi_new, int d0, int d1,
                                   const double* __restrict__ prefix, double* __restrict__ out) {
    const int64_t N = (int64_t)pr.nel * pr.nb;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        double ph = prefix ? prefix[i] : 0.0;
        for (int d = d0; d < d1; ++d) ph = fma(pr.weight[d], psi_new[(size_t)d * N + i], ph);
        out[i] = ph;
    }
}

void dev_phi_partial(const DevProblem& P, const double* psi_new, int d0, int d1, const double* prefix, double* out,
                     void* stream) {
    const int64_t N = (int64_t)P.nel * P.nb;
    const int nblk = (int)std::min<int64_t>(4096, (N + 255) / 256);
    phi_partial_kernel<<<nblk, 256, 0, (cudaStream_t)stream>>>(P, psi_new, d0, d1, prefix, out);
    KCHECK(cudaGetLastError());
}

// sum (phi_new - phi_old)^2 and sum phi_new^2 with phi_norms_kernel's exact tree
__global__ void __launch_bounds__(kRedThreads)
phi_norms2_kernel(int64_t N, const double* __restrict__ phi_new, const double* __restrict__ phi_old,
                  double* __restrict__ part) {
    double num = 0.0, den = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < N; i += (int64_t)gridDim.x * kRedThreads) {
        const double ph = phi_new[i];
        const double df = ph - phi_old[i];
        num = fma(df, df, num);
        den = fma(ph, ph, den);
    }
    __shared__ double s1[kRedThreads], s2[kRedThreads];
    s1[threadIdx.x] = num; s2[threadIdx.x] = den;
    __syncthreads();
    for (int off = kRedThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s1[threadIdx.x] += s1[threadIdx.x + off];
            s2[threadIdx.x] += s2[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = 0.0;
        part[gridDim.x + blockIdx.x] = s1[0];
        part[2 * gridDim.x + blockIdx.x] = s2[0];
    }
}

void dev_phi_norms2(const DevProblem& P, const double* phi_new, const double* phi_old, double* scratch, double* out3,
                    void* stream) {
    const int64_t N = (int64_t)P.nel * P.nb;
    const int nblk = (int)std::min<int64_t>(kRedBlocks, (N + kRedThreads - 1) / kRedThreads);
    cudaStream_t st = (cudaStream_t)stream;
    phi_norms2_kernel<<<nblk, kRedThreads, 0, st>>>(N, phi_new, phi_old, scratch);
    KCHECK(cudaGetLastError());
    finish3_kernel<<<1, kRedThreads, 0, st>>>(scratch, nblk, out3);
    KCHECK(cudaGetLastError());
}

void dev_max_abs_diff(const double* a, const double* b, int64_t n, double* scratch, double* out, void* stream) {
    const int nblk = (int)std::min<int64_t>(kRedBlocks, (n + kRedThreads - 1) / kRedThreads);
    cudaStream_t st = (cudaStream_t)stream;
    maxdiff_kernel<<<nblk, kRedThreads, 0, st>>>(a, b, n, scratch);
    KCHECK(cudaGetLastError());
    finish3_kernel<<<1, kRedThreads, 0, st>>>(scratch, nblk, out, 1);
    KCHECK(cudaGetLastError());
}

// ConvergenceHistory::per_ordinate (solver.hpp:36,150-156): out[d] =
// ||psi_new_d - psi_old_d||_inf for every ordinate.  max is order-independent, so
// the bit patterns of the non-negative maxima are combined with an integer
// atomicMax (exact, deterministic); out must be zeroed first.
__global__ void __launch_bounds__(kRedThreads)
per_ordinate_maxdiff_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n, int chunks,
                            unsigned long long* out) {
    const int d = blockIdx.x / chunks, c = blockIdx.x % chunks;
    const double* ad = a + (size_t)d * n;
    const double* bd = b + (size_t)d * n;
    double mx = 0.0;
    for (int64_t i = (int64_t)c * kRedThreads + threadIdx.x; i < n; i += (int64_t)chunks * kRedThreads)
        mx = fmax(mx, fabs(ad[i] - bd[i]));
    for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out + d, (unsigned long long)__double_as_longlong(mx));
}

void dev_per_ordinate_maxdiff(const double* a, const double* b, int nd, int64_t n, double* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    KCHECK(cudaMemsetAsync(out, 0, (size_t)nd * sizeof(double), st));
    const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(64, (n + kRedThreads - 1) / kRedThreads));
    per_ordinate_maxdiff_kernel<<<nd * chunks, kRedThreads, 0, st>>>(a, b, n, chunks,
                                                                   reinterpret_cast<unsigned long long*>(out));
    KCHECK(cudaGetLastError());
}

}  // namespace hsw
