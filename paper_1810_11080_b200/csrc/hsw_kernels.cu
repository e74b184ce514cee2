// CUDA kernels of the B200 transport sweep (sm_100a).
//
//   K1 sweep_pairs_kernel   SweepSolver::sweep (solver.hpp:98-117) for one level of the
//                           (element, ordinate) worklist: assemble
//                           A = sum_k Omega_k G_k + F_out + sigma_t M   (assembly.hpp:393)
//                           and rhs = s_e + upwind traces (retained: psi_new,
//                           lagged: psi_old), then dense FP64 LU with partial pivoting
//                           (solver.hpp:69,114) and the two triangular solves.
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

__constant__ int c_fnode[kMaxFaces][kMaxFaceNodes];
__constant__ double c_trace[kMaxFacePoints][kMaxFaceNodes];

#define KCHECK(x)                                                                              \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess)                                                                 \
            throw Error(-8, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x);       \
    } while (0)

void dev_upload_tables(const ConstTables& t) {
    KCHECK(cudaMemcpyToSymbol(c_fnode, t.fnode, sizeof(t.fnode)));
    KCHECK(cudaMemcpyToSymbol(c_trace, t.trace, sizeof(t.trace)));
}

template <int DIM, int P>
struct Shape {
    static constexpr int N1 = P + 1;
    static constexpr int NB = DIM == 2 ? N1 * N1 : N1 * N1 * N1;
    static constexpr int NFN = DIM == 2 ? N1 : N1 * N1;
    static constexpr int NF = 2 * DIM;
    static constexpr int LD = NB + 1;  // augmented column NB holds the rhs
    static constexpr int NT = NB <= 16 ? 64 : (NB <= 32 ? 128 : (NB <= 64 ? 256 : 512));
};

__device__ __forceinline__ void orient_index_dev(int dim, int code, int r, int a, int b, int& ao, int& bo) {
    if (dim == 2) { ao = code ? r - a : a; bo = 0; return; }
    int u = a, v = b;
    if (code & 4) { u = b; v = a; }
    if (code & 2) u = r - u;
    if (code & 1) v = r - v;
    ao = u; bo = v;
}

template <int NT>
__device__ __forceinline__ double block_max(double v, double* red) {
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < NT / 32; ++w) r = fmax(r, red[w]);
    return r;
}

// Assemble the local system of pair (e, d) into A (NB x LD, shared) and run
// the partial-pivot LU + solves.  mode 0: sweep (rhs = src + upwind traces);
// mode 1: local solve (rhs given, no inflow terms).
template <int DIM, int P>
__device__ void solve_pair(const DevProblem& pr, int e, int d, const double* __restrict__ src,
                           const double* __restrict__ psi_old, const double* __restrict__ psi_new_in,
                           double* __restrict__ out, int64_t psi_stride, const double* __restrict__ rhs_given,
                           unsigned long long* err_key, int64_t zero_pair, double* sm) {
    using S = Shape<DIM, P>;
    constexpr int NB = S::NB, LD = S::LD, NFN = S::NFN, NF = S::NF, NT = S::NT, N1 = S::N1;
    double* A = sm;
    double* wq = A + NB * LD;
    double* wi = wq + kMaxFacePoints;
    double* tr = wi + kMaxFacePoints;
    double* up = tr + kMaxFacePoints;
    double* red = up + kMaxFaceNodes;
    __shared__ int s_piv;
    const int tid = threadIdx.x;
    const int nqf = pr.nqf;
    const double om0 = pr.omega[d * 4 + 0], om1 = pr.omega[d * 4 + 1], om2 = pr.omega[d * 4 + 2];
    const double st = pr.sig_t[e];
    const int64_t pair = (int64_t)e * pr.nd + d;

    // ---- volume: A = Omega . G + sigma_t M (T[e][m][n] = {M, Gx, Gy, Gz})
    const double4* Te = reinterpret_cast<const double4*>(pr.T) + (size_t)e * NB * NB;
    for (int idx = tid; idx < NB * NB; idx += NT) {
        const int m = idx / NB, n = idx - (idx / NB) * NB;
        const double4 t = Te[(size_t)n * NB + m];  // column-major T
        double g = om0 * t.y + om1 * t.z;
        if (DIM == 3) g += om2 * t.w;
        A[m * LD + n] = g + st * t.x;
    }
    for (int m = tid; m < NB; m += NT) A[m * LD + NB] = rhs_given ? rhs_given[m] : src[(size_t)e * NB + m];
    __syncthreads();

    // ---- faces: outflow block (own normal, w+) and upwind inflow (w-)
    const unsigned flags = rhs_given ? 0u : pr.inflags[(size_t)d * pr.nel + e];
    for (int f = 0; f < NF; ++f) {
        const double* geo = pr.fgeom + (((size_t)e * NF + f) * nqf) * 4;
        const int* nb4 = pr.fnbr + ((size_t)e * NF + f) * 4;
        const int nbr = nb4[0];
        const bool incoming = (flags >> (2 * f)) & 1u;
        const bool lag = (flags >> (2 * f + 1)) & 1u;
        const bool inflow_bc = !rhs_given && nbr < 0 && pr.inflow != 0.0;
        int any_out = 0;
        for (int q = tid; q < nqf; q += NT) {
            const double4 g = reinterpret_cast<const double4*>(geo)[q];
            double on = om0 * g.x + om1 * g.y;
            if (DIM == 3) on += om2 * g.z;
            const double wp = on > 0.0 ? on * g.w : 0.0;
            wq[q] = wp;
            wi[q] = on < 0.0 ? -on * g.w : 0.0;
            any_out |= wp != 0.0;
        }
        if (incoming) {
            const double* srcpsi = (lag ? psi_old : psi_new_in) + (size_t)d * psi_stride + (size_t)nbr * NB;
            const int nface = nb4[1], code = nb4[2];
            for (int a = tid; a < NFN; a += NT) {
                int ao, bo;
                orient_index_dev(DIM, code, P, a % N1, a / N1, ao, bo);
                up[a] = srcpsi[c_fnode[nface][bo * N1 + ao]];
            }
        }
        any_out = __syncthreads_or(any_out);
        if (incoming || inflow_bc) {
            for (int q = tid; q < nqf; q += NT) {
                double t;
                if (incoming) {
                    t = 0.0;
                    for (int a = 0; a < NFN; ++a) t += c_trace[q][a] * up[a];
                } else {
                    t = pr.inflow;
                }
                tr[q] = t * wi[q];
            }
        }
        __syncthreads();
        if (any_out) {
            for (int idx = tid; idx < NFN * NFN; idx += NT) {
                const int a = idx / NFN, b = idx - (idx / NFN) * NFN;
                double s = 0.0;
                for (int q = 0; q < nqf; ++q) s += wq[q] * c_trace[q][a] * c_trace[q][b];
                A[c_fnode[f][a] * LD + c_fnode[f][b]] += s;
            }
        }
        if (incoming || inflow_bc) {
            for (int a = tid; a < NFN; a += NT) {
                double s = 0.0;
                for (int q = 0; q < nqf; ++q) s += tr[q] * c_trace[q][a];
                A[c_fnode[f][a] * LD + NB] += s;
            }
        }
        __syncthreads();
    }
    if (pair == zero_pair) {
        for (int idx = tid; idx < NB * NB; idx += NT) A[(idx / NB) * LD + idx % NB] = 0.0;
        __syncthreads();
    }
    // scale for the singularity test (pivot-based stand-in for rcond > 1e-14, solver.hpp:70)
    double amax = 0.0;
    for (int idx = tid; idx < NB * NB; idx += NT) amax = fmax(amax, fabs(A[(idx / NB) * LD + idx % NB]));
    amax = block_max<NT>(amax, red);

    // ---- LU with partial pivoting on [A | rhs]
    bool singular = false;
    for (int k = 0; k < NB; ++k) {
        if (tid < 32) {
            double best = -1.0;
            int bi = k;
            for (int i = k + tid; i < NB; i += 32) {
                const double v = fabs(A[i * LD + k]);
                if (v > best) { best = v; bi = i; }
            }
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, best, off);
                const int oi = __shfl_down_sync(0xffffffffu, bi, off);
                if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
            }
            if (tid == 0) s_piv = bi;
        }
        __syncthreads();
        const int p = s_piv;
        if (p != k)
            for (int j = k + tid; j <= NB; j += NT) {
                const double t = A[k * LD + j];
                A[k * LD + j] = A[p * LD + j];
                A[p * LD + j] = t;
            }
        __syncthreads();
        const double piv = A[k * LD + k];
        if (!(fabs(piv) > 1e-14 * amax)) singular = true;
        const double inv = 1.0 / piv;
        const int w = NB - k;  // columns k+1..NB
        for (int idx = tid; idx < (NB - 1 - k) * w; idx += NT) {
            const int i = k + 1 + idx / w, j = k + 1 + idx % w;
            A[i * LD + j] -= (A[i * LD + k] * inv) * A[k * LD + j];
        }
        __syncthreads();
    }
    for (int k = NB - 1; k >= 0; --k) {
        if (tid == 0) A[k * LD + NB] = A[k * LD + NB] / A[k * LD + k];
        __syncthreads();
        const double xk = A[k * LD + NB];
        for (int i = tid; i < k; i += NT) A[i * LD + NB] -= A[i * LD + k] * xk;
        __syncthreads();
    }
    if (singular && tid == 0) atomicMin(err_key, (unsigned long long)pair);
    for (int m = tid; m < NB; m += NT) out[m] = A[m * LD + NB];
}

template <int DIM, int P>
__global__ void __launch_bounds__(Shape<DIM, P>::NT)
sweep_pairs_kernel(const DevProblem pr, const double* __restrict__ src, const double* __restrict__ psi_old,
                   double* psi_new, const int* __restrict__ pairs, unsigned long long* err_key,
                   int64_t zero_pair) {
    extern __shared__ double sm[];
    const int pair = pairs[blockIdx.x];
    const int e = pair / pr.nd, d = pair - (pair / pr.nd) * pr.nd;
    const int64_t stride = (int64_t)pr.nel * Shape<DIM, P>::NB;
    double* out = psi_new + (size_t)d * stride + (size_t)e * Shape<DIM, P>::NB;
    solve_pair<DIM, P>(pr, e, d, src, psi_old, psi_new, out, stride, nullptr, err_key, zero_pair, sm);
}

template <int DIM, int P>
__global__ void __launch_bounds__(Shape<DIM, P>::NT)
local_solve_kernel(const DevProblem pr, int e, int d, const double* rhs, double* out,
                   unsigned long long* err_key, int64_t zero_pair) {
    extern __shared__ double sm[];
    solve_pair<DIM, P>(pr, e, d, nullptr, nullptr, nullptr, out, 0, rhs, err_key, zero_pair, sm);
}

template <int DIM, int P>
static size_t smem_bytes() {
    using S = Shape<DIM, P>;
    return (size_t)(S::NB * S::LD + 3 * kMaxFacePoints + kMaxFaceNodes + 32) * sizeof(double);
}

template <int DIM, int P>
static void launch_sweep(const DevProblem& pr, const double* src, const double* psi_old, double* psi_new,
                         const int* pairs, int npairs, unsigned long long* err, int64_t zero_pair,
                         cudaStream_t st) {
    const size_t sm = smem_bytes<DIM, P>();
    static bool configured = false;
    if (!configured) {
        KCHECK(cudaFuncSetAttribute(sweep_pairs_kernel<DIM, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        KCHECK(cudaFuncSetAttribute(local_solve_kernel<DIM, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        configured = true;
    }
    sweep_pairs_kernel<DIM, P><<<npairs, Shape<DIM, P>::NT, sm, st>>>(pr, src, psi_old, psi_new, pairs, err, zero_pair);
    KCHECK(cudaGetLastError());
}

template <int DIM, int P>
static void launch_local(const DevProblem& pr, int e, int d, const double* rhs, double* out,
                         unsigned long long* err, int64_t zero_pair, cudaStream_t st) {
    const size_t sm = smem_bytes<DIM, P>();
    KCHECK(cudaFuncSetAttribute(local_solve_kernel<DIM, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    local_solve_kernel<DIM, P><<<1, Shape<DIM, P>::NT, sm, st>>>(pr, e, d, rhs, out, err, zero_pair);
    KCHECK(cudaGetLastError());
}

#define HSW_DISPATCH(DIMV, PV, CALL)                                                  \
    do {                                                                              \
        if (DIMV == 2) {                                                              \
            switch (PV) {                                                             \
                case 1: CALL(2, 1); break;                                            \
                case 2: CALL(2, 2); break;                                            \
                case 3: CALL(2, 3); break;                                            \
                case 4: CALL(2, 4); break;                                            \
                case 5: CALL(2, 5); break;                                            \
                case 6: CALL(2, 6); break;                                            \
                default: throw Error(-1, "unsupported 2D order");                    \
            }                                                                         \
        } else {                                                                      \
            switch (PV) {                                                             \
                case 1: CALL(3, 1); break;                                            \
                case 2: CALL(3, 2); break;                                            \
                case 3: CALL(3, 3); break;                                            \
                case 4: CALL(3, 4); break;                                            \
                default: throw Error(-1, "unsupported 3D order");                    \
            }                                                                         \
        }                                                                             \
    } while (0)

void dev_sweep_pairs(const DevProblem& P, const double* src, const double* psi_old, double* psi_new,
                     const int* pairs, int npairs, unsigned long long* err_key, int64_t zero_pair,
                     void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
#define CALL_SWEEP(D_, P_) launch_sweep<D_, P_>(P, src, psi_old, psi_new, pairs, npairs, err_key, zero_pair, st)
    HSW_DISPATCH(P.dim, P.p, CALL_SWEEP);
#undef CALL_SWEEP
}

void dev_local_solve(const DevProblem& P, int e, int d, const double* rhs, double* out,
                     unsigned long long* err_key, int64_t zero_pair, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
#define CALL_LOCAL(D_, P_) launch_local<D_, P_>(P, e, d, rhs, out, err_key, zero_pair, st)
    HSW_DISPATCH(P.dim, P.p, CALL_LOCAL);
#undef CALL_LOCAL
}

int dev_max_dynamic_smem_needed(int dim, int p) {
    size_t r = 0;
#define CALL_SM(D_, P_) r = smem_bytes<D_, P_>()
    HSW_DISPATCH(dim, p, CALL_SM);
#undef CALL_SM
    return (int)r;
}

// ------------------------------------------------------------ scatter source
__global__ void scatter_source_kernel(const DevProblem pr, const double* __restrict__ phi, double* __restrict__ src) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int nb = pr.nb;
    if (i >= (int64_t)pr.nel * nb) return;
    const int e = (int)(i / nb), m = (int)(i - (i / nb) * nb);
    const double* Tm = pr.T + ((size_t)e * nb * nb + (size_t)m) * 4;  // entry (m, n) at (n*nb + m)
    const double* ph = phi + (size_t)e * nb;
    double s = 0.0;
    for (int n = 0; n < nb; ++n) s += Tm[(size_t)n * nb * 4] * ph[n];
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

__global__ void __launch_bounds__(kRedThreads) finish3_kernel(const double* __restrict__ part, int nblk, double* out) {
    __shared__ double s0[kRedThreads], s1[kRedThreads], s2[kRedThreads];
    double a = 0.0, b = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < nblk; i += kRedThreads) {
        a = fmax(a, part[i]);
        b += part[nblk + i];
        c += part[2 * nblk + i];
    }
    s0[threadIdx.x] = a; s1[threadIdx.x] = b; s2[threadIdx.x] = c;
    __syncthreads();
    for (int off = kRedThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s0[threadIdx.x] = fmax(s0[threadIdx.x], s0[threadIdx.x + off]);
            s1[threadIdx.x] += s1[threadIdx.x + off];
            s2[threadIdx.x] += s2[threadIdx.x + off];
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
    double mx = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kRedThreads)
        mx = fmax(mx, fabs(a[i] - b[i]));
    __shared__ double s0[kRedThreads];
    s0[threadIdx.x] = mx;
    __syncthreads();
    for (int off = kRedThreads / 2; off > 0; off >>= 1) {
        if (threadIdx.x < off) s0[threadIdx.x] = fmax(s0[threadIdx.x], s0[threadIdx.x + off]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = s0[0];
        part[gridDim.x + blockIdx.x] = 0.0;
        part[2 * gridDim.x + blockIdx.x] = 0.0;
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
    finish3_kernel<<<1, kRedThreads, 0, st>>>(scratch, nblk, out);
    KCHECK(cudaGetLastError());
}

}  // namespace hsw
