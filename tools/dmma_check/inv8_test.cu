// Unit check of the kernel's fraction-free 8x8 tile inversion (copied at build time from hsw_dmma1.cu).
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ void inv8_tile(double& d0, double& d1, double sc, double rthr, bool& bad, int g, int q) {
    constexpr unsigned FULL = 0xffffffffu;
    d0 *= sc;
    d1 *= sc;
    double dg = 1.0, pp = 1.0;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int ql = s >> 1;
        const double dk = (s & 1) ? d1 : d0;            // column s of this row where q == ql
        const double rk0 = __shfl_sync(FULL, d0, 4 * s + q), rk1 = __shfl_sync(FULL, d1, 4 * s + q);
        const double f = __shfl_sync(FULL, dk, 4 * g + ql);
        const double pv = __shfl_sync(FULL, dk, 4 * s + ql);
        if (!(fabs(pv) > rthr * fabs(pp))) bad = true;
        const double s2 = __hiloint2double(0x7fe00000 - (__double2hiint(pv) & 0x7ff00000), 0);   // 2^-exponent(pv)
        const double pvn = pv * s2, fn = f * s2;
        const bool prow = g == s;
        double n0 = prow ? d0 : fma(-fn, rk0, pvn * d0);
        double n1 = prow ? d1 : fma(-fn, rk1, pvn * d1);
        const double ck = prow ? pp : -fn * pp;         // column s of the inverse (unnormalised)
        if (s & 1) n1 = q == ql ? ck : n1;
        else n0 = q == ql ? ck : n0;
        d0 = n0;
        d1 = n1;
        dg = prow ? pv : dg * pvn;
        pp *= pvn;
    }
    double rinv;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rinv) : "d"(dg));
    {
        double er = fma(-dg, rinv, 1.0);
        rinv = fma(rinv, er, rinv);
        er = fma(-dg, rinv, 1.0);
        rinv = fma(rinv, er, rinv);
    }
    rinv *= sc;
    d0 *= rinv;
    d1 *= rinv;
}

__global__ void k(const double* A, double* X, int* badf, double amax_in) {
    const int lane = threadIdx.x, g = lane >> 2, q = lane & 3;
    const double* a = A + blockIdx.x * 64;
    double d0 = a[g * 8 + 2 * q], d1 = a[g * 8 + 2 * q + 1];
    double amax = amax_in;
    const int iex = ilogb(amax);
    const double isc = scalbn(1.0, -iex);
    bool bad = false;
    inv8_tile(d0, d1, isc, 1e-14 * (amax * isc), bad, g, q);
    X[blockIdx.x * 64 + g * 8 + 2 * q] = d0;
    X[blockIdx.x * 64 + g * 8 + 2 * q + 1] = d1;
    if (bad) badf[blockIdx.x] = 1;
}
int main() {
    const int nt = 1000;
    double* hA = new double[nt * 64]; double* hX = new double[nt * 64]; int* hb = new int[nt];
    srand(1);
    const double scale = 3e-7;
    for (int t = 0; t < nt; ++t)
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) hA[t * 64 + i * 8 + j] = scale * ((rand() / (double)RAND_MAX - 0.5) * (t % 3 == 0 ? 0.02 : 1.0) + (i == j ? ((t & 1) ? -1.5 : 1.5) * (t % 5 == 0 ? 0.05 : 1.0) : 0.0));
    double *dA, *dX; int* db;
    cudaMalloc(&dA, nt * 64 * 8); cudaMalloc(&dX, nt * 64 * 8); cudaMalloc(&db, nt * 4); cudaMemset(db, 0, nt * 4);
    cudaMemcpy(dA, hA, nt * 64 * 8, cudaMemcpyHostToDevice);
    k<<<nt, 32>>>(dA, dX, db, 5.0 * scale);
    cudaMemcpy(hX, dX, nt * 64 * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hb, db, nt * 4, cudaMemcpyDeviceToHost);
    double worst = 0; int nbad = 0;
    for (int t = 0; t < nt; ++t) {
        nbad += hb[t];
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) {
                double s = 0; for (int k2 = 0; k2 < 8; ++k2) s += hX[t * 64 + i * 8 + k2] * hA[t * 64 + k2 * 8 + j];
                worst = fmax(worst, fabs(s - (i == j)));
            }
    }
    printf("inv8_tile: max |X A - I| = %.3e over %d tiles, flagged bad: %d\n", worst, nt, nbad);
    return 0;
}
