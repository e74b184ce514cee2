// Checks the mma.m8n8k4 f64 fragment layout assumed by hsw_dmma.cu:
// A[g][q], B[q][g], C[g][2q+s] with g = lane>>2, q = lane&3.
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* C) {
    int l = threadIdx.x, g = l >> 2, q = l & 3;
    double a = A[g * 4 + q], b = B[q * 8 + g];
    double c0 = 0, c1 = 0;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    C[g * 8 + 2 * q] = c0; C[g * 8 + 2 * q + 1] = c1;
}
int main() {
    double hA[32], hB[32], hC[64], ref[64];
    for (int i = 0; i < 32; ++i) { hA[i] = i + 1; hB[i] = 0.5 * i - 3; }
    for (int m = 0; m < 8; ++m) for (int n = 0; n < 8; ++n) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[m * 4 + k] * hB[k * 8 + n]; ref[m * 8 + n] = s; }
    double *dA, *dB, *dC; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC); cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
    double err = 0; for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hC[i] - ref[i]));
    printf("dmma layout max err %g (%s)\n", err, err < 1e-12 ? "OK" : "MISMATCH");
    return err < 1e-12 ? 0 : 1;
}
