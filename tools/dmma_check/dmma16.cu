// Checks the m16n8k4 f64 fragment layout assumed by the sweep kernel against a CPU product.
// a0 = A[g][q], a1 = A[g+8][q]; b0 = B[q][g]; c0,c1 = C[g][2q,2q+1], c2,c3 = C[g+8][2q,2q+1].
#include <cstdio>
__global__ void k(const double* A, const double* B, double* C) {
    const int lane = threadIdx.x, g = lane >> 2, q = lane & 3;
    double a0 = A[g * 4 + q], a1 = A[(g + 8) * 4 + q];
    double b0 = B[q * 8 + g];
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b0));
    C[g * 8 + 2 * q] = c0; C[g * 8 + 2 * q + 1] = c1; C[(g + 8) * 8 + 2 * q] = c2; C[(g + 8) * 8 + 2 * q + 1] = c3;
}
int main() {
    double hA[64], hB[32], hC[128], ref[128];
    for (int i = 0; i < 64; ++i) hA[i] = 1.0 + i * 0.37;
    for (int i = 0; i < 32; ++i) hB[i] = 2.0 - i * 0.11;
    for (int r = 0; r < 16; ++r) for (int c = 0; c < 8; ++c) { double s = 0; for (int k2 = 0; k2 < 4; ++k2) s += hA[r * 4 + k2] * hB[k2 * 8 + c]; ref[r * 8 + c] = s; }
    double *A, *B, *C; cudaMalloc(&A, 512); cudaMalloc(&B, 256); cudaMalloc(&C, 1024);
    cudaMemcpy(A, hA, 512, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(A, B, C); cudaMemcpy(hC, C, 1024, cudaMemcpyDeviceToHost);
    double err = 0; for (int i = 0; i < 128; ++i) { double d = hC[i] - ref[i]; err = d * d > err ? d * d : err; }
    printf("m16n8k4 f64 layout max sq err %g (%s)\n", err, err < 1e-20 ? "OK" : "MISMATCH");
    return 0;
}
