// Device-side setup: per-element tensors T = [M, G_x, G_y, G_z] and volume
// source moments, computed where they are used instead of on the host and
// uploaded (C4: 4.3 GB of T, ~8 s of host time on 8 cores -> milliseconds).
//
// Replaces the direction-independent half of assemble_volume / assemble_source
// (assembly.hpp:143-163, 292-300) hoisted out of the ordinate loop
// (SURVEY §8a A4-A7):
//   M[m][n]   =  sum_q w_q det_q u_m(x_q) u_n(x_q)
//   G_k[m][n] = -sum_q w_q det_q (d_k u_m)(x_q) u_n(x_q),  grad = J^{-T} grad_ref
//   qvol[m]   =  sum_q w_q det_q q(x_q) u_m(x_q)
// Layout: T[e][n][m][k] (column-major per element, k = 0..3) as hsw_host.cpp's
// host path; tolerance-level (not bit-level) agreement with it: T feeds only
// the FP64 solves, never an integer decision.
#include "hsw_internal.hpp"

#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace hsw {

#define SCHECK(x)                                                                              \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess)                                                                 \
            throw Error(-8, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x);       \
    } while (0)

namespace {

constexpr int kSetupThreads = 256;
constexpr int kMaxQ = 216;   // (p + 2)^3 volume points, p <= 4

template <int DIM>
__global__ void __launch_bounds__(kSetupThreads)
element_tensor_kernel(int nel, int nb, int npe, int nq, const double* __restrict__ pts, const int* __restrict__ enodes,
                      const double* __restrict__ U, const double* __restrict__ DU, const double* __restrict__ GG,
                      const double* __restrict__ GV, const double* __restrict__ wq, int source_kind,
                      SourceParams sp, double* __restrict__ T, double* __restrict__ qvol,
                      unsigned long long* __restrict__ bad_elem) {
    __shared__ double sK[kMaxQ][DIM * DIM];   // J^{-1}
    __shared__ double sW[kMaxQ];              // w_q det_q
    __shared__ double sS[kMaxQ];              // w_q det_q q(x_q)
    const int e = blockIdx.x;
    const int* en = enodes + (size_t)e * npe;
    // 1. geometry at the volume points (mesh.hpp:157-170)
    for (int q = threadIdx.x; q < nq; q += kSetupThreads) {
        double J[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, x[3] = {0, 0, 0};
        const double* g = GG + (size_t)q * npe * DIM;
        const double* v = GV + (size_t)q * npe;
        for (int m = 0; m < npe; ++m) {
            const double* X = pts + (size_t)en[m] * DIM;
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
#pragma unroll
                for (int b = 0; b < DIM; ++b) J[a * 3 + b] += X[a] * g[m * DIM + b];
                x[a] += v[m] * X[a];
            }
        }
        double det, K[9];
        if (DIM == 2) {
            det = J[0] * J[4] - J[3] * J[1];
            const double id = 1.0 / det;
            K[0] = J[4] * id; K[3] = -J[3] * id; K[1] = -J[1] * id; K[4] = J[0] * id;
        } else {
            const double c00 = J[4] * J[8] - J[5] * J[7];
            const double c01 = J[5] * J[6] - J[3] * J[8];
            const double c02 = J[3] * J[7] - J[4] * J[6];
            det = J[0] * c00 + J[1] * c01 + J[2] * c02;
            const double id = 1.0 / det;
            K[0] = c00 * id; K[1] = (J[2] * J[7] - J[1] * J[8]) * id; K[2] = (J[1] * J[5] - J[2] * J[4]) * id;
            K[3] = c01 * id; K[4] = (J[0] * J[8] - J[2] * J[6]) * id; K[5] = (J[2] * J[3] - J[0] * J[5]) * id;
            K[6] = c02 * id; K[7] = (J[1] * J[6] - J[0] * J[7]) * id; K[8] = (J[0] * J[4] - J[1] * J[3]) * id;
        }
        if (!(det > 0.0) || !isfinite(det)) atomicMin(bad_elem, (unsigned long long)e);
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
            for (int b = 0; b < DIM; ++b) sK[q][a * DIM + b] = K[a * 3 + b];
        const double wd = wq[q] * det;
        sW[q] = wd;
        double src = sp.v[0];
        if (source_kind != 0) {   // disc / ball (assembly.hpp:298 at the quadrature point)
            double d2 = 0.0;
#pragma unroll
            for (int a = 0; a < DIM; ++a) d2 += (x[a] - sp.v[a]) * (x[a] - sp.v[a]);
            src = d2 < sp.v[3] * sp.v[3] ? sp.v[4] : sp.v[5];
        }
        sS[q] = wd * src;
    }
    __syncthreads();
    // 2. source moments
    for (int m = threadIdx.x; m < nb; m += kSetupThreads) {
        double s = 0.0;
        for (int q = 0; q < nq; ++q) s += sS[q] * U[(size_t)q * nb + m];
        qvol[(size_t)e * nb + m] = s;
    }
    // 3. T in 4 x 4 (m, n) blocks per thread, all DIM + 1 components
    const int nbb = (nb + 3) / 4;
    for (int blk = threadIdx.x; blk < nbb * nbb; blk += kSetupThreads) {
        const int m0 = 4 * (blk / nbb), n0 = 4 * (blk % nbb);
        double acc[4][4][DIM + 1];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int k = 0; k <= DIM; ++k) acc[i][j][k] = 0.0;
        for (int q = 0; q < nq; ++q) {
            const double wd = sW[q];
            double wm[4][DIM + 1], un[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int m = min(m0 + i, nb - 1);
                wm[i][0] = U[(size_t)q * nb + m] * wd;
                const double* du = DU + ((size_t)q * nb + m) * DIM;
#pragma unroll
                for (int k = 0; k < DIM; ++k) {
                    double v = 0.0;
#pragma unroll
                    for (int j = 0; j < DIM; ++j) v += sK[q][j * DIM + k] * du[j];
                    wm[i][k + 1] = v * wd;
                }
                un[i] = U[(size_t)q * nb + min(n0 + i, nb - 1)];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int k = 0; k <= DIM; ++k) acc[i][j][k] += wm[i][k] * un[j];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int m = m0 + i, n = n0 + j;
                if (m < nb && n < nb) {
                    T[t_idx(e, nb, m, n, 0)] = acc[i][j][0];
#pragma unroll
                    for (int k = 1; k <= DIM; ++k) T[t_idx(e, nb, m, n, k)] = -acc[i][j][k];
                    if (DIM == 2) T[t_idx(e, nb, m, n, 3)] = 0.0;
                }
            }
    }
}

// absorption = sum_e (sigma_t - sigma_s) 1^T M_e phi_e (balance_report, solver.hpp:220-245)
__global__ void __launch_bounds__(256)
absorption_kernel(int nel, int nb, const double* __restrict__ T, const double* __restrict__ sig_t,
                  const double* __restrict__ sig_s, const double* __restrict__ phi, double* __restrict__ part) {
    double s = 0.0;
    const int64_t total = (int64_t)nel * nb;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)(i / nb), n = (int)(i % nb);
        double cs = 0.0;   // column n of M: M[m][n], m = 0..nb-1
        for (int m = 0; m < nb; ++m) cs += T[t_idx(e, nb, m, n, 0)];
        s += (sig_t[e] - sig_s[e]) * cs * phi[i];
    }
    __shared__ double red[256];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// per element: max over the n x n entries of sig_t |M| + |Gx| + |Gy| + |Gz| (an
// ordinate-independent upper bound of max |sigma_t M + sum_k Omega_k G_k|, |Omega_k| <= 1)
__global__ void __launch_bounds__(kSetupThreads) block_scale_kernel(int nb, const double* __restrict__ T,
                                                                    const double* __restrict__ sig_t,
                                                                    double* __restrict__ out) {
    __shared__ double red[kSetupThreads];
    const int e = blockIdx.x;
    const double st = sig_t[e];
    double m = 0.0;
    for (int i = threadIdx.x; i < nb * nb; i += blockDim.x) {
        const int col = i / nb, row = i - (i / nb) * nb;
        m = fmax(m, st * fabs(T[t_idx(e, nb, row, col, 0)]) + fabs(T[t_idx(e, nb, row, col, 1)]) +
                        fabs(T[t_idx(e, nb, row, col, 2)]) + fabs(T[t_idx(e, nb, row, col, 3)]));
    }
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[e] = red[0];
}

}  // namespace

void dev_block_scale(int nel, int nb, const double* T, const double* sig_t, double* out, void* stream) {
    block_scale_kernel<<<nel, kSetupThreads, 0, (cudaStream_t)stream>>>(nb, T, sig_t, out);
    SCHECK(cudaGetLastError());
}

void dev_element_tensors(int dim, int nel, int nb, int npe, int nq, const double* pts, const int* enodes,
                         const double* U, const double* DU, const double* GG, const double* GV, const double* wq,
                         int source_kind, const SourceParams& sp, double* T, double* qvol,
                         unsigned long long* bad_elem, void* stream) {
    if (nq > kMaxQ) throw Error(-1, "dev_element_tensors: too many volume points");
    cudaStream_t st = (cudaStream_t)stream;
    if (dim == 2)
        element_tensor_kernel<2><<<nel, kSetupThreads, 0, st>>>(nel, nb, npe, nq, pts, enodes, U, DU, GG, GV, wq,
                                                                source_kind, sp, T, qvol, bad_elem);
    else
        element_tensor_kernel<3><<<nel, kSetupThreads, 0, st>>>(nel, nb, npe, nq, pts, enodes, U, DU, GG, GV, wq,
                                                                source_kind, sp, T, qvol, bad_elem);
    SCHECK(cudaGetLastError());
}

// balance_report's boundary terms on the device (solver.hpp:220-245): per boundary face,
// summed over the ordinates in ascending order, the outflow w_d 1^T B_d psi_d and the
// inflow w_d sum(source_boundary_d) — Gauss rule from the face tables (as the kernels
// assemble B), Romberg rule from the integrated blocks.  One thread per face: fixed order.
__global__ void __launch_bounds__(128)
balance_faces_kernel(const DevProblem pr, const double* __restrict__ psi, int nbf, const int* __restrict__ bfaces,
                     double* __restrict__ out) {
    const int bi = blockIdx.x * blockDim.x + threadIdx.x;
    if (bi >= nbf) return;
    const int e = bfaces[3 * bi], f = bfaces[3 * bi + 1];
    const int nfn = pr.nfn, nqf = pr.nqf, nb = pr.nb;
    const size_t N = (size_t)pr.nel * nb;
    double otot = 0.0, itot = 0.0;
    for (int d = 0; d < pr.nd; ++d) {
        const double* ps = psi + (size_t)d * N + (size_t)e * nb;
        double o = 0.0, in = 0.0;
        if (pr.rom_ob) {
            const size_t fb = ((size_t)d * pr.nel + e) * pr.nfaces + f;
            const double* blk = pr.rom_ob + fb * nfn * nfn;
            for (int m = 0; m < nfn; ++m) {
                double r = 0.0;
                for (int n = 0; n < nfn; ++n) r += blk[m * nfn + n] * ps[pr.g_fnode[f * kMaxFaceNodes + n]];
                o += r;
            }
            for (int m = 0; m < nfn; ++m) in += pr.rom_bin[fb * nfn + m];
        } else {
            const double* om = pr.omega + 4 * d;
            const double4* geo = reinterpret_cast<const double4*>(pr.fgeom) + ((size_t)e * pr.nfaces + f) * nqf;
            for (int q = 0; q < nqf; ++q) {
                const double4 gm = geo[q];
                double on = om[0] * gm.x + om[1] * gm.y;
                if (pr.dim == 3) on += om[2] * gm.z;
                const double wplus = 0.5 * (on + fabs(on)), wminus = 0.5 * (fabs(on) - on);
                double tr = 0.0, ts = 0.0;
                for (int a = 0; a < nfn; ++a) {
                    const double t = pr.g_trace[q * kMaxFaceNodes + a];
                    tr += t * ps[pr.g_fnode[f * kMaxFaceNodes + a]];
                    ts += t;
                }
                o += gm.w * wplus * tr * ts;
                in += gm.w * wminus * pr.inflow * ts;
            }
        }
        otot += pr.weight[d] * o;
        itot += pr.weight[d] * in;
    }
    out[2 * bi] = otot;
    out[2 * bi + 1] = itot;
}

void dev_balance_faces(const DevProblem& P, const double* psi, int nbf, const int* bfaces, double* out, void* stream) {
    if (nbf <= 0) return;
    balance_faces_kernel<<<(nbf + 127) / 128, 128, 0, (cudaStream_t)stream>>>(P, psi, nbf, bfaces, out);
    SCHECK(cudaGetLastError());
}

double dev_absorption(int nel, int nb, const double* T, const double* sig_t, const double* sig_s, const double* phi,
                      double* scratch, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int nblk = 1024;
    absorption_kernel<<<nblk, 256, 0, st>>>(nel, nb, T, sig_t, sig_s, phi, scratch);
    SCHECK(cudaGetLastError());
    std::vector<double> h(nblk);
    SCHECK(cudaMemcpyAsync(h.data(), scratch, nblk * sizeof(double), cudaMemcpyDeviceToHost, st));
    SCHECK(cudaStreamSynchronize(st));
    double s = 0.0;
    for (double v : h) s += v;
    return s;
}


// ---- per-(ordinate, interior face) coupling magnitudes
// max|LR| and max|RL| of the two coupling blocks of every interior face for a
// block of ordinates: the edge-existence test (> 1e-12 * length) and the `face`
// edge weight of sweepgraph.hpp:60-64.  Bit-identical to the host
// (hsw_host.cpp Setup::ordinates, itself the restatement of
// assembly.hpp:197-241): same inputs, ascending quadrature order, every
// product / sum rounded separately (__dmul_rn / __dadd_rn: no FMA contraction).
namespace {
constexpr int kCplThreads = 256;

__global__ void __launch_bounds__(kCplThreads)
coupling_max_kernel(int dim, int nfi, int nf, int nqf, int nfn, const int* __restrict__ iface /*[nfi][5]*/,
                    const double* __restrict__ fgeom, const double* __restrict__ fsj, const double* __restrict__ fqw,
                    const double* __restrict__ trace /*[nqf][nfn]*/, const double* __restrict__ traceR /*[code][nqf][nfn]*/,
                    const double* __restrict__ odir /*[nd][3]*/, int d0, int d1, double* __restrict__ out /*[d][nfi][2]*/) {
    __shared__ double s_geo[64 * 4], s_sj[64], s_wm[64], s_wp[64];
    __shared__ double s_red[2][kCplThreads / 32];
    const int fi = blockIdx.x;
    const int el = iface[fi * 5 + 0], fl = iface[fi * 5 + 2], orient = iface[fi * 5 + 4];
    for (int i = threadIdx.x; i < nqf * 4; i += kCplThreads) s_geo[i] = fgeom[((size_t)el * nf + fl) * nqf * 4 + i];
    for (int i = threadIdx.x; i < nqf; i += kCplThreads) s_sj[i] = fsj[((size_t)el * nf + fl) * nqf + i];
    const double* uR = traceR + (size_t)orient * nqf * nfn;
    for (int d = d0; d < d1; ++d) {
        __syncthreads();   // s_wm / s_wp reuse
        int any_p = 0, any_m = 0;
        for (int q = threadIdx.x; q < nqf; q += kCplThreads) {
            double on = 0.0;
            for (int k = 0; k < dim; ++k) on = __dadd_rn(on, __dmul_rn(odir[d * 3 + k], s_geo[q * 4 + k]));
            s_wp[q] = __dmul_rn(0.5, __dadd_rn(on, fabs(on)));
            s_wm[q] = __dmul_rn(0.5, __dadd_rn(fabs(on), -on));
            any_p |= s_wp[q] != 0.0;
            any_m |= s_wm[q] != 0.0;
        }
        // a face the ordinate crosses one way only has w- == 0 (or w+ == 0) at every point: that
        // block is a sum of zero products, |.| = 0 exactly, and is skipped (as the host does)
        const bool do_lr = __syncthreads_or(any_m) != 0;
        const bool do_rl = __syncthreads_or(any_p) != 0;
        double mlr = 0.0, mrl = 0.0;
        for (int mn = threadIdx.x; mn < nfn * nfn; mn += kCplThreads) {
            const int m = mn / nfn, n = mn - m * nfn;
            double lr = 0.0, rl = 0.0;
            // row[n] += w * (c * ur[n] * sj), c = w- * ul[m]   (and the mirrored RL term)
            if (do_lr)
                for (int q = 0; q < nqf; ++q) {
                    const double ul_m = trace[q * nfn + m], ur_n = uR[q * nfn + n];
                    lr = __dadd_rn(lr, __dmul_rn(fqw[q], __dmul_rn(__dmul_rn(__dmul_rn(s_wm[q], ul_m), ur_n), s_sj[q])));
                }
            if (do_rl)
                for (int q = 0; q < nqf; ++q) {
                    const double ur_m = uR[q * nfn + m], ul_n = trace[q * nfn + n];
                    rl = __dadd_rn(rl, __dmul_rn(fqw[q], __dmul_rn(__dmul_rn(__dmul_rn(s_wp[q], ur_m), ul_n), s_sj[q])));
                }
            mlr = fmax(mlr, fabs(lr));
            mrl = fmax(mrl, fabs(rl));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            mlr = fmax(mlr, __shfl_xor_sync(0xffffffffu, mlr, off));
            mrl = fmax(mrl, __shfl_xor_sync(0xffffffffu, mrl, off));
        }
        if ((threadIdx.x & 31) == 0) {
            s_red[0][threadIdx.x >> 5] = mlr;
            s_red[1][threadIdx.x >> 5] = mrl;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, b = 0.0;
            for (int w = 0; w < kCplThreads / 32; ++w) {
                a = fmax(a, s_red[0][w]);
                b = fmax(b, s_red[1][w]);
            }
            out[((size_t)(d - d0) * nfi + fi) * 2 + 0] = a;
            out[((size_t)(d - d0) * nfi + fi) * 2 + 1] = b;
        }
    }
}
}  // namespace

void dev_coupling_max(int dim, int nfi, int nf, int nqf, int nfn, const int* iface, const double* fgeom,
                      const double* fsj, const double* fqw, const double* trace, const double* traceR,
                      const double* odir, int d0, int d1, double* out, void* stream) {
    if (nqf > 64) throw Error(-1, "dev_coupling_max: too many face points");
    if (nfi == 0 || d1 <= d0) return;
    coupling_max_kernel<<<nfi, kCplThreads, 0, (cudaStream_t)stream>>>(dim, nfi, nf, nqf, nfn, iface, fgeom, fsj, fqw,
                                                                       trace, traceR, odir, d0, d1, out);
    SCHECK(cudaGetLastError());
}

}  // namespace hsw
