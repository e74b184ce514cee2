// K1 production sweep kernel (r1b): blocked Gauss-Jordan with FP64 tensor-core
// (DMMA m8n8k4) trailing updates on the augmented local system [A | rhs].
//
// Replaces SweepSolver::sweep's per-element step (solver.hpp:104-114): assemble
//   A = sum_k Omega_k G_k + F_out + sigma_t M   (assembly.hpp:393; T tensors)
//   rhs = s_e + incoming upwind traces (retained psi_new / lagged psi_old)
// and solve with partial pivoting (PartialPivLU, solver.hpp:69,114).
//
// Layout: [A | rhs] (N x (N+1), padded to 8x8 tiles) lives in
// DMMA accumulator fragments: lane (g = lane/4, q = lane%4) holds rows 8tr+g,
// columns 8tc + 2q + {0,1}.  W warps per pair own tile-columns tc % W == w.
// Panels of 4 columns (the DMMA k): the owner warp copies the panel to SMEM,
// reads it back row-per-lane and eliminates its 4 columns with partial pivoting
// (redux.sync on the high word of |a|, ties -> lowest lane) keeping every
// multiplier; then every warp gathers the 4 pivot rows of its columns,
// applies L11^{-1} (U = L11^{-1} A[P,:], zero on the panel's own columns) and
// updates all its tiles with one DMMA per tile: C -= L_panel * U.  Gauss-Jordan
// (every row except the pivot is eliminated) removes the back substitution:
// x_k = rhs(p_k) / pivot_k.  One-panel lookahead: the owner of panel P+1
// updates that tile-column first, factors P+1 and publishes its multipliers
// before finishing panel P's update of its other tiles.
#include "hsw_internal.hpp"

#include <cuda_runtime.h>

#include <cassert>
#include <cstdint>
#include <cstdlib>
#include <string>

#ifdef HSW_DEBUG_BOUNDS
#define HSW_ASSERT(c) assert(c)
#else
#define HSW_ASSERT(c) ((void)0)
#endif

namespace hsw {

#define DCHECK(x)                                                                              \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess)                                                                 \
            throw Error(-8, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x);       \
    } while (0)

template <int DIM, int P, int W>
struct DG {
    static constexpr int N1 = P + 1;
    static constexpr int N = DIM == 2 ? N1 * N1 : N1 * N1 * N1;
    static constexpr int NTR = (N + 7) / 8;             // tile rows
    static constexpr int NTC = (N + 1 + 7) / 8;         // tile columns (rhs = column N)
    static constexpr int TCW = (NTC + W - 1) / W;       // tile columns per warp
    static constexpr int NR = 8 * NTR;                  // padded rows
    static constexpr int RP = (NR + 31) / 32;           // panel rows per lane (row layout)
    static constexpr int NPANEL = (N + 3) / 4;
    static constexpr int NFN = DIM == 2 ? N1 : N1 * N1;
    static constexpr int NF = 2 * DIM;
    static constexpr int NQ1 = P + 2;
    static constexpr int NQF = DIM == 2 ? NQ1 : NQ1 * NQ1;
    static constexpr int GROUPS = W == 1 ? 4 : 1;
    static constexpr int THREADS = 32 * W * GROUPS;
    static constexpr int REGS = 4 * TCW * NTR + 16 * RP + 72;
    static constexpr int MINB0 = 65536 / (THREADS * REGS);
    static constexpr int MINB = MINB0 < 1 ? 1 : (MINB0 > 8 ? 8 : MINB0);
    static constexpr int T1SZ = DIM == 3 ? NQ1 * N1 * N1 : 0;
    // per-pair scratch (doubles)
    static constexpr int SM_WQ = 0;
    static constexpr int SM_WI = SM_WQ + NF * NQF;
    static constexpr int SM_TR = SM_WI + NF * NQF;
    static constexpr int SM_UP = SM_TR + NF * NQF;
    static constexpr int SM_T1 = SM_UP + NF * NFN;
    static constexpr int SM_F = SM_T1 + NF * T1SZ;
    static constexpr int SM_FLAGS = SM_F + NF * NFN * NFN;          // 2 ints + 2 ints
    static constexpr int SM_PIVV = SM_FLAGS + 2;                    // [N]
    static constexpr int SM_ROWS = SM_PIVV + N;                     // [N] ints
    static constexpr int SM_PAN = (SM_ROWS + (N + 1) / 2 + 1) & ~1; // [NR][4]
    static constexpr int SM_LP = SM_PAN + NR * 4;                   // [4 bufs][4][NR]
    static constexpr int SM_PROW = SM_LP + 16 * NR;                 // [4 bufs][4] ints -> 8 doubles
    static constexpr int SM_AMX = SM_PROW + 8;                      // [W] + ready
    static constexpr int SM_PAIR = (SM_AMX + W + 2 + 1) & ~1;
    static constexpr int SM_UW = 2 * 4 * 8 * TCW;                   // per warp: Uraw + U
    static constexpr int SM_GROUP = SM_PAIR + W * SM_UW;
    static constexpr int TAB_INTS = NF * N + N + NF * NFN;
    static constexpr int TAB_TRACE = ((TAB_INTS + 1) / 2 + 1) & ~1;
    static constexpr int TAB_TOTAL = (TAB_TRACE + NQF * NFN + NQ1 * N1 + 1) & ~1;
    static constexpr size_t SMEM = (size_t)(TAB_TOTAL + GROUPS * SM_GROUP) * sizeof(double);
};

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void bar_named(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int DIM, int P, int W>
__global__ void __launch_bounds__(DG<DIM, P, W>::THREADS, DG<DIM, P, W>::MINB)
dmma_sweep_kernel(const DevProblem pr, const double* __restrict__ src, const double* __restrict__ psi_old,
                  const double* psi_new_in, double* psi_out, int64_t psi_stride, const int* __restrict__ pairs,
                  int npairs, const double* __restrict__ rhs_given, unsigned long long* err_key, int64_t zero_pair) {
    using G = DG<DIM, P, W>;
    constexpr int N = G::N, NTR = G::NTR, TCW = G::TCW, NR = G::NR, RP = G::RP, NPANEL = G::NPANEL;
    constexpr int NFN = G::NFN, NF = G::NF, NQ1 = G::NQ1, NQF = G::NQF, N1 = G::N1, T1SZ = G::T1SZ;
    extern __shared__ double smem[];

    const long long t_start = clock64();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = warp / W, w = warp - group * W;
    const int g = lane >> 2, q = lane & 3;

    // element tables staged in SMEM (lane-varying indices)
    int* s_fidx = reinterpret_cast<int*>(smem);
    int* s_nmask = s_fidx + NF * N;
    int* s_fnode = s_nmask + N;
    double* s_trace = smem + G::TAB_TRACE;
    double* s_line = s_trace + NQF * NFN;
    for (int idx = threadIdx.x; idx < NF * N; idx += G::THREADS)
        s_fidx[idx] = __ldg(pr.g_fidx + (idx / N) * 128 + idx % N);
    for (int idx = threadIdx.x; idx < N; idx += G::THREADS) s_nmask[idx] = __ldg(pr.g_nmask + idx);
    for (int idx = threadIdx.x; idx < NF * NFN; idx += G::THREADS)
        s_fnode[idx] = __ldg(pr.g_fnode + (idx / NFN) * kMaxFaceNodes + idx % NFN);
    for (int idx = threadIdx.x; idx < NQF * NFN; idx += G::THREADS)
        s_trace[idx] = __ldg(pr.g_trace + (idx / NFN) * kMaxFaceNodes + idx % NFN);
    for (int idx = threadIdx.x; idx < NQ1 * N1; idx += G::THREADS)
        s_line[idx] = __ldg(pr.g_line + (idx / N1) * 8 + idx % N1);
    __syncthreads();
    const long long t_tab = clock64();

    double* psm = smem + G::TAB_TOTAL + (size_t)group * G::SM_GROUP;
    double* uw = psm + G::SM_PAIR + w * G::SM_UW;   // this warp's Uraw[4][8TCW], U[4][8TCW]
    double* Uraw = uw;
    double* Ub = uw + 4 * 8 * TCW;
    double* WQ = psm + G::SM_WQ;
    double* WI = psm + G::SM_WI;
    double* TR = psm + G::SM_TR;
    double* UP = psm + G::SM_UP;
    double* T1 = psm + G::SM_T1;
    double* FM = psm + G::SM_F;
    int* flg = reinterpret_cast<int*>(psm + G::SM_FLAGS);
    double* pivval = psm + G::SM_PIVV;
    int* rowstep = reinterpret_cast<int*>(psm + G::SM_ROWS);
    double* Pan = psm + G::SM_PAN;
    double* Lp = psm + G::SM_LP;
    int* prows = reinterpret_cast<int*>(psm + G::SM_PROW);
    double* amx = psm + G::SM_AMX;
    volatile int* ready = reinterpret_cast<volatile int*>(amx + W);

    const int pidx = blockIdx.x * G::GROUPS + group;
    const bool active = pidx < npairs;
    const int pair = pairs[active ? pidx : 0];
    const int e = pair / pr.nd, d = pair - (pair / pr.nd) * pr.nd;
    const double om0 = pr.omega[d * 4 + 0], om1 = pr.omega[d * 4 + 1], om2 = pr.omega[d * 4 + 2];
    const int gthreads = 32 * W;
    const int ctid = w * 32 + lane;
    auto pair_sync = [&]() {
        if (W > 1) bar_named(1 + group, gthreads);
        else __syncwarp();
    };
    const int dbg = pr.debug_flags;

    // ------------------------------------------------ volume terms into the accumulator tiles
    double acc[TCW][NTR][2];
    {
        const double st = pr.sig_t[e];
        const double2* Te = reinterpret_cast<const double2*>(pr.T) + (size_t)e * (t_elem_doubles(N) / 2);   // fragment order (t_idx)
#pragma unroll
        for (int j = 0; j < TCW; ++j)
#pragma unroll
            for (int tr = 0; tr < NTR; ++tr)
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int r = 8 * tr + g, c = 8 * (j * W + w) + 2 * q + s;
                    double v = 0.0;
                    if (r < N && c < N) {
                        const double4 t = (dbg & 4) ? make_double4(r == c ? 1.0 : 0.0, 0.0, 0.0, 0.0)
                                                    : make_double4(Te[t_idx2(N, r, c, 0)].x, Te[t_idx2(N, r, c, 0)].y, Te[t_idx2(N, r, c, 1)].x,
                                                                  Te[t_idx2(N, r, c, 1)].y);
                        double gg = om0 * t.y + om1 * t.z;
                        if (DIM == 3) gg += om2 * t.w;
                        v = gg + st * t.x;
                    } else if (r < N && c == N) {
                        v = rhs_given ? rhs_given[r] : src[(size_t)e * N + r];
                    }
                    acc[j][tr][s] = v;
                }
    }

    // ------------------------------------------------ faces (same scheme as hsw_gj.cu)
    const unsigned inflags = rhs_given ? 0u : pr.inflags[(size_t)d * pr.nel + e];
    if (ctid == 0) { flg[0] = 0; flg[1] = 0; }
    pair_sync();
    int outm = 0, inm = 0;
    // Romberg face rule (2D): face blocks integrated at create (assembly.hpp:121-131)
    const bool romb = DIM == 2 && pr.rom_ob != nullptr;
    const size_t rfb = ((size_t)d * pr.nel + e) * NF;
    if (!(dbg & 1)) {
        if (romb && ctid == 0) outm = (int)pr.rom_omask[(size_t)d * pr.nel + e];
        for (int idx = ctid; idx < (romb ? 0 : NF * NQF); idx += gthreads) {
            const int f = idx / NQF, qq = idx - (idx / NQF) * NQF;
            const double4 gm = reinterpret_cast<const double4*>(pr.fgeom)[((size_t)e * NF + f) * NQF + qq];
            double on = om0 * gm.x + om1 * gm.y;
            if (DIM == 3) on += om2 * gm.z;
            const double wp = on > 0.0 ? on * gm.w : 0.0;
            WQ[idx] = wp;
            WI[idx] = on < 0.0 ? -on * gm.w : 0.0;
            if (wp != 0.0) outm |= 1 << f;
        }
        for (int idx = ctid; idx < NF * NFN; idx += gthreads) {
            const int f = idx / NFN, aa = idx - (idx / NFN) * NFN;
            const int4 nb4 = reinterpret_cast<const int4*>(pr.fnbr)[(size_t)e * NF + f];
            if ((inflags >> (2 * f)) & 1u) {
                const bool lag = (inflags >> (2 * f + 1)) & 1u;
                const double* sp = (lag ? psi_old : psi_new_in) + (size_t)d * psi_stride + (size_t)nb4.x * N;
                const int a0 = aa % N1, b0 = aa / N1, code = nb4.z;
                int ao, bo;
                if (DIM == 2) { ao = code ? P - a0 : a0; bo = 0; }
                else {
                    int u = a0, v = b0;
                    if (code & 4) { u = b0; v = a0; }
                    if (code & 2) u = P - u;
                    if (code & 1) v = P - v;
                    ao = u; bo = v;
                }
                UP[idx] = sp[s_fnode[nb4.y * NFN + bo * N1 + ao]];
                if (aa == 0) inm |= 1 << f;
            } else if (!rhs_given && nb4.x < 0 && pr.inflow != 0.0) {
                if (aa == 0) inm |= 1 << (f + 8);
            }
        }
        if (outm) atomicOr(flg, outm);
        if (inm) atomicOr(flg + 1, inm);
        pair_sync();
        outm = flg[0];
        inm = flg[1];
        for (int idx = ctid; idx < (romb ? 0 : NF * NQF); idx += gthreads) {
            const int f = idx / NQF, qq = idx - (idx / NQF) * NQF;
            double t = 0.0;
            if ((inm >> f) & 1) {
#pragma unroll
                for (int aa = 0; aa < NFN; ++aa) t += s_trace[qq * NFN + aa] * UP[f * NFN + aa];
            } else if ((inm >> (f + 8)) & 1) {
                t = pr.inflow;
            }
            TR[idx] = t * WI[idx];
        }
        if (DIM == 3 && !romb) {
            for (int idx = ctid; idx < NF * T1SZ; idx += gthreads) {
                const int f = idx / (T1SZ > 0 ? T1SZ : 1), rem = idx - f * T1SZ;
                if (!((outm >> f) & 1)) continue;
                const int jq = rem / (N1 * N1), r2 = rem - jq * N1 * N1;
                const int aa = r2 / N1, ab = r2 - aa * N1;
                double s = 0.0;
#pragma unroll
                for (int iq = 0; iq < NQ1; ++iq)
                    s += WQ[f * NQF + jq * NQ1 + iq] * (s_line[iq * N1 + aa] * s_line[iq * N1 + ab]);
                T1[idx] = s;
            }
            pair_sync();
        }
        for (int idx = ctid; idx < NF * NFN * NFN; idx += gthreads) {
            const int f = idx / (NFN * NFN), rem = idx - f * NFN * NFN;
            if (!((outm >> f) & 1)) continue;
            const int fa = rem / NFN, fb = rem - fa * NFN;
            double s = 0.0;
            if (romb) {
                s = pr.rom_ob[(rfb + f) * NFN * NFN + rem];
            } else if (DIM == 3) {
                const int a0 = fa % N1, b0 = fa / N1, a1 = fb % N1, b1 = fb / N1;
#pragma unroll
                for (int jq = 0; jq < NQ1; ++jq)
                    s += T1[f * T1SZ + (jq * N1 + a0) * N1 + a1] * (s_line[jq * N1 + b0] * s_line[jq * N1 + b1]);
            } else {
#pragma unroll
                for (int iq = 0; iq < NQ1; ++iq) s += WQ[f * NQF + iq] * (s_line[iq * N1 + fa] * s_line[iq * N1 + fb]);
            }
            FM[idx] = s;
        }
        pair_sync();
    }
    const long long t_face = clock64();
    // face contributions into the tiles
#pragma unroll
    for (int tr = 0; tr < NTR; ++tr) {
        const int r = 8 * tr + g;
        const int rm = r < N ? s_nmask[r] : 0;
#pragma unroll
        for (int j = 0; j < TCW; ++j)
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int c = 8 * (j * W + w) + 2 * q + s;
                if (r < N && c < N) {
                    int m = rm & outm & s_nmask[c];
                    while (m) {
                        const int f = __ffs(m) - 1;
                        m &= m - 1;
                        acc[j][tr][s] += FM[f * NFN * NFN + s_fidx[f * N + r] * NFN + s_fidx[f * N + c]];
                    }
                } else if (r < N && c == N) {
                    int m = rm & (inm | (inm >> 8)) & 63;
                    while (m) {
                        const int f = __ffs(m) - 1;
                        m &= m - 1;
                        const int fr = s_fidx[f * N + r];
                        double s2 = 0.0;
                        if (romb) {   // coupling block times the gathered upwind traces, or the inflow moments
                            if ((inm >> f) & 1) {
                                const double* ib = pr.rom_ib + ((rfb + f) * NFN + fr) * NFN;
                                for (int aa = 0; aa < NFN; ++aa) s2 += ib[aa] * UP[f * NFN + aa];
                            } else {
                                s2 = pr.rom_bin[(rfb + f) * NFN + fr];
                            }
                        } else {
                            for (int qq = 0; qq < NQF; ++qq) s2 += TR[f * NQF + qq] * s_trace[qq * NFN + fr];
                        }
                        acc[j][tr][s] += s2;
                    }
                }
            }
    }
    if ((int64_t)pair == zero_pair) {
#pragma unroll
        for (int j = 0; j < TCW; ++j)
#pragma unroll
            for (int tr = 0; tr < NTR; ++tr)
#pragma unroll
                for (int s = 0; s < 2; ++s)
                    if (8 * (j * W + w) + 2 * q + s < N) acc[j][tr][s] = 0.0;
    }
    // matrix scale for the singularity test (stand-in for rcond > 1e-14, solver.hpp:70)
    double amax = 0.0;
#pragma unroll
    for (int j = 0; j < TCW; ++j)
#pragma unroll
        for (int tr = 0; tr < NTR; ++tr)
#pragma unroll
            for (int s = 0; s < 2; ++s)
                if (8 * (j * W + w) + 2 * q + s < N) amax = fmax(amax, fabs(acc[j][tr][s]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    if (W > 1) {
        if (lane == 0) amx[w] = amax;
        if (ctid == 0) *ready = -1;
        pair_sync();
#pragma unroll
        for (int qq = 0; qq < W; ++qq) amax = fmax(amax, amx[qq]);
    }
    const long long t_asm = clock64();

    // ------------------------------------------------ blocked Gauss-Jordan
    unsigned rdone = 0;  // row layout: bit i = row lane + 32 i pivoted (or padding)
#pragma unroll
    for (int i = 0; i < RP; ++i)
        if (lane + 32 * i >= N) rdone |= 1u << i;
    bool singular = false;

    // factor panel Pn (owner warp): copy its 4 columns to row layout, eliminate, publish multipliers
    auto factor = [&](int Pn) {
        const int TCp = Pn >> 1, h = Pn & 1, jp = TCp / W;
        double* lp = Lp + (Pn & 3) * 4 * NR;
        int* prw = prows + (Pn & 3) * 4;
        if ((q >> 1) == h) {
#pragma unroll
            for (int j = 0; j < TCW; ++j)
                if (j == jp) {
#pragma unroll
                    for (int tr = 0; tr < NTR; ++tr)
                        *reinterpret_cast<double2*>(Pan + (8 * tr + g) * 4 + 2 * (q - 2 * h)) =
                            make_double2(acc[j][tr][0], acc[j][tr][1]);
                }
        }
        __syncwarp();
        double pv[RP][4];
#pragma unroll
        for (int i = 0; i < RP; ++i) {
            const int r = lane + 32 * i;
            if (r < NR) {
                const double2 x0 = *reinterpret_cast<const double2*>(Pan + r * 4);
                const double2 x1 = *reinterpret_cast<const double2*>(Pan + r * 4 + 2);
                pv[i][0] = x0.x; pv[i][1] = x0.y; pv[i][2] = x1.x; pv[i][3] = x1.y;
            } else {
                pv[i][0] = pv[i][1] = pv[i][2] = pv[i][3] = 0.0;
            }
        }
        double lr[RP][4];
        int pst[4] = {-1, -1, -1, -1};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int k = 4 * Pn + t;
            if (k >= N) {
#pragma unroll
                for (int i = 0; i < RP; ++i) lr[i][t] = 0.0;
                if (lane == 0) prw[t] = -1;
                continue;
            }
            unsigned key = 0u;
            int ks = 0;
#pragma unroll
            for (int i = 0; i < RP; ++i) {
                const unsigned hi = (unsigned)(__double_as_longlong(fabs(pv[i][t])) >> 32) + 1u;
                if (!((rdone >> i) & 1u) && hi > key) { key = hi; ks = i; }
            }
            double mine[4];
#pragma unroll
            for (int tt = 0; tt < 4; ++tt) {
                mine[tt] = pv[0][tt];
#pragma unroll
                for (int i = 1; i < RP; ++i)
                    if (i == ks) mine[tt] = pv[i][tt];
            }
            const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
            const unsigned bal = __ballot_sync(0xffffffffu, key == kmax && key != 0u);
            const int src_lane = __ffs(bal) - 1;
            HSW_ASSERT(src_lane >= 0 && src_lane < 32);
            const int prow = __shfl_sync(0xffffffffu, lane + 32 * ks, src_lane);
            HSW_ASSERT(prow >= 0 && prow < N);
            const double piv = __shfl_sync(0xffffffffu, mine[t], src_lane);
            if (!(fabs(piv) > 1e-14 * amax)) singular = true;
            const double rinv = 1.0 / piv;
#pragma unroll
            for (int i = 0; i < RP; ++i) lr[i][t] = (lane + 32 * i == prow) ? 0.0 : pv[i][t] * rinv;
#pragma unroll
            for (int tt = t + 1; tt < 4; ++tt) {
                const double u = __shfl_sync(0xffffffffu, mine[tt], src_lane);
#pragma unroll
                for (int i = 0; i < RP; ++i) pv[i][tt] -= lr[i][t] * u;
            }
            if (lane == (prow & 31)) rdone |= 1u << (prow >> 5);
            pst[t] = prow;
            if (lane == 0) {
                pivval[k] = piv;
                rowstep[prow] = k;
                prw[t] = prow;
            }
        }
        // L~ = L * L11^{-1}, L11[t2][t] = l_t(p_t2) (t < t2): then the trailing update is
        // A -= L~ * A[P,:] with the raw pre-panel pivot rows as the B operand.
        double l11[4][4];
#pragma unroll
        for (int t2 = 1; t2 < 4; ++t2)
#pragma unroll
            for (int t = 0; t < t2; ++t) {
                const int p2 = pst[t2];
                double v = lr[0][t];
#pragma unroll
                for (int i = 1; i < RP; ++i)
                    if (p2 >= 0 && i == (p2 >> 5)) v = lr[i][t];
                v = __shfl_sync(0xffffffffu, v, p2 >= 0 ? (p2 & 31) : 0);
                l11[t2][t] = p2 >= 0 ? v : 0.0;
            }
#pragma unroll
        for (int i = 0; i < RP; ++i) {
            double lt3 = lr[i][3];
            double lt2 = lr[i][2] - lt3 * l11[3][2];
            double lt1 = lr[i][1] - lt2 * l11[2][1] - lt3 * l11[3][1];
            double lt0 = lr[i][0] - lt1 * l11[1][0] - lt2 * l11[2][0] - lt3 * l11[3][0];
            lr[i][0] = lt0; lr[i][1] = lt1; lr[i][2] = lt2; lr[i][3] = lt3;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < RP; ++i)
                if (lane + 32 * i < NR) lp[t * NR + lane + 32 * i] = lr[i][t];
        __syncwarp();
        if (W > 1 && lane == 0) {
            __threadfence_block();
            *ready = Pn;
        }
    };

    // DMMA update of local tile-column j with panel multipliers (bufp) and this warp's U
    auto update_tc = [&](int j, const double* lpb, const double (&bfr)[TCW]) {
#pragma unroll
        for (int jj = 0; jj < TCW; ++jj)
            if (jj == j) {
                const double b = bfr[jj];
#pragma unroll
                for (int tr = 0; tr < NTR; ++tr) {
                    const double a = -lpb[q * NR + 8 * tr + g];
                    dmma_884(acc[jj][tr][0], acc[jj][tr][1], a, b);
                }
            }
    };

    if (!(dbg & 2)) {
        long long c_wait = 0, c_u = 0, c_mma = 0, c_fac = 0, c0, c1;
        c0 = clock64();
        if (w == 0) factor(0);
        c_fac += clock64() - c0;
#pragma unroll 1
        for (int Pn = 0; Pn < NPANEL; ++Pn) {
            const int owner = (Pn >> 1) % W;
            c0 = clock64();
            if (W > 1 && w != owner) {
                while (*ready < Pn) __nanosleep(20);
                __threadfence_block();
            }
            c1 = clock64();
            c_wait += c1 - c0;
            const double* lpb = Lp + (Pn & 3) * 4 * NR;
            const int* prw = prows + (Pn & 3) * 4;
            int pr4[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                pr4[t] = prw[t];
                HSW_ASSERT(pr4[t] >= -1 && pr4[t] < N);
                // every warp tracks the pivot set (the owner of a later panel searches with it)
                if (pr4[t] >= 0 && lane == (pr4[t] & 31)) rdone |= 1u << (pr4[t] >> 5);
            }
            // B fragments = raw pre-panel pivot rows over this warp's columns (L11^{-1} is
            // folded into the published multipliers): the quad holding pivot row p_t
            // writes it to SMEM, lane (g, q) reads B[q][8j + g].
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int p = pr4[t];
                if (p >= 0) {
                    const bool holder = g == (p & 7);
                    double* dst = Uraw + t * 8 * TCW + 2 * q;
                    switch (p >> 3) {  // uniform tile-row of the pivot row
#define HSW_TP(T_)                                                                            \
    case T_:                                                                                  \
        if (holder) {                                                                         \
            _Pragma("unroll") for (int j = 0; j < TCW; ++j)                                   \
                *reinterpret_cast<double2*>(dst + 8 * j) =                                    \
                    make_double2(acc[j][T_ < NTR ? T_ : 0][0], acc[j][T_ < NTR ? T_ : 0][1]); \
        }                                                                                     \
        break;
                        HSW_TP(0) HSW_TP(1) HSW_TP(2) HSW_TP(3) HSW_TP(4) HSW_TP(5) HSW_TP(6) HSW_TP(7)
                        HSW_TP(8) HSW_TP(9) HSW_TP(10) HSW_TP(11) HSW_TP(12) HSW_TP(13) HSW_TP(14) HSW_TP(15)
#undef HSW_TP
                        default: break;
                    }
                }
            }
            __syncwarp();
            double bfr[TCW];
            {
                const bool qv = pr4[q] >= 0;
#pragma unroll
                for (int j = 0; j < TCW; ++j) bfr[j] = qv ? Uraw[q * 8 * TCW + 8 * j + g] : 0.0;
            }
            // lookahead: the owner of panel Pn+1 updates that tile-column first and factors it
            const int Pn1 = Pn + 1;
            const int own1 = (Pn1 >> 1) % W, jn = (Pn1 >> 1) / W;
            const bool look = Pn1 < NPANEL && w == own1;
            c0 = clock64();
            c_u += c0 - c1;
            if (look) {
                update_tc(jn, lpb, bfr);
                c1 = clock64();
                factor(Pn1);
                c_fac += clock64() - c1;
            }
            c1 = clock64();
#pragma unroll
            for (int j = 0; j < TCW; ++j) {
                const int tcg = j * W + w;
                const bool live = 8 * tcg + 7 >= 4 * Pn + 4 || tcg == N / 8;  // the rhs tile stays live
                if (live && !(look && j == jn)) update_tc(j, lpb, bfr);
            }
            __syncwarp();  // Uraw reuse by the next panel's gather
            c_mma += clock64() - c1;
            c0 = clock64();
            if (W > 1 && (Pn & 1)) pair_sync();  // bounds the 4-deep multiplier ring
            c_wait += clock64() - c0;
        }
        if ((dbg & 8) && lane == 0 && w == 0 && active) {
            atomicAdd(pr.prof + 8, (unsigned long long)c_wait);
            atomicAdd(pr.prof + 9, (unsigned long long)c_u);
            atomicAdd(pr.prof + 10, (unsigned long long)c_mma);
            atomicAdd(pr.prof + 11, (unsigned long long)c_fac);
        }
        if (W > 1) pair_sync();
        else __syncwarp();
    }
    const long long t_gj = clock64();

    // ------------------------------------------------ solution x_k = rhs(p_k) / pivot_k
    if (singular && active && lane == 0) atomicMin(err_key, (unsigned long long)pair);
    constexpr int TCR = N / 8, OWR = TCR % W, JR = TCR / W, QR = (N % 8) / 2, SR = N % 2;
    if (active && w == OWR && q == QR) {
        double* out = rhs_given ? psi_out : psi_out + (size_t)d * psi_stride + (size_t)e * N;
#pragma unroll
        for (int tr = 0; tr < NTR; ++tr) {
            const int r = 8 * tr + g;
            if (r < N) {
                if (dbg & 2) {
                    out[r] = acc[JR][tr][SR];
                } else {
                    const int kk = rowstep[r];
                    HSW_ASSERT(kk >= 0 && kk < N);
                    out[kk] = acc[JR][tr][SR] / pivval[kk];
                }
            }
        }
    }
    if ((dbg & 8) && lane == 0 && w == 0 && active) {
        const long long t_end = clock64();
        atomicAdd(pr.prof + 0, (unsigned long long)(t_tab - t_start));
        atomicAdd(pr.prof + 1, (unsigned long long)(t_face - t_tab));
        atomicAdd(pr.prof + 2, (unsigned long long)(t_asm - t_face));
        atomicAdd(pr.prof + 3, (unsigned long long)(t_gj - t_asm));
        atomicAdd(pr.prof + 4, (unsigned long long)(t_end - t_gj));
        atomicAdd(pr.prof + 5, 1ull);
    }
}

template <int DIM, int P, int W>
static void launch_dmma(const DevProblem& pr, const double* src, const double* psi_old, const double* psi_new_in,
                        double* psi_out, int64_t stride, const int* pairs, int npairs, const double* rhs_given,
                        unsigned long long* err, int64_t zero_pair, cudaStream_t st) {
    using G = DG<DIM, P, W>;
    static int slots[64] = {};
    static std::mutex mu;
    int dev = 0;
    DCHECK(cudaGetDevice(&dev));
    per_device_once(slots, mu, dev, [&] {
        DCHECK(cudaFuncSetAttribute(dmma_sweep_kernel<DIM, P, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)G::SMEM));
        return 1;
    });
    const int blocks = (npairs + G::GROUPS - 1) / G::GROUPS;
    dmma_sweep_kernel<DIM, P, W><<<blocks, G::THREADS, G::SMEM, st>>>(pr, src, psi_old, psi_new_in, psi_out, stride,
                                                                      pairs, npairs, rhs_given, err, zero_pair);
    DCHECK(cudaGetLastError());
}

// debug: HSW_DMMA_ALT=1 swaps the warp split (n=64: W=8, n=125: W=4) for bisection
static bool dmma_alt() {
    static const bool v = [] { const char* e = std::getenv("HSW_DMMA_ALT"); return e && e[0] == '1'; }();
    return v;
}

#define DMMA_DISPATCH(DIMV, PV, CALL)                                   \
    do {                                                                \
        if (DIMV == 2) {                                                \
            switch (PV) {                                               \
                case 1: CALL(2, 1, 1); break;                           \
                case 2: CALL(2, 2, 1); break;                           \
                case 3: CALL(2, 3, 1); break;                           \
                case 4: CALL(2, 4, 1); break;                           \
                case 5: CALL(2, 5, 1); break;                           \
                case 6: CALL(2, 6, 2); break;                           \
                default: throw Error(-1, "unsupported 2D order");      \
            }                                                           \
        } else {                                                        \
            switch (PV) {                                               \
                case 1: CALL(3, 1, 1); break;                           \
                case 2: CALL(3, 2, 1); break;                           \
                case 3: if (dmma_alt()) CALL(3, 3, 8); else CALL(3, 3, 3); break; \
                case 4: if (dmma_alt()) CALL(3, 4, 4); else CALL(3, 4, 8); break; \
                default: throw Error(-1, "unsupported 3D order");      \
            }                                                           \
        }                                                               \
    } while (0)

void dev_dmma_sweep(const DevProblem& P, const double* src, const double* psi_old, double* psi_new, int64_t stride,
                    const int* pairs, int npairs, unsigned long long* err_key, int64_t zero_pair, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
#define CALL_D(D_, P_, W_) \
    launch_dmma<D_, P_, W_>(P, src, psi_old, psi_new, psi_new, stride, pairs, npairs, nullptr, err_key, zero_pair, st)
    DMMA_DISPATCH(P.dim, P.p, CALL_D);
#undef CALL_D
}

void dev_dmma_local_solve(const DevProblem& P, const int* pair_dev, const double* rhs, double* out,
                          unsigned long long* err_key, int64_t zero_pair, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
#define CALL_DL(D_, P_, W_) \
    launch_dmma<D_, P_, W_>(P, nullptr, nullptr, nullptr, out, 0, pair_dev, 1, rhs, err_key, zero_pair, st)
    DMMA_DISPATCH(P.dim, P.p, CALL_DL);
#undef CALL_DL
}

}  // namespace hsw
