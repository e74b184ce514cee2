// K1 production sweep kernel: register-resident Gauss-Jordan on the augmented
// local system [A | rhs] of each (element, ordinate) pair.
//
// Replaces SweepSolver::sweep's per-element step (solver.hpp:104-114): assemble
//   A = sum_k Omega_k G_k + F_out + sigma_t M      (assembly.hpp:393; T tensors)
//   rhs = s_e + sum_{incoming faces} w_in * trace(psi_upwind)   (solver.hpp:105-113)
// and solve with partial pivoting (PartialPivLU, solver.hpp:69,114).
//
// Layout: lane `ll` of a pair owns rows r = ll + L*i (i < R);
// warp w of the pair owns augmented columns j = s*W + w (s < CW, cyclic).  The
// matrix never leaves registers.  Per elimination step k only the owner warp
// of column k searches the pivot (packed 64-bit key butterfly: |a| high word,
// then lowest row), computes the multipliers of its rows (local — no load) and
// publishes them for the other warps (double-buffered SMEM + named barrier);
// the pivot row segment of each warp is broadcast through a per-warp SMEM
// line (STS by the owner lane, LDS.128 broadcast by all).
//
// Gauss-Jordan keeps every lane busy (no idle pivoted rows) and removes the
// back substitution: x_k = rhs(p_k) / pivot_k.  Columns <= k are dead after
// step k (never read again), so the update may touch them: the step body
// updates whole blocks of SB slots starting at the block that holds column k,
// entered through one fall-through switch — no per-slot predicates, one copy
// of the body (the kernel stays in the instruction cache).  Pivots are chosen
// by |a| to ~2^-20 relative precision (ties -> lowest row): a valid
// partial-pivoting choice.
#include "hsw_internal.hpp"

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace hsw {

__constant__ int c_fnode[kMaxFaces][kMaxFaceNodes];          // face node a -> element node
__constant__ double c_trace[kMaxFacePoints][kMaxFaceNodes];  // phi_a at face point q
__constant__ int c_fidx[kMaxFaces][128];                      // element node -> face node index, or -1
__constant__ unsigned char c_nmask[128];                      // element node -> bitmask of its faces
__constant__ double c_line[8][8];                             // L_a(x_i) at the face Gauss points [i][a]

#define GCHECK(x)                                                                              \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess)                                                                 \
            throw Error(-8, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x);       \
    } while (0)

void dev_upload_gj_tables(const ConstTables& t, const int* fidx /*6*128*/, const double* line /*8*8*/) {
    GCHECK(cudaMemcpyToSymbol(c_fnode, t.fnode, sizeof(t.fnode)));
    GCHECK(cudaMemcpyToSymbol(c_trace, t.trace, sizeof(t.trace)));
    GCHECK(cudaMemcpyToSymbol(c_fidx, fidx, sizeof(int) * kMaxFaces * 128));
    unsigned char mask[128] = {0};
    for (int f = 0; f < kMaxFaces; ++f)
        for (int m = 0; m < 128; ++m)
            if (fidx[f * 128 + m] >= 0) mask[m] |= (unsigned char)(1u << f);
    GCHECK(cudaMemcpyToSymbol(c_nmask, mask, sizeof(mask)));
    GCHECK(cudaMemcpyToSymbol(c_line, line, sizeof(double) * 64));
}

template <int DIM, int P, int W, int PPW>
struct GJ {
    static constexpr int N1 = P + 1;
    static constexpr int N = DIM == 2 ? N1 * N1 : N1 * N1 * N1;
    static constexpr int NC = N + 1;                         // augmented columns
    static constexpr int L = 32 / PPW;                       // lanes per pair
    static constexpr int R = (N + L - 1) / L;                // rows per lane
    static constexpr int SB = 4;                             // column slots per skip block
    // block-cyclic columns: blocks of SB consecutive columns, block b -> warp b % W
    static constexpr int NBLK = ((NC + SB - 1) / SB + W - 1) / W;  // blocks per warp
    static constexpr int CW = NBLK * SB;                     // slots per warp
    static constexpr int NFN = DIM == 2 ? N1 : N1 * N1;
    static constexpr int NF = 2 * DIM;
    static constexpr int NQ1 = P + 2;                        // face Gauss points per axis
    static constexpr int NQF = DIM == 2 ? NQ1 : NQ1 * NQ1;
    static constexpr int GROUPS = W == 1 ? 4 : (W == 2 ? 2 : 1);  // pair groups per CTA
    static constexpr int THREADS = 32 * W * GROUPS;
    static constexpr int PAIRS_PER_CTA = GROUPS * PPW;
    // CTAs per SM from the register budget (matrix slots + ~64 bookkeeping registers)
    static constexpr int REGS = 2 * R * CW + 64;
    static constexpr int MINB0 = 65536 / (THREADS * REGS);
    static constexpr int MINB = MINB0 < 1 ? 1 : (MINB0 > 4 ? 4 : MINB0);
    static constexpr int T1SZ = DIM == 3 ? NQ1 * N1 * N1 : 0;
    // per-pair shared scratch (doubles)
    static constexpr int SM_WQ = 0;                          // [NF][NQF] outflow weights w+ * w * |J|
    static constexpr int SM_WI = SM_WQ + NF * NQF;           // [NF][NQF] inflow weights
    static constexpr int SM_TR = SM_WI + NF * NQF;           // [NF][NQF] inflow trace * weight
    static constexpr int SM_UP = SM_TR + NF * NQF;           // [NF][NFN] upwind face values
    static constexpr int SM_T1 = SM_UP + NF * NFN;           // [NF][T1SZ]
    static constexpr int SM_F = SM_T1 + NF * T1SZ;           // [NF][NFN*NFN] outflow blocks
    static constexpr int SM_FLAGS = SM_F + NF * NFN * NFN;   // 2 ints: outflow mask, inflow mask
    static constexpr int SM_PIVV = SM_FLAGS + 2;             // [N] pivot value of step k
    static constexpr int SM_ROWS = SM_PIVV + N;              // [N] ints: step at which row r pivots
    static constexpr int SM_PAIR = (SM_ROWS + (N + 1) / 2 + 1) & ~1;
    static constexpr int SM_LBUF = W > 1 ? 8 * (L * R + 2) : 0;   // per group, W > 1 multiplier ring
    static constexpr int SM_UBUF = PPW * (CW + 2);           // per warp: pivot row lines
    static constexpr int SM_GROUP = PPW * SM_PAIR + SM_LBUF + W * SM_UBUF + 2 * W + 2;
    static constexpr int TAB_INTS = NF * N + N + NF * NFN;
    static constexpr int TAB_TRACE = ((TAB_INTS + 1) / 2 + 1) & ~1;   // doubles offset
    static constexpr int TAB_TOTAL = (TAB_TRACE + NQF * NFN + NQ1 * N1 + 1) & ~1;
    static constexpr size_t SMEM = (size_t)(TAB_TOTAL + GROUPS * SM_GROUP) * sizeof(double);
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int DIM, int P, int W, int PPW>
__global__ void __launch_bounds__(GJ<DIM, P, W, PPW>::THREADS, GJ<DIM, P, W, PPW>::MINB)
gj_sweep_kernel(const DevProblem pr, const double* __restrict__ src, const double* __restrict__ psi_old,
                const double* psi_new_in, double* psi_out, int64_t psi_stride, const int* __restrict__ pairs,
                int npairs, const double* __restrict__ rhs_given, unsigned long long* err_key,
                int64_t zero_pair) {
    using G = GJ<DIM, P, W, PPW>;
    constexpr int N = G::N, L = G::L, R = G::R, CW = G::CW, NFN = G::NFN, NF = G::NF;
    constexpr int NQ1 = G::NQ1, NQF = G::NQF, N1 = G::N1, SB = G::SB, NBLK = G::NBLK, T1SZ = G::T1SZ;
    extern __shared__ double smem[];

    const long long t_start = clock64();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = warp / W, w = warp - group * W;       // pair group, warp within group
    const int ps = lane / L, ll = lane - ps * L;             // pair slot within warp, lane within pair
    // element tables staged in SMEM (lane-varying indices: constant memory would serialise)
    int* s_fidx = reinterpret_cast<int*>(smem);                  // [NF][N] face-node index or -1
    int* s_nmask = s_fidx + NF * N;                              // [N] face bitmask of node m
    int* s_fnode = s_nmask + N;                                  // [NF][NFN] face node -> element node
    double* s_trace = smem + G::TAB_TRACE;                       // [NQF][NFN]
    double* s_line = s_trace + NQF * NFN;                        // [NQ1][N1]
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
    double* gsm = smem + G::TAB_TOTAL + (size_t)group * G::SM_GROUP;
    double* psm = gsm + ps * G::SM_PAIR;                      // this pair's scratch
    double* lbuf = gsm + PPW * G::SM_PAIR;                    // W > 1 multipliers (double-buffered)
    double* ubuf = lbuf + G::SM_LBUF + w * G::SM_UBUF + ps * (CW + 2);  // this warp's pivot row line
    double* amx = lbuf + G::SM_LBUF + W * G::SM_UBUF;           // W > 1: per-warp |A| max

    const int pidx = blockIdx.x * G::PAIRS_PER_CTA + group * PPW + ps;
    const bool active = pidx < npairs;
    const int pair = pairs[active ? pidx : 0];
    const int e = pair / pr.nd, d = pair - (pair / pr.nd) * pr.nd;
    const double om0 = pr.omega[d * 4 + 0], om1 = pr.omega[d * 4 + 1], om2 = pr.omega[d * 4 + 2];
    const int gthreads = 32 * W;
    const int ctid = PPW > 1 ? ll : w * 32 + lane;   // cooperative index over the pair's threads
    const int cnt = PPW > 1 ? L : gthreads;
    auto pair_sync = [&]() {
        if (W > 1) named_bar(1 + group, gthreads);
        else __syncwarp();
    };

    double* WQ = psm + G::SM_WQ;
    double* WI = psm + G::SM_WI;
    double* TR = psm + G::SM_TR;
    double* UP = psm + G::SM_UP;
    double* T1 = psm + G::SM_T1;
    double* FM = psm + G::SM_F;
    int* flg = reinterpret_cast<int*>(psm + G::SM_FLAGS);
    const unsigned inflags = rhs_given ? 0u : pr.inflags[(size_t)d * pr.nel + e];

    // ------------------------------------------------ faces, phase 1: weights + upwind gathers
    const int dbg = pr.debug_flags;
    // ------------------------------------------------ volume terms straight into registers
    // (issued before the face phase so the T-tensor loads overlap it; branch-free
    // so the compiler can batch the loads)
    double a[R][CW];
    {
        const double st = pr.sig_t[e];
        const double4* Te = reinterpret_cast<const double4*>(pr.T) + (size_t)e * N * N;
#pragma unroll
        for (int s = 0; s < CW; ++s) {
            const int j = ((s / SB) * W + w) * SB + (s % SB);
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int r = ll + L * i;
                double v = 0.0;
                if (r < N && j < N) {
                    const double4 t = (dbg & 4) ? make_double4(r == j ? 1.0 : 0.0, 0.0, 0.0, 0.0)
                                                : Te[(size_t)j * N + r];  // column-major: coalesced over rows
                    double g = om0 * t.y + om1 * t.z;
                    if (DIM == 3) g += om2 * t.w;
                    v = g + st * t.x;
                } else if (r < N && j == N) {
                    v = rhs_given ? rhs_given[r] : src[(size_t)e * N + r];
                }
                a[i][s] = v;
            }
        }
    }
    if (ctid == 0) { flg[0] = 0; flg[1] = 0; }
    pair_sync();
    int outm = 0, inm = 0;
    if (!(dbg & 1)) {
    for (int idx = ctid; idx < NF * NQF; idx += cnt) {
        const int f = idx / NQF, q = idx - (idx / NQF) * NQF;
        const double4 g = reinterpret_cast<const double4*>(pr.fgeom)[((size_t)e * NF + f) * NQF + q];
        double on = om0 * g.x + om1 * g.y;
        if (DIM == 3) on += om2 * g.z;
        const double wp = on > 0.0 ? on * g.w : 0.0;
        WQ[idx] = wp;
        WI[idx] = on < 0.0 ? -on * g.w : 0.0;
        if (wp != 0.0) outm |= 1 << f;
    }
    for (int idx = ctid; idx < NF * NFN; idx += cnt) {
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
            if (aa == 0) inm |= 1 << (f + 8);  // boundary inflow
        }
    }
    if (outm) atomicOr(flg, outm);
    if (inm) atomicOr(flg + 1, inm);
    pair_sync();
    outm = flg[0];
    inm = flg[1];
    // phase 2: inflow traces and the first sum-factorisation stage of the outflow blocks
    for (int idx = ctid; idx < NF * NQF; idx += cnt) {
        const int f = idx / NQF, q = idx - (idx / NQF) * NQF;
        double t = 0.0;
        if ((inm >> f) & 1) {
#pragma unroll
            for (int aa = 0; aa < NFN; ++aa) t += s_trace[q * NFN + aa] * UP[f * NFN + aa];
        } else if ((inm >> (f + 8)) & 1) {
            t = pr.inflow;
        }
        TR[idx] = t * WI[idx];
    }
    if (DIM == 3) {
        for (int idx = ctid; idx < NF * T1SZ; idx += cnt) {
            const int f = idx / T1SZ, rem = idx - f * T1SZ;
            if (!((outm >> f) & 1)) continue;
            const int jq = rem / (N1 * N1), r2 = rem - jq * N1 * N1;
            const int aa = r2 / N1, ab = r2 - aa * N1;
            double s = 0.0;
#pragma unroll
            for (int iq = 0; iq < NQ1; ++iq) s += WQ[f * NQF + jq * NQ1 + iq] * (s_line[iq * N1 + aa] * s_line[iq * N1 + ab]);
            T1[idx] = s;
        }
        pair_sync();
    }
    // phase 3: outflow blocks F_f[(a,b),(a',b')] = sum_ij wq_ij L_a L_a'(s_i) L_b L_b'(t_j)
    for (int idx = ctid; idx < NF * NFN * NFN; idx += cnt) {
        const int f = idx / (NFN * NFN), rem = idx - f * NFN * NFN;
        if (!((outm >> f) & 1)) continue;
        const int fa = rem / NFN, fb = rem - fa * NFN;
        double s = 0.0;
        if (DIM == 3) {
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
    }  // dbg & 1

    const long long t_face = clock64();
    // ------------------------------------------------ assemble into registers
    {
        // face contributions: outflow blocks on (face-node row, face-node column)
        // entries and inflow projections on the rhs column
        int rmask[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int r = ll + L * i;
            rmask[i] = r < N ? s_nmask[r] & outm : 0;
        }
#pragma unroll
        for (int s = 0; s < CW; ++s) {
            const int j = ((s / SB) * W + w) * SB + (s % SB);
            const int cmask = j < N ? s_nmask[j] : 0;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int r = ll + L * i;
                if (r < N && j < N) {
                    int m = rmask[i] & cmask;
                    while (m) {  // outflow blocks of the faces shared by node r and node j
                        const int f = __ffs(m) - 1;
                        m &= m - 1;
                        a[i][s] += FM[f * NFN * NFN + s_fidx[f * N + r] * NFN + s_fidx[f * N + j]];
                    }
                } else if (r < N && j == N) {
                    int m = s_nmask[r] & (inm | (inm >> 8)) & 63;
                    while (m) {
                        const int f = __ffs(m) - 1;
                        m &= m - 1;
                        const int fr = s_fidx[f * N + r];
                        double s2 = 0.0;
                        for (int q = 0; q < NQF; ++q) s2 += TR[f * NQF + q] * s_trace[q * NFN + fr];
                        a[i][s] += s2;
                    }
                }
            }
        }
    }
    if ((int64_t)pair == zero_pair) {
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int s = 0; s < CW; ++s)
                if (((s / SB) * W + w) * SB + (s % SB) < N) a[i][s] = 0.0;
    }
    // matrix scale for the singularity test (stand-in for rcond > 1e-14, solver.hpp:70)
    double amax = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
        for (int s = 0; s < CW; ++s)
            if (((s / SB) * W + w) * SB + (s % SB) < N) amax = fmax(amax, fabs(a[i][s]));
#pragma unroll
    for (int off = L / 2; off > 0; off >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    if (W > 1) {
        if (lane == 0) amx[w] = amax;
        pair_sync();
#pragma unroll
        for (int q = 0; q < W; ++q) amax = fmax(amax, amx[q]);
    }

    const long long t_asm = clock64();
    // ------------------------------------------------ Gauss-Jordan
    // Lookahead 1: inside step k the owner warp of column k+1 updates that
    // column first, searches pivot k+1 and publishes its multipliers before its
    // own bulk update of step k.  W > 1: multipliers travel through an 8-slot
    // SMEM ring with a ready counter (no per-step rendezvous); a named barrier
    // every 4 steps bounds the ring.  Columns <= k are dead after step k, so
    // every warp updates all its slots >= s unconditionally (no predicates).
    double* pivval = psm + G::SM_PIVV;                               // [N] pivot of step k
    int* rowstep = reinterpret_cast<int*>(psm + G::SM_ROWS);        // [N] step where row r pivots
    double* ring = lbuf;                                              // W > 1: [8][L*R + 2]
    volatile int* ready = reinterpret_cast<volatile int*>(amx + W);  // W > 1: last published step
    constexpr int RS = L * R + 2;
    unsigned done = 0;     // bit i: row slot i already pivoted (or padding)
#pragma unroll
    for (int i = 0; i < R; ++i)
        if (ll + L * i >= N) done |= 1u << i;
    bool singular = false;
    const unsigned gbits = PPW > 1 ? (((1u << L) - 1u) << (ps * L)) : 0xffffffffu;
    if (W > 1 && lane == 0 && w == 0) *ready = -1;

    // pivot search on a candidate column (this warp's copy of the rows)
    auto search = [&](const double (&cv)[R], double (&lo)[R], int& prow_o, double& piv_o) {
        if (PPW == 1) {
            // one packed key per lane [|a| high word >> KLB, + 1][row slot][31 - lane]
            // (pivoted rows 0): a single redux.max yields the pivot row; pivot chosen
            // within 2^-14 of max |a| (ties -> higher slot, then lower lane)
            constexpr int KLB = 5 + (R <= 1 ? 0 : R <= 2 ? 1 : R <= 4 ? 2 : 3);
            unsigned key = 0u;
            int ks = 0;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const unsigned hi = (unsigned)(__double_as_longlong(cv[i]) >> 32) & 0x7fffffffu;
                const unsigned kk = ((((hi >> KLB) + 1u) << KLB) | ((unsigned)i << 5) | (31u - ll));
                if (!((done >> i) & 1u) && kk > key) { key = kk; ks = i; }
            }
            double cm = cv[0];
#pragma unroll
            for (int i = 1; i < R; ++i)
                if (i == ks) cm = cv[i];
            const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
            const int src_lane = 31 - (int)(kmax & 31u);
            prow_o = src_lane + 32 * (int)((kmax >> 5) & ((1u << (KLB - 5)) - 1u));
            piv_o = __shfl_sync(0xffffffffu, cm, src_lane);
        } else {
            unsigned key = 0u;
            int ks = 0;
            double cm = cv[0];
#pragma unroll
            for (int i = 0; i < R; ++i) {
                // high word of |a| + 1: every unpivoted row is a candidate, ties -> lowest lane
                const unsigned hi = (unsigned)(__double_as_longlong(fabs(cv[i])) >> 32) + 1u;
                if (!((done >> i) & 1u) && hi > key) { key = hi; ks = i; cm = cv[i]; }
            }
            unsigned kmax = 0u;
#pragma unroll
            for (int pp = 0; pp < PPW; ++pp) {
                const unsigned t = __reduce_max_sync(0xffffffffu, ps == pp ? key : 0u);
                if (ps == pp) kmax = t;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, key == kmax && key != 0u) & gbits;
            const int src_lane = __ffs(bal) - 1;
            prow_o = __shfl_sync(0xffffffffu, ll + L * ks, src_lane);
            piv_o = __shfl_sync(0xffffffffu, cm, src_lane);
        }
        if (!(fabs(piv_o) > 1e-14 * amax)) singular = true;
        const double rinv = 1.0 / piv_o;
#pragma unroll
        for (int i = 0; i < R; ++i) lo[i] = (ll + L * i == prow_o) ? 0.0 : cv[i] * rinv;
    };
    auto produce = [&](int k, const double (&lo)[R], int prow_o, double piv_o) {
        double* slot = ring + (k & 7) * RS;
#pragma unroll
        for (int i = 0; i < R; ++i) slot[ll + L * i] = lo[i];
        if (lane == 0) {
            slot[L * R] = __longlong_as_double((long long)prow_o);
            slot[L * R + 1] = piv_o;
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            *ready = k;
        }
    };
    auto consume = [&](int k, double (&lo)[R], int& prow_o, double& piv_o) {
        while (*ready < k) __nanosleep(8);
        __threadfence_block();
        const double* slot = ring + (k & 7) * RS;
#pragma unroll
        for (int i = 0; i < R; ++i) lo[i] = slot[ll + L * i];
        prow_o = (int)__double_as_longlong(slot[L * R]);
        piv_o = slot[L * R + 1];
    };
    auto mark = [&](int k, int prow_o, double piv_o) {
        if (ll == prow_o % L) done |= 1u << (prow_o / L);
        if (w == 0 && ll == 0) {
            pivval[k] = piv_o;
            rowstep[prow_o] = k;
        }
    };

    double l[R];
    int prow;
    double piv;
    if (W > 1) pair_sync();  // ready initialised
    if (dbg & 2) {
        if (active && w == 0)
            for (int i = 0; i < R; ++i)
                if (ll + L * i < N) psi_out[(rhs_given ? 0 : (size_t)d * psi_stride + (size_t)e * N) + ll + L * i] = a[i][0];
        return;
    }
    if (w == 0) {
        double cv[R];
#pragma unroll
        for (int i = 0; i < R; ++i) cv[i] = a[i][0];
        search(cv, l, prow, piv);
        if (W > 1) produce(0, l, prow, piv);
    }
    if (W > 1 && w != 0) consume(0, l, prow, piv);
    mark(0, prow, piv);

    // step k = ((sb * W + o) * SB + t): block sb of owner warp o, slot sb*SB + t
#pragma unroll
    for (int sb = 0; sb < NBLK; ++sb) {
#pragma unroll 1
        for (int o = 0; o < W; ++o) {
#pragma unroll
            for (int t = 0; t < SB; ++t) {
                const int s = sb * SB + t;
                const int k = (sb * W + o) * SB + t;
                if (k < N) {
                    // publish the pivot row's segment of this warp's blocks >= sb
                    const int pslot = prow / L, plane = prow % L;
#pragma unroll
                    for (int i = 0; i < R; ++i) {
                        if (i == pslot && ll == plane) {
#pragma unroll
                            for (int s2 = sb * SB; s2 < CW; s2 += 2)
                                *reinterpret_cast<double2*>(ubuf + s2) = make_double2(a[i][s2], a[i][s2 + 1]);
                        }
                    }
                    __syncwarp();
                    // block sb (+ the first pair of block sb+1) first: they hold column k+1
                    const int FIRST_END = (sb + 1) * SB + 2 < CW ? (sb + 1) * SB + 2 : CW;
#pragma unroll
                    for (int s2 = sb * SB; s2 < FIRST_END; s2 += 2) {
                        const double2 u2 = *reinterpret_cast<const double2*>(ubuf + s2);
#pragma unroll
                        for (int i = 0; i < R; ++i) {
                            a[i][s2] -= l[i] * u2.x;
                            a[i][s2 + 1] -= l[i] * u2.y;
                        }
                    }
                    const int kn = k + 1;
                    const int own_n = W == 1 ? 0 : (t < SB - 1 ? o : (o + 1 == W ? 0 : o + 1));
                    double ln[R];
                    int prown = 0;
                    double pivn = 1.0;
                    if (kn < N && w == own_n) {
                        double cv[R];
#pragma unroll
                        for (int i = 0; i < R; ++i) {
                            if (t < SB - 1) cv[i] = a[i][s + 1 < CW ? s + 1 : 0];
                            else if (W > 1 && o + 1 < W) cv[i] = a[i][sb * SB];
                            else cv[i] = a[i][(sb + 1) * SB < CW ? (sb + 1) * SB : 0];
                        }
                        search(cv, ln, prown, pivn);
                        if (W > 1) produce(kn, ln, prown, pivn);
                    }
                    // bulk update of the remaining slots with step k
#pragma unroll
                    for (int s2 = FIRST_END; s2 < CW; s2 += 2) {
                        const double2 u2 = *reinterpret_cast<const double2*>(ubuf + s2);
#pragma unroll
                        for (int i = 0; i < R; ++i) {
                            a[i][s2] -= l[i] * u2.x;
                            a[i][s2 + 1] -= l[i] * u2.y;
                        }
                    }
                    __syncwarp();  // ubuf reads complete before the next publication
                    if (kn < N) {
                        if (W > 1 && w != own_n) consume(kn, ln, prown, pivn);
#pragma unroll
                        for (int i = 0; i < R; ++i) l[i] = ln[i];
                        prow = prown;
                        piv = pivn;
                        mark(kn, prow, piv);
                    }
                    if (W > 1 && t == SB - 1) pair_sync();  // bounds the 8-slot multiplier ring
                }
            }
        }
    }
    if (W > 1) pair_sync();
    else __syncwarp();

    const long long t_gj = clock64();
    // ------------------------------------------------ solution x_k = rhs(p_k) / pivot_k
    if (singular && active && ll == 0) atomicMin(err_key, (unsigned long long)pair);
    constexpr int SN = (N / SB) % W, SSLOT = ((N / SB) / W) * SB + N % SB;  // warp / slot of the rhs column
    if (active && w == SN) {
        double* out = rhs_given ? psi_out : psi_out + (size_t)d * psi_stride + (size_t)e * N;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int r = ll + L * i;
            if (r < N) {
                const int kk = rowstep[r];
                out[kk] = a[i][SSLOT] / pivval[kk];
            }
        }
    }
    if ((dbg & 8) && lane == 0 && w == 0 && ps == 0 && active) {
        const long long t_end = clock64();
        atomicAdd(pr.prof + 0, (unsigned long long)(t_tab - t_start));
        atomicAdd(pr.prof + 1, (unsigned long long)(t_face - t_tab));
        atomicAdd(pr.prof + 2, (unsigned long long)(t_asm - t_face));
        atomicAdd(pr.prof + 3, (unsigned long long)(t_gj - t_asm));
        atomicAdd(pr.prof + 4, (unsigned long long)(t_end - t_gj));
        atomicAdd(pr.prof + 5, 1ull);
    }
}

template <int DIM, int P, int W, int PPW>
static void launch_gj(const DevProblem& pr, const double* src, const double* psi_old, const double* psi_new_in,
                      double* psi_out, int64_t stride, const int* pairs, int npairs, const double* rhs_given,
                      unsigned long long* err, int64_t zero_pair, cudaStream_t st) {
    using G = GJ<DIM, P, W, PPW>;
    static_assert(G::NBLK <= 16, "slot blocks exceed the unrolled switch");
    static bool configured = false;
    if (!configured) {
        GCHECK(cudaFuncSetAttribute(gj_sweep_kernel<DIM, P, W, PPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)G::SMEM));
        configured = true;
    }
    const int blocks = (npairs + G::PAIRS_PER_CTA - 1) / G::PAIRS_PER_CTA;
    gj_sweep_kernel<DIM, P, W, PPW><<<blocks, G::THREADS, G::SMEM, st>>>(
        pr, src, psi_old, psi_new_in, psi_out, stride, pairs, npairs, rhs_given, err, zero_pair);
    GCHECK(cudaGetLastError());
}

// (dim, p) -> (W, PPW): lanes own whole rows; W warps split the columns when
// a lane's rows would not fit in registers; PPW pairs share a warp when n is small.
#define GJ_DISPATCH(DIMV, PV, CALL)                                      \
    do {                                                                 \
        if (DIMV == 2) {                                                 \
            switch (PV) {                                                \
                case 1: CALL(2, 1, 1, 8); break;                         \
                case 2: CALL(2, 2, 1, 4); break;                         \
                case 3: CALL(2, 3, 1, 4); break;                         \
                case 4: CALL(2, 4, 1, 2); break;                         \
                case 5: CALL(2, 5, 2, 1); break;                         \
                case 6: CALL(2, 6, 2, 1); break;                         \
                default: throw Error(-1, "unsupported 2D order");       \
            }                                                            \
        } else {                                                         \
            switch (PV) {                                                \
                case 1: CALL(3, 1, 1, 8); break;                         \
                case 2: CALL(3, 2, 1, 2); break;                         \
                case 3: CALL(3, 3, 4, 1); break;                         \
                case 4: CALL(3, 4, 8, 1); break;                         \
                default: throw Error(-1, "unsupported 3D order");       \
            }                                                            \
        }                                                                \
    } while (0)

void dev_gj_sweep(const DevProblem& P, const double* src, const double* psi_old, double* psi_new, int64_t stride,
                  const int* pairs, int npairs, unsigned long long* err_key, int64_t zero_pair, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
#define CALL_GJ(D_, P_, W_, PPW_) \
    launch_gj<D_, P_, W_, PPW_>(P, src, psi_old, psi_new, psi_new, stride, pairs, npairs, nullptr, err_key, zero_pair, st)
    GJ_DISPATCH(P.dim, P.p, CALL_GJ);
#undef CALL_GJ
}

void dev_gj_local_solve(const DevProblem& P, const int* pair_dev, const double* rhs, double* out,
                        unsigned long long* err_key, int64_t zero_pair, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
#define CALL_GJL(D_, P_, W_, PPW_) \
    launch_gj<D_, P_, W_, PPW_>(P, nullptr, nullptr, nullptr, out, 0, pair_dev, 1, rhs, err_key, zero_pair, st)
    GJ_DISPATCH(P.dim, P.p, CALL_GJL);
#undef CALL_GJL
}

int dev_gj_smem(int dim, int p) {
    size_t r = 0;
#define CALL_SM(D_, P_, W_, PPW_) r = GJ<D_, P_, W_, PPW_>::SMEM
    GJ_DISPATCH(dim, p, CALL_SM);
#undef CALL_SM
    return (int)r;
}

}  // namespace hsw
