// K1 sweep kernel, two-warp pairs (3D): TWO warps per (element, ordinate) pair.
//
// Same arithmetic as hsw_dmma1.cu (SweepSolver::sweep's per-element step,
// solver.hpp:104-114: A = sum_k Omega_k G_k + F_out + sigma_t M, rhs = s_e + upwind
// traces, partial-pivot elimination; blocked Gauss-Jordan with DMMA m8n8k4 FP64
// trailing updates, x_k = rhs(p_k) / pivot_k), re-partitioned for the shapes where
// one warp per pair leaves the SM latency-bound (C5: n = 125, 16 x 16 tiles, only
// three one-warp pairs fit an SM).
//
// Ownership.  The augmented matrix's tile-columns alternate between the pair's two
// warps (column c belongs to role c & 1); storage by column range: the first NL in
// shared memory, the next NT in tensor memory, the rest in registers (NRW per warp).
// The two warps of a pair are w and w + PAIRS, PAIRS a multiple of 4, so both map to
// the same TMEM lane quarter: the pair's TMEM tile-columns are one column range of
// that quarter.  Every tile is written only by its owner, so the only cross-warp data
// are the panel multipliers L~ (three buffers), the pivot rows' steps / reciprocal
// pivots, and the face matrices.
//
// Elimination with look-ahead.  Panel Pn lives in tile-column Pn*PW/8 and is factored
// by that column's owner.  After the multipliers of Pn are published, the owner of
// panel Pn+1's column updates that column first, factors Pn+1 and publishes it
// (bar.arrive, no wait), and only then finishes its other updates with Pn; the other
// warp waits for each panel with bar.sync.  So a panel's pivot chain overlaps the
// other warp's trailing updates.  A warp that factors two consecutive panels runs at
// most two panels ahead of the other warp's register copy of an earlier panel's L~,
// so three multiplier buffers suffice.  Each warp gathers the pivot rows (the B
// operand) from its own columns only.
#include "hsw_internal.hpp"

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

namespace hsw {
namespace {

#define D2CHECK(x)                                                                             \
    do {                                                                                       \
        cudaError_t _e = (x);                                                                  \
        if (_e != cudaSuccess)                                                                 \
            throw Error(-8, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #x);       \
    } while (0)

template <int P, int NL_, int NT_, int PAIRS_, bool SP_ = false>
struct D2 {
    static constexpr int PW = 4;                        // panel width (one m8n8k4 k-chunk)
    static constexpr int N1 = P + 1;
    static constexpr int N = N1 * N1 * N1;
    static constexpr int NTR = (N + 7) / 8;             // tile rows
    static constexpr int NTC = (N + 1 + 7) / 8;         // tile columns (rhs = column N)
    static constexpr int NL = NL_;                      // shared-memory tile-columns [0, NL)
    static constexpr int NT = NT_;                      // tensor-memory tile-columns [NL, RB)
    static constexpr int RB = NL + NT;                  // register tile-columns [RB, NTC)
    static constexpr int NRW = (NTC - RB) / 2;          // register tile-columns per warp
    static_assert((NTC - RB) % 2 == 0 && NRW >= 1, "register tile-columns split evenly over the two warps");
    static_assert(NT % 2 == 0, "TMEM tile-columns split evenly over the two warps (role = column parity)");
    static constexpr int TCR = N / 8, QR = (N % 8) / 2, SR = N % 2;   // rhs tile-column / quad column / slot
    static constexpr int RHS_ROLE = TCR & 1;
    static constexpr int JR = (TCR - NL_ - NT_ - ((RHS_ROLE - NL_ - NT_) & 1)) / 2;   // register slot of the rhs column
    static_assert(TCR >= RB, "the rhs tile-column must be register resident");
    static constexpr int PAIRS = PAIRS_;
    static_assert(PAIRS % 4 == 0, "a pair's two warps must share a TMEM lane quarter");
    static constexpr int NBAR = SP_ ? 1 : 3;            // named barriers per pair (the static-pivot form needs one)
    static_assert(1 + NBAR * PAIRS <= 16, "named barriers per pair (ids 1..15)");
    static constexpr int WARPS = 2 * PAIRS;
    static constexpr int THREADS = 32 * WARPS;
    static constexpr int PPQ = PAIRS / 4;               // pairs per TMEM lane quarter
    static constexpr int TCOLS = NT * NTR * 4;          // TMEM columns per pair
    static_assert(NT == 0 || (NTR % 4 == 0 && TCOLS * PPQ <= 512), "TMEM tile-columns do not fit");
    static constexpr int NR = 8 * NTR;
    static constexpr int RP = (NR + 31) / 32;           // panel rows per lane (row layout)
    static constexpr int NPANEL = (N + PW - 1) / PW;
    static constexpr int NFN = N1 * N1, NF = 6, NQ1 = P + 2, NQF = NQ1 * NQ1;
    static constexpr int T1SZ = NQ1 * N1 * N1;
    static constexpr int NSF = NFN * (NFN + 1) / 2, NS1 = N1 * (N1 + 1) / 2;
    // per-pair shared memory (doubles)
    static constexpr int SM_AL = 0;                                   // [NL][NTR][32][2]
    static constexpr int SM_X = SM_AL + NL * NTR * 64;                // union: faces | elimination
    static constexpr int SM_WQ = SM_X;                                // [NF][NQF] signed (Omega.n) w|J|
    static constexpr int SM_UP = SM_WQ + NF * NQF;                    // [NF][NFN] upwind values / projections
    static constexpr int SM_TR = SM_UP + NF * NFN;                    // [NF][NQF] inflow traces * weight
    static constexpr int SM_T1 = SM_TR + NF * NQF;                    // [2 roles][T1SZ]
    static constexpr int FMS = NFN + 1;
    static constexpr int SM_F = SM_T1 + 2 * T1SZ;                     // [2 face parities][NFN][FMS]
    static constexpr int FACE_END = SM_F + 2 * NFN * FMS;
    static constexpr int LPS = NR + (4 - NR % 16 + 16) % 16;           // = 4 (mod 16)
    static constexpr int NOWN = (NT + 1) / 2 + NRW;                   // TMEM + register tile-columns of a warp (max)
    static constexpr int URS = 8 * NOWN + (4 - (8 * NOWN) % 16 + 16) % 16;
    static constexpr int LPB = (NR * PW > PW * LPS ? NR * PW : PW * LPS);   // one multiplier buffer (panel overlay)
    // three multiplier buffers: a panel's producer can be two panels ahead of the other
    // warp's read of an earlier panel's multipliers (see the kernel header)
    static constexpr int NLP = 3;
    static constexpr int SM_LP = SM_X;                                // [NLP][LPB]
    static constexpr int SM_UR = SM_LP + NLP * LPB;                   // [2 roles][PW][URS]
    static constexpr int SM_PIVV = SM_UR + 2 * PW * URS;              // [N]
    static constexpr int SM_ROWS = SM_PIVV + N;                       // [N] ints
    static constexpr int SM_PST = SM_ROWS + (N + 1) / 2;              // [NLP][PW] ints
    static constexpr int ELIM_END = SM_PST + (NLP * PW + 1) / 2;
    // static-pivot two-warp left-looking LU (SP): the negated inverse diagonal tiles, two tile
    // transposition buffers per warp, the published -L~ tiles of the register tile-columns, the
    // rhs / solution vector
    static constexpr int XIS = 10;
    static constexpr int SM_XI = SM_X;                                // [NTR][8][XIS]
    static constexpr int SM_TB = SM_XI + NTR * 8 * XIS;               // [2 roles][2][8][XIS]
    static constexpr int LRR = NTR - 1 - RB > 0 ? NTR - 1 - RB : 1;   // tile rows below the first register diagonal
    static constexpr int LRC = NTC - 1 - RB > 0 ? NTC - 1 - RB : 1;   // register tile-columns with tiles below
    static constexpr int SM_LR = SM_TB + 2 * 2 * 8 * XIS;             // [LRC][LRR][32][2]
    static constexpr int SM_YX = SM_LR + LRC * LRR * 64;              // [NR]
    static constexpr int LL_END = SM_YX + NR;
    static constexpr int EL_END = SP_ ? LL_END : ELIM_END;
    static constexpr int X_END = FACE_END > EL_END ? FACE_END : EL_END;
    static constexpr int SM_PAIR = (X_END + 4) & ~1;                  // + the claimed pair index and the column counter
    static constexpr int TAB_INTS = NF * N + (N + 3) / 4 + NF * NFN + NSF + NS1;
    static constexpr int TAB_TRACE = ((TAB_INTS + 1) / 2 + 1) & ~1;
    static constexpr int TRS = NFN + (2 - NFN % 16 + 16) % 16;
    static constexpr int TAB_TOTAL = (TAB_TRACE + NQF * TRS + NQ1 * N1 + NQ1 * N1 * N1 + 1) & ~1;
    static constexpr size_t SMEM = (size_t)(TAB_TOTAL + PAIRS * SM_PAIR) * sizeof(double);
};

__device__ __forceinline__ void mma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void tm_ld16(uint32_t a, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(a));
}
__device__ __forceinline__ void tm_ld4(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void tm_st16(uint32_t a, const uint32_t (&r)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
template <int K>
__device__ __forceinline__ void tm_pin(uint32_t (&r)[K]) {
#pragma unroll
    for (int i = 0; i < K; ++i) asm volatile("" : "+r"(r[i]));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st_shared_v2_if(double* p, double x, double y, bool on) {
    asm volatile("{\n .reg .pred q;\n setp.ne.s32 q, %3, 0;\n @q st.shared.v2.f64 [%0], {%1, %2};\n}"
                 ::"r"((uint32_t)__cvta_generic_to_shared(p)), "d"(x), "d"(y), "r"((int)on) : "memory");
}
__device__ __forceinline__ double u2d(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }
// 4 tile fragments (8 doubles) of TMEM: load + wait + pairing in ONE asm statement, so the
// compiler sees doubles (no register moves re-pairing the b32 halves, no pins after the wait)
__device__ __forceinline__ void tm_ld16w(uint32_t a, double (&v)[8]) {
    asm volatile("{\n .reg .b32 t<16>;\n"
                 " tcgen05.ld.sync.aligned.32x32b.x16.b32 {t0,t1,t2,t3,t4,t5,t6,t7,t8,t9,t10,t11,t12,t13,t14,t15}, [%8];\n"
                 " tcgen05.wait::ld.sync.aligned;\n"
                 " mov.b64 %0, {t0,t1};\n mov.b64 %1, {t2,t3};\n mov.b64 %2, {t4,t5};\n mov.b64 %3, {t6,t7};\n"
                 " mov.b64 %4, {t8,t9};\n mov.b64 %5, {t10,t11};\n mov.b64 %6, {t12,t13};\n mov.b64 %7, {t14,t15};\n}"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
                 : "r"(a) : "memory");
}
__device__ __forceinline__ void tm_st16w(uint32_t a, const double (&v)[8]) {
    asm volatile("{\n .reg .b32 t<16>;\n"
                 " mov.b64 {t0,t1}, %1;\n mov.b64 {t2,t3}, %2;\n mov.b64 {t4,t5}, %3;\n mov.b64 {t6,t7}, %4;\n"
                 " mov.b64 {t8,t9}, %5;\n mov.b64 {t10,t11}, %6;\n mov.b64 {t12,t13}, %7;\n mov.b64 {t14,t15}, %8;\n"
                 " tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {t0,t1,t2,t3,t4,t5,t6,t7,t8,t9,t10,t11,t12,t13,t14,t15};\n}"
                 ::"r"(a), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]), "d"(v[4]), "d"(v[5]), "d"(v[6]), "d"(v[7])
                 : "memory");
}
// one x4 fragment (2 doubles) from each of 4 TMEM column addresses, one wait
__device__ __forceinline__ void tm_ld4x4w(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, double (&v)[8]) {
    asm volatile("{\n .reg .b32 t<16>;\n"
                 " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t0,t1,t2,t3}, [%8];\n"
                 " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t4,t5,t6,t7}, [%9];\n"
                 " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t8,t9,t10,t11}, [%10];\n"
                 " tcgen05.ld.sync.aligned.32x32b.x4.b32 {t12,t13,t14,t15}, [%11];\n"
                 " tcgen05.wait::ld.sync.aligned;\n"
                 " mov.b64 %0, {t0,t1};\n mov.b64 %1, {t2,t3};\n mov.b64 %2, {t4,t5};\n mov.b64 %3, {t6,t7};\n"
                 " mov.b64 %4, {t8,t9};\n mov.b64 %5, {t10,t11};\n mov.b64 %6, {t12,t13};\n mov.b64 %7, {t14,t15};\n}"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3) : "memory");
}
// named barriers of a pair (64 threads: its two warps)
__device__ __forceinline__ void pbar_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void pbar_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }

template <int P, int NL_, int NT_, int PAIRS_, bool SP_ = false>
__global__ void __launch_bounds__(64 * PAIRS_, 1)
dmma2_sweep_kernel(const DevProblem pr, const double* __restrict__ src, const double* __restrict__ psi_old,
                   const double* psi_new_in, double* psi_out, int64_t psi_stride, const int* __restrict__ pairs,
                   int npairs, const double* __restrict__ rhs_given, unsigned long long* err_key, int64_t zero_pair,
                   unsigned* done_flags, unsigned epoch) {
    using G = D2<P, NL_, NT_, PAIRS_, SP_>;
    constexpr int PW = G::PW, N = G::N, NTR = G::NTR, NL = G::NL, NT = G::NT, RB = G::RB, NRW = G::NRW;
    constexpr int NR = G::NR, RP = G::RP, NPANEL = G::NPANEL, TCR = G::TCR, QR = G::QR, SR = G::SR;
    constexpr int NFN = G::NFN, NF = G::NF, NQ1 = G::NQ1, NQF = G::NQF, N1 = G::N1, NSF = G::NSF, NS1 = G::NS1;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int KLB = 5 + (RP <= 1 ? 0 : RP <= 2 ? 1 : RP <= 4 ? 2 : 3);
    extern __shared__ double smem[];
    __shared__ uint32_t s_tmem_base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q = lane & 3;
    const int role = warp / G::PAIRS;          // 0 or 1: owns the tile-columns c with (c & 1) == role
    const int ps = warp % G::PAIRS;            // pair slot of the CTA
    const bool rhs_owner = role == G::RHS_ROLE;
    // named barrier ids of this pair: 1 + 3 ps + {0: pair start, each outflow face block, faces
    // done (both sync); 1, 2: panel parity 0 / 1 (the producer arrives, the other syncs)}
    const int bid = 1 + G::NBAR * ps;
    if (NT > 0) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&s_tmem_base)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
    }
    int* s_fidx = reinterpret_cast<int*>(smem);
    unsigned char* s_nmask = reinterpret_cast<unsigned char*>(s_fidx + NF * N);
    int* s_fnode = s_fidx + NF * N + (N + 3) / 4;
    int* s_tri = s_fnode + NF * NFN;
    int* s_tri1 = s_tri + NSF;
    double* s_trace = smem + G::TAB_TRACE;
    double* s_line = s_trace + NQF * G::TRS;
    double* s_l2 = s_line + NQ1 * N1;
    for (int idx = threadIdx.x; idx < NF * N; idx += G::THREADS) s_fidx[idx] = __ldg(pr.g_fidx + (idx / N) * 128 + idx % N);
    for (int idx = threadIdx.x; idx < N; idx += G::THREADS) s_nmask[idx] = (unsigned char)__ldg(pr.g_nmask + idx);
    if (threadIdx.x == 0) {
        int k = 0;
        for (int a = 0; a < NFN; ++a)
            for (int b = a; b < NFN; ++b) s_tri[k++] = a | (b << 8);
        k = 0;
        for (int a = 0; a < N1; ++a)
            for (int b = a; b < N1; ++b) s_tri1[k++] = a | (b << 8);
    }
    for (int idx = threadIdx.x; idx < NF * NFN; idx += G::THREADS)
        s_fnode[idx] = __ldg(pr.g_fnode + (idx / NFN) * kMaxFaceNodes + idx % NFN);
    for (int idx = threadIdx.x; idx < NQF * NFN; idx += G::THREADS)
        s_trace[(idx / NFN) * G::TRS + idx % NFN] = __ldg(pr.g_trace + (idx / NFN) * kMaxFaceNodes + idx % NFN);
    for (int idx = threadIdx.x; idx < NQ1 * N1; idx += G::THREADS) s_line[idx] = __ldg(pr.g_line + (idx / N1) * 8 + idx % N1);
    for (int idx = threadIdx.x; idx < NQ1 * N1 * N1; idx += G::THREADS) {
        const int iq = idx / (N1 * N1), ab = idx % (N1 * N1);
        s_l2[idx] = __ldg(pr.g_line + iq * 8 + ab / N1) * __ldg(pr.g_line + iq * 8 + ab % N1);
    }
    __syncthreads();
    if (NT > 0) asm volatile("tcgen05.fence::after_thread_sync;");
    // the pair's TMEM: lane quarter ps % 4, column range (ps / 4) * TCOLS
    const uint32_t tmw = NT > 0 ? s_tmem_base + ((uint32_t)(32 * (ps & 3)) << 16) + (uint32_t)((ps >> 2) * G::TCOLS) : 0u;
    auto tm_get4 = [&](int tt, int grp, double (&v)[4][2]) {
        tm_wait_st();
        tm_ld16w(tmw + (uint32_t)((tt * NTR + 4 * grp) * 4), *reinterpret_cast<double (*)[8]>(&v[0][0]));
    };
    auto tm_put4 = [&](int tt, int grp, const double (&v)[4][2]) {
        tm_st16w(tmw + (uint32_t)((tt * NTR + 4 * grp) * 4), *reinterpret_cast<const double (*)[8]>(&v[0][0]));
    };

    double* psm = smem + G::TAB_TOTAL + (size_t)ps * G::SM_PAIR;
    const int lsw = lane ^ ((lane >> 3) & 3);
    double* AL = psm + G::SM_AL;
    double* WQ = psm + G::SM_WQ;
    double* UP = psm + G::SM_UP;
    double* TR = psm + G::SM_TR;
    double* T1 = psm + G::SM_T1;
    double* FM = psm + G::SM_F;
    double* UR = psm + G::SM_UR + role * PW * G::URS;    // own pivot rows (TMEM and register columns)
    double* pivval = psm + G::SM_PIVV;
    int* rowstep = reinterpret_cast<int*>(psm + G::SM_ROWS);
    int* s_pst = reinterpret_cast<int*>(psm + G::SM_PST);  // [NLP][PW]
    int* s_claim = reinterpret_cast<int*>(psm + G::SM_PAIR - 1);
    // (SP) finished tile-columns of the pair: column k's owner publishes k + 1
    volatile int* ndone = reinterpret_cast<volatile int*>(psm + G::SM_PAIR - 2);
    if (SP_ && role == 0 && lane == 0) *ndone = 0;
    // own tile-columns: storage index of column c of this role
    // TMEM: tt = c - NL; own TMEM columns c = NL + t0 + 2 i, t0 = (NL ^ role) & 1 parity fix
    // role w owns the columns of parity w: SMEM columns w, w + 2, ...; TMEM columns NL + tt,
    // tt = t0, t0 + 2, ...; register columns RB + r0 + 2 j
    const int l0 = role, t0 = (role - NL) & 1, r0 = (role - RB) & 1;
    constexpr int NTOWN = NT / 2;
    auto owner_of = [](int c) { return c & 1; };
    unsigned* claim = done_flags ? done_flags + (size_t)pr.nel * pr.nd + 1 : nullptr;
    int pidx_next = blockIdx.x * G::PAIRS + ps;

    for (;;) {
        // ------------------------------------------------ claim (role 0), shared with role 1
        if (role == 0) {
            int pi;
            if (claim) {
                unsigned c = 0;
                if (lane == 0) c = atomicAdd(claim, 1u);
                pi = (int)__shfl_sync(FULL, c, 0);
            } else {
                pi = pidx_next;
                pidx_next += gridDim.x * G::PAIRS;
            }
            if (lane == 0) *s_claim = pi;
        }
        pbar_sync(bid);   // pair start: the previous pair is finished by both warps, the claim is visible
        const int pidx = *s_claim;
        if (pidx >= npairs) break;
        const int pair = pairs[pidx];
        const int e = pair / pr.nd, d = pair - (pair / pr.nd) * pr.nd;
        const double om0 = pr.omega[d * 4 + 0], om1 = pr.omega[d * 4 + 1], om2 = pr.omega[d * 4 + 2];
        const double amax = pr.bscale[e];
        const int iex = SP_ ? ilogb(amax > 0.0 ? amax : 1.0) : 0;
        const double isc = scalbn(1.0, -iex), iun = scalbn(1.0, iex);   // power of two ~ 1 / amax; isc * iun == 1
        if (role == 0 && !(pr.tune & 1)) {   // TMA L2 prefetch of the pair's element tensor
            constexpr unsigned TB = (unsigned)(t_elem_doubles(N) * sizeof(double));
            constexpr unsigned CH = 32768u;
            const char* tb = reinterpret_cast<const char*>(pr.T) + (size_t)e * TB;
            if (lane < (int)((TB + CH - 1) / CH)) {
                const unsigned off = (unsigned)lane * CH, sz = TB - off < CH ? TB - off : CH;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tb + off), "r"(sz) : "memory");
            }
        }

        // ------------------------------------------------ volume terms of the own tile-columns
        double acc[NRW][NTR][2];
        {
            const double st = pr.sig_t[e];
            const double2* Te = reinterpret_cast<const double2*>(pr.T) + (size_t)e * (t_elem_doubles(N) / 2);
            const double* se = rhs_given ? rhs_given : src + (size_t)e * N;
            auto tload = [&](int r, int c) -> double4 {
                const double2 a = __ldg(Te + t_idx2(N, r, c, 0)), b = __ldg(Te + t_idx2(N, r, c, 1));
                return make_double4(a.x, a.y, b.x, b.y);
            };
            auto comb = [&](const double4 t) { return om0 * t.y + om1 * t.z + om2 * t.w + st * t.x; };
            auto vol = [&](int r, int c) -> double {
                if (r < N && c < N) return comb(tload(r, c));
                if (c == N) {
                    const double sv = se[r < N ? r : N - 1];
                    return r < N ? sv : 0.0;
                }
                return 0.0;
            };
            for (int tl = l0; tl < NL; tl += 2) {
#pragma unroll 4
                for (int tr = 0; tr < NTR; ++tr) {
                    const int r = 8 * tr + g, c = 8 * tl + 2 * q;
                    *reinterpret_cast<double2*>(AL + ((tl * NTR + tr) * 32 + lsw) * 2) = make_double2(vol(r, c), vol(r, c + 1));
                }
            }
            if (NT > 0) {
                constexpr int GPC = NTR / 4;
                auto ldgrp = [&](int tt, int grp, double4 (&b)[4][2]) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int s2 = 0; s2 < 2; ++s2) {
                            const int r = 8 * (4 * grp + k) + g, c = 8 * (NL + tt) + 2 * q + s2;
                            b[k][s2] = (r < N && c < N) ? tload(r, c) : make_double4(0.0, 0.0, 0.0, 0.0);
                        }
                };
                auto combine = [&](int tt, int grp, const double4 (&b)[4][2]) {
                    double v[4][2];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
#pragma unroll
                        for (int s2 = 0; s2 < 2; ++s2) {
                            const int r = 8 * (4 * grp + k) + g, c = 8 * (NL + tt) + 2 * q + s2;
                            v[k][s2] = r < N && c < N ? comb(b[k][s2]) : (r < N && c == N ? se[r] : 0.0);
                        }
                    tm_put4(tt, grp, v);
                };
                constexpr int NGR = NTOWN * GPC;
                auto gi_tt = [&](int gi) { return t0 + 2 * (gi / GPC); };
                if (G::PAIRS >= 8) {
                    // many warps, 128 registers: one group in flight
#pragma unroll 1
                    for (int gi = 0; gi < NGR; ++gi) {
                        double4 b[4][2];
                        ldgrp(gi_tt(gi), gi % GPC, b);
                        combine(gi_tt(gi), gi % GPC, b);
                    }
                } else {
                    // loads one group ahead, two groups per (rolled) iteration: a small code
                    // footprint (eight warps per SM share the instruction cache).  Two groups ahead
                    // (three 64-register buffers) spills in this loop: C5 1501 vs 766 ms.
                    double4 b0[4][2], b1[4][2];
                    ldgrp(gi_tt(0), 0, b0);
#pragma unroll 1
                    for (int gi = 0; gi < NGR; gi += 2) {
                        if (gi + 1 < NGR) ldgrp(gi_tt(gi + 1), (gi + 1) % GPC, b1);
                        combine(gi_tt(gi), gi % GPC, b0);
                        if (gi + 2 < NGR) ldgrp(gi_tt(gi + 2), (gi + 2) % GPC, b0);
                        if (gi + 1 < NGR) combine(gi_tt(gi + 1), (gi + 1) % GPC, b1);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NRW; ++j)
#pragma unroll
                for (int tr = 0; tr < NTR; ++tr)
#pragma unroll
                    for (int s = 0; s < 2; ++s) acc[j][tr][s] = vol(8 * tr + g, 8 * (RB + r0 + 2 * j) + 2 * q + s);
        }

        // ------------------------------------------------ faces
        const unsigned inflags = rhs_given ? 0u : pr.inflags[(size_t)d * pr.nel + e];
        int outm = 0, inm = 0;
        {
            constexpr int KG = (NF * NQF + 31) / 32, KU = (NF * NFN + 31) / 32;
            double4 gmv[KG];
#pragma unroll
            for (int k = 0; k < KG; ++k) {
                const int idx = lane + 32 * k;
                if (idx < NF * NQF) gmv[k] = reinterpret_cast<const double4*>(pr.fgeom)[(size_t)e * NF * NQF + idx];
            }
            // both warps: the signed face weights (identical values) and the outflow mask
#pragma unroll
            for (int k = 0; k < KG; ++k) {
                const int idx = lane + 32 * k;
                if (idx < NF * NQF) {
                    const double4 gm = gmv[k];
                    const double on = om0 * gm.x + om1 * gm.y + om2 * gm.z;
                    const double onw = on * gm.w;
                    WQ[idx] = onw;
                    if (on > 0.0 && onw != 0.0) outm |= 1 << (idx / NQF);
                }
            }
            outm = (int)__reduce_or_sync(FULL, (unsigned)outm);
            if (rhs_owner) {
                // inflow: dataflow wait, upwind gathers, traces, projections, rhs adds
                int4 nbv[KU];
#pragma unroll
                for (int k = 0; k < KU; ++k) {
                    const int idx = lane + 32 * k;
                    if (idx < NF * NFN) nbv[k] = reinterpret_cast<const int4*>(pr.fnbr)[(size_t)e * NF + idx / NFN];
                }
                if (done_flags) {
                    if (lane < NF && ((inflags >> (2 * lane)) & 3u) == 1u) {
                        const int nb = reinterpret_cast<const int4*>(pr.fnbr)[(size_t)e * NF + lane].x;
                        const unsigned* fl = done_flags + (size_t)nb * pr.nd + d;
                        unsigned v;
                        const long long t_wait = clock64();
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
                        while (v != epoch) {
                            __nanosleep(64);
                            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
                            if (v == epoch) {
                                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(fl) : "memory");
                                break;
                            }
                            if (clock64() - t_wait > (1ll << 34)) {
                                atomicExch(done_flags + (size_t)pr.nel * pr.nd, 1u);
                                break;
                            }
                        }
                    }
                    __syncwarp();
                }
#pragma unroll
                for (int k = 0; k < KU; ++k) {
                    const int idx = lane + 32 * k;
                    const int f = idx / NFN, aa = idx - (idx / NFN) * NFN;
                    double u = 0.0;
                    if (idx < NF * NFN && ((inflags >> (2 * f)) & 1u)) {
                        const int4 nb4 = nbv[k];
                        const bool lag = (inflags >> (2 * f + 1)) & 1u;
                        const double* sp = (lag ? psi_old : psi_new_in) + (size_t)d * psi_stride + (size_t)nb4.x * N;
                        const int a0 = aa % N1, b0 = aa / N1, code = nb4.z;
                        int uu = a0, vv = b0;
                        if (code & 4) { uu = b0; vv = a0; }
                        if (code & 2) uu = P - uu;
                        if (code & 1) vv = P - vv;
                        u = __ldcg(sp + s_fnode[nb4.y * NFN + vv * N1 + uu]);
                        inm |= 1 << f;
                    } else if (idx < NF * NFN && !rhs_given && nbv[k].x < 0 && pr.inflow != 0.0) {
                        inm |= 1 << (f + 8);
                    }
                    if (idx < NF * NFN) UP[idx] = u;
                }
                inm = (int)__reduce_or_sync(FULL, (unsigned)inm);
                __syncwarp();
                const int infm = (inm | (inm >> 8)) & 63;
                const int nin = __popc(infm);
                auto nth_face = [&](int sl) {
                    int m = infm;
                    for (int i = 0; i < sl; ++i) m &= m - 1;
                    return __ffs(m) - 1;
                };
                for (int idx = lane; idx < nin * NQF; idx += 32) {
                    const int sl = idx / NQF, qq = idx - sl * NQF;
                    const int f = nth_face(sl);
                    double t = pr.inflow;
                    if ((inm >> f) & 1) {
                        t = 0.0;
#pragma unroll 5
                        for (int aa = 0; aa < NFN; ++aa) t += s_trace[qq * G::TRS + aa] * UP[f * NFN + aa];
                    }
                    TR[sl * NQF + qq] = t * fmax(-WQ[f * NQF + qq], 0.0);
                }
                __syncwarp();
                for (int idx = lane; idx < nin * NFN; idx += 32) {
                    const int sl = idx / NFN, a = idx - sl * NFN;
                    double t = 0.0;
#pragma unroll 6
                    for (int qq = 0; qq < NQF; ++qq) t += TR[sl * NQF + qq] * s_trace[qq * G::TRS + a];
                    UP[idx] = t;
                }
                __syncwarp();
                if (infm && q == QR) {   // the rhs lanes: a short data-dependent loop per row
#pragma unroll
                    for (int tr = 0; tr < NTR; ++tr) {
                        const int r = 8 * tr + g;
                        int m = r < N ? s_nmask[r] & infm : 0;
                        while (m) {
                            const int f = __ffs(m) - 1;
                            m &= m - 1;
                            acc[G::JR][tr][SR] += UP[__popc(infm & ((1 << f) - 1)) * NFN + s_fidx[f * N + r]];
                        }
                    }
                }
            }
            // outflow blocks: both warps form half of each face's block (double-buffered by
            // face parity; the first stage T1 privately), one barrier, then each adds it to
            // its own tile-columns
            const int nout = __popc(outm);
            int om = outm;
            for (int k = 0; k < nout; ++k) {
                const int f = __ffs(om) - 1;
                om &= om - 1;
                double* T1w = T1 + role * G::T1SZ;
                double* FMk = FM + (k & 1) * NFN * G::FMS;
                {
                    for (int idx = lane; idx < NQ1 * NS1; idx += 32) {
                        const int jq = idx / NS1;
                        const int tri = s_tri1[idx - jq * NS1];
                        const int aa = tri & 255, ab = tri >> 8;
                        double t = 0.0;
#pragma unroll
                        for (int iq = 0; iq < NQ1; ++iq) t += fmax(WQ[f * NQF + jq * NQ1 + iq], 0.0) * s_l2[(iq * N1 + aa) * N1 + ab];
                        T1w[(jq * N1 + aa) * N1 + ab] = t;
                        T1w[(jq * N1 + ab) * N1 + aa] = t;
                    }
                    __syncwarp();
                    for (int idx = 2 * lane + role; idx < NSF; idx += 64) {
                        const int tri = s_tri[idx];
                        const int fa = tri & 255, fb = tri >> 8;
                        const int a0 = fa % N1, b0 = fa / N1, a1 = fb % N1, b1 = fb / N1;
                        double t = 0.0;
#pragma unroll
                        for (int jq = 0; jq < NQ1; ++jq) t += T1w[(jq * N1 + a0) * N1 + a1] * s_l2[(jq * N1 + b0) * N1 + b1];
                        FMk[fa * G::FMS + fb] = t;
                        FMk[fb * G::FMS + fa] = t;
                    }
                }
                pbar_sync(bid);   // the block is complete (and the other warp is past face k - 1)
                int rf[NTR];
#pragma unroll
                for (int tr = 0; tr < NTR; ++tr) {
                    const int r = 8 * tr + g;
                    rf[tr] = r < N ? s_fidx[f * N + r] * G::FMS : -1;
                }
#pragma unroll
                for (int j = 0; j < NRW; ++j)
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        const int c = 8 * (RB + r0 + 2 * j) + 2 * q + s;
                        const int cf = c < N ? s_fidx[f * N + c] : -1;
                        if (__any_sync(FULL, cf >= 0)) {
#pragma unroll
                            for (int tr = 0; tr < NTR; ++tr)
                                if (cf >= 0 && rf[tr] >= 0) acc[j][tr][s] += FMk[rf[tr] + cf];
                        }
                    }
                for (int tl = l0; tl < NL; tl += 2)
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        const int cf = s_fidx[f * N + 8 * tl + 2 * q + s];
                        if (__any_sync(FULL, cf >= 0)) {
#pragma unroll
                            for (int tr = 0; tr < NTR; ++tr)
                                if (cf >= 0 && rf[tr] >= 0) AL[((tl * NTR + tr) * 32 + lsw) * 2 + s] += FMk[rf[tr] + cf];
                        }
                    }
                for (int tt = t0; tt < NT; tt += 2) {
                    const int c0 = 8 * (NL + tt) + 2 * q;
                    const int cf0 = c0 < N ? s_fidx[f * N + c0] : -1, cf1 = c0 + 1 < N ? s_fidx[f * N + c0 + 1] : -1;
                    if (__any_sync(FULL, cf0 >= 0 || cf1 >= 0)) {
#pragma unroll
                        for (int grp = 0; grp < NTR / 4; ++grp) {
                            double v[4][2];
                            tm_get4(tt, grp, v);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const int rr = rf[4 * grp + kk];
                                if (rr >= 0 && cf0 >= 0) v[kk][0] += FMk[rr + cf0];
                                if (rr >= 0 && cf1 >= 0) v[kk][1] += FMk[rr + cf1];
                            }
                            tm_put4(tt, grp, v);
                        }
                    }
                }
                __syncwarp();
            }
        }
        if ((int64_t)pair == zero_pair) {   // test hook: zero the (e, d) block (own columns)
#pragma unroll
            for (int j = 0; j < NRW; ++j)
#pragma unroll
                for (int tr = 0; tr < NTR; ++tr)
#pragma unroll
                    for (int s = 0; s < 2; ++s)
                        if (8 * (RB + r0 + 2 * j) + 2 * q + s < N) acc[j][tr][s] = 0.0;
            for (int tl = l0; tl < NL; tl += 2)
                for (int i = lane * 2; i < NTR * 64; i += 64) AL[tl * NTR * 64 + i] = AL[tl * NTR * 64 + i + 1] = 0.0;
            for (int tt = t0; tt < NT; tt += 2)
                for (int grp = 0; grp < NTR / 4; ++grp) {
                    const double z[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
                    tm_put4(tt, grp, z);
                }
        }
        __syncwarp();
        // faces done by both warps: the face scratch becomes the elimination buffers
        pbar_sync(bid);
        if (!SP_ && owner_of(0) == role) {   // the first factoring warp; the other reads steps only after a panel barrier
            for (int r = lane; r < N; r += 32) rowstep[r] = -1;
            __syncwarp();
        }

        if constexpr (SP_) {
        // ------------------------------------------------ static-pivot tile LU, left-looking, two warps
        // A = L~ U over the 8x8 tiles (U unscaled, L~_ik = A_ik A_kk^-1; see the one-warp form in
        // hsw_dmma1.cu).  A warp works through its OWN tile-columns in increasing order: column k is
        // read once, receives c_i -= L~_ij U_jk for every finished column j < k in registers (the -L~
        // tiles of the other warp's columns come from shared memory / TMEM, those of its register
        // columns from the Lr buffer), its diagonal tile is inverted, the -L~ tiles below are formed
        // and stored, and k + 1 is published in `ndone`.  Columns finish strictly in order, so the
        // only wait is for the latest column of the other warp, and everything older is applied
        // before that wait: a column's critical section is one update step, one tile inversion and
        // the L~ tiles.  No row searches, no pivot-row gathers, 2/3 n^3 flops.
        {
            constexpr int XIS = G::XIS, NTC = G::NTC, LRR = G::LRR;
            constexpr bool TAILC = N % 8 != 0;
            static_assert(NTR % 4 == 0, "two-warp static-pivot LU: whole 4-tile groups");
            double* Xi = psm + G::SM_XI;
            double* Tb = psm + G::SM_TB + role * (2 * 8 * XIS);
            double* Lr = psm + G::SM_LR;
            double* yx = psm + G::SM_YX;
            unsigned xmaxh = 0u;
            int tbsel = 0;
            auto tb_put = [&](double p0, double p1) {
                *reinterpret_cast<double2*>(Tb + tbsel + g * XIS + 2 * q) = make_double2(p0, p1);
            };
            auto tb_get = [&](double& b0, double& b1) {
                __syncwarp();
                b0 = Tb[tbsel + (2 * q) * XIS + g];
                b1 = Tb[tbsel + (2 * q + 1) * XIS + g];
                tbsel ^= 8 * XIS;
            };
            auto st4 = [&](uint32_t a, double v0, double v1) {
                asm volatile("{\n .reg .b32 t<4>;\n mov.b64 {t0,t1}, %1;\n mov.b64 {t2,t3}, %2;\n"
                             " tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {t0,t1,t2,t3};\n}" ::"r"(a), "d"(v0), "d"(v1) : "memory");
            };
            // tile (tr, k) of an own column k < RB
            auto home_store = [&](int tr, int k, double v0, double v1) {
                if (k < NL) *reinterpret_cast<double2*>(AL + ((k * NTR + tr) * 32 + lsw) * 2) = make_double2(v0, v1);
                else st4(tmw + (uint32_t)(((k - NL) * NTR + tr) * 4), v0, v1);
            };
            auto lr_tile = [&](int c, int tr) { return Lr + (((c - RB) * LRR + (tr - RB - 1)) * 32 + lane) * 2; };
            double c[NTR][2];
#pragma unroll 1
            for (int k = role; k < NTC; k += 2) {
                // (1) the column
                if (k < NL) {
#pragma unroll
                    for (int tr = 0; tr < NTR; ++tr) {
                        const double2 v = *reinterpret_cast<const double2*>(AL + ((k * NTR + tr) * 32 + lsw) * 2);
                        c[tr][0] = v.x;
                        c[tr][1] = v.y;
                    }
                } else if (k < RB) {
#pragma unroll
                    for (int grp = 0; grp < NTR / 4; ++grp) {
                        double v[4][2];
                        tm_get4(k - NL, grp, v);
#pragma unroll
                        for (int k4 = 0; k4 < 4; ++k4) {
                            c[4 * grp + k4][0] = v[k4][0];
                            c[4 * grp + k4][1] = v[k4][1];
                        }
                    }
                } else {
                    static_row<0, NRW>((k - RB - r0) >> 1, [&](auto J_) {
                        constexpr int jr = decltype(J_)::value;
#pragma unroll
                        for (int tr = 0; tr < NTR; ++tr) {
                            c[tr][0] = acc[jr][tr][0];
                            c[tr][1] = acc[jr][tr][1];
                        }
                    });
                }
                // (2) left-looking updates with the finished columns j < k
                if (k > 0) {
                    double b0, b1;
                    tb_put(c[0][0], c[0][1]);   // row 0 never changes: U_0k as assembled
                    tb_get(b0, b1);
#pragma unroll 1
                    for (int j = 0; j < k; ++j) {
                        if ((j ^ role) & 1) {   // the other warp's column: published?
                            if (*ndone <= j) {
                                const long long t_wait = clock64();
                                while (*ndone <= j) {
                                    // ~4 s without the other warp's column: flag it instead of hanging
                                    if (clock64() - t_wait > (1ll << 33)) {
                                        if (done_flags) atomicExch(done_flags + (size_t)pr.nel * pr.nd, 1u);
                                        else atomicMin(err_key, (unsigned long long)pair);   // level launches: fail loudly too
                                        break;
                                    }
                                }
                            }
                            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                            __threadfence_block();
                            __syncwarp();
                        }
                        const bool more = j + 1 < k;
                        static_row<0, NTC - 1>(j, [&](auto J_) {
                            constexpr int J = decltype(J_)::value;
                            constexpr int G0 = (J + 1) / 4, NG = NTR / 4;
                            double nb0 = 0.0, nb1 = 0.0;
                            // the -L~ tiles of group grp + 1 are requested before the DMMAs of group grp
                            // (TMEM: asynchronous tcgen05.ld, waited for just before its use)
                            uint32_t rt[2][16];
                            double lfs[2][4][2];
                            auto request = [&](auto GRP_, auto BUF_) {
                                constexpr int grp = decltype(GRP_)::value, buf = decltype(BUF_)::value;
                                if constexpr (J < NL) {
#pragma unroll
                                    for (int k4 = 0; k4 < 4; ++k4)
                                        if (4 * grp + k4 > J) {
                                            const double2 l = *reinterpret_cast<const double2*>(
                                                AL + ((J * NTR + 4 * grp + k4) * 32 + lsw) * 2);
                                            lfs[buf][k4][0] = l.x;
                                            lfs[buf][k4][1] = l.y;
                                        }
                                } else if constexpr (J < RB) {
                                    tm_ld16(tmw + (uint32_t)(((J - NL) * NTR + 4 * grp) * 4), rt[buf]);
                                } else {
#pragma unroll
                                    for (int k4 = 0; k4 < 4; ++k4)
                                        if (4 * grp + k4 > J) {
                                            const double2 l = *reinterpret_cast<const double2*>(lr_tile(J, 4 * grp + k4));
                                            lfs[buf][k4][0] = l.x;
                                            lfs[buf][k4][1] = l.y;
                                        }
                                }
                            };
                            if constexpr (J >= NL && J < RB) tm_wait_st();
                            if constexpr (G0 < NG) request(std::integral_constant<int, G0>{}, std::integral_constant<int, 0>{});
#pragma unroll
                            for (int grp = G0; grp < NG; ++grp) {
                                const int buf = (grp - G0) & 1;
                                if constexpr (J >= NL && J < RB) {   // the group's TMEM load has landed
                                    tm_wait_ld();
                                    tm_pin(rt[buf]);
#pragma unroll
                                    for (int k4 = 0; k4 < 4; ++k4) {
                                        lfs[buf][k4][0] = u2d(rt[buf][4 * k4], rt[buf][4 * k4 + 1]);
                                        lfs[buf][k4][1] = u2d(rt[buf][4 * k4 + 2], rt[buf][4 * k4 + 3]);
                                    }
                                }
                                if (grp + 1 < NG) {
                                    if (buf == 0) static_row<0, NG>(grp + 1, [&](auto G_) { request(G_, std::integral_constant<int, 1>{}); });
                                    else static_row<0, NG>(grp + 1, [&](auto G_) { request(G_, std::integral_constant<int, 0>{}); });
                                }
#pragma unroll
                                for (int k4 = 0; k4 < 4; ++k4)
                                    if (4 * grp + k4 > J) {
                                        mma884(c[4 * grp + k4][0], c[4 * grp + k4][1], lfs[buf][k4][0], b0);
                                        mma884(c[4 * grp + k4][0], c[4 * grp + k4][1], lfs[buf][k4][1], b1);
                                    }
                                if (grp == G0 && more) {   // U_{j+1,k} is final: store it, transpose it for the next step
                                    if (k < RB) home_store(J + 1, k, c[J + 1][0], c[J + 1][1]);
                                    tb_put(c[J + 1][0], c[J + 1][1]);
                                    tb_get(nb0, nb1);
                                }
                            }
                            b0 = nb0;
                            b1 = nb1;
                        });
                    }
                }
                // (3) the diagonal tile's inverse (the rhs-only tile-column of n % 8 == 0 has none)
                if (k < NTR) {
                    double d0 = 0.0, d1 = 0.0;
                    static_row<0, NTR>(k, [&](auto T_) {
                        constexpr int t = decltype(T_)::value;
                        d0 = c[t][0];
                        d1 = c[t][1];
                    });
                    if (TAILC && k == NTR - 1) {   // padding rows, the rhs and padding columns -> identity
                        const int r = 8 * k + g, cc = 8 * k + 2 * q;
                        if (cc >= N) d0 = r == cc ? iun : 0.0;
                        if (cc + 1 >= N) d1 = r == cc + 1 ? iun : 0.0;
                    }
                    inv8_tile(d0, d1, isc, g, q);
                    const unsigned h0 = (unsigned)__double2hiint(d0) & 0x7fffffffu, h1 = (unsigned)__double2hiint(d1) & 0x7fffffffu;
                    xmaxh = max(xmaxh, max(h0, h1));
                    *reinterpret_cast<double2*>(Xi + k * 8 * XIS + g * XIS + 2 * q) = make_double2(-d0, -d1);
                    __syncwarp();
                }
                // (4) -L~_ik = A_ik (-X), i > k, stored over the column's tiles (register columns: Lr)
                if (k < NTR - 1) {
                    static_row<0, NTR - 1>(k, [&](auto K_) {
                        constexpr int K = decltype(K_)::value;
                        const double xb0 = Xi[K * 8 * XIS + (2 * q) * XIS + g], xb1 = Xi[K * 8 * XIS + (2 * q + 1) * XIS + g];
#pragma unroll
                        for (int tr = K + 1; tr < NTR; ++tr) {
                            double l0 = 0.0, l1 = 0.0;
                            mma884(l0, l1, c[tr][0], xb0);
                            mma884(l0, l1, c[tr][1], xb1);
                            if constexpr (K < RB) home_store(tr, K, l0, l1);
                            else *reinterpret_cast<double2*>(lr_tile(K, tr)) = make_double2(l0, l1);
                        }
                    });
                }
                // a register column keeps its U tiles (rows <= k) in acc
                if (k >= RB) {
                    static_row<0, NRW>((k - RB - r0) >> 1, [&](auto J_) {
                        constexpr int jr = decltype(J_)::value;
#pragma unroll
                        for (int tr = 0; tr < NTR; ++tr) {
                            acc[jr][tr][0] = c[tr][0];
                            acc[jr][tr][1] = c[tr][1];
                        }
                    });
                }
                // (5) publish the column
                tm_wait_st();
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __threadfence_block();
                __syncwarp();
                if (lane == 0) *ndone = k + 1;
            }
            {
                const unsigned xm = __reduce_max_sync(FULL, xmaxh);
                if (!(__hiloint2double((int)xm, 0) * amax <= 1e5) && lane == 0)
                    atomicMin(err_key + 1, (unsigned long long)pair);
            }
            // ---------------------------------------------- back substitution, column by column:
            // x_k = X_k y_k, then y_i -= U_ik x_k (i < k) by the column's owner; y and x share yx.
            // (Measured slower at C5: splitting the rows of the shared-memory / TMEM columns between
            // both warps, two barriers per column, 804 vs 778 ms; claiming the next pair here to
            // prefetch its 512 KB tensor early, 833 ms: 592 pairs' tensors do not fit the L2.)
            if (rhs_owner && q == QR) {
#pragma unroll
                for (int tr = 0; tr < NTR; ++tr) yx[8 * tr + g] = 8 * tr + g < N ? acc[G::JR][tr][SR] : 0.0;
            }
            pbar_sync(bid);
#pragma unroll 1
            for (int k = NTR - 1; k >= 0; --k) {
                if ((k & 1) == role) {
                    const double2 z = *reinterpret_cast<const double2*>(yx + 8 * k + 2 * q);
                    const double2 xn = *reinterpret_cast<const double2*>(Xi + k * 8 * XIS + g * XIS + 2 * q);
                    double t = fma(xn.x, z.x, xn.y * z.y);
                    t += __shfl_xor_sync(FULL, t, 1);
                    t += __shfl_xor_sync(FULL, t, 2);
                    __syncwarp();
                    if (q == 0) yx[8 * k + g] = 8 * k + g < N ? -t : 0.0;
                    __syncwarp();
                    const double2 x2 = *reinterpret_cast<const double2*>(yx + 8 * k + 2 * q);
                    auto axpy = [&](int i, double u0, double u1) {
                        double part = fma(u0, x2.x, u1 * x2.y);
                        part += __shfl_xor_sync(FULL, part, 1);
                        part += __shfl_xor_sync(FULL, part, 2);
                        if (q == 0) yx[8 * i + g] -= part;
                    };
                    if (k < NL) {
#pragma unroll 1
                        for (int i = 0; i < k; ++i) {
                            const double2 u = *reinterpret_cast<const double2*>(AL + ((k * NTR + i) * 32 + lsw) * 2);
                            axpy(i, u.x, u.y);
                        }
                    } else if (k < RB) {
#pragma unroll 1
                        for (int grp = 0; 4 * grp < k; ++grp) {
                            double v[4][2];
                            tm_get4(k - NL, grp, v);
#pragma unroll
                            for (int k4 = 0; k4 < 4; ++k4)
                                if (4 * grp + k4 < k) axpy(4 * grp + k4, v[k4][0], v[k4][1]);
                        }
                    } else {
                        static_row<0, NRW>((k - RB - r0) >> 1, [&](auto J_) {
                            constexpr int jr = decltype(J_)::value;
#pragma unroll
                            for (int i = 0; i < NTR - 1; ++i)
                                if (i < k) axpy(i, acc[jr][i][0], acc[jr][i][1]);
                        });
                    }
                    __syncwarp();
                }
                pbar_sync(bid);
            }
            if (role == 0 && lane == 0) *ndone = 0;   // both warps are past their last read of it
            if (rhs_owner) {
                double* out = rhs_given ? psi_out : psi_out + (size_t)d * psi_stride + (size_t)e * N;
                for (int r = lane; r < N; r += 32) out[r] = yx[r];
                if (done_flags) {
                    __threadfence();
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(done_flags + pair), "r"(epoch) : "memory");
                }
            }
        }
        } else {
        // ------------------------------------------------ blocked Gauss-Jordan, two warps
        unsigned am[RP];
        bool singular = false;
        // factor panel Pn (its tile-column is own): partial pivoting in row layout; publish
        // L~ = L L11^{-1} into Lp[Pn & 1], the pivot rows into s_pst[Pn & 1], the steps
        bool pan_ready = false;   // the next panel (a TMEM column) is already in the panel buffer
        auto factor = [&](int Pn) {
            const int TCp = (Pn * PW) >> 3, h = ((Pn * PW) >> 2) & 1;
            double* Lp = psm + G::SM_LP + (Pn % G::NLP) * G::LPB;
            double* Pan = Lp;   // the panel in row layout overlays this panel's multiplier buffer
            auto psl = [](int r, int j) { return j ^ ((r >> 2) & 1); };
            double pv[RP][PW];
            if (TCp < NL) {
#pragma unroll
                for (int i = 0; i < RP; ++i) {
                    const int r = lane + 32 * i;
                    const double* sp = AL + (TCp * NTR + (r >> 3)) * 64;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int sl = (r & 7) * 4 + 2 * h + j;
                        if (r < NR) {
                            const double2 x = *reinterpret_cast<const double2*>(sp + 2 * (sl ^ ((sl >> 3) & 3)));
                            pv[i][2 * j] = x.x;
                            pv[i][2 * j + 1] = x.y;
                        } else {
                            pv[i][2 * j] = pv[i][2 * j + 1] = 0.0;
                        }
                    }
                }
            } else {
                const bool wr = (q >> 1) == h;
                const int js = q - 2 * h;
                if (TCp < RB && !pan_ready) {
#pragma unroll
                    for (int grp = 0; grp < NTR / 4; ++grp) {
                        double v[4][2];
                        tm_get4(TCp - NL, grp, v);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int r = 8 * (4 * grp + k) + g;
                            st_shared_v2_if(Pan + r * PW + 2 * psl(r, js), v[k][0], v[k][1], wr);
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < NRW; ++j)
                    if (RB + r0 + 2 * j == TCp) {
#pragma unroll
                        for (int tr = 0; tr < NTR; ++tr) {
                            const int r = 8 * tr + g;
                            st_shared_v2_if(Pan + r * PW + 2 * psl(r, js), acc[j][tr][0], acc[j][tr][1], wr);
                        }
                    }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < RP; ++i) {
                    const int r = lane + 32 * i;
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        if (r < NR) {
                            const double2 x = *reinterpret_cast<const double2*>(Pan + r * PW + 2 * psl(r, j));
                            pv[i][2 * j] = x.x;
                            pv[i][2 * j + 1] = x.y;
                        } else {
                            pv[i][2 * j] = pv[i][2 * j + 1] = 0.0;
                        }
                    }
                }
                __syncwarp();
            }
            double lr[RP][PW];
            double kv[RP];
            int pst[PW];
#pragma unroll
            for (int i = 0; i < RP; ++i) kv[i] = pv[i][0];
#pragma unroll
            for (int t = 0; t < PW; ++t) {
                const int k = PW * Pn + t;
                if (N % PW != 0 && k >= N) {
#pragma unroll
                    for (int i = 0; i < RP; ++i) lr[i][t] = 0.0;
                    pst[t] = -1;
                    continue;
                }
                unsigned key = 0u;
                int ks = 0;
#pragma unroll
                for (int i = 0; i < RP; ++i) {
                    const unsigned hi = (unsigned)__double2hiint(kv[i]);
                    const unsigned lowk = ((unsigned)i << 5) | (31u - lane);
                    const unsigned kk = (hi & am[i]) + (am[i] ? (1u << KLB) | lowk : lowk);
                    if (i == 0 || kk > key) { key = kk; ks = i; }
                }
                double mine[PW];
#pragma unroll
                for (int tt = t; tt < PW; ++tt) {
                    mine[tt] = pv[0][tt];
#pragma unroll
                    for (int i = 1; i < RP; ++i)
                        if (i == ks) mine[tt] = pv[i][tt];
                }
                const unsigned kmax = __reduce_max_sync(FULL, key);
                const int src_lane = 31 - (int)(kmax & 31u);
                const int prow = src_lane + 32 * (int)((kmax >> 5) & ((1u << (KLB - 5)) - 1u));
                const double piv = __shfl_sync(FULL, mine[t], src_lane);
                double u[PW];
#pragma unroll
                for (int tt = t + 1; tt < PW; ++tt) u[tt] = __shfl_sync(FULL, mine[tt], src_lane);
                if (t < PW - 1) {
                    constexpr int L = PW - 1;
#pragma unroll
                    for (int i = 0; i < RP; ++i) kv[i] = piv * pv[i][t + 1 < PW ? t + 1 : L] - pv[i][t] * u[t + 1 < PW ? t + 1 : L];
                }
                if (!(fabs(piv) > 1e-14 * amax)) singular = true;
                double rinv;
                asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rinv) : "d"(piv));
                {
                    double ee = fma(-piv, rinv, 1.0);
                    rinv = fma(rinv, ee, rinv);
                    ee = fma(-piv, rinv, 1.0);
                    rinv = fma(rinv, ee, rinv);
                }
#pragma unroll
                for (int i = 0; i < RP; ++i) lr[i][t] = (lane + 32 * i == prow) ? 0.0 : pv[i][t] * rinv;
#pragma unroll
                for (int tt = t + 1; tt < PW; ++tt)
#pragma unroll
                    for (int i = 0; i < RP; ++i) pv[i][tt] -= lr[i][t] * u[tt];
#pragma unroll
                for (int i = 0; i < RP; ++i) am[i] = (lane + 32 * i == prow) ? 0u : am[i];
                pst[t] = prow;
                if (lane == 0) {
                    pivval[k] = rinv;
                    rowstep[prow] = k;
                }
            }
#pragma unroll
            for (int t = PW - 2; t >= 0; --t) {
                double l11[PW];
#pragma unroll
                for (int t2 = t + 1; t2 < PW; ++t2) {
                    const int p2 = pst[t2];
                    double v = lr[0][t];
#pragma unroll
                    for (int i = 1; i < RP; ++i)
                        if (p2 >= 0 && i == (p2 >> 5)) v = lr[i][t];
                    v = __shfl_sync(FULL, v, p2 >= 0 ? (p2 & 31) : 0);
                    l11[t2] = p2 >= 0 ? v : 0.0;
                }
#pragma unroll
                for (int t2 = t + 1; t2 < PW; ++t2)
#pragma unroll
                    for (int i = 0; i < RP; ++i) lr[i][t] -= lr[i][t2] * l11[t2];
            }
            __syncwarp();   // Pan reads done before Lp (same buffer) is written
#pragma unroll
            for (int t = 0; t < PW; ++t)
#pragma unroll
                for (int i = 0; i < RP; ++i)
                    if (lane + 32 * i < NR) Lp[t * G::LPS + lane + 32 * i] = -lr[i][t];
            if (lane < PW) s_pst[(Pn % G::NLP) * PW + lane] = pst[lane];
            __syncwarp();
        };
        // both warps track the retired rows (the pivot rows of every panel)
#pragma unroll
        for (int i = 0; i < RP; ++i) am[i] = lane + 32 * i >= N ? 0u : (0x7fffffffu & ~((1u << KLB) - 1u));
        auto owner = [](int c) { return c & 1; };
        auto panel_col = [](int Pn) { return (Pn * PW) >> 3; };
        (void)owner;
        // Per-panel state of the update (registers): L~ fragments, pivot rows, row steps
        const double* afp = nullptr;   // this panel's L~ fragments: afp[8 tr] (read where used: fewer live registers)
        int pstv[PW], tsv[NTR];
        int pq = -1;
        // update of an own SHARED-MEMORY tile-column c with the current panel
        auto upd_smem = [&](int c) __attribute__((always_inline)) {
            const double b = pq >= 0 ? AL[((c * NTR + (pq >> 3)) * 32 + (((pq & 7) * 4 + (g >> 1)) ^ ((pq & 7) >> 1))) * 2 + (g & 1)]
                                     : 0.0;
            __syncwarp();
            double* base = AL + (c * NTR * 32 + lsw) * 2;
#pragma unroll
            for (int tr = 0; tr < NTR; ++tr) {
                double2 cc = *reinterpret_cast<const double2*>(base + tr * 64);
                mma884(cc.x, cc.y, afp[8 * tr], b);
                *reinterpret_cast<double2*>(base + tr * 64) = cc;
            }
            __syncwarp();
        };
        // update of an own TMEM tile-column c: its pivot rows (one x4 load per row, the
        // holders write UR), then the software-pipelined tile pass
        auto upd_tmem = [&](int c, double* pan, int h) __attribute__((always_inline)) {
            // pan != nullptr: this is the next panel's column; its half h is also written to the
            // panel buffer in row layout (the factorization then skips its TMEM reload)
            const int tt = c - NL;
            const int us = (tt - t0) >> 1;
            tm_wait_st();
            {
                auto pa = [&](int t) { return tmw + (uint32_t)((tt * NTR + ((pstv[t] >= 0 ? pstv[t] : 0) >> 3)) * 4); };
                double rv[8];
                tm_ld4x4w(pa(0), pa(1), pa(2), pa(3), rv);
#pragma unroll
                for (int t = 0; t < PW; ++t) {
                    const int p = pstv[t] >= 0 ? pstv[t] : 0;
                    st_shared_v2_if(UR + t * G::URS + 2 * q + 8 * us, rv[2 * t], rv[2 * t + 1], pstv[t] >= 0 && g == (p & 7));
                }
            }
            __syncwarp();
            const double b = pq >= 0 ? UR[q * G::URS + 8 * us + g] : 0.0;
            constexpr int GPC = NTR / 4;
#pragma unroll
            for (int grp = 0; grp < GPC; ++grp) {
                double v[4][2];
                tm_ld16w(tmw + (uint32_t)((tt * NTR + 4 * grp) * 4), *reinterpret_cast<double (*)[8]>(&v[0][0]));
#pragma unroll
                for (int k = 0; k < 4; ++k) mma884(v[k][0], v[k][1], afp[8 * (4 * grp + k)], b);
                tm_put4(tt, grp, v);
                if (pan) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int r = 8 * (4 * grp + k) + g;
                        st_shared_v2_if(pan + r * PW + 2 * ((q - 2 * h) ^ ((r >> 2) & 1)), v[k][0], v[k][1],
                                        (q >> 1) == h);
                    }
                }
            }
            __syncwarp();   // UR reuse (and the panel written)
        };
        // update of own REGISTER tile-column j (column RB + role + 2 j)
        auto upd_reg = [&](int j) __attribute__((always_inline)) {
#pragma unroll
            for (int jj = 0; jj < NRW; ++jj)
                if (jj == j) {
                    const int us = NTOWN + jj;
#pragma unroll
                    for (int tr = 0; tr < NTR; ++tr)
                        st_shared_v2_if(UR + (tsv[tr] & (PW - 1)) * G::URS + 2 * q + 8 * us, acc[jj][tr][0], acc[jj][tr][1],
                                        (unsigned)tsv[tr] < (unsigned)PW);
                    __syncwarp();
                    const double b = pq >= 0 ? UR[q * G::URS + 8 * us + g] : 0.0;
#pragma unroll
                    for (int tr = 0; tr < NTR; ++tr) mma884(acc[jj][tr][0], acc[jj][tr][1], afp[8 * tr], b);
                    __syncwarp();
                }
        };
        // Pn = -1 only factors panel 0; factor() has one call site.
#pragma unroll 1
        for (int Pn = -1; Pn < NPANEL; ++Pn) {
            // look-ahead: the owner of panel Pn + 1's column updates it first (it is this warp's
            // first live column) and factors Pn + 1 before its other updates
            const bool la = Pn + 1 < NPANEL && owner(panel_col(Pn + 1)) == role;
            int c = G::NTC;   // first own live column not yet updated
            pan_ready = false;
            if (Pn >= 0) {
                if (owner(panel_col(Pn)) != role) pbar_sync(bid + 1 + (Pn & 1));   // published by the other warp
                const double* Lp = psm + G::SM_LP + (Pn % G::NLP) * G::LPB;
                afp = Lp + q * G::LPS + g;
#pragma unroll
                for (int t = 0; t < PW; ++t) pstv[t] = s_pst[(Pn % G::NLP) * PW + t];
                if (owner(panel_col(Pn)) != role) {   // the other warp retired these rows
#pragma unroll
                    for (int t = 0; t < PW; ++t)
#pragma unroll
                        for (int i = 0; i < RP; ++i) am[i] = (lane + 32 * i == pstv[t]) ? 0u : am[i];
                }
#pragma unroll
                for (int tr = 0; tr < NTR; ++tr) tsv[tr] = 8 * tr + g < N ? rowstep[8 * tr + g] - PW * Pn : -1;
                pq = pstv[0];
                pq = q == 1 ? pstv[1] : pq;
                pq = q == 2 ? pstv[2] : pq;
                pq = q == 3 ? pstv[3] : pq;
                const int tcn = min(((Pn + 1) * PW) >> 3, TCR);   // first live column (= the next panel's)
                c = tcn + ((tcn & 1) != role);
                if (la) {   // the next panel's column
                    if (c < NL) {
                        upd_smem(c);
                    } else if (c < RB) {
                        upd_tmem(c, psm + G::SM_LP + ((Pn + 1) % G::NLP) * G::LPB, (((Pn + 1) * PW) >> 2) & 1);
                        pan_ready = true;
                    } else {
                        upd_reg((c - RB - r0) >> 1);
                    }
                    c += 2;
                }
            }
            if (la) {
                factor(Pn + 1);
                pbar_arrive(bid + 1 + ((Pn + 1) & 1));
            }
            // the remaining own live columns, by storage class
#pragma unroll 1
            for (; c < NL; c += 2) upd_smem(c);
#pragma unroll 1
            for (; c < RB; c += 2) upd_tmem(c, nullptr, 0);
#pragma unroll
            for (int j = 0; j < NRW; ++j)
                if (RB + r0 + 2 * j >= c) upd_reg(j);
        }

        // ------------------------------------------------ solution x_k = rhs(p_k) * (1 / pivot_k)
        if (singular && lane == 0) atomicMin(err_key, (unsigned long long)pair);
        if (rhs_owner) {
            if (q == QR) {
                double* out = rhs_given ? psi_out : psi_out + (size_t)d * psi_stride + (size_t)e * N;
                constexpr int JR = G::JR;
#pragma unroll
                for (int tr = 0; tr < NTR; ++tr) {
                    const int r = 8 * tr + g;
                    if (r < N) {
                        const int kk = rowstep[r];
                        out[kk] = acc[JR][tr][SR] * pivval[kk];
                    }
                }
            }
            if (done_flags) {
                __threadfence();
                __syncwarp();
                if (lane == 0)
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(done_flags + pair), "r"(epoch) : "memory");
            }
        }
        }
        __syncwarp();
    }
    if (NT > 0) {
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem_base));
    }
}

template <int P, int NL, int NT, int PAIRS, bool SP = false>
void launch_dmma2(const DevProblem& pr, const double* src, const double* psi_old, const double* psi_new_in,
                  double* psi_out, int64_t stride, const int* pairs, int npairs, const double* rhs_given,
                  unsigned long long* err, int64_t zero_pair, cudaStream_t st, unsigned* done_flags, unsigned epoch) {
    using G = D2<P, NL, NT, PAIRS, SP>;
    static int slots[64] = {};
    static std::mutex mu;
    int dev = 0;
    D2CHECK(cudaGetDevice(&dev));
    const int max_blocks = per_device_once(slots, mu, dev, [&] {
        D2CHECK(cudaFuncSetAttribute(dmma2_sweep_kernel<P, NL, NT, PAIRS, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)G::SMEM));
        int sms = 0, per_sm = 0;
        D2CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        D2CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dmma2_sweep_kernel<P, NL, NT, PAIRS, SP>, G::THREADS,
                                                              G::SMEM));
        if (per_sm < 1) throw Error(-8, "dmma2 kernel does not fit on an SM");
        return sms * (per_sm > 1 ? 1 : per_sm);   // one CTA per SM: it owns all TMEM columns
    });
    int blocks = (npairs + G::PAIRS - 1) / G::PAIRS;
    if (blocks > max_blocks) blocks = max_blocks;
    dmma2_sweep_kernel<P, NL, NT, PAIRS, SP><<<blocks, G::THREADS, G::SMEM, st>>>(
        pr, src, psi_old, psi_new_in, psi_out, stride, pairs, npairs, rhs_given, err, zero_pair, done_flags, epoch);
    D2CHECK(cudaGetLastError());
}

}  // namespace

// The two-warp kernel's shape: 3D p = 4 (C5).  Measured for 3D p = 3 (C4) too, with four
// two-warp pairs per SM: 544 ms vs the one-warp kernel's 319 ms (twelve pairs per SM).
bool dev_dmma2_supported(int dim, int p) { return dim == 3 && p == 4; }

void dev_dmma2_sweep(const DevProblem& P, const double* src, const double* psi_old, double* psi_new, int64_t stride,
                     const int* pairs, int npairs, unsigned long long* err_key, int64_t zero_pair, void* stream,
                     unsigned* done_flags, unsigned epoch, bool static_pivot) {
    cudaStream_t st = (cudaStream_t)stream;
    if (P.dim == 3 && P.p == 3 && static_pivot)   // C4 shape: eight two-warp pairs per SM (HSW_D2_Q3=1)
        launch_dmma2<3, 1, 6, 8, true>(P, src, psi_old, psi_new, psi_new, stride, pairs, npairs, nullptr, err_key,
                                       zero_pair, st, done_flags, epoch);
    else if (P.dim == 3 && P.p == 4 && static_pivot)
        launch_dmma2<4, 4, 8, 4, true>(P, src, psi_old, psi_new, psi_new, stride, pairs, npairs, nullptr, err_key,
                                       zero_pair, st, done_flags, epoch);
    else if (P.dim == 3 && P.p == 4)
        launch_dmma2<4, 4, 8, 4>(P, src, psi_old, psi_new, psi_new, stride, pairs, npairs, nullptr, err_key, zero_pair,
                                 st, done_flags, epoch);
    else
        throw Error(-1, "dmma2 kernel: unsupported (dim, order)");
}

void dev_dmma2_local_solve(const DevProblem& P, const int* pair_dev, const double* rhs, double* out,
                           unsigned long long* err_key, int64_t zero_pair, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (P.dim == 3 && P.p == 4)
        launch_dmma2<4, 4, 8, 4>(P, nullptr, nullptr, nullptr, out, 0, pair_dev, 1, rhs, err_key, zero_pair, st,
                                 nullptr, 0);

    else
        throw Error(-1, "dmma2 kernel: unsupported (dim, order)");
}

}  // namespace hsw
