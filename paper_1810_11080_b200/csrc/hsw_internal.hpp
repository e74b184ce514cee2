// Internal declarations shared by the host setup (hsw_host.cpp), the C ABI
// (hsw_capi.cpp) and the CUDA kernels (hsw_kernels.cu).  Not installed.
#pragma once

#include <type_traits>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace hsw {

// Exception types mapped 1:1 onto hsw_status codes by the C ABI and back onto
// the reference's exception types by include/hosweep_b200/solver.hpp.
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

// Per-device launch configuration of one kernel instantiation: the dynamic
// shared-memory attribute is per device, so it is set (and the resident grid
// size measured) once for every device a process launches on.  Thread-safe.
template <typename Init>
int per_device_once(int (&slots)[64], std::mutex& mu, int dev, Init&& init) {
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64) throw std::runtime_error("device ordinal out of range");
    if (slots[dev] == 0) slots[dev] = init();
    return slots[dev];
}

constexpr int kMaxFaces = 6;
constexpr int kMaxFaceNodes = 49;     // (p+1)^2 for p <= 6 (3D p <= 4 -> 25)
constexpr int kMaxFacePoints = 64;    // (p+2)^2 for p <= 6

#ifdef __CUDACC__
#define HSW_HD __host__ __device__
#else
#define HSW_HD
#endif
// Device layout of the element tensors T = (M, Gx, Gy, Gz), entry (row m, column n): DMMA-fragment
// order.  The n x n matrix is cut into 8x8 tiles (padded with zeros to a multiple of 8); per tile
// (column-major over tiles), per column parity s = n & 1 and per plane ((M, Gx) | (Gy, Gz)) the 32
// lanes' double2 values are contiguous: lane 4 (m & 7) + ((n & 7) >> 1).  A warp loading a tile in the
// m8n8k4 accumulator layout (rows 8 tr + g, columns 8 tc + 2 q + s) therefore reads 512 contiguous
// bytes per LDG.128 — one L1TEX wavefront per 128-byte line.  (The earlier planar layout
// [column][plane][row] fetched the same sectors as four lines of eight lanes each: one wavefront per
// 32-byte sector, measured 30.5 vs 76.2 B/clk/SM, tools/dmma_check/ldg_pattern.cu.)
HSW_HD constexpr inline size_t t_tiles(int nb) { return (size_t)((nb + 7) / 8); }
HSW_HD constexpr inline size_t t_elem_doubles(int nb) { return t_tiles(nb) * t_tiles(nb) * 256; }
// double2 index, within one element, of plane p of entry (m, n)
HSW_HD constexpr inline size_t t_idx2(int nb, int m, int n, int p) {
    const size_t tile = (size_t)(n >> 3) * t_tiles(nb) + (size_t)(m >> 3);
    return ((tile * 2 + (size_t)(n & 1)) * 2 + (size_t)p) * 32 + (size_t)(4 * (m & 7) + ((n & 7) >> 1));
}
HSW_HD inline size_t t_idx(size_t e, int nb, int m, int n, int k) {
    return e * t_elem_doubles(nb) + 2 * t_idx2(nb, m, n, k >> 1) + (size_t)(k & 1);
}

// Kernel-facing problem tables (device pointers), POD.
struct DevProblem {
    int dim, p, nb, nfn, nqf, nfaces, nel, nd;
    const double* T;          // fragment order, see t_idx (planes (M, Gx) | (Gy, Gz)), G_k = -(d_k u)^T W u
    const double* sig_t;      // [E]
    const double* sig_s;      // [E]
    const double* bscale;     // [E] max_ij (sig_t |M| + |Gx| + |Gy| + |Gz|)_ij >= max |volume part of A(Omega)|:
                              //     the matrix scale of the singular-block test (dmma1 kernel)
    const double* qvol;       // [E][nb] volume source moments
    const double* fgeom;      // [E][nfaces][nqf][4]: outward normal (own side), w_q*|J_Gamma|
    const int* fnbr;          // [E][nfaces][4]: neighbour elem (-1 boundary), neighbour face,
                              //                 orientation code (own -> neighbour), unused
    const uint16_t* inflags;  // [nd][E]: bit 2f incoming coupling through face f, bit 2f+1 lagged
    const double* omega;      // [nd][4]
    const double* weight;     // [nd]
    double inflow;
    // reference-element tables in global memory (staged into SMEM by the kernels)
    const int* g_fnode;       // [6][kMaxFaceNodes]
    const double* g_trace;    // [kMaxFacePoints][kMaxFaceNodes]
    const int* g_fidx;        // [6][128]
    const int* g_nmask;       // [128]
    const double* g_line;     // [8][8]
    int debug_flags;          // ablation (tools/ablate.py): 1 skip faces, 2 skip elimination, 4 skip T loads,
                              // 8 per-phase clock64 counters into prof[], 16/32 warp subsets (dmma1
                              // profiling instantiations only)
    unsigned long long* prof; // [16] debug phase-cycle accumulators
    int tune;                 // development knobs (HSW_TUNE, bit flags; 0 = production defaults)
    // FaceIntegration::Rule::romberg (2D; null with the Gauss rule): per (ordinate, element,
    // local face) blocks integrated at create (assembly.hpp:121-131, romberg.hpp)
    const double* rom_ob;     // [nd][E][nf][nfn*nfn] outflow block, own face nodes
    const double* rom_ib;     // [nd][E][nf][nfn*nfn] incoming coupling block (positive integral;
                              // columns in own face-node order of the gathered upwind traces)
    const double* rom_bin;    // [nd][E][nf][nfn] boundary inflow moments
    const unsigned char* rom_omask;   // [nd][E] faces with a nonzero outflow block
};

// Host-computed reference-face tables (uploaded as the g_* global tables).
struct SourceParams {
    double v[8];
};

struct ConstTables {
    int fnode[kMaxFaces][kMaxFaceNodes];                 // local element node of face node a
    double trace[kMaxFacePoints][kMaxFaceNodes];         // phi_a(point q) on the reference face
};

// Device-side launch wrappers (hsw_kernels.cu).
struct DevState;
struct LaunchCounters { int64_t launches = 0; };

// scattering + volume source s[e][m] = qvol + (1/4pi) sigma_s M phi
void dev_scatter_source(const DevProblem& P, const double* phi, double* src, void* stream);
// phi = sum_d w_d psi[d] (d ascending), plus max|psi_new - psi_old| and the
// phi L2 partial sums; deterministic fixed-shape reductions.
void dev_phi_and_norms(const DevProblem& P, const double* psi_new, const double* psi_old,
                       const double* phi_old, double* phi_new, double* scratch, double* out3,
                       void* stream);
// out[d] = max_i |a[d][i] - b[d][i]| for d < nd (per-ordinate error history)
void dev_per_ordinate_maxdiff(const double* a, const double* b, int nd, int64_t n, double* out, void* stream);
// out[0] = max_i |a_i - b_i|, out[2] = max_i |a_i| over n values
void dev_max_abs_diff(const double* a, const double* b, int64_t n, double* scratch, double* out,
                      void* stream);
double dev_fp64_peak_tflops(int device);
double dev_dmma_peak_tflops(int device);
// W warps per pair, DMMA trailing updates (hsw_dmma.cu): the shapes dmma1 does not instantiate
void dev_dmma_sweep(const DevProblem& P, const double* src, const double* psi_old, double* psi_new, int64_t stride,
                    const int* pairs, int npairs, unsigned long long* err_key, int64_t zero_pair, void* stream);
void dev_dmma_local_solve(const DevProblem& P, const int* pair_dev, const double* rhs, double* out,
                          unsigned long long* err_key, int64_t zero_pair, void* stream);
// device-side setup (hsw_setup.cu): element tensors + volume source moments, absorption
void dev_block_scale(int nel, int nb, const double* T, const double* sig_t, double* out, void* stream);
void dev_element_tensors(int dim, int nel, int nb, int npe, int nq, const double* pts, const int* enodes,
                         const double* U, const double* DU, const double* GG, const double* GV, const double* wq,
                         int source_kind, const SourceParams& sp, double* T, double* qvol,
                         unsigned long long* bad_elem, void* stream);
double dev_absorption(int nel, int nb, const double* T, const double* sig_t, const double* sig_s, const double* phi,
                      double* scratch, void* stream);
// per boundary face (elem, face, attr triples): out[2 bi] = sum_d w_d 1^T B psi_d (outflow),
// out[2 bi + 1] = sum_d w_d * inflow moments (device balance_report, solver.hpp:220-245)
void dev_balance_faces(const DevProblem& P, const double* psi, int nbf, const int* bfaces, double* out, void* stream);
void dev_coupling_max(int dim, int nfi, int nf, int nqf, int nfn, const int* iface, const double* fgeom,
                      const double* fsj, const double* fqw, const double* trace, const double* traceR,
                      const double* odir, int d0, int d1, double* out, void* stream);
// direction-sharded source iteration (hsw_kernels.cu)
void dev_phi_partial(const DevProblem& P, const double* psi_new, int d0, int d1, const double* prefix, double* out,
                     void* stream);
void dev_phi_norms2(const DevProblem& P, const double* phi_new, const double* phi_old, double* scratch, double* out3,
                    void* stream);
// one warp per pair, persistent, register + shared-memory DMMA tiles (hsw_dmma1.cu)
bool dev_dmma1_supported(int dim, int p);
// done_flags != nullptr: dataflow schedule over the whole worklist (one launch;
// a pair waits for its retained upwind pairs' flags == epoch, then publishes its own).
// static_pivot: the tile-LU instantiation without row searches; a pair whose block it
// refuses (tiny pivot / large inverse tile) is recorded in err_key[1] (atomicMin of the
// pair id) and the caller redoes the sweep with static_pivot = false.  err_key points
// at TWO 64-bit keys: [0] singular block, [1] static pivoting refused.
void dev_dmma1_sweep(const DevProblem& P, const double* src, const double* psi_old, double* psi_new, int64_t stride,
                     const int* pairs, int npairs, unsigned long long* err_key, int64_t zero_pair, void* stream,
                     unsigned* done_flags = nullptr, unsigned epoch = 0, bool static_pivot = false);
void dev_dmma1_local_solve(const DevProblem& P, const int* pair_dev, const double* rhs, double* out,
                           unsigned long long* err_key, int64_t zero_pair, void* stream);
// two warps per pair (hsw_dmma2.cu): the latency-bound 3D Q4 shape
bool dev_dmma2_supported(int dim, int p);
void dev_dmma2_sweep(const DevProblem& P, const double* src, const double* psi_old, double* psi_new, int64_t stride,
                     const int* pairs, int npairs, unsigned long long* err_key, int64_t zero_pair, void* stream,
                     unsigned* done_flags = nullptr, unsigned epoch = 0, bool static_pivot = false);
void dev_dmma2_local_solve(const DevProblem& P, const int* pair_dev, const double* rhs, double* out,
                           unsigned long long* err_key, int64_t zero_pair, void* stream);

#ifdef __CUDACC__
// ---- device helpers shared by the sweep kernels (hsw_dmma1.cu, hsw_dmma2.cu)
// dispatch a warp-uniform runtime index i in [LO, HI) to code with a compile-time index
// (register tiles are addressed statically): a binary tree of uniform branches
template <int LO, int HI, class F>
__device__ __forceinline__ void static_row(int i, F&& f) {
    if constexpr (HI - LO <= 1) {
        f(std::integral_constant<int, LO>{});
    } else {
        constexpr int MID = (LO + HI) / 2;
        if (i < MID) static_row<LO, MID>(i, static_cast<F&&>(f));
        else static_row<MID, HI>(i, static_cast<F&&>(f));
    }
}
// In-register inverse of an 8x8 tile held in the m8n8k4 accumulator layout (lane (g, q): row g,
// columns 2q, 2q+1), static pivot order.  Fraction-free Gauss-Jordan: step s leaves the pivot row as
// it is and forms  row_i <- pvn row_i - fn_i row_s  for the other rows, with the pivot and the
// multipliers scaled by 2^-exponent(pv) (an integer operation on the high word; |pvn| in [1, 2), so
// the row scales grow by < 2 per step).  The inverse's column s takes the slot of the eliminated
// column; each row carries its diagonal dg.  The step-to-step chain is shuffle + DMUL + DMUL + DFMA
// with no reciprocal in it; one reciprocal per row at the end.  The tile is scaled by sc (a power
// of two ~ 1 / matrix scale).  The true pivot of step s is pv_s / pp (pp = product of the pvn so
// far = the scale of row s); a tiny or zero pivot shows as a huge / non-finite inverse, which
// the caller's max |X| monitor refuses (no per-step test on the chain).
__device__ __forceinline__ void inv8_tile(double& d0, double& d1, double sc, int g, int q) {
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

#endif  // __CUDACC__

}  // namespace hsw
