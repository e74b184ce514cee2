/*
 * hosweep_b200.h — C ABI of the B200-native transport sweep.
 *
 * Drop-in boundary for the reference's solver/sweep path
 * (/root/reference/proj/include/hosweep/solver.hpp:50-203 over
 * assembly.hpp:333-409).  Plain C: POD structs, pointers + sizes, int status
 * codes, no exceptions and no torch/Eigen types.  One handle owns the device
 * state of one assembled problem; calls on a handle are stream-ordered on the
 * handle's CUDA stream, serialised by a per-handle lock (so a reference-style
 * parallel_for over ordinates calling sweep(d) concurrently is safe,
 * solver.hpp:145-149) and run on the handle's device whatever device is
 * current on the calling thread (restored on return).
 *
 * Error model: every call returns HSW_OK (0) or a negative status; the message
 * of the last failure on the calling thread is available from hsw_last_error()
 * and carries the reference's context, e.g.
 *   "local streaming+collision block is singular (element E, ordinate D)"
 *   (solver.hpp:70-74) for HSW_ERR_SOLVER.
 * The C++ wrapper in include/hosweep_b200/solver.hpp rethrows these as the
 * reference's exception types (SolverError, MeshError, AssemblyError,
 * std::out_of_range, std::logic_error).
 */
#ifndef HOSWEEP_B200_H
#define HOSWEEP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSW_ABI_VERSION 4

enum hsw_status {
    HSW_OK = 0,
    HSW_ERR_INVALID = -1,   /* std::invalid_argument: bad descriptor / options        */
    HSW_ERR_MESH = -2,      /* MeshError (mesh.hpp:23-25): connectivity, pairing, det<=0 */
    HSW_ERR_GEOMETRY = -3,  /* GeometryError (mesh.hpp:27-29): degenerate face tangent  */
    HSW_ERR_ASSEMBLY = -4,  /* AssemblyError (assembly.hpp:24-26): singular Jacobian     */
    HSW_ERR_SOLVER = -5,    /* SolverError (solver.hpp:21-23): singular local block      */
    HSW_ERR_LOGIC = -6,     /* std::logic_error (sweepgraph.hpp:379-380,391-392)          */
    HSW_ERR_RANGE = -7,     /* std::out_of_range (solver.hpp:80 ordering(d).at())         */
    HSW_ERR_CUDA = -8,      /* CUDA runtime failure / no device                          */
    HSW_ERR_NOMEM = -9      /* device or host allocation failure                          */
};

/* Edge weighting (sweepgraph.hpp:40): unity, face (default), siginvface. */
enum hsw_weighting { HSW_WEIGHT_UNITY = 0, HSW_WEIGHT_FACE = 1, HSW_WEIGHT_SIGINVFACE = 2 };

/* Volumetric source q(x) (SourceSpec::volumetric, assembly.hpp:317-327),
 * evaluated at physical volume quadrature points (assembly.hpp:298). */
enum hsw_source_kind {
    HSW_SOURCE_CONSTANT = 0, /* params[0] = q                                           */
    HSW_SOURCE_BALL = 1      /* params = cx, cy, cz, R, q_in, q_out: q_in if |x-c|^2<R^2 */
};

/*
 * Problem descriptor: the arguments of assemble_transport_operator
 * (assembly.hpp:362-366) flattened to C: HighOrderMesh (mesh.hpp:121-134),
 * basis order (ReferenceBasis, basis.hpp:65-72), AngularQuadrature
 * (angular.hpp:23-33), CrossSectionField::by_region (xsec.hpp:22-27),
 * SourceSpec::isotropic (assembly.hpp:321-326), AssemblyOptions with the
 * Gauss face rule (assembly.hpp:33-45), plus the SolveOptions graph knobs
 * (solver.hpp:25-32).  All arrays are host memory, copied during hsw_create.
 */
typedef struct hsw_problem_desc {
    int abi_version;            /* HSW_ABI_VERSION                                     */
    int dim;                    /* 2 (quads) or 3 (hexes)                               */
    int geom_order;             /* r: mesh mapping order                                */
    int basis_order;            /* p: DG order, n = (p+1)^dim dofs per element          */
    int num_points;
    const double* points;       /* num_points * dim, interleaved                        */
    int num_elements;
    const int* element_nodes;   /* num_elements * (r+1)^dim, lexicographic, x fastest   */
    const int* element_region;  /* num_elements region ids (NULL: all 1)                */
    int num_boundary_faces;
    const int* boundary_faces;  /* (elem, local_face, attr) triples                     */
    int num_ordinates;
    const double* ordinate_weight; /* sum 4*pi (angular.hpp:22)                         */
    const double* ordinate_dir;    /* 3 per ordinate: (mu, eta, xi)                     */
    int num_regions;
    const int* region_ids;
    const double* sigma_t;      /* per region; requires sigma_t >= sigma_s >= 0          */
    const double* sigma_s;
    int source_kind;            /* hsw_source_kind                                      */
    double source_params[8];
    double inflow;              /* isotropic incident flux on all boundary faces        */
    int volume_points;          /* per axis; 0 -> p+2 (assembly.hpp:146)               */
    int face_points;            /* Gauss points per face axis; 0 -> p+2                 */
    int weighting;              /* hsw_weighting                                        */
    int exact_fas_threshold;    /* solver.hpp:31, default 10                            */
    int validate_geometry;      /* MeshValidation::full checks (mesh.hpp:128-131)        */
    int check_local_blocks;     /* factor every (e,d) block once at create and report
                                   the first singular one, like the SweepSolver ctor
                                   (solver.hpp:67-75)                                   */
    int device;                 /* CUDA device ordinal                                  */
    /* FaceIntegration (assembly.hpp:33-40): HSW_FACE_GAUSS (face_points per axis) or
       HSW_FACE_ROMBERG, the reference's default: adaptive Romberg per (face, ordinate)
       with tol / max_levels / min_levels (romberg.hpp:33-88; 2D meshes, as the
       reference).  Zero-initialised fields select Gauss.                              */
    int face_rule;
    double romberg_tol;         /* default 1e-10 when <= 0                               */
    int romberg_max_levels;     /* default 16 when <= 0                                  */
    int romberg_min_levels;     /* default 6 when < 0 (0 is a valid value)              */
    /* Ordinate shard [ordinate_begin, ordinate_end) of a multi-GPU rank:
       only these ordinates' graphs, orders, worklists and psi are built / allocated;
       the hsw_shard_* primitives, hsw_sweep_resident and single-ordinate calls inside
       the shard work, all-ordinate calls (source_iteration, balance, d = -1 sweeps)
       report HSW_ERR_RANGE.  ordinate_end == 0: every ordinate.                      */
    int ordinate_begin, ordinate_end;
} hsw_problem_desc;
enum hsw_face_rule { HSW_FACE_GAUSS = 0, HSW_FACE_ROMBERG = 1 };

/* SolveOptions (solver.hpp:25-32) + the configs' relative-phi criterion. */
enum hsw_criterion { HSW_CRIT_PSI_LINF = 0, HSW_CRIT_PHI_REL_L2 = 1 };
enum hsw_mode { HSW_MODE_SWEEP = 0, HSW_MODE_DIRECT = 1 };
typedef struct hsw_si_options {
    double tolerance;           /* default 1e-14 (solver.hpp:27)                        */
    int max_iterations;         /* default 400 (solver.hpp:28)                          */
    int criterion;              /* hsw_criterion                                       */
    int mode;                   /* hsw_mode: sweep or direct_oracle (solver.hpp:26)     */
} hsw_si_options;

/* ConvergenceHistory + SolverState metadata (solver.hpp:34-45). */
typedef struct hsw_si_result {
    int iterations;
    int converged;
    double final_error;         /* max_d ||psi_new - psi_old||_inf of the last iteration */
    double final_phi_rel;       /* ||phi_new - phi_old||_2 / ||phi_new||_2              */
    double seconds;             /* device time of the whole iteration (CUDA events)      */
} hsw_si_result;

typedef struct hsw_handle hsw_handle;

/* Thread-local message of the last failing call (always NUL terminated). */
int hsw_last_error(char* buf, size_t len);

/* Build the operator tensors, face tables, per-ordinate graphs, orderings,
 * lag flags and level worklists; upload to the device.  Replaces
 * assemble_transport_operator (assembly.hpp:362-409) + the SweepSolver
 * constructor (solver.hpp:52-78). */
int hsw_create(const hsw_problem_desc* desc, hsw_handle** out);
void hsw_destroy(hsw_handle* h);

/* Sizes: num_elements, block_size n, num_ordinates, num_dofs = N_el*n,
 * num_interior_faces, num_levels (of the all-ordinate worklist). */
int hsw_sizes(const hsw_handle* h, int64_t out[6]);

/* SweepSolver::ordering(d) (solver.hpp:80) -> SweepOrdering (sweepgraph.hpp:318-325):
 * order/position (N_el each, may be NULL), lagged edge ids ascending (capacity
 * lagged_cap; *num_lagged gets the true count), lagged weight, per-element
 * level (N_el, may be NULL).  HSW_ERR_RANGE for d out of range. */
int hsw_ordering(const hsw_handle* h, int d, int* order, int* position, int* lagged,
                 int lagged_cap, int* num_lagged, double* lagged_weight, int* level);

/* SweepSolver::total_lagged_edges (solver.hpp:83-87). */
int hsw_total_lagged_edges(const hsw_handle* h, int64_t* out);

/* The ordinate's face couplings in the reference's coupling order
 * (assembly.hpp:236-241): per coupling (face, downwind, upwind, lagged) and
 * the graph edge weight.  Capacity cap; *count gets the true count. */
int hsw_couplings(const hsw_handle* h, int d, int* ints4, double* weights, int cap, int* count);

/* Interior faces in the reference's face order (mesh.hpp:290-332): per face
 * (elem_left, elem_right, face_left, face_right, orientation). */
int hsw_interior_faces(const hsw_handle* h, int* ints5, int cap, int* count);

/* SweepSolver::local_solve (solver.hpp:91-93): psi = A_{e,d}^{-1} rhs. */
int hsw_local_solve(hsw_handle* h, int e, int d, const double* rhs, double* out);

/* SweepSolver::sweep (solver.hpp:98-117) for one ordinate d, or for every
 * ordinate when d == -1 (then psi_old/psi_new are [num_ordinates][N]).
 * Host pointers; H2D/D2H copies are part of the call. */
int hsw_sweep(hsw_handle* h, int d, const double* phi, const double* psi_old, double* psi_new);

/* Same on device pointers already resident in HBM (stream-ordered on the
 * handle's stream, no host synchronisation unless an error check needs it). */
int hsw_sweep_device(hsw_handle* h, int d, const double* phi_dev, const double* psi_old_dev,
                     double* psi_new_dev);

/* SweepSolver::direct_oracle (solver.hpp:121-133): the per-ordinate global
 * system solved with phi fixed (lagged sweeps iterated to a fixpoint on the
 * device; converges to machine precision on these block-triangular-plus-cut
 * systems). */
int hsw_direct_oracle(hsw_handle* h, int d, const double* phi, double* psi);

/* SweepSolver::source_iteration (solver.hpp:136-168).  psi_out ([nd][N]) and
 * phi_out (N) may be NULL; err_hist / phi_hist (max_iterations) may be NULL;
 * per_ordinate_hist ([max_iterations][nd], may be NULL) receives
 * ConvergenceHistory::per_ordinate, error[it][d] = ||dpsi_d||_inf
 * (solver.hpp:36,150-156). */
int hsw_source_iteration(hsw_handle* h, const hsw_si_options* opts, hsw_si_result* res,
                         double* psi_out, double* phi_out, double* err_hist, double* phi_hist,
                         double* per_ordinate_hist);

/* balance_report (solver.hpp:220-245) on a state; out5 = source_volume,
 * inflow, absorption, outflow, residual; attrs/vals: outflow by boundary
 * attribute (up to cap entries, *count true count). */
int hsw_balance(hsw_handle* h, const double* psi, const double* phi, double out5[5], int* attrs,
                double* vals, int cap, int* count);
/* balance_report of the handle's RESIDENT state (after hsw_source_iteration: its
 * converged psi / phi; after hsw_set_state: the state set), evaluated on the
 * device: per boundary face a deterministic sum over the ordinates, absorption
 * by a fixed-shape reduction.  Same outputs as hsw_balance. */
int hsw_balance_resident(hsw_handle* h, double out5[5], int* attrs, double* vals, int cap, int* count);

/* ---- device-resident state for benchmarking / advanced callers ---------- */
/* Device pointers of the handle's psi (two buffers, [nd][N] each) and phi. */
int hsw_device_state(hsw_handle* h, double** psi_a, double** psi_b, double** phi);
/* Copy host phi (N) and/or psi (nd*N, into psi_a) into the resident device
 * state; either pointer may be NULL. */
int hsw_set_state(hsw_handle* h, const double* phi, const double* psi);
/* One all-ordinate sweep psi_a -> psi_b with the current device phi (the
 * scattering source is rebuilt inside), stream-ordered; no host sync. */
int hsw_sweep_resident(hsw_handle* h);
/* Synchronise the handle's stream; returns the sweep error flag as a status. */
int hsw_synchronize(hsw_handle* h);
/* The handle's CUDA stream (cudaStream_t as void*). */
void* hsw_stream(hsw_handle* h);
/* Kernel launches issued by the last hsw_sweep_resident call. */
int64_t hsw_last_launch_count(const hsw_handle* h);
/* How many API calls were redone with the pivoted (partial-pivoting Gauss-Jordan) kernel because the
 * static-pivot tile LU refused a local block (tiny pivot / large inverse tile); after the first one the
 * handle keeps to the pivoted kernel.  0 on every BASELINE.json config. */
int64_t hsw_pivot_fallbacks(const hsw_handle* h);
/* Device time of the main sweep kernel launches of the last
 * hsw_sweep_resident call, measured with CUDA events on the handle's stream. */
double hsw_last_sweep_kernel_ms(const hsw_handle* h);

/* ---- direction-sharded source iteration ----------------------
 * source_iteration's sweeps are independent per ordinate (solver.hpp:145-149),
 * so a rank owns an ordinate block [d0, d1) and exchanges only phi.  These are
 * the per-rank device primitives; the collective driver is
 * paper_1810_11080_b200/sharded.py.  Pointers named *_dev are DEVICE pointers on
 * the handle's device; all work is ordered on hsw_stream(h), no host sync unless
 * a host output is returned.  HSW_ERR_RANGE unless 0 <= d0 < d1 <= nd. */
/* psi_old = psi_new = 0 for every ordinate, resident phi = 0 (solver.hpp:139-141). */
int hsw_shard_reset(hsw_handle* h);
/* Scattering source from phi_dev (NULL: the resident phi), then sweep the
 * ordinates [d0, d1): psi_new from the resident psi_old (lagged couplings) and
 * the block's own retained upwind values.  Worklist: the block's pairs sorted
 * by (level, element, ordinate), built once per block and cached. */
int hsw_shard_sweep(hsw_handle* h, int d0, int d1, const double* phi_dev);
/* The same block sweep end to end with HOST buffers: phi (N doubles) and the
 * block's psi_old / psi_new ((d1 - d0) x N, row d - d0), H2D / sweep / D2H
 * pipelined over ordinate sub-blocks as in hsw_sweep(d = -1); the block's
 * psi_new also stays on the device for hsw_shard_phi_partial.  Synchronous. */
int hsw_shard_sweep_host(hsw_handle* h, int d0, int d1, const double* phi, const double* psi_old, double* psi_new);
/* out_dev = prefix_dev + sum_{d0 <= d < d1} w_d psi_new_d, accumulated per
 * (e, m) in ascending d with one FMA per ordinate (prefix_dev NULL: 0).
 * Chaining blocks in rank order reproduces hsw_source_iteration's phi bit for
 * bit (solver.hpp:157-158). */
int hsw_shard_phi_partial(hsw_handle* h, int d0, int d1, const double* prefix_dev, double* out_dev);
/* *err = max over d in [d0, d1) of ||psi_new_d - psi_old_d||_inf (solver.hpp:150-156). */
int hsw_shard_psi_error(hsw_handle* h, int d0, int d1, double* err);
/* out2 = { sum (phi_new - phi_old)^2, sum phi_new^2 } with the same fixed-shape
 * reduction tree as hsw_source_iteration (identical bits for identical phi). */
int hsw_shard_phi_norms(hsw_handle* h, const double* phi_new_dev, const double* phi_old_dev, double out2[2]);
/* psi_old <- psi_new (buffer swap) and resident phi <- phi_dev (NULL: keep). */
int hsw_shard_advance(hsw_handle* h, const double* phi_dev);
/* Copy psi_old (the latest completed iterate) of ordinates [d0, d1) to host
 * psi ((d1-d0)*N doubles, ordinate-major). */
int hsw_shard_psi(hsw_handle* h, int d0, int d1, double* psi);

/* Measured FP64 FMA throughput of the device (TFLOP/s) from a DFMA-chain
 * microbenchmark over all SMs (~0.1 s); the roofline denominator of the
 * sweep kernel.  device: CUDA ordinal. */
int hsw_fp64_peak(int device, double* tflops);

/* Ablation switches for development timing (results are NOT valid solves):
 * 1 skip the face terms, 2 skip the elimination, 4 skip the tensor loads,
 * 8 phase clocks, 16 / 32 only warp 0 / warps 0-3 of each CTA work.  Honoured
 * by the one-warp DMMA kernel's profiling instantiations (3D Q3 and Q4); the
 * production kernels carry no debug code. */
int hsw_debug_flags(hsw_handle* h, int flags);
/* Debug phase-cycle counters of flag 8 (0-5: volume, faces, assembly,
 * elimination, write-back, pair count; 6-7: register / TMEM volume parts;
 * 8-11: pivot-row gather, update, dependency wait, factor; 12-14: factor
 * load, pivot steps, gather TMEM + register part). */
int hsw_debug_profile(hsw_handle* h, unsigned long long out[16]);

/* Test hook: the library's graph ordering (Tarjan SCC, exact FAS DP for SCCs
 * <= threshold else the weighted Eades-Lin-Smyth heuristic, min-heap Kahn on
 * the condensation; sweepgraph.hpp:54-396) on an arbitrary digraph with
 * edges[2*ne] (from, to) and weights[ne]; writes order[nv], lagged[<= ne]
 * (edge ids, ascending) and the cut weight.  Returns the number of lagged
 * edges, or a negative status. */
int hsw_debug_graph_order(int nv, int ne, const int* edges, const double* weights, int threshold, int* order,
                          int* lagged, double* lagged_weight);

/* Test hook mirroring test_solver.cpp:332-344 for the constructor check: the
 * next hsw_create on the calling thread zeroes the (e, d) local block from the
 * start, so check_local_blocks reports it as SolverError at construction. */
int hsw_debug_create_zero_block(int e, int d);

/* Test hook mirroring test_solver.cpp:332-344 (op.ordinates[d].diag[e].setZero()):
 * zero the assembled local block of (e, d) in every later factorization. */
int hsw_debug_zero_block(hsw_handle* h, int e, int d);

#ifdef __cplusplus
}
#endif
#endif /* HOSWEEP_B200_H */
