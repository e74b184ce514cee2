// hosweep_b200/solver.hpp — C++ drop-in for hosweep::SweepSolver
// (/root/reference/proj/include/hosweep/solver.hpp:50-203) over the C ABI in
// hosweep_b200.h.  Same method names, argument meaning, result types (with
// std::vector<double> in place of Eigen::VectorXd, element-major layout
// e*n + m) and exception types (SolverError, MeshError, GeometryError,
// AssemblyError, std::out_of_range, std::logic_error, std::invalid_argument).
// Header-only; link against libhosweep_b200.so.
#pragma once

#include "hosweep_b200.h"

#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace hosweep_b200 {

struct SolverError : std::runtime_error { using std::runtime_error::runtime_error; };    // solver.hpp:21-23
struct MeshError : std::runtime_error { using std::runtime_error::runtime_error; };      // mesh.hpp:23-25
struct GeometryError : std::runtime_error { using std::runtime_error::runtime_error; };  // mesh.hpp:27-29
struct AssemblyError : std::runtime_error { using std::runtime_error::runtime_error; };  // assembly.hpp:24-26
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

inline std::string last_error() {
    char buf[2048];
    hsw_last_error(buf, sizeof(buf));
    return buf;
}

inline void check(int rc) {
    if (rc == HSW_OK) return;
    const std::string msg = last_error();
    switch (rc) {
        case HSW_ERR_MESH: throw MeshError(msg);
        case HSW_ERR_GEOMETRY: throw GeometryError(msg);
        case HSW_ERR_ASSEMBLY: throw AssemblyError(msg);
        case HSW_ERR_SOLVER: throw SolverError(msg);
        case HSW_ERR_LOGIC: throw std::logic_error(msg);
        case HSW_ERR_RANGE: throw std::out_of_range(msg);
        case HSW_ERR_NOMEM: throw std::bad_alloc();
        case HSW_ERR_CUDA: throw DeviceError(msg);
        default: throw std::invalid_argument(msg);
    }
}

enum class EdgeWeighting { unity = HSW_WEIGHT_UNITY, face = HSW_WEIGHT_FACE, sig_inv_face = HSW_WEIGHT_SIGINVFACE };

// solver.hpp:25-32 (+ the configs' relative-phi stopping criterion)
struct SolveOptions {
    enum class Mode { sweep, direct_oracle };
    enum class Criterion { psi_linf, phi_rel_l2 };
    double tolerance = 1e-14;
    int max_iterations = 400;
    Mode mode = Mode::sweep;
    EdgeWeighting weighting = EdgeWeighting::face;
    int exact_fas_threshold = 10;
    Criterion criterion = Criterion::psi_linf;
};

// sweepgraph.hpp:318-325 (+ the level of each element in the B200 worklist)
struct SweepOrdering {
    std::vector<int> order, position, lagged_edges, level;
    double lagged_weight = 0.0;
    bool is_lagged_position(int from, int to) const { return position[from] > position[to]; }
};

struct ConvergenceHistory {  // solver.hpp:34-39
    std::vector<double> error;                      // per iteration, max over ordinates of ||dpsi||_inf
    std::vector<std::vector<double>> per_ordinate;  // error[it][d] (solver.hpp:36)
    std::vector<double> phi_rel;                    // per iteration ||dphi||_2 / ||phi||_2
    bool converged = false;
    double seconds = 0.0;         // device time
    int iterations() const { return static_cast<int>(error.size()); }
};

struct SolverState {  // solver.hpp:41-45
    std::vector<std::vector<double>> psi;
    std::vector<double> phi;
    int iterations = 0;
};

class SweepSolver {
  public:
    // Replaces assemble_transport_operator + SweepSolver(op, opts): the
    // descriptor carries the mesh, basis order, ordinates, cross sections and
    // source (see hosweep_b200.h); options.weighting / exact_fas_threshold
    // override the descriptor's graph knobs.
    // The reference constructor factors every local block and throws SolverError
    // for a singular one (solver.hpp:67-75); check_local_blocks is therefore forced
    // on here (one sweep on zero data at construction).
    explicit SweepSolver(hsw_problem_desc desc, const SolveOptions& opts = {}) : opts_(opts) {
        desc.abi_version = HSW_ABI_VERSION;
        desc.check_local_blocks = 1;
        desc.weighting = static_cast<int>(opts.weighting);
        desc.exact_fas_threshold = opts.exact_fas_threshold;
        hsw_handle* h = nullptr;
        check(hsw_create(&desc, &h));
        h_.reset(h);
        int64_t sz[6];
        check(hsw_sizes(h, sz));
        nel_ = (int)sz[0];
        nb_ = (int)sz[1];
        nd_ = (int)sz[2];
        orderings_.resize(nd_);
        ordering_once_ = std::make_unique<std::once_flag[]>(nd_);
    }

    const SolveOptions& options() const { return opts_; }
    int num_ordinates() const { return nd_; }
    int block_size() const { return nb_; }
    int num_elements() const { return nel_; }
    int num_dofs() const { return nel_ * nb_; }

    // solver.hpp:80 (throws std::out_of_range like .at())
    const SweepOrdering& ordering(int d) const {
        if (d < 0 || d >= nd_) throw std::out_of_range("SweepSolver::ordering: ordinate " + std::to_string(d));
        auto& slot = orderings_[d];
        // filled once per ordinate; safe under concurrent callers (the reference's
        // orderings_ are built in the constructor and only read afterwards)
        std::call_once(ordering_once_[d], [&] {
            auto o = std::make_unique<SweepOrdering>();
            o->order.resize(nel_);
            o->position.resize(nel_);
            o->level.resize(nel_);
            int nl = 0;
            check(hsw_ordering(h_.get(), d, o->order.data(), o->position.data(), nullptr, 0, &nl, &o->lagged_weight,
                               o->level.data()));
            o->lagged_edges.resize(nl);
            check(hsw_ordering(h_.get(), d, nullptr, nullptr, o->lagged_edges.data(), nl, nullptr, nullptr, nullptr));
            slot = std::move(o);
        });
        return *slot;
    }

    int total_lagged_edges() const {  // solver.hpp:83-87
        int64_t n = 0;
        check(hsw_total_lagged_edges(h_.get(), &n));
        return static_cast<int>(n);
    }

    std::vector<double> local_solve(int e, int d, const std::vector<double>& rhs) const {  // solver.hpp:91-93
        std::vector<double> out(nb_);
        check(hsw_local_solve(h_.get(), e, d, rhs.data(), out.data()));
        return out;
    }

    // solver.hpp:98-117: one lagged sweep of ordinate d
    std::vector<double> sweep(int d, const std::vector<double>& phi, const std::vector<double>& psi_old) const {
        std::vector<double> out(psi_old.size());
        check(hsw_sweep(h_.get(), d, phi.data(), psi_old.data(), out.data()));
        return out;
    }

    // solver.hpp:121-133
    std::vector<double> direct_oracle(int d, const std::vector<double>& phi) const {
        std::vector<double> out(num_dofs());
        check(hsw_direct_oracle(h_.get(), d, phi.data(), out.data()));
        return out;
    }

    // solver.hpp:136-168
    std::pair<SolverState, ConvergenceHistory> source_iteration() const {
        hsw_si_options o{};
        o.tolerance = opts_.tolerance;
        o.max_iterations = opts_.max_iterations;
        o.criterion = opts_.criterion == SolveOptions::Criterion::psi_linf ? HSW_CRIT_PSI_LINF : HSW_CRIT_PHI_REL_L2;
        o.mode = opts_.mode == SolveOptions::Mode::sweep ? HSW_MODE_SWEEP : HSW_MODE_DIRECT;
        hsw_si_result r{};
        const size_t N = (size_t)num_dofs();
        std::vector<double> psi(N * nd_), phi(N), err(opts_.max_iterations), rel(opts_.max_iterations);
        std::vector<double> per((size_t)opts_.max_iterations * nd_);
        check(hsw_source_iteration(h_.get(), &o, &r, psi.data(), phi.data(), err.data(), rel.data(), per.data()));
        SolverState s;
        s.psi.resize(nd_);
        for (int d = 0; d < nd_; ++d) s.psi[d].assign(psi.begin() + d * N, psi.begin() + (d + 1) * N);
        s.phi = std::move(phi);
        s.iterations = r.iterations;
        ConvergenceHistory hst;
        hst.error.assign(err.begin(), err.begin() + r.iterations);
        hst.phi_rel.assign(rel.begin(), rel.begin() + r.iterations);
        for (int it = 0; it < r.iterations; ++it)
            hst.per_ordinate.emplace_back(per.begin() + (size_t)it * nd_, per.begin() + (size_t)(it + 1) * nd_);
        hst.converged = r.converged != 0;
        hst.seconds = r.seconds;
        return {std::move(s), std::move(hst)};
    }

    hsw_handle* handle() const { return h_.get(); }

  private:
    struct Del { void operator()(hsw_handle* h) const { hsw_destroy(h); } };
    std::unique_ptr<hsw_handle, Del> h_;
    SolveOptions opts_;
    int nel_ = 0, nb_ = 0, nd_ = 0;
    mutable std::vector<std::unique_ptr<SweepOrdering>> orderings_;
    std::unique_ptr<std::once_flag[]> ordering_once_;
};

// solver.hpp:209-245 balance_report: conservation functionals of a state
struct BalanceReport {
    double source_volume = 0.0, inflow = 0.0, source_total = 0.0, absorption = 0.0, outflow = 0.0,
           net_leakage = 0.0, residual = 0.0;
    std::map<int, double> outflow_by_attr;   // keyed by boundary attribute
};

namespace detail {
inline BalanceReport balance_from(const double out5[5], const int* attrs, const double* vals, int n) {
    BalanceReport r;
    r.source_volume = out5[0];
    r.inflow = out5[1];
    r.source_total = out5[0] + out5[1];
    r.absorption = out5[2];
    r.outflow = out5[3];
    r.net_leakage = out5[3] - out5[1];
    r.residual = out5[4];
    for (int i = 0; i < n; ++i) r.outflow_by_attr[attrs[i]] = vals[i];
    return r;
}
}  // namespace detail

// balance_report(op, state) for a state held on the host
inline BalanceReport balance_report(const SweepSolver& s, const SolverState& st) {
    const size_t N = (size_t)s.num_dofs();
    std::vector<double> psi(N * (size_t)s.num_ordinates());
    for (int d = 0; d < s.num_ordinates(); ++d) std::copy(st.psi[d].begin(), st.psi[d].end(), psi.begin() + d * N);
    double out5[5];
    int attrs[64], cnt = 0;
    double vals[64];
    check(hsw_balance(s.handle(), psi.data(), st.phi.data(), out5, attrs, vals, 64, &cnt));
    return detail::balance_from(out5, attrs, vals, cnt < 64 ? cnt : 64);
}

// balance_report of the solver's converged state while it is still on the device
// (after source_iteration(); no host round trip of psi)
inline BalanceReport balance_report_resident(const SweepSolver& s) {
    double out5[5];
    int attrs[64], cnt = 0;
    double vals[64];
    check(hsw_balance_resident(s.handle(), out5, attrs, vals, 64, &cnt));
    return detail::balance_from(out5, attrs, vals, cnt < 64 ? cnt : 64);
}

}  // namespace hosweep_b200
