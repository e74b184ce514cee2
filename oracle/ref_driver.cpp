// Driver for the REFERENCE'S OWN solver path — TEST INFRASTRUCTURE ONLY.
//
// Compiled by `make -C oracle ref` from the reference headers where they lie
// (/root/reference/proj/include/hosweep: solver.hpp -> assembly.hpp,
// sweepgraph.hpp, mesh.hpp, basis.hpp, quadrature.hpp, romberg.hpp, xsec.hpp,
// angular.hpp, parallel.hpp) against the Eigen-subset shim in
// oracle/eigen_shim/, into oracle/_ref/ref_driver (git-ignored; nothing is
// copied from the reference).  tests/golden/make_ref_golden.py feeds it a 2D
// problem written as raw arrays and turns its outputs into the committed
// fixtures tests/golden/ref_*.npz, which pin the CPU oracle
// (oracle/hosweep_oracle.cpp) and the B200 product to the reference itself.
//
// usage: ref_driver IN_DIR OUT_DIR
//   IN_DIR/meta.txt: "p r np ne nbf nd nreg src_kind face_rule face_points
//                     volume_points inflow si_tol si_max direct_count"
//   raw arrays: pts (np x 2 f64), nodes (ne x (r+1)^2 i32), reg (ne i32),
//   bf (nbf x 3 i32), w (nd f64), dir (nd x 3 f64), ids/st/ss (nreg),
//   src (8 f64), phi (N f64), psi_old (nd x N f64), rhs (n f64)
// Calls made (the reference API, solver.hpp:50-245):
//   HighOrderMesh::build, assemble_transport_operator (Gauss or Romberg face
//   rule), SweepSolver(op, opts), ordering(d), total_lagged_edges(),
//   sweep(d, phi, psi_old) for every d, local_solve(e, d, rhs),
//   direct_oracle(d, phi) for the first `direct_count` ordinates,
//   source_iteration() and balance_report().
#include "hosweep/solver.hpp"

#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

using namespace hosweep;

template <typename T>
static std::vector<T> rd(const std::string& dir, const char* name, size_t n) {
    std::vector<T> v(n);
    std::ifstream f(dir + "/" + name, std::ios::binary);
    if (!f) throw std::runtime_error(std::string("ref_driver: missing input ") + name);
    f.read(reinterpret_cast<char*>(v.data()), (std::streamsize)(n * sizeof(T)));
    if ((size_t)f.gcount() != n * sizeof(T)) throw std::runtime_error(std::string("ref_driver: short input ") + name);
    return v;
}

struct Out {
    std::string dir;
    std::ofstream manifest;
    explicit Out(const std::string& d) : dir(d), manifest(d + "/manifest.txt") {}
    template <typename T>
    void put(const std::string& name, const std::vector<T>& v, const char* dtype) {
        std::ofstream f(dir + "/" + name + ".bin", std::ios::binary);
        f.write(reinterpret_cast<const char*>(v.data()), (std::streamsize)(v.size() * sizeof(T)));
        manifest << name << " " << dtype << " " << v.size() << "\n";
    }
    void f64(const std::string& n, const std::vector<double>& v) { put(n, v, "f8"); }
    void i32(const std::string& n, const std::vector<int>& v) { put(n, v, "i4"); }
};

static std::vector<double> vec(const Eigen::VectorXd& v) { return std::vector<double>(v.data(), v.data() + v.size()); }

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: ref_driver IN_DIR OUT_DIR\n");
        return 2;
    }
    const std::string in = argv[1];
    Out out(argv[2]);
    std::ifstream mf(in + "/meta.txt");
    int p, r, np, ne, nbf, nd, nreg, src_kind, face_rule, face_points, volume_points, si_max, direct_count;
    double inflow, si_tol;
    mf >> p >> r >> np >> ne >> nbf >> nd >> nreg >> src_kind >> face_rule >> face_points >> volume_points >> inflow >>
        si_tol >> si_max >> direct_count;
    if (!mf) throw std::runtime_error("ref_driver: bad meta.txt");
    const int npe = (r + 1) * (r + 1);
    const auto pts = rd<double>(in, "pts", (size_t)np * 2);
    const auto nodes = rd<int>(in, "nodes", (size_t)ne * npe);
    const auto reg = rd<int>(in, "reg", ne);
    const auto bf = rd<int>(in, "bf", (size_t)nbf * 3);
    const auto w = rd<double>(in, "w", nd);
    const auto dir = rd<double>(in, "dir", (size_t)nd * 3);
    const auto ids = rd<int>(in, "ids", nreg);
    const auto st = rd<double>(in, "st", nreg);
    const auto ss = rd<double>(in, "ss", nreg);
    const auto sp = rd<double>(in, "src", 8);

    // ---- mesh (mesh.hpp:121-134) from the raw arrays
    std::vector<Vec2> cps(np);
    for (int i = 0; i < np; ++i) cps[i] = Vec2(pts[2 * i], pts[2 * i + 1]);
    std::vector<ElementRecord> els(ne);
    for (int e = 0; e < ne; ++e) {
        els[e].nodes.assign(nodes.begin() + (size_t)e * npe, nodes.begin() + (size_t)(e + 1) * npe);
        els[e].region = reg[e];
    }
    std::vector<BoundaryFace> bfs(nbf);
    for (int b = 0; b < nbf; ++b) bfs[b] = {bf[3 * b], bf[3 * b + 1], bf[3 * b + 2]};
    const HighOrderMesh mesh = HighOrderMesh::build(r, cps, els, bfs);
    const ReferenceBasis basis(p);
    AngularQuadrature quad;
    for (int d = 0; d < nd; ++d) quad.ordinates.push_back({w[d], {dir[3 * d], dir[3 * d + 1], dir[3 * d + 2]}});
    std::map<int, CrossSections> table;
    for (int i = 0; i < nreg; ++i) table[ids[i]] = {st[i], ss[i]};
    const CrossSectionField xsec = CrossSectionField::by_region(table);
    SourceSpec src;
    if (src_kind == 0) {
        src = SourceSpec::isotropic(sp[0], inflow);
    } else {   // disc indicator at physical quadrature points (assembly.hpp:298)
        const double cx = sp[0], cy = sp[1], R = sp[3], qin = sp[4], qout = sp[5];
        src.volumetric = [=](int, const Vec2& x) {
            const double dx = x[0] - cx, dy = x[1] - cy;
            return dx * dx + dy * dy < R * R ? qin : qout;
        };
        src.incident = [inflow](int, const Vec2&) { return inflow; };
    }
    AssemblyOptions ao;
    ao.volume_points_per_axis = volume_points;
    ao.face.rule = face_rule == 0 ? FaceIntegration::Rule::gauss : FaceIntegration::Rule::romberg;
    ao.face.gauss_points = face_points > 0 ? face_points : p + 2;
    const TransportOperator op = assemble_transport_operator(mesh, basis, quad, xsec, src, ao);

    // ---- interior faces (mesh.hpp:275-339)
    {
        std::vector<int> f;
        for (const FaceRecord& fr : mesh.interior_faces())
            for (int x : {fr.elem_left, fr.elem_right, fr.local_face_left, fr.local_face_right, fr.orientation})
                f.push_back(x);
        out.i32("interior_faces", f);
    }
    SolveOptions so;
    so.tolerance = si_tol;
    so.max_iterations = si_max;
    const SweepSolver solver(op, so);

    // ---- per-ordinate plan: couplings, weights, lag flags, ordering (sweepgraph.hpp:54-396)
    std::vector<int> cpl, cpl_off{0}, order, lag, lag_off{0}, unconv;
    std::vector<double> weights, lag_w;
    for (int d = 0; d < nd; ++d) {
        const auto& o = op.ordinates[d];
        const DependencyGraph g = build_graph(op, d, so.weighting);
        const SweepOrdering& so_d = solver.ordering(d);
        for (size_t c = 0; c < o.couplings.size(); ++c) {
            const FaceCoupling& fc = o.couplings[c];
            cpl.insert(cpl.end(), {fc.face, fc.downwind, fc.upwind,
                                   so_d.is_lagged_position(fc.upwind, fc.downwind) ? 1 : 0});
            weights.push_back(g.edges[c].weight);
        }
        cpl_off.push_back((int)(cpl.size() / 4));
        order.insert(order.end(), so_d.order.begin(), so_d.order.end());
        lag.insert(lag.end(), so_d.lagged_edges.begin(), so_d.lagged_edges.end());
        lag_off.push_back((int)lag.size());
        lag_w.push_back(so_d.lagged_weight);
        unconv.push_back(o.unconverged_faces);
    }
    out.i32("couplings", cpl);
    out.i32("couplings_offsets", cpl_off);
    out.f64("edge_weights", weights);
    out.i32("order", order);
    out.i32("lagged_edges", lag);
    out.i32("lagged_offsets", lag_off);
    out.f64("lagged_weight", lag_w);
    out.i32("unconverged_faces", unconv);
    out.i32("total_lagged_edges", {solver.total_lagged_edges()});

    // ---- one lagged sweep of every ordinate (solver.hpp:98-117)
    const int nu = op.block_size();
    const size_t N = (size_t)op.num_dofs();
    const auto phi_v = rd<double>(in, "phi", N);
    const auto psi_old_v = rd<double>(in, "psi_old", N * nd);
    Eigen::VectorXd phi(N);
    for (size_t i = 0; i < N; ++i) phi[i] = phi_v[i];
    std::vector<double> sw;
    for (int d = 0; d < nd; ++d) {
        Eigen::VectorXd po(N);
        for (size_t i = 0; i < N; ++i) po[i] = psi_old_v[(size_t)d * N + i];
        const auto x = vec(solver.sweep(d, phi, po));
        sw.insert(sw.end(), x.begin(), x.end());
    }
    out.f64("sweep", sw);

    // ---- local_solve of element 0 / last, every ordinate (solver.hpp:91-93)
    {
        const auto rhs_v = rd<double>(in, "rhs", nu);
        Eigen::VectorXd rhs(nu);
        for (int i = 0; i < nu; ++i) rhs[i] = rhs_v[i];
        std::vector<double> ls;
        for (int d = 0; d < nd; ++d)
            for (int e : {0, ne - 1}) {
                const auto x = vec(solver.local_solve(e, d, rhs));
                ls.insert(ls.end(), x.begin(), x.end());
            }
        out.f64("local_solve", ls);
    }
    // ---- direct_oracle (solver.hpp:121-133)
    {
        std::vector<double> dor;
        for (int d = 0; d < std::min(direct_count, nd); ++d) {
            const auto x = vec(solver.direct_oracle(d, phi));
            dor.insert(dor.end(), x.begin(), x.end());
        }
        out.f64("direct_oracle", dor);
    }
    // ---- source iteration + balance (solver.hpp:136-168, 220-245)
    if (si_max > 0) {
        const auto [state, hist] = solver.source_iteration();
        std::vector<double> psi;
        for (const auto& v : state.psi) {
            const auto x = vec(v);
            psi.insert(psi.end(), x.begin(), x.end());
        }
        out.f64("si_psi", psi);
        out.f64("si_phi", vec(state.phi));
        out.f64("si_error", hist.error);
        std::vector<double> per;
        for (const auto& row : hist.per_ordinate) per.insert(per.end(), row.begin(), row.end());
        out.f64("si_per_ordinate", per);
        out.i32("si_iterations", {state.iterations, hist.converged ? 1 : 0});
        const BalanceReport b = balance_report(op, state);
        out.f64("balance", {b.source_volume, b.inflow, b.absorption, b.outflow, b.residual});
        std::vector<int> attrs;
        std::vector<double> vals;
        for (const auto& [a, v] : b.outflow_by_attr) {
            attrs.push_back(a);
            vals.push_back(v);
        }
        out.i32("balance_attrs", attrs);
        out.f64("balance_attr_outflow", vals);
    }
    std::puts("ref_driver ok");
    return 0;
}
