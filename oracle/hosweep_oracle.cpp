// =============================================================================
// hosweep ORACLE — CPU restatement of the reference transport-sweep path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load this library, and
// only as the checker or the timed CPU baseline.  The product
// (paper_1810_11080_b200/) never links, loads or calls it.
//
// It restates, file by file and in the same arithmetic order, the reference
// header-only library under /root/reference/proj/include/hosweep/:
//   quadrature.hpp:23-104   gauss_legendre, gauss_lobatto, tensor rule
//   basis.hpp:15-133        Lagrange1D (product form), nodal tensor basis
//   mesh.hpp:64-365         reference faces, map/jacobian/face_geometry,
//                           build_faces (corner-key std::map pairing), checks
//   xsec.hpp:20-67          per-region cross sections
//   assembly.hpp:58-409     element quad data, volume blocks, Gauss face rule
//                           (FaceIntegration::Rule::gauss), source moments
//   sweepgraph.hpp:54-396   build_graph, tarjan_scc, min_fas_exact,
//                           min_fas_heuristic, sweep_ordering
//   solver.hpp:52-168       SweepSolver ctor (lag flags, LU + rcond check),
//                           local_solve, sweep, direct_oracle, source_iteration
//   solver.hpp:220-245      balance_report
//   parallel.hpp:16-54      per-ordinate worker pool (HOSWEEP_THREADS)
// and generalises it to 3D hexahedra (the reference is 2D only,
// SPEC.md:11): tensor basis with m = (iz*(p+1)+iy)*(p+1)+ix, six faces,
// sorted-4-corner face keys with an 8-case orientation code, surface
// Jacobian |J t1 x J t2|, normal normalize(J^-T n_ref).  See DESIGN.md §3 for
// the exact conventions; the product's host code restates the same
// arithmetic independently so graph weights and cut sets are bit-identical.
//
// Eigen is absent in this image, so the dense kernels (LU with partial
// pivoting, products) are written out here; the arithmetic order of every
// quantity that feeds an integer decision (edge existence, FAS weights) is
// the reference's element-wise order, which is Eigen-independent
// (assembly.hpp:197-241).  Compile with -ffp-contract=off.
// =============================================================================
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

struct MeshError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GeometryError : std::runtime_error { using std::runtime_error::runtime_error; };
struct AssemblyError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IntegrationError : std::runtime_error { using std::runtime_error::runtime_error; };  // romberg.hpp:15-17

// romberg.hpp:33-88: Romberg tableau over successive trapezoid halvings of [0,1] for a
// vector integrand f(t, out[nv]) (all components share one sampling).  Converged when two
// successive diagonal entries agree to tol in the max norm, not before min_levels
// halvings; otherwise the last diagonal entry is returned unconverged.  Elementwise
// arithmetic in the reference's order (Eigen expressions evaluate coefficient-wise).
template <typename F>
static bool romberg_vec(F&& f, size_t nv, double tol, int max_levels, int min_levels, std::vector<double>& out) {
    if (tol <= 0.0) throw std::invalid_argument("romberg: tol must be positive");
    if (max_levels < 1) throw std::invalid_argument("romberg: need max_levels >= 1");
    min_levels = std::min(min_levels, max_levels);
    auto nan_check = [&](const std::vector<double>& v) {
        for (double x : v)
            if (std::isnan(x)) throw IntegrationError("romberg: integrand returned NaN");
    };
    std::vector<double> f0(nv), f1(nv), trap(nv), sum(nv), fi(nv);
    f(0.0, f0.data());
    f(1.0, f1.data());
    nan_check(f0);
    nan_check(f1);
    for (size_t i = 0; i < nv; ++i) trap[i] = 0.5 * (f0[i] + f1[i]);
    std::vector<std::vector<double>> diag{trap}, row;
    bool converged = false;
    long n = 1;
    for (int k = 1; k <= max_levels; ++k) {
        const double h = 1.0 / (2.0 * n);
        f(h, sum.data());
        nan_check(sum);
        for (long i = 1; i < n; ++i) {
            f((2 * i + 1) * h, fi.data());
            nan_check(fi);
            for (size_t j = 0; j < nv; ++j) sum[j] += fi[j];
        }
        for (size_t j = 0; j < nv; ++j) trap[j] = 0.5 * trap[j] + h * sum[j];
        n *= 2;
        row.assign(1, trap);
        double pow4 = 1.0;
        for (int j = 1; j <= k; ++j) {
            pow4 *= 4.0;
            std::vector<double> r(nv);
            for (size_t i = 0; i < nv; ++i) r[i] = row[j - 1][i] + (row[j - 1][i] - diag[j - 1][i]) / (pow4 - 1.0);
            row.push_back(std::move(r));
        }
        double diff = 0.0;
        for (size_t i = 0; i < nv; ++i) diff = std::max(diff, std::abs(row[k][i] - diag[k - 1][i]));
        diag.swap(row);
        if (diff < tol && k >= min_levels) {
            converged = true;
            break;
        }
    }
    out = diag.back();
    return converged;
}
struct SolverError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- parallel.hpp
// parallel.hpp:16-23
static int max_workers() {
    if (const char* env = std::getenv("HOSWEEP_THREADS")) {
        const int n = std::atoi(env);
        if (n >= 1) return n;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}

// parallel.hpp:27-54 (first exception rethrown on the caller)
template <typename Fn>
static void parallel_for(int n, Fn&& fn) {
    const int workers = std::min(n, max_workers());
    if (workers <= 1) {
        for (int i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    std::exception_ptr error;
    std::mutex error_mutex;
    std::atomic<int> next{0};
    for (int w = 0; w < workers; ++w)
        pool.emplace_back([&] {
            for (;;) {
                const int i = next.fetch_add(1);
                if (i >= n) return;
                try {
                    fn(i);
                } catch (...) {
                    std::lock_guard<std::mutex> lock(error_mutex);
                    if (!error) error = std::current_exception();
                    return;
                }
            }
        });
    for (auto& t : pool) t.join();
    if (error) std::rethrow_exception(error);
}

// -------------------------------------------------------------- quadrature.hpp
struct Quad1D {
    std::vector<double> points, weights;
    int size() const { return (int)points.size(); }
};

// quadrature.hpp:23-34
static void legendre(int n, double x, double& p, double& dp) {
    double p0 = 1.0, p1 = x;
    if (n == 0) { p = p0; dp = 0.0; return; }
    for (int k = 2; k <= n; ++k) {
        const double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
    }
    p = p1;
    dp = n * (x * p1 - p0) / (x * x - 1.0);
}

// quadrature.hpp:38-59
static Quad1D gauss_legendre(int n) {
    if (n < 1) throw std::invalid_argument("gauss_legendre: need n >= 1");
    Quad1D r;
    r.points.resize(n);
    r.weights.resize(n);
    for (int i = 0; i < n; ++i) {
        double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        double p = 0.0, dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            legendre(n, x, p, dp);
            const double dx = p / dp;
            x -= dx;
            if (std::abs(dx) < 1e-15) break;
        }
        legendre(n, x, p, dp);
        r.points[n - 1 - i] = 0.5 * (x + 1.0);
        r.weights[n - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);
    }
    return r;
}

// quadrature.hpp:62-82
static std::vector<double> gauss_lobatto(int n) {
    if (n < 2) throw std::invalid_argument("gauss_lobatto: need n >= 2");
    std::vector<double> pts(n);
    pts.front() = 0.0;
    pts.back() = 1.0;
    const int m = n - 1;
    for (int i = 1; i < m; ++i) {
        double x = std::cos(M_PI * i / m);
        for (int it = 0; it < 100; ++it) {
            double p, dp;
            legendre(m, x, p, dp);
            const double ddp = (2.0 * x * dp - m * (m + 1) * p) / (1.0 - x * x);
            const double dx = dp / ddp;
            x -= dx;
            if (std::abs(dx) < 1e-15) break;
        }
        pts[m - i] = 0.5 * (x + 1.0);
    }
    return pts;
}

// quadrature.hpp:85-104, generalised to dim 3 (i fastest, weight (wi*wj)*wk)
struct VolQuad {
    int dim = 2;
    std::vector<std::array<double, 3>> points;
    std::vector<double> weights;
    int size() const { return (int)weights.size(); }
};
static VolQuad tensor_gauss(int dim, int per_axis) {
    const Quad1D line = gauss_legendre(per_axis);
    VolQuad q;
    q.dim = dim;
    if (dim == 2) {
        for (int j = 0; j < per_axis; ++j)
            for (int i = 0; i < per_axis; ++i) {
                q.points.push_back({line.points[i], line.points[j], 0.0});
                q.weights.push_back(line.weights[i] * line.weights[j]);
            }
    } else {
        for (int k = 0; k < per_axis; ++k)
            for (int j = 0; j < per_axis; ++j)
                for (int i = 0; i < per_axis; ++i) {
                    q.points.push_back({line.points[i], line.points[j], line.points[k]});
                    q.weights.push_back(line.weights[i] * line.weights[j] * line.weights[k]);
                }
    }
    return q;
}

// ------------------------------------------------------------------- basis.hpp
// basis.hpp:15-60
struct Lagrange1D {
    std::vector<double> nodes;
    int size() const { return (int)nodes.size(); }
    double value(int j, double x) const {
        const int n = size();
        double v = 1.0;
        for (int k = 0; k < n; ++k) {
            if (k == j) continue;
            v *= (x - nodes[k]) / (nodes[j] - nodes[k]);
        }
        return v;
    }
    double derivative(int j, double x) const {
        const int n = size();
        double d = 0.0;
        for (int i = 0; i < n; ++i) {
            if (i == j) continue;
            double term = 1.0 / (nodes[j] - nodes[i]);
            for (int k = 0; k < n; ++k) {
                if (k == j || k == i) continue;
                term *= (x - nodes[k]) / (nodes[j] - nodes[k]);
            }
            d += term;
        }
        return d;
    }
};

// basis.hpp:62-133 (2D), generalised: node m = (iz*n1 + iy)*n1 + ix.
struct Basis {
    int dim = 2, order = 1, n1 = 2, nb = 4;
    Lagrange1D line;
    Basis() = default;
    Basis(int d, int p) : dim(d), order(p), n1(p + 1) {
        if (p < 1 || p >= 32) throw std::invalid_argument("ReferenceBasis: order out of range");
        line.nodes = gauss_lobatto(p + 1);
        nb = d == 2 ? n1 * n1 : n1 * n1 * n1;
    }
    int size() const { return nb; }
    void node(int m, double* xi) const {
        xi[0] = line.nodes[m % n1];
        xi[1] = line.nodes[(m / n1) % n1];
        if (dim == 3) xi[2] = line.nodes[m / (n1 * n1)];
    }
    // basis.hpp:98-108
    void values(const double* xi, double* out) const {
        double vx[32], vy[32], vz[32];
        for (int j = 0; j < n1; ++j) vx[j] = line.value(j, xi[0]);
        for (int j = 0; j < n1; ++j) vy[j] = line.value(j, xi[1]);
        if (dim == 2) {
            for (int iy = 0; iy < n1; ++iy)
                for (int ix = 0; ix < n1; ++ix) out[iy * n1 + ix] = vx[ix] * vy[iy];
        } else {
            for (int j = 0; j < n1; ++j) vz[j] = line.value(j, xi[2]);
            for (int iz = 0; iz < n1; ++iz)
                for (int iy = 0; iy < n1; ++iy)
                    for (int ix = 0; ix < n1; ++ix)
                        out[(iz * n1 + iy) * n1 + ix] = vx[ix] * vy[iy] * vz[iz];
        }
    }
    // basis.hpp:111-126; out[m*dim + k] = d u_m / d xi_k
    void gradients(const double* xi, double* out) const {
        double vx[32], vy[32], vz[32], dx[32], dy[32], dz[32];
        for (int j = 0; j < n1; ++j) vx[j] = line.value(j, xi[0]);
        for (int j = 0; j < n1; ++j) vy[j] = line.value(j, xi[1]);
        for (int j = 0; j < n1; ++j) dx[j] = line.derivative(j, xi[0]);
        for (int j = 0; j < n1; ++j) dy[j] = line.derivative(j, xi[1]);
        if (dim == 2) {
            for (int iy = 0; iy < n1; ++iy)
                for (int ix = 0; ix < n1; ++ix) {
                    const int m = iy * n1 + ix;
                    out[m * 2 + 0] = dx[ix] * vy[iy];
                    out[m * 2 + 1] = vx[ix] * dy[iy];
                }
        } else {
            for (int j = 0; j < n1; ++j) vz[j] = line.value(j, xi[2]);
            for (int j = 0; j < n1; ++j) dz[j] = line.derivative(j, xi[2]);
            for (int iz = 0; iz < n1; ++iz)
                for (int iy = 0; iy < n1; ++iy)
                    for (int ix = 0; ix < n1; ++ix) {
                        const int m = (iz * n1 + iy) * n1 + ix;
                        out[m * 3 + 0] = dx[ix] * vy[iy] * vz[iz];
                        out[m * 3 + 1] = vx[ix] * dy[iy] * vz[iz];
                        out[m * 3 + 2] = vx[ix] * vy[iy] * dz[iz];
                    }
        }
    }
};

// ------------------------------------------------------------ reference faces
// 2D: mesh.hpp:64-109.  3D (new): 0 z=0 (s,t,0); 1 y=0 (s,0,t); 2 x=1 (1,s,t);
// 3 y=1 (s,1,t); 4 x=0 (0,s,t); 5 z=1 (s,t,1).
static int num_faces(int dim) { return dim == 2 ? 4 : 6; }

static void param_point(int dim, int f, double s, double t, double* xi) {
    if (dim == 2) {
        switch (f) {
            case 0: xi[0] = s; xi[1] = 0.0; return;
            case 1: xi[0] = 1.0; xi[1] = s; return;
            case 2: xi[0] = s; xi[1] = 1.0; return;
            case 3: xi[0] = 0.0; xi[1] = s; return;
        }
    } else {
        switch (f) {
            case 0: xi[0] = s; xi[1] = t; xi[2] = 0.0; return;
            case 1: xi[0] = s; xi[1] = 0.0; xi[2] = t; return;
            case 2: xi[0] = 1.0; xi[1] = s; xi[2] = t; return;
            case 3: xi[0] = s; xi[1] = 1.0; xi[2] = t; return;
            case 4: xi[0] = 0.0; xi[1] = s; xi[2] = t; return;
            case 5: xi[0] = s; xi[1] = t; xi[2] = 1.0; return;
        }
    }
    throw std::out_of_range("reface: bad local face index");
}
// reference-space axes of the face parameters (s -> axis0, t -> axis1)
static void face_axes(int dim, int f, int& a0, int& a1) {
    if (dim == 2) { a0 = (f == 0 || f == 2) ? 0 : 1; a1 = -1; return; }
    switch (f) {
        case 0: case 5: a0 = 0; a1 = 1; return;
        case 1: case 3: a0 = 0; a1 = 2; return;
        default: a0 = 1; a1 = 2; return;
    }
}
static void outward_normal(int dim, int f, double* n) {
    n[0] = n[1] = n[2] = 0.0;
    if (dim == 2) {
        static const double t[4][2] = {{0, -1}, {1, 0}, {0, 1}, {-1, 0}};
        n[0] = t[f][0]; n[1] = t[f][1];
    } else {
        static const double t[6][3] = {{0, 0, -1}, {0, -1, 0}, {1, 0, 0},
                                       {0, 1, 0},  {-1, 0, 0}, {0, 0, 1}};
        n[0] = t[f][0]; n[1] = t[f][1]; n[2] = t[f][2];
    }
}
// Local node indices on a face, ordered (s fastest, then t); ascending.
// 2D: mesh.hpp:93-107.
static std::vector<int> face_nodes(int dim, int f, int order) {
    const int n1 = order + 1;
    std::vector<int> idx;
    if (dim == 2) {
        for (int k = 0; k < n1; ++k) {
            switch (f) {
                case 0: idx.push_back(k); break;
                case 1: idx.push_back(order + k * n1); break;
                case 2: idx.push_back(order * n1 + k); break;
                case 3: idx.push_back(k * n1); break;
            }
        }
        return idx;
    }
    for (int b = 0; b < n1; ++b)
        for (int a = 0; a < n1; ++a) {
            int ix = 0, iy = 0, iz = 0;
            switch (f) {
                case 0: ix = a; iy = b; iz = 0; break;
                case 1: ix = a; iy = 0; iz = b; break;
                case 2: ix = order; iy = a; iz = b; break;
                case 3: ix = a; iy = order; iz = b; break;
                case 4: ix = 0; iy = a; iz = b; break;
                case 5: ix = a; iy = b; iz = order; break;
            }
            idx.push_back((iz * n1 + iy) * n1 + ix);
        }
    return idx;
}
// Orientation code: 2D 0 = same direction, 1 = reversed (mesh.hpp:299-309).
// 3D: bit2 swap (s,t), bit1 flip s, bit0 flip t, applied in that order.
static void orient_param(int dim, int code, double s, double t, double& so, double& to) {
    if (dim == 2) { so = code ? 1.0 - s : s; to = 0.0; return; }
    double u = s, v = t;
    if (code & 4) { u = t; v = s; }
    if (code & 2) u = 1.0 - u;
    if (code & 1) v = 1.0 - v;
    so = u; to = v;
}
static void orient_index(int dim, int code, int r, int a, int b, int& ao, int& bo) {
    if (dim == 2) { ao = code ? r - a : a; bo = 0; return; }
    int u = a, v = b;
    if (code & 4) { u = b; v = a; }
    if (code & 2) u = r - u;
    if (code & 1) v = r - v;
    ao = u; bo = v;
}

// -------------------------------------------------------------------- mesh.hpp
struct FaceRecord { int elem_left, elem_right, face_left, face_right, orientation; };
struct BoundaryFace { int elem, local_face, attr; };
struct FaceGeom { double point[3]; double normal[3]; double sj; };

struct Mesh {
    int dim = 2, order = 1;
    Basis geom;
    std::vector<double> pts;              // num_points * dim
    std::vector<std::vector<int>> elems;  // control node ids
    std::vector<int> region;
    std::vector<BoundaryFace> bfaces;
    std::vector<FaceRecord> ifaces;

    int num_elements() const { return (int)elems.size(); }
    int num_points() const { return (int)(pts.size() / dim); }

    // mesh.hpp:147-154
    void map_point(int e, const double* xi, double* x) const {
        std::vector<double> v(geom.size());
        geom.values(xi, v.data());
        x[0] = x[1] = x[2] = 0.0;
        const auto& el = elems[e];
        for (int m = 0; m < geom.size(); ++m)
            for (int a = 0; a < dim; ++a) x[a] += v[m] * pts[(size_t)el[m] * dim + a];
    }
    // mesh.hpp:157-170; J[a*3+b] = d x_a / d xi_b.  Returns det(J).
    double jacobian(int e, const double* xi, double* J) const {
        std::vector<double> g(geom.size() * dim);
        geom.gradients(xi, g.data());
        for (int i = 0; i < 9; ++i) J[i] = 0.0;
        const auto& el = elems[e];
        for (int m = 0; m < geom.size(); ++m) {
            const double* x = &pts[(size_t)el[m] * dim];
            for (int a = 0; a < dim; ++a)
                for (int b = 0; b < dim; ++b) J[a * 3 + b] += x[a] * g[m * dim + b];
        }
        return det(J);
    }
    double det(const double* J) const {
        if (dim == 2) return J[0] * J[4] - J[3] * J[1];  // Eigen 2x2 determinant
        const double c0 = J[4] * J[8] - J[5] * J[7];
        const double c1 = J[5] * J[6] - J[3] * J[8];
        const double c2 = J[3] * J[7] - J[4] * J[6];
        return J[0] * c0 + J[1] * c1 + J[2] * c2;
    }
    // K = J^{-1}, K[a*3+b]
    void inverse(const double* J, double* K) const {
        if (dim == 2) {  // Eigen compute_inverse_size2
            const double invdet = 1.0 / (J[0] * J[4] - J[3] * J[1]);
            K[0] = J[4] * invdet;
            K[3] = -J[3] * invdet;
            K[1] = -J[1] * invdet;
            K[4] = J[0] * invdet;
            return;
        }
        const double c00 = J[4] * J[8] - J[5] * J[7];
        const double c01 = J[5] * J[6] - J[3] * J[8];
        const double c02 = J[3] * J[7] - J[4] * J[6];
        const double invdet = 1.0 / (J[0] * c00 + J[1] * c01 + J[2] * c02);
        K[0] = c00 * invdet;
        K[1] = (J[2] * J[7] - J[1] * J[8]) * invdet;
        K[2] = (J[1] * J[5] - J[2] * J[4]) * invdet;
        K[3] = c01 * invdet;
        K[4] = (J[0] * J[8] - J[2] * J[6]) * invdet;
        K[5] = (J[2] * J[3] - J[0] * J[5]) * invdet;
        K[6] = c02 * invdet;
        K[7] = (J[1] * J[6] - J[0] * J[7]) * invdet;
        K[8] = (J[0] * J[4] - J[1] * J[3]) * invdet;
    }
    // mesh.hpp:204-217 (3D: max over the 8 corners)
    double element_diameter(int e) const {
        const int r = order, n1 = r + 1;
        std::vector<int> corners;
        if (dim == 2) corners = {0, r, r * n1, r * n1 + r};
        else
            for (int cz : {0, r})
                for (int cy : {0, r})
                    for (int cx : {0, r}) corners.push_back((cz * n1 + cy) * n1 + cx);
        double d = 0.0;
        const auto& el = elems[e];
        for (size_t i = 0; i < corners.size(); ++i)
            for (size_t j = i + 1; j < corners.size(); ++j) {
                double s = 0.0;
                for (int a = 0; a < dim; ++a) {
                    const double df = pts[(size_t)el[corners[i]] * dim + a] -
                                      pts[(size_t)el[corners[j]] * dim + a];
                    s += df * df;
                }
                d = std::max(d, std::sqrt(s));
            }
        return d;
    }
    // mesh.hpp:180-200; 3D: |J t1 x J t2|, normal = normalize(J^-T n_ref)
    FaceGeom face_geometry(int e, int f, double s, double t) const {
        double xi[3] = {0, 0, 0};
        param_point(dim, f, s, t, xi);
        double J[9];
        jacobian(e, xi, J);
        int a0, a1;
        face_axes(dim, f, a0, a1);
        double sj;
        if (dim == 2) {
            const double t0 = J[0 * 3 + a0], t1 = J[1 * 3 + a0];  // J * e_a0
            sj = std::sqrt(t0 * t0 + t1 * t1);
        } else {
            const double u0 = J[0 * 3 + a0], u1 = J[1 * 3 + a0], u2 = J[2 * 3 + a0];
            const double v0 = J[0 * 3 + a1], v1 = J[1 * 3 + a1], v2 = J[2 * 3 + a1];
            const double c0 = u1 * v2 - u2 * v1;
            const double c1 = u2 * v0 - u0 * v2;
            const double c2 = u0 * v1 - u1 * v0;
            sj = std::sqrt(c0 * c0 + c1 * c1 + c2 * c2);
        }
        if (sj < 1e-14 * element_diameter(e))
            throw GeometryError("face_geometry: degenerate tangent on element " +
                                std::to_string(e) + " face " + std::to_string(f));
        double K[9];
        inverse(J, K);
        double nref[3];
        outward_normal(dim, f, nref);
        FaceGeom fg{};
        double z = 0.0;
        for (int i = 0; i < dim; ++i) {
            double v = 0.0;
            for (int j = 0; j < dim; ++j) v += K[j * 3 + i] * nref[j];
            fg.normal[i] = v;
        }
        for (int i = 0; i < dim; ++i) z += fg.normal[i] * fg.normal[i];
        if (z > 0.0) {
            const double rt = std::sqrt(z);
            for (int i = 0; i < dim; ++i) fg.normal[i] /= rt;
        }
        map_point(e, xi, fg.point);
        fg.sj = sj;
        return fg;
    }
    std::vector<int> face_global_nodes(int e, int f) const {
        std::vector<int> out;
        for (int m : face_nodes(dim, f, order)) out.push_back(elems[e][m]);
        return out;
    }

    // mesh.hpp:242-262
    void check_connectivity() const {
        const int expected = geom.size();
        for (int e = 0; e < num_elements(); ++e) {
            if ((int)elems[e].size() != expected)
                throw MeshError("mesh: element " + std::to_string(e) + " has " +
                                std::to_string(elems[e].size()) + " nodes, expected " +
                                std::to_string(expected));
            for (int idx : elems[e])
                if (idx < 0 || idx >= num_points())
                    throw MeshError("mesh: element " + std::to_string(e) +
                                    " references control point " + std::to_string(idx) +
                                    " out of range");
        }
        for (const auto& b : bfaces)
            if (b.elem < 0 || b.elem >= num_elements() || b.local_face < 0 ||
                b.local_face >= num_faces(dim))
                throw MeshError("mesh: boundary face record (elem " + std::to_string(b.elem) +
                                ", face " + std::to_string(b.local_face) + ") out of range");
    }

    // mesh.hpp:275-339.  Key: 2D sorted (front, back) corner pair; 3D the sorted
    // four corner ids.  std::map iteration order defines interior-face ids.
    void build_faces() {
        ifaces.clear();
        const int nf = num_faces(dim);
        const int r = order, n1 = r + 1;
        std::map<std::array<int, 4>, std::vector<std::pair<int, int>>> by_corners;
        for (int e = 0; e < num_elements(); ++e)
            for (int f = 0; f < nf; ++f) {
                const std::vector<int> nodes = face_global_nodes(e, f);
                std::array<int, 4> key{};
                if (dim == 2) {
                    key = {nodes.front(), nodes.back(), -1, -1};
                    if (key[0] > key[1]) std::swap(key[0], key[1]);
                } else {
                    key = {nodes[0], nodes[r], nodes[r * n1], nodes[r * n1 + r]};
                    std::sort(key.begin(), key.end());
                }
                by_corners[key].push_back({e, f});
            }
        std::vector<std::vector<bool>> paired(num_elements(), std::vector<bool>(nf, false));
        for (const auto& kv : by_corners) {
            const auto& sides = kv.second;
            if (sides.size() > 2)
                throw MeshError("mesh: face shared by " + std::to_string(sides.size()) +
                                " elements");
            if (sides.size() != 2) continue;
            const auto [e0, f0] = sides[0];
            const auto [e1, f1] = sides[1];
            const std::vector<int> g0 = face_global_nodes(e0, f0);
            const std::vector<int> g1 = face_global_nodes(e1, f1);
            int orientation = -1;
            const int ncodes = dim == 2 ? 2 : 8;
            for (int code = 0; code < ncodes && orientation < 0; ++code) {
                bool ok = true;
                for (int b = 0; b < (dim == 2 ? 1 : n1) && ok; ++b)
                    for (int a = 0; a < n1 && ok; ++a) {
                        int ao, bo;
                        orient_index(dim, code, r, a, b, ao, bo);
                        if (g1[bo * n1 + ao] != g0[b * n1 + a]) ok = false;
                    }
                if (ok) orientation = code;
            }
            if (orientation < 0)
                throw MeshError("mesh: elements " + std::to_string(e0) + " and " +
                                std::to_string(e1) +
                                " share face corners but edge nodes do not match");
            ifaces.push_back({e0, e1, f0, f1, orientation});
            paired[e0][f0] = paired[e1][f1] = true;
        }
        std::vector<std::vector<bool>> declared(num_elements(), std::vector<bool>(nf, false));
        for (const auto& b : bfaces) {
            if (paired[b.elem][b.local_face])
                throw MeshError("mesh: boundary record for interior face (elem " +
                                std::to_string(b.elem) + ", face " +
                                std::to_string(b.local_face) + ")");
            if (declared[b.elem][b.local_face])
                throw MeshError("mesh: duplicate boundary record (elem " +
                                std::to_string(b.elem) + ", face " +
                                std::to_string(b.local_face) + ")");
            declared[b.elem][b.local_face] = true;
        }
        for (int e = 0; e < num_elements(); ++e)
            for (int f = 0; f < nf; ++f)
                if (!paired[e][f] && !declared[e][f])
                    throw MeshError("mesh: face (elem " + std::to_string(e) + ", face " +
                                    std::to_string(f) +
                                    ") is neither interior nor declared boundary");
    }

    // mesh.hpp:219-228, 341-344: det(J) on an (order+2)^dim lattice
    int first_invalid_element() const {
        const int ns = order + 2;
        double J[9];
        for (int e = 0; e < num_elements(); ++e) {
            const int nz = dim == 3 ? ns : 1;
            for (int k = 0; k < nz; ++k)
                for (int j = 0; j < ns; ++j)
                    for (int i = 0; i < ns; ++i) {
                        const double xi[3] = {i / double(ns - 1), j / double(ns - 1),
                                              dim == 3 ? k / double(ns - 1) : 0.0};
                        if (jacobian(e, xi, J) <= 0.0) return e;
                    }
        }
        return -1;
    }
    // mesh.hpp:346-365 (3D: 5x5 sample grid on the face)
    void check_face_traces() const {
        for (size_t i = 0; i < ifaces.size(); ++i) {
            const FaceRecord& fr = ifaces[i];
            const double tol = 1e-12 * element_diameter(fr.elem_left);
            const int nt = dim == 3 ? 5 : 1;
            for (int kt = 0; kt < nt; ++kt)
                for (int k = 0; k < 5; ++k) {
                    const double s = k / 4.0, t = dim == 3 ? kt / 4.0 : 0.0;
                    double so, to;
                    orient_param(dim, fr.orientation, s, t, so, to);
                    double xil[3] = {0, 0, 0}, xir[3] = {0, 0, 0}, xl[3], xr[3];
                    param_point(dim, fr.face_left, s, t, xil);
                    param_point(dim, fr.face_right, so, to, xir);
                    map_point(fr.elem_left, xil, xl);
                    map_point(fr.elem_right, xir, xr);
                    double d2 = 0.0;
                    for (int a = 0; a < dim; ++a) d2 += (xl[a] - xr[a]) * (xl[a] - xr[a]);
                    if (std::sqrt(d2) > tol)
                        throw MeshError("mesh: interior face " + std::to_string(i) +
                                        " traces disagree between elements " +
                                        std::to_string(fr.elem_left) + " and " +
                                        std::to_string(fr.elem_right));
                }
        }
    }
};

// --------------------------------------------------------------- problem input
struct CrossSections { double sigma_t, sigma_s; };

struct SourceSpec {
    int kind = 0;           // 0 constant, 1 ball indicator
    double params[8] = {0}; // kind 0: [q]; kind 1: [cx,cy,cz,radius,q_in,q_out]
    double inflow = 0.0;    // isotropic incident flux on boundary faces
    double volumetric(const double* x, int dim) const {
        if (kind == 0) return params[0];
        double d2 = 0.0;
        for (int a = 0; a < dim; ++a) d2 += (x[a] - params[a]) * (x[a] - params[a]);
        return d2 < params[3] * params[3] ? params[4] : params[5];
    }
};

struct Ordinate { double weight; double dir[3]; };

// ---------------------------------------------------------------- small dense
// Row-major n x n LU with partial pivoting (first max on ties), as Eigen's
// PartialPivLU semantics (solver.hpp:69,92,114).
struct DenseLU {
    int n = 0;
    std::vector<double> lu;
    std::vector<int> perm;  // row k of U came from original row perm[k]
    double l1_norm = 0.0;
    void factor(const double* A, int nn) {
        n = nn;
        lu.assign(A, A + (size_t)n * n);
        perm.resize(n);
        l1_norm = 0.0;
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int i = 0; i < n; ++i) s += std::abs(A[(size_t)i * n + j]);
            l1_norm = std::max(l1_norm, s);
        }
        std::iota(perm.begin(), perm.end(), 0);
        for (int k = 0; k < n; ++k) {
            int p = k;
            double best = std::abs(lu[(size_t)k * n + k]);
            for (int i = k + 1; i < n; ++i) {
                const double v = std::abs(lu[(size_t)i * n + k]);
                if (v > best) { best = v; p = i; }
            }
            if (p != k) {
                for (int j = 0; j < n; ++j) std::swap(lu[(size_t)k * n + j], lu[(size_t)p * n + j]);
                std::swap(perm[k], perm[p]);
            }
            const double piv = lu[(size_t)k * n + k];
            if (piv == 0.0) continue;
            for (int i = k + 1; i < n; ++i) {
                double& lik = lu[(size_t)i * n + k];
                lik /= piv;
                const double l = lik;
                if (l == 0.0) continue;
                const double* urow = &lu[(size_t)k * n];
                double* row = &lu[(size_t)i * n];
                for (int j = k + 1; j < n; ++j) row[j] -= l * urow[j];
            }
        }
    }
    void solve(const double* b, double* x) const {
        std::vector<double> y(n);
        for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
        for (int i = 0; i < n; ++i) {
            double s = y[i];
            for (int j = 0; j < i; ++j) s -= lu[(size_t)i * n + j] * y[j];
            y[i] = s;
        }
        for (int i = n - 1; i >= 0; --i) {
            double s = y[i];
            for (int j = i + 1; j < n; ++j) s -= lu[(size_t)i * n + j] * y[j];
            y[i] = s / lu[(size_t)i * n + i];
        }
        for (int i = 0; i < n; ++i) x[i] = y[i];
    }
    // reciprocal condition number in the 1-norm (exact ||A^-1||_1 from n solves)
    double rcond() const {
        for (int k = 0; k < n; ++k)
            if (!(lu[(size_t)k * n + k] != 0.0) || !std::isfinite(lu[(size_t)k * n + k])) return 0.0;
        double inv_norm = 0.0;
        std::vector<double> e(n), x(n);
        for (int j = 0; j < n; ++j) {
            std::fill(e.begin(), e.end(), 0.0);
            e[j] = 1.0;
            solve(e.data(), x.data());
            double s = 0.0;
            for (int i = 0; i < n; ++i) s += std::abs(x[i]);
            inv_norm = std::max(inv_norm, s);
        }
        if (!(inv_norm > 0.0) || !(l1_norm > 0.0)) return 0.0;
        return (1.0 / inv_norm) / l1_norm;
    }
};

// ----------------------------------------------------------------- assembly.hpp
struct ElementQuadData {  // assembly.hpp:50-93
    std::vector<double> u;     // nq x nb
    std::vector<double> g;     // dim x nq x nb (physical gradients)
    std::vector<double> wdet, sigma_t, sigma_s;
    std::vector<double> x;     // nq x 3
};

// Restricted face blocks: rows/cols indexed over face nodes (n_f each).
// Entries outside the face nodes of the full n x n reference blocks are exact
// zeros (GLL endpoint traces vanish exactly), so restriction is lossless.
struct Coupling { int face, downwind, upwind, down_face, up_face; std::vector<double> block; };

struct Problem {
    Mesh mesh;
    Basis basis;
    int p = 1;
    std::vector<Ordinate> quad;
    std::map<int, CrossSections> xs;
    SourceSpec source;
    int vol_points = 0, face_points = 0;
    // FaceIntegration (assembly.hpp:33-40): 0 gauss (face_points), 1 romberg (2D, the reference default)
    int face_rule = 0;
    double romberg_tol = 1e-10;
    int romberg_max_levels = 16, romberg_min_levels = 6;
    int weighting = 1;      // 0 unity, 1 face, 2 siginvface (sweepgraph.hpp:40)
    int fas_threshold = 10; // solver.hpp:31
};

struct PerOrdinate {
    std::vector<Coupling> couplings;
    std::vector<std::vector<int>> incoming;
    std::vector<std::vector<double>> ll, rr;  // per interior face, restricted outflow parts
    std::vector<std::vector<double>> bout;    // per boundary face, restricted outflow
    std::vector<double> src_bnd;              // N*nb
    std::vector<double> face_length;
    int unconverged = 0;                      // Romberg faces that hit max_levels (assembly.hpp:349)
    // graph / ordering
    std::vector<int> order, position, lagged_edges;
    double lagged_weight = 0.0;
    std::vector<char> lagged;  // per coupling
    std::vector<double> weights;
    std::vector<int> level;
};

class Oracle {
  public:
    Problem P;
    int nb = 0, nf_nodes = 0, nel = 0;
    VolQuad vq;
    Quad1D fq;  // face Gauss rule (FaceIntegration::Rule::gauss)
    std::vector<std::vector<int>> fnodes;  // per local face: element node ids
    std::vector<ElementQuadData> eqd;      // cached per element
    std::vector<std::vector<double>> mass_total, mass_scatter;  // per element nb x nb
    std::vector<double> src_vol;                                // N*nb (isotropic)
    std::vector<PerOrdinate> ords;
    // element -> list of (kind, index) faces in the reference accumulation order
    std::vector<std::vector<std::pair<int, int>>> elem_faces;
    bool cache_lu = true;
    std::vector<int> active;  // ordinates set up (all by default)
    std::vector<std::vector<DenseLU>> lu;  // [d][e] when cached
    std::vector<std::vector<double>> diag_override_zero;  // test hook

    explicit Oracle(Problem prob, bool cache) : P(std::move(prob)), cache_lu(cache) {
        Mesh& M = P.mesh;
        M.check_connectivity();
        M.build_faces();
        P.basis = Basis(M.dim, P.p);
        nb = P.basis.size();
        nel = M.num_elements();
        const int npa = P.vol_points > 0 ? P.vol_points : P.p + 2;
        vq = tensor_gauss(M.dim, npa);
        fq = gauss_legendre(P.face_points > 0 ? P.face_points : P.p + 2);
        for (int f = 0; f < num_faces(M.dim); ++f) fnodes.push_back(face_nodes(M.dim, f, P.p));
        nf_nodes = (int)fnodes[0].size();
        elem_faces.assign(nel, {});
        for (size_t fi = 0; fi < M.ifaces.size(); ++fi) {
            elem_faces[M.ifaces[fi].elem_left].push_back({0, (int)fi});
            elem_faces[M.ifaces[fi].elem_right].push_back({1, (int)fi});
        }
        for (size_t bi = 0; bi < M.bfaces.size(); ++bi)
            elem_faces[M.bfaces[bi].elem].push_back({2, (int)bi});
    }

    void validate_geometry() {
        const int bad = P.mesh.first_invalid_element();
        if (bad >= 0)
            throw MeshError("mesh: element " + std::to_string(bad) + " has non-positive Jacobian");
        P.mesh.check_face_traces();
    }

    CrossSections xs_at(int region) const {  // xsec.hpp:37-51
        auto it = P.xs.find(region);
        if (it == P.xs.end()) {
            it = P.xs.find(0);
            if (it == P.xs.end())
                throw std::out_of_range("cross sections: no entry for region " +
                                        std::to_string(region));
        }
        return it->second;
    }

    // assembly.hpp:58-93
    ElementQuadData element_quad_data(int e) const {
        const Mesh& M = P.mesh;
        const int dim = M.dim, nq = vq.size();
        ElementQuadData d;
        d.u.resize((size_t)nq * nb);
        d.g.resize((size_t)dim * nq * nb);
        d.wdet.resize(nq);
        d.sigma_t.resize(nq);
        d.sigma_s.resize(nq);
        d.x.resize((size_t)nq * 3);
        std::vector<double> grads((size_t)nb * dim);
        const CrossSections xs = xs_at(M.region[e]);
        for (int q = 0; q < nq; ++q) {
            const double* xi = vq.points[q].data();
            double J[9], K[9];
            const double det = M.jacobian(e, xi, J);
            if (det <= 0.0 || !std::isfinite(det))
                throw AssemblyError("assembly: singular Jacobian in element " + std::to_string(e));
            M.inverse(J, K);
            P.basis.values(xi, &d.u[(size_t)q * nb]);
            P.basis.gradients(xi, grads.data());
            for (int m = 0; m < nb; ++m)
                for (int k = 0; k < dim; ++k) {
                    // (K^T grad)_k = sum_j K(j,k) dhat_j   (assembly.hpp:84-85)
                    double v = 0.0;
                    for (int j = 0; j < dim; ++j) v += K[j * 3 + k] * grads[m * dim + j];
                    d.g[((size_t)k * nq + q) * nb + m] = v;
                }
            d.wdet[q] = vq.weights[q] * det;
            M.map_point(e, xi, &d.x[(size_t)q * 3]);
            d.sigma_t[q] = xs.sigma_t;
            d.sigma_s[q] = xs.sigma_s;
        }
        return d;
    }

    const ElementQuadData& quad_data(int e) const { return eqd[e]; }

    void precompute_elements() {
        eqd.resize(nel);
        mass_total.resize(nel);
        mass_scatter.resize(nel);
        src_vol.assign((size_t)nel * nb, 0.0);
        const int nq = vq.size();
        parallel_for(nel, [&](int e) {
            ElementQuadData local;
            if (cache_lu) eqd[e] = element_quad_data(e);
            else local = element_quad_data(e);
            const ElementQuadData& d = cache_lu ? eqd[e] : local;
            // assembly.hpp:157-160
            std::vector<double>& mt = mass_total[e];
            std::vector<double>& ms = mass_scatter[e];
            mt.assign((size_t)nb * nb, 0.0);
            ms.assign((size_t)nb * nb, 0.0);
            for (int m = 0; m < nb; ++m)
                for (int n = 0; n < nb; ++n) {
                    double st = 0.0, ss = 0.0;
                    for (int q = 0; q < nq; ++q) {
                        const double um = d.u[(size_t)q * nb + m], un = d.u[(size_t)q * nb + n];
                        st += um * (d.wdet[q] * d.sigma_t[q]) * un;
                        ss += um * (d.wdet[q] * d.sigma_s[q]) * un;
                    }
                    mt[(size_t)m * nb + n] = st;
                    ms[(size_t)m * nb + n] = ss;
                }
            // assembly.hpp:292-300 volume source moments (isotropic)
            double J[9];
            for (int q = 0; q < nq; ++q) {
                const double* xi = vq.points[q].data();
                const double det = P.mesh.jacobian(e, xi, J);
                double x[3];
                P.mesh.map_point(e, xi, x);
                const double s = vq.weights[q] * det * P.source.volumetric(x, P.mesh.dim);
                for (int m = 0; m < nb; ++m) src_vol[(size_t)e * nb + m] += s * d.u[(size_t)q * nb + m];
            }
        });
    }

    // assembly.hpp:143-163 streaming block G_e(Omega) = -(Omega.grad u)^T W u
    void stream_block(int e, const double* omega, double* G) const {
        ElementQuadData local;
        if (!cache_lu) local = element_quad_data(e);
        const ElementQuadData& d = cache_lu ? eqd[e] : local;
        const int nq = vq.size(), dim = P.mesh.dim;
        std::vector<double> dir((size_t)nq * nb);
        for (int q = 0; q < nq; ++q)
            for (int m = 0; m < nb; ++m) {
                double v = 0.0;
                for (int k = 0; k < dim; ++k) v += omega[k] * d.g[((size_t)k * nq + q) * nb + m];
                dir[(size_t)q * nb + m] = v;
            }
        for (int m = 0; m < nb; ++m)
            for (int n = 0; n < nb; ++n) {
                double s = 0.0;
                for (int q = 0; q < nq; ++q)
                    s += (dir[(size_t)q * nb + m] * d.wdet[q]) * d.u[(size_t)q * nb + n];
                G[(size_t)m * nb + n] = -s;
            }
    }

    // Trace values of the face nodes of local face f at face parameter (s,t):
    // exact products of 1D Lagrange values (the other factor is exactly 1.0).
    void face_trace(int f, double s, double t, double* out) const {
        const int dim = P.mesh.dim, n1 = P.p + 1;
        std::vector<double> full(nb);
        double xi[3] = {0, 0, 0};
        param_point(dim, f, s, t, xi);
        P.basis.values(xi, full.data());
        for (int a = 0; a < (int)fnodes[f].size(); ++a) out[a] = full[fnodes[f][a]];
        (void)n1;
    }

    // assembly.hpp:185-268 + 302-313 with FaceIntegration::Rule::romberg (:121-131, the
    // reference default; 2D): per interior face ONE Romberg tableau over the packed
    // integrand [LL+ | RR- | LR- | RL+ | |J|] (face-node restriction: the other entries
    // are exact zeros in every sample, so the max-norm convergence test is unchanged);
    // per boundary face one over [LL+] and one over the inflow moments.
    void assemble_faces_romberg(int d, PerOrdinate& ord) const {
        const Mesh& M = P.mesh;
        if (M.dim != 2) throw std::invalid_argument("romberg face rule: 2D meshes only (the reference is 2D)");
        const double* omega = P.quad[d].dir;
        const int nfn = nf_nodes, nn = nfn * nfn;
        const int nfi = (int)M.ifaces.size();
        ord.ll.assign(nfi, {});
        ord.rr.assign(nfi, {});
        ord.face_length.assign(nfi, 0.0);
        ord.couplings.clear();
        ord.unconverged = 0;
        std::vector<double> ul(nfn), ur(nfn), packed;
        for (int fi = 0; fi < nfi; ++fi) {
            const FaceRecord& fr = M.ifaces[fi];
            auto integrand = [&](double t, double* v) {   // assembly.hpp:197-220
                const FaceGeom fg = M.face_geometry(fr.elem_left, fr.face_left, t, 0.0);
                const double on = omega[0] * fg.normal[0] + omega[1] * fg.normal[1];
                face_trace(fr.face_left, t, 0.0, ul.data());
                double so, to;
                orient_param(2, fr.orientation, t, 0.0, so, to);
                face_trace(fr.face_right, so, to, ur.data());
                const double wplus = 0.5 * (on + std::abs(on));
                const double wminus = 0.5 * (std::abs(on) - on);
                int k = 0;
                for (int m = 0; m < nfn; ++m)
                    for (int n = 0; n < nfn; ++n) v[k++] = wplus * ul[m] * ul[n] * fg.sj;
                for (int m = 0; m < nfn; ++m)
                    for (int n = 0; n < nfn; ++n) v[k++] = wminus * ur[m] * ur[n] * fg.sj;
                for (int m = 0; m < nfn; ++m)
                    for (int n = 0; n < nfn; ++n) v[k++] = wminus * ul[m] * ur[n] * fg.sj;
                for (int m = 0; m < nfn; ++m)
                    for (int n = 0; n < nfn; ++n) v[k++] = wplus * ur[m] * ul[n] * fg.sj;
                v[k] = fg.sj;
            };
            if (!romberg_vec(integrand, (size_t)4 * nn + 1, P.romberg_tol, P.romberg_max_levels,
                             P.romberg_min_levels, packed))
                ord.unconverged++;
            const double length = packed[(size_t)4 * nn];
            ord.face_length[fi] = length;
            const double eps_edge = 1e-12 * length;
            ord.ll[fi].assign(packed.begin(), packed.begin() + nn);
            ord.rr[fi].assign(packed.begin() + nn, packed.begin() + 2 * nn);
            std::vector<double> LR(packed.begin() + 2 * nn, packed.begin() + 3 * nn),
                RL(packed.begin() + 3 * nn, packed.begin() + 4 * nn);
            double mlr = 0.0, mrl = 0.0;
            for (int k = 0; k < nn; ++k) {
                mlr = std::max(mlr, std::abs(LR[k]));
                mrl = std::max(mrl, std::abs(RL[k]));
            }
            if (mlr > eps_edge) {
                Coupling c{fi, fr.elem_left, fr.elem_right, fr.face_left, fr.face_right, LR};
                for (double& x : c.block) x = -x;
                ord.couplings.push_back(std::move(c));
            }
            if (mrl > eps_edge) {
                Coupling c{fi, fr.elem_right, fr.elem_left, fr.face_right, fr.face_left, RL};
                for (double& x : c.block) x = -x;
                ord.couplings.push_back(std::move(c));
            }
        }
        const int nfb = (int)M.bfaces.size();
        ord.bout.assign(nfb, {});
        ord.src_bnd.assign((size_t)nel * nb, 0.0);
        for (int bi = 0; bi < nfb; ++bi) {
            const BoundaryFace& bf = M.bfaces[bi];
            auto outflow = [&](double t, double* v) {   // assembly.hpp:244-258
                const FaceGeom fg = M.face_geometry(bf.elem, bf.local_face, t, 0.0);
                const double on = omega[0] * fg.normal[0] + omega[1] * fg.normal[1];
                face_trace(bf.local_face, t, 0.0, ul.data());
                const double wplus = 0.5 * (on + std::abs(on));
                int k = 0;
                for (int m = 0; m < nfn; ++m)
                    for (int n = 0; n < nfn; ++n) v[k++] = wplus * ul[m] * ul[n] * fg.sj;
            };
            if (!romberg_vec(outflow, (size_t)nn, P.romberg_tol, P.romberg_max_levels, P.romberg_min_levels,
                             ord.bout[bi]))
                ord.unconverged++;
        }
        // assemble_source's boundary functional (assembly.hpp:302-313), after the volume part
        for (int bi = 0; bi < nfb; ++bi) {
            const BoundaryFace& bf = M.bfaces[bi];
            auto incident = [&](double t, double* v) {
                const FaceGeom fg = M.face_geometry(bf.elem, bf.local_face, t, 0.0);
                const double on = omega[0] * fg.normal[0] + omega[1] * fg.normal[1];
                face_trace(bf.local_face, t, 0.0, ul.data());
                const double wminus = 0.5 * (std::abs(on) - on);
                const double c = wminus * P.source.inflow * fg.sj;
                for (int m = 0; m < nfn; ++m) v[m] = c * ul[m];
            };
            std::vector<double> mom;
            romberg_vec(incident, (size_t)nfn, P.romberg_tol, P.romberg_max_levels, P.romberg_min_levels, mom);
            const auto& fn = fnodes[bf.local_face];
            for (int m = 0; m < nfn; ++m) ord.src_bnd[(size_t)bf.elem * nb + fn[m]] += mom[m];
        }
        ord.incoming.assign(nel, {});
        for (size_t c = 0; c < ord.couplings.size(); ++c)
            ord.incoming[ord.couplings[c].downwind].push_back((int)c);
    }

    // assembly.hpp:185-268 with FaceIntegration::Rule::gauss (:121-128)
    void assemble_faces(int d, PerOrdinate& ord) const {
        if (P.face_rule == 1) {
            assemble_faces_romberg(d, ord);
            return;
        }
        const Mesh& M = P.mesh;
        const int dim = M.dim;
        const double* omega = P.quad[d].dir;
        const int nfn = nf_nodes;
        const int ng = fq.size();
        const int npts = dim == 2 ? ng : ng * ng;
        const int nfi = (int)M.ifaces.size();
        ord.ll.assign(nfi, {});
        ord.rr.assign(nfi, {});
        ord.face_length.assign(nfi, 0.0);
        ord.couplings.clear();
        std::vector<double> ul(nfn), ur(nfn);
        std::vector<double> LL(nfn * nfn), RR(nfn * nfn), LR(nfn * nfn), RL(nfn * nfn);
        for (int fi = 0; fi < nfi; ++fi) {
            const FaceRecord& fr = M.ifaces[fi];
            std::fill(LL.begin(), LL.end(), 0.0);
            std::fill(RR.begin(), RR.end(), 0.0);
            std::fill(LR.begin(), LR.end(), 0.0);
            std::fill(RL.begin(), RL.end(), 0.0);
            double length = 0.0;
            for (int ip = 0; ip < npts; ++ip) {
                const int is = ip % ng, it = ip / ng;
                const double s = fq.points[is], t = dim == 3 ? fq.points[it] : 0.0;
                const double w = dim == 3 ? fq.weights[is] * fq.weights[it] : fq.weights[is];
                // assembly.hpp:103-117 face_sample
                const FaceGeom fg = M.face_geometry(fr.elem_left, fr.face_left, s, t);
                double on = 0.0;
                for (int k = 0; k < dim; ++k) on += omega[k] * fg.normal[k];
                face_trace(fr.face_left, s, t, ul.data());
                double so, to;
                orient_param(dim, fr.orientation, s, t, so, to);
                face_trace(fr.face_right, so, to, ur.data());
                const double wplus = 0.5 * (on + std::abs(on));
                const double wminus = 0.5 * (std::abs(on) - on);
                const double sj = fg.sj;
                for (int m = 0; m < nfn; ++m)
                    for (int n = 0; n < nfn; ++n) {
                        LL[m * nfn + n] += w * (wplus * ul[m] * ul[n] * sj);
                        RR[m * nfn + n] += w * (wminus * ur[m] * ur[n] * sj);
                        LR[m * nfn + n] += w * (wminus * ul[m] * ur[n] * sj);
                        RL[m * nfn + n] += w * (wplus * ur[m] * ul[n] * sj);
                    }
                length += w * sj;
            }
            ord.face_length[fi] = length;
            const double eps_edge = 1e-12 * length;
            ord.ll[fi] = LL;
            ord.rr[fi] = RR;
            double mlr = 0.0, mrl = 0.0;
            for (int k = 0; k < nfn * nfn; ++k) {
                mlr = std::max(mlr, std::abs(LR[k]));
                mrl = std::max(mrl, std::abs(RL[k]));
            }
            if (mlr > eps_edge) {
                Coupling c{fi, fr.elem_left, fr.elem_right, fr.face_left, fr.face_right, LR};
                for (double& v : c.block) v = -v;
                ord.couplings.push_back(std::move(c));
            }
            if (mrl > eps_edge) {
                Coupling c{fi, fr.elem_right, fr.elem_left, fr.face_right, fr.face_left, RL};
                for (double& v : c.block) v = -v;
                ord.couplings.push_back(std::move(c));
            }
        }
        // boundary faces: outflow (assembly.hpp:244-266) and inflow source (:302-313)
        const int nfb = (int)M.bfaces.size();
        ord.bout.assign(nfb, {});
        ord.src_bnd.assign((size_t)nel * nb, 0.0);
        for (int bi = 0; bi < nfb; ++bi) {
            const BoundaryFace& bf = M.bfaces[bi];
            std::vector<double> B(nfn * nfn, 0.0), inflow(nfn, 0.0);
            for (int ip = 0; ip < npts; ++ip) {
                const int is = ip % ng, it = ip / ng;
                const double s = fq.points[is], t = dim == 3 ? fq.points[it] : 0.0;
                const double w = dim == 3 ? fq.weights[is] * fq.weights[it] : fq.weights[is];
                const FaceGeom fg = M.face_geometry(bf.elem, bf.local_face, s, t);
                double on = 0.0;
                for (int k = 0; k < dim; ++k) on += omega[k] * fg.normal[k];
                face_trace(bf.local_face, s, t, ul.data());
                const double wplus = 0.5 * (on + std::abs(on));
                const double wminus = 0.5 * (std::abs(on) - on);
                for (int m = 0; m < nfn; ++m)
                    for (int n = 0; n < nfn; ++n)
                        B[m * nfn + n] += w * (wplus * ul[m] * ul[n] * fg.sj);
                const double c = wminus * P.source.inflow * fg.sj;
                for (int m = 0; m < nfn; ++m) inflow[m] += w * (c * ul[m]);
            }
            ord.bout[bi] = B;
            const auto& fn = fnodes[bf.local_face];
            for (int m = 0; m < nfn; ++m) ord.src_bnd[(size_t)bf.elem * nb + fn[m]] += inflow[m];
        }
        // incoming lists (assembly.hpp:398-400)
        ord.incoming.assign(nel, {});
        for (size_t c = 0; c < ord.couplings.size(); ++c)
            ord.incoming[ord.couplings[c].downwind].push_back((int)c);
    }

    // diag = stream + outflow + M_t (assembly.hpp:393); outflow accumulated in
    // the reference's face order (interior faces by id, then boundary faces).
    void diag_block(int e, int d, const PerOrdinate& ord, double* A) const {
        stream_block(e, P.quad[d].dir, A);
        std::vector<double> out((size_t)nb * nb, 0.0);
        const Mesh& M = P.mesh;
        const int nfn = nf_nodes;
        // interior faces first (face id order), then boundary faces
        std::vector<std::pair<int, int>> faces = elem_faces[e];
        std::stable_sort(faces.begin(), faces.end(), [](auto a, auto b) {
            const int ka = a.first == 2 ? 1 : 0, kb = b.first == 2 ? 1 : 0;
            if (ka != kb) return ka < kb;
            return a.second < b.second;
        });
        for (const auto& [kind, idx] : faces) {
            const std::vector<double>* blk;
            int lf;
            if (kind == 0) { blk = &ord.ll[idx]; lf = M.ifaces[idx].face_left; }
            else if (kind == 1) { blk = &ord.rr[idx]; lf = M.ifaces[idx].face_right; }
            else { blk = &ord.bout[idx]; lf = M.bfaces[idx].local_face; }
            const auto& fn = fnodes[lf];
            for (int m = 0; m < nfn; ++m)
                for (int n = 0; n < nfn; ++n)
                    out[(size_t)fn[m] * nb + fn[n]] += (*blk)[m * nfn + n];
        }
        const auto& mt = mass_total[e];
        for (size_t k = 0; k < (size_t)nb * nb; ++k) A[k] = (A[k] + out[k]) + mt[k];
        if (!diag_override_zero.empty() && !diag_override_zero[d].empty() &&
            diag_override_zero[d][e] != 0.0)
            std::fill(A, A + (size_t)nb * nb, 0.0);
    }

    // ----------------------------------------------------------- sweepgraph.hpp
    struct Edge { int from, to; double weight; int coupling; };
    struct Graph { int nv; std::vector<Edge> edges; };

    // sweepgraph.hpp:54-77
    Graph build_graph(int d, const PerOrdinate& ord) const {
        Graph g;
        g.nv = nel;
        const int nfn = nf_nodes;
        for (size_t c = 0; c < ord.couplings.size(); ++c) {
            const Coupling& fc = ord.couplings[c];
            double w = 1.0;
            if (P.weighting == 1) {
                w = 0.0;
                for (double v : fc.block) w = std::max(w, std::abs(v));
            } else if (P.weighting == 2) {
                DenseLU mlu;
                mlu.factor(mass_total[fc.downwind].data(), nb);
                w = 0.0;
                std::vector<double> col(nb), x(nb);
                for (int n = 0; n < nfn; ++n) {
                    std::fill(col.begin(), col.end(), 0.0);
                    for (int m = 0; m < nfn; ++m) col[fnodes[fc.down_face][m]] = fc.block[m * nfn + n];
                    mlu.solve(col.data(), x.data());
                    for (int i = 0; i < nb; ++i) {
                        if (!std::isfinite(x[i]))
                            throw AssemblyError("sig_inv_face weighting: singular mass matrix on element " +
                                                std::to_string(fc.downwind));
                        w = std::max(w, std::abs(x[i]));
                    }
                }
            }
            g.edges.push_back({fc.upwind, fc.downwind, w, (int)c});
        }
        (void)d;
        return g;
    }

    // sweepgraph.hpp:82-136
    static std::vector<std::vector<int>> tarjan_scc(const Graph& g) {
        const int n = g.nv;
        std::vector<std::vector<int>> adj(n);
        for (size_t i = 0; i < g.edges.size(); ++i) adj[g.edges[i].from].push_back((int)i);
        std::vector<int> index(n, -1), lowlink(n, 0);
        std::vector<char> on_stack(n, 0);
        std::vector<int> stack;
        std::vector<std::vector<int>> sccs;
        int next_index = 0;
        struct Frame { int v; size_t child; };
        std::vector<Frame> call;
        for (int root = 0; root < n; ++root) {
            if (index[root] != -1) continue;
            call.push_back({root, 0});
            index[root] = lowlink[root] = next_index++;
            stack.push_back(root);
            on_stack[root] = 1;
            while (!call.empty()) {
                Frame& fr = call.back();
                if (fr.child < adj[fr.v].size()) {
                    const int w = g.edges[adj[fr.v][fr.child++]].to;
                    if (index[w] == -1) {
                        index[w] = lowlink[w] = next_index++;
                        stack.push_back(w);
                        on_stack[w] = 1;
                        call.push_back({w, 0});
                    } else if (on_stack[w]) {
                        lowlink[fr.v] = std::min(lowlink[fr.v], index[w]);
                    }
                } else {
                    if (lowlink[fr.v] == index[fr.v]) {
                        std::vector<int> comp;
                        int w;
                        do {
                            w = stack.back();
                            stack.pop_back();
                            on_stack[w] = 0;
                            comp.push_back(w);
                        } while (w != fr.v);
                        std::sort(comp.begin(), comp.end());
                        sccs.push_back(std::move(comp));
                    }
                    const int v = fr.v;
                    call.pop_back();
                    if (!call.empty())
                        lowlink[call.back().v] = std::min(lowlink[call.back().v], lowlink[v]);
                }
            }
        }
        return sccs;
    }

    struct Fas { std::vector<int> order, lagged; double weight = 0.0; };
    struct Local { std::vector<int> verts; std::vector<std::array<int, 2>> edges; std::vector<double> w; std::vector<int> parent; };

    // sweepgraph.hpp:156-170
    static Local induce(const Graph& g, const std::vector<int>& vs) {
        Local lg;
        lg.verts = vs;
        std::vector<int> local(g.nv, -1);
        for (size_t i = 0; i < vs.size(); ++i) local[vs[i]] = (int)i;
        for (size_t e = 0; e < g.edges.size(); ++e) {
            const auto& ed = g.edges[e];
            if (local[ed.from] >= 0 && local[ed.to] >= 0) {
                lg.edges.push_back({local[ed.from], local[ed.to]});
                lg.w.push_back(ed.weight);
                lg.parent.push_back((int)e);
            }
        }
        return lg;
    }
    // sweepgraph.hpp:173-186
    static Fas order_to_result(const Local& lg, const std::vector<int>& lo) {
        Fas r;
        std::vector<int> pos(lg.verts.size());
        for (size_t k = 0; k < lo.size(); ++k) pos[lo[k]] = (int)k;
        for (size_t e = 0; e < lg.edges.size(); ++e)
            if (pos[lg.edges[e][0]] > pos[lg.edges[e][1]]) {
                r.lagged.push_back(lg.parent[e]);
                r.weight += lg.w[e];
            }
        for (int v : lo) r.order.push_back(lg.verts[v]);
        return r;
    }
    // sweepgraph.hpp:192-232
    static Fas min_fas_exact(const Graph& g, const std::vector<int>& vs) {
        const int n = (int)vs.size();
        if (n > 22) throw std::invalid_argument("min_fas_exact: component too large");
        Local lg = induce(g, vs);
        std::vector<std::vector<double>> wout(n, std::vector<double>(n, 0.0));
        for (size_t e = 0; e < lg.edges.size(); ++e) wout[lg.edges[e][0]][lg.edges[e][1]] += lg.w[e];
        const uint32_t full = (uint32_t(1) << n) - 1;
        std::vector<double> dp(full + 1, std::numeric_limits<double>::infinity());
        std::vector<int8_t> choice(full + 1, -1);
        dp[0] = 0.0;
        for (uint32_t mask = 1; mask <= full; ++mask) {
            for (int v = 0; v < n; ++v) {
                if (!(mask & (uint32_t(1) << v))) continue;
                const uint32_t rest = mask & ~(uint32_t(1) << v);
                if (dp[rest] == std::numeric_limits<double>::infinity()) continue;
                double back = 0.0;
                for (int u = 0; u < n; ++u)
                    if (rest & (uint32_t(1) << u)) back += wout[v][u];
                const double cand = dp[rest] + back;
                if (cand < dp[mask]) {
                    dp[mask] = cand;
                    choice[mask] = (int8_t)v;
                }
            }
        }
        std::vector<int> lo(n);
        uint32_t mask = full;
        for (int k = n - 1; k >= 0; --k) {
            const int v = choice[mask];
            lo[k] = v;
            mask &= ~(uint32_t(1) << v);
        }
        return order_to_result(lg, lo);
    }
    // sweepgraph.hpp:238-315
    static Fas min_fas_heuristic(const Graph& g, const std::vector<int>& vs) {
        Local lg = induce(g, vs);
        const int n = (int)lg.verts.size();
        std::vector<std::vector<std::pair<int, double>>> out(n), in(n);
        std::vector<double> wout(n, 0.0), win(n, 0.0);
        std::vector<int> dout(n, 0), din(n, 0);
        for (size_t e = 0; e < lg.edges.size(); ++e) {
            const int u = lg.edges[e][0], v = lg.edges[e][1];
            const double w = lg.w[e];
            out[u].push_back({v, w});
            in[v].push_back({u, w});
            wout[u] += w;
            win[v] += w;
            dout[u]++;
            din[v]++;
        }
        std::vector<char> removed(n, 0);
        std::vector<int> head, tail;
        auto drop = [&](int v) {
            removed[v] = 1;
            for (const auto& [u, w] : out[v]) {
                if (removed[u]) continue;
                din[u]--;
                win[u] -= w;
            }
            for (const auto& [u, w] : in[v]) {
                if (removed[u]) continue;
                dout[u]--;
                wout[u] -= w;
            }
        };
        int left = n;
        while (left > 0) {
            bool progressed = true;
            while (progressed) {
                progressed = false;
                for (int v = 0; v < n; ++v)
                    if (!removed[v] && dout[v] == 0) {
                        drop(v);
                        tail.push_back(v);
                        left--;
                        progressed = true;
                    }
            }
            progressed = true;
            while (progressed) {
                progressed = false;
                for (int v = 0; v < n; ++v)
                    if (!removed[v] && dout[v] > 0 && din[v] == 0) {
                        drop(v);
                        head.push_back(v);
                        left--;
                        progressed = true;
                    }
            }
            if (left == 0) break;
            int best = -1;
            double best_delta = -std::numeric_limits<double>::infinity();
            for (int v = 0; v < n; ++v) {
                if (removed[v]) continue;
                const double delta = wout[v] - win[v];
                if (delta > best_delta) {
                    best_delta = delta;
                    best = v;
                }
            }
            drop(best);
            head.push_back(best);
            left--;
        }
        std::vector<int> lo = std::move(head);
        lo.insert(lo.end(), tail.rbegin(), tail.rend());
        return order_to_result(lg, lo);
    }
    // sweepgraph.hpp:331-396
    static void sweep_ordering(const Graph& g, int thr, PerOrdinate& res) {
        const auto sccs = tarjan_scc(g);
        const int n = g.nv;
        std::vector<int> comp_of(n, -1);
        for (size_t c = 0; c < sccs.size(); ++c)
            for (int v : sccs[c]) comp_of[v] = (int)c;
        const int nc = (int)sccs.size();
        std::vector<std::vector<int>> cond_out(nc);
        std::vector<int> cond_in(nc, 0);
        for (const auto& e : g.edges) {
            const int cu = comp_of[e.from], cv = comp_of[e.to];
            if (cu != cv) cond_out[cu].push_back(cv);
        }
        for (int c = 0; c < nc; ++c) {
            std::sort(cond_out[c].begin(), cond_out[c].end());
            cond_out[c].erase(std::unique(cond_out[c].begin(), cond_out[c].end()), cond_out[c].end());
            for (int t : cond_out[c]) cond_in[t]++;
        }
        using Key = std::pair<int, int>;
        std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
        for (int c = 0; c < nc; ++c)
            if (cond_in[c] == 0) ready.push({sccs[c].front(), c});
        res.order.clear();
        res.lagged_edges.clear();
        res.lagged_weight = 0.0;
        while (!ready.empty()) {
            const int c = ready.top().second;
            ready.pop();
            if (sccs[c].size() == 1) {
                res.order.push_back(sccs[c].front());
            } else {
                const Fas fas = (int)sccs[c].size() <= std::min(thr, 22) ? min_fas_exact(g, sccs[c])
                                                                       : min_fas_heuristic(g, sccs[c]);
                res.order.insert(res.order.end(), fas.order.begin(), fas.order.end());
                res.lagged_edges.insert(res.lagged_edges.end(), fas.lagged.begin(), fas.lagged.end());
                res.lagged_weight += fas.weight;
            }
            for (int t : cond_out[c])
                if (--cond_in[t] == 0) ready.push({sccs[t].front(), t});
        }
        if ((int)res.order.size() != n) throw std::logic_error("sweep_ordering: condensation was not acyclic");
        res.position.assign(n, -1);
        for (int k = 0; k < n; ++k) res.position[res.order[k]] = k;
        std::vector<char> lag(g.edges.size(), 0);
        for (int e : res.lagged_edges) lag[e] = 1;
        for (size_t e = 0; e < g.edges.size(); ++e) {
            const bool backward = res.position[g.edges[e].from] > res.position[g.edges[e].to];
            if (backward != (bool)lag[e]) throw std::logic_error("sweep_ordering: retained edge set is inconsistent");
        }
        std::sort(res.lagged_edges.begin(), res.lagged_edges.end());
    }

    // ---------------------------------------------------------------- solver.hpp
    // SweepSolver ctor (solver.hpp:52-78) + levels (new).
    void setup(bool check_rcond) {
        precompute_elements();
        const int nd = (int)P.quad.size();
        ords.assign(nd, {});
        if (cache_lu) lu.assign(nd, {});
        if (active.empty()) {
            active.resize(nd);
            std::iota(active.begin(), active.end(), 0);
        }
        parallel_for((int)active.size(), [&](int ai) {
            const int d = active[ai];
            PerOrdinate& ord = ords[d];
            assemble_faces(d, ord);
            const Graph g = build_graph(d, ord);
            ord.weights.clear();
            for (const auto& e : g.edges) ord.weights.push_back(e.weight);
            sweep_ordering(g, P.fas_threshold, ord);
            ord.lagged.assign(ord.couplings.size(), 0);
            for (size_t c = 0; c < ord.couplings.size(); ++c)
                ord.lagged[c] = ord.position[ord.couplings[c].upwind] > ord.position[ord.couplings[c].downwind];
            // levels over retained edges, in sweep order
            ord.level.assign(nel, 0);
            for (int e : ord.order) {
                int lv = 0;
                for (int c : ord.incoming[e])
                    if (!ord.lagged[c]) lv = std::max(lv, ord.level[ord.couplings[c].upwind] + 1);
                ord.level[e] = lv;
            }
            if (cache_lu) {
                lu[d].resize(nel);
                std::vector<double> A((size_t)nb * nb);
                for (int e = 0; e < nel; ++e) {
                    diag_block(e, d, ord, A.data());
                    lu[d][e].factor(A.data(), nb);
                    if (check_rcond) {
                        const double rc = lu[d][e].rcond();
                        if (!(rc > 1e-14))
                            throw SolverError("local streaming+collision block is singular (element " +
                                              std::to_string(e) + ", ordinate " + std::to_string(d) + ")");
                    }
                }
            }
        });
    }

    void local_solve(int e, int d, const double* rhs, double* out) const {
        if (cache_lu) { lu[d][e].solve(rhs, out); return; }
        std::vector<double> A((size_t)nb * nb);
        diag_block(e, d, ords[d], A.data());
        DenseLU l;
        l.factor(A.data(), nb);
        l.solve(rhs, out);
    }

    // solver.hpp:98-117
    void sweep(int d, const double* phi, const double* psi_old, double* psi_new) const {
        const PerOrdinate& ord = ords[d];
        const int nfn = nf_nodes;
        const double c4pi = 1.0 / (4.0 * M_PI);
        std::vector<double> rhs(nb), A, tmp(nfn);
        DenseLU l;
        if (!cache_lu) A.resize((size_t)nb * nb);
        for (int e : ord.order) {
            for (int m = 0; m < nb; ++m)
                rhs[m] = src_vol[(size_t)e * nb + m] + ord.src_bnd[(size_t)e * nb + m];
            const auto& ms = mass_scatter[e];
            for (int m = 0; m < nb; ++m) {
                double s = 0.0;
                for (int n = 0; n < nb; ++n) s += ms[(size_t)m * nb + n] * phi[(size_t)e * nb + n];
                rhs[m] += c4pi * s;
            }
            for (int c : ord.incoming[e]) {
                const Coupling& fc = ord.couplings[c];
                const double* src = ord.lagged[c] ? psi_old : psi_new;
                const auto& dn = fnodes[fc.down_face];
                const auto& un = fnodes[fc.up_face];
                for (int m = 0; m < nfn; ++m) {
                    double s = 0.0;
                    for (int n = 0; n < nfn; ++n) s += fc.block[m * nfn + n] * src[(size_t)fc.upwind * nb + un[n]];
                    rhs[dn[m]] -= s;
                }
            }
            if (cache_lu) {
                lu[d][e].solve(rhs.data(), &psi_new[(size_t)e * nb]);
            } else {
                diag_block(e, d, ord, A.data());
                l.factor(A.data(), nb);
                l.solve(rhs.data(), &psi_new[(size_t)e * nb]);
            }
        }
    }

    // solver.hpp:121-133 direct_oracle via a dense global LU (small meshes only)
    void direct_oracle(int d, const double* phi, double* psi) const {
        const int N = nel * nb;
        if (N > 6000) throw std::invalid_argument("direct_oracle: system too large for the dense oracle");
        const PerOrdinate& ord = ords[d];
        std::vector<double> A((size_t)N * N, 0.0), blk((size_t)nb * nb), rhs(N);
        for (int e = 0; e < nel; ++e) {
            diag_block(e, d, ord, blk.data());
            for (int i = 0; i < nb; ++i)
                for (int j = 0; j < nb; ++j) A[(size_t)(e * nb + i) * N + e * nb + j] = blk[(size_t)i * nb + j];
        }
        const int nfn = nf_nodes;
        for (const Coupling& fc : ord.couplings) {
            const auto& dn = fnodes[fc.down_face];
            const auto& un = fnodes[fc.up_face];
            for (int m = 0; m < nfn; ++m)
                for (int n = 0; n < nfn; ++n)
                    A[(size_t)(fc.downwind * nb + dn[m]) * N + fc.upwind * nb + un[n]] += fc.block[m * nfn + n];
        }
        const double c4pi = 1.0 / (4.0 * M_PI);
        for (int e = 0; e < nel; ++e) {
            const auto& ms = mass_scatter[e];
            for (int m = 0; m < nb; ++m) {
                double s = 0.0;
                for (int n = 0; n < nb; ++n) s += ms[(size_t)m * nb + n] * phi[(size_t)e * nb + n];
                rhs[e * nb + m] = (src_vol[(size_t)e * nb + m] + ord.src_bnd[(size_t)e * nb + m]) + c4pi * s;
            }
        }
        DenseLU g;
        g.factor(A.data(), N);
        g.solve(rhs.data(), psi);
    }

    // solver.hpp:136-168; criterion 0 = reference max_d ||dpsi||_inf,
    // 1 = configs' ||dphi||_2 / ||phi||_2.
    int source_iteration(double tol, int max_it, int criterion, double* psi, double* phi,
                         double* err_hist, double* phi_hist, int* converged) const {
        const int nd = (int)P.quad.size();
        const size_t N = (size_t)nel * nb;
        std::vector<std::vector<double>> cur(nd, std::vector<double>(N, 0.0)), nxt(nd, std::vector<double>(N));
        std::vector<double> ph(N, 0.0), ph_old(N);
        *converged = 0;
        int it = 0;
        for (; it < max_it; ++it) {
            parallel_for(nd, [&](int d) { sweep(d, ph.data(), cur[d].data(), nxt[d].data()); });
            double err = 0.0;
            for (int d = 0; d < nd; ++d) {
                double e = 0.0;
                for (size_t i = 0; i < N; ++i) e = std::max(e, std::abs(nxt[d][i] - cur[d][i]));
                err = std::max(err, e);
                std::swap(cur[d], nxt[d]);
            }
            ph_old = ph;
            std::fill(ph.begin(), ph.end(), 0.0);
            for (int d = 0; d < nd; ++d) {
                const double w = P.quad[d].weight;
                for (size_t i = 0; i < N; ++i) ph[i] += w * cur[d][i];
            }
            double num = 0.0, den = 0.0;
            for (size_t i = 0; i < N; ++i) {
                num += (ph[i] - ph_old[i]) * (ph[i] - ph_old[i]);
                den += ph[i] * ph[i];
            }
            const double rel = den > 0.0 ? std::sqrt(num) / std::sqrt(den) : (num > 0.0 ? INFINITY : 0.0);
            if (err_hist) err_hist[it] = err;
            if (phi_hist) phi_hist[it] = rel;
            const double crit = criterion == 0 ? err : rel;
            if (crit < tol) {
                *converged = 1;
                ++it;
                break;
            }
        }
        if (psi)
            for (int d = 0; d < nd; ++d) std::copy(cur[d].begin(), cur[d].end(), psi + (size_t)d * N);
        if (phi) std::copy(ph.begin(), ph.end(), phi);
        return it;
    }

    // solver.hpp:220-245 balance_report (out: src_vol, inflow, absorption, outflow, residual, per attr)
    void balance(const double* psi, const double* phi, double* out, std::map<int, double>& by_attr) const {
        const Mesh& M = P.mesh;
        const int nfn = nf_nodes;
        const size_t N = (size_t)nel * nb;
        double sv = 0.0, inflow = 0.0, absorption = 0.0, outflow = 0.0;
        for (int d = 0; d < (int)P.quad.size(); ++d) {
            const double w = P.quad[d].weight;
            double s1 = 0.0, s2 = 0.0;
            for (size_t i = 0; i < N; ++i) { s1 += src_vol[i]; s2 += ords[d].src_bnd[i]; }
            sv += w * s1;
            inflow += w * s2;
            for (size_t bi = 0; bi < M.bfaces.size(); ++bi) {
                const BoundaryFace& bf = M.bfaces[bi];
                const auto& fn = fnodes[bf.local_face];
                double o = 0.0;
                for (int m = 0; m < nfn; ++m) {
                    double s = 0.0;
                    for (int n = 0; n < nfn; ++n)
                        s += ords[d].bout[bi][m * nfn + n] * psi[(size_t)d * N + (size_t)bf.elem * nb + fn[n]];
                    o += s;
                }
                o *= w;
                outflow += o;
                by_attr[bf.attr] += o;
            }
        }
        for (int e = 0; e < nel; ++e)
            for (int m = 0; m < nb; ++m) {
                double s = 0.0;
                for (int n = 0; n < nb; ++n)
                    s += (mass_total[e][(size_t)m * nb + n] - mass_scatter[e][(size_t)m * nb + n]) *
                         phi[(size_t)e * nb + n];
                absorption += s;
            }
        out[0] = sv;
        out[1] = inflow;
        out[2] = absorption;
        out[3] = outflow;
        out[4] = sv + inflow - absorption - outflow;
    }
};

}  // namespace orc

// =============================================================== C interface
extern "C" {

struct orc_problem {
    int dim, geom_order, basis_order;
    int num_points;
    const double* points;
    int num_elements;
    const int* element_nodes;
    const int* element_region;
    int num_bfaces;
    const int* bfaces;  // (elem, local_face, attr) triples
    int num_ordinates;
    const double* ord_weight;
    const double* ord_dir;  // 3 per ordinate
    int num_regions;
    const int* region_ids;
    const double* sigma_t;
    const double* sigma_s;
    int source_kind;
    double source_params[8];
    double inflow;
    int volume_points, face_points;
    int weighting, fas_threshold;
    int validate_geometry;
    int cache_lu;
    int check_rcond;
    int num_active;           // 0: all ordinates
    const int* active;        // ordinates to set up (C4/C5 sampled parity)
    int face_rule;            // 0 gauss, 1 romberg
    double romberg_tol;
    int romberg_max_levels, romberg_min_levels;
};

static thread_local std::string g_err;

static void set_err(const char* what, char* buf, int len) {
    g_err = what;
    if (buf && len > 0) {
        std::snprintf(buf, (size_t)len, "%s", what);
    }
}

void* orc_create(const orc_problem* p, char* err, int errlen) {
    try {
        orc::Problem P;
        P.mesh.dim = p->dim;
        P.mesh.order = p->geom_order;
        P.mesh.geom = orc::Basis(p->dim, p->geom_order);
        P.mesh.pts.assign(p->points, p->points + (size_t)p->num_points * p->dim);
        const int npe = P.mesh.geom.size();
        P.mesh.elems.resize(p->num_elements);
        P.mesh.region.resize(p->num_elements);
        for (int e = 0; e < p->num_elements; ++e) {
            P.mesh.elems[e].assign(p->element_nodes + (size_t)e * npe, p->element_nodes + (size_t)(e + 1) * npe);
            P.mesh.region[e] = p->element_region ? p->element_region[e] : 1;
        }
        for (int b = 0; b < p->num_bfaces; ++b)
            P.mesh.bfaces.push_back({p->bfaces[3 * b], p->bfaces[3 * b + 1], p->bfaces[3 * b + 2]});
        P.p = p->basis_order;
        for (int d = 0; d < p->num_ordinates; ++d)
            P.quad.push_back({p->ord_weight[d], {p->ord_dir[3 * d], p->ord_dir[3 * d + 1], p->ord_dir[3 * d + 2]}});
        for (int r = 0; r < p->num_regions; ++r) {
            if (!(p->sigma_t[r] >= p->sigma_s[r] && p->sigma_s[r] >= 0.0))
                throw std::invalid_argument("cross sections: need sigma_t >= sigma_s >= 0 (region " +
                                            std::to_string(p->region_ids[r]) + ")");
            P.xs[p->region_ids[r]] = {p->sigma_t[r], p->sigma_s[r]};
        }
        P.source.kind = p->source_kind;
        for (int i = 0; i < 8; ++i) P.source.params[i] = p->source_params[i];
        P.source.inflow = p->inflow;
        P.vol_points = p->volume_points;
        P.face_points = p->face_points;
        P.face_rule = p->face_rule;
        if (p->face_rule == 1) {
            P.romberg_tol = p->romberg_tol;
            P.romberg_max_levels = p->romberg_max_levels;
            P.romberg_min_levels = p->romberg_min_levels;
        }
        P.weighting = p->weighting;
        P.fas_threshold = p->fas_threshold;
        auto* o = new orc::Oracle(std::move(P), p->cache_lu != 0);
        if (p->num_active > 0) o->active.assign(p->active, p->active + p->num_active);
        try {
            if (p->validate_geometry) o->validate_geometry();
            o->setup(p->check_rcond != 0);
        } catch (...) {
            delete o;
            throw;
        }
        return o;
    } catch (const std::exception& ex) {
        set_err(ex.what(), err, errlen);
        return nullptr;
    }
}

void orc_destroy(void* h) { delete static_cast<orc::Oracle*>(h); }

int orc_block_size(void* h) { return static_cast<orc::Oracle*>(h)->nb; }
int orc_face_nodes(void* h) { return static_cast<orc::Oracle*>(h)->nf_nodes; }
int orc_num_interior_faces(void* h) { return (int)static_cast<orc::Oracle*>(h)->P.mesh.ifaces.size(); }
void orc_interior_faces(void* h, int* out) {  // 5 ints per face
    auto* o = static_cast<orc::Oracle*>(h);
    for (size_t i = 0; i < o->P.mesh.ifaces.size(); ++i) {
        const auto& f = o->P.mesh.ifaces[i];
        out[5 * i] = f.elem_left; out[5 * i + 1] = f.elem_right;
        out[5 * i + 2] = f.face_left; out[5 * i + 3] = f.face_right; out[5 * i + 4] = f.orientation;
    }
}
int orc_num_couplings(void* h, int d) { return (int)static_cast<orc::Oracle*>(h)->ords[d].couplings.size(); }
// per coupling: face, downwind, upwind, lagged; weight
void orc_couplings(void* h, int d, int* ints, double* weights) {
    auto* o = static_cast<orc::Oracle*>(h);
    const auto& ord = o->ords[d];
    for (size_t c = 0; c < ord.couplings.size(); ++c) {
        ints[4 * c] = ord.couplings[c].face;
        ints[4 * c + 1] = ord.couplings[c].downwind;
        ints[4 * c + 2] = ord.couplings[c].upwind;
        ints[4 * c + 3] = ord.lagged[c];
        if (weights) weights[c] = ord.weights[c];
    }
}
void orc_coupling_block(void* h, int d, int c, double* out) {
    auto* o = static_cast<orc::Oracle*>(h);
    const auto& b = o->ords[d].couplings[c].block;
    std::copy(b.begin(), b.end(), out);
}
int orc_num_lagged(void* h, int d) { return (int)static_cast<orc::Oracle*>(h)->ords[d].lagged_edges.size(); }
double orc_ordering(void* h, int d, int* order, int* position, int* lagged, int* level) {
    auto* o = static_cast<orc::Oracle*>(h);
    const auto& ord = o->ords[d];
    if (order) std::copy(ord.order.begin(), ord.order.end(), order);
    if (position) std::copy(ord.position.begin(), ord.position.end(), position);
    if (lagged) std::copy(ord.lagged_edges.begin(), ord.lagged_edges.end(), lagged);
    if (level) std::copy(ord.level.begin(), ord.level.end(), level);
    return ord.lagged_weight;
}
void orc_mass(void* h, int e, double* mt, double* ms) {
    auto* o = static_cast<orc::Oracle*>(h);
    std::copy(o->mass_total[e].begin(), o->mass_total[e].end(), mt);
    std::copy(o->mass_scatter[e].begin(), o->mass_scatter[e].end(), ms);
}
void orc_source(void* h, int d, double* vol, double* bnd) {
    auto* o = static_cast<orc::Oracle*>(h);
    if (vol) std::copy(o->src_vol.begin(), o->src_vol.end(), vol);
    if (bnd) std::copy(o->ords[d].src_bnd.begin(), o->ords[d].src_bnd.end(), bnd);
}
void orc_diag_block(void* h, int e, int d, double* A) {
    auto* o = static_cast<orc::Oracle*>(h);
    o->diag_block(e, d, o->ords[d], A);
}
int orc_local_solve(void* h, int e, int d, const double* rhs, double* out, char* err, int errlen) {
    try {
        static_cast<orc::Oracle*>(h)->local_solve(e, d, rhs, out);
        return 0;
    } catch (const std::exception& ex) { set_err(ex.what(), err, errlen); return 1; }
}
int orc_sweep(void* h, int d, const double* phi, const double* psi_old, double* psi_new, char* err, int errlen) {
    try {
        static_cast<orc::Oracle*>(h)->sweep(d, phi, psi_old, psi_new);
        return 0;
    } catch (const std::exception& ex) { set_err(ex.what(), err, errlen); return 1; }
}
// all ordinates, in parallel over d (psi_* are [nd][N])
int orc_sweep_all(void* h, const double* phi, const double* psi_old, double* psi_new, char* err, int errlen) {
    try {
        auto* o = static_cast<orc::Oracle*>(h);
        const size_t N = (size_t)o->nel * o->nb;
        orc::parallel_for((int)o->P.quad.size(),
                          [&](int d) { o->sweep(d, phi, psi_old + d * N, psi_new + d * N); });
        return 0;
    } catch (const std::exception& ex) { set_err(ex.what(), err, errlen); return 1; }
}
// sweep a subset of ordinates (timed CPU baseline sample)
int orc_sweep_subset(void* h, int nd, const int* ds, const double* phi, double* psi_scratch, char* err, int errlen) {
    try {
        auto* o = static_cast<orc::Oracle*>(h);
        const size_t N = (size_t)o->nel * o->nb;
        std::vector<double> zero(N, 0.0);
        orc::parallel_for(nd, [&](int i) { o->sweep(ds[i], phi, zero.data(), psi_scratch + i * N); });
        return 0;
    } catch (const std::exception& ex) { set_err(ex.what(), err, errlen); return 1; }
}
// Bounded CPU-baseline sample: for each listed ordinate, the first max_elems
// elements of its sweep order (the reference's per-element work: assemble the
// local block on the fly, factor, solve), psi_old = 0, one ordinate per thread.
// Returns the number of (element, ordinate) solves performed.
long long orc_sweep_sample(void* h, int nd, const int* ds, int max_elems, const double* phi, char* err,
                           int errlen) {
    try {
        auto* o = static_cast<orc::Oracle*>(h);
        const size_t N = (size_t)o->nel * o->nb;
        std::atomic<long long> count{0};
        orc::parallel_for(nd, [&](int i) {
            const int d = ds[i];
            const orc::PerOrdinate& ord = o->ords[d];
            std::vector<double> psi(N, 0.0), zero(N, 0.0), rhs(o->nb), A((size_t)o->nb * o->nb);
            orc::DenseLU lu;
            const int nfn = o->nf_nodes;
            const double c4pi = 1.0 / (4.0 * M_PI);
            const int ne = std::min<int>(max_elems, (int)ord.order.size());
            for (int q = 0; q < ne; ++q) {
                const int e = ord.order[q];
                for (int m = 0; m < o->nb; ++m)
                    rhs[m] = o->src_vol[(size_t)e * o->nb + m] + ord.src_bnd[(size_t)e * o->nb + m];
                const auto& ms = o->mass_scatter[e];
                for (int m = 0; m < o->nb; ++m) {
                    double s = 0.0;
                    for (int n = 0; n < o->nb; ++n) s += ms[(size_t)m * o->nb + n] * phi[(size_t)e * o->nb + n];
                    rhs[m] += c4pi * s;
                }
                for (int c : ord.incoming[e]) {
                    const orc::Coupling& fc = ord.couplings[c];
                    const double* src = ord.lagged[c] ? zero.data() : psi.data();
                    const auto& dn = o->fnodes[fc.down_face];
                    const auto& un = o->fnodes[fc.up_face];
                    for (int m = 0; m < nfn; ++m) {
                        double s = 0.0;
                        for (int n = 0; n < nfn; ++n) s += fc.block[m * nfn + n] * src[(size_t)fc.upwind * o->nb + un[n]];
                        rhs[dn[m]] -= s;
                    }
                }
                o->diag_block(e, d, ord, A.data());
                lu.factor(A.data(), o->nb);
                lu.solve(rhs.data(), &psi[(size_t)e * o->nb]);
            }
            count += ne;
        });
        return count.load();
    } catch (const std::exception& ex) { set_err(ex.what(), err, errlen); return -1; }
}

int orc_direct_oracle(void* h, int d, const double* phi, double* psi, char* err, int errlen) {
    try {
        static_cast<orc::Oracle*>(h)->direct_oracle(d, phi, psi);
        return 0;
    } catch (const std::exception& ex) { set_err(ex.what(), err, errlen); return 1; }
}
int orc_source_iteration(void* h, double tol, int max_it, int criterion, double* psi, double* phi,
                         double* err_hist, double* phi_hist, int* converged, char* err, int errlen) {
    try {
        return static_cast<orc::Oracle*>(h)->source_iteration(tol, max_it, criterion, psi, phi, err_hist,
                                                              phi_hist, converged);
    } catch (const std::exception& ex) { set_err(ex.what(), err, errlen); return -1; }
}
// out[5] = src_vol, inflow, absorption, outflow, residual; attrs/vals up to max_attr entries
int orc_balance(void* h, const double* psi, const double* phi, double* out, int* attrs, double* vals, int max_attr) {
    auto* o = static_cast<orc::Oracle*>(h);
    std::map<int, double> by;
    o->balance(psi, phi, out, by);
    int k = 0;
    for (const auto& kv : by) {
        if (k >= max_attr) break;
        attrs[k] = kv.first;
        vals[k] = kv.second;
        ++k;
    }
    return k;
}

// Standalone graph algorithms on caller-supplied graphs (sweepgraph tests).
// edges: (from, to) pairs; returns number of SCCs; comp_out: scc id per vertex
// in Tarjan emission order; order/position/lagged output of sweep_ordering.
int orc_graph_tarjan(int nv, int ne, const int* edges, int* comp_out) {
    orc::Oracle::Graph g;
    g.nv = nv;
    for (int i = 0; i < ne; ++i) g.edges.push_back({edges[2 * i], edges[2 * i + 1], 1.0, i});
    const auto sccs = orc::Oracle::tarjan_scc(g);
    for (size_t c = 0; c < sccs.size(); ++c)
        for (int v : sccs[c]) comp_out[v] = (int)c;
    return (int)sccs.size();
}
// mode 0 exact, 1 heuristic, 2 sweep_ordering(threshold)
double orc_graph_order(int nv, int ne, const int* edges, const double* w, int mode, int threshold,
                       int* order, int* nlagged, int* lagged) {
    orc::Oracle::Graph g;
    g.nv = nv;
    for (int i = 0; i < ne; ++i) g.edges.push_back({edges[2 * i], edges[2 * i + 1], w[i], i});
    std::vector<int> all(nv);
    std::iota(all.begin(), all.end(), 0);
    if (mode == 2) {
        orc::PerOrdinate res;
        orc::Oracle::sweep_ordering(g, threshold, res);
        std::copy(res.order.begin(), res.order.end(), order);
        *nlagged = (int)res.lagged_edges.size();
        std::copy(res.lagged_edges.begin(), res.lagged_edges.end(), lagged);
        return res.lagged_weight;
    }
    const auto r = mode == 0 ? orc::Oracle::min_fas_exact(g, all) : orc::Oracle::min_fas_heuristic(g, all);
    std::copy(r.order.begin(), r.order.end(), order);
    *nlagged = (int)r.lagged.size();
    std::copy(r.lagged.begin(), r.lagged.end(), lagged);
    return r.weight;
}

// Quadrature / basis known answers (quadrature.hpp, basis.hpp)
void orc_gauss_legendre(int n, double* pts, double* wts) {
    const auto q = orc::gauss_legendre(n);
    std::copy(q.points.begin(), q.points.end(), pts);
    std::copy(q.weights.begin(), q.weights.end(), wts);
}
void orc_gauss_lobatto(int n, double* pts) {
    const auto q = orc::gauss_lobatto(n);
    std::copy(q.begin(), q.end(), pts);
}
void orc_basis_eval(int dim, int order, const double* xi, double* vals, double* grads) {
    orc::Basis b(dim, order);
    if (vals) b.values(xi, vals);
    if (grads) b.gradients(xi, grads);
}
// mesh geometry probes
int orc_face_geometry(void* h, int e, int f, double s, double t, double* out7) {
    auto* o = static_cast<orc::Oracle*>(h);
    const auto fg = o->P.mesh.face_geometry(e, f, s, t);
    for (int i = 0; i < 3; ++i) { out7[i] = fg.point[i]; out7[3 + i] = fg.normal[i]; }
    out7[6] = fg.sj;
    return 0;
}
double orc_jacobian(void* h, int e, const double* xi, double* J9) {
    return static_cast<orc::Oracle*>(h)->P.mesh.jacobian(e, xi, J9);
}
// test hook: zero the assembled local block of (e, d) before factorization
// (the reference test pokes op.ordinates[d].diag[e].setZero(), test_solver.cpp:332-344)
void* orc_create_with_zero_block(const orc_problem* p, int e, int d, char* err, int errlen) {
    try {
        orc_problem q = *p;
        q.check_rcond = 0;
        q.cache_lu = 0;
        void* h = orc_create(&q, err, errlen);
        if (!h) return nullptr;
        std::unique_ptr<orc::Oracle> guard(static_cast<orc::Oracle*>(h));
        auto* o = guard.get();
        o->diag_override_zero.assign(o->P.quad.size(), {});
        o->diag_override_zero[d].assign(o->nel, 0.0);
        o->diag_override_zero[d][e] = 1.0;
        // re-run the constructor's factorization check with the poked block
        // (the handle stays in on-the-fly mode, cache_lu = false)
        orc::parallel_for((int)o->P.quad.size(), [&](int dd) {
            std::vector<double> A((size_t)o->nb * o->nb);
            orc::DenseLU lu;
            for (int ee = 0; ee < o->nel; ++ee) {
                o->diag_block(ee, dd, o->ords[dd], A.data());
                lu.factor(A.data(), o->nb);
                if (!(lu.rcond() > 1e-14))
                    throw orc::SolverError("local streaming+collision block is singular (element " +
                                           std::to_string(ee) + ", ordinate " + std::to_string(dd) + ")");
            }
        });
        return guard.release();
    } catch (const std::exception& ex) {
        set_err(ex.what(), err, errlen);
        return nullptr;
    }
}

}  // extern "C"
