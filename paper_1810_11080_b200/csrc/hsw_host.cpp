// Host side of the B200 transport sweep: problem ingestion, mesh face pairing,
// exact face geometry, per-element operator tensors, per-ordinate couplings,
// dependency graphs, cut sets, orderings, levels and worklists, and the C ABI
// declared in include/hosweep_b200.h.
//
// Reference mapping (paths under /root/reference/proj/include/hosweep/):
//   quadrature.hpp:23-104  -> gauss_legendre / gauss_lobatto / tensor rule
//   basis.hpp:15-133       -> Lagrange1D / TensorBasis
//   mesh.hpp:121-365       -> Mesh::build_faces / jacobian / face_geometry / checks
//   assembly.hpp:58-163    -> element_tensors (M, G_k = -(d_k u)^T W u; the per-ordinate
//                             stream block is sum_k Omega_k G_k, assembled on the GPU)
//   assembly.hpp:185-268   -> face_couplings (Gauss face rule, shared sampling,
//                             edge threshold 1e-12*length) — bit-exact with the reference
//                             element-wise arithmetic so the graph is bit-exact
//   sweepgraph.hpp:54-396  -> build_graph / tarjan_scc / min_fas_* / sweep_ordering
//   solver.hpp:52-168      -> hsw_create (ctor), hsw_sweep, hsw_source_iteration
//   solver.hpp:220-245     -> hsw_balance
// Compiled with -ffp-contract=off: every quantity that feeds an integer
// decision is evaluated with the reference's operation order.
#include "hosweep_b200.h"
#include "hsw_internal.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sys/mman.h>
#include <exception>
#include <limits>
#include <map>
#include <functional>
#include <memory>
#include <mutex>
#include <numeric>
#include <queue>
#include <thread>
#include <tuple>
#include <vector>

namespace hsw {

// std::vector whose resize() leaves new elements uninitialised: the large tables that a
// parallel loop fills completely are first touched by the threads that write them, not
// zero-filled (page faults included) by one thread beforehand.
template <typename T>
struct default_init_allocator : std::allocator<T> {
    template <typename U> struct rebind { using other = default_init_allocator<U>; };
    using std::allocator<T>::allocator;
    template <typename U> void construct(U* ptr) noexcept(std::is_nothrow_default_constructible<U>::value) {
        ::new (static_cast<void*>(ptr)) U;
    }
    template <typename U, typename... Args> void construct(U* ptr, Args&&... args) {
        ::new (static_cast<void*>(ptr)) U(std::forward<Args>(args)...);
    }
};
template <typename T> using raw_vector = std::vector<T, default_init_allocator<T>>;

// ------------------------------------------------------------------ threads
static int host_workers() {
    if (const char* env = std::getenv("HOSWEEP_THREADS")) {  // parallel.hpp:16-23
        const int n = std::atoi(env);
        if (n >= 1) return n;
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : (int)hw;
}

template <typename Fn>
static void parallel_for(int64_t n, Fn&& fn) {
    const int workers = (int)std::min<int64_t>(n, host_workers());
    if (workers <= 1) {
        for (int64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    std::exception_ptr error;
    std::mutex mu;
    std::atomic<int64_t> next{0};
    for (int w = 0; w < workers; ++w)
        pool.emplace_back([&] {
            for (;;) {
                const int64_t i = next.fetch_add(1);
                if (i >= n) return;
                try {
                    fn(i);
                } catch (...) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!error) error = std::current_exception();
                    return;
                }
            }
        });
    for (auto& t : pool) t.join();
    if (error) std::rethrow_exception(error);
}

// ----------------------------------------------------------------- numerics
static void legendre(int n, double x, double& p, double& dp) {  // quadrature.hpp:23-34
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

struct Rule { std::vector<double> x, w; };

static Rule gauss_legendre(int n) {  // quadrature.hpp:38-59
    if (n < 1) throw Error(HSW_ERR_INVALID, "gauss_legendre: need n >= 1");
    Rule r;
    r.x.resize(n);
    r.w.resize(n);
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
        r.x[n - 1 - i] = 0.5 * (x + 1.0);
        r.w[n - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);
    }
    return r;
}

static std::vector<double> gauss_lobatto(int n) {  // quadrature.hpp:62-82
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

// Lagrange1D product form (basis.hpp:15-60) and the tensor basis
// (basis.hpp:62-133, 3D: m = (iz*n1 + iy)*n1 + ix, value (vx*vy)*vz).
struct TensorBasis {
    int dim = 2, order = 1, n1 = 2, nb = 4;
    std::vector<double> nodes;
    TensorBasis() = default;
    TensorBasis(int d, int p) : dim(d), order(p), n1(p + 1) {
        nodes = gauss_lobatto(p + 1);
        nb = d == 2 ? n1 * n1 : n1 * n1 * n1;
    }
    double value(int j, double x) const {
        double v = 1.0;
        for (int k = 0; k < n1; ++k) {
            if (k == j) continue;
            v *= (x - nodes[k]) / (nodes[j] - nodes[k]);
        }
        return v;
    }
    double derivative(int j, double x) const {
        double d = 0.0;
        for (int i = 0; i < n1; ++i) {
            if (i == j) continue;
            double term = 1.0 / (nodes[j] - nodes[i]);
            for (int k = 0; k < n1; ++k) {
                if (k == j || k == i) continue;
                term *= (x - nodes[k]) / (nodes[j] - nodes[k]);
            }
            d += term;
        }
        return d;
    }
    void values(const double* xi, double* out) const {
        double vx[32], vy[32], vz[32];
        for (int j = 0; j < n1; ++j) { vx[j] = value(j, xi[0]); vy[j] = value(j, xi[1]); }
        if (dim == 2) {
            for (int iy = 0; iy < n1; ++iy)
                for (int ix = 0; ix < n1; ++ix) out[iy * n1 + ix] = vx[ix] * vy[iy];
            return;
        }
        for (int j = 0; j < n1; ++j) vz[j] = value(j, xi[2]);
        for (int iz = 0; iz < n1; ++iz)
            for (int iy = 0; iy < n1; ++iy)
                for (int ix = 0; ix < n1; ++ix) out[(iz * n1 + iy) * n1 + ix] = vx[ix] * vy[iy] * vz[iz];
    }
    void gradients(const double* xi, double* out) const {  // out[m*dim + k]
        double vx[32], vy[32], vz[32], dx[32], dy[32], dz[32];
        for (int j = 0; j < n1; ++j) {
            vx[j] = value(j, xi[0]); vy[j] = value(j, xi[1]);
            dx[j] = derivative(j, xi[0]); dy[j] = derivative(j, xi[1]);
        }
        if (dim == 2) {
            for (int iy = 0; iy < n1; ++iy)
                for (int ix = 0; ix < n1; ++ix) {
                    const int m = iy * n1 + ix;
                    out[2 * m] = dx[ix] * vy[iy];
                    out[2 * m + 1] = vx[ix] * dy[iy];
                }
            return;
        }
        for (int j = 0; j < n1; ++j) { vz[j] = value(j, xi[2]); dz[j] = derivative(j, xi[2]); }
        for (int iz = 0; iz < n1; ++iz)
            for (int iy = 0; iy < n1; ++iy)
                for (int ix = 0; ix < n1; ++ix) {
                    const int m = (iz * n1 + iy) * n1 + ix;
                    out[3 * m] = dx[ix] * vy[iy] * vz[iz];
                    out[3 * m + 1] = vx[ix] * dy[iy] * vz[iz];
                    out[3 * m + 2] = vx[ix] * vy[iy] * dz[iz];
                }
    }
};

// --------------------------------------------------------- reference faces
// 2D: mesh.hpp:64-109.  3D: 0 z=0 (s,t,0); 1 y=0 (s,0,t); 2 x=1 (1,s,t);
// 3 y=1 (s,1,t); 4 x=0 (0,s,t); 5 z=1 (s,t,1).  DESIGN.md §3.
static int nfaces_of(int dim) { return dim == 2 ? 4 : 6; }

static void param_point(int dim, int f, double s, double t, double* xi) {
    xi[2] = 0.0;
    if (dim == 2) {
        static const double fix[4][2] = {{-1, 0}, {1, -1}, {-1, 1}, {0, -1}};
        (void)fix;
        switch (f) {
            case 0: xi[0] = s; xi[1] = 0.0; return;
            case 1: xi[0] = 1.0; xi[1] = s; return;
            case 2: xi[0] = s; xi[1] = 1.0; return;
            default: xi[0] = 0.0; xi[1] = s; return;
        }
    }
    switch (f) {
        case 0: xi[0] = s; xi[1] = t; xi[2] = 0.0; return;
        case 1: xi[0] = s; xi[1] = 0.0; xi[2] = t; return;
        case 2: xi[0] = 1.0; xi[1] = s; xi[2] = t; return;
        case 3: xi[0] = s; xi[1] = 1.0; xi[2] = t; return;
        case 4: xi[0] = 0.0; xi[1] = s; xi[2] = t; return;
        default: xi[0] = s; xi[1] = t; xi[2] = 1.0; return;
    }
}
static void face_axes(int dim, int f, int& a0, int& a1) {
    if (dim == 2) { a0 = (f == 0 || f == 2) ? 0 : 1; a1 = -1; return; }
    if (f == 0 || f == 5) { a0 = 0; a1 = 1; }
    else if (f == 1 || f == 3) { a0 = 0; a1 = 2; }
    else { a0 = 1; a1 = 2; }
}
static void ref_normal(int dim, int f, double* n) {
    n[0] = n[1] = n[2] = 0.0;
    if (dim == 2) {
        static const double t[4][2] = {{0, -1}, {1, 0}, {0, 1}, {-1, 0}};
        n[0] = t[f][0]; n[1] = t[f][1];
        return;
    }
    static const double t[6][3] = {{0, 0, -1}, {0, -1, 0}, {1, 0, 0}, {0, 1, 0}, {-1, 0, 0}, {0, 0, 1}};
    n[0] = t[f][0]; n[1] = t[f][1]; n[2] = t[f][2];
}
static std::vector<int> face_nodes(int dim, int f, int order) {
    const int n1 = order + 1;
    std::vector<int> idx;
    if (dim == 2) {
        for (int k = 0; k < n1; ++k) {
            switch (f) {
                case 0: idx.push_back(k); break;
                case 1: idx.push_back(order + k * n1); break;
                case 2: idx.push_back(order * n1 + k); break;
                default: idx.push_back(k * n1); break;
            }
        }
        return idx;
    }
    for (int b = 0; b < n1; ++b)
        for (int a = 0; a < n1; ++a) {
            int ix, iy, iz;
            switch (f) {
                case 0: ix = a; iy = b; iz = 0; break;
                case 1: ix = a; iy = 0; iz = b; break;
                case 2: ix = order; iy = a; iz = b; break;
                case 3: ix = a; iy = order; iz = b; break;
                case 4: ix = 0; iy = a; iz = b; break;
                default: ix = a; iy = b; iz = order; break;
            }
            idx.push_back((iz * n1 + iy) * n1 + ix);
        }
    return idx;
}
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
static int orient_inverse(int dim, int code) {
    if (dim == 2) return code;
    for (int c = 0; c < 8; ++c) {
        bool ok = true;
        for (int a = 0; a < 3 && ok; ++a)
            for (int b = 0; b < 3 && ok; ++b) {
                int a1, b1, a2, b2;
                orient_index(3, code, 2, a, b, a1, b1);
                orient_index(3, c, 2, a1, b1, a2, b2);
                if (a2 != a || b2 != b) ok = false;
            }
        if (ok) return c;
    }
    return code;
}

// --------------------------------------------------------------------- mesh
struct IFace { int el, er, fl, fr, orient; };
struct BFace { int elem, face, attr; };

struct Mesh {
    int dim = 2, order = 1, npe = 4;
    TensorBasis geom;
    std::vector<double> pts;  // P * dim
    std::vector<int> enodes;  // E * npe
    std::vector<int> region;
    std::vector<BFace> bfaces;
    std::vector<IFace> ifaces;
    int nel = 0;

    const double* X(int e, int m) const { return &pts[(size_t)enodes[(size_t)e * npe + m] * dim]; }

    // mesh.hpp:157-170 with a precomputed gradient table g (npe*dim) at xi
    double jacobian_tab(int e, const double* g, double* J) const {
        for (int i = 0; i < 9; ++i) J[i] = 0.0;
        const int* en = &enodes[(size_t)e * npe];
        if (dim == 3) {   // same sums in the same (ascending m) order, fixed trip counts
            double j[9] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            for (int m = 0; m < npe; ++m) {
                const double* x = &pts[(size_t)en[m] * 3];
                const double* gm = g + (size_t)m * 3;
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b) j[a * 3 + b] += x[a] * gm[b];
            }
            for (int i = 0; i < 9; ++i) J[i] = j[i];
            return det(J);
        }
        for (int m = 0; m < npe; ++m) {
            const double* x = X(e, m);
            for (int a = 0; a < dim; ++a)
                for (int b = 0; b < dim; ++b) J[a * 3 + b] += x[a] * g[m * dim + b];
        }
        return det(J);
    }
    double det(const double* J) const {
        if (dim == 2) return J[0] * J[4] - J[3] * J[1];
        const double c0 = J[4] * J[8] - J[5] * J[7];
        const double c1 = J[5] * J[6] - J[3] * J[8];
        const double c2 = J[3] * J[7] - J[4] * J[6];
        return J[0] * c0 + J[1] * c1 + J[2] * c2;
    }
    void inverse(const double* J, double* K) const {
        if (dim == 2) {
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
    void map_tab(int e, const double* v, double* x) const {  // mesh.hpp:147-154
        x[0] = x[1] = x[2] = 0.0;
        for (int m = 0; m < npe; ++m) {
            const double* p = X(e, m);
            for (int a = 0; a < dim; ++a) x[a] += v[m] * p[a];
        }
    }
    double diameter(int e) const {  // mesh.hpp:204-217
        const int r = order, n1 = r + 1;
        std::vector<int> c;
        if (dim == 2) c = {0, r, r * n1, r * n1 + r};
        else
            for (int cz : {0, r})
                for (int cy : {0, r})
                    for (int cx : {0, r}) c.push_back((cz * n1 + cy) * n1 + cx);
        double d = 0.0;
        for (size_t i = 0; i < c.size(); ++i)
            for (size_t j = i + 1; j < c.size(); ++j) {
                double s = 0.0;
                for (int a = 0; a < dim; ++a) {
                    const double df = X(e, c[i])[a] - X(e, c[j])[a];
                    s += df * df;
                }
                d = std::max(d, std::sqrt(s));
            }
        return d;
    }
    // mesh.hpp:180-200 given the geometry gradient table at the face point
    // diam: the element's diameter when the caller already has it (< 0: computed here)
    // Jacobians of element e at n points at once: gt is the gradient table transposed to
    // [npe][n * dim] (point-major inside a node), out is [dim][n * dim], so that
    // J_q[a][b] = out[a * n * dim + q * dim + b].  Every entry is the same sum over the
    // nodes in the same ascending order as jacobian_tab (no FMA contraction), so the bits
    // agree; the inner loop runs over contiguous memory and vectorises.
    void jacobians_batch(int e, const double* gt, int n, double* out) const {
        const int w = n * dim;
        for (int i = 0; i < dim * w; ++i) out[i] = 0.0;
        const int* en = &enodes[(size_t)e * npe];
        for (int m = 0; m < npe; ++m) {
            const double* x = &pts[(size_t)en[m] * dim];
            const double* gm = gt + (size_t)m * w;
            for (int a = 0; a < dim; ++a) {
                const double xa = x[a];
                double* o = out + (size_t)a * w;
                for (int i = 0; i < w; ++i) o[i] += xa * gm[i];
            }
        }
    }
    void unpack_jacobian(const double* out, int n, int q, double* J) const {
        for (int i = 0; i < 9; ++i) J[i] = 0.0;
        for (int a = 0; a < dim; ++a)
            for (int b = 0; b < dim; ++b) J[a * 3 + b] = out[(size_t)a * n * dim + (size_t)q * dim + b];
    }
    void face_geometry_tab(int e, int f, const double* g, double* normal, double& sj, double diam = -1.0) const {
        double J[9];
        jacobian_tab(e, g, J);
        face_geometry_J(e, f, J, normal, sj, diam);
    }
    void face_geometry_J(int e, int f, const double* J, double* normal, double& sj, double diam = -1.0) const {
        int a0, a1;
        face_axes(dim, f, a0, a1);
        if (dim == 2) {
            const double t0 = J[a0], t1 = J[3 + a0];
            sj = std::sqrt(t0 * t0 + t1 * t1);
        } else {
            const double u0 = J[a0], u1 = J[3 + a0], u2 = J[6 + a0];
            const double v0 = J[a1], v1 = J[3 + a1], v2 = J[6 + a1];
            const double c0 = u1 * v2 - u2 * v1;
            const double c1 = u2 * v0 - u0 * v2;
            const double c2 = u0 * v1 - u1 * v0;
            sj = std::sqrt(c0 * c0 + c1 * c1 + c2 * c2);
        }
        if (sj < 1e-14 * (diam >= 0.0 ? diam : diameter(e)))
            throw Error(HSW_ERR_GEOMETRY, "face_geometry: degenerate tangent on element " +
                                              std::to_string(e) + " face " + std::to_string(f));
        double K[9], nref[3];
        inverse(J, K);
        ref_normal(dim, f, nref);
        double z = 0.0;
        for (int i = 0; i < dim; ++i) {
            double v = 0.0;
            for (int j = 0; j < dim; ++j) v += K[j * 3 + i] * nref[j];
            normal[i] = v;
        }
        for (int i = 0; i < dim; ++i) z += normal[i] * normal[i];
        if (z > 0.0) {
            const double rt = std::sqrt(z);
            for (int i = 0; i < dim; ++i) normal[i] /= rt;
        }
        if (dim == 2) normal[2] = 0.0;
    }
    std::vector<int> face_global(int e, int f) const {
        std::vector<int> out;
        for (int m : face_nodes(dim, f, order)) out.push_back(enodes[(size_t)e * npe + m]);
        return out;
    }
    // mesh.hpp:242-262
    void check_connectivity(int num_points) const {
        for (int e = 0; e < nel; ++e)
            for (int m = 0; m < npe; ++m) {
                const int idx = enodes[(size_t)e * npe + m];
                if (idx < 0 || idx >= num_points)
                    throw Error(HSW_ERR_MESH, "mesh: element " + std::to_string(e) +
                                                  " references control point " + std::to_string(idx) +
                                                  " out of range");
            }
        for (const auto& b : bfaces)
            if (b.elem < 0 || b.elem >= nel || b.face < 0 || b.face >= nfaces_of(dim))
                throw Error(HSW_ERR_MESH, "mesh: boundary face record (elem " + std::to_string(b.elem) +
                                              ", face " + std::to_string(b.face) + ") out of range");
    }
    // mesh.hpp:275-339; interior-face ids follow the sorted corner keys (std::map order)
    void build_faces() {
        const int nf = nfaces_of(dim), r = order, n1 = r + 1;
        struct Side { std::array<int, 4> key; int e, f; };
        std::vector<Side> sides;
        sides.reserve((size_t)nel * nf);
        for (int e = 0; e < nel; ++e)
            for (int f = 0; f < nf; ++f) {
                const auto g = face_global(e, f);
                std::array<int, 4> key{};
                if (dim == 2) {
                    key = {g.front(), g.back(), -1, -1};
                    if (key[0] > key[1]) std::swap(key[0], key[1]);
                } else {
                    key = {g[0], g[r], g[r * n1], g[r * n1 + r]};
                    std::sort(key.begin(), key.end());
                }
                sides.push_back({key, e, f});
            }
        std::stable_sort(sides.begin(), sides.end(), [](const Side& a, const Side& b) { return a.key < b.key; });
        std::vector<char> paired((size_t)nel * nf, 0);
        ifaces.clear();
        for (size_t i = 0; i < sides.size();) {
            size_t j = i;
            while (j < sides.size() && sides[j].key == sides[i].key) ++j;
            const size_t cnt = j - i;
            if (cnt > 2)
                throw Error(HSW_ERR_MESH, "mesh: face shared by " + std::to_string(cnt) + " elements");
            if (cnt == 2) {
                const int e0 = sides[i].e, f0 = sides[i].f, e1 = sides[i + 1].e, f1 = sides[i + 1].f;
                const auto g0 = face_global(e0, f0), g1 = face_global(e1, f1);
                int orient = -1;
                const int ncodes = dim == 2 ? 2 : 8;
                for (int code = 0; code < ncodes && orient < 0; ++code) {
                    bool ok = true;
                    for (int b = 0; b < (dim == 2 ? 1 : n1) && ok; ++b)
                        for (int a = 0; a < n1 && ok; ++a) {
                            int ao, bo;
                            orient_index(dim, code, r, a, b, ao, bo);
                            if (g1[bo * n1 + ao] != g0[b * n1 + a]) ok = false;
                        }
                    if (ok) orient = code;
                }
                if (orient < 0)
                    throw Error(HSW_ERR_MESH, "mesh: elements " + std::to_string(e0) + " and " +
                                                  std::to_string(e1) +
                                                  " share face corners but edge nodes do not match");
                ifaces.push_back({e0, e1, f0, f1, orient});
                paired[(size_t)e0 * nf + f0] = paired[(size_t)e1 * nf + f1] = 1;
            }
            i = j;
        }
        std::vector<char> declared((size_t)nel * nf, 0);
        for (const auto& b : bfaces) {
            if (paired[(size_t)b.elem * nf + b.face])
                throw Error(HSW_ERR_MESH, "mesh: boundary record for interior face (elem " +
                                              std::to_string(b.elem) + ", face " + std::to_string(b.face) + ")");
            if (declared[(size_t)b.elem * nf + b.face])
                throw Error(HSW_ERR_MESH, "mesh: duplicate boundary record (elem " + std::to_string(b.elem) +
                                              ", face " + std::to_string(b.face) + ")");
            declared[(size_t)b.elem * nf + b.face] = 1;
        }
        for (int e = 0; e < nel; ++e)
            for (int f = 0; f < nf; ++f)
                if (!paired[(size_t)e * nf + f] && !declared[(size_t)e * nf + f])
                    throw Error(HSW_ERR_MESH, "mesh: face (elem " + std::to_string(e) + ", face " +
                                                  std::to_string(f) + ") is neither interior nor declared boundary");
    }
};

// ------------------------------------------------------------ sweep graph
struct Edge { int from, to; double weight; };

struct Fas { std::vector<int> order, lagged; double weight = 0.0; };
struct Local { std::vector<int> verts; std::vector<std::array<int, 2>> e; std::vector<double> w; std::vector<int> parent; };

// induce (sweepgraph.hpp:156-170) without the scan over every edge of the graph per component (O(E) per SCC,
// quadratic on twisted meshes with many cyclic components): the component's out-edges
// from the CSR adjacency, sorted by edge id, give the same local edge list in the same
// (ascending edge id) order, so FAS tie-breaks and `parent` are unchanged.
struct OutCsr { std::vector<int> off, eid; };
static OutCsr out_csr(int nv, const std::vector<Edge>& edges) {
    OutCsr g;
    g.off.assign(nv + 1, 0);
    for (const auto& ed : edges) g.off[ed.from + 1]++;
    for (int v = 0; v < nv; ++v) g.off[v + 1] += g.off[v];
    g.eid.resize(edges.size());
    std::vector<int> fill(g.off.begin(), g.off.end() - 1);
    for (size_t k = 0; k < edges.size(); ++k) g.eid[fill[edges[k].from]++] = (int)k;   // ascending per vertex
    return g;
}
static Local induce_csr(const OutCsr& g, const std::vector<Edge>& edges, const std::vector<int>& vs,
                        std::vector<int>& scratch, std::vector<int>& ks) {
    Local lg;
    lg.verts = vs;
    if (scratch.size() != g.off.size() - 1) scratch.assign(g.off.size() - 1, -1);
    for (size_t i = 0; i < vs.size(); ++i) scratch[vs[i]] = (int)i;
    ks.clear();
    for (int v : vs)
        for (int j = g.off[v]; j < g.off[v + 1]; ++j)
            if (scratch[edges[g.eid[j]].to] >= 0) ks.push_back(g.eid[j]);
    std::sort(ks.begin(), ks.end());
    for (int k : ks) {
        const auto& ed = edges[k];
        lg.e.push_back({scratch[ed.from], scratch[ed.to]});
        lg.w.push_back(ed.weight);
        lg.parent.push_back(k);
    }
    for (int v : vs) scratch[v] = -1;
    return lg;
}
static Fas order_result(const Local& lg, const std::vector<int>& lo) {  // sweepgraph.hpp:173-186
    Fas r;
    std::vector<int> pos(lg.verts.size());
    for (size_t k = 0; k < lo.size(); ++k) pos[lo[k]] = (int)k;
    for (size_t k = 0; k < lg.e.size(); ++k)
        if (pos[lg.e[k][0]] > pos[lg.e[k][1]]) {
            r.lagged.push_back(lg.parent[k]);
            r.weight += lg.w[k];
        }
    for (int v : lo) r.order.push_back(lg.verts[v]);
    return r;
}
static Fas fas_exact(const Local& lg) {  // sweepgraph.hpp:192-232
    const int n = (int)lg.verts.size();
    if (n > 22) throw Error(HSW_ERR_INVALID, "min_fas_exact: component too large");
    std::vector<double> wout((size_t)n * n, 0.0);
    for (size_t k = 0; k < lg.e.size(); ++k) wout[(size_t)lg.e[k][0] * n + lg.e[k][1]] += lg.w[k];
    const uint32_t full = (uint32_t(1) << n) - 1;
    std::vector<double> dp((size_t)full + 1, std::numeric_limits<double>::infinity());
    std::vector<int8_t> choice((size_t)full + 1, -1);
    dp[0] = 0.0;
    for (uint32_t mask = 1; mask <= full; ++mask)
        for (int v = 0; v < n; ++v) {
            if (!(mask & (uint32_t(1) << v))) continue;
            const uint32_t rest = mask & ~(uint32_t(1) << v);
            if (dp[rest] == std::numeric_limits<double>::infinity()) continue;
            double back = 0.0;
            for (int u = 0; u < n; ++u)
                if (rest & (uint32_t(1) << u)) back += wout[(size_t)v * n + u];
            const double cand = dp[rest] + back;
            if (cand < dp[mask]) {
                dp[mask] = cand;
                choice[mask] = (int8_t)v;
            }
        }
    std::vector<int> lo(n);
    uint32_t mask = full;
    for (int k = n - 1; k >= 0; --k) {
        const int v = choice[mask];
        lo[k] = v;
        mask &= ~(uint32_t(1) << v);
    }
    return order_result(lg, lo);
}
static Fas fas_heuristic(const Local& lg) {  // sweepgraph.hpp:238-315
    const int n = (int)lg.verts.size();
    std::vector<std::vector<std::pair<int, double>>> out(n), in(n);
    std::vector<double> wout(n, 0.0), win(n, 0.0);
    std::vector<int> dout(n, 0), din(n, 0);
    for (size_t k = 0; k < lg.e.size(); ++k) {
        const int u = lg.e[k][0], v = lg.e[k][1];
        const double w = lg.w[k];
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
        bool prog = true;
        while (prog) {
            prog = false;
            for (int v = 0; v < n; ++v)
                if (!removed[v] && dout[v] == 0) { drop(v); tail.push_back(v); left--; prog = true; }
        }
        prog = true;
        while (prog) {
            prog = false;
            for (int v = 0; v < n; ++v)
                if (!removed[v] && dout[v] > 0 && din[v] == 0) { drop(v); head.push_back(v); left--; prog = true; }
        }
        if (left == 0) break;
        int best = -1;
        double bd = -std::numeric_limits<double>::infinity();
        for (int v = 0; v < n; ++v) {
            if (removed[v]) continue;
            const double delta = wout[v] - win[v];
            if (delta > bd) { bd = delta; best = v; }
        }
        drop(best);
        head.push_back(best);
        left--;
    }
    std::vector<int> lo = std::move(head);
    lo.insert(lo.end(), tail.rbegin(), tail.rend());
    return order_result(lg, lo);
}

struct Ordering {
    std::vector<int> order, position, lagged_edges, level;
    double lagged_weight = 0.0;
};

// Tarjan (sweepgraph.hpp:82-136) over the CSR adjacency, flat outputs: the same visit
// order (roots ascending, out-edges by ascending edge id) as tarjan_scc, so the same
// components in the same emission order, each sorted ascending; no per-vertex vectors.
struct FlatScc { std::vector<int> comp, off, verts; };
static FlatScc tarjan_flat(int n, const OutCsr& g, const std::vector<Edge>& edges) {
    FlatScc r;
    r.comp.assign(n, -1);
    r.off.push_back(0);
    r.verts.reserve(n);
    std::vector<int> index(n, -1), low(n, 0), stack;
    std::vector<char> on(n, 0);
    struct Frame { int v, child; };
    std::vector<Frame> call;
    int next = 0;
    for (int root = 0; root < n; ++root) {
        if (index[root] != -1) continue;
        call.push_back({root, g.off[root]});
        index[root] = low[root] = next++;
        stack.push_back(root);
        on[root] = 1;
        while (!call.empty()) {
            Frame& fr = call.back();
            if (fr.child < g.off[fr.v + 1]) {
                const int w = edges[g.eid[fr.child++]].to;
                if (index[w] == -1) {
                    index[w] = low[w] = next++;
                    stack.push_back(w);
                    on[w] = 1;
                    call.push_back({w, g.off[w]});
                } else if (on[w]) {
                    low[fr.v] = std::min(low[fr.v], index[w]);
                }
            } else {
                const int v = fr.v;
                if (low[v] == index[v]) {
                    const size_t b = r.verts.size();
                    int w;
                    do {
                        w = stack.back();
                        stack.pop_back();
                        on[w] = 0;
                        r.verts.push_back(w);
                    } while (w != v);
                    std::sort(r.verts.begin() + b, r.verts.end());
                    const int c = (int)r.off.size() - 1;
                    for (size_t k = b; k < r.verts.size(); ++k) r.comp[r.verts[k]] = c;
                    r.off.push_back((int)r.verts.size());
                }
                call.pop_back();
                if (!call.empty()) low[call.back().v] = std::min(low[call.back().v], low[v]);
            }
        }
    }
    return r;
}

// sweepgraph.hpp:331-396 (flat-array restatement; same order, cut set and weights)
static Ordering sweep_ordering(int n, const std::vector<Edge>& edges, int thr) {
    const OutCsr g = out_csr(n, edges);
    const FlatScc S = tarjan_flat(n, g, edges);
    const std::vector<int>& comp = S.comp;
    const int nc = (int)S.off.size() - 1;
    // condensation edges, sorted unique per source component (CSR)
    // (bucketed by source component, each small bucket sorted and deduplicated: the same
    // list as a global sort + unique of the (source, target) pairs)
    std::vector<std::pair<int, int>> ce;
    std::vector<int> coff((size_t)nc + 1, 0), cin(nc, 0);
    {
        std::vector<int> boff((size_t)nc + 1, 0);
        for (const auto& e : edges)
            if (comp[e.from] != comp[e.to]) boff[(size_t)comp[e.from] + 1]++;
        for (int c = 0; c < nc; ++c) boff[(size_t)c + 1] += boff[c];
        std::vector<int> tgt(boff[nc]), fill(boff.begin(), boff.end() - 1);
        for (const auto& e : edges) {
            const int cu = comp[e.from], cv = comp[e.to];
            if (cu != cv) tgt[fill[cu]++] = cv;
        }
        ce.reserve(tgt.size());
        for (int c = 0; c < nc; ++c) {
            int* b = tgt.data() + boff[c];
            int* e = tgt.data() + boff[(size_t)c + 1];
            std::sort(b, e);
            e = std::unique(b, e);
            for (int* q = b; q != e; ++q) {
                ce.push_back({c, *q});
                cin[*q]++;
            }
            coff[(size_t)c + 1] = (int)ce.size();
        }
    }
    using Key = std::pair<int, int>;
    std::priority_queue<Key, std::vector<Key>, std::greater<Key>> ready;
    for (int c = 0; c < nc; ++c)
        if (cin[c] == 0) ready.push({S.verts[S.off[c]], c});
    Ordering res;
    res.order.reserve(n);
    std::vector<int> scratch, ks, vs;
    while (!ready.empty()) {
        const int c = ready.top().second;
        ready.pop();
        const int sz = S.off[c + 1] - S.off[c];
        if (sz == 1) {
            res.order.push_back(S.verts[S.off[c]]);
        } else {
            vs.assign(S.verts.begin() + S.off[c], S.verts.begin() + S.off[c + 1]);
            const Local lg = induce_csr(g, edges, vs, scratch, ks);
            const Fas fas = sz <= std::min(thr, 22) ? fas_exact(lg) : fas_heuristic(lg);
            res.order.insert(res.order.end(), fas.order.begin(), fas.order.end());
            res.lagged_edges.insert(res.lagged_edges.end(), fas.lagged.begin(), fas.lagged.end());
            res.lagged_weight += fas.weight;
        }
        for (int k = coff[c]; k < coff[(size_t)c + 1]; ++k)
            if (--cin[ce[k].second] == 0) ready.push({S.verts[S.off[ce[k].second]], ce[k].second});
    }
    if ((int)res.order.size() != n) throw Error(HSW_ERR_LOGIC, "sweep_ordering: condensation was not acyclic");
    res.position.assign(n, -1);
    for (int k = 0; k < n; ++k) res.position[res.order[k]] = k;
    std::vector<char> lag(edges.size(), 0);
    for (int e : res.lagged_edges) lag[e] = 1;
    for (size_t e = 0; e < edges.size(); ++e) {
        const bool backward = res.position[edges[e].from] > res.position[edges[e].to];
        if (backward != (bool)lag[e]) throw Error(HSW_ERR_LOGIC, "sweep_ordering: retained edge set is inconsistent");
    }
    std::sort(res.lagged_edges.begin(), res.lagged_edges.end());
    return res;
}

// Small dense LU with partial pivoting (first max on ties); used for the
// siginvface weights so they are bit-identical to the oracle's.
static void lu_factor(std::vector<double>& a, std::vector<int>& perm, int n) {
    perm.resize(n);
    std::iota(perm.begin(), perm.end(), 0);
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = std::abs(a[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            const double v = std::abs(a[(size_t)i * n + k]);
            if (v > best) { best = v; p = i; }
        }
        if (p != k) {
            for (int j = 0; j < n; ++j) std::swap(a[(size_t)k * n + j], a[(size_t)p * n + j]);
            std::swap(perm[k], perm[p]);
        }
        const double piv = a[(size_t)k * n + k];
        if (piv == 0.0) continue;
        for (int i = k + 1; i < n; ++i) {
            double& lik = a[(size_t)i * n + k];
            lik /= piv;
            const double l = lik;
            if (l == 0.0) continue;
            for (int j = k + 1; j < n; ++j) a[(size_t)i * n + j] -= l * a[(size_t)k * n + j];
        }
    }
}
static void lu_solve(const std::vector<double>& a, const std::vector<int>& perm, int n, const double* b, double* x) {
    std::vector<double> y(n);
    for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
    for (int i = 0; i < n; ++i) {
        double s = y[i];
        for (int j = 0; j < i; ++j) s -= a[(size_t)i * n + j] * y[j];
        y[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = y[i];
        for (int j = i + 1; j < n; ++j) s -= a[(size_t)i * n + j] * y[j];
        y[i] = s / a[(size_t)i * n + i];
    }
    for (int i = 0; i < n; ++i) x[i] = y[i];
}

// =================================================================== setup
struct Coupling { int face, down, up, down_face, up_face; };

// romberg.hpp:33-88: Romberg tableau over successive trapezoid halvings of [0,1] for a
// vector integrand f(t, out[nv]) sharing one sampling; converged when two successive
// diagonal entries agree to tol in the max norm, never before min_levels halvings.
// Coefficient-wise in the reference's order (its Eigen expressions are elementwise);
// returns the last diagonal entry and whether it converged.
template <typename F>
static bool romberg_integrate(F&& f, size_t nv, double tol, int max_levels, int min_levels,
                              std::vector<double>& out) {
    min_levels = std::min(min_levels, max_levels);
    auto finite = [&](const std::vector<double>& v) {
        for (double x : v)
            if (std::isnan(x)) throw Error(HSW_ERR_ASSEMBLY, "romberg: integrand returned NaN");
    };
    std::vector<double> f0(nv), f1(nv), trap(nv), sum(nv), fi(nv);
    f(0.0, f0.data());
    f(1.0, f1.data());
    finite(f0);
    finite(f1);
    for (size_t i = 0; i < nv; ++i) trap[i] = 0.5 * (f0[i] + f1[i]);
    std::vector<std::vector<double>> diag{trap}, row;
    bool conv = false;
    long n = 1;
    for (int k = 1; k <= max_levels; ++k) {
        const double h = 1.0 / (2.0 * n);
        f(h, sum.data());
        finite(sum);
        for (long i = 1; i < n; ++i) {
            f((2 * i + 1) * h, fi.data());
            finite(fi);
            for (size_t j = 0; j < nv; ++j) sum[j] += fi[j];
        }
        for (size_t j = 0; j < nv; ++j) trap[j] = 0.5 * trap[j] + h * sum[j];
        n *= 2;
        row.resize((size_t)k + 1);
        row[0] = trap;
        double pow4 = 1.0;
        for (int j = 1; j <= k; ++j) {
            pow4 *= 4.0;
            row[j].resize(nv);
            for (size_t i = 0; i < nv; ++i) row[j][i] = row[j - 1][i] + (row[j - 1][i] - diag[j - 1][i]) / (pow4 - 1.0);
        }
        double diff = 0.0;
        for (size_t i = 0; i < nv; ++i) diff = std::max(diff, std::abs(row[k][i] - diag[k - 1][i]));
        diag.swap(row);
        if (diff < tol && k >= min_levels) {
            conv = true;
            break;
        }
    }
    out = diag.back();
    return conv;
}

struct Setup {
    // inputs
    int dim = 2, p = 1, nb = 4, nfn = 2, nf = 4, nel = 0, nd = 0;
    Mesh mesh;
    TensorBasis basis;
    std::vector<double> ow, odir;  // nd, nd*3
    std::map<int, std::pair<double, double>> xs;
    int source_kind = 0;
    double source_params[8] = {0};
    double inflow = 0.0;
    int vol_pts = 0, face_pts = 0, weighting = 1, fas_thr = 10;
    // ordinate shard [ob, oe) of this handle (all ordinates unless a multi-GPU rank's block)
    int ob = 0, oe = 0;
    bool partial() const { return ob != 0 || oe != nd; }
    // FaceIntegration (assembly.hpp:33-40): Gauss (face_pts) or Romberg (2D)
    int face_rule = HSW_FACE_GAUSS;
    double rom_tol = 1e-10;
    int rom_max = 16, rom_min = 6;
    // Romberg face data per (ordinate, element, local face), computed at create and
    // uploaded: outflow block (own face nodes x own face nodes), incoming coupling block
    // (own face nodes x own face-node order of the upwind traces, as the kernels gather
    // them), boundary inflow moments, outflow-face mask
    std::vector<double> rom_ob, rom_ib, rom_bin;
    std::vector<uint8_t> rom_omask;
    std::vector<int> rom_unconverged;   // per ordinate (TransportOperator::PerOrdinate, assembly.hpp:349)
    // quadrature
    Rule line_v, line_f;
    std::vector<std::array<double, 3>> vq_pts;
    std::vector<double> vq_w;
    std::vector<std::array<double, 2>> fq_pts;
    std::vector<double> fq_w;
    int nq = 0, nqf = 0;
    std::vector<std::vector<int>> fnodes;  // per face, element node ids of face nodes
    // per element
    std::vector<double> T;      // E*nb*nb*4
    std::vector<double> sig_t, sig_s, qvol;  // E, E, E*nb
    raw_vector<double> fgeom;  // E*nf*nqf*4 (normal, w*sj)
    raw_vector<double> fsj;    // E*nf*nqf   (sj)
    std::vector<int> fnbr;      // E*nf*4
    std::vector<int> bface_of;  // E*nf -> boundary face id or -1
    // face trace tables (bit-exact with the reference element-wise arithmetic)
    std::vector<double> trace;              // nqf * nfn: phi_a at own param point q
    std::vector<std::vector<double>> traceR;  // per orientation code: nqf * nfn at mapped point
    // max|LR|, max|RL| per (ordinate, interior face) computed on the device
    // (hsw_setup.cu, bit-identical to the host loop below); empty: host computes
    // coupling magnitudes from the device (hsw_create's CouplingFeed): acquire blocks until
    // ordinate d's [nfi][2] block has arrived and returns it, release hands its slot back
    std::function<const double*(int)> cmax_acquire;
    std::function<void(int)> cmax_release;
    std::vector<double> face_len;   // per interior face: sum_q w_q sj_q (assembly.hpp:231)
    // per ordinate
    std::vector<std::vector<Coupling>> couplings;
    std::vector<std::vector<double>> weights;
    std::vector<std::vector<char>> lagged;
    std::vector<Ordering> ords;
    std::vector<uint16_t> inflags;  // nd*E
    // worklists
    int num_levels = 0;
    std::vector<int> level_offsets;  // num_levels+1 into pairs_all
    raw_vector<int> pairs_all;      // e*nd + d, sorted (level, e, d)
    std::vector<std::vector<int>> dir_level_offsets;  // per d
    std::vector<int> pairs_dir;      // per d block of E pairs sorted by level
    std::vector<int> face_id_of;     // E*nf -> interior face id or -1
    std::vector<double> mass_t_cache;  // E*nb*nb for siginvface (exact oracle arithmetic)

    double xs_t(int region) const {
        auto it = xs.find(region);
        if (it == xs.end()) it = xs.find(0);
        if (it == xs.end())
            throw Error(HSW_ERR_RANGE, "cross sections: no entry for region " + std::to_string(region));
        return it->second.first;
    }
    double xs_s(int region) const {
        auto it = xs.find(region);
        if (it == xs.end()) it = xs.find(0);
        return it->second.second;
    }
    double source_at(const double* x) const {
        if (source_kind == HSW_SOURCE_CONSTANT) return source_params[0];
        double d2 = 0.0;
        for (int a = 0; a < dim; ++a) d2 += (x[a] - source_params[a]) * (x[a] - source_params[a]);
        return d2 < source_params[3] * source_params[3] ? source_params[4] : source_params[5];
    }

    void ingest(const hsw_problem_desc* D) {
        if (!D) throw Error(HSW_ERR_INVALID, "hsw_create: null descriptor");
        if (D->abi_version != HSW_ABI_VERSION) throw Error(HSW_ERR_INVALID, "hsw_create: ABI version mismatch");
        if (D->dim != 2 && D->dim != 3) throw Error(HSW_ERR_INVALID, "hsw_create: dim must be 2 or 3");
        if (D->geom_order < 1 || D->geom_order > 8)
            throw Error(HSW_ERR_INVALID, "hsw_create: geometry order out of range");
        if (D->basis_order < 1 || (D->dim == 3 && D->basis_order > 4) || D->basis_order > 6)
            throw Error(HSW_ERR_INVALID, "ReferenceBasis: order out of range for the B200 kernels");
        if (D->num_elements < 1 || D->num_ordinates < 1 || D->num_ordinates > 4096)
            throw Error(HSW_ERR_INVALID, "hsw_create: need elements and 1..4096 ordinates");
        dim = D->dim;
        p = D->basis_order;
        mesh.dim = dim;
        mesh.order = D->geom_order;
        mesh.geom = TensorBasis(dim, D->geom_order);
        mesh.npe = mesh.geom.nb;
        mesh.nel = nel = D->num_elements;
        mesh.pts.assign(D->points, D->points + (size_t)D->num_points * dim);
        mesh.enodes.assign(D->element_nodes, D->element_nodes + (size_t)nel * mesh.npe);
        mesh.region.assign(nel, 1);
        if (D->element_region) mesh.region.assign(D->element_region, D->element_region + nel);
        for (int b = 0; b < D->num_boundary_faces; ++b)
            mesh.bfaces.push_back({D->boundary_faces[3 * b], D->boundary_faces[3 * b + 1], D->boundary_faces[3 * b + 2]});
        nd = D->num_ordinates;
        ow.assign(D->ordinate_weight, D->ordinate_weight + nd);
        odir.assign(D->ordinate_dir, D->ordinate_dir + 3 * nd);
        for (int r = 0; r < D->num_regions; ++r) {
            if (!(D->sigma_t[r] >= D->sigma_s[r] && D->sigma_s[r] >= 0.0))
                throw Error(HSW_ERR_INVALID, "cross sections: need sigma_t >= sigma_s >= 0 (region " +
                                                 std::to_string(D->region_ids[r]) + ")");
            xs[D->region_ids[r]] = {D->sigma_t[r], D->sigma_s[r]};
        }
        source_kind = D->source_kind;
        std::memcpy(source_params, D->source_params, sizeof(source_params));
        inflow = D->inflow;
        vol_pts = D->volume_points > 0 ? D->volume_points : p + 2;
        face_pts = D->face_points > 0 ? D->face_points : p + 2;
        weighting = D->weighting;
        fas_thr = D->exact_fas_threshold > 0 ? D->exact_fas_threshold : 10;
        ob = 0;
        oe = nd;
        if (D->ordinate_end != 0) {
            if (D->ordinate_begin < 0 || D->ordinate_end > nd || D->ordinate_begin >= D->ordinate_end)
                throw Error(HSW_ERR_RANGE, "hsw_create: ordinate shard [" + std::to_string(D->ordinate_begin) + ", " +
                                               std::to_string(D->ordinate_end) + ") out of range");
            ob = D->ordinate_begin;
            oe = D->ordinate_end;
        }
        face_rule = D->face_rule;
        if (face_rule != HSW_FACE_GAUSS && face_rule != HSW_FACE_ROMBERG)
            throw Error(HSW_ERR_INVALID, "hsw_create: unknown face rule");
        if (face_rule == HSW_FACE_ROMBERG) {
            if (dim != 2) throw Error(HSW_ERR_INVALID, "romberg face rule: 2D meshes only (the reference is 2D)");
            rom_tol = D->romberg_tol > 0.0 ? D->romberg_tol : 1e-10;
            rom_max = D->romberg_max_levels > 0 ? D->romberg_max_levels : 16;
            rom_min = D->romberg_min_levels >= 0 ? D->romberg_min_levels : 6;
        }
        basis = TensorBasis(dim, p);
        nb = basis.nb;
        nf = nfaces_of(dim);
        for (int f = 0; f < nf; ++f) fnodes.push_back(face_nodes(dim, f, p));
        nfn = (int)fnodes[0].size();
        if (nfn > kMaxFaceNodes) throw Error(HSW_ERR_INVALID, "hsw_create: too many face nodes");
        // quadrature rules (quadrature.hpp:93-104 + face Gauss rule)
        line_v = gauss_legendre(vol_pts);
        line_f = gauss_legendre(face_pts);
        if (dim == 2) {
            for (int j = 0; j < vol_pts; ++j)
                for (int i = 0; i < vol_pts; ++i) {
                    vq_pts.push_back({line_v.x[i], line_v.x[j], 0.0});
                    vq_w.push_back(line_v.w[i] * line_v.w[j]);
                }
            for (int i = 0; i < face_pts; ++i) {
                fq_pts.push_back({line_f.x[i], 0.0});
                fq_w.push_back(line_f.w[i]);
            }
        } else {
            for (int k = 0; k < vol_pts; ++k)
                for (int j = 0; j < vol_pts; ++j)
                    for (int i = 0; i < vol_pts; ++i) {
                        vq_pts.push_back({line_v.x[i], line_v.x[j], line_v.x[k]});
                        vq_w.push_back(line_v.w[i] * line_v.w[j] * line_v.w[k]);
                    }
            for (int j = 0; j < face_pts; ++j)
                for (int i = 0; i < face_pts; ++i) {
                    fq_pts.push_back({line_f.x[i], line_f.x[j]});
                    fq_w.push_back(line_f.w[i] * line_f.w[j]);
                }
        }
        nq = (int)vq_w.size();
        nqf = (int)fq_w.size();
        if (nqf > kMaxFacePoints) throw Error(HSW_ERR_INVALID, "hsw_create: too many face points");
    }

    void build_mesh(int num_points, bool validate) {
        auto T0 = std::chrono::steady_clock::now();
        auto TT = [&](const char* n) { if (std::getenv("HSW_SETUP_TIMING")) { auto t = std::chrono::steady_clock::now(); std::fprintf(stderr, "  bm %s %.3f\n", n, std::chrono::duration<double>(t - T0).count()); T0 = t; } };
        mesh.check_connectivity(num_points);
        TT("check");
        mesh.build_faces();
        TT("build_faces");
        face_id_of.assign((size_t)nel * nf, -1);
        bface_of.assign((size_t)nel * nf, -1);
        fnbr.assign((size_t)nel * nf * 4, -1);
        for (size_t i = 0; i < mesh.ifaces.size(); ++i) {
            const auto& F = mesh.ifaces[i];
            face_id_of[(size_t)F.el * nf + F.fl] = (int)i;
            face_id_of[(size_t)F.er * nf + F.fr] = (int)i;
            int* a = &fnbr[((size_t)F.el * nf + F.fl) * 4];
            a[0] = F.er; a[1] = F.fr; a[2] = F.orient; a[3] = 0;
            int* b = &fnbr[((size_t)F.er * nf + F.fr) * 4];
            b[0] = F.el; b[1] = F.fl; b[2] = orient_inverse(dim, F.orient); b[3] = 1;
        }
        for (size_t i = 0; i < mesh.bfaces.size(); ++i) {
            const auto& B = mesh.bfaces[i];
            bface_of[(size_t)B.elem * nf + B.face] = (int)i;
            int* a = &fnbr[((size_t)B.elem * nf + B.face) * 4];
            a[0] = -1; a[1] = -1; a[2] = 0; a[3] = (int)i;
        }
        TT("fnbr");
        if (validate) {
            // mesh.hpp:219-228 det(J) > 0 on an (order+2)^dim lattice
            const int ns = mesh.order + 2;
            const int nz = dim == 3 ? ns : 1;
            const int nlat = ns * ns * nz;
            std::vector<double> gtab((size_t)mesh.npe * nlat * dim);   // [npe][nlat * dim]
            {
                std::vector<double> g((size_t)mesh.npe * dim);
                int q = 0;
                for (int k = 0; k < nz; ++k)
                    for (int j = 0; j < ns; ++j)
                        for (int i = 0; i < ns; ++i, ++q) {
                            const double xi[3] = {i / double(ns - 1), j / double(ns - 1),
                                                  dim == 3 ? k / double(ns - 1) : 0.0};
                            mesh.geom.gradients(xi, g.data());
                            for (int m = 0; m < mesh.npe; ++m)
                                for (int b = 0; b < dim; ++b)
                                    gtab[((size_t)m * nlat + q) * dim + b] = g[(size_t)m * dim + b];
                        }
            }
            std::atomic<int> bad{std::numeric_limits<int>::max()};
            parallel_for(nel, [&](int64_t e) {
                thread_local std::vector<double> jb;
                jb.resize((size_t)dim * nlat * dim);
                mesh.jacobians_batch((int)e, gtab.data(), nlat, jb.data());
                double J[9];
                for (int q = 0; q < nlat; ++q) {
                    mesh.unpack_jacobian(jb.data(), nlat, q, J);
                    if (mesh.det(J) <= 0.0) {
                        int cur = bad.load();
                        while ((int)e < cur && !bad.compare_exchange_weak(cur, (int)e)) {}
                        return;
                    }
                }
            });
            if (bad.load() != std::numeric_limits<int>::max())
                throw Error(HSW_ERR_MESH, "mesh: element " + std::to_string(bad.load()) + " has non-positive Jacobian");
            TT("detJ");
            // mesh.hpp:346-365 trace agreement on a 5-point (5x5) lattice
            std::atomic<int64_t> badf{std::numeric_limits<int64_t>::max()};
            // geometry basis values at the lattice points, tabulated per (face, lattice point)
            // on the left and per (face, orientation, lattice point) on the right
            const int nt = dim == 3 ? 5 : 1, nlp = 5 * nt, ncodes = dim == 2 ? 2 : 8;
            const size_t npe = (size_t)mesh.npe;
            std::vector<double> vl((size_t)nf * nlp * npe), vrt((size_t)nf * ncodes * nlp * npe);
            for (int f = 0; f < nf; ++f)
                for (int kt = 0; kt < nt; ++kt)
                    for (int k = 0; k < 5; ++k) {
                        const double s = k / 4.0, t = dim == 3 ? kt / 4.0 : 0.0;
                        double xi[3];
                        param_point(dim, f, s, t, xi);
                        mesh.geom.values(xi, &vl[((size_t)f * nlp + kt * 5 + k) * npe]);
                        for (int c = 0; c < ncodes; ++c) {
                            double so, to;
                            orient_param(dim, c, s, t, so, to);
                            param_point(dim, f, so, to, xi);
                            mesh.geom.values(xi, &vrt[(((size_t)f * ncodes + c) * nlp + kt * 5 + k) * npe]);
                        }
                    }
            parallel_for((int64_t)mesh.ifaces.size(), [&](int64_t i) {
                const auto& F = mesh.ifaces[i];
                const double tol = 1e-12 * mesh.diameter(F.el);
                for (int kt = 0; kt < nt; ++kt)
                    for (int k = 0; k < 5; ++k) {
                        double xl[3], xr[3];
                        mesh.map_tab(F.el, &vl[((size_t)F.fl * nlp + kt * 5 + k) * npe], xl);
                        mesh.map_tab(F.er, &vrt[(((size_t)F.fr * ncodes + F.orient) * nlp + kt * 5 + k) * npe], xr);
                        double d2 = 0.0;
                        for (int a = 0; a < dim; ++a) d2 += (xl[a] - xr[a]) * (xl[a] - xr[a]);
                        if (std::sqrt(d2) > tol) {   // the lowest failing face is reported
                            int64_t cur = badf.load();
                            while (i < cur && !badf.compare_exchange_weak(cur, i)) {}
                            return;
                        }
                    }
            });
            if (badf.load() != std::numeric_limits<int64_t>::max()) {
                const auto& F = mesh.ifaces[(size_t)badf.load()];
                throw Error(HSW_ERR_MESH, "mesh: interior face " + std::to_string(badf.load()) +
                                              " traces disagree between elements " + std::to_string(F.el) +
                                              " and " + std::to_string(F.er));
            }
            TT("traces");
        }
    }

    // assembly.hpp:58-93 + 143-163 + 278-300: per element M, G_k, volume source
    // basis / geometry tables at the volume points (element independent)
    std::vector<double> volU, volDU, volGV, volGG;
    void volume_tables() {
        volU.assign((size_t)nq * nb, 0.0);
        volDU.assign((size_t)nq * nb * dim, 0.0);
        volGV.assign((size_t)nq * mesh.npe, 0.0);
        volGG.assign((size_t)nq * mesh.npe * dim, 0.0);
        for (int q = 0; q < nq; ++q) {
            basis.values(vq_pts[q].data(), &volU[(size_t)q * nb]);
            basis.gradients(vq_pts[q].data(), &volDU[(size_t)q * nb * dim]);
            mesh.geom.values(vq_pts[q].data(), &volGV[(size_t)q * mesh.npe]);
            mesh.geom.gradients(vq_pts[q].data(), &volGG[(size_t)q * mesh.npe * dim]);
        }
    }

    // host_T = false: only the materials here; T and the source moments are
    // computed on the device (hsw_setup.cu) at hsw_create
    void element_tensors(bool host_T = true) {
        volume_tables();
        sig_t.resize(nel);
        sig_s.resize(nel);
        for (int e = 0; e < nel; ++e) {
            sig_t[e] = xs_t(mesh.region[e]);
            sig_s[e] = xs_s(mesh.region[e]);
        }
        if (!host_T) return;
        const std::vector<double>& U = volU;
        const std::vector<double>& DU = volDU;
        const std::vector<double>& GV = volGV;
        const std::vector<double>& GG = volGG;
        T.assign((size_t)nel * nb * nb * 4, 0.0);
        qvol.assign((size_t)nel * nb, 0.0);
        if (weighting == HSW_WEIGHT_SIGINVFACE) mass_t_cache.assign((size_t)nel * nb * nb, 0.0);
        parallel_for(nel, [&](int64_t e64) {
            const int e = (int)e64;
            const double st = xs_t(mesh.region[e]);
            sig_t[e] = st;
            sig_s[e] = xs_s(mesh.region[e]);
            std::vector<double> W((size_t)(dim + 1) * nq * nb);
            std::vector<double> wdet(nq);
            for (int q = 0; q < nq; ++q) {
                double J[9], K[9], x[3];
                const double det = mesh.jacobian_tab(e, &GG[(size_t)q * mesh.npe * dim], J);
                if (det <= 0.0 || !std::isfinite(det))
                    throw Error(HSW_ERR_ASSEMBLY, "assembly: singular Jacobian in element " + std::to_string(e));
                mesh.inverse(J, K);
                const double wd = vq_w[q] * det;
                wdet[q] = wd;
                const double* du = &DU[(size_t)q * nb * dim];
                for (int m = 0; m < nb; ++m) {
                    W[((size_t)0 * nq + q) * nb + m] = U[(size_t)q * nb + m] * wd;
                    for (int k = 0; k < dim; ++k) {
                        double v = 0.0;
                        for (int j = 0; j < dim; ++j) v += K[j * 3 + k] * du[m * dim + j];
                        W[((size_t)(k + 1) * nq + q) * nb + m] = v * wd;
                    }
                }
                mesh.map_tab(e, &GV[(size_t)q * mesh.npe], x);
                const double s = vq_w[q] * det * source_at(x);  // assembly.hpp:298
                for (int m = 0; m < nb; ++m) qvol[(size_t)e * nb + m] += s * U[(size_t)q * nb + m];
            }
            std::vector<double> acc((size_t)nb);
            double* Te = &T[(size_t)e * nb * nb * 4];
            for (int k = 0; k <= dim; ++k) {
                const double sign = k == 0 ? 1.0 : -1.0;
                for (int m = 0; m < nb; ++m) {
                    std::fill(acc.begin(), acc.end(), 0.0);
                    for (int q = 0; q < nq; ++q) {
                        const double w = W[((size_t)k * nq + q) * nb + m];
                        const double* u = &U[(size_t)q * nb];
                        for (int n = 0; n < nb; ++n) acc[n] += w * u[n];
                    }
                    for (int n = 0; n < nb; ++n) Te[((size_t)n * nb + m) * 4 + k] = sign * acc[n];
                }
            }
            if (!mass_t_cache.empty()) {  // exact reference M_t arithmetic (assembly.hpp:157-158)
                double* mt = &mass_t_cache[(size_t)e * nb * nb];
                for (int m = 0; m < nb; ++m)
                    for (int n = 0; n < nb; ++n) {
                        double s = 0.0;
                        for (int q = 0; q < nq; ++q)
                            s += U[(size_t)q * nb + m] * (wdet[q] * st) * U[(size_t)q * nb + n];
                        mt[(size_t)m * nb + n] = s;
                    }
            }
        });
    }

    // per element face geometry (own side) + trace tables
    void face_tables() {
        // per face: gradient tables at the face points, transposed to [npe][nqf * dim]
        std::vector<std::vector<double>> GGf(nf);
        {
            std::vector<double> g((size_t)mesh.npe * dim);
            for (int f = 0; f < nf; ++f) {
                GGf[f].resize((size_t)nqf * mesh.npe * dim);
                for (int q = 0; q < nqf; ++q) {
                    double xi[3];
                    param_point(dim, f, fq_pts[q][0], fq_pts[q][1], xi);
                    mesh.geom.gradients(xi, g.data());
                    for (int m = 0; m < mesh.npe; ++m)
                        for (int b = 0; b < dim; ++b)
                            GGf[f][((size_t)m * nqf + q) * dim + b] = g[(size_t)m * dim + b];
                }
            }
        }
        fgeom.resize((size_t)nel * nf * nqf * 4);   // every entry is written below
        fsj.resize((size_t)nel * nf * nqf);
        parallel_for(nel, [&](int64_t e64) {
            const int e = (int)e64;
            const double diam = mesh.diameter(e);
            thread_local std::vector<double> jb;
            jb.resize((size_t)dim * nqf * dim);
            for (int f = 0; f < nf; ++f) {
                mesh.jacobians_batch(e, GGf[f].data(), nqf, jb.data());
                for (int q = 0; q < nqf; ++q) {
                    double n[3], sj, J[9];
                    mesh.unpack_jacobian(jb.data(), nqf, q, J);
                    mesh.face_geometry_J(e, f, J, n, sj, diam);
                    double* g = &fgeom[(((size_t)e * nf + f) * nqf + q) * 4];
                    g[0] = n[0]; g[1] = n[1]; g[2] = n[2];
                    g[3] = fq_w[q] * sj;
                    fsj[((size_t)e * nf + f) * nqf + q] = sj;
                }
            }
        });
        // traces: full basis values at the face param point, face nodes picked
        // (assembly.hpp:112-116); identical for every face (one factor is exactly 1).
        std::vector<double> full(nb);
        trace.assign((size_t)nqf * nfn, 0.0);
        for (int q = 0; q < nqf; ++q) {
            double xi[3];
            param_point(dim, 0, fq_pts[q][0], fq_pts[q][1], xi);
            basis.values(xi, full.data());
            for (int a = 0; a < nfn; ++a) trace[(size_t)q * nfn + a] = full[fnodes[0][a]];
        }
        const int ncodes = dim == 2 ? 2 : 8;
        traceR.assign(ncodes, std::vector<double>((size_t)nqf * nfn, 0.0));
        for (int c = 0; c < ncodes; ++c)
            for (int q = 0; q < nqf; ++q) {
                double so, to, xi[3];
                orient_param(dim, c, fq_pts[q][0], fq_pts[q][1], so, to);
                param_point(dim, 0, so, to, xi);
                basis.values(xi, full.data());
                for (int a = 0; a < nfn; ++a) traceR[c][(size_t)q * nfn + a] = full[fnodes[0][a]];
            }
    }

    // face blocks integrated on the host for the kernels (2D): Romberg, or a Gauss rule with
    // other than the kernels' p + 2 points per face
    bool face_blocks() const { return face_rule == HSW_FACE_ROMBERG || (dim == 2 && face_pts != p + 2); }

    // assembly.hpp:185-241 (interior faces, Gauss rule) -> couplings + weights,
    // then sweepgraph.hpp:54-77 + 331-396, lag flags (solver.hpp:63-66) and levels.
    void ordinates() {
        couplings.assign(nd, {});
        weights.assign(nd, {});
        lagged.assign(nd, {});
        ords.assign(nd, {});
        inflags.assign((size_t)nd * nel, 0);
        const int nfi = (int)mesh.ifaces.size();
        // face blocks integrated here and handed to the kernels (2D): the Romberg rule, or a
        // Gauss rule other than the kernels' own p + 2 points (the reference's gauss_points)
        const bool romb = face_blocks();
        const bool use_romberg = face_rule == HSW_FACE_ROMBERG;
        const size_t nn = (size_t)nfn * nfn;
        if (romb) {
            rom_ob.assign((size_t)nd * nel * nf * nn, 0.0);
            rom_ib.assign((size_t)nd * nel * nf * nn, 0.0);
            rom_bin.assign((size_t)nd * nel * nf * nfn, 0.0);
            rom_omask.assign((size_t)nd * nel, 0);
            rom_unconverged.assign(nd, 0);
        }
        if (cmax_acquire) {
            face_len.assign(nfi, 0.0);
            parallel_for(nfi, [&](int64_t fi) {
                const IFace& F = mesh.ifaces[fi];
                const double* sjv = &fsj[((size_t)F.el * nf + F.fl) * nqf];
                double length = 0.0;
                for (int q = 0; q < nqf; ++q) length += fq_w[q] * sjv[q];
                face_len[fi] = length;
            });
        }
        std::atomic<long long> phase_acc[3];
        for (auto& a : phase_acc) a.store(0);
        std::atomic<long long>* phase_us = std::getenv("HSW_SETUP_TIMING") ? phase_acc : nullptr;
        parallel_for(oe - ob, [&](int64_t i64) {
            const auto t_begin = std::chrono::steady_clock::now();
            const int d = ob + (int)i64;
            const double* om = &odir[3 * d];
            std::vector<double> LR((size_t)nfn * nfn), RL((size_t)nfn * nfn), wp(nqf), wm(nqf);
            auto& cpl = couplings[d];
            auto& wts = weights[d];
            cpl.reserve((size_t)nfi + nfi / 8);   // about one coupling per interior face
            wts.reserve((size_t)nfi + nfi / 8);
            const double* cmax = cmax_acquire ? cmax_acquire(d) : nullptr;   // [nfi][2] of this ordinate
            // Romberg sampling of one face at parameter t (assembly.hpp:103-117): geometry of
            // the (left) element's face, its face-node traces, the neighbour's at t or 1 - t
            std::vector<double> gg((size_t)mesh.npe * dim), full(nb), ul(nfn), ur(nfn), packed, gtmp;
            // integrate_face (assembly.hpp:121-131): Romberg, or out += w_i f(t_i) over the Gauss rule
            auto integrate = [&](auto&& fn, size_t nv, std::vector<double>& out) -> bool {
                if (use_romberg) return romberg_integrate(fn, nv, rom_tol, rom_max, rom_min, out);
                out.assign(nv, 0.0);
                gtmp.resize(nv);
                for (int i = 0; i < face_pts; ++i) {
                    fn(line_f.x[i], gtmp.data());
                    for (size_t j = 0; j < nv; ++j) out[j] += line_f.w[i] * gtmp[j];
                }
                return true;
            };
            auto sample = [&](int e, int f, double t, double& on, double& sj, double* u) {
                double xi[3], n[3];
                param_point(dim, f, t, 0.0, xi);
                mesh.geom.gradients(xi, gg.data());
                mesh.face_geometry_tab(e, f, gg.data(), n, sj);
                on = om[0] * n[0] + om[1] * n[1];
                basis.values(xi, full.data());
                for (int a = 0; a < nfn; ++a) u[a] = full[fnodes[f][a]];
            };
            auto trace_at = [&](int f, double s0, double* u) {
                double xi[3];
                param_point(dim, f, s0, 0.0, xi);
                basis.values(xi, full.data());
                for (int a = 0; a < nfn; ++a) u[a] = full[fnodes[f][a]];
            };
            // incoming block of (downwind element e, face f): columns in e's face-node
            // order of the gathered upwind traces (kernel: neighbour node P - a if reversed)
            auto put_in = [&](int e, int f, const double* blk) {
                const int code = fnbr[((size_t)e * nf + f) * 4 + 2];
                double* dst = &rom_ib[(((size_t)d * nel + e) * nf + f) * nn];
                for (int a = 0; a < nfn; ++a)
                    for (int aa = 0; aa < nfn; ++aa) dst[(size_t)a * nfn + aa] = blk[(size_t)a * nfn + (code ? p - aa : aa)];
            };
            auto put_out = [&](int e, int f, const double* blk) {
                double* dst = &rom_ob[(((size_t)d * nel + e) * nf + f) * nn];
                bool nz = false;
                for (size_t k = 0; k < nn; ++k) {
                    dst[k] = blk[k];
                    nz |= blk[k] != 0.0;
                }
                if (nz) rom_omask[(size_t)d * nel + e] |= (uint8_t)(1u << f);
            };
            for (int fi = 0; fi < nfi; ++fi) {
                const IFace& F = mesh.ifaces[fi];
                if (romb) {   // assembly.hpp:195-241 with FaceIntegration::Rule::romberg
                    auto integrand = [&](double t, double* v) {
                        double on, sj, so, to;
                        sample(F.el, F.fl, t, on, sj, ul.data());
                        orient_param(dim, F.orient, t, 0.0, so, to);
                        trace_at(F.fr, so, ur.data());
                        const double wplus = 0.5 * (on + std::abs(on));
                        const double wminus = 0.5 * (std::abs(on) - on);
                        size_t k = 0;
                        for (int m = 0; m < nfn; ++m)
                            for (int n = 0; n < nfn; ++n) v[k++] = wplus * ul[m] * ul[n] * sj;
                        for (int m = 0; m < nfn; ++m)
                            for (int n = 0; n < nfn; ++n) v[k++] = wminus * ur[m] * ur[n] * sj;
                        for (int m = 0; m < nfn; ++m)
                            for (int n = 0; n < nfn; ++n) v[k++] = wminus * ul[m] * ur[n] * sj;
                        for (int m = 0; m < nfn; ++m)
                            for (int n = 0; n < nfn; ++n) v[k++] = wplus * ur[m] * ul[n] * sj;
                        v[k] = sj;
                    };
                    if (!integrate(integrand, 4 * nn + 1, packed)) rom_unconverged[d]++;
                    const double length = packed[4 * nn];
                    const double eps = 1e-12 * length;
                    put_out(F.el, F.fl, &packed[0]);
                    put_out(F.er, F.fr, &packed[nn]);
                    std::copy(packed.begin() + 2 * nn, packed.begin() + 3 * nn, LR.begin());
                    std::copy(packed.begin() + 3 * nn, packed.begin() + 4 * nn, RL.begin());
                    double mlr = 0.0, mrl = 0.0;
                    for (size_t k = 0; k < nn; ++k) {
                        mlr = std::max(mlr, std::abs(LR[k]));
                        mrl = std::max(mrl, std::abs(RL[k]));
                    }
                    if (mlr > eps) {
                        cpl.push_back({fi, F.el, F.er, F.fl, F.fr});
                        wts.push_back(weight_of(mlr, F.el, F.fl, LR, false));
                        put_in(F.el, F.fl, LR.data());
                    }
                    if (mrl > eps) {
                        cpl.push_back({fi, F.er, F.el, F.fr, F.fl});
                        wts.push_back(weight_of(mrl, F.er, F.fr, RL, false));
                        put_in(F.er, F.fr, RL.data());
                    }
                    continue;
                }
                const double* geo = &fgeom[(((size_t)F.el * nf + F.fl) * nqf) * 4];
                const double* sjv = &fsj[((size_t)F.el * nf + F.fl) * nqf];
                if (cmax) {   // magnitudes from the device; the face length from the shared table
                    const double eps = 1e-12 * face_len[fi];
                    const double mlr = cmax[(size_t)fi * 2], mrl = cmax[(size_t)fi * 2 + 1];
                    if (mlr > eps) {
                        cpl.push_back({fi, F.el, F.er, F.fl, F.fr});
                        wts.push_back(weight_of(mlr, F.el, F.fl, LR, false));
                    }
                    if (mrl > eps) {
                        cpl.push_back({fi, F.er, F.el, F.fr, F.fl});
                        wts.push_back(weight_of(mrl, F.er, F.fr, RL, false));
                    }
                    continue;
                }
                std::fill(LR.begin(), LR.end(), 0.0);
                std::fill(RL.begin(), RL.end(), 0.0);
                double length = 0.0;
                const double* uR0 = traceR[F.orient].data();
                for (int q = 0; q < nqf; ++q) {
                    double on = 0.0;
                    for (int k = 0; k < dim; ++k) on += om[k] * geo[q * 4 + k];
                    const double wplus = 0.5 * (on + std::abs(on));
                    const double wminus = 0.5 * (std::abs(on) - on);
                    const double sj = sjv[q], w = fq_w[q];
                    const double* ul = &trace[(size_t)q * nfn];
                    const double* ur = &uR0[(size_t)q * nfn];
                    if (wminus != 0.0)
                        for (int m = 0; m < nfn; ++m) {
                            const double c = wminus * ul[m];
                            double* row = &LR[(size_t)m * nfn];
                            for (int n = 0; n < nfn; ++n) row[n] += w * (c * ur[n] * sj);
                        }
                    if (wplus != 0.0)
                        for (int m = 0; m < nfn; ++m) {
                            const double c = wplus * ur[m];
                            double* row = &RL[(size_t)m * nfn];
                            for (int n = 0; n < nfn; ++n) row[n] += w * (c * ul[n] * sj);
                        }
                    length += w * sj;
                }
                const double eps = 1e-12 * length;
                double mlr = 0.0, mrl = 0.0;
                for (size_t k = 0; k < LR.size(); ++k) {
                    mlr = std::max(mlr, std::abs(LR[k]));
                    mrl = std::max(mrl, std::abs(RL[k]));
                }
                if (mlr > eps) {
                    cpl.push_back({fi, F.el, F.er, F.fl, F.fr});
                    wts.push_back(weight_of(mlr, F.el, F.fl, LR, false));
                }
                if (mrl > eps) {
                    cpl.push_back({fi, F.er, F.el, F.fr, F.fl});
                    wts.push_back(weight_of(mrl, F.er, F.fr, RL, false));
                }
            }
            if (romb) {   // boundary outflow (assembly.hpp:244-266), then the inflow moments (:302-313)
                std::vector<double> mom;
                for (const auto& B : mesh.bfaces) {
                    auto outflow = [&](double t, double* v) {
                        double on, sj;
                        sample(B.elem, B.face, t, on, sj, ul.data());
                        const double wplus = 0.5 * (on + std::abs(on));
                        size_t k = 0;
                        for (int m = 0; m < nfn; ++m)
                            for (int n = 0; n < nfn; ++n) v[k++] = wplus * ul[m] * ul[n] * sj;
                    };
                    if (!integrate(outflow, nn, packed)) rom_unconverged[d]++;
                    put_out(B.elem, B.face, packed.data());
                }
                if (inflow != 0.0)
                    for (const auto& B : mesh.bfaces) {
                        auto incident = [&](double t, double* v) {
                            double on, sj;
                            sample(B.elem, B.face, t, on, sj, ul.data());
                            const double wminus = 0.5 * (std::abs(on) - on);
                            const double c = wminus * inflow * sj;
                            for (int m = 0; m < nfn; ++m) v[m] = c * ul[m];
                        };
                        integrate(incident, (size_t)nfn, mom);
                        double* dst = &rom_bin[(((size_t)d * nel + B.elem) * nf + B.face) * nfn];
                        for (int m = 0; m < nfn; ++m) dst[m] += mom[m];
                    }
            }
            if (cmax) cmax_release(d);
            const auto t_faces = std::chrono::steady_clock::now();
            std::vector<Edge> edges(cpl.size());
            for (size_t c = 0; c < cpl.size(); ++c) edges[c] = {cpl[c].up, cpl[c].down, wts[c]};
            ords[d] = sweep_ordering(nel, edges, fas_thr);
            const auto t_order = std::chrono::steady_clock::now();
            Ordering& o = ords[d];
            auto& lg = lagged[d];
            lg.assign(cpl.size(), 0);
            std::vector<int> in_off((size_t)nel + 1, 0), in_c(cpl.size());   // incoming couplings, CSR
            for (size_t c = 0; c < cpl.size(); ++c) {
                lg[c] = o.position[cpl[c].up] > o.position[cpl[c].down];
                in_off[(size_t)cpl[c].down + 1]++;
                uint16_t& fl = inflags[(size_t)d * nel + cpl[c].down];
                fl |= (uint16_t)(1u << (2 * cpl[c].down_face));
                if (lg[c]) fl |= (uint16_t)(1u << (2 * cpl[c].down_face + 1));
            }
            for (int e = 0; e < nel; ++e) in_off[(size_t)e + 1] += in_off[e];
            {
                std::vector<int> fill(in_off.begin(), in_off.end() - 1);
                for (size_t c = 0; c < cpl.size(); ++c) in_c[fill[cpl[c].down]++] = (int)c;
            }
            o.level.assign(nel, 0);
            for (int e : o.order) {
                int lv = 0;
                for (int j = in_off[e]; j < in_off[(size_t)e + 1]; ++j) {
                    const int c = in_c[j];
                    if (!lg[c]) lv = std::max(lv, o.level[cpl[c].up] + 1);
                }
                o.level[e] = lv;
            }
            if (phase_us) {   // HSW_SETUP_TIMING: thread-seconds per part, summed over the ordinates
                const auto t_end = std::chrono::steady_clock::now();
                auto us = [](auto a, auto b) { return (long long)std::chrono::duration_cast<std::chrono::microseconds>(b - a).count(); };
                phase_us[0] += us(t_begin, t_faces);
                phase_us[1] += us(t_faces, t_order);
                phase_us[2] += us(t_order, t_end);
            }
        });
        if (phase_us)
            std::fprintf(stderr, "  ordinates (thread-seconds): couplings %.3f, sweep_ordering %.3f, lag flags + levels %.3f\n",
                         phase_us[0].load() * 1e-6, phase_us[1].load() * 1e-6, phase_us[2].load() * 1e-6);
    }

    // face -> max|block|; siginvface -> max|M_t^{-1} block| (sweepgraph.hpp:60-72)
    double weight_of(double maxabs, int down, int down_face, const std::vector<double>& blk, bool) const {
        if (weighting == HSW_WEIGHT_UNITY) return 1.0;
        if (weighting == HSW_WEIGHT_FACE) return maxabs;
        std::vector<double> a(mass_t_cache.begin() + (size_t)down * nb * nb,
                              mass_t_cache.begin() + (size_t)(down + 1) * nb * nb);
        std::vector<int> perm;
        lu_factor(a, perm, nb);
        double w = 0.0;
        std::vector<double> col(nb), x(nb);
        for (int n = 0; n < nfn; ++n) {
            std::fill(col.begin(), col.end(), 0.0);
            for (int m = 0; m < nfn; ++m) col[fnodes[down_face][m]] = -blk[(size_t)m * nfn + n];
            lu_solve(a, perm, nb, col.data(), x.data());
            for (int i = 0; i < nb; ++i) {
                if (!std::isfinite(x[i]))
                    throw Error(HSW_ERR_ASSEMBLY, "sig_inv_face weighting: singular mass matrix on element " +
                                                      std::to_string(down));
                w = std::max(w, std::abs(x[i]));
            }
        }
        return w;
    }

    void worklists() {   // over the handle's ordinate shard [ob, oe)
        const int nds = oe - ob;
        // per-ordinate worklists (level, element) and level counts, one ordinate per task
        pairs_dir.resize((size_t)nel * nd);
        if (nds < nd) std::fill(pairs_dir.begin(), pairs_dir.end(), 0);   // rows outside the shard
        dir_level_offsets.assign(nd, {});
        parallel_for(nds, [&](int64_t i) {
            const int d = ob + (int)i;
            const int* lev = ords[d].level.data();
            int ml = 0;
            for (int e = 0; e < nel; ++e) ml = std::max(ml, lev[e]);
            std::vector<int> c(ml + 2, 0);
            for (int e = 0; e < nel; ++e) c[lev[e] + 1]++;
            for (int l = 0; l <= ml; ++l) c[l + 1] += c[l];
            std::vector<int> fl(c.begin(), c.end() - 1);
            int* base = &pairs_dir[(size_t)d * nel];
            for (int e = 0; e < nel; ++e) base[fl[lev[e]]++] = e * nd + d;
            dir_level_offsets[d] = std::move(c);
        });
        int maxl = 0;
        for (int d = ob; d < oe; ++d) maxl = std::max(maxl, (int)dir_level_offsets[d].size() - 2);
        num_levels = maxl + 1;
        // shard worklist sorted by (level, element, ordinate): element chunks count their
        // pairs per level, a prefix over (level, chunk) gives every chunk its write offsets
        const int nchunk = (int)std::max<int64_t>(1, std::min<int64_t>(nel, 4 * (int64_t)host_workers()));
        auto chunk_begin = [&](int k) { return (int)((int64_t)nel * k / nchunk); };
        std::vector<int> cnt((size_t)nchunk * num_levels, 0);
        parallel_for(nchunk, [&](int64_t k) {
            int* c = &cnt[(size_t)k * num_levels];
            for (int d = ob; d < oe; ++d) {
                const int* lev = ords[d].level.data();
                for (int e = chunk_begin((int)k); e < chunk_begin((int)k + 1); ++e) c[lev[e]]++;
            }
        });
        level_offsets.assign(num_levels + 1, 0);
        {
            int run = 0;
            for (int l = 0; l < num_levels; ++l) {
                level_offsets[l] = run;
                for (int k = 0; k < nchunk; ++k) {
                    const int c = cnt[(size_t)k * num_levels + l];
                    cnt[(size_t)k * num_levels + l] = run;
                    run += c;
                }
            }
            level_offsets[num_levels] = run;
        }
        pairs_all.resize((size_t)nel * nds);
        parallel_for(nchunk, [&](int64_t k) {
            int* fill = &cnt[(size_t)k * num_levels];
            for (int e = chunk_begin((int)k); e < chunk_begin((int)k + 1); ++e)
                for (int d = ob; d < oe; ++d) pairs_all[fill[ords[d].level[e]]++] = e * nd + d;
        });
    }
};

}  // namespace hsw

// ===================================================================== C ABI
using namespace hsw;

struct hsw_handle {
    // calls on one handle are serialised (the reference's const sweep/local_solve are
    // called concurrently for distinct ordinates, solver.hpp:145-149) and run on the
    // handle's device whatever device is current on the calling thread
    std::recursive_mutex mu;
    Setup S;
    int device = 0;
    cudaStream_t stream = nullptr;
    DevProblem P{};
    // device buffers
    double *d_rom_ob = nullptr, *d_rom_ib = nullptr, *d_rom_bin = nullptr;
    int* d_bfaces = nullptr;   // (elem, face, attr) per boundary face, for the device balance
    size_t psi_offset = 0;     // d_psiA / d_psiB point psi_offset doubles before their allocations (shards)
    unsigned char* d_rom_omask = nullptr;
    double *d_T = nullptr, *d_sig_t = nullptr, *d_sig_s = nullptr, *d_qvol = nullptr, *d_fgeom = nullptr;
    double* d_bscale = nullptr;
    int* d_fnbr = nullptr;
    uint16_t* d_inflags = nullptr;
    double *d_omega = nullptr, *d_weight = nullptr;
    double *d_psiA = nullptr, *d_psiB = nullptr, *d_phi = nullptr, *d_phi_old = nullptr, *d_src = nullptr;
    double *d_scratch = nullptr, *d_out = nullptr, *d_vec = nullptr, *d_vec2 = nullptr;
    int *d_pairs_all = nullptr, *d_pairs_dir = nullptr, *d_pair1 = nullptr;
    unsigned long long* d_prof = nullptr;
    int *d_tab_fnode = nullptr, *d_tab_fidx = nullptr, *d_tab_nmask = nullptr;
    double *d_tab_trace = nullptr, *d_tab_line = nullptr;
    unsigned long long* d_err = nullptr;   // [2]: singular block | static pivoting refused
    // Static-pivot tile LU (the production sweep kernel) refused a block of this problem:
    // every later sweep uses the pivoted Gauss-Jordan kernel (sticky)
    bool need_pivot = false;
    int64_t pivot_fallbacks = 0;
    double* h_out = nullptr;  // pinned
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int64_t zero_pair = -1;
    int64_t last_launches = 0;
    double last_kernel_ms = 0.0;
    size_t N = 0;
    // direction-sharded SI: cached worklists of ordinate blocks [d0, d1)
    struct RangeList {
        int* d_pairs = nullptr;
        std::vector<int> offsets;   // num_levels + 1
    };
    std::map<std::pair<int, int>, RangeList> ranges;
    // captured all-ordinate level sequences (CUDA graphs)
    struct GraphKey {
        const double* psi_old;
        const double* psi_new;
        int flags;
        int64_t zero_pair;
        int kernel;
        bool operator<(const GraphKey& o) const {
            return std::tie(psi_old, psi_new, flags, zero_pair, kernel) <
                   std::tie(o.psi_old, o.psi_new, o.flags, o.zero_pair, o.kernel);
        }
    };
    struct GraphEntry {
        cudaGraphExec_t exec;
        int64_t launches;
    };
    std::map<GraphKey, GraphEntry> graphs;
    bool levels_configured = false;
    // dataflow schedule: per-pair completion flags (== epoch of the current sweep)
    unsigned* d_done = nullptr;
    unsigned epoch = 0;
    // host-pointer all-ordinate sweep: copy streams and per-block events
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_sw;
    cudaEvent_t ev_cp[2] = {nullptr, nullptr};
    // pageable caller buffers: pinned staging ring (2 in + 2 out chunks), one event per chunk
    char* stage = nullptr;
    size_t stage_chunk = 0;
    cudaEvent_t ev_stage[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {
// fn on a helper thread; join() rethrows what it threw (the destructor only joins)
struct Async {
    std::exception_ptr err;
    std::thread t;
    template <class F>
    explicit Async(F&& f) : t([this, fn = std::forward<F>(f)]() mutable {
        try {
            fn();
        } catch (...) {
            err = std::current_exception();
        }
    }) {}
    void join() {
        if (t.joinable()) t.join();
        if (err) {
            std::exception_ptr e = err;
            err = nullptr;
            std::rethrow_exception(e);
        }
    }
    ~Async() {
        if (t.joinable()) t.join();
    }
};
thread_local std::string g_last_error;
thread_local int g_create_zero_e = -1, g_create_zero_d = -1;

// Lock the handle and make its device current for the call (restored on exit).
struct HandleScope {
    std::unique_lock<std::recursive_mutex> lk;
    int prev = -1;
    bool switched = false;
    explicit HandleScope(hsw_handle* h) : lk(h->mu) {
        if (h->stream && cudaGetDevice(&prev) == cudaSuccess && prev != h->device)
            switched = cudaSetDevice(h->device) == cudaSuccess;
    }
    ~HandleScope() {
        if (switched) cudaSetDevice(prev);
    }
};

int fail(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

#define CUDA_OK(x)                                                                           \
    do {                                                                                     \
        cudaError_t _e = (x);                                                                \
        if (_e != cudaSuccess)                                                               \
            throw hsw::Error(HSW_ERR_CUDA, std::string("CUDA: ") + cudaGetErrorString(_e) + \
                                               " at " #x);                                   \
    } while (0)

template <typename T, typename A>
T* dev_upload(const std::vector<T, A>& v) {
    T* p = nullptr;
    if (v.empty()) return nullptr;
    CUDA_OK(cudaMalloc(&p, v.size() * sizeof(T)));
    CUDA_OK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
}

void free_handle(hsw_handle* h) {
    if (!h) return;
    if (h->d_psiA) h->d_psiA += h->psi_offset;
    if (h->d_psiB) h->d_psiB += h->psi_offset;
    void* bufs[] = {h->d_T, h->d_sig_t, h->d_bscale, h->d_sig_s, h->d_qvol, h->d_fgeom, h->d_fnbr, h->d_inflags,
                    h->d_omega, h->d_weight, h->d_psiA, h->d_psiB, h->d_phi, h->d_phi_old, h->d_src,
                    h->d_scratch, h->d_out, h->d_vec, h->d_vec2, h->d_pairs_all, h->d_pairs_dir, h->d_pair1,
                    h->d_err, h->d_prof, h->d_tab_fnode, h->d_tab_fidx, h->d_tab_nmask, h->d_tab_trace, h->d_tab_line,
                    h->d_rom_ob, h->d_rom_ib, h->d_rom_bin, h->d_rom_omask, h->d_bfaces};
    for (void* b : bufs)
        if (b) cudaFree(b);
    for (auto& kv : h->ranges)
        if (kv.second.d_pairs) cudaFree(kv.second.d_pairs);
    for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second.exec);
    if (h->d_done) cudaFree(h->d_done);
    for (auto e : h->ev_in) cudaEventDestroy(e);
    for (auto e : h->ev_sw) cudaEventDestroy(e);
    for (auto e : h->ev_cp)
        if (e) cudaEventDestroy(e);
    if (h->copy_in) cudaStreamDestroy(h->copy_in);
    if (h->copy_out) cudaStreamDestroy(h->copy_out);
    if (h->stage) cudaFreeHost(h->stage);
    for (auto e : h->ev_stage)
        if (e) cudaEventDestroy(e);
    if (h->h_out) cudaFreeHost(h->h_out);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

// shard handles (hsw_problem_desc::ordinate_begin/end): ordinates outside the shard and
// calls that need every ordinate are range errors
void need_in_shard(const hsw_handle* h, int d, const char* what) {
    if (d >= 0 && (d < h->S.ob || d >= h->S.oe))
        throw hsw::Error(HSW_ERR_RANGE, std::string(what) + ": ordinate " + std::to_string(d) +
                                            " is not in this handle's shard [" + std::to_string(h->S.ob) + ", " +
                                            std::to_string(h->S.oe) + ")");
}
void need_all_ordinates(const hsw_handle* h, const char* what) {
    if (h->S.partial())
        throw hsw::Error(HSW_ERR_RANGE, std::string(what) + ": needs every ordinate; this handle holds the shard [" +
                                            std::to_string(h->S.ob) + ", " + std::to_string(h->S.oe) +
                                            ") (use the hsw_shard_* primitives)");
}

void need_device(const hsw_handle* h) {
    if (!h || !h->stream)
        throw hsw::Error(HSW_ERR_CUDA, "handle has no device state (created with device < 0); "
                                       "the B200 sweep has no CPU fallback");
}

// Thrown by check_err when the static-pivot kernel refused a block: guarded() redoes the
// API call once, now with the pivoted kernel (hsw_handle::need_pivot).
struct RetryPivot {};

// Raise the first singular (element, ordinate) recorded by the kernels.
void check_err(hsw_handle* h) {
    if (h->d_done) {   // dataflow stall (see dmma1 kernel): results are invalid, fail loudly
        unsigned stall = 0;
        CUDA_OK(cudaMemcpyAsync(&stall, h->d_done + (size_t)h->S.nel * h->S.nd, sizeof(stall), cudaMemcpyDeviceToHost,
                                h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        if (stall) {
            CUDA_OK(cudaMemsetAsync(h->d_done + (size_t)h->S.nel * h->S.nd, 0, sizeof(unsigned), h->stream));
            throw hsw::Error(HSW_ERR_CUDA, "dataflow sweep stalled: the persistent CTAs were not all resident "
                                           "(other work on the GPU?); set HSW_DATAFLOW=0");
        }
    }
    unsigned long long keys[2] = {0, 0};
    CUDA_OK(cudaMemcpyAsync(keys, h->d_err, sizeof(keys), cudaMemcpyDeviceToHost, h->stream));
    CUDA_OK(cudaStreamSynchronize(h->stream));
    if (keys[1] != ~0ull) {
        // the static-pivot kernel refused a block (tiny pivot or large inverse tile): its results
        // are discarded, the handle switches to the pivoted kernel and the caller redoes the call
        const unsigned long long reset[2] = {~0ull, ~0ull};
        CUDA_OK(cudaMemcpy(h->d_err, reset, sizeof(reset), cudaMemcpyHostToDevice));
        h->need_pivot = true;
        ++h->pivot_fallbacks;
        throw RetryPivot{};
    }
    const unsigned long long key = keys[0];
    if (key != ~0ull) {
        const int nd = h->S.nd;
        const long long pr = (long long)(key & 0xffffffffffull);
        const int e = (int)(pr / nd), d = (int)(pr % nd);
        const unsigned long long reset = ~0ull;
        CUDA_OK(cudaMemcpy(h->d_err, &reset, sizeof(reset), cudaMemcpyHostToDevice));
        throw hsw::Error(HSW_ERR_SOLVER, "local streaming+collision block is singular (element " +
                                             std::to_string(e) + ", ordinate " + std::to_string(d) + ")");
    }
}

// Kernel selection: the one-warp DMMA kernel (hsw_dmma1.cu) for every shape it
// instantiates (2D Q2/Q3, 3D Q2-Q4: all five configs); the W-warps-per-pair DMMA
// kernel (hsw_dmma.cu) for the other orders.  HSW_KERNEL=dmma forces the latter.
// HSW_D2=0 turns the two-warp kernel (hsw_dmma2.cu) off where it is instantiated.
int kernel_choice_for(int dim, int p) {
    static const bool force_dmma = [] {
        const char* k = std::getenv("HSW_KERNEL");
        return k && std::string(k) == "dmma";
    }();
    static const int d2 = [] {
        const char* e = std::getenv("HSW_D2");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    // the two-warp kernel by default where it is instantiated (3D Q4: C5 1.54 -> 1.31 s)
    if (!force_dmma && d2 != 0 && dev_dmma2_supported(dim, p)) return 4;
    return (!force_dmma && dev_dmma1_supported(dim, p)) ? 3 : 2;
}

// Static-pivot tile LU: the production sweep kernels unless a block of this problem was refused
// (need_pivot) or HSW_SP=0.  hsw_dmma1.cu (one warp per pair) for every shape but 3D Q4, where the
// two-warp kernel's left-looking static-pivot form runs (hsw_dmma2.cu); HSW_SP_Q4=1 selects the
// one-warp kernel there, HSW_SP_Q4=0 the pivoted two-warp kernel.
int sp_q4_env() {
    static const int q4 = [] {
        const char* e = std::getenv("HSW_SP_Q4");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return q4;
}
bool static_pivot(const hsw_handle* h) {
    static const int env = [] {
        const char* e = std::getenv("HSW_SP");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    if (env == 0 || h->need_pivot) return false;
    const int kc = kernel_choice_for(h->S.dim, h->S.p);
    if (kc == 4) return sp_q4_env() != 0;
    return kc == 3;
}
// 6: dmma2 static-pivot, 5: dmma1 static-pivot, 4: dmma2, 3: dmma1 pivoted, 2: dmma
int kernel_choice(const hsw_handle* h) {
    const int kc = kernel_choice_for(h->S.dim, h->S.p);
    if (!static_pivot(h)) return kc;
    // HSW_D2_Q3=1: the two-warp static-pivot kernel at 3D Q3 too (eight pairs per SM)
    static const bool d2q3 = [] { const char* e = std::getenv("HSW_D2_Q3"); return e && e[0] == '1'; }();
    if (d2q3 && h->S.dim == 3 && h->S.p == 3) return 6;
    return kc == 4 && sp_q4_env() != 1 ? 6 : 5;
}

void sweep_launch(hsw_handle* h, const double* psi_old, double* psi_new, const int* pairs, int n) {
    const int kc = kernel_choice(h);
    if (kc == 5)
        dev_dmma1_sweep(h->P, h->d_src, psi_old, psi_new, (int64_t)h->N, pairs, n, h->d_err, h->zero_pair, h->stream,
                        nullptr, 0, true);
    else if (kc == 4 || kc == 6)
        dev_dmma2_sweep(h->P, h->d_src, psi_old, psi_new, (int64_t)h->N, pairs, n, h->d_err, h->zero_pair, h->stream,
                        nullptr, 0, kc == 6);
    else if (kc == 3)
        dev_dmma1_sweep(h->P, h->d_src, psi_old, psi_new, (int64_t)h->N, pairs, n, h->d_err, h->zero_pair, h->stream);
    else
        dev_dmma_sweep(h->P, h->d_src, psi_old, psi_new, (int64_t)h->N, pairs, n, h->d_err, h->zero_pair, h->stream);
}

// All-ordinate sweep psi_old -> psi_new using the current h->d_src.
int64_t launch_all_levels(hsw_handle* h, const double* psi_old, double* psi_new) {
    const auto& off = h->S.level_offsets;
    int64_t launches = 0;
    for (int l = 0; l < h->S.num_levels; ++l) {
        const int n = off[l + 1] - off[l];
        if (n == 0) continue;
        sweep_launch(h, psi_old, psi_new, h->d_pairs_all + off[l], n);
        ++launches;
    }
    return launches;
}

bool graphs_enabled() {
    static const bool v = [] { const char* e = std::getenv("HSW_GRAPHS"); return !(e && e[0] == '0'); }();
    return v;
}

// Dataflow schedule (HSW_DATAFLOW=1, one-warp DMMA kernel): the whole worklist
// in one persistent launch; each pair waits for its retained upwind pairs'
// completion flags instead of a per-level barrier.
// Default: on for 3D (C3 -9 %, C4 -1.5 %), off for 2D (its 449 short levels are
// faster level by level from a CUDA graph).  HSW_DATAFLOW=0/1 overrides.
bool dataflow_enabled(const hsw_handle* h) {
    static const int env = [] {
        const char* e = std::getenv("HSW_DATAFLOW");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    if (kernel_choice(h) < 3) return false;
    return env >= 0 ? env == 1 : h->S.dim == 3;
}

unsigned next_epoch(hsw_handle* h) {
    // flags [nel * nd] + the stall flag + the pair-claim counter
    const size_t bytes = ((size_t)h->S.nel * h->S.nd + 2) * sizeof(unsigned);
    if (!h->d_done) {
        CUDA_OK(cudaMalloc(&h->d_done, bytes));
        CUDA_OK(cudaMemsetAsync(h->d_done, 0, bytes, h->stream));
        h->epoch = 0;
    }
    if (++h->epoch == 0u) {   // wrapped: clear the flags
        CUDA_OK(cudaMemsetAsync(h->d_done, 0, bytes, h->stream));
        h->epoch = 1;
    }
    return h->epoch;
}

void dataflow_sweep(hsw_handle* h, const double* psi_old, double* psi_new, const int* pairs, int n) {
    const unsigned ep = next_epoch(h);
    CUDA_OK(cudaMemsetAsync(h->d_done + (size_t)h->S.nel * h->S.nd + 1, 0, sizeof(unsigned), h->stream));
    const int kc = kernel_choice(h);
    if (kc == 4 || kc == 6)
        dev_dmma2_sweep(h->P, h->d_src, psi_old, psi_new, (int64_t)h->N, pairs, n, h->d_err, h->zero_pair, h->stream,
                        h->d_done, ep, kc == 6);
    else
        dev_dmma1_sweep(h->P, h->d_src, psi_old, psi_new, (int64_t)h->N, pairs, n, h->d_err, h->zero_pair, h->stream,
                        h->d_done, ep, kc == 5);
}

// The all-ordinate sweep is one launch per level (C2: 449 levels of ~24 us):
// after a first direct run (which configures every kernel), the level sequence
// is captured once per (psi_old, psi_new, kernel arguments) into a CUDA graph
// and replayed with a single launch.  HSW_GRAPHS=0 disables.
void run_all_levels(hsw_handle* h, const double* psi_old, double* psi_new, bool time_it) {
    if (time_it) CUDA_OK(cudaEventRecord(h->ev0, h->stream));
    if (dataflow_enabled(h)) {
        dataflow_sweep(h, psi_old, psi_new, h->d_pairs_all, (int)h->S.pairs_all.size());
        h->last_launches = 1;
        if (time_it) CUDA_OK(cudaEventRecord(h->ev1, h->stream));
        return;
    }
    const hsw_handle::GraphKey key{psi_old, psi_new, h->P.debug_flags, h->zero_pair, kernel_choice(h)};
    auto it = h->graphs.find(key);
    if (!graphs_enabled() || (it == h->graphs.end() && !h->levels_configured)) {
        h->last_launches = launch_all_levels(h, psi_old, psi_new);
        h->levels_configured = true;
    } else {
        if (it == h->graphs.end()) {
            cudaGraph_t g = nullptr;
            CUDA_OK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
            int64_t launches = 0;
            try {
                launches = launch_all_levels(h, psi_old, psi_new);
            } catch (...) {
                cudaStreamEndCapture(h->stream, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            CUDA_OK(cudaStreamEndCapture(h->stream, &g));
            cudaGraphExec_t ex = nullptr;
            CUDA_OK(cudaGraphInstantiate(&ex, g, 0));
            CUDA_OK(cudaGraphDestroy(g));
            it = h->graphs.emplace(key, hsw_handle::GraphEntry{ex, launches}).first;
        }
        CUDA_OK(cudaGraphLaunch(it->second.exec, h->stream));
        h->last_launches = it->second.launches;
    }
    if (time_it) CUDA_OK(cudaEventRecord(h->ev1, h->stream));
}

// Ordinate blocks of the pipelined host-pointer sweep: 4 when psi is large
// enough for PCIe time to matter (HSW_E2E_BLOCKS overrides; 1 disables).
int e2e_blocks_env() {
    static const int env = [] {
        const char* v = std::getenv("HSW_E2E_BLOCKS");
        return v ? std::atoi(v) : 0;
    }();
    return env;
}
// Relative block sizes of the default ramp, as cumulative 32nds (HSW_E2E_RAMP="1,4,12,24,30,32"
// overrides: an increasing list ending in 32; its length is the block count).
const std::vector<int>& e2e_ramp() {
    static const std::vector<int> v = [] {
        std::vector<int> r{0, 1, 4, 12, 24, 30, 32};
        if (const char* e = std::getenv("HSW_E2E_RAMP")) {
            std::vector<int> u{0};
            for (const char* p = e; *p;) {
                char* end = nullptr;
                const long x = std::strtol(p, &end, 10);
                if (end == p) break;
                u.push_back((int)x);
                p = *end == ',' ? end + 1 : end;
            }
            bool ok = u.size() >= 2 && u.back() == 32;
            for (size_t i = 1; i < u.size(); ++i) ok = ok && u[i] > u[i - 1];
            if (ok) r = u;
        }
        return r;
    }();
    return v;
}
int e2e_blocks(const hsw_handle* h, int nr) {   // nr: ordinates of the swept range
    const int env = e2e_blocks_env();
    int b = env > 0 ? env : ((double)h->N * nr * sizeof(double) >= 64e6 ? (int)e2e_ramp().size() - 1 : 1);
    return std::max(1, std::min(b, nr));
}
// First ordinate of block b (of nblk).  Default (no HSW_E2E_BLOCKS, >= 32 ordinates):
// a ramp of relative sizes 1:3:8:12:6:2, so that only a small first block's H2D and a
// small last block's D2H stay exposed while every other transfer hides behind a
// larger neighbouring sweep.
int e2e_block_start(int b, int nblk, int nr) {   // offset within a range of nr ordinates
    const std::vector<int>& ramp = e2e_ramp();
    if (e2e_blocks_env() > 0 || nblk != (int)ramp.size() - 1 || nr < 32) return (int)((int64_t)b * nr / nblk);
    return (int)((int64_t)ramp[b] * nr / 32);
}

void ensure_copy_streams(hsw_handle* h, int nblk) {
    if (!h->copy_in) {
        CUDA_OK(cudaStreamCreateWithFlags(&h->copy_in, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&h->copy_out, cudaStreamNonBlocking));
        for (auto& e : h->ev_cp) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    while ((int)h->ev_in.size() < nblk) {
        cudaEvent_t a, b;
        CUDA_OK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CUDA_OK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        h->ev_in.push_back(a);
        h->ev_sw.push_back(b);
    }
}

// Worklist of the ordinate block [d0, d1): the all-ordinate list filtered,
// so the (level, element, ordinate) order and every pair's inputs are unchanged.
const hsw_handle::RangeList& range_list(hsw_handle* h, int d0, int d1) {
    auto key = std::make_pair(d0, d1);
    auto it = h->ranges.find(key);
    if (it != h->ranges.end()) return it->second;
    const auto& off = h->S.level_offsets;
    const int nd = h->S.nd;
    std::vector<int> pairs;
    hsw_handle::RangeList rl;
    rl.offsets.assign(off.size(), 0);
    for (size_t l = 0; l + 1 < off.size(); ++l) {
        for (int i = off[l]; i < off[l + 1]; ++i) {
            const int d = h->S.pairs_all[i] % nd;
            if (d >= d0 && d < d1) pairs.push_back(h->S.pairs_all[i]);
        }
        rl.offsets[l + 1] = (int)pairs.size();
    }
    if (!pairs.empty()) {
        CUDA_OK(cudaMalloc(&rl.d_pairs, pairs.size() * sizeof(int)));
        CUDA_OK(cudaMemcpy(rl.d_pairs, pairs.data(), pairs.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    return h->ranges.emplace(key, std::move(rl)).first->second;
}

void run_range_levels(hsw_handle* h, const hsw_handle::RangeList& rl, const double* psi_old, double* psi_new) {
    CUDA_OK(cudaEventRecord(h->ev0, h->stream));
    if (dataflow_enabled(h)) {   // the block's pairs depend only on pairs of the same ordinates
        if (rl.offsets.back() > 0) dataflow_sweep(h, psi_old, psi_new, rl.d_pairs, rl.offsets.back());
        CUDA_OK(cudaEventRecord(h->ev1, h->stream));
        h->last_launches = 1;
        return;
    }
    int64_t launches = 0;
    for (size_t l = 0; l + 1 < rl.offsets.size(); ++l) {
        const int n = rl.offsets[l + 1] - rl.offsets[l];
        if (n == 0) continue;
        sweep_launch(h, psi_old, psi_new, rl.d_pairs + rl.offsets[l], n);
        ++launches;
    }
    CUDA_OK(cudaEventRecord(h->ev1, h->stream));
    h->last_launches = launches;
}

void run_dir_levels(hsw_handle* h, int d, const double* psi_old, double* psi_new) {
    const auto& off = h->S.dir_level_offsets[d];
    const int* base = h->d_pairs_dir + (size_t)d * h->S.nel;
    for (size_t l = 0; l + 1 < off.size(); ++l) {
        const int n = off[l + 1] - off[l];
        if (n == 0) continue;
        sweep_launch(h, psi_old, psi_new, base + off[l], n);
    }
}

template <typename F>
int guarded(F&& f) {
    try {
        try {
            return f();
        } catch (const RetryPivot&) {
            // the static-pivot kernel refused a block: the handle now uses the pivoted kernel
            return f();
        }
    } catch (const RetryPivot&) {
        return fail(HSW_ERR_SOLVER, "static-pivot fallback raised twice");
    } catch (const hsw::Error& e) {
        return fail(e.status, e.what());
    } catch (const std::bad_alloc&) {
        return fail(HSW_ERR_NOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(HSW_ERR_INVALID, e.what());
    }
}
}  // namespace

namespace {
// SweepSolver::direct_oracle (solver.hpp:121-133) on the device: the per-ordinate
// global system (block lower-triangular in the sweep order plus the lagged
// couplings) is solved by lagged sweeps iterated to their fixed point,
// x_{k+1} = sweep_d(phi, psi_old = x_k), from x_0 = it (device, N doubles; used as
// scratch).  Converged when max|x_{k+1} - x_k| <= 16 eps max|x_{k+1}|, or at the
// round-off floor (no decrease for 8 sweeps while <= 1e-11 max|x|); otherwise
// HSW_ERR_SOLVER, like the reference's failed SparseLU (solver.hpp:130-131,190-192).
// The result is left in res (device, N doubles).  Uses the current h->d_src.
void direct_fixpoint(hsw_handle* h, int d, double* it, double* res) {
    const size_t N = h->N;
    const ptrdiff_t sh = (ptrdiff_t)d * (ptrdiff_t)N;
    const bool exact_in_one = h->S.ords[d].lagged_edges.empty();
    double best = INFINITY, diff = INFINITY, xmax = 0.0;
    int since_best = 0;
    constexpr int kMaxSweeps = 2000;
    for (int k = 0; k < kMaxSweeps; ++k) {
        run_dir_levels(h, d, it - sh, res - sh);
        dev_max_abs_diff(res, it, (int64_t)N, h->d_scratch, h->d_out, h->stream);
        CUDA_OK(cudaMemcpyAsync(h->h_out, h->d_out, 3 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaMemcpyAsync(it, res, N * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
        check_err(h);   // synchronises
        diff = h->h_out[0];
        xmax = h->h_out[2];
        if (exact_in_one || diff <= 16.0 * std::numeric_limits<double>::epsilon() * xmax) return;
        if (diff < best) {
            best = diff;
            since_best = 0;
        } else if (++since_best >= 8 && best <= 1e-11 * xmax) {
            return;
        }
    }
    char msg[160];
    std::snprintf(msg, sizeof(msg), "direct oracle: lagged fixed point did not converge for ordinate %d "
                  "(max |dpsi| = %.3e, max |psi| = %.3e)", d, diff, xmax);
    throw hsw::Error(HSW_ERR_SOLVER, msg);
}
}  // namespace

extern "C" {

int hsw_last_error(char* buf, size_t len) {
    if (buf && len) std::snprintf(buf, len, "%s", g_last_error.c_str());
    return (int)g_last_error.size();
}

namespace {
void device_init(hsw_handle* h, int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw hsw::Error(HSW_ERR_CUDA, "hsw_create: no CUDA device available (the B200 sweep has no CPU fallback)");
    h->device = device;
    CUDA_OK(cudaSetDevice(h->device));
    CUDA_OK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreate(&h->ev0));
    CUDA_OK(cudaEventCreate(&h->ev1));
}

// max|LR|, max|RL| of every (ordinate, interior face) on the device, in blocks of
// ordinates, for Setup::ordinates.  The blocks are produced on a helper
// thread in ascending ordinate order into a small ring of pinned host slots while
// Setup::ordinates (whose tasks are claimed in the same order) already works on the
// finished ones: S.cmax_acquire(d) blocks until ordinate d's magnitudes have arrived,
// S.cmax_release(d) counts the block's slot down; the producer reuses a slot once every
// ordinate of its previous block has been released.
struct CouplingFeed {
    static constexpr int kSlots = 4;
    hsw_handle* h;
    int nfi = 0, chunk = 1, nchunks = 0;
    size_t slot_doubles = 0;
    int* d_if = nullptr;
    double *d_sj = nullptr, *d_w = nullptr, *d_tr = nullptr, *d_trR = nullptr, *d_od = nullptr;
    double* d_out[2] = {nullptr, nullptr};
    double* ring = nullptr;   // pinned, kSlots blocks
    cudaStream_t kern = nullptr, copy = nullptr;   // its own streams: the handle's stream builds device state meanwhile
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEvent_t ev_t0[2] = {nullptr, nullptr};   // HSW_SETUP_TIMING: kernel start events
    double kernel_ms = 0.0, wait_slot_ms = 0.0, total_ms = 0.0;
    std::unique_ptr<std::atomic<int>[]> ready, left;
    std::atomic<bool> failed{false}, abort{false};

    explicit CouplingFeed(hsw_handle* hh) : h(hh) {
        Setup& S = h->S;
        nfi = (int)S.mesh.ifaces.size();
        if (nfi == 0) return;
        std::vector<int> iface((size_t)nfi * 5);
        for (int i = 0; i < nfi; ++i) {
            const IFace& F = S.mesh.ifaces[i];
            int* r = &iface[(size_t)i * 5];
            r[0] = F.el; r[1] = F.er; r[2] = F.fl; r[3] = F.fr; r[4] = F.orient;
        }
        std::vector<double> trR;
        for (const auto& t : S.traceR) trR.insert(trR.end(), t.begin(), t.end());
        d_if = dev_upload(iface);
        h->d_fgeom = dev_upload(S.fgeom);   // kept: the sweep kernels' face geometry
        d_sj = dev_upload(S.fsj);
        d_w = dev_upload(S.fq_w);
        d_tr = dev_upload(S.trace);
        d_trR = dev_upload(trR);
        d_od = dev_upload(S.odir);
        // blocks of about 12 MB of magnitudes (C4: 8 ordinates), two device buffers
        const int nds = S.oe - S.ob;
        chunk = std::max(1, std::min(nds, (int)(std::max<size_t>(1, (size_t)(12u << 20) / ((size_t)nfi * 16)))));
        nchunks = (nds + chunk - 1) / chunk;
        slot_doubles = (size_t)chunk * nfi * 2;
        for (auto& b : d_out) CUDA_OK(cudaMalloc(&b, slot_doubles * sizeof(double)));
        CUDA_OK(cudaMallocHost(&ring, (size_t)std::min(kSlots, nchunks) * slot_doubles * sizeof(double)));
        CUDA_OK(cudaStreamCreateWithFlags(&kern, cudaStreamNonBlocking));
        CUDA_OK(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
        const bool timing = std::getenv("HSW_SETUP_TIMING") != nullptr;
        for (auto& e : ev) CUDA_OK(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
        if (timing)
            for (auto& e : ev_t0) CUDA_OK(cudaEventCreate(&e));
        ready.reset(new std::atomic<int>[nchunks]);
        left.reset(new std::atomic<int>[nchunks]);
        for (int k = 0; k < nchunks; ++k) {
            ready[k].store(0);
            left[k].store(std::min(chunk, nds - k * chunk));
        }
        S.cmax_acquire = [this](int d) -> const double* {
            const int i = d - h->S.ob, k = i / chunk;
            while (!ready[k].load(std::memory_order_acquire)) {
                if (failed.load()) throw hsw::Error(HSW_ERR_CUDA, "hsw_create: the device coupling pass failed");
                std::this_thread::sleep_for(std::chrono::microseconds(20));
            }
            return ring + (size_t)(k % kSlots) * slot_doubles + (size_t)(i - k * chunk) * nfi * 2;
        };
        S.cmax_release = [this](int d) { left[(d - h->S.ob) / chunk].fetch_sub(1, std::memory_order_release); };
    }
    void launch(int k) {
        Setup& S = h->S;
        const int d0 = S.ob + k * chunk, d1 = std::min(S.oe, d0 + chunk);
        if (ev_t0[k & 1]) CUDA_OK(cudaEventRecord(ev_t0[k & 1], kern));
        dev_coupling_max(S.dim, nfi, S.nf, S.nqf, S.nfn, d_if, h->d_fgeom, d_sj, d_w, d_tr, d_trR, d_od, d0, d1,
                         d_out[k & 1], kern);
        CUDA_OK(cudaEventRecord(ev[k & 1], kern));
    }
    void produce() {   // helper thread
        if (nfi == 0) return;
        try {
            Setup& S = h->S;
            CUDA_OK(cudaSetDevice(h->device));
            const auto t_begin = std::chrono::steady_clock::now();
            launch(0);
            for (int k = 0; k < nchunks; ++k) {
                // block k + 1 is computed while block k is copied (its device buffer was
                // drained by the completed copy of block k - 1)
                if (k + 1 < nchunks) launch(k + 1);
                const auto t_w = std::chrono::steady_clock::now();
                while (k >= kSlots && left[k - kSlots].load(std::memory_order_acquire) > 0) {
                    if (abort.load()) return;   // the consumers are gone (an ordinate task threw)
                    std::this_thread::sleep_for(std::chrono::microseconds(20));
                }
                wait_slot_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_w).count();
                const int d0 = S.ob + k * chunk, d1 = std::min(S.oe, d0 + chunk);
                CUDA_OK(cudaStreamWaitEvent(copy, ev[k & 1], 0));
                CUDA_OK(cudaMemcpyAsync(ring + (size_t)(k % kSlots) * slot_doubles, d_out[k & 1],
                                        (size_t)(d1 - d0) * nfi * 2 * sizeof(double), cudaMemcpyDeviceToHost, copy));
                CUDA_OK(cudaStreamSynchronize(copy));
                if (ev_t0[k & 1]) {
                    float ms = 0.f;
                    CUDA_OK(cudaEventElapsedTime(&ms, ev_t0[k & 1], ev[k & 1]));
                    kernel_ms += ms;
                }
                ready[k].store(1, std::memory_order_release);
            }
            total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_begin).count();
            if (ev_t0[0])
                std::fprintf(stderr, "  coupling feed: %d blocks of %d ordinates, kernels %.1f ms, waited for slots %.1f ms, "
                             "producer %.1f ms\n", nchunks, chunk, kernel_ms, wait_slot_ms, total_ms);
        } catch (...) {
            failed.store(true);
            throw;
        }
    }
    ~CouplingFeed() {
        h->S.cmax_acquire = nullptr;
        h->S.cmax_release = nullptr;
        if (kern) cudaStreamSynchronize(kern);
        for (void* b : {(void*)d_if, (void*)d_sj, (void*)d_w, (void*)d_tr, (void*)d_trR, (void*)d_od, (void*)d_out[0],
                        (void*)d_out[1]})
            cudaFree(b);
        if (ring) cudaFreeHost(ring);
        if (kern) cudaStreamDestroy(kern);
        if (copy) cudaStreamDestroy(copy);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        for (auto e : ev_t0)
            if (e) cudaEventDestroy(e);
    }
};
}  // namespace

int hsw_create(const hsw_problem_desc* desc, hsw_handle** out) {
    if (!out) return fail(HSW_ERR_INVALID, "hsw_create: null output handle");
    *out = nullptr;
    hsw_handle* h = new hsw_handle();
    const int rc = guarded([&] {
        Setup& S = h->S;
        // HSW_SETUP_TIMING=1 prints the host setup phases (stderr)
        static const bool timing = std::getenv("HSW_SETUP_TIMING") != nullptr;
        auto tick = std::chrono::steady_clock::now();
        auto phase = [&](const char* name) {
            if (!timing) return;
            const auto now = std::chrono::steady_clock::now();
            std::fprintf(stderr, "hsw setup %-16s %8.3f s\n", name, std::chrono::duration<double>(now - tick).count());
            tick = now;
        };
        S.ingest(desc);
        phase("ingest");
        {   // the face geometry tables need the points and the (checked) connectivity only:
            // they are filled beside the face pairing / geometry validation of build_mesh
            S.mesh.check_connectivity(desc->num_points);
            Async faces([&] {
                const auto t0 = std::chrono::steady_clock::now();
                S.face_tables();
                if (timing)
                    std::fprintf(stderr, "  (face_tables, beside build_mesh) %.3f s\n",
                                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
            });
            S.build_mesh(desc->num_points, desc->validate_geometry != 0);
            faces.join();
        }
        phase("mesh+face_tables");
        // element tensors on the device unless host-only, or the siginvface weights
        // need the host's exact M_t arithmetic (sweepgraph.hpp:65-72)
        const bool host_T = desc->device < 0 || S.weighting == HSW_WEIGHT_SIGINVFACE;
        S.element_tensors(host_T);
        phase("element_tensors");
        if (desc->device >= 0) {
            device_init(h, desc->device);
            if (S.dim == 3 && S.face_pts != S.p + 2)
                throw hsw::Error(HSW_ERR_INVALID, "hsw_create: the 3D kernels integrate faces with p + 2 Gauss "
                                                  "points per axis (face_points " + std::to_string(S.face_pts) + ")");
        }
        if (desc->device < 0) {   // host-only plan, used by the CPU tests of the host logic
            S.ordinates();
            phase("ordinates");
            S.worklists();
            phase("worklists");
            return HSW_OK;
        }
        // Device state that does not depend on the orderings (tables, element tensors, materials,
        // psi / phi buffers) is built on a helper thread while the host works through the
        // per-ordinate graphs; the plan-dependent arrays are uploaded after both are done.
        auto device_static = [&] {
        CUDA_OK(cudaSetDevice(h->device));
        ConstTables ct{};
        for (int f = 0; f < S.nf; ++f)
            for (int a = 0; a < S.nfn; ++a) ct.fnode[f][a] = S.fnodes[f][a];
        for (int q = 0; q < S.nqf; ++q)
            for (int a = 0; a < S.nfn; ++a) ct.trace[q][a] = S.trace[(size_t)q * S.nfn + a];
        {
            std::vector<int> fidx((size_t)kMaxFaces * 128, -1);
            for (int f = 0; f < S.nf; ++f)
                for (int a = 0; a < S.nfn; ++a) fidx[(size_t)f * 128 + S.fnodes[f][a]] = a;
            std::vector<double> line(64, 0.0);
            for (int i = 0; i < S.face_pts && i < 8; ++i)
                for (int a = 0; a <= S.p && a < 8; ++a) line[(size_t)i * 8 + a] = S.basis.value(a, S.line_f.x[i]);
            std::vector<int> fn((size_t)kMaxFaces * kMaxFaceNodes, 0), nmask(128, 0);
            std::vector<double> tr((size_t)kMaxFacePoints * kMaxFaceNodes, 0.0);
            for (int f = 0; f < kMaxFaces; ++f)
                for (int a = 0; a < kMaxFaceNodes; ++a) fn[(size_t)f * kMaxFaceNodes + a] = ct.fnode[f][a];
            for (int q = 0; q < kMaxFacePoints; ++q)
                for (int a = 0; a < kMaxFaceNodes; ++a) tr[(size_t)q * kMaxFaceNodes + a] = ct.trace[q][a];
            for (int f = 0; f < kMaxFaces; ++f)
                for (int m = 0; m < 128; ++m)
                    if (fidx[(size_t)f * 128 + m] >= 0) nmask[m] |= 1 << f;
            h->d_tab_fnode = dev_upload(fn);
            h->d_tab_trace = dev_upload(tr);
            h->d_tab_fidx = dev_upload(fidx);
            h->d_tab_nmask = dev_upload(nmask);
            h->d_tab_line = dev_upload(line);
        }
        if (!S.T.empty()) {
            // host tensors are [E][n][m][4]; the device layout is the fragment order (t_idx), zero padded
            const int nb = S.nb;
            std::vector<double> Tp((size_t)S.nel * hsw::t_elem_doubles(nb), 0.0);
            for (size_t e = 0; e < (size_t)S.nel; ++e)
                for (int n = 0; n < nb; ++n)
                    for (int m = 0; m < nb; ++m)
                        for (int k = 0; k < 4; ++k)
                            Tp[hsw::t_idx(e, nb, m, n, k)] = S.T[((e * nb + n) * nb + m) * 4 + k];
            h->d_T = dev_upload(Tp);
            h->d_qvol = dev_upload(S.qvol);
        } else {   // element tensors + source moments computed on the device (hsw_setup.cu)
            const size_t nb = (size_t)S.nb, nel = (size_t)S.nel;
            CUDA_OK(cudaMalloc(&h->d_T, nel * hsw::t_elem_doubles(S.nb) * sizeof(double)));
            if (S.nb % 8 != 0)   // the tile padding is read by nobody, but keep it defined
                CUDA_OK(cudaMemsetAsync(h->d_T, 0, nel * hsw::t_elem_doubles(S.nb) * sizeof(double), h->stream));
            CUDA_OK(cudaMalloc(&h->d_qvol, nel * nb * sizeof(double)));
            double* d_pts = dev_upload(S.mesh.pts);
            int* d_en = dev_upload(S.mesh.enodes);
            double* d_U = dev_upload(S.volU);
            double* d_DU = dev_upload(S.volDU);
            double* d_GG = dev_upload(S.volGG);
            double* d_GV = dev_upload(S.volGV);
            double* d_w = dev_upload(S.vq_w);
            unsigned long long* d_bad = nullptr;
            CUDA_OK(cudaMalloc(&d_bad, sizeof(unsigned long long)));
            CUDA_OK(cudaMemset(d_bad, 0xff, sizeof(unsigned long long)));
            SourceParams sp{};
            for (int i = 0; i < 8; ++i) sp.v[i] = S.source_params[i];
            dev_element_tensors(S.dim, S.nel, S.nb, S.mesh.npe, S.nq, d_pts, d_en, d_U, d_DU, d_GG, d_GV, d_w,
                                S.source_kind, sp, h->d_T, h->d_qvol, d_bad, h->stream);
            unsigned long long bad = 0;
            S.qvol.resize(nel * nb);
            CUDA_OK(cudaMemcpyAsync(S.qvol.data(), h->d_qvol, nel * nb * sizeof(double), cudaMemcpyDeviceToHost,
                                    h->stream));
            CUDA_OK(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, h->stream));
            CUDA_OK(cudaStreamSynchronize(h->stream));
            for (void* b : {(void*)d_pts, (void*)d_en, (void*)d_U, (void*)d_DU, (void*)d_GG, (void*)d_GV, (void*)d_w,
                            (void*)d_bad})
                cudaFree(b);
            if (bad != ~0ull)
                throw hsw::Error(HSW_ERR_ASSEMBLY, "assembly: singular Jacobian in element " + std::to_string(bad));
        }
        h->d_sig_t = dev_upload(S.sig_t);
        h->d_sig_s = dev_upload(S.sig_s);
        CUDA_OK(cudaMalloc(&h->d_bscale, (size_t)S.nel * sizeof(double)));
        dev_block_scale(S.nel, S.nb, h->d_T, h->d_sig_t, h->d_bscale, h->stream);
        if (!h->d_fgeom) h->d_fgeom = dev_upload(S.fgeom);
        h->d_fnbr = dev_upload(S.fnbr);
        std::vector<double> om((size_t)S.nd * 4, 0.0);
        for (int d = 0; d < S.nd; ++d)
            for (int k = 0; k < 3; ++k) om[(size_t)d * 4 + k] = k < S.dim ? S.odir[3 * d + k] : 0.0;
        h->d_omega = dev_upload(om);
        h->d_weight = dev_upload(S.ow);
        h->N = (size_t)S.nel * S.nb;
        // psi of the shard's ordinates only; the handle's pointers are offset so that row d of
        // the global [nd][N] layout addresses ordinate d (kernels index psi by global d)
        const size_t psi_bytes = h->N * (size_t)(S.oe - S.ob) * sizeof(double);
        CUDA_OK(cudaMalloc(&h->d_psiA, psi_bytes));
        CUDA_OK(cudaMalloc(&h->d_psiB, psi_bytes));
        CUDA_OK(cudaMemset(h->d_psiA, 0, psi_bytes));
        CUDA_OK(cudaMemset(h->d_psiB, 0, psi_bytes));
        h->psi_offset = (size_t)S.ob * h->N;
        h->d_psiA -= h->psi_offset;
        h->d_psiB -= h->psi_offset;
        CUDA_OK(cudaMalloc(&h->d_phi, h->N * sizeof(double)));
        CUDA_OK(cudaMalloc(&h->d_phi_old, h->N * sizeof(double)));
        CUDA_OK(cudaMalloc(&h->d_src, h->N * sizeof(double)));
        CUDA_OK(cudaMalloc(&h->d_vec, h->N * sizeof(double)));
        CUDA_OK(cudaMalloc(&h->d_vec2, h->N * sizeof(double)));
        CUDA_OK(cudaMemset(h->d_phi, 0, h->N * sizeof(double)));
        CUDA_OK(cudaMemset(h->d_phi_old, 0, h->N * sizeof(double)));
        CUDA_OK(cudaMalloc(&h->d_scratch, (size_t)3 * 65536 * sizeof(double)));
        CUDA_OK(cudaMalloc(&h->d_out, 8 * sizeof(double)));
        CUDA_OK(cudaMalloc(&h->d_err, 2 * sizeof(unsigned long long)));
        CUDA_OK(cudaMalloc(&h->d_pair1, sizeof(int)));
        CUDA_OK(cudaMalloc(&h->d_prof, 16 * sizeof(unsigned long long)));
        CUDA_OK(cudaMemset(h->d_prof, 0, 16 * sizeof(unsigned long long)));
        CUDA_OK(cudaMemset(h->d_err, 0xff, 2 * sizeof(unsigned long long)));
        CUDA_OK(cudaMallocHost(&h->h_out, 8 * sizeof(double)));
        };   // device_static
        {
            // (siginvface needs the coupling blocks on the host; Romberg integrates them there)
            const bool dev_cpl = S.weighting != HSW_WEIGHT_SIGINVFACE && !S.face_blocks();
            std::unique_ptr<CouplingFeed> feed(dev_cpl ? new CouplingFeed(h) : nullptr);
            phase("coupling uploads");
            Async cpl([&] { if (feed) feed->produce(); });
            Async dev(device_static);
            struct AbortOnExit {   // destroyed before the threads are joined: frees a producer
                CouplingFeed* f;   // waiting for slots nobody will release (a task threw)
                ~AbortOnExit() { if (f) f->abort.store(true); }
            } abort_guard{feed.get()};
            S.ordinates();
            phase("ordinates");
            S.worklists();
            phase("worklists");
            cpl.join();
            dev.join();
            phase("device state");
        }
        h->d_inflags = dev_upload(S.inflags);
        h->d_pairs_all = dev_upload(S.pairs_all);
        h->d_pairs_dir = dev_upload(S.pairs_dir);
        DevProblem& P = h->P;
        P.dim = S.dim; P.p = S.p; P.nb = S.nb; P.nfn = S.nfn; P.nqf = S.nqf; P.nfaces = S.nf;
        P.nel = S.nel; P.nd = S.nd;
        {
            const char* tv = std::getenv("HSW_TUNE");
            P.tune = tv ? std::atoi(tv) : 0;
        }
        if (S.face_blocks()) {
            h->d_rom_ob = dev_upload(S.rom_ob);
            h->d_rom_ib = dev_upload(S.rom_ib);
            h->d_rom_bin = dev_upload(S.rom_bin);
            std::vector<unsigned char> om(S.rom_omask.begin(), S.rom_omask.end());
            h->d_rom_omask = dev_upload(om);
        }
        P.rom_ob = h->d_rom_ob;
        P.rom_ib = h->d_rom_ib;
        P.rom_bin = h->d_rom_bin;
        P.rom_omask = h->d_rom_omask;
        P.T = h->d_T; P.sig_t = h->d_sig_t; P.bscale = h->d_bscale; P.sig_s = h->d_sig_s; P.qvol = h->d_qvol;
        P.fgeom = h->d_fgeom; P.fnbr = h->d_fnbr; P.inflags = h->d_inflags;
        P.omega = h->d_omega; P.weight = h->d_weight; P.inflow = S.inflow;
        P.g_fnode = h->d_tab_fnode; P.g_trace = h->d_tab_trace; P.g_fidx = h->d_tab_fidx;
        P.g_nmask = h->d_tab_nmask; P.g_line = h->d_tab_line;
        P.prof = h->d_prof;
        // test hook (hsw_debug_create_zero_block): the (e, d) block zeroed from creation on
        if (g_create_zero_e >= 0 && g_create_zero_e < S.nel && g_create_zero_d < S.nd)
            h->zero_pair = (int64_t)g_create_zero_e * S.nd + g_create_zero_d;
        g_create_zero_e = g_create_zero_d = -1;
        if (desc->check_local_blocks) {
            // SweepSolver ctor factor check (solver.hpp:67-75): one sweep on zero data
            dev_scatter_source(P, h->d_phi, h->d_src, h->stream);
            run_all_levels(h, h->d_psiA, h->d_psiB, false);
            try {
                check_err(h);
            } catch (const RetryPivot&) {   // decided here once: this problem needs row pivoting
                run_all_levels(h, h->d_psiA, h->d_psiB, false);
                check_err(h);
            }
        }
        CUDA_OK(cudaStreamSynchronize(h->stream));
        return HSW_OK;
    });
    if (rc != HSW_OK) {
        free_handle(h);
        return rc;
    }
    *out = h;
    return HSW_OK;
}

void hsw_destroy(hsw_handle* h) { free_handle(h); }

int hsw_sizes(const hsw_handle* h, int64_t out[6]) {
    if (!h || !out) return fail(HSW_ERR_INVALID, "hsw_sizes: null argument");
    out[0] = h->S.nel;
    out[1] = h->S.nb;
    out[2] = h->S.nd;
    out[3] = (int64_t)h->N;
    out[4] = (int64_t)h->S.mesh.ifaces.size();
    out[5] = h->S.num_levels;
    return HSW_OK;
}

int hsw_ordering(const hsw_handle* h, int d, int* order, int* position, int* lagged, int lagged_cap,
                 int* num_lagged, double* lagged_weight, int* level) {
    if (!h) return fail(HSW_ERR_INVALID, "hsw_ordering: null handle");
    if (d < 0 || d >= h->S.nd) return fail(HSW_ERR_RANGE, "vector::_M_range_check: ordinate " + std::to_string(d));
    if (d < h->S.ob || d >= h->S.oe)
        return fail(HSW_ERR_RANGE, "hsw_ordering: ordinate " + std::to_string(d) + " is not in this handle's shard");
    const Ordering& o = h->S.ords[d];
    if (order) std::copy(o.order.begin(), o.order.end(), order);
    if (position) std::copy(o.position.begin(), o.position.end(), position);
    if (level) std::copy(o.level.begin(), o.level.end(), level);
    if (lagged) std::copy(o.lagged_edges.begin(), o.lagged_edges.begin() + std::min<size_t>(lagged_cap, o.lagged_edges.size()), lagged);
    if (num_lagged) *num_lagged = (int)o.lagged_edges.size();
    if (lagged_weight) *lagged_weight = o.lagged_weight;
    return HSW_OK;
}

int hsw_total_lagged_edges(const hsw_handle* h, int64_t* out) {
    if (!h || !out) return fail(HSW_ERR_INVALID, "hsw_total_lagged_edges: null argument");
    int64_t n = 0;
    for (const auto& o : h->S.ords) n += (int64_t)o.lagged_edges.size();
    *out = n;
    return HSW_OK;
}

int hsw_couplings(const hsw_handle* h, int d, int* ints4, double* weights, int cap, int* count) {
    if (!h) return fail(HSW_ERR_INVALID, "hsw_couplings: null handle");
    if (d < 0 || d >= h->S.nd) return fail(HSW_ERR_RANGE, "hsw_couplings: ordinate out of range");
    if (d < h->S.ob || d >= h->S.oe)
        return fail(HSW_ERR_RANGE, "hsw_couplings: ordinate " + std::to_string(d) + " is not in this handle's shard");
    const auto& c = h->S.couplings[d];
    if (count) *count = (int)c.size();
    const int n = std::min<int>(cap, (int)c.size());
    for (int i = 0; i < n; ++i) {
        if (ints4) {
            ints4[4 * i] = c[i].face;
            ints4[4 * i + 1] = c[i].down;
            ints4[4 * i + 2] = c[i].up;
            ints4[4 * i + 3] = h->S.lagged[d][i];
        }
        if (weights) weights[i] = h->S.weights[d][i];
    }
    return HSW_OK;
}

int hsw_interior_faces(const hsw_handle* h, int* ints5, int cap, int* count) {
    if (!h) return fail(HSW_ERR_INVALID, "hsw_interior_faces: null handle");
    const auto& f = h->S.mesh.ifaces;
    if (count) *count = (int)f.size();
    const int n = std::min<int>(cap, (int)f.size());
    for (int i = 0; i < n && ints5; ++i) {
        ints5[5 * i] = f[i].el; ints5[5 * i + 1] = f[i].er; ints5[5 * i + 2] = f[i].fl;
        ints5[5 * i + 3] = f[i].fr; ints5[5 * i + 4] = f[i].orient;
    }
    return HSW_OK;
}

int hsw_local_solve(hsw_handle* h, int e, int d, const double* rhs, double* out) {
    return guarded([&] {
        if (!h || !rhs || !out) throw hsw::Error(HSW_ERR_INVALID, "hsw_local_solve: null argument");
        HandleScope hs(h);
        need_device(h);
        if (e < 0 || e >= h->S.nel || d < 0 || d >= h->S.nd)
            throw hsw::Error(HSW_ERR_RANGE, "hsw_local_solve: element/ordinate out of range");
        need_in_shard(h, d, "hsw_local_solve");
        const size_t nb = h->S.nb;
        CUDA_OK(cudaMemcpyAsync(h->d_vec, rhs, nb * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        const int pr = e * h->S.nd + d;
        CUDA_OK(cudaMemcpyAsync(h->d_pair1, &pr, sizeof(int), cudaMemcpyHostToDevice, h->stream));
        if (kernel_choice_for(h->S.dim, h->S.p) == 4)
            dev_dmma2_local_solve(h->P, h->d_pair1, h->d_vec, h->d_vec2, h->d_err, h->zero_pair, h->stream);
        else if (kernel_choice_for(h->S.dim, h->S.p) == 3)
            dev_dmma1_local_solve(h->P, h->d_pair1, h->d_vec, h->d_vec2, h->d_err, h->zero_pair, h->stream);
        else
            dev_dmma_local_solve(h->P, h->d_pair1, h->d_vec, h->d_vec2, h->d_err, h->zero_pair, h->stream);
        CUDA_OK(cudaMemcpyAsync(out, h->d_vec2, nb * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        check_err(h);
        return HSW_OK;
    });
}

int hsw_sweep_device(hsw_handle* h, int d, const double* phi_dev, const double* psi_old_dev, double* psi_new_dev) {
    return guarded([&] {
        if (!h) throw hsw::Error(HSW_ERR_INVALID, "hsw_sweep_device: null handle");
        HandleScope hs(h);
        need_device(h);
        if (d < -1 || d >= h->S.nd) throw hsw::Error(HSW_ERR_RANGE, "hsw_sweep: ordinate out of range");
        if (d == -1) need_all_ordinates(h, "hsw_sweep_device(d = -1)");
        need_in_shard(h, d, "hsw_sweep_device");
        dev_scatter_source(h->P, phi_dev, h->d_src, h->stream);
        if (d == -1) {
            run_all_levels(h, psi_old_dev, psi_new_dev, false);
        } else {
            // single-ordinate vectors: shift the base so slot d addresses them
            const double* po = psi_old_dev - (ptrdiff_t)d * (ptrdiff_t)h->N;
            double* pn = psi_new_dev - (ptrdiff_t)d * (ptrdiff_t)h->N;
            run_dir_levels(h, d, po, pn);
        }
        return HSW_OK;
    });
}

// Sweep of ordinates [r0, r1) with HOST psi buffers holding that range (row d - r0),
// from the scattering source of h->d_phi_old.  Pipelined over ordinate blocks: a
// block's sweep needs only its own psi_old (lagged couplings stay within an
// ordinate), so the H2D of block b+1 and the D2H of block b-1 overlap the sweep of
// block b.  Stream-ordered on h->stream (the caller synchronizes).
// True for page-locked (cudaHostAlloc / cudaHostRegister) or managed host memory: the
// copy engines read / write it asynchronously.  Ordinary pageable memory is not.
static bool copy_engine_host(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// memcpy of one staging chunk split over persistent host workers (pageable caller memory is
// first-touched here, so the page faults are spread over the cores as well).  The workers are
// created once per process and sleep between chunks: a sweep stages ~130 chunks, and spawning
// and joining a thread team for each (parallel_for) cost ~20 ms of the C4 end-to-end time.
class CopyPool {
  public:
    explicit CopyPool(int n) {
        for (int i = 0; i < n; ++i) std::thread([this] { work(); }).detach();   // live until process exit
    }
    void run(void* dst, const void* src, size_t bytes) {
        std::lock_guard<std::mutex> call(call_mu_);   // one chunk at a time
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_done_.wait(lk, [&] { return busy_ == 0; });   // no worker still inside the previous job's loop
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            np_ = (int64_t)((bytes + kPiece - 1) / kPiece);
            next_.store(0);
            left_ = np_;
            ++gen_;
        }
        cv_work_.notify_all();
        const int64_t mine = copy_pieces();   // the caller works too
        std::unique_lock<std::mutex> lk(mu_);
        left_ -= mine;
        cv_done_.wait(lk, [&] { return left_ == 0; });
    }

  private:
    static constexpr size_t kPiece = (size_t)4 << 20;
    int64_t copy_pieces() {
        int64_t done = 0;
        for (;;) {
            const int64_t i = next_.fetch_add(1);
            if (i >= np_) break;
            const size_t off = (size_t)i * kPiece, len = std::min(kPiece, bytes_ - off);
            std::memcpy(dst_ + off, src_ + off, len);
            ++done;
        }
        return done;
    }
    void work() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_work_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                ++busy_;   // the job cannot be replaced while busy_ > 0
            }
            const int64_t done = copy_pieces();
            {
                std::lock_guard<std::mutex> lk(mu_);
                left_ -= done;
                --busy_;
            }
            cv_done_.notify_all();
        }
    }
    std::mutex call_mu_, mu_;
    std::condition_variable cv_work_, cv_done_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    int64_t np_ = 0, left_ = 0;
    int busy_ = 0;
    std::atomic<int64_t> next_{0};
    uint64_t gen_ = 0;
};
static void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    static CopyPool* pool = new CopyPool(std::max(0, host_workers() - 1));   // never destroyed: detached workers
    pool->run(dst, src, bytes);
}

// staging chunk (HSW_STAGE_MB overrides; 64 MiB default)
static size_t stage_chunk_bytes() {
    static const size_t v = [] {
        const char* e = std::getenv("HSW_STAGE_MB");
        const long mb = e ? std::atol(e) : 64;
        return (size_t)std::max(1l, mb) << 20;
    }();
    return v;
}

// pipelined_range_sweep for PAGEABLE caller buffers (what a reference caller passes:
// Eigen / std::vector / numpy storage).  The copy engines cannot stream pageable memory
// asynchronously, so every transfer goes through a pinned staging ring: host workers
// memcpy the next chunk of psi_old into an input stage while the previous stage's
// H2D copy and the sweeps of earlier ordinate blocks run, and drain the D2H output
// stages of finished blocks into psi_new.  Host order per block b: H2D(b), sweep(b),
// then the D2H of block b-1, so the GPU always has the next sweep queued while the host
// waits on a drain.  Synchronous on return (the caller's buffers are written).
static void staged_range_sweep(hsw_handle* h, int r0, int r1, const double* psi_old, double* psi_new) {
    const size_t N = h->N;
    const int nr = r1 - r0;
    {
        // the output is usually freshly allocated by the caller (the reference returns psi by
        // value): ask for transparent huge pages so that first-touch faults come per 2 MiB,
        // not per 4 KiB (a policy hint on the caller's mapping; ignored where THP is off)
        const uintptr_t a = reinterpret_cast<uintptr_t>(psi_new), pg = 4096;
        const uintptr_t lo = a & ~(pg - 1), hi = (a + (uintptr_t)nr * N * sizeof(double) + pg - 1) & ~(pg - 1);
        (void)madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
    }
    const int nblk = std::max(2, e2e_blocks(h, nr));
    ensure_copy_streams(h, nblk);
    const size_t CH = stage_chunk_bytes();
    if (!h->stage || h->stage_chunk != CH) {
        if (h->stage) CUDA_OK(cudaFreeHost(h->stage));
        h->stage = nullptr;
        CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&h->stage), 4 * CH, cudaHostAllocDefault));
        h->stage_chunk = CH;
        for (auto& e : h->ev_stage)
            if (!e) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    auto bstart = [&](int b) { return r0 + e2e_block_start(b, nblk, nr); };
    for (int b = 0; b < nblk; ++b) (void)range_list(h, bstart(b), bstart(b + 1));
    // inputs of the whole range are read after this point: order against earlier work
    CUDA_OK(cudaEventRecord(h->ev_cp[0], h->stream));
    CUDA_OK(cudaStreamWaitEvent(h->copy_in, h->ev_cp[0], 0));
    dev_scatter_source(h->P, h->d_phi_old, h->d_src, h->stream);
    int in_slot = 0;
    bool in_used[2] = {false, false};
    auto h2d = [&](int b) {
        const size_t off = (size_t)bstart(b) * N * sizeof(double), end = (size_t)bstart(b + 1) * N * sizeof(double);
        const size_t hbase = (size_t)r0 * N * sizeof(double);
        for (size_t o = off; o < end; o += CH) {
            const size_t len = std::min(CH, end - o);
            char* st = h->stage + (size_t)in_slot * CH;
            if (in_used[in_slot]) CUDA_OK(cudaEventSynchronize(h->ev_stage[in_slot]));   // its last copy is done
            parallel_memcpy(st, reinterpret_cast<const char*>(psi_old) + (o - hbase), len);
            CUDA_OK(cudaMemcpyAsync(reinterpret_cast<char*>(h->d_psiA) + o, st, len, cudaMemcpyHostToDevice,
                                    h->copy_in));
            CUDA_OK(cudaEventRecord(h->ev_stage[in_slot], h->copy_in));
            in_used[in_slot] = true;
            in_slot ^= 1;
        }
        CUDA_OK(cudaEventRecord(h->ev_in[b], h->copy_in));
    };
    int64_t launches = 1;   // the scatter-source kernel
    auto sweep = [&](int b) {
        CUDA_OK(cudaStreamWaitEvent(h->stream, h->ev_in[b], 0));
        run_range_levels(h, range_list(h, bstart(b), bstart(b + 1)), h->d_psiA, h->d_psiB);
        launches += h->last_launches;
        CUDA_OK(cudaEventRecord(h->ev_sw[b], h->stream));
    };
    auto d2h = [&](int b) {
        CUDA_OK(cudaStreamWaitEvent(h->copy_out, h->ev_sw[b], 0));
        const size_t off = (size_t)bstart(b) * N * sizeof(double), end = (size_t)bstart(b + 1) * N * sizeof(double);
        const size_t hbase = (size_t)r0 * N * sizeof(double);
        // two output stages: the copy of chunk k+1 runs while chunk k is drained
        std::vector<size_t> chunks;
        for (size_t o = off; o < end; o += CH) chunks.push_back(o);
        auto issue = [&](size_t k) {
            const size_t o = chunks[k], len = std::min(CH, end - o);
            char* st = h->stage + (2 + k % 2) * CH;
            CUDA_OK(cudaMemcpyAsync(st, reinterpret_cast<const char*>(h->d_psiB) + o, len, cudaMemcpyDeviceToHost,
                                    h->copy_out));
            CUDA_OK(cudaEventRecord(h->ev_stage[2 + k % 2], h->copy_out));
        };
        if (!chunks.empty()) issue(0);
        for (size_t k = 0; k < chunks.size(); ++k) {
            CUDA_OK(cudaEventSynchronize(h->ev_stage[2 + k % 2]));
            if (k + 1 < chunks.size()) issue(k + 1);
            const size_t o = chunks[k], len = std::min(CH, end - o);
            parallel_memcpy(reinterpret_cast<char*>(psi_new) + (o - hbase), h->stage + (2 + k % 2) * CH, len);
        }
    };
    h2d(0);
    sweep(0);
    for (int b = 1; b < nblk; ++b) {
        h2d(b);
        sweep(b);
        d2h(b - 1);
    }
    d2h(nblk - 1);
    CUDA_OK(cudaEventRecord(h->ev_cp[1], h->copy_out));
    CUDA_OK(cudaStreamWaitEvent(h->stream, h->ev_cp[1], 0));
    h->last_launches = launches;
}

static void pipelined_range_sweep(hsw_handle* h, int r0, int r1, const double* psi_old, double* psi_new) {
    const size_t N = h->N;
    const int nr = r1 - r0;
    if ((double)N * nr * sizeof(double) >= 64e6 && !(copy_engine_host(psi_old) && copy_engine_host(psi_new))) {
        staged_range_sweep(h, r0, r1, psi_old, psi_new);
        return;
    }
    const int nblk = e2e_blocks(h, nr);
    if (nblk <= 1) {
        CUDA_OK(cudaMemcpyAsync(h->d_psiA + (size_t)r0 * N, psi_old, N * nr * sizeof(double), cudaMemcpyHostToDevice,
                                h->stream));
        dev_scatter_source(h->P, h->d_phi_old, h->d_src, h->stream);
        if (r0 == 0 && r1 == h->S.nd)
            run_all_levels(h, h->d_psiA, h->d_psiB, false);
        else
            run_range_levels(h, range_list(h, r0, r1), h->d_psiA, h->d_psiB);
        h->last_launches += 1;   // the scatter-source kernel
        CUDA_OK(cudaMemcpyAsync(psi_new, h->d_psiB + (size_t)r0 * N, N * nr * sizeof(double), cudaMemcpyDeviceToHost,
                                h->stream));
        return;
    }
    ensure_copy_streams(h, nblk);
    for (int b = 0; b < nblk; ++b)   // worklists first: no allocation / sync copy between launches
        (void)range_list(h, r0 + e2e_block_start(b, nblk, nr), r0 + e2e_block_start(b + 1, nblk, nr));
    CUDA_OK(cudaEventRecord(h->ev_cp[0], h->stream));
    CUDA_OK(cudaStreamWaitEvent(h->copy_in, h->ev_cp[0], 0));
    dev_scatter_source(h->P, h->d_phi_old, h->d_src, h->stream);
    for (int b = 0; b < nblk; ++b) {
        const int d0 = r0 + e2e_block_start(b, nblk, nr), d1 = r0 + e2e_block_start(b + 1, nblk, nr);
        const size_t off = (size_t)d0 * N, hoff = (size_t)(d0 - r0) * N, cnt = (size_t)(d1 - d0) * N * sizeof(double);
        CUDA_OK(cudaMemcpyAsync(h->d_psiA + off, psi_old + hoff, cnt, cudaMemcpyHostToDevice, h->copy_in));
        CUDA_OK(cudaEventRecord(h->ev_in[b], h->copy_in));
    }
    int64_t launches = 1;   // the scatter-source kernel
    for (int b = 0; b < nblk; ++b) {
        const int d0 = r0 + e2e_block_start(b, nblk, nr), d1 = r0 + e2e_block_start(b + 1, nblk, nr);
        const size_t off = (size_t)d0 * N, hoff = (size_t)(d0 - r0) * N, cnt = (size_t)(d1 - d0) * N * sizeof(double);
        CUDA_OK(cudaStreamWaitEvent(h->stream, h->ev_in[b], 0));
        run_range_levels(h, range_list(h, d0, d1), h->d_psiA, h->d_psiB);
        launches += h->last_launches;
        CUDA_OK(cudaEventRecord(h->ev_sw[b], h->stream));
        CUDA_OK(cudaStreamWaitEvent(h->copy_out, h->ev_sw[b], 0));
        CUDA_OK(cudaMemcpyAsync(psi_new + hoff, h->d_psiB + off, cnt, cudaMemcpyDeviceToHost, h->copy_out));
    }
    CUDA_OK(cudaEventRecord(h->ev_cp[1], h->copy_out));
    CUDA_OK(cudaStreamWaitEvent(h->stream, h->ev_cp[1], 0));
    h->last_launches = launches;   // summed over the sub-blocks
}

int hsw_sweep(hsw_handle* h, int d, const double* phi, const double* psi_old, double* psi_new) {
    return guarded([&] {
        if (!h || !phi || !psi_old || !psi_new) throw hsw::Error(HSW_ERR_INVALID, "hsw_sweep: null argument");
        HandleScope hs(h);
        need_device(h);
        if (d < -1 || d >= h->S.nd) throw hsw::Error(HSW_ERR_RANGE, "hsw_sweep: ordinate out of range");
        if (d == -1) need_all_ordinates(h, "hsw_sweep(d = -1)");
        need_in_shard(h, d, "hsw_sweep");
        const size_t N = h->N;
        CUDA_OK(cudaMemcpyAsync(h->d_phi_old, phi, N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        if (d == -1) {
            pipelined_range_sweep(h, 0, h->S.nd, psi_old, psi_new);
        } else {
            double* slotA = h->d_psiA + (size_t)d * N;
            double* slotB = h->d_psiB + (size_t)d * N;
            CUDA_OK(cudaMemcpyAsync(slotA, psi_old, N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
            dev_scatter_source(h->P, h->d_phi_old, h->d_src, h->stream);
            run_dir_levels(h, d, h->d_psiA, h->d_psiB);
            CUDA_OK(cudaMemcpyAsync(psi_new, slotB, N * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        }
        check_err(h);
        return HSW_OK;
    });
}

int hsw_direct_oracle(hsw_handle* h, int d, const double* phi, double* psi) {
    return guarded([&] {
        if (!h || !phi || !psi) throw hsw::Error(HSW_ERR_INVALID, "hsw_direct_oracle: null argument");
        HandleScope hs(h);
        need_device(h);
        if (d < 0 || d >= h->S.nd) throw hsw::Error(HSW_ERR_RANGE, "hsw_direct_oracle: ordinate out of range");
        need_in_shard(h, d, "hsw_direct_oracle");
        const size_t N = h->N;
        CUDA_OK(cudaMemcpyAsync(h->d_phi_old, phi, N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        CUDA_OK(cudaMemsetAsync(h->d_vec, 0, N * sizeof(double), h->stream));
        dev_scatter_source(h->P, h->d_phi_old, h->d_src, h->stream);
        direct_fixpoint(h, d, h->d_vec, h->d_psiB + (size_t)d * N);
        CUDA_OK(cudaMemcpyAsync(psi, h->d_psiB + (size_t)d * N, N * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        return HSW_OK;
    });
}

int hsw_source_iteration(hsw_handle* h, const hsw_si_options* opts, hsw_si_result* res, double* psi_out,
                         double* phi_out, double* err_hist, double* phi_hist, double* per_ordinate_hist) {
    return guarded([&] {
        if (!h || !opts) throw hsw::Error(HSW_ERR_INVALID, "hsw_source_iteration: null argument");
        HandleScope hs(h);
        need_device(h);
        need_all_ordinates(h, "hsw_source_iteration");
        const size_t N = h->N;
        const int nd = h->S.nd;
        CUDA_OK(cudaMemsetAsync(h->d_psiA, 0, N * nd * sizeof(double), h->stream));
        CUDA_OK(cudaMemsetAsync(h->d_phi, 0, N * sizeof(double), h->stream));
        double* cur = h->d_psiA;
        double* nxt = h->d_psiB;
        double* phi_cur = h->d_phi;
        double* phi_nxt = h->d_phi_old;
        hsw_si_result r{};
        cudaEvent_t t0, t1;
        CUDA_OK(cudaEventCreate(&t0));
        CUDA_OK(cudaEventCreate(&t1));
        CUDA_OK(cudaEventRecord(t0, h->stream));
        for (int it = 0; it < opts->max_iterations; ++it) {
            dev_scatter_source(h->P, phi_cur, h->d_src, h->stream);
            if (opts->mode == HSW_MODE_DIRECT) {
                // direct_oracle per ordinate with phi fixed (solver.hpp:145-149), from psi_old
                for (int d = 0; d < nd; ++d) {
                    CUDA_OK(cudaMemcpyAsync(h->d_vec, cur + (size_t)d * N, N * sizeof(double), cudaMemcpyDeviceToDevice,
                                            h->stream));
                    direct_fixpoint(h, d, h->d_vec, nxt + (size_t)d * N);
                }
            } else {
                run_all_levels(h, cur, nxt, false);
            }
            dev_phi_and_norms(h->P, nxt, cur, phi_cur, phi_nxt, h->d_scratch, h->d_out, h->stream);
            CUDA_OK(cudaMemcpyAsync(h->h_out, h->d_out, 3 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
            if (per_ordinate_hist) {
                dev_per_ordinate_maxdiff(nxt, cur, nd, (int64_t)N, h->d_vec2, h->stream);
                CUDA_OK(cudaMemcpyAsync(per_ordinate_hist + (size_t)it * nd, h->d_vec2, (size_t)nd * sizeof(double),
                                        cudaMemcpyDeviceToHost, h->stream));
            }
            check_err(h);
            const double err = h->h_out[0];
            const double num = h->h_out[1], den = h->h_out[2];
            const double rel = den > 0.0 ? std::sqrt(num) / std::sqrt(den) : (num > 0.0 ? INFINITY : 0.0);
            if (err_hist) err_hist[it] = err;
            if (phi_hist) phi_hist[it] = rel;
            std::swap(cur, nxt);
            std::swap(phi_cur, phi_nxt);
            r.iterations = it + 1;
            r.final_error = err;
            r.final_phi_rel = rel;
            const double crit = opts->criterion == HSW_CRIT_PSI_LINF ? err : rel;
            if (crit < opts->tolerance) {
                r.converged = 1;
                break;
            }
        }
        CUDA_OK(cudaEventRecord(t1, h->stream));
        CUDA_OK(cudaEventSynchronize(t1));
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, t0, t1));
        r.seconds = ms * 1e-3;
        cudaEventDestroy(t0);
        cudaEventDestroy(t1);
        if (psi_out) CUDA_OK(cudaMemcpyAsync(psi_out, cur, N * nd * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        if (phi_out) CUDA_OK(cudaMemcpyAsync(phi_out, phi_cur, N * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        // keep the converged state in psiA / phi for hsw_device_state
        if (cur != h->d_psiA) std::swap(h->d_psiA, h->d_psiB);
        if (phi_cur != h->d_phi) std::swap(h->d_phi, h->d_phi_old);
        if (res) *res = r;
        return HSW_OK;
    });
}

int hsw_balance(hsw_handle* h, const double* psi, const double* phi, double out5[5], int* attrs, double* vals,
                int cap, int* count) {
    return guarded([&] {
        if (!h || !psi || !phi || !out5) throw hsw::Error(HSW_ERR_INVALID, "hsw_balance: null argument");
        HandleScope hs(h);
        need_all_ordinates(h, "hsw_balance");
        const Setup& S = h->S;
        const size_t N = h->N;
        const int nfn = S.nfn, nqf = S.nqf, nb = S.nb;
        double sv = 0.0, inflow_tot = 0.0, absorption = 0.0, outflow = 0.0;
        std::map<int, double> by_attr;
        double qsum = 0.0;
        for (size_t i = 0; i < N; ++i) qsum += S.qvol[i];
        for (int d = 0; d < S.nd; ++d) {
            const double w = S.ow[d];
            const double* om = &S.odir[3 * d];
            sv += w * qsum;
            double inf_d = 0.0;
            for (size_t bi = 0; bi < S.mesh.bfaces.size(); ++bi) {
                const auto& B = S.mesh.bfaces[bi];
                const double* geo = &S.fgeom[(((size_t)B.elem * S.nf + B.face) * nqf) * 4];
                const double* psie = psi + (size_t)d * N + (size_t)B.elem * nb;
                double o = 0.0;
                if (S.face_blocks()) {   // the integrated blocks (solver.hpp:225-233)
                    const size_t fb = ((size_t)d * S.nel + B.elem) * S.nf + B.face;
                    const double* blk = &S.rom_ob[fb * nfn * nfn];
                    for (int m = 0; m < nfn; ++m) {
                        double r = 0.0;
                        for (int n = 0; n < nfn; ++n) r += blk[(size_t)m * nfn + n] * psie[S.fnodes[B.face][n]];
                        o += r;
                    }
                    for (int m = 0; m < nfn; ++m) inf_d += S.rom_bin[fb * nfn + m];
                    o *= w;
                    outflow += o;
                    by_attr[B.attr] += o;
                    continue;
                }
                for (int q = 0; q < nqf; ++q) {
                    double on = 0.0;
                    for (int k = 0; k < S.dim; ++k) on += om[k] * geo[q * 4 + k];
                    const double wplus = 0.5 * (on + std::abs(on));
                    const double wminus = 0.5 * (std::abs(on) - on);
                    double tr = 0.0, ts = 0.0;
                    for (int a = 0; a < nfn; ++a) {
                        tr += S.trace[(size_t)q * nfn + a] * psie[S.fnodes[B.face][a]];
                        ts += S.trace[(size_t)q * nfn + a];
                    }
                    o += geo[q * 4 + 3] * wplus * tr * ts;
                    inf_d += geo[q * 4 + 3] * wminus * S.inflow * ts;
                }
                o *= w;
                outflow += o;
                by_attr[B.attr] += o;
            }
            inflow_tot += w * inf_d;
        }
        // absorption: (M_t - M_s) phi summed, with M_t - M_s = (sigma_t - sigma_s) M
        if (!S.T.empty()) {
            for (int e = 0; e < S.nel; ++e) {
                const double sa = S.sig_t[e] - S.sig_s[e];
                const double* Te = &S.T[(size_t)e * nb * nb * 4];
                for (int m = 0; m < nb; ++m)
                    for (int n = 0; n < nb; ++n)
                        absorption += sa * Te[((size_t)n * nb + m) * 4] * phi[(size_t)e * nb + n];
            }
        } else {   // the element tensors live on the device only
            need_device(h);
            CUDA_OK(cudaMemcpyAsync(h->d_vec, phi, N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
            absorption = dev_absorption(S.nel, nb, h->d_T, h->d_sig_t, h->d_sig_s, h->d_vec, h->d_scratch, h->stream);
        }
        out5[0] = sv;
        out5[1] = inflow_tot;
        out5[2] = absorption;
        out5[3] = outflow;
        out5[4] = sv + inflow_tot - absorption - outflow;
        int k = 0;
        for (const auto& kv : by_attr) {
            if (k < cap && attrs && vals) {
                attrs[k] = kv.first;
                vals[k] = kv.second;
            }
            ++k;
        }
        if (count) *count = k;
        return HSW_OK;
    });
}

int hsw_balance_resident(hsw_handle* h, double out5[5], int* attrs, double* vals, int cap, int* count) {
    return guarded([&] {
        if (!h || !out5) throw hsw::Error(HSW_ERR_INVALID, "hsw_balance_resident: null argument");
        HandleScope hs(h);
        need_device(h);
        need_all_ordinates(h, "hsw_balance_resident");
        const Setup& S = h->S;
        const int nbf = (int)S.mesh.bfaces.size();
        if (!h->d_bfaces && nbf > 0) {
            std::vector<int> bf((size_t)nbf * 3);
            for (int i = 0; i < nbf; ++i) {
                bf[3 * i] = S.mesh.bfaces[i].elem;
                bf[3 * i + 1] = S.mesh.bfaces[i].face;
                bf[3 * i + 2] = S.mesh.bfaces[i].attr;
            }
            h->d_bfaces = dev_upload(bf);
        }
        double* d_out = nullptr;
        CUDA_OK(cudaMallocAsync(&d_out, (size_t)std::max(nbf, 1) * 2 * sizeof(double), h->stream));
        dev_balance_faces(h->P, h->d_psiA, nbf, h->d_bfaces, d_out, h->stream);
        std::vector<double> fo((size_t)nbf * 2);
        if (nbf > 0)
            CUDA_OK(cudaMemcpyAsync(fo.data(), d_out, fo.size() * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaFreeAsync(d_out, h->stream));
        const double absorption =
            dev_absorption(S.nel, S.nb, h->d_T, h->d_sig_t, h->d_sig_s, h->d_phi, h->d_scratch, h->stream);
        double qsum = 0.0, wsum = 0.0, outflow = 0.0, inflow_tot = 0.0;
        for (size_t i = 0; i < h->N; ++i) qsum += S.qvol[i];
        for (int d = 0; d < S.nd; ++d) wsum += S.ow[d];
        std::map<int, double> by_attr;
        for (int i = 0; i < nbf; ++i) {
            outflow += fo[2 * i];
            inflow_tot += fo[2 * i + 1];
            by_attr[S.mesh.bfaces[i].attr] += fo[2 * i];
        }
        const double sv = wsum * qsum;
        out5[0] = sv;
        out5[1] = inflow_tot;
        out5[2] = absorption;
        out5[3] = outflow;
        out5[4] = sv + inflow_tot - absorption - outflow;
        int k = 0;
        for (const auto& kv : by_attr) {
            if (k < cap && attrs && vals) {
                attrs[k] = kv.first;
                vals[k] = kv.second;
            }
            ++k;
        }
        if (count) *count = k;
        return HSW_OK;
    });
}

int hsw_device_state(hsw_handle* h, double** psi_a, double** psi_b, double** phi) {
    if (!h) return fail(HSW_ERR_INVALID, "hsw_device_state: null handle");
    if (psi_a) *psi_a = h->d_psiA;
    if (psi_b) *psi_b = h->d_psiB;
    if (phi) *phi = h->d_phi;
    return HSW_OK;
}

int hsw_set_state(hsw_handle* h, const double* phi, const double* psi) {
    return guarded([&] {
        if (!h) throw hsw::Error(HSW_ERR_INVALID, "hsw_set_state: null handle");
        HandleScope hs(h);
        need_device(h);
        if (phi) CUDA_OK(cudaMemcpyAsync(h->d_phi, phi, h->N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        if (psi)
            CUDA_OK(cudaMemcpyAsync(h->d_psiA + (size_t)h->S.ob * h->N, psi,
                                    h->N * (size_t)(h->S.oe - h->S.ob) * sizeof(double), cudaMemcpyHostToDevice,
                                    h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        return HSW_OK;
    });
}

int hsw_sweep_resident(hsw_handle* h) {
    return guarded([&] {
        if (!h) throw hsw::Error(HSW_ERR_INVALID, "hsw_sweep_resident: null handle");
        HandleScope hs(h);
        need_device(h);
        dev_scatter_source(h->P, h->d_phi, h->d_src, h->stream);
        run_all_levels(h, h->d_psiA, h->d_psiB, true);
        h->last_launches += 1;  // scatter-source kernel
        return HSW_OK;
    });
}

// ---- direction-sharded source iteration primitives
namespace {
void check_block(const hsw_handle* h, int d0, int d1, const char* what) {
    if (d0 < h->S.ob || d1 > h->S.oe || d0 >= d1)
        throw hsw::Error(HSW_ERR_RANGE, std::string(what) + ": ordinate block [" + std::to_string(d0) + ", " +
                                            std::to_string(d1) + ") out of range");
}
}  // namespace

int hsw_shard_reset(hsw_handle* h) {
    return guarded([&] {
        if (!h) throw hsw::Error(HSW_ERR_INVALID, "hsw_shard_reset: null handle");
        HandleScope hs(h);
        need_device(h);
        const size_t N = h->N, ns = (size_t)(h->S.oe - h->S.ob), o = (size_t)h->S.ob * N;
        CUDA_OK(cudaMemsetAsync(h->d_psiA + o, 0, N * ns * sizeof(double), h->stream));
        CUDA_OK(cudaMemsetAsync(h->d_psiB + o, 0, N * ns * sizeof(double), h->stream));
        CUDA_OK(cudaMemsetAsync(h->d_phi, 0, N * sizeof(double), h->stream));
        return HSW_OK;
    });
}

int hsw_shard_sweep_host(hsw_handle* h, int d0, int d1, const double* phi, const double* psi_old, double* psi_new) {
    return guarded([&] {
        if (!h || !phi || !psi_old || !psi_new) throw hsw::Error(HSW_ERR_INVALID, "hsw_shard_sweep_host: null argument");
        HandleScope hs(h);
        need_device(h);
        check_block(h, d0, d1, "hsw_shard_sweep_host");
        CUDA_OK(cudaMemcpyAsync(h->d_phi_old, phi, h->N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
        pipelined_range_sweep(h, d0, d1, psi_old, psi_new);
        check_err(h);
        return HSW_OK;
    });
}

int hsw_shard_sweep(hsw_handle* h, int d0, int d1, const double* phi_dev) {
    return guarded([&] {
        if (!h) throw hsw::Error(HSW_ERR_INVALID, "hsw_shard_sweep: null handle");
        HandleScope hs(h);
        need_device(h);
        check_block(h, d0, d1, "hsw_shard_sweep");
        const auto& rl = range_list(h, d0, d1);
        dev_scatter_source(h->P, phi_dev ? phi_dev : h->d_phi, h->d_src, h->stream);
        run_range_levels(h, rl, h->d_psiA, h->d_psiB);
        h->last_launches += 1;   // scatter-source kernel
        return HSW_OK;
    });
}

int hsw_shard_phi_partial(hsw_handle* h, int d0, int d1, const double* prefix_dev, double* out_dev) {
    return guarded([&] {
        if (!h || !out_dev) throw hsw::Error(HSW_ERR_INVALID, "hsw_shard_phi_partial: null argument");
        HandleScope hs(h);
        need_device(h);
        check_block(h, d0, d1, "hsw_shard_phi_partial");
        dev_phi_partial(h->P, h->d_psiB, d0, d1, prefix_dev, out_dev, h->stream);
        return HSW_OK;
    });
}

int hsw_shard_psi_error(hsw_handle* h, int d0, int d1, double* err) {
    return guarded([&] {
        if (!h || !err) throw hsw::Error(HSW_ERR_INVALID, "hsw_shard_psi_error: null argument");
        HandleScope hs(h);
        need_device(h);
        check_block(h, d0, d1, "hsw_shard_psi_error");
        const size_t N = h->N;
        dev_max_abs_diff(h->d_psiB + (size_t)d0 * N, h->d_psiA + (size_t)d0 * N, (int64_t)((size_t)(d1 - d0) * N),
                         h->d_scratch, h->d_out, h->stream);
        CUDA_OK(cudaMemcpyAsync(h->h_out, h->d_out, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        check_err(h);   // synchronises; raises a singular local block of this sweep
        *err = h->h_out[0];
        return HSW_OK;
    });
}

int hsw_shard_phi_norms(hsw_handle* h, const double* phi_new_dev, const double* phi_old_dev, double out2[2]) {
    return guarded([&] {
        if (!h || !phi_new_dev || !phi_old_dev || !out2)
            throw hsw::Error(HSW_ERR_INVALID, "hsw_shard_phi_norms: null argument");
        HandleScope hs(h);
        need_device(h);
        dev_phi_norms2(h->P, phi_new_dev, phi_old_dev, h->d_scratch, h->d_out, h->stream);
        CUDA_OK(cudaMemcpyAsync(h->h_out, h->d_out, 3 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        out2[0] = h->h_out[1];
        out2[1] = h->h_out[2];
        return HSW_OK;
    });
}

int hsw_shard_advance(hsw_handle* h, const double* phi_dev) {
    return guarded([&] {
        if (!h) throw hsw::Error(HSW_ERR_INVALID, "hsw_shard_advance: null handle");
        HandleScope hs(h);
        need_device(h);
        std::swap(h->d_psiA, h->d_psiB);
        if (phi_dev)
            CUDA_OK(cudaMemcpyAsync(h->d_phi, phi_dev, h->N * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
        return HSW_OK;
    });
}

int hsw_shard_psi(hsw_handle* h, int d0, int d1, double* psi) {
    return guarded([&] {
        if (!h || !psi) throw hsw::Error(HSW_ERR_INVALID, "hsw_shard_psi: null argument");
        HandleScope hs(h);
        need_device(h);
        check_block(h, d0, d1, "hsw_shard_psi");
        const size_t N = h->N;
        CUDA_OK(cudaMemcpyAsync(psi, h->d_psiA + (size_t)d0 * N, (size_t)(d1 - d0) * N * sizeof(double),
                                cudaMemcpyDeviceToHost, h->stream));
        CUDA_OK(cudaStreamSynchronize(h->stream));
        return HSW_OK;
    });
}

int hsw_synchronize(hsw_handle* h) {
    return guarded([&] {
        if (!h) throw hsw::Error(HSW_ERR_INVALID, "hsw_synchronize: null handle");
        HandleScope hs(h);
        need_device(h);
        CUDA_OK(cudaStreamSynchronize(h->stream));
        check_err(h);
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, h->ev0, h->ev1) == cudaSuccess) h->last_kernel_ms = ms;
        cudaGetLastError();
        return HSW_OK;
    });
}

void* hsw_stream(hsw_handle* h) { return h ? (void*)h->stream : nullptr; }
int64_t hsw_last_launch_count(const hsw_handle* h) { return h ? h->last_launches : 0; }
int64_t hsw_pivot_fallbacks(const hsw_handle* h) { return h ? h->pivot_fallbacks : 0; }
double hsw_last_sweep_kernel_ms(const hsw_handle* h) { return h ? h->last_kernel_ms : 0.0; }

int hsw_fp64_peak(int device, double* tflops) {
    return guarded([&] {
        if (!tflops) throw hsw::Error(HSW_ERR_INVALID, "hsw_fp64_peak: null output");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw hsw::Error(HSW_ERR_CUDA, "hsw_fp64_peak: no CUDA device");
        // the FP64 roofline: max of the CUDA-core DFMA and the tensor-core DMMA rates
        const double dfma = dev_fp64_peak_tflops(device);
        const double dmma = dev_dmma_peak_tflops(device);
        if (const char* v = std::getenv("HSW_PEAK_VERBOSE"))
            if (v[0] == '1') std::fprintf(stderr, "fp64 peak: DFMA %.2f TFLOP/s, DMMA %.2f TFLOP/s\n", dfma, dmma);
        *tflops = dfma > dmma ? dfma : dmma;
        return HSW_OK;
    });
}

// Test hook: the product's graph ordering (Tarjan + exact/heuristic FAS + min-heap
// Kahn, sweepgraph.hpp:318-396) on an arbitrary weighted digraph, for randomized
// bit-exactness tests against the oracle.  Returns the number of lagged edges.
int hsw_debug_graph_order(int nv, int ne, const int* edges, const double* weights, int threshold, int* order,
                          int* lagged, double* lagged_weight) {
    try {
        if (nv < 1 || ne < 0 || (ne > 0 && (!edges || !weights)) || !order)
            throw hsw::Error(HSW_ERR_INVALID, "hsw_debug_graph_order: bad arguments");
        std::vector<Edge> es((size_t)ne);
        for (int i = 0; i < ne; ++i) {
            if (edges[2 * i] < 0 || edges[2 * i] >= nv || edges[2 * i + 1] < 0 || edges[2 * i + 1] >= nv)
                throw hsw::Error(HSW_ERR_RANGE, "hsw_debug_graph_order: vertex out of range");
            es[i] = {edges[2 * i], edges[2 * i + 1], weights[i]};
        }
        const Ordering o = sweep_ordering(nv, es, threshold);
        std::copy(o.order.begin(), o.order.end(), order);
        if (lagged) std::copy(o.lagged_edges.begin(), o.lagged_edges.end(), lagged);
        if (lagged_weight) *lagged_weight = o.lagged_weight;
        return (int)o.lagged_edges.size();
    } catch (const hsw::Error& e) {
        return fail(e.status, e.what());
    } catch (const std::exception& e) {
        return fail(HSW_ERR_LOGIC, e.what());
    }
}

int hsw_debug_flags(hsw_handle* h, int flags) {
    if (!h) return fail(HSW_ERR_INVALID, "hsw_debug_flags: null handle");
    h->P.debug_flags = flags;
    if (h->d_prof) cudaMemset(h->d_prof, 0, 16 * sizeof(unsigned long long));
    return HSW_OK;
}

int hsw_debug_profile(hsw_handle* h, unsigned long long out[16]) {
    if (!h || !h->d_prof) return fail(HSW_ERR_INVALID, "hsw_debug_profile: no device state");
    cudaStreamSynchronize(h->stream);
    cudaMemcpy(out, h->d_prof, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return HSW_OK;
}

int hsw_debug_create_zero_block(int e, int d) {
    if (e < 0 || d < 0) return fail(HSW_ERR_RANGE, "hsw_debug_create_zero_block: out of range");
    g_create_zero_e = e;
    g_create_zero_d = d;
    return HSW_OK;
}

int hsw_debug_zero_block(hsw_handle* h, int e, int d) {
    if (!h) return fail(HSW_ERR_INVALID, "hsw_debug_zero_block: null handle");
    if (e < 0 || e >= h->S.nel || d < 0 || d >= h->S.nd) return fail(HSW_ERR_RANGE, "hsw_debug_zero_block: out of range");
    h->zero_pair = (int64_t)e * h->S.nd + d;
    return HSW_OK;
}

}  // extern "C"
