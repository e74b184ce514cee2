"""The C++ drop-in header (include/hosweep_b200/solver.hpp) compiles against the
C ABI, and its SweepSolver surface works on a host-only plan (no GPU): ordering(d),
total_lagged_edges(), out_of_range on a bad ordinate, MeshError on a bad mesh."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r'''
#include "hosweep_b200/solver.hpp"
#include <cmath>
#include <cstdio>
#include <vector>
int main() {
    // 2x1 linear quads on [0,2]x[0,1] (generators.hpp:24-67 layout), one ordinate along +x
    std::vector<double> pts = {0,0, 1,0, 2,0, 0,1, 1,1, 2,1};
    std::vector<int> nodes = {0,1,3,4, 1,2,4,5};
    std::vector<int> bf = {0,0,1, 1,0,1, 0,2,3, 1,2,3, 1,1,2, 0,3,4};
    double w[1] = {12.566370614359172}; double dir[3] = {1.0, 0.0, 0.0};
    int ids[1] = {1}; double st[1] = {1.0}; double ss[1] = {0.0};
    hsw_problem_desc d{};
    d.dim = 2; d.geom_order = 1; d.basis_order = 1;
    d.num_points = 6; d.points = pts.data(); d.num_elements = 2; d.element_nodes = nodes.data();
    d.num_boundary_faces = 6; d.boundary_faces = bf.data();
    d.num_ordinates = 1; d.ordinate_weight = w; d.ordinate_dir = dir;
    d.num_regions = 1; d.region_ids = ids; d.sigma_t = st; d.sigma_s = ss;
    d.source_params[0] = 1.0; d.validate_geometry = 1; d.device = -1;
    hosweep_b200::SweepSolver s(d);
    const auto& o = s.ordering(0);
    if (o.order.size() != 2 || o.order[0] != 0 || o.order[1] != 1 || !o.lagged_edges.empty()) return 2;
    if (s.total_lagged_edges() != 0 || o.level[1] != 1) return 3;
    try { s.ordering(1); return 4; } catch (const std::out_of_range&) {}
    try { s.sweep(0, std::vector<double>(8), std::vector<double>(8)); return 5; }
    catch (const hosweep_b200::DeviceError&) {}
    // balance_report (solver.hpp:220-245) of a host state: psi = phi = 1, Omega = +x ->
    // outflow only through the x = 2 face (attribute 2), its length times 4 pi
    hosweep_b200::SolverState stt;
    stt.psi.assign(1, std::vector<double>(8, 1.0));
    stt.phi.assign(8, 1.0);
    const auto br = hosweep_b200::balance_report(s, stt);
    if (br.outflow_by_attr.size() != 4 || std::abs(br.outflow - 12.566370614359172) > 1e-12 ||
        std::abs(br.outflow_by_attr.at(2) - br.outflow) > 1e-12) return 7;
    d.num_boundary_faces = 5;  // face left undeclared -> MeshError (mesh.hpp:333-337)
    try { hosweep_b200::SweepSolver bad(d); return 6; } catch (const hosweep_b200::MeshError&) {}
    std::puts("cpp wrapper ok");
    return 0;
}
'''


def test_cpp_wrapper_compiles_and_runs(tmp_path):
    from paper_1810_11080_b200 import _capi
    src = tmp_path / "w.cpp"
    src.write_text(SRC)
    exe = tmp_path / "w"
    libdir = os.path.dirname(_capi.LIB_PATH)
    subprocess.check_call(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                           "-L", libdir, "-lhosweep_b200", f"-Wl,-rpath,{libdir}"])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stdout, out.stderr)
    assert "cpp wrapper ok" in out.stdout
