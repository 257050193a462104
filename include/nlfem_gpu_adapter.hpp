// nlfem_gpu_adapter.hpp -- header-only C++ adapter: the reference's own types
// in, the reference's own LinearSystem out, the B200 assembler in between.
//
//   #include "nlfem/assembly.hpp"        // reference headers
//   #include "nlfem_gpu_adapter.hpp"     // this file
//   LinearSystem sys = nlfem::gpu::assemble(et, dofs, kernel, f_poly, g_poly, cfg, &stats);
//
// Same contract as nlfem::assemble (reference proj/include/nlfem/assembly.hpp:71-73):
// borrowed const inputs, LinearSystem returned by value, optional stats, and
// nlfem::Error with the reference's ErrorCode on BadConfig / BallExitsMesh.
// f and g are nlfem::Polynomial instead of ScalarFn: a std::function cannot
// cross to the device, and every caller in the reference builds them from
// polynomials anyway (study.cpp:30-33, nlfem_module.cpp:134-137).
//
// The ElementTable and DofMap arrays are passed zero-copy: nlfem::Vec is three
// doubles and std::array<Index, 4> four int32, both contiguous.  A 2D table
// (et.n == 2, P1 triangles) goes to nlfem_gpu_assemble_2d, its three-slot
// arrays compacted from the table's four slots.
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "nlfem/assembly.hpp"
#include "nlfem/polynomial.hpp"
#include "nlfem_gpu.h"

namespace nlfem::gpu {

struct PolyArrays {
  std::vector<double> coef;
  std::vector<int32_t> exps;
  nlfem_gpu_poly view() const {
    return nlfem_gpu_poly{int32_t(coef.size()), coef.data(), exps.data()};
  }
};

inline PolyArrays flatten(const Polynomial& p) {
  PolyArrays a;
  for (const auto& t : p.terms) {  // Polynomial sort order is kept
    a.coef.push_back(t.c);
    for (int k = 0; k < 3; ++k) a.exps.push_back(t.e[k]);
  }
  return a;
}

inline LinearSystem assemble(const ElementTable& et, const DofMap& dofs, const Kernel& kernel,
                             const Polynomial& f, const Polynomial& g,
                             const AssemblyConfig& cfg, AssemblyStats* stats = nullptr,
                             int device = -1) {
  static_assert(sizeof(Vec) == 3 * sizeof(double), "Vec must be three packed doubles");
  static_assert(sizeof(std::array<Index, 4>) == 4 * sizeof(int32_t), "Index must be int32");
  if (kernel.n != et.n) fail(ErrorCode::BadConfig, "kernel dimension does not match mesh");
  const nlfem_gpu_dofs d{dofs.node_count, dofs.unknowns, dofs.dof_of_node.data()};
  const nlfem_gpu_kernel k{kernel.C, kernel.delta};
  const PolyArrays fa = flatten(f), ga = flatten(g);
  const nlfem_gpu_poly fp = fa.view(), gp = ga.view();
  const nlfem_gpu_config c{int32_t(cfg.strategy), cfg.mc_samples, cfg.seed,
                           NLFEM_SAMPLER_PHILOX, device};
  nlfem_gpu_csr out{};
  nlfem_gpu_stats st{};
  char err[512] = {0};
  int rc = 0;
  if (et.n == 2) {
    // the 2D table keeps four slots per element (reference ball_approx.hpp);
    // the 2D entry takes three vertices / neighbours and the four 2x2 inverse
    // entries per element
    std::vector<int32_t> v3(3 * size_t(et.count)), n3(3 * size_t(et.count));
    std::vector<double> inv4(4 * size_t(et.count));
    for (Index t = 0; t < et.count; ++t) {
      for (int i = 0; i < 3; ++i) {
        v3[3 * size_t(t) + i] = et.verts[t][i];
        n3[3 * size_t(t) + i] = et.neighbor[t][i];
      }
      for (int i = 0; i < 4; ++i) inv4[4 * size_t(t) + i] = et.inv_edges[t][i];
    }
    const nlfem_gpu_mesh2d mesh2{et.node_count,
                                 et.count,
                                 reinterpret_cast<const double*>(et.node.data()),
                                 v3.data(),
                                 n3.data(),
                                 reinterpret_cast<const double*>(et.center.data()),
                                 et.radius.data(),
                                 et.volume.data(),
                                 et.diam.data(),
                                 et.region.data(),
                                 inv4.data()};
    rc = nlfem_gpu_assemble_2d(&mesh2, &d, &k, &fp, &gp, &c, &out, &st, err, sizeof(err));
  } else {
    if (et.n != 3) fail(ErrorCode::BadConfig, "mesh dimension must be 2 or 3");
    const nlfem_gpu_mesh mesh{
      et.node_count,
      et.count,
      reinterpret_cast<const double*>(et.node.data()),
      reinterpret_cast<const int32_t*>(et.verts.data()),
      reinterpret_cast<const int32_t*>(et.neighbor.data()),
      reinterpret_cast<const double*>(et.center.data()),
      et.radius.data(),
      et.volume.data(),
      et.diam.data(),
      et.region.data(),
      reinterpret_cast<const double*>(et.inv_edges.data())};
    rc = nlfem_gpu_assemble(&mesh, &d, &k, &fp, &gp, &c, &out, &st, err, sizeof(err));
  }
  if (rc >= 1 && rc <= 8) throw Error(ErrorCode(rc - 1), err);
  if (rc != 0) throw std::runtime_error(std::string("nlfem_gpu_assemble: ") + err);
  LinearSystem sys;
  sys.rows = out.rows;
  sys.row_ptr.assign(out.row_ptr, out.row_ptr + out.rows + 1);
  sys.col_idx.assign(out.col_idx, out.col_idx + out.nnz);
  sys.values.assign(out.values, out.values + out.nnz);
  sys.rhs.assign(out.rhs, out.rhs + out.rows);
  nlfem_gpu_free_csr(&out);
  if (stats) {
    stats->seconds = st.seconds;
    stats->threads = st.threads;
    stats->blocks = st.blocks;
    stats->mc_samples = st.mc_samples;
    stats->mc_hits = st.mc_hits;
  }
  return sys;
}

}  // namespace nlfem::gpu
