// oracle/adapter_demo.cpp -- TEST INFRASTRUCTURE: the drop-in, end to end.
// The reference's own upstream (generate_mesh, build_cmap, build_element_table,
// build_dofmap, make_kernel, make_problem_from) feeds both the reference's
// nlfem::assemble and nlfem::gpu::assemble (include/nlfem_gpu_adapter.hpp);
// prints one JSON line comparing them.  Built into oracle/_ref/ by
// `make -C oracle ref`; run by tests/test_gpu_adapter.py on a B200.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "nlfem/assembly.hpp"
#include "nlfem/mesh.hpp"
#include "nlfem/problem.hpp"
#include "nlfem_gpu_adapter.hpp"

using namespace nlfem;

int main(int argc, char** argv) {
  const int res = argc > 1 ? std::atoi(argv[1]) : 6;
  const double delta = argc > 2 ? std::atof(argv[2]) : 0.34;
  const std::string strat = argc > 3 ? argv[3] : "nocaps";
  const int dim = argc > 4 ? std::atoi(argv[4]) : 3;
  const MeshData md = generate_mesh(dim, res, delta);
  const ElementTable et = build_element_table(build_cmap(dim, md.coords, md.cells, md.region));
  const DofMap dofs = build_dofmap(et);
  const Kernel k = make_kernel(dim, delta, Normalization::SecondMoment);
  Polynomial u = Polynomial::monomial({2, 0, 0}, 1.0) + Polynomial::monomial({0, 2, 0}, 1.0);
  if (dim == 3) u = u + Polynomial::monomial({0, 0, 2}, 1.0);
  const ManufacturedProblem mp = make_problem_from(u, k);
  AssemblyConfig cfg;
  cfg.strategy = parse_strategy(strat);
  cfg.seed = 1234;
  cfg.mc_samples = 16;
  cfg.threads = 0;
  const Polynomial f = mp.f, g = mp.u;
  AssemblyStats rs, gs;
  const LinearSystem ref = assemble(
      et, dofs, k, [f](Vec p) { return f.eval(p); }, [g](Vec p) { return g.eval(p); }, cfg, &rs);
  LinearSystem gpu;
  try {
    gpu = gpu::assemble(et, dofs, k, f, g, cfg, &gs);
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 2;
  }
  const bool pattern = ref.row_ptr == gpu.row_ptr && ref.col_idx == gpu.col_idx;
  double err = 0, rerr = 0, bmax = 0;
  if (pattern) {
    for (Index i = 0; i < ref.rows; ++i) {
      double rmax = 0;
      for (Index q = ref.row_ptr[i]; q < ref.row_ptr[i + 1]; ++q)
        rmax = std::max(rmax, std::abs(ref.values[q]));
      for (Index q = ref.row_ptr[i]; q < ref.row_ptr[i + 1]; ++q)
        err = std::max(err, std::abs(gpu.values[q] - ref.values[q]) / rmax);
      bmax = std::max(bmax, std::abs(ref.rhs[i]));
    }
    for (Index i = 0; i < ref.rows; ++i) rerr = std::max(rerr, std::abs(gpu.rhs[i] - ref.rhs[i]));
  }
  std::printf("{\"strategy\": \"%s\", \"rows\": %d, \"nnz\": %zu, \"pattern_equal\": %s, "
              "\"max_row_rel_err\": %.3e, \"rhs_rel_err\": %.3e, \"ref_s\": %.4f, \"gpu_s\": %.4f, "
              "\"mc_samples_ref\": %llu, \"mc_samples_gpu\": %llu}\n",
              strat.c_str(), ref.rows, ref.values.size(), pattern ? "true" : "false", err,
              bmax > 0 ? rerr / bmax : 0.0, rs.seconds, gs.seconds,
              (unsigned long long)rs.mc_samples, (unsigned long long)gs.mc_samples);
  return pattern ? 0 : 1;
}
