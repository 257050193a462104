// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin C-ABI shim over the *unmodified* reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests and bench.py's reference arm drive the reference's own public
// API through ctypes:
//   generate_mesh            (reference proj/src/mesh.cpp:115)
//   build_cmap               (reference proj/src/cmap.cpp:56)
//   build_element_table      (reference proj/src/ball_approx.cpp:33)
//   build_dofmap             (reference proj/src/assembly.cpp:16)
//   make_kernel              (reference proj/src/polynomial.cpp:112)
//   make_problem_from        (reference proj/src/problem.cpp:5)
//   assemble                 (reference proj/src/assembly.cpp:617)   <- the hot path
//   walk_ball                (reference proj/include/nlfem/ball_approx.hpp:163)
//   cg_solve / l2_error      (reference proj/src/solver.cpp:26, study.cpp:76)
// Nothing here re-implements reference logic; it only marshals arrays.

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "nlfem/assembly.hpp"
#include "nlfem/ball_approx.hpp"
#include "nlfem/cmap.hpp"
#include "nlfem/mesh.hpp"
#include "nlfem/polynomial.hpp"
#include "nlfem/problem.hpp"
#include "nlfem/solver.hpp"
#include "nlfem/study.hpp"

using namespace nlfem;

namespace {

void set_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, std::size_t(errlen - 1));
    err[errlen - 1] = 0;
  }
}

Strategy strategy_of(int s) {
  switch (s) {
    case 0: return Strategy::Inside;
    case 1: return Strategy::Overlap;
    case 2: return Strategy::Barycenter;
    case 3: return Strategy::Nocaps;
    case 4: return Strategy::Approxcaps;
    default: return Strategy::Fullcaps;
  }
}

Polynomial poly_of(const double* terms, int nterms) {
  Polynomial p;
  for (int i = 0; i < nterms; ++i) {
    p = p + Polynomial::monomial({int(terms[4 * i + 1]), int(terms[4 * i + 2]),
                                  int(terms[4 * i + 3])},
                                 terms[4 * i + 0]);
  }
  return p;
}

struct Problem {
  ElementTable et;
  DofMap dofs;
  int n = 3;
};

struct Result {
  LinearSystem sys;
  AssemblyStats stats;
};

}  // namespace

extern "C" {

// ---- meshes ---------------------------------------------------------------

void* ref_mesh_generate(int res, double delta) {
  try {
    return new MeshData(generate_mesh(3, res, delta));
  } catch (...) {
    return nullptr;
  }
}

// generate_mesh in dimension n (2: triangles, the reference's 2D path)
void* ref_mesh_generate_n(int n, int res, double delta) {
  try {
    return new MeshData(generate_mesh(n, res, delta));
  } catch (...) {
    return nullptr;
  }
}

int ref_mesh_dim(void* h) { return static_cast<MeshData*>(h)->n; }

// Config-3 jitter (builder-defined): the reference's own
// nlfem::Rng (core.hpp:108-133) seeded with `seed`; for every node in id
// order draw u0, u1, u2; a node strictly inside (0,1)^3 (lattice index
// 0 < i < res per axis) moves by h (0.4 u - 0.2) per axis.
void* ref_mesh_generate_jittered(int res, double delta, std::int64_t seed) {
  try {
    auto* md = new MeshData(generate_mesh(3, res, delta));
    nlfem::Rng rng(static_cast<std::uint64_t>(seed));
    const double h = 1.0 / res;
    for (auto& p : md->coords) {
      const double u0 = rng.uniform(), u1 = rng.uniform(), u2 = rng.uniform();
      const long i = std::lround(p.x * res), j = std::lround(p.y * res), k = std::lround(p.z * res);
      if (i > 0 && i < res && j > 0 && j < res && k > 0 && k < res) {
        p.x = p.x + h * (0.4 * u0 - 0.2);
        p.y = p.y + h * (0.4 * u1 - 0.2);
        p.z = p.z + h * (0.4 * u2 - 0.2);
      }
    }
    return md;
  } catch (...) {
    return nullptr;
  }
}

void* ref_mesh_from_arrays(const double* coords, std::int64_t nnodes,
                           const std::int32_t* cells, const std::uint8_t* region,
                           std::int64_t ncells) {
  auto* md = new MeshData;
  md->n = 3;
  md->coords.resize(std::size_t(nnodes));
  for (std::int64_t i = 0; i < nnodes; ++i)
    md->coords[i] = {coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]};
  md->cells.resize(std::size_t(ncells));
  md->region.resize(std::size_t(ncells));
  for (std::int64_t k = 0; k < ncells; ++k) {
    md->cells[k] = {cells[4 * k], cells[4 * k + 1], cells[4 * k + 2], cells[4 * k + 3]};
    md->region[k] = region[k];
  }
  return md;
}

void ref_mesh_sizes(void* h, std::int64_t* nnodes, std::int64_t* ncells) {
  auto* md = static_cast<MeshData*>(h);
  *nnodes = std::int64_t(md->coords.size());
  *ncells = std::int64_t(md->cells.size());
}

void ref_mesh_copy(void* h, double* coords, std::int32_t* cells, std::uint8_t* region) {
  auto* md = static_cast<MeshData*>(h);
  for (std::size_t i = 0; i < md->coords.size(); ++i) {
    coords[3 * i] = md->coords[i].x;
    coords[3 * i + 1] = md->coords[i].y;
    coords[3 * i + 2] = md->coords[i].z;
  }
  for (std::size_t k = 0; k < md->cells.size(); ++k) {
    for (int j = 0; j < 4; ++j) cells[4 * k + j] = md->cells[k][j];
    region[k] = md->region[k];
  }
}

void ref_mesh_free(void* h) { delete static_cast<MeshData*>(h); }

// ---- element table + dof map ------------------------------------------------

void* ref_problem_build(void* mesh, char* err, int errlen) {
  try {
    auto* md = static_cast<MeshData*>(mesh);
    auto* p = new Problem;
    p->et = build_element_table(build_cmap(md->n, md->coords, md->cells, md->region));
    p->dofs = build_dofmap(p->et);
    p->n = md->n;
    return p;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void ref_problem_sizes(void* h, std::int64_t* nodes, std::int64_t* elems,
                       std::int64_t* unknowns) {
  auto* p = static_cast<Problem*>(h);
  *nodes = p->et.node_count;
  *elems = p->et.count;
  *unknowns = p->dofs.unknowns;
}

// Copies every ElementTable field (AoS -> flat arrays) plus the dof map.
void ref_problem_copy(void* h, std::int32_t* verts, std::int32_t* neighbor,
                      double* center, double* radius, double* volume, double* diam,
                      std::uint8_t* region, double* inv_edges, double* simplex,
                      std::int32_t* dof_of_node, std::uint8_t* constrained) {
  auto* p = static_cast<Problem*>(h);
  const ElementTable& et = p->et;
  for (Index t = 0; t < et.count; ++t) {
    for (int j = 0; j < 4; ++j) {
      verts[4 * t + j] = et.verts[t][j];
      neighbor[4 * t + j] = et.neighbor[t][j];
      simplex[12 * t + 3 * j] = et.simplex[t].v[j].x;
      simplex[12 * t + 3 * j + 1] = et.simplex[t].v[j].y;
      simplex[12 * t + 3 * j + 2] = et.simplex[t].v[j].z;
    }
    center[3 * t] = et.center[t].x;
    center[3 * t + 1] = et.center[t].y;
    center[3 * t + 2] = et.center[t].z;
    radius[t] = et.radius[t];
    volume[t] = et.volume[t];
    diam[t] = et.diam[t];
    region[t] = et.region[t];
    for (int j = 0; j < 9; ++j) inv_edges[9 * t + j] = et.inv_edges[t][j];
  }
  for (Index v = 0; v < et.node_count; ++v) {
    dof_of_node[v] = p->dofs.dof_of_node[v];
    constrained[v] = p->dofs.constrained[v];
  }
}

void ref_problem_free(void* h) { delete static_cast<Problem*>(h); }

// ---- kernel constant and manufactured forcing --------------------------------

// Writes C and the forcing polynomial f = -L u (at most maxterms terms).
int ref_forcing_n(int dim, double delta, int moment2, const double* uterms, int nu, double* C,
                  double* fterms, int maxterms) {
  const Kernel k = make_kernel(dim, delta, moment2 ? Normalization::SecondMoment
                                                   : Normalization::Mass);
  const ManufacturedProblem mp = make_problem_from(poly_of(uterms, nu), k);
  *C = k.C;
  int n = 0;
  for (const auto& t : mp.f.terms) {
    if (n >= maxterms) break;
    fterms[4 * n] = t.c;
    for (int a = 0; a < 3; ++a) fterms[4 * n + 1 + a] = t.e[a];
    ++n;
  }
  return n;
}

int ref_forcing(double delta, int moment2, const double* uterms, int nu, double* C,
                double* fterms, int maxterms) {
  return ref_forcing_n(3, delta, moment2, uterms, nu, C, fterms, maxterms);
}

// ---- the hot path: unmodified nlfem::assemble ---------------------------------

void* ref_assemble(void* problem, double delta, int strategy, int moment2,
                   const double* uterms, int nu, int threads, std::uint64_t seed,
                   int mc_samples, char* err, int errlen) {
  try {
    auto* p = static_cast<Problem*>(problem);
    const Kernel k = make_kernel(p->n, delta, moment2 ? Normalization::SecondMoment
                                                      : Normalization::Mass);
    const ManufacturedProblem mp = make_problem_from(poly_of(uterms, nu), k);
    const Polynomial f = mp.f, u = mp.u;
    AssemblyConfig cfg;
    cfg.strategy = strategy_of(strategy);
    cfg.threads = threads;
    cfg.seed = seed;
    cfg.mc_samples = mc_samples;
    auto* r = new Result;
    r->sys = assemble(
        p->et, p->dofs, k, [f](Vec x) { return f.eval(x); },
        [u](Vec x) { return u.eval(x); }, cfg, &r->stats);
    return r;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void ref_result_sizes(void* h, std::int64_t* rows, std::int64_t* nnz) {
  auto* r = static_cast<Result*>(h);
  *rows = r->sys.rows;
  *nnz = std::int64_t(r->sys.col_idx.size());
}

void ref_result_copy(void* h, std::int32_t* row_ptr, std::int32_t* col_idx,
                     double* values, double* rhs) {
  auto* r = static_cast<Result*>(h);
  std::memcpy(row_ptr, r->sys.row_ptr.data(), r->sys.row_ptr.size() * sizeof(Index));
  std::memcpy(col_idx, r->sys.col_idx.data(), r->sys.col_idx.size() * sizeof(Index));
  std::memcpy(values, r->sys.values.data(), r->sys.values.size() * sizeof(double));
  std::memcpy(rhs, r->sys.rhs.data(), r->sys.rhs.size() * sizeof(double));
}

void ref_result_stats(void* h, double* seconds, std::int32_t* threads,
                      std::int64_t* blocks, std::uint64_t* samples,
                      std::uint64_t* hits) {
  auto* r = static_cast<Result*>(h);
  *seconds = r->stats.seconds;
  *threads = r->stats.threads;
  *blocks = r->stats.blocks;
  *samples = r->stats.mc_samples;
  *hits = r->stats.mc_hits;
}

void ref_result_free(void* h) { delete static_cast<Result*>(h); }

// ---- per-point piece sets through the public walk_ball ------------------------
//
// For outer element t and outer quadrature point k (degree-2 rule), records the
// pieces walk_ball emits: (parent, kind) with kind 0 = whole, 1 = sub-simplex,
// 2 = Monte Carlo cap; sub-simplex pieces are recorded once per sub-simplex.
// Returns the number of pieces (or -1 on error / -2 if maxout too small).
int ref_walk_pieces(void* problem, std::int32_t t, int k, double delta, int strategy,
                    std::int32_t* parent, std::int32_t* kind, int maxout) {
  auto* p = static_cast<Problem*>(problem);
  const ElementTable& et = p->et;
  const QuadratureRule& rule = gauss_rule(et.n, 2);
  Vec x = rule.bary[k][0] * et.simplex[t].v[0];
  for (int i = 1; i <= et.n; ++i) x = x + rule.bary[k][i] * et.simplex[t].v[i];
  struct Rec {
    std::int32_t* parent;
    std::int32_t* kind;
    int maxout;
    int n = 0;
    void put(Index t, int kd) {
      if (n < maxout) {
        parent[n] = t;
        kind[n] = kd;
      }
      ++n;
    }
    void whole(Index t) { put(t, 0); }
    void sub(Index t, const Simplex&) { put(t, 1); }
    void cap(Index t, std::span<const Simplex>) { put(t, 2); }
  } rec{parent, kind, maxout};
  try {
    WalkScratch ws;
    walk_ball(et, ws, x, delta, t, strategy_of(strategy), rec);
  } catch (...) {
    return -1;
  }
  return rec.n > maxout ? -2 : rec.n;
}

// ---- harness helpers: CG + L2 error (reference solver.cpp / study.cpp) -------

int ref_solve_l2(void* problem, const std::int32_t* row_ptr, const std::int32_t* col_idx,
                 const double* values, const double* rhs, const double* uterms, int nu,
                 double tol, double* l2, double* max_nodal, std::int32_t* iters) {
  auto* p = static_cast<Problem*>(problem);
  LinearSystem sys;
  sys.rows = p->dofs.unknowns;
  sys.row_ptr.assign(row_ptr, row_ptr + sys.rows + 1);
  sys.col_idx.assign(col_idx, col_idx + sys.row_ptr.back());
  sys.values.assign(values, values + sys.row_ptr.back());
  sys.rhs.assign(rhs, rhs + sys.rows);
  const Polynomial u = poly_of(uterms, nu);
  SolveReport rep;
  std::vector<double> x = cg_solve(sys, sys.rhs, tol, 100 * std::max<Index>(sys.rows, 1), &rep);
  auto uf = [u](Vec y) { return u.eval(y); };
  std::vector<double> nv = node_values(p->et, p->dofs, x, uf);
  *l2 = l2_error(p->et, nv, uf);
  double mx = 0;
  for (Index v = 0; v < p->et.node_count; ++v) {
    if (p->dofs.constrained[v]) continue;
    mx = std::max(mx, std::abs(nv[v] - u.eval(p->et.node[v])));
  }
  *max_nodal = mx;
  *iters = rep.iterations;
  return rep.converged ? 0 : 1;
}

}  // extern "C"
