// host_setup.cpp -- the reference's upstream setup, restated for the host.
//
// Compiled with -ffp-contract=off: every expression keeps the reference's
// operation order and rounding (the reference binary is FMA-free), so the
// element table is bit-identical to build_element_table's.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "nlfem_gpu.h"
#include "nlfem_host.h"

namespace {

struct V3 {
  double x, y, z;
};
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 scale(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}

void put_err(char* err, size_t len, const std::string& m) {
  if (!err || len == 0) return;
  std::strncpy(err, m.c_str(), len - 1);
  err[len - 1] = 0;
}

// splitmix64 / xoshiro256++ as nlfem::Rng (reference core.hpp:90-133).
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
struct Xoshiro {
  uint64_t s[4];
  explicit Xoshiro(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s) w = x = mix64(x);
  }
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return double(next() >> 11) * 0x1.0p-53; }
};

// ---- polynomials (reference polynomial.cpp) -----------------------------------
struct Term {
  std::array<int, 3> e;
  double c;
};
using Poly = std::vector<Term>;

void normalize(Poly& ts) {
  std::sort(ts.begin(), ts.end(), [](const Term& a, const Term& b) { return a.e < b.e; });
  Poly out;
  for (const Term& t : ts) {
    if (!out.empty() && out.back().e == t.e) out.back().c += t.c;
    else out.push_back(t);
  }
  out.erase(std::remove_if(out.begin(), out.end(), [](const Term& t) { return t.c == 0.0; }),
            out.end());
  ts = std::move(out);
}
Poly padd(const Poly& a, const Poly& b) {
  Poly r = a;
  r.insert(r.end(), b.begin(), b.end());
  normalize(r);
  return r;
}
Poly pscale(double s, const Poly& a) {
  Poly r = a;
  for (Term& t : r) t.c *= s;
  if (s == 0) r.clear();
  return r;
}
Poly pderiv(const Poly& p, int axis) {
  Poly d;
  for (const Term& t : p) {
    if (t.e[axis] == 0) continue;
    Term nt = t;
    nt.c *= t.e[axis];
    nt.e[axis] -= 1;
    d.push_back(nt);
  }
  normalize(d);
  return d;
}
int pdegree(const Poly& p) {
  int d = 0;
  for (const Term& t : p) d = std::max(d, t.e[0] + t.e[1] + t.e[2]);
  return d;
}
Poly poly_from_rows(const double* rows, int n) {
  Poly p;
  for (int i = 0; i < n; ++i) {
    const double c = rows[4 * i];
    if (c == 0) continue;  // Polynomial::monomial drops zero coefficients
    Poly m{{{int(rows[4 * i + 1]), int(rows[4 * i + 2]), int(rows[4 * i + 3])}, c}};
    p = padd(p, m);
  }
  return p;
}

double ball_moment3(std::array<int, 3> e, double r) {
  const int n = 3;
  int total = 0;
  for (int a = 0; a < n; ++a) {
    if (e[a] % 2 != 0) return 0.0;
    total += e[a];
  }
  double dfac = 1;
  for (int a = 0; a < n; ++a)
    for (int k = e[a] - 1; k >= 2; k -= 2) dfac *= k;
  const double num = dfac * std::pow(M_PI, 0.5 * n);
  const double den = std::pow(2.0, 0.5 * total) * std::tgamma(0.5 * (n + total) + 1.0);
  return num / den * std::pow(r, n + total);
}

double kernel_C(double delta, bool moment2) {
  const double mass = ball_moment3({0, 0, 0}, delta);
  if (!moment2) return 3.0 / mass;
  const double m2 = ball_moment3({2, 0, 0}, delta) * 3;
  return 3.0 / m2;
}

Poly apply_L(const Poly& u, double delta, double C) {
  Poly acc;
  const int deg = pdegree(u);
  std::array<int, 3> a{0, 0, 0};
  for (a[0] = 0; a[0] <= deg; a[0] += 2) {
    for (a[1] = 0; a[0] + a[1] <= deg; a[1] += 2) {
      const int zmax = deg - a[0] - a[1];
      for (a[2] = 0; a[2] <= zmax; a[2] += 2) {
        if (a[0] + a[1] + a[2] == 0) continue;
        Poly d = u;
        double fact = 1;
        for (int ax = 0; ax < 3; ++ax)
          for (int i = 0; i < a[ax]; ++i) {
            d = pderiv(d, ax);
            fact *= (i + 1);
          }
        if (d.empty()) continue;
        acc = padd(acc, pscale(ball_moment3(a, delta) / fact, d));
      }
    }
  }
  return pscale(2.0 * C, acc);
}

int sort_parity3(const int32_t* t) {
  int inv = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = i + 1; j < 3; ++j)
      if (t[i] > t[j]) ++inv;
  return inv & 1;
}

}  // namespace

extern "C" {

int nlfem_host_lattice_mesh(int32_t res, double delta, int64_t jitter_seed,
                            int64_t* nnodes, int64_t* ncells, double* coords,
                            int32_t* cells, uint8_t* region) {
  if (res < 1 || !(delta > 0)) return NLFEM_GPU_BAD_CONFIG;
  const int32_t L = int32_t(std::ceil(delta * res - 1e-9));
  const int32_t lo = -L, hi = res + L;
  const int64_t nv1 = int64_t(hi - lo + 1);
  const double h = 1.0 / res;
  *nnodes = nv1 * nv1 * nv1;
  *ncells = 6 * (nv1 - 1) * (nv1 - 1) * (nv1 - 1);
  if (!coords) return 0;
  auto vid = [&](int64_t i, int64_t j, int64_t k) {
    return int32_t(((k - lo) * nv1 + (j - lo)) * nv1 + (i - lo));
  };
  int64_t v = 0;
  for (int32_t k = lo; k <= hi; ++k)
    for (int32_t j = lo; j <= hi; ++j)
      for (int32_t i = lo; i <= hi; ++i, ++v) {
        coords[3 * v] = i * h;
        coords[3 * v + 1] = j * h;
        coords[3 * v + 2] = k * h;
      }
  // Kuhn split: one tet per axis permutation, odd permutations swap the last
  // two vertices so every volume is positive (reference mesh.cpp:20-26).
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                  {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  static const bool odd[6] = {false, true, true, false, false, true};
  auto interior = [&](int32_t x) { return x >= 0 && x < res; };
  int64_t c = 0;
  for (int32_t k = lo; k < hi; ++k)
    for (int32_t j = lo; j < hi; ++j)
      for (int32_t i = lo; i < hi; ++i) {
        const uint8_t tag = !(interior(i) && interior(j) && interior(k));
        for (int t = 0; t < 6; ++t, ++c) {
          int64_t ix[3] = {i, j, k};
          int32_t* tet = cells + 4 * c;
          tet[0] = vid(ix[0], ix[1], ix[2]);
          for (int s = 0; s < 3; ++s) {
            ++ix[perms[t][s]];
            tet[s + 1] = vid(ix[0], ix[1], ix[2]);
          }
          if (odd[t]) std::swap(tet[2], tet[3]);
          region[c] = tag;
        }
      }
  if (jitter_seed >= 0) {
    Xoshiro rng{uint64_t(jitter_seed)};
    v = 0;
    for (int32_t k = lo; k <= hi; ++k)
      for (int32_t j = lo; j <= hi; ++j)
        for (int32_t i = lo; i <= hi; ++i, ++v) {
          const double u0 = rng.uniform(), u1 = rng.uniform(), u2 = rng.uniform();
          if (i > 0 && i < res && j > 0 && j < res && k > 0 && k < res) {
            coords[3 * v] = coords[3 * v] + h * (0.4 * u0 - 0.2);
            coords[3 * v + 1] = coords[3 * v + 1] + h * (0.4 * u1 - 0.2);
            coords[3 * v + 2] = coords[3 * v + 2] + h * (0.4 * u2 - 0.2);
          }
        }
  }
  return 0;
}

int nlfem_host_element_table(const double* coords, int64_t nnodes, const int32_t* cells,
                             const uint8_t* region, int64_t ncells, int32_t* verts,
                             int32_t* neighbor, double* center, double* radius,
                             double* volume, double* diam, double* inv_edges, char* err,
                             size_t errlen) {
  (void)region;
  const int64_t K = ncells, Vn = nnodes;
  // --- validation (reference cmap.cpp:66-83)
  std::vector<uint8_t> used(size_t(Vn), 0);
  for (int64_t k = 0; k < K; ++k) {
    for (int i = 0; i < 4; ++i) {
      const int32_t v = cells[4 * k + i];
      if (v < 0 || v >= Vn) {
        put_err(err, errlen, "BadIndex: cell " + std::to_string(k) + " references vertex " +
                                 std::to_string(v));
        return NLFEM_GPU_BAD_INDEX;
      }
      for (int j = i + 1; j < 4; ++j)
        if (cells[4 * k + j] == v) {
          put_err(err, errlen, "BadIndex: cell " + std::to_string(k) + " repeats vertex " +
                                   std::to_string(v));
          return NLFEM_GPU_BAD_INDEX;
        }
      used[size_t(v)] = 1;
    }
  }
  for (int64_t v = 0; v < Vn; ++v)
    if (!used[size_t(v)]) {
      put_err(err, errlen,
              "DanglingVertex: vertex " + std::to_string(v) + " is not used by any cell");
      return NLFEM_GPU_DANGLING_VERTEX;
    }

  // --- facet incidence: sort (sorted triple, cell, slot) records
  struct Facet {
    int32_t a, b, c;
    int32_t cell;
    int8_t slot, par;
  };
  std::vector<Facet> fs(size_t(4 * K));
  for (int64_t k = 0; k < K; ++k)
    for (int s = 0; s < 4; ++s) {
      int32_t tup[3];
      int m = 0;
      for (int i = 0; i < 4; ++i)
        if (i != s) tup[m++] = cells[4 * k + i];
      const int par = sort_parity3(tup) ^ (s & 1);
      std::sort(tup, tup + 3);
      fs[size_t(4 * k + s)] = {tup[0], tup[1], tup[2], int32_t(k), int8_t(s), int8_t(par)};
    }
  std::sort(fs.begin(), fs.end(), [](const Facet& x, const Facet& y) {
    if (x.a != y.a) return x.a < y.a;
    if (x.b != y.b) return x.b < y.b;
    if (x.c != y.c) return x.c < y.c;
    if (x.cell != y.cell) return x.cell < y.cell;
    return x.slot < y.slot;
  });
  // partner[4k+s] = (other cell, other slot) across the facet opposite input slot s
  std::vector<int32_t> other(size_t(4 * K), -1);
  std::vector<int8_t> psum(size_t(4 * K), 0);
  for (size_t i = 0; i < fs.size();) {
    size_t j = i + 1;
    while (j < fs.size() && fs[j].a == fs[i].a && fs[j].b == fs[i].b && fs[j].c == fs[i].c) ++j;
    if (j - i > 2) {
      put_err(err, errlen, "NonManifold: facet shared by more than two cells");
      return NLFEM_GPU_NON_MANIFOLD;
    }
    if (j - i == 2) {
      const Facet& A = fs[i];
      const Facet& B = fs[i + 1];
      other[size_t(4 * A.cell + A.slot)] = B.cell;
      other[size_t(4 * B.cell + B.slot)] = A.cell;
      psum[size_t(4 * A.cell + A.slot)] = int8_t(A.par ^ B.par);
      psum[size_t(4 * B.cell + B.slot)] = int8_t(A.par ^ B.par);
    }
    i = j;
  }
  // --- orientation: BFS from each unseen root; adjacent cells must induce
  // opposite facet orientations (reference cmap.cpp:107-140).  The flip state
  // is unique per component given its lowest-id root, so traversal order is free.
  std::vector<uint8_t> flipped(size_t(K), 0), seen(size_t(K), 0);
  std::vector<int32_t> queue;
  for (int64_t root = 0; root < K; ++root) {
    if (seen[size_t(root)]) continue;
    seen[size_t(root)] = 1;
    queue.assign(1, int32_t(root));
    for (size_t qi = 0; qi < queue.size(); ++qi) {
      const int32_t c = queue[qi];
      for (int s = 0; s < 4; ++s) {
        const int32_t o = other[size_t(4 * c + s)];
        if (o < 0) continue;
        const uint8_t want = uint8_t(flipped[size_t(c)] ^ psum[size_t(4 * c + s)] ^ 1);
        if (!seen[size_t(o)]) {
          seen[size_t(o)] = 1;
          flipped[size_t(o)] = want;
          queue.push_back(o);
        } else if (flipped[size_t(o)] != want) {
          put_err(err, errlen, "NonManifold: mesh is not orientable");
          return NLFEM_GPU_NON_MANIFOLD;
        }
      }
    }
  }
  // --- per-element fields (reference ball_approx.cpp:51-95)
  for (int64_t t = 0; t < K; ++t) {
    int32_t w[4] = {cells[4 * t], cells[4 * t + 1], cells[4 * t + 2], cells[4 * t + 3]};
    if (flipped[size_t(t)]) std::swap(w[2], w[3]);
    for (int s = 0; s < 4; ++s) {
      verts[4 * t + s] = w[s];
      // input slot s sits at effective slot s, except 2 <-> 3 when flipped
      const int eff = flipped[size_t(t)] ? (s == 2 ? 3 : (s == 3 ? 2 : s)) : s;
      neighbor[4 * t + eff] = other[size_t(4 * t + s)];
    }
    V3 v[4];
    for (int i = 0; i < 4; ++i)
      v[i] = {coords[3 * int64_t(w[i])], coords[3 * int64_t(w[i]) + 1],
              coords[3 * int64_t(w[i]) + 2]};
    V3 c = v[0];
    for (int i = 1; i < 4; ++i) c = add(c, v[i]);
    const V3 cen = scale(1.0 / 4, c);
    double r2 = 0, d2 = 0;
    for (int i = 0; i < 4; ++i) {
      r2 = std::max(r2, dot(sub(v[i], cen), sub(v[i], cen)));
      for (int j = i + 1; j < 4; ++j) d2 = std::max(d2, dot(sub(v[i], v[j]), sub(v[i], v[j])));
    }
    center[3 * t] = cen.x;
    center[3 * t + 1] = cen.y;
    center[3 * t + 2] = cen.z;
    radius[t] = std::sqrt(r2);
    diam[t] = std::sqrt(d2);
    volume[t] = std::abs(dot(cross(sub(v[1], v[0]), sub(v[2], v[0])), sub(v[3], v[0]))) / 6.0;
    const V3 e1 = sub(v[1], v[0]), e2 = sub(v[2], v[0]), e3 = sub(v[3], v[0]);
    const double det = dot(e1, cross(e2, e3));
    if (det == 0) {
      put_err(err, errlen, "BadConfig: degenerate element " + std::to_string(t));
      return NLFEM_GPU_BAD_CONFIG;
    }
    const V3 r1 = cross(e2, e3), rr2 = cross(e3, e1), r3 = cross(e1, e2);
    double* inv = inv_edges + 9 * t;
    inv[0] = r1.x / det;
    inv[1] = r1.y / det;
    inv[2] = r1.z / det;
    inv[3] = rr2.x / det;
    inv[4] = rr2.y / det;
    inv[5] = rr2.z / det;
    inv[6] = r3.x / det;
    inv[7] = r3.y / det;
    inv[8] = r3.z / det;
  }
  return 0;
}

int32_t nlfem_host_dofmap(const int32_t* verts, const uint8_t* region, int64_t ncells,
                          int64_t nnodes, int32_t* dof_of_node, uint8_t* constrained) {
  std::fill(constrained, constrained + nnodes, uint8_t(0));
  for (int64_t t = 0; t < ncells; ++t)
    if (region[t])
      for (int i = 0; i < 4; ++i) constrained[verts[4 * t + i]] = 1;
  int32_t u = 0;
  for (int64_t v = 0; v < nnodes; ++v) dof_of_node[v] = constrained[v] ? -1 : u++;
  return u;
}

double nlfem_host_kernel_constant(double delta, int32_t moment2) {
  return kernel_C(delta, moment2 != 0);
}

int32_t nlfem_host_forcing(double delta, int32_t moment2, const double* uterms, int32_t nu,
                           double* fterms, int32_t maxterms) {
  const Poly u = poly_from_rows(uterms, nu);
  const double C = kernel_C(delta, moment2 != 0);
  const Poly f = pscale(-1.0, apply_L(u, delta, C));
  int32_t n = 0;
  for (const Term& t : f) {
    if (n >= maxterms) break;
    fterms[4 * n] = t.c;
    for (int a = 0; a < 3; ++a) fterms[4 * n + 1 + a] = t.e[a];
    ++n;
  }
  return n;
}

int32_t nlfem_host_normalize_poly(const double* terms, int32_t n, double* out,
                                  int32_t maxterms) {
  const Poly p = poly_from_rows(terms, n);
  int32_t m = 0;
  for (const Term& t : p) {
    if (m >= maxterms) break;
    out[4 * m] = t.c;
    for (int a = 0; a < 3; ++a) out[4 * m + 1 + a] = t.e[a];
    ++m;
  }
  return m;
}

}  // extern "C"
