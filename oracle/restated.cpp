// oracle/restated.cpp -- TEST INFRASTRUCTURE ONLY: a CPU restatement of the
// reference's assembly (proj/src/assembly.cpp:617-843 and the geometry it
// calls) with a pluggable Monte Carlo sampler.  Never linked into the product;
// only tests/, __graft_entry__.smoke() and bench.py's baseline legs load it.
//
//   sampler 1 ("R"): xoshiro256++ seeded by mix_seed(seed, T, q, piece_idx)
//     with the walk-order piece index (reference assembly.cpp:383-399,
//     core.hpp:100-133) -- reproduces the unmodified reference, which pins
//     this restatement (tests/test_oracle.py against oracle/_ref).
//   sampler 0 ("P"): the counter-based Philox stream of include/nlfem_mc_stream.h
//     (the one the GPU kernels draw), same regions and estimator.
//
// Arithmetic order follows the reference expression by expression and the
// file is compiled with -ffp-contract=off, so mode R agrees with the reference
// bit for bit; the block-of-32 accumulation with a fixed pairwise merge tree
// (assembly.cpp:80-160) is restated too, so results do not depend on threads.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "nlfem_mc_stream.h"

namespace orc {

struct V {
  double x = 0, y = 0, z = 0;
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
inline V operator+(V a, V b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V operator-(V a, V b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V operator*(double s, V a) { return {s * a.x, s * a.y, s * a.z}; }
inline double dot(V a, V b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V cross(V a, V b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double n2(V a) { return dot(a, a); }
inline double dist(V a, V b) { return std::sqrt(n2(a - b)); }

struct Tet {
  V v[4];
};

struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// degree-2 rule (reference quadrature.cpp:22-29)
const double QA = 0.5854101966249685, QB = 0.1381966011250105;
inline double qb(int k, int i) { return k == i ? QA : QB; }

struct Poly {
  std::vector<double> c;
  std::vector<std::array<int, 3>> e;
  double eval(V p) const {  // Polynomial::eval, reference polynomial.cpp:28-37
    double acc = 0;
    for (size_t t = 0; t < c.size(); ++t) {
      double v = c[t];
      for (int a = 0; a < 3; ++a)
        for (int i = 0; i < e[t][a]; ++i) v *= p[a];
      acc += v;
    }
    return acc;
  }
};

struct Mesh {
  int K = 0, J = 0;
  const double* node;
  const int32_t* verts;
  const int32_t* nbr;
  const double* center;
  const double* radius;
  const double* volume;
  const double* diam;
  const uint8_t* region;
  const double* inv;
  V vert(int t, int i) const {
    const int v = verts[4 * t + i];
    return {node[3 * v], node[3 * v + 1], node[3 * v + 2]};
  }
  Tet tet(int t) const { return {{vert(t, 0), vert(t, 1), vert(t, 2), vert(t, 3)}}; }
  V cen(int t) const { return {center[3 * t], center[3 * t + 1], center[3 * t + 2]}; }
  std::array<double, 4> bary(int t, V p) const {  // ball_approx.cpp:100-115
    const double* iv = inv + 9 * (int64_t)t;
    const V d = p - vert(t, 0);
    std::array<double, 4> o{};
    o[1] = iv[0] * d.x + iv[1] * d.y + iv[2] * d.z;
    o[2] = iv[3] * d.x + iv[4] * d.y + iv[5] * d.z;
    o[3] = iv[6] * d.x + iv[7] * d.y + iv[8] * d.z;
    o[0] = 1.0 - o[1] - o[2] - o[3];
    return o;
  }
};

// ---- geometry (reference geometry.cpp, ball_approx.cpp) -------------------------

double tvol(V a, V b, V c, V d) { return std::abs(dot(cross(b - a, c - a), d - a)) / 6.0; }

int in_mask(const Tet& s, V c, double r) {
  const double ri = r - 1e-10 * r;
  const double r2 = ri * ri;
  int m = 0;
  for (int i = 0; i < 4; ++i)
    if (n2(s.v[i] - c) < r2) m |= 1 << i;
  return m;
}

double crossing_t(V a, V b, V c, double r) {
  const V d = b - a, u = a - c;
  const double A = n2(d), B = dot(u, d), C = n2(u) - r * r;
  double disc = B * B - A * C;
  if (disc < 0) disc = 0;
  const double sq = std::sqrt(disc);
  const double t = (B <= 0) ? (-B + sq) / A : -C / (B + sq);
  return std::clamp(t, 0.0, 1.0);
}

int crossings(const Tet& s, int mask, V c, double r, V q[4]) {
  int n = 0;
  for (int i = 0; i < 4; ++i) {
    if (!(mask >> i & 1)) continue;
    for (int o = 0; o < 4; ++o) {
      if (mask >> o & 1) continue;
      const double t = crossing_t(s.v[i], s.v[o], c, r);
      q[n++] = s.v[i] + t * (s.v[o] - s.v[i]);
    }
  }
  return n;
}

void keep(std::vector<Tet>& out, V a, V b, V c, V d, double tau) {
  if (tvol(a, b, c, d) > tau) out.push_back({{a, b, c, d}});
}
void prism3(std::vector<Tet>& out, const V A[3], const V B[3], double tau) {
  keep(out, A[0], A[1], A[2], B[0], tau);
  keep(out, A[1], A[2], B[0], B[1], tau);
  keep(out, A[2], B[0], B[1], B[2], tau);
}
void warped3(std::vector<Tet>& out, const V A[3], const V B[3], double tau) {
  const double va = tvol(A[0], A[1], A[2], B[0]) + tvol(A[1], A[2], B[0], B[1]) +
                    tvol(A[2], B[0], B[1], B[2]);
  const double vb = tvol(A[0], A[2], A[1], B[0]) + tvol(A[2], A[1], B[0], B[2]) +
                    tvol(A[1], B[0], B[2], B[1]);
  if (vb > va) {
    const V A2[3] = {A[0], A[2], A[1]}, B2[3] = {B[0], B[2], B[1]};
    prism3(out, A2, B2, tau);
  } else {
    prism3(out, A, B, tau);
  }
}

void inner_pieces(const Tet& s, int mask, V c, double r, double tau, std::vector<Tet>& out) {
  out.clear();
  V q[4];
  crossings(s, mask, c, r, q);
  int in[4], m = 0;
  for (int i = 0; i < 4; ++i)
    if (mask >> i & 1) in[m++] = i;
  if (m == 1) {
    keep(out, s.v[in[0]], q[0], q[1], q[2], tau);
  } else if (m == 2) {
    const V A[3] = {s.v[in[0]], q[0], q[1]}, B[3] = {s.v[in[1]], q[2], q[3]};
    warped3(out, A, B, tau);
  } else {
    const V A[3] = {s.v[in[0]], s.v[in[1]], s.v[in[2]]}, B[3] = {q[0], q[1], q[2]};
    prism3(out, A, B, tau);
  }
}

// ---- approxcaps: inner polytope with sphere points, as a convex hull --------------
// Points (reference ball_approx.cpp:210-229): the inside vertices, the
// crossings, and per crossing pair sharing an inside or an outside endpoint the
// radial projection of their midpoint onto the sphere.  Incremental hull with
// the reference's seeds, eps tests and face order (geometry.cpp:198-298), fan
// from the centroid of the hull vertices (geometry.cpp:310-328), pieces above
// the volume floor (ball_approx.cpp:177-192).  Empty on a degenerate hull.
void approx_pieces(const Tet& s, int mask, V c, double r, double tau, std::vector<Tet>& out) {
  out.clear();
  V q[4];
  const int nq = crossings(s, mask, c, r, q);
  int qi[4], qo[4];
  {
    int k = 0;
    for (int i = 0; i < 4; ++i) {
      if (!(mask >> i & 1)) continue;
      for (int o = 0; o < 4; ++o)
        if (!(mask >> o & 1)) qi[k] = i, qo[k] = o, ++k;
    }
  }
  std::vector<V> pts;
  for (int i = 0; i < 4; ++i)
    if (mask >> i & 1) pts.push_back(s.v[i]);
  for (int k = 0; k < nq; ++k) pts.push_back(q[k]);
  for (int i = 0; i < nq; ++i)
    for (int j = i + 1; j < nq; ++j) {
      if (qi[i] != qi[j] && qo[i] != qo[j]) continue;
      const V mid = 0.5 * (q[i] + q[j]) - c;
      const double len = std::sqrt(n2(mid));
      if (len <= 0) continue;
      pts.push_back(c + (r / len) * mid);
    }
  const int n = int(pts.size());
  // hull3d
  V lo = pts[0], hi = pts[0];
  for (const V& p : pts) {
    lo = {std::min(lo.x, p.x), std::min(lo.y, p.y), std::min(lo.z, p.z)};
    hi = {std::max(hi.x, p.x), std::max(hi.y, p.y), std::max(hi.z, p.z)};
  }
  const double scale = std::max(std::sqrt(n2(hi - lo)), 1e-300);
  const double eps = 1e-12 * scale;
  int s0 = 0, s1 = -1, s2 = -1, s3 = -1;
  for (int i = 1; i < n; ++i)
    if (dist(pts[i], pts[s0]) > eps) {
      s1 = i;
      break;
    }
  if (s1 < 0) return;
  const V d01 = pts[s1] - pts[s0];
  for (int i = 0; i < n; ++i)
    if (std::sqrt(n2(cross(d01, pts[i] - pts[s0]))) / std::sqrt(n2(d01)) > eps) {
      s2 = i;
      break;
    }
  if (s2 < 0) return;
  const V nrm = cross(d01, pts[s2] - pts[s0]);
  for (int i = 0; i < n; ++i)
    if (std::abs(dot(nrm, pts[i] - pts[s0])) / std::sqrt(n2(nrm)) > eps) {
      s3 = i;
      break;
    }
  if (s3 < 0) return;
  if (dot(nrm, pts[s3] - pts[s0]) > 0) std::swap(s1, s2);
  using F = std::array<int, 3>;
  std::vector<F> faces{{s0, s2, s1}, {s0, s1, s3}, {s1, s2, s3}, {s0, s3, s2}};
  const V inner = 0.25 * (pts[s0] + pts[s1] + pts[s2] + pts[s3]);
  auto outward = [&](F& f) {
    const V nn = cross(pts[f[1]] - pts[f[0]], pts[f[2]] - pts[f[0]]);
    if (dot(nn, inner - pts[f[0]]) > 0) std::swap(f[1], f[2]);
  };
  for (auto& f : faces) outward(f);
  std::vector<char> used(n, 0), vis;
  used[s0] = used[s1] = used[s2] = used[s3] = 1;
  for (int pi = 0; pi < n; ++pi) {
    if (used[pi]) continue;
    used[pi] = 1;
    const V p = pts[pi];
    bool dup = false;
    for (const F& f : faces)
      for (int v : f)
        if (dist(p, pts[v]) <= eps) dup = true;
    if (dup) continue;
    vis.assign(faces.size(), 0);
    bool any = false;
    for (size_t fi = 0; fi < faces.size(); ++fi) {
      const F& f = faces[fi];
      const V nn = cross(pts[f[1]] - pts[f[0]], pts[f[2]] - pts[f[0]]);
      if (dot(nn, p - pts[f[0]]) > eps * std::sqrt(n2(nn))) vis[fi] = 1, any = true;
    }
    if (!any) continue;
    std::vector<std::array<int, 2>> horizon;
    for (size_t fi = 0; fi < faces.size(); ++fi) {
      if (!vis[fi]) continue;
      for (int e = 0; e < 3; ++e) {
        const int a = faces[fi][e], b = faces[fi][(e + 1) % 3];
        bool open = true;
        for (size_t fj = 0; fj < faces.size() && open; ++fj) {
          if (vis[fj]) continue;
          for (int e2 = 0; e2 < 3; ++e2)
            if (faces[fj][e2] == b && faces[fj][(e2 + 1) % 3] == a) open = false;
        }
        if (!open) horizon.push_back({a, b});
      }
    }
    std::vector<F> next;
    for (size_t fi = 0; fi < faces.size(); ++fi)
      if (!vis[fi]) next.push_back(faces[fi]);
    for (auto [a, b] : horizon) {
      F f{a, b, pi};
      outward(f);
      next.push_back(f);
    }
    faces.swap(next);
  }
  // triangulate_polytope: fan from the centroid of the distinct hull vertices
  std::vector<int> vs;
  for (const F& f : faces)
    for (int i = 0; i < 3; ++i) vs.push_back(f[i]);
  std::sort(vs.begin(), vs.end());
  vs.erase(std::unique(vs.begin(), vs.end()), vs.end());
  V cen{};
  for (int v : vs) cen = cen + pts[v];
  cen = (1.0 / double(vs.size())) * cen;
  for (const F& f : faces) keep(out, cen, pts[f[0]], pts[f[1]], pts[f[2]], tau);
}

void outer_pieces(const Tet& s, int mask, V c, double r, double tau, std::vector<Tet>& out) {
  out.clear();
  V q[4];
  crossings(s, mask, c, r, q);
  int os[4], m = 0, mo = 0;
  for (int i = 0; i < 4; ++i) {
    if (mask >> i & 1) ++m;
    else os[mo++] = i;
  }
  if (m == 1) {
    const V A[3] = {q[0], q[1], q[2]}, B[3] = {s.v[os[0]], s.v[os[1]], s.v[os[2]]};
    prism3(out, A, B, tau);
  } else if (m == 2) {
    const V A[3] = {s.v[os[0]], q[0], q[2]}, B[3] = {s.v[os[1]], q[1], q[3]};
    warped3(out, A, B, tau);
  } else {
    keep(out, s.v[os[0]], q[0], q[1], q[2], tau);
  }
}

double tri_dist(V p, V a, V b, V c) {  // geometry.cpp:98-127
  const V ab = b - a, ac = c - a, ap = p - a;
  const double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0 && d2 <= 0) return dist(p, a);
  const V bp = p - b;
  const double d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0 && d4 <= d3) return dist(p, b);
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) return dist(p, a + (d1 / (d1 - d3)) * ab);
  const V cp = p - c;
  const double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0 && d5 <= d6) return dist(p, c);
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) return dist(p, a + (d2 / (d2 - d6)) * ac);
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0)
    return dist(p, b + ((d4 - d3) / ((d4 - d3) + (d5 - d6))) * (c - b));
  const double den = 1.0 / (va + vb + vc);
  const double vv = vb * den, w = vc * den;
  return dist(p, a + vv * ab + w * ac);
}

double tet_dist(V p, const Tet& s) {  // geometry.cpp:129-144
  const V e1 = s.v[1] - s.v[0], e2 = s.v[2] - s.v[0], e3 = s.v[3] - s.v[0], b = p - s.v[0];
  const double det = dot(e1, cross(e2, e3));
  const double l1 = dot(b, cross(e2, e3)) / det;
  const double l2 = dot(e1, cross(b, e3)) / det;
  const double l3 = dot(e1, cross(e2, b)) / det;
  const double l0 = 1.0 - l1 - l2 - l3;
  if (!(l0 < 0) && !(l1 < 0) && !(l2 < 0) && !(l3 < 0)) return 0.0;
  double d = tri_dist(p, s.v[1], s.v[2], s.v[3]);
  d = std::min(d, tri_dist(p, s.v[0], s.v[2], s.v[3]));
  d = std::min(d, tri_dist(p, s.v[0], s.v[1], s.v[3]));
  return std::min(d, tri_dist(p, s.v[0], s.v[1], s.v[2]));
}

double face_dist(const Tet& s, int slot, V p) {
  V f[3];
  int k = 0;
  for (int i = 0; i < 4; ++i)
    if (i != slot) f[k++] = s.v[i];
  return tri_dist(p, f[0], f[1], f[2]);
}

V qpoint(const Tet& s, int k) {
  V p = qb(k, 0) * s.v[0];
  for (int i = 1; i < 4; ++i) p = p + qb(k, i) * s.v[i];
  return p;
}

// ---- samplers -------------------------------------------------------------------

uint64_t smix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
struct Xo {
  uint64_t s[4];
  explicit Xo(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s) w = x = smix(x);
  }
  static uint64_t rl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rl(s[3], 45);
    return r;
  }
  double u() { return double(next() >> 11) * 0x1.0p-53; }
};

// ---- accumulation: blocks of 32 outer elements, sorted runs, fixed merge tree -----

constexpr uint64_t kRhs = 0xFFFFFFFFull;
struct Ent {
  uint64_t key;
  double val;
};
using Run = std::vector<Ent>;

Run merge(const Run& a, const Run& b) {
  Run o;
  o.reserve(a.size() + b.size());
  size_t i = 0, j = 0;
  while (i < a.size() && j < b.size()) {
    if (a[i].key < b[j].key) o.push_back(a[i++]);
    else if (b[j].key < a[i].key) o.push_back(b[j++]);
    else {
      o.push_back({a[i].key, a[i].val + b[j].val});
      ++i, ++j;
    }
  }
  while (i < a.size()) o.push_back(a[i++]);
  while (j < b.size()) o.push_back(b[j++]);
  return o;
}

struct Job {
  Mesh m;
  const int32_t* dof;
  int unknowns;
  double C, delta;
  Poly f, g;
  int strategy;  // 0 inside, 1 overlap, 2 barycenter, 3 nocaps, 4 approxcaps, 5 fullcaps
  uint64_t seed;
  int M;
  int sampler;  // 0 Philox (P), 1 xoshiro walk order (R)
  std::vector<double> tau, gnode;
  std::vector<int> interior;
};

// Per-(outer element, quad point) piece sink with per-parent moment aggregation
// (reference AsmSink, assembly.cpp:257-473).
struct Acc {
  const Job& J;
  std::unordered_map<uint64_t, double> pm;  // block accumulator, key order irrelevant:
  std::vector<uint64_t> order;              // first-touch keys (sorted at block end)
  std::unordered_map<int, double> rh;
  uint64_t mc_done = 0, mc_hit = 0;
  // outer state
  int elemN = -1, q = 0;
  int nodeN[4], dofN[4];
  double wN = 0;
  V p;
  double cN[4];
  // parent state
  int cur = -1;
  bool ccon = false;
  double S0 = 0, Sg = 0, S1[4], S2[4][4];
  int piece = 0;
  std::vector<Tet> scratch;
  // element pairs (T, T') with a piece for some quad point of T
  std::vector<int> seen;
  uint64_t pairs = 0;

  explicit Acc(const Job& j) : J(j), seen(size_t(j.m.K), -1) {}
  void mark(int t) {
    if (seen[t] != elemN) {
      seen[t] = elemN;
      ++pairs;
    }
  }

  double& slot(uint64_t k) {
    auto it = pm.find(k);
    if (it == pm.end()) {
      order.push_back(k);
      return pm[k] = 0.0;
    }
    return it->second;
  }
  double& rhs(int d) { return rh[d]; }

  void pair(int da, int na, int db, int nb, double v) {  // add_pair, 401-411
    if (da >= 0 && db >= 0) {
      const uint64_t lo = uint64_t(std::min(da, db)), hi = uint64_t(std::max(da, db));
      slot((lo << 32) | hi) += v;
    } else if (da >= 0) {
      rhs(da) -= v * J.gnode[nb];
    } else if (db >= 0) {
      rhs(db) -= v * J.gnode[na];
    }
  }

  void open(int t) {
    mark(t);
    if (cur >= 0) close();
    cur = t;
    ccon = J.m.region[t] != 0;
    S0 = Sg = 0;
    for (int i = 0; i < 4; ++i) {
      S1[i] = 0;
      for (int k = 0; k < 4; ++k) S2[i][k] = 0;
    }
  }

  void point(V y, double w) {  // accumulate_point, 332-344
    S0 += w;
    if (ccon) {
      Sg += w * J.g.eval(y);
      return;
    }
    const auto b = J.m.bary(cur, y);
    for (int i = 0; i < 4; ++i) {
      const double wb = w * b[i];
      S1[i] += wb;
      for (int k = 0; k < 4; ++k) S2[i][k] += wb * b[k];
    }
  }

  void whole(int t) {  // 346-370
    if (t != cur) open(t);
    ++piece;
    const double vol = J.m.volume[t];
    if (ccon) {
      S0 += vol;
      const Tet s = J.m.tet(t);
      for (int k = 0; k < 4; ++k) Sg += vol * 0.25 * J.g.eval(qpoint(s, k));
      return;
    }
    S0 += vol;
    const double s1 = vol / 4, off = vol / double(20);
    for (int i = 0; i < 4; ++i) {
      S1[i] += s1;
      for (int k = 0; k < 4; ++k) S2[i][k] += off * (i == k ? 2.0 : 1.0);
    }
  }

  void sub(int t, const Tet& s) {  // 372-381
    if (t != cur) open(t);
    ++piece;
    const double vol = tvol(s.v[0], s.v[1], s.v[2], s.v[3]);
    for (int k = 0; k < 4; ++k) point(qpoint(s, k), vol * 0.25);
  }

  void cap(int t, const std::vector<Tet>& outer) {  // 383-399 (sampler pluggable)
    if (t != cur) open(t);
    ++piece;
    const double r2 = J.delta * J.delta;
    if (J.sampler == 1) {
      uint64_t h = smix(J.seed ^ 0x243f6a8885a308d3ull);
      h = smix(h ^ uint64_t(elemN));
      h = smix(h ^ uint64_t(q));
      Xo rng(smix(h ^ uint64_t(piece)));
      for (const Tet& s : outer) {
        const double w = tvol(s.v[0], s.v[1], s.v[2], s.v[3]) / J.M;
        for (int k = 0; k < J.M; ++k) {
          double u[3] = {rng.u(), rng.u(), rng.u()};  // sample_simplex, quadrature.cpp:94-108
          if (u[0] > u[1]) std::swap(u[0], u[1]);
          if (u[1] > u[2]) std::swap(u[1], u[2]);
          if (u[0] > u[1]) std::swap(u[0], u[1]);
          const double l0 = u[0], l1 = u[1] - u[0], l2 = u[2] - u[1], l3 = 1.0 - u[2];
          const V y = l0 * s.v[0] + l1 * s.v[1] + l2 * s.v[2] + l3 * s.v[3];
          ++mc_done;
          if (n2(y - p) >= r2) continue;
          ++mc_hit;
          point(y, w);
        }
      }
      return;
    }
    // mode P: include/nlfem_mc_stream.h
    const double xq[3] = {p.x, p.y, p.z};
    for (size_t sb = 0; sb < outer.size(); ++sb) {
      const Tet& s = outer[sb];
      const double w = tvol(s.v[0], s.v[1], s.v[2], s.v[3]) / J.M;
      const double v0[3] = {s.v[0].x, s.v[0].y, s.v[0].z}, v1[3] = {s.v[1].x, s.v[1].y, s.v[1].z},
                   v2[3] = {s.v[2].x, s.v[2].y, s.v[2].z}, v3[3] = {s.v[3].x, s.v[3].y, s.v[3].z};
      nlfem_mc_quad Q;
      nlfem_mc_make_quad(v0, v1, v2, v3, xq, &Q);
      uint32_t W[8];
      for (int k = 0; k < J.M; ++k) {
        if (k % 4 == 0)
          nlfem_mc_block(J.seed, uint32_t(elemN), uint32_t(t), uint32_t(q), uint32_t(sb),
                         uint32_t(k / 4), W);
        double d[3], r[3];
        ++mc_done;
        if (!nlfem_mc_sample(W, k % 4, &Q, r2, d)) continue;
        ++mc_hit;
        nlfem_mc_r(&Q, d[0], d[1], d[2], r);
        point({p.x + r[0], p.y + r[1], p.z + r[2]}, w);
      }
    }
  }

  void close() {  // flush, 413-473
    const int Mx = cur;
    const double C = J.C;
    if (ccon) {
      const double base = wN * 2.0 * C;
      for (int a = 0; a < 4; ++a) {
        if (dofN[a] >= 0) rhs(dofN[a]) += base * Sg * cN[a];
        for (int b = a; b < 4; ++b) pair(dofN[a], nodeN[a], dofN[b], nodeN[b], base * S0 * cN[a] * cN[b]);
      }
      cur = -1;
      return;
    }
    struct U {
      int node, dof;
      double c;
      int ms;
    } u[8];
    int n = 0;
    const int32_t* vm = J.m.verts + 4 * Mx;
    for (int a = 0; a < 4; ++a) {
      int ms = -1;
      for (int j = 0; j < 4; ++j)
        if (vm[j] == nodeN[a]) {
          ms = j;
          break;
        }
      u[n++] = {nodeN[a], dofN[a], cN[a], ms};
    }
    for (int j = 0; j < 4; ++j) {
      bool shared = false;
      for (int a = 0; a < 4; ++a)
        if (nodeN[a] == vm[j]) shared = true;
      if (!shared) u[n++] = {vm[j], J.dof[vm[j]], 0.0, j};
    }
    const double sc = C * wN;
    for (int x = 0; x < n; ++x) {
      const double s1x = u[x].ms >= 0 ? S1[u[x].ms] : 0.0;
      for (int y = x; y < n; ++y) {
        const double s1y = u[y].ms >= 0 ? S1[u[y].ms] : 0.0;
        const double s2 = (u[x].ms >= 0 && u[y].ms >= 0) ? S2[u[x].ms][u[y].ms] : 0.0;
        pair(u[x].dof, u[x].node, u[y].dof, u[y].node,
             sc * (s2 - u[x].c * s1y - u[y].c * s1x + u[x].c * u[y].c * S0));
      }
    }
    cur = -1;
  }

  // core_whole, 479-549 (rW sums of the outer rule)
  void core(int t, double rW0, const double* rWA, const double (*rWAB)[4], double volN) {
    mark(t);
    const double C = J.C;
    const double vol = J.m.volume[t];
    if (J.m.region[t]) {
      double sg = 0;
      const Tet s = J.m.tet(t);
      for (int k = 0; k < 4; ++k) sg += vol * 0.25 * J.g.eval(qpoint(s, k));
      const double base = 2.0 * C * volN;
      for (int a = 0; a < 4; ++a) {
        if (dofN[a] >= 0) rhs(dofN[a]) += base * rWA[a] * sg;
        for (int b = a; b < 4; ++b) pair(dofN[a], nodeN[a], dofN[b], nodeN[b], base * rWAB[a][b] * vol);
      }
      return;
    }
    const double s1 = vol / 4, off = vol / double(20);
    struct U {
      int node, dof, ms, ns;
    } u[8];
    int n = 0;
    const int32_t* vm = J.m.verts + 4 * t;
    for (int a = 0; a < 4; ++a) {
      int ms = -1;
      for (int j = 0; j < 4; ++j)
        if (vm[j] == nodeN[a]) {
          ms = j;
          break;
        }
      u[n++] = {nodeN[a], dofN[a], ms, a};
    }
    for (int j = 0; j < 4; ++j) {
      bool shared = false;
      for (int a = 0; a < 4; ++a)
        if (nodeN[a] == vm[j]) shared = true;
      if (!shared) u[n++] = {vm[j], J.dof[vm[j]], j, -1};
    }
    const double sc = C * volN;
    for (int x = 0; x < n; ++x) {
      const double s1x = u[x].ms >= 0 ? s1 : 0.0;
      const double wax = u[x].ns >= 0 ? rWA[u[x].ns] : 0.0;
      for (int y = x; y < n; ++y) {
        const double s1y = u[y].ms >= 0 ? s1 : 0.0;
        const double way = u[y].ns >= 0 ? rWA[u[y].ns] : 0.0;
        const double s2 = (u[x].ms >= 0 && u[y].ms >= 0) ? off * (u[x].ms == u[y].ms ? 2.0 : 1.0) : 0.0;
        const double wab = (u[x].ns >= 0 && u[y].ns >= 0) ? rWAB[u[x].ns][u[y].ns] : 0.0;
        pair(u[x].dof, u[x].node, u[y].dof, u[y].node,
             sc * (rW0 * s2 - wax * s1y - way * s1x + wab * vol));
      }
    }
  }
};

// collect_candidates: BFS with radius delta + spread (reference assembly.cpp:569-613)
struct Cand {
  std::vector<int> core, rest, bnd;
};
void candidates(const Mesh& m, std::vector<uint32_t>& stamp, uint32_t& epoch, int seed, V cN,
                const V* qp, double delta, Cand& out) {
  double spread = 0;
  for (int k = 0; k < 4; ++k) spread = std::max(spread, dist(qp[k], cN));
  const double R = delta + spread;
  const double cut = delta - 1e-10 * delta - 1e-12 * delta - spread;
  out.core.clear();
  out.rest.clear();
  out.bnd.clear();
  ++epoch;
  std::vector<int> queue{seed};
  std::vector<double> gaps{dist(m.cen(seed), cN)};
  stamp[seed] = epoch;
  for (size_t qi = 0; qi < queue.size(); ++qi) {
    const int t = queue[qi];
    for (int f = 0; f < 4; ++f)
      if (m.nbr[4 * t + f] < 0) {
        out.bnd.push_back(t);
        break;
      }
    if (gaps[qi] + m.radius[t] < cut) out.core.push_back(t);
    else out.rest.push_back(t);
    for (int f = 0; f < 4; ++f) {
      const int nb = m.nbr[4 * t + f];
      if (nb < 0 || stamp[nb] == epoch) continue;
      stamp[nb] = epoch;
      const double gap = dist(m.cen(nb), cN);
      if (gap >= m.radius[nb] + R) continue;
      if (gap + m.radius[nb] >= R && tet_dist(cN, m.tet(nb)) >= R) continue;
      queue.push_back(nb);
      gaps.push_back(gap);
    }
  }
}

struct Result {
  std::vector<int32_t> row_ptr, col_idx;
  std::vector<double> values, rhs;
  uint64_t mc_done = 0, mc_hit = 0, pairs = 0;
  int blocks = 0, threads = 1;
  double seconds = 0;
};

Run do_block(const Job& J, int b, std::vector<uint32_t>& stamp, uint32_t& epoch, uint64_t& md,
             uint64_t& mh, uint64_t& np) {
  const Mesh& m = J.m;
  double rW0 = 0, rWA[4] = {0, 0, 0, 0}, rWAB[4][4] = {};
  for (int k = 0; k < 4; ++k) {  // assembly.cpp:636-648
    rW0 += 0.25;
    for (int a = 0; a < 4; ++a) {
      rWA[a] += 0.25 * qb(k, a);
      for (int c = 0; c < 4; ++c) rWAB[a][c] += 0.25 * qb(k, a) * qb(k, c);
    }
  }
  const double delta = J.delta;
  const double slack = 1e-10 * delta;
  const double icut = delta - slack - 1e-12 * delta;
  Acc A(J);
  Cand cand;
  const size_t lo = size_t(b) * 32, hi = std::min(lo + 32, J.interior.size());
  for (size_t e = lo; e < hi; ++e) {
    const int T = J.interior[e];
    const Tet s = m.tet(T);
    const double vol = m.volume[T];
    V qp[4];
    for (int k = 0; k < 4; ++k) qp[k] = qpoint(s, k);
    A.elemN = T;
    for (int a = 0; a < 4; ++a) {
      A.nodeN[a] = m.verts[4 * T + a];
      A.dofN[a] = J.dof[A.nodeN[a]];
    }
    candidates(m, stamp, epoch, T, m.cen(T), qp, delta, cand);
    for (int t : cand.core) A.core(t, rW0, rWA, rWAB, vol);
    for (int k = 0; k < 4; ++k) {
      const V p = qp[k];
      const double w = 0.25 * vol;
      const double fv = J.f.eval(p);
      A.q = k;
      A.wN = w;
      A.p = p;
      for (int a = 0; a < 4; ++a) A.cN[a] = qb(k, a);
      A.cur = -1;
      A.piece = 0;
      for (int a = 0; a < 4; ++a)
        if (A.dofN[a] >= 0) A.rhs(A.dofN[a]) += w * A.cN[a] * fv;
      for (int t : cand.bnd) {
        const Tet st = m.tet(t);
        for (int f = 0; f < 4; ++f)
          if (m.nbr[4 * t + f] < 0 && face_dist(st, f, p) < delta - slack)
            throw Err(5, "BallExitsMesh: ball reaches past an unglued facet of element " +
                             std::to_string(t));
      }
      for (int t : cand.rest) {
        const V ct = m.cen(t);
        const double gap = dist(ct, p);
        if (gap >= m.radius[t] + delta) continue;
        if (J.strategy == 2) {  // barycenter, assembly.cpp:725-727
          if (gap < delta) A.whole(t);
          continue;
        }
        if (J.strategy == 1) {  // overlap, assembly.cpp:728-733
          if (gap + m.radius[t] < delta || tet_dist(p, m.tet(t)) < delta) A.whole(t);
          continue;
        }
        if (gap + m.radius[t] < icut) {
          A.whole(t);
          continue;
        }
        const Tet st = m.tet(t);
        const int mask = in_mask(st, p, delta);
        if (mask == 15) {
          A.whole(t);
        } else if (mask != 0) {
          if (J.strategy == 0) continue;  // inside: straddlers dropped, assembly.cpp:744
          if (J.strategy == 4)  // approxcaps: straddle_inner with sphere points
            approx_pieces(st, mask, p, delta, J.tau[t], A.scratch);
          else
            inner_pieces(st, mask, p, delta, J.tau[t], A.scratch);
          for (const Tet& sb : A.scratch) A.sub(t, sb);
          if (J.strategy == 5) {
            outer_pieces(st, mask, p, delta, J.tau[t], A.scratch);
            if (!A.scratch.empty()) {
              const std::vector<Tet> outer = A.scratch;
              A.cap(t, outer);
            }
          }
        } else if (J.strategy == 5 && tet_dist(p, st) < delta) {
          A.cap(t, std::vector<Tet>{st});
        }
      }
      if (A.cur >= 0) A.close();
    }
  }
  md += A.mc_done;
  mh += A.mc_hit;
  np += A.pairs;
  Run run;
  run.reserve(A.order.size() + A.rh.size());
  for (uint64_t k : A.order) run.push_back({k, A.pm[k]});
  for (auto& kv : A.rh) run.push_back({(uint64_t(uint32_t(kv.first)) << 32) | kRhs, kv.second});
  std::sort(run.begin(), run.end(), [](const Ent& a, const Ent& b) { return a.key < b.key; });
  return run;
}

Result assemble(const Job& J, int threads) {
  Result R;
  const int nb = int((J.interior.size() + 31) / 32);
  R.blocks = nb;
  std::vector<Run> runs(std::max(nb, 1));
  std::atomic<int> next{0};
  std::atomic<uint64_t> md{0}, mh{0}, npairs{0};
  std::mutex emu;
  int ecode = 0;
  std::string emsg;
  auto work = [&]() {
    std::vector<uint32_t> stamp(J.m.K, 0);
    uint32_t epoch = 0;
    uint64_t a = 0, b = 0, c = 0;
    while (true) {
      const int k = next.fetch_add(1);
      if (k >= nb) break;
      try {
        runs[k] = do_block(J, k, stamp, epoch, a, b, c);
      } catch (const Err& e) {
        std::lock_guard<std::mutex> lk(emu);
        if (!ecode) {
          ecode = e.code;
          emsg = e.what();
        }
        next = nb;
      }
    }
    md += a;
    mh += b;
    npairs += c;
  };
  const int T = std::max(1, std::min(threads, std::max(nb, 1)));
  R.threads = T;
  std::vector<std::thread> pool;
  for (int i = 1; i < T; ++i) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (ecode) throw Err(ecode, emsg);
  // fixed pairwise merge tree over block indices (reference assembly.cpp:114-160)
  while (runs.size() > 1) {
    std::vector<Run> up((runs.size() + 1) / 2);
    for (size_t i = 0; i < up.size(); ++i)
      up[i] = (2 * i + 1 < runs.size()) ? merge(runs[2 * i], runs[2 * i + 1]) : std::move(runs[2 * i]);
    runs.swap(up);
  }
  const Run& run = runs[0];
  // upper-triangle run -> full CSR (reference assembly.cpp:789-833)
  const int U = J.unknowns;
  R.rhs.assign(U, 0.0);
  std::vector<int32_t> deg(U, 0), lower(U, 0);
  for (const Ent& e : run) {
    const int r = int(e.key >> 32);
    const uint64_t c = e.key & 0xFFFFFFFFull;
    if (c == kRhs) {
      R.rhs[r] += e.val;
      continue;
    }
    ++deg[r];
    if (int(c) != r) {
      ++deg[c];
      ++lower[c];
    }
  }
  R.row_ptr.assign(U + 1, 0);
  for (int r = 0; r < U; ++r) R.row_ptr[r + 1] = R.row_ptr[r] + deg[r];
  R.col_idx.assign(R.row_ptr.back(), 0);
  R.values.assign(R.row_ptr.back(), 0.0);
  std::vector<int32_t> up(U), lc(U);
  for (int r = 0; r < U; ++r) {
    lc[r] = R.row_ptr[r];
    up[r] = R.row_ptr[r] + lower[r];
  }
  for (const Ent& e : run) {
    const int r = int(e.key >> 32);
    const uint64_t c = e.key & 0xFFFFFFFFull;
    if (c == kRhs) continue;
    R.col_idx[up[r]] = int(c);
    R.values[up[r]] = e.val;
    ++up[r];
    if (int(c) != r) {
      R.col_idx[lc[c]] = r;
      R.values[lc[c]] = e.val;
      ++lc[c];
    }
  }
  R.mc_done = md;
  R.mc_hit = mh;
  R.pairs = npairs;
  return R;
}

Poly make_poly(const double* t, int n) {
  Poly p;
  for (int i = 0; i < n; ++i) {
    p.c.push_back(t[4 * i]);
    p.e.push_back({int(t[4 * i + 1]), int(t[4 * i + 2]), int(t[4 * i + 3])});
  }
  return p;
}

}  // namespace orc

extern "C" {

void* oracle_assemble(int K, int Jn, const double* node, const int32_t* verts,
                      const int32_t* nbr, const double* center, const double* radius,
                      const double* volume, const double* diam, const uint8_t* region,
                      const double* inv, const int32_t* dof_of_node, int unknowns, double C,
                      double delta, const double* fterms, int nf, const double* gterms, int ng,
                      int strategy, uint64_t seed, int M, int sampler, int threads,
                      const int32_t* outer, int64_t n_outer, int* code, char* err, int errlen) {
  // outer != NULL: integrate only these outer elements (interior ids, in the
  // given order) -- a partial system for sampled parity at full mesh sizes;
  // NULL: every interior element, as assembly.cpp:624-627
  using namespace orc;
  *code = 0;
  try {
    if (!(delta > 0)) throw Err(8, "BadConfig: delta must be positive");
    if (M <= 0) throw Err(8, "BadConfig: mc_samples must be positive");
    if (strategy < 0 || strategy > 5) throw Err(8, "BadConfig: unknown strategy");
    Job J{Mesh{K, Jn, node, verts, nbr, center, radius, volume, diam, region, inv},
          dof_of_node, unknowns, C, delta, make_poly(fterms, nf), make_poly(gterms, ng),
          strategy, seed, M, sampler, {}, {}, {}};
    J.tau.resize(K);
    for (int t = 0; t < K; ++t) {
      J.tau[t] = 1e-14 * std::pow(diam[t], 3);
      if (!region[t] && !outer) J.interior.push_back(t);
    }
    if (outer)
      for (int64_t i = 0; i < n_outer; ++i) {
        if (outer[i] < 0 || outer[i] >= K || region[outer[i]])
          throw Err(8, "BadConfig: outer element is not interior");
        J.interior.push_back(outer[i]);
      }
    J.gnode.assign(Jn, 0.0);
    for (int v = 0; v < Jn; ++v)
      if (dof_of_node[v] < 0) J.gnode[v] = J.g.eval({node[3 * v], node[3 * v + 1], node[3 * v + 2]});
    auto* R = new Result(assemble(J, threads));
    return R;
  } catch (const orc::Err& e) {
    *code = e.code;
    std::strncpy(err, e.what(), size_t(errlen - 1));
    err[errlen - 1] = 0;
    return nullptr;
  }
}

void oracle_result_sizes(void* h, int64_t* rows, int64_t* nnz) {
  auto* R = static_cast<orc::Result*>(h);
  *rows = int64_t(R->rhs.size());
  *nnz = int64_t(R->values.size());
}

void oracle_result_copy(void* h, int32_t* rp, int32_t* ci, double* v, double* rhs) {
  auto* R = static_cast<orc::Result*>(h);
  std::memcpy(rp, R->row_ptr.data(), R->row_ptr.size() * 4);
  std::memcpy(ci, R->col_idx.data(), R->col_idx.size() * 4);
  std::memcpy(v, R->values.data(), R->values.size() * 8);
  std::memcpy(rhs, R->rhs.data(), R->rhs.size() * 8);
}

void oracle_result_stats(void* h, uint64_t* md, uint64_t* mh, int32_t* blocks,
                         uint64_t* pairs) {
  auto* R = static_cast<orc::Result*>(h);
  *md = R->mc_done;
  *mh = R->mc_hit;
  *blocks = R->blocks;
  *pairs = R->pairs;
}

void oracle_result_free(void* h) { delete static_cast<orc::Result*>(h); }

// Philox4x32-10 known-answer helper for the tests.
void oracle_philox(const uint32_t ctr[4], uint32_t k0, uint32_t k1, uint32_t out[4]) {
  nlfem_philox4x32_10(ctr, k0, k1, out);
}

// The unsorted 21-bit fields (3 per sample, 4 samples per block) of sample
// blocks j0 .. j0 + nblocks - 1 of sub-simplex `sub` of item (T, q, T') of the
// 3D Monte Carlo stream (include/nlfem_mc_stream.h), for the stream tests.
void oracle_mc_fields(uint64_t seed, uint32_t T, uint32_t Tp, uint32_t q, uint32_t sub,
                      uint32_t j0, int nblocks, uint32_t* out) {
  for (int b = 0; b < nblocks; ++b) {
    uint32_t W[8];
    nlfem_mc_block(seed, T, Tp, q, sub, j0 + uint32_t(b), W);
    for (int i = 0; i < 4; ++i) nlfem_mc_fields(W, i, out + 12 * b + 3 * i);
  }
}

// Plain CG from zero (reference solver.cpp:26-66).
int oracle_cg(int n, const int32_t* rp, const int32_t* ci, const double* v, const double* b,
              double tol, int maxit, double* x, int32_t* iters) {
  std::vector<double> r(b, b + n), p(b, b + n), Ap(n);
  std::fill(x, x + n, 0.0);
  auto dotv = [&](const std::vector<double>& a, const std::vector<double>& c) {
    double s = 0;
    for (int i = 0; i < n; ++i) s += a[i] * c[i];
    return s;
  };
  double bb = 0;
  for (int i = 0; i < n; ++i) bb += b[i] * b[i];
  const double bn = std::sqrt(bb);
  *iters = 0;
  if (bn == 0) return 0;
  double rr = dotv(r, r);
  for (int it = 0; it < maxit; ++it) {
    if (std::sqrt(rr) <= tol * bn) return 0;
    for (int i = 0; i < n; ++i) {
      double s = 0;
      for (int k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * p[ci[k]];
      Ap[i] = s;
    }
    const double alpha = rr / dotv(p, Ap);
    for (int i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * Ap[i];
    }
    const double rr2 = dotv(r, r);
    const double beta = rr2 / rr;
    rr = rr2;
    for (int i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
    *iters = it + 1;
  }
  return std::sqrt(rr) <= tol * bn ? 0 : 1;
}

// L2 error of the P1 field with the 14-point degree-5 rule (reference
// study.cpp:76-99, quadrature.cpp:42-62).
double oracle_l2_error(int K, const double* node, const int32_t* verts, const uint8_t* region,
                       const double* volume, const double* node_vals, const double* uterms,
                       int nu) {
  using namespace orc;
  const Poly u = make_poly(uterms, nu);
  double bary[14][4], w[14];
  const double a = 0.3108859192633005, wa = 0.1126879257180162;
  const double b = 0.0927352503108912, wb = 0.0734930431163619;
  const double c = 0.0455037041256497, d = 0.5 - c, wc = 0.0425460207770812;
  const double a4 = 1.0 - 3.0 * a, b4 = 1.0 - 3.0 * b;
  const double rows[14][5] = {{a4, a, a, a, wa}, {a, a4, a, a, wa}, {a, a, a4, a, wa},
                              {a, a, a, a4, wa}, {b4, b, b, b, wb}, {b, b4, b, b, wb},
                              {b, b, b4, b, wb}, {b, b, b, b4, wb}, {c, c, d, d, wc},
                              {c, d, c, d, wc}, {c, d, d, c, wc}, {d, c, c, d, wc},
                              {d, c, d, c, wc}, {d, d, c, c, wc}};
  for (int q = 0; q < 14; ++q) {
    for (int i = 0; i < 4; ++i) bary[q][i] = rows[q][i];
    w[q] = rows[q][4];
  }
  double acc = 0;
  for (int t = 0; t < K; ++t) {
    if (region[t]) continue;
    for (int q = 0; q < 14; ++q) {
      V p{};
      double uh = 0;
      for (int i = 0; i < 4; ++i) {
        const int v = verts[4 * t + i];
        p = p + bary[q][i] * V{node[3 * v], node[3 * v + 1], node[3 * v + 2]};
        uh += bary[q][i] * node_vals[v];
      }
      const double e = uh - u.eval(p);
      acc += volume[t] * w[q] * e * e;
    }
  }
  return std::sqrt(acc);
}

}  // extern "C"
