// geom.cuh -- device restatement of the reference's simplex/ball geometry.
//
// Every function keeps the reference's operation order; the translation unit
// is compiled with -fmad=false so nvcc cannot contract a*b+c into DFMA.  With
// IEEE +,-,*,/,sqrt on both sides the results are bit-identical to the
// reference's (x86-64, FMA-free) binary, which is what makes the element-pair
// sets, the straddle sub-simplices and hence the sparsity pattern bit-exact.
#pragma once
#include <cstdint>

struct Vd {
  double x, y, z;
};

__device__ __forceinline__ Vd vsub(Vd a, Vd b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ Vd vadd(Vd a, Vd b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ Vd vscale(double s, Vd a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double vdot(Vd a, Vd b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ Vd vcross(Vd a, Vd b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double vnorm2(Vd a) { return vdot(a, a); }
__device__ __forceinline__ double vdist(Vd a, Vd b) { return sqrt(vnorm2(vsub(a, b))); }

// Outer/inner degree-2 tetrahedral rule (reference quadrature.cpp:22-29).
#define NLFEM_QA 0.5854101966249685
#define NLFEM_QB 0.1381966011250105
__device__ __forceinline__ double qbary(int k, int i) { return k == i ? NLFEM_QA : NLFEM_QB; }

// Quadrature point: p = b0*v0; p = p + b_i*v_i (reference assembly.cpp:689-694).
__device__ __forceinline__ Vd quad_point(const Vd v[4], int k) {
  Vd p = vscale(qbary(k, 0), v[0]);
  for (int i = 1; i < 4; ++i) p = vadd(p, vscale(qbary(k, i), v[i]));
  return p;
}

// simplex_volume (reference geometry.cpp:59-62); tet_volume (ball_approx.cpp:144-146).
__device__ __forceinline__ double tet_volume(Vd a, Vd b, Vd c, Vd d) {
  return fabs(vdot(vcross(vsub(b, a), vsub(c, a)), vsub(d, a))) / 6.0;
}

// edge_sphere_crossing (reference geometry.cpp:26-37).
__device__ __forceinline__ double edge_crossing(Vd a, Vd b, Vd c, double r) {
  const Vd d = vsub(b, a);
  const Vd u = vsub(a, c);
  const double A = vnorm2(d);
  const double B = vdot(u, d);
  const double C = vnorm2(u) - r * r;
  double disc = B * B - A * C;
  if (disc < 0) disc = 0;
  const double sq = sqrt(disc);
  double t = (B <= 0) ? (-B + sq) / A : -C / (B + sq);
  return t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
}

// point_triangle_distance, Ericson's region walk (reference geometry.cpp:98-127).
__device__ __forceinline__ double point_triangle_distance(Vd p, Vd a, Vd b, Vd c) {
  const Vd ab = vsub(b, a), ac = vsub(c, a), ap = vsub(p, a);
  const double d1 = vdot(ab, ap), d2 = vdot(ac, ap);
  if (d1 <= 0 && d2 <= 0) return vdist(p, a);
  const Vd bp = vsub(p, b);
  const double d3 = vdot(ab, bp), d4 = vdot(ac, bp);
  if (d3 >= 0 && d4 <= d3) return vdist(p, b);
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    const double t = d1 / (d1 - d3);
    return vdist(p, vadd(a, vscale(t, ab)));
  }
  const Vd cp = vsub(p, c);
  const double d5 = vdot(ab, cp), d6 = vdot(ac, cp);
  if (d6 >= 0 && d5 <= d6) return vdist(p, c);
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    const double t = d2 / (d2 - d6);
    return vdist(p, vadd(a, vscale(t, ac)));
  }
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    const double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return vdist(p, vadd(b, vscale(t, vsub(c, b))));
  }
  const double denom = 1.0 / (va + vb + vc);
  const double vv = vb * denom, w = vc * denom;
  return vdist(p, vadd(vadd(a, vscale(vv, ab)), vscale(w, ac)));
}

// distance_point_simplex (reference geometry.cpp:64-82, 129-144).
__device__ __forceinline__ double distance_point_simplex(Vd p, const Vd v[4]) {
  const Vd e1 = vsub(v[1], v[0]), e2 = vsub(v[2], v[0]), e3 = vsub(v[3], v[0]);
  const Vd b = vsub(p, v[0]);
  const double det = vdot(e1, vcross(e2, e3));
  const double l1 = vdot(b, vcross(e2, e3)) / det;
  const double l2 = vdot(e1, vcross(b, e3)) / det;
  const double l3 = vdot(e1, vcross(e2, b)) / det;
  const double l0 = 1.0 - l1 - l2 - l3;
  if (!(l0 < 0) && !(l1 < 0) && !(l2 < 0) && !(l3 < 0)) return 0.0;
  double d = point_triangle_distance(p, v[1], v[2], v[3]);
  d = fmin(d, point_triangle_distance(p, v[0], v[2], v[3]));
  d = fmin(d, point_triangle_distance(p, v[0], v[1], v[3]));
  return fmin(d, point_triangle_distance(p, v[0], v[1], v[2]));
}

// detail::facet_distance (reference ball_approx.cpp:122-131).
__device__ __forceinline__ double facet_distance(const Vd v[4], int slot, Vd p) {
  Vd f[3];
  int k = 0;
  for (int i = 0; i < 4; ++i)
    if (i != slot) f[k++] = v[i];
  return point_triangle_distance(p, f[0], f[1], f[2]);
}

// ---------------------------------------------------------------------------
// Compact form of the straddle decompositions.  Both straddle_inner and
// straddle_outer emit either one tet (A0, A1, A2, B0) or the three-tet split of
// a prism (A0 A1 A2 | B0 B1 B2): (A0,A1,A2,B0), (A1,A2,B0,B1), (A2,B0,B1,B2)
// (reference ball_approx.cpp:150-155); a warped prism first picks the
// orientation with the larger total volume (160-175).  Holding the six points
// and selecting piece k with conditional moves keeps one copy of the consumer
// code in the instruction stream; results are bit-identical to the reference
// because every point and volume is computed by the same expressions.
struct Straddle {
  Vd A0, A1, A2, B0, B1, B2;
  int n;  // 1 (single tet) or 3 (prism split)
};

__device__ __forceinline__ Vd pick(const Vd v[4], int i) {
  return i == 0 ? v[0] : (i == 1 ? v[1] : (i == 2 ? v[2] : v[3]));
}

__device__ __forceinline__ void orient_warped(Straddle& s) {
  const double va = tet_volume(s.A0, s.A1, s.A2, s.B0) + tet_volume(s.A1, s.A2, s.B0, s.B1) +
                    tet_volume(s.A2, s.B0, s.B1, s.B2);
  const double vb = tet_volume(s.A0, s.A2, s.A1, s.B0) + tet_volume(s.A2, s.A1, s.B0, s.B2) +
                    tet_volume(s.A1, s.B0, s.B2, s.B1);
  if (vb > va) {
    const Vd t = s.A1;
    s.A1 = s.A2;
    s.A2 = t;
    const Vd u = s.B1;
    s.B1 = s.B2;
    s.B2 = u;
  }
}

// position of the r-th set bit (r = 0..3) of a 4-bit mask: a 2-bit table
// lookup (__fns is emulated with a loop on sm_100)
__host__ __device__ constexpr unsigned long long nth_bit_table(int half) {
  unsigned long long t = 0;
  for (int m = 8 * half; m < 8 * half + 8; ++m)
    for (int r = 0; r < 4; ++r) {
      int cnt = 0, pos = 0;
      for (int b = 0; b < 4; ++b)
        if (m >> b & 1) {
          if (cnt == r) pos = b;
          ++cnt;
        }
      t |= (unsigned long long)pos << (2 * ((m - 8 * half) * 4 + r));
    }
  return t;
}
constexpr unsigned long long kNthBit0 = nth_bit_table(0), kNthBit1 = nth_bit_table(1);
__device__ __forceinline__ int nth_bit4(unsigned mask, int r) {
  const unsigned long long t = mask < 8 ? kNthBit0 : kNthBit1;
  return (int)((t >> (2 * (((mask & 7u) << 2) | (unsigned)r))) & 3u);
}

// crossing_points (reference geometry.cpp:39-50) in one loop: crossing k is
// edge (k-th inside slot -> j-th outside slot), k = i_rank * (4 - m) + j
struct Crossings {
  Vd q[4];
};

__device__ __forceinline__ void crossings4(const Vd v[4], int mask, Vd c, double r, Crossings& X) {
  const int m = __popc(mask), mo = 4 - m, n = m * mo;
  const unsigned inm = (unsigned)mask, outm = (unsigned)(~mask & 15);
#pragma unroll
  for (int k = 0; k < 4; ++k) X.q[k] = v[0];
#pragma unroll 1
  for (int k = 0; k < n; ++k) {
    const int ir = k / mo, orr = k - ir * mo;
    const int i = nth_bit4(inm, ir), o = nth_bit4(outm, orr);
    const Vd a = pick(v, i), b = pick(v, o);
    const double t = edge_crossing(a, b, c, r);
    const Vd p = vadd(a, vscale(t, vsub(b, a)));
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (k == j) X.q[j] = p;
  }
}

__device__ __forceinline__ int nth_slot(int mask, int n) { return nth_bit4((unsigned)mask, n); }

// detail::straddle_inner (reference ball_approx.cpp:195-255), from the item's
// crossings (shared with straddle_outer: both start from crossing_points)
__device__ __forceinline__ Straddle inner_straddle_x(const Vd v[4], int mask, const Crossings& X) {
  const int m = __popc(mask);
  const int s0 = nth_slot(mask, 0), s1 = nth_slot(mask, m > 1 ? 1 : 0),
            s2 = nth_slot(mask, m > 2 ? 2 : 0);
  const Vd i0 = pick(v, s0), i1 = pick(v, s1), i2 = pick(v, s2);
  Straddle s;
  if (m == 1) {  // tet (a, a->o0, a->o1, a->o2)
    s.A0 = i0; s.A1 = X.q[0]; s.A2 = X.q[1]; s.B0 = X.q[2]; s.B1 = X.q[2]; s.B2 = X.q[2];
    s.n = 1;
  } else if (m == 2) {  // warped prism {a, a->o0, a->o1} | {b, b->o0, b->o1}
    s.A0 = i0; s.A1 = X.q[0]; s.A2 = X.q[1]; s.B0 = i1; s.B1 = X.q[2]; s.B2 = X.q[3];
    s.n = 3;
    orient_warped(s);
  } else {  // frustum {a, b, d} | {a->o, b->o, d->o}
    s.A0 = i0; s.A1 = i1; s.A2 = i2; s.B0 = X.q[0]; s.B1 = X.q[1]; s.B2 = X.q[2];
    s.n = 3;
  }
  return s;
}

// detail::straddle_outer (reference ball_approx.cpp:257-298)
__device__ __forceinline__ Straddle outer_straddle_x(const Vd v[4], int mask, const Crossings& X) {
  const int m = __popc(mask), om = ~mask & 15;
  const int t0 = nth_slot(om, 0), t1 = nth_slot(om, m < 3 ? 1 : 0), t2 = nth_slot(om, m < 2 ? 2 : 0);
  const Vd o0 = pick(v, t0), o1 = pick(v, t1), o2 = pick(v, t2);
  Straddle s;
  if (m == 1) {  // frustum {a->o0, a->o1, a->o2} | {o0, o1, o2}
    s.A0 = X.q[0]; s.A1 = X.q[1]; s.A2 = X.q[2]; s.B0 = o0; s.B1 = o1; s.B2 = o2;
    s.n = 3;
  } else if (m == 2) {  // warped prism {c, a->c, b->c} | {d, a->d, b->d}
    s.A0 = o0; s.A1 = X.q[0]; s.A2 = X.q[2]; s.B0 = o1; s.B1 = X.q[1]; s.B2 = X.q[3];
    s.n = 3;
    orient_warped(s);
  } else {  // corner tet (o, a->o, b->o, d->o)
    s.A0 = o0; s.A1 = X.q[0]; s.A2 = X.q[1]; s.B0 = X.q[2]; s.B1 = X.q[2]; s.B2 = X.q[2];
    s.n = 1;
  }
  return s;
}

__device__ __forceinline__ Straddle inner_straddle(const Vd v[4], int mask, Vd c, double r) {
  Crossings X;
  crossings4(v, mask, c, r, X);
  return inner_straddle_x(v, mask, X);
}

__device__ __forceinline__ Straddle outer_straddle(const Vd v[4], int mask, Vd c, double r) {
  Crossings X;
  crossings4(v, mask, c, r, X);
  return outer_straddle_x(v, mask, X);
}

// piece k (0..n-1) of the decomposition
__device__ __forceinline__ void straddle_piece(const Straddle& s, int k, Vd& a, Vd& b, Vd& c,
                                               Vd& d) {
  a = k == 0 ? s.A0 : (k == 1 ? s.A1 : s.A2);
  b = k == 0 ? s.A1 : (k == 1 ? s.A2 : s.B0);
  c = k == 0 ? s.A2 : (k == 1 ? s.B0 : s.B1);
  d = k == 0 ? s.B0 : (k == 1 ? s.B1 : s.B2);
}


// ---------------------------------------------------------------------------
// approxcaps: detail::straddle_inner with sphere_points (reference
// ball_approx.cpp:210-229): the inside vertices, the crossings, and for every
// crossing pair sharing an inside or an outside endpoint the radial projection
// of their midpoint onto the sphere (<= 10 points); their convex hull by the
// reference's incremental algorithm (geometry.cpp:198-298: seeds, eps tests,
// horizon order, face order), fanned from the centroid of the hull vertices
// (geometry.cpp:310-328).  `fn(a, b, c, d, vol)` is called for every fan piece
// above the volume floor (hull_pieces, ball_approx.cpp:177-192), in the
// reference's order.  A degenerate hull emits nothing (DegenerateHull is
// swallowed there).  Returns false if the face table overflowed (cannot happen
// for <= 10 points: a triangulated hull has <= 2V - 4 = 16 faces).
constexpr int kHullFaces = 32;   // faces after an insertion (a closed hull of <= 10 points has <= 16)
constexpr int kHullScratch = 48; // faces + new horizon faces during an insertion (<= 16 + 10)

template <class Fn>
__device__ __forceinline__ bool approx_pieces(const Vd v[4], int mask, Vd c, double r, double tau,
                                              Fn&& fn) {
  const int m = __popc(mask), mo = 4 - m, nq = m * mo;
  Crossings X;
  crossings4(v, mask, c, r, X);
  Vd pts[10];
  int n = 0;
  for (int i = 0; i < m; ++i) pts[n++] = pick(v, nth_bit4((unsigned)mask, i));
  for (int k = 0; k < nq; ++k) pts[n++] = X.q[k];
  // crossing k = (inside rank k / mo, outside rank k % mo)
  for (int i = 0; i < nq; ++i)
    for (int j = i + 1; j < nq; ++j) {
      if (i / mo != j / mo && i % mo != j % mo) continue;
      const Vd mid = vsub(vscale(0.5, vadd(X.q[i], X.q[j])), c);
      const double len = sqrt(vnorm2(mid));
      if (len <= 0) continue;
      pts[n++] = vadd(c, vscale(r / len, mid));
    }
  // hull3d: scale and eps
  Vd lo = pts[0], hi = pts[0];
  for (int i = 0; i < n; ++i) {
    lo = {fmin(lo.x, pts[i].x), fmin(lo.y, pts[i].y), fmin(lo.z, pts[i].z)};
    hi = {fmax(hi.x, pts[i].x), fmax(hi.y, pts[i].y), fmax(hi.z, pts[i].z)};
  }
  const double eps = 1e-12 * fmax(sqrt(vnorm2(vsub(hi, lo))), 1e-300);
  // affinely independent seed
  int s0 = 0, s1 = -1, s2 = -1, s3 = -1;
  for (int i = 1; i < n; ++i)
    if (vdist(pts[i], pts[s0]) > eps) {
      s1 = i;
      break;
    }
  if (s1 < 0) return true;
  const Vd d01 = vsub(pts[s1], pts[s0]);
  for (int i = 0; i < n; ++i)
    if (sqrt(vnorm2(vcross(d01, vsub(pts[i], pts[s0])))) / sqrt(vnorm2(d01)) > eps) {
      s2 = i;
      break;
    }
  if (s2 < 0) return true;
  const Vd nrm = vcross(d01, vsub(pts[s2], pts[s0]));
  for (int i = 0; i < n; ++i)
    if (fabs(vdot(nrm, vsub(pts[i], pts[s0]))) / sqrt(vnorm2(nrm)) > eps) {
      s3 = i;
      break;
    }
  if (s3 < 0) return true;
  if (vdot(nrm, vsub(pts[s3], pts[s0])) > 0) {
    const int t = s1;
    s1 = s2;
    s2 = t;
  }
  const Vd inner = vscale(0.25, vadd(vadd(vadd(pts[s0], pts[s1]), pts[s2]), pts[s3]));
  // faces packed one per word (a | b << 8 | c << 16): the table stays small
  // enough for L1 (the data-dependent indexing puts it in local memory)
  auto pack = [](int a, int b, int cc) { return (unsigned)a | ((unsigned)b << 8) | ((unsigned)cc << 16); };
  auto outward = [&](int a, int b, int cc) {
    const Vd nn = vcross(vsub(pts[b], pts[a]), vsub(pts[cc], pts[a]));
    return vdot(nn, vsub(inner, pts[a])) > 0 ? pack(a, cc, b) : pack(a, b, cc);
  };
  // faces [0, nf); horizon faces are built at [nf, nf + nh) and moved down
  unsigned F[kHullScratch];
  int nf = 4;
  F[0] = outward(s0, s2, s1);
  F[1] = outward(s0, s1, s3);
  F[2] = outward(s1, s2, s3);
  F[3] = outward(s0, s3, s2);
  unsigned used = (1u << s0) | (1u << s1) | (1u << s2) | (1u << s3);
  unsigned hv = used;  // vertices of the current faces
  for (int pi = 0; pi < n; ++pi) {
    if (used >> pi & 1) continue;
    used |= 1u << pi;
    const Vd p = pts[pi];
    // duplicate of a face corner (the reference tests every face's corners;
    // the distinct corners give the same answer)
    bool dup = false;
    for (int i = 0; i < n; ++i)
      if ((hv >> i & 1) && vdist(p, pts[i]) <= eps) dup = true;
    if (dup) continue;
    unsigned vis = 0;  // kHullFaces <= 32
    for (int f = 0; f < nf; ++f) {
      const int a = F[f] & 255, b = (F[f] >> 8) & 255, cc = F[f] >> 16;
      const Vd nn = vcross(vsub(pts[b], pts[a]), vsub(pts[cc], pts[a]));
      if (vdot(nn, vsub(p, pts[a])) > eps * sqrt(vnorm2(nn))) vis |= 1u << f;
    }
    if (!vis) continue;
    // horizon: directed edges of visible faces whose reverse lies in an
    // invisible face, in (face, edge) order -> new faces (a, b, pi).  The
    // directed edges of the invisible faces are marked in a 10 x 10 bit
    // matrix (bit 10 x + y for edge x -> y), so each test is one bit probe.
    unsigned long long em[2] = {0ull, 0ull};
    for (int g = 0; g < nf; ++g) {
      if (vis >> g & 1) continue;
      const int x = F[g] & 255, y = (F[g] >> 8) & 255, z = F[g] >> 16;
      const int k1 = 10 * x + y, k2 = 10 * y + z, k3 = 10 * z + x;
      em[k1 >> 6] |= 1ull << (k1 & 63);
      em[k2 >> 6] |= 1ull << (k2 & 63);
      em[k3 >> 6] |= 1ull << (k3 & 63);
    }
    int nh = 0;
    for (int f = 0; f < nf; ++f) {
      if (!(vis >> f & 1)) continue;
      const int e3[3] = {(int)(F[f] & 255), (int)((F[f] >> 8) & 255), (int)(F[f] >> 16)};
      for (int e = 0; e < 3; ++e) {
        const int a = e3[e], b = e3[e == 2 ? 0 : e + 1];
        const int kb = 10 * b + a;  // the reverse edge b -> a
        const bool open = !((em[kb >> 6] >> (kb & 63)) & 1ull);
        if (!open) {
          if (nf + nh >= kHullScratch) return false;
          F[nf + nh++] = outward(a, b, pi);
        }
      }
    }
    int k = 0;
    for (int f = 0; f < nf; ++f)
      if (!(vis >> f & 1)) F[k++] = F[f];
    if (k + nh > kHullFaces) return false;
    for (int h = 0; h < nh; ++h) F[k + h] = F[nf + h];
    nf = k + nh;
    hv = 0;
    for (int f = 0; f < nf; ++f) hv |= (1u << (F[f] & 255)) | (1u << ((F[f] >> 8) & 255)) | (1u << (F[f] >> 16));
  }
  // triangulate_polytope: centroid of the distinct hull vertices, summed in
  // ascending vertex order, times 1/count
  const unsigned vs = hv;
  Vd cen = {0.0, 0.0, 0.0};
  for (int i = 0; i < n; ++i)
    if (vs >> i & 1) cen = vadd(cen, pts[i]);
  cen = vscale(1.0 / (double)__popc(vs), cen);
  for (int f = 0; f < nf; ++f) {
    const Vd a = pts[F[f] & 255], b = pts[(F[f] >> 8) & 255], cc = pts[F[f] >> 16];
    const double vol = tet_volume(cen, a, b, cc);
    if (vol > tau) fn(cen, a, b, cc, vol);
  }
  return true;
}
